"""The gradient kernels divide by the launch-constant h as RN(1/h) times r with
two FMA residual corrections (common.cuh div_by, Markstein's correctly rounded
step) instead of __ddiv_rn. Same binary64 operations on the host: the result must
equal IEEE r/h bit for bit over random, all-ones-significand, binade-edge and
near-midpoint cases (tests/csrc/div_by_check.c)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_div_by_matches_ieee_division(tmp_path):
    exe = tmp_path / "div_by_check"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(HERE, "csrc", "div_by_check.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "4000000", "3"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout
