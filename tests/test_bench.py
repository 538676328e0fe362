"""bench.py's host-side pieces, on CPU: the reference arm's JSON contract, the
renumbering used by the locality study's parity, and the lattice closed form
used for C5's sampled-row parity."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, NCCL_DEBUG="VERSION")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def _brute_renumber(off, it, perm):
    n = len(perm)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rows = [sorted(int(inv[j]) for j in it[off[p]:off[p + 1]]) for p in perm]
    new_off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return new_off, np.array([j for r in rows for j in r], np.int32)


def test_renumber_table_matches_brute_force():
    rng = np.random.default_rng(4)
    n = 300
    lens = rng.integers(0, 9, n)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    it = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int32)
    for perm in (rng.permutation(n), np.arange(n)[::-1].copy(), np.arange(n)):
        got = bench.renumber_table(off, it, perm)
        want = _brute_renumber(off, it, perm)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_lattice_offsets_closed_form():
    # the 56 lattice sites within 2.4 ds of a site (interior C5 rows)
    assert len(bench.LATTICE_OFFSETS) == 56
    assert all(0 < a * a + b * b + c * c < 5.76 for a, b, c in bench.LATTICE_OFFSETS)


def test_workloads_name_the_baseline_configs():
    assert {"C1", "C2", "C3", "C4", "C5"} <= set(bench.WORKLOADS)
    assert bench.WORKLOADS["C2"]["dim"] == 2 and bench.WORKLOADS["C2"]["ds"] == 0.001
    assert bench.WORKLOADS["C5"]["jitter"] == 0.0
