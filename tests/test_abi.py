"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/sphx_cuda.h declares, computes grid descriptors exactly like the
reference CellGrid, and fails loudly (no CPU fallback) without a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sphx_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sphx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2401_08586_b200 import capi
    L = capi.lib()
    names = _declared()
    assert len(names) >= 19
    for name in names:
        assert hasattr(L, name), f"{name} not exported"
    assert set(capi.EXPORTED) <= set(names)


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2401_08586_b200", "lib", "libsphx_cuda.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_grid_init_matches_reference_cellgrid():
    import oracle as O
    from paper_2401_08586_b200 import capi
    if not os.path.exists(O.REF_SO):
        pytest.skip("reference not built")
    for dim, ds, per in [(2, 0.01, (0, 0, 0)), (3, 0.013, (1, 0, 1)), (1, 0.05, (1, 0, 0)),
                         (2, 0.0007, (0, 1, 0))]:
        r = O.RefSystem.lattice(dim, ds, 0.0, 1).make_grid(periodic=per, rebin=False, rel=False)
        want = r.grid_desc()
        g = capi.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.0 * r.h, per)
        assert list(g.counts)[:dim] == want["counts"][:dim]
        assert g.cutoff_norm == want["cutoff_norm"] and g.radius_phys == want["radius"]
        for k in range(dim):
            assert g.hc[k] == want["hc"][k] and g.origin[k] == want["origin"][k]


def test_grid_init_errors():
    from paper_2401_08586_b200 import capi
    with pytest.raises(ValueError, match="periodic axis needs at least 3 cells"):
        capi.grid_init(2, (0, 0, 0), (1, 1, 1), 0.4, (1, 0, 0))
    with pytest.raises(ValueError, match="search radius must be positive"):
        capi.grid_init(2, (0, 0, 0), (1, 1, 1), 0.0)
    with pytest.raises(ValueError, match="lo < hi"):
        capi.grid_init(2, (0, 0, 0), (1, 0, 1), 0.1)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2401_08586_b200 import capi
    with pytest.raises(capi.SphxCudaError):
        capi.Context(0)


@pytest.mark.parametrize("dim,ds,jit,seed", [(2, 0.01, 0.3, 1), (3, 0.05, 0.2, 7), (1, 0.1, 0.0, 3)])
def test_generators_match_reference(dim, ds, jit, seed):
    import oracle as O
    import paper_2401_08586_b200 as P
    want = O.Oracle().lattice(dim, ds, jit, seed)
    got = P.build_lattice(dim, ds, jit, seed)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    want, wds = O.Oracle().random(dim, 777, seed)
    got, gds = P.build_random_uniform(dim, 777, seed)
    assert gds == wds
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
