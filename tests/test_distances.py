"""Per-pair distances of RCLL tables (sphx_table_distances / sphx_rcll_distances_device).

north_star: per-pair distances must match the reference within a stated FP16/FP32
tolerance. The tolerance here is zero: for every entry (i, j) the device value
must equal the reference's rel_distance(rc, i, j, grid, prec) (cell_grid.cpp:
135-178; the oracle restates it and tests/test_oracle.py pins the oracle to the
reference) bit for bit -- with j's cell taken at its minimum image when the pair
wraps a periodic axis, as rcll's search does -- and every listed pair must be
closer than round_to(prec, cutoff), the test rcll applied.
"""
import numpy as np
import pytest

import oracle as O
from golden_cases import load_cases, load_configs

pytestmark = pytest.mark.gpu

PREC = {"fp64": 0, "fp32": 1, "fp16": 2}


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _min_image_cells(case, counts, i, j):
    """Cell arrays in which j's cell is replaced by its minimum image seen from i
    (what rcll's dc = -off is on a wrapping axis, nnps.cpp:359-362), so that
    rel_distance's raw cell difference becomes the minimum-image one."""
    cell = [np.array(c, dtype=np.int32) for c in case.cell]
    for k in range(case.dim):
        dc = int(cell[k][i]) - int(cell[k][j])
        if dc > 1:
            cell[k][j] += counts[k]
        elif dc < -1:
            cell[k][j] -= counts[k]
    return cell


@pytest.mark.parametrize("prec", ["fp64", "fp32", "fp16"])
@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c.name)
def test_distances_equal_rel_distance(ctx, case, prec):
    import paper_2401_08586_b200 as P
    m = case.meta
    if case.n < 2:
        pytest.skip("no pairs")
    g = P.grid_init(case.dim, m["lo"], m["hi"], 2.0 * m["h"], m["periodic"])
    p = PREC[prec]
    off, it = ctx.rcll(g, case.rel, case.cell, case.items, case.start, p)
    dist = ctx.table_distances(g, p)
    assert dist.shape == it.shape
    orc = O.Oracle()
    og = orc.grid(case.dim, 2.0 * m["h"], m["lo"], m["hi"], m["periodic"])
    cutoff = orc.round_to(p, og.cutoff_norm)
    assert np.all(dist < cutoff), "a listed pair is not within the cutoff"
    counts = list(g.counts)
    for i in range(case.n):
        for e in range(off[i], off[i + 1]):
            j = int(it[e])
            wraps = any(abs(int(case.cell[k][i]) - int(case.cell[k][j])) > 1
                        for k in range(case.dim))
            cell = _min_image_cells(case, counts, i, j) if wraps else case.cell
            want = orc.rel_distance(og, case.rel, cell, i, j, p)
            assert dist[e] == want, f"pair ({i},{j}): {dist[e]!r} != {want!r}"


def test_distances_device_c1(ctx):
    """C1 (10K, FP16): the device entry point on device-resident inputs, every pair
    against the oracle."""
    import torch

    import paper_2401_08586_b200 as P
    cfg = load_configs()["C1"]
    orc = O.Oracle()
    x = orc.lattice(2, 0.01, 0.0, 1)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * 0.01)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    off, it = ctx.rcll(g, rel, cell, items, start, 2)
    assert len(it) == cfg["tables"]["rcll_fp16"]["total"]
    dev = torch.device("cuda", 0)
    rd = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in rel]
    cd = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in cell]
    od = torch.from_numpy(off).to(dev)
    idd = torch.from_numpy(it).to(dev)
    dist = torch.empty(len(it), dtype=torch.float64, device=dev)
    ctx.rcll_distances_device(g, rd, cd, 2, od, idd, dist)
    torch.cuda.synchronize()
    d = dist.cpu().numpy()
    og = orc.grid(2, 2.4 * 0.01)
    want = np.array([orc.rel_distance(og, rel, cell, i, int(it[e]), 2)
                     for i in range(len(off) - 1) for e in range(off[i], off[i + 1])])
    assert np.array_equal(d, want)
