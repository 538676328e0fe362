"""Device RCLL maintenance: RelCoords stay resident on the
device across steps -- update_relative (cell_grid.cpp:180-212) for every particle,
rebuild_members (cell_grid.cpp:86-108), FP16 RCLL -- exactly as step_mixed does
(dynamics.cpp:191-198, FP64 maintenance). Every step's rel, cell, CSR and table
must equal the oracle's."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _rebuild_members(cell, counts):
    """CellGrid::build_csr from per-axis cells (stable counting sort by id)."""
    dim = len(cell)
    lin = np.zeros(len(cell[0]), np.int64)
    for k in reversed(range(dim)):
        lin = lin * counts[k] + cell[k]
    items = np.argsort(lin, kind="stable").astype(np.int32)
    total = int(np.prod(counts[:dim]))
    start = np.zeros(total + 1, np.int32)
    start[1:] = np.cumsum(np.bincount(lin, minlength=total))
    return lin.astype(np.int32), start, items


@pytest.mark.parametrize("dim", [2, 3])
def test_resident_rcll_steps(ctx, dim):
    import torch

    import paper_2401_08586_b200 as P
    ds = 0.02 if dim == 2 else 0.05
    per = (1, 1, 1 if dim == 3 else 0)
    orc = O.Oracle()
    x = orc.lattice(dim, ds, 0.3, 1)
    og = orc.grid(dim, 2.4 * ds, periodic=per)
    rel, cell, _, start, items = orc.build_rel(og, x)
    g = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.4 * ds, per)
    counts = list(g.counts)
    dev = torch.device("cuda", 0)
    drel = [torch.from_numpy(a.copy()).to(dev) for a in rel]
    dcell = [torch.from_numpy(a.copy()).to(dev) for a in cell]
    n = len(x[0])
    cell_of = torch.empty(n, dtype=torch.int32, device=dev)
    dstart = torch.empty(g.cell_total + 1, dtype=torch.int32, device=dev)
    ditems = torch.empty(n, dtype=torch.int32, device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.empty(n * 80, dtype=torch.int32, device=dev)
    rng = np.random.default_rng(3)
    for step in range(4):
        dx = [rng.uniform(-0.4, 0.4, n) * og.edge[k] for k in range(dim)]
        assert orc.update_relative(og, rel, cell, dx, 0) == 0
        ctx.update_relative_device(g, drel, dcell, [torch.from_numpy(a).to(dev) for a in dx], 0,
                                   status)
        ctx.rebuild_members_device(g, dcell, cell_of, dstart, ditems)
        ctx.rcll_device(g, drel, dcell, ditems, dstart, 2, offsets, out)
        torch.cuda.synchronize()
        assert int(status.item()) == -1, "no particle may throw"
        for k in range(dim):
            assert np.array_equal(drel[k].cpu().numpy(), rel[k]), f"step {step}: rel {k}"
            assert np.array_equal(dcell[k].cpu().numpy(), cell[k]), f"step {step}: cell {k}"
        _, start, items = _rebuild_members(cell, counts)
        assert np.array_equal(dstart.cpu().numpy(), start)
        assert np.array_equal(ditems.cpu().numpy(), items)
        want = orc.rcll(og, rel, cell, items, start, 2)
        off = offsets.cpu().numpy()
        assert np.array_equal(off, want.offsets), f"step {step}: offsets"
        assert np.array_equal(out[:off[-1]].cpu().numpy(), want.items), f"step {step}: items"


def test_update_relative_errors(ctx):
    import paper_2401_08586_b200 as P
    ds = 0.05
    orc = O.Oracle()
    x = orc.lattice(2, ds, 0.0, 1)
    og = orc.grid(2, 2.4 * ds)
    rel, cell, _, _, _ = orc.build_rel(og, x)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    n = len(x[0])
    dx = [np.zeros(n), np.zeros(n)]
    dx[1][7] = 1.5 * og.edge[1]
    with pytest.raises(RuntimeError, match="displacement skips a cell on axis 1"):
        ctx.update_relative(g, [a.copy() for a in rel], [a.copy() for a in cell], dx, 0)
    dx = [np.zeros(n), np.zeros(n)]
    dx[0][0] = -0.9 * og.edge[0]  # particle 0 sits in cell 0 near the wall
    with pytest.raises(RuntimeError, match="particle leaves the grid on axis 0"):
        ctx.update_relative(g, [a.copy() for a in rel], [a.copy() for a in cell], dx, 0)
