"""The windowed 2-D FP16 RCLL path (csrc/cuda/window.cu, the default; SPHX_W2=0
selects the encode + k_rcll16 path).

Every table bit-identical to the reference's: the small 2-D cases (periodic
seams, ties, random, empty), C1/C2 against the reference's golden hashes, the
dense clusters that overflow the window and the 32-position segments (the exact
per-row path), a stale grid (RelCoords cells that disagree with the CSR
membership), a shuffled particle order (no compact bands), periodic domains
(windows that would wrap x) and tiles that straddle the end of a lattice row
(two bands).
"""
import os

import numpy as np
import pytest

import oracle as O
from golden_cases import load_cases, load_configs

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["128", "256"], ids=["bt128", "bt256"])
def windowed(request):
    """Both tile sizes (SPHX_W2BT) of the windowed path."""
    old = {k: os.environ.get(k) for k in ("SPHX_W2", "SPHX_W2BT")}
    os.environ["SPHX_W2"] = "1"
    os.environ["SPHX_W2BT"] = request.param
    yield
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _grid(P, meta):
    return P.grid_init(meta["dim"], meta["lo"], meta["hi"], 2.0 * meta["h"], meta["periodic"])


@pytest.mark.parametrize("case", [c for c in load_cases() if c.dim == 2], ids=lambda c: c.name)
def test_small_cases(ctx, case):
    import paper_2401_08586_b200 as P
    g = _grid(P, case.meta)
    off, it = ctx.rcll(g, case.rel, case.cell, case.items, case.start, 2)
    woff, wit = case.table("rcll", "fp16")
    assert np.array_equal(off, woff) and np.array_equal(it, wit)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_golden_hash(ctx, name):
    import paper_2401_08586_b200 as P
    c = load_configs()[name]
    x = O.Oracle().lattice(c["dim"], c["ds"], c["jitter"], c["seed"])
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * c["ds"])
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    t = ctx.rcll(g, rel, cell, items, start, 2)
    want = c["tables"]["rcll_fp16"]
    assert int(t[0][-1]) == want["total"]
    assert f"{O.fnv_hash(*t):016x}" == want["hash"]


def _blob(n_blob, sigma, n_back, seed):
    rs = np.random.default_rng(seed)
    x = np.concatenate([0.45 + sigma * rs.standard_normal((2, n_blob)), rs.random((2, n_back))], axis=1)
    return [np.ascontiguousarray(a) for a in np.clip(x, 0.0, 1.0 - 1e-12)]


@pytest.mark.parametrize("n_blob,sigma,ds", [(3000, 0.012, 0.02), (1500, 0.05, 0.01), (400, 0.004, 0.05)])
def test_dense_clusters(ctx, n_blob, sigma, ds):
    import paper_2401_08586_b200 as P
    x = _blob(n_blob, sigma, 600, 5)
    orc = O.Oracle()
    og = orc.grid(2, 2.4 * ds)
    orel, ocell, _, ostart, oitems = orc.build_rel(og, x)
    want = orc.rcll(og, orel, ocell, oitems, ostart, O.FP16)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    off, it = ctx.rcll(g, rel, cell, items, start, 2)
    assert np.array_equal(off, want.offsets) and np.array_equal(it, want.items)


def test_stale_grid(ctx):
    """RelCoords moved on (update_relative) while the CSR still holds the old
    membership: rows follow RelCoords::cell, candidates the CSR (nnps.cpp:349-372)."""
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    x = orc.lattice(2, 0.02, 0.3, 3)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 0.048)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    rs = np.random.default_rng(9)
    moved = rs.choice(len(rel[0]), 40, replace=False)
    cell = [c.copy() for c in cell]
    for i in moved:  # to a neighbouring cell inside the grid, rel kept
        cell[0][i] = min(max(cell[0][i] + rs.integers(-1, 2), 0), g.counts[0] - 1)
        cell[1][i] = min(max(cell[1][i] + rs.integers(-1, 2), 0), g.counts[1] - 1)
    og = orc.grid(2, 0.048)
    want = orc.rcll(og, rel, cell, items, start, O.FP16)
    off, it = ctx.rcll(g, rel, cell, items, start, 2)
    assert np.array_equal(off, want.offsets) and np.array_equal(it, want.items)


def _table(ctx, P, g, x):
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    return ctx.rcll(g, rel, cell, items, start, 2), (rel, cell, items, start)


@pytest.mark.parametrize("order", ["shuffled", "reversed", "blocks"])
def test_particle_orders(ctx, order):
    """Renumbered lattices: rows in any id order, same table up to the renumbering."""
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    x = orc.lattice(2, 0.004, 0.3, 2)  # 250 x 250
    n = len(x[0])
    rs = np.random.default_rng(4)
    if order == "shuffled":
        perm = rs.permutation(n)
    elif order == "reversed":
        perm = np.arange(n)[::-1].copy()
    else:  # blocks of 37 consecutive ids in random block order
        nb = (n + 36) // 37
        perm = np.concatenate([np.arange(b * 37, min(n, b * 37 + 37)) for b in rs.permutation(nb)])
    xp = [np.ascontiguousarray(a[perm]) for a in x]
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * 0.004)
    (off, it), (rel, cell, items, start) = _table(ctx, P, g, xp)
    og = orc.grid(2, 2.4 * 0.004)
    want = orc.rcll(og, rel, cell, items, start, O.FP16)
    assert np.array_equal(off, want.offsets) and np.array_equal(it, want.items)


@pytest.mark.parametrize("periodic", [(1, 0, 0), (0, 1, 0), (1, 1, 0)])
@pytest.mark.parametrize("nside", [60, 253])
def test_periodic_lattices(ctx, periodic, nside):
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    ds = 1.0 / nside
    x = orc.lattice(2, ds, 0.3, 7)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * ds, periodic)
    (off, it), (rel, cell, items, start) = _table(ctx, P, g, x)
    og = orc.grid(2, 2.4 * ds, periodic=periodic)
    want = orc.rcll(og, rel, cell, items, start, O.FP16)
    assert np.array_equal(off, want.offsets) and np.array_equal(it, want.items)


def test_matches_encode_path(ctx):
    """C2-sized lattice with lattice rows of 999 particles (tiles straddle row ends
    at every phase): the windowed table equals the encode + k_rcll16 table."""
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    x = orc.lattice(2, 1.0 / 999, 0.3, 5)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 / 999)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    a = ctx.rcll(g, rel, cell, items, start, 2)
    os.environ["SPHX_W2"] = "0"
    b = ctx.rcll(g, rel, cell, items, start, 2)
    os.environ["SPHX_W2"] = "1"
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("nx_cells", [2048, 2200])
def test_wide_grids(ctx, nx_cells):
    """A strip domain at and past the windowed path's 2048-cell row limit (past it
    the rows go to the encode path): the table equals the oracle's either way."""
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    ds = 0.002
    radius = 2.4 * ds
    hi = (nx_cells * radius - 1e-9, 12 * ds, 1.0)
    x = orc.lattice(2, ds, 0.3, 11, (0, 0, 0), hi)
    g = P.grid_init(2, (0, 0, 0), hi, radius)
    assert g.counts[0] == nx_cells
    (off, it), (rel, cell, items, start) = _table(ctx, P, g, x)
    og = orc.grid(2, radius, (0, 0, 0), hi)
    want = orc.rcll(og, rel, cell, items, start, O.FP16)
    assert np.array_equal(off, want.offsets) and np.array_equal(it, want.items)
