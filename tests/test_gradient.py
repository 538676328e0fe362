"""Fused FP16 RCLL -> grad_normalized against the oracle.

The reference's mixed step computes grad_normalized(f, ps, rcll(rel, grid, fp16),
make_kernel(h, dim)) (dynamics.cpp:145-155, gradient.cpp:44-82). The fused kernel
never writes the table; its FP64 gradient and degenerate count must be bit-identical
to the oracle's restatement applied to the oracle's FP16 RCLL table
(tests/test_oracle.py pins that restatement to the reference's gradient.cpp).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _fields(x):
    dim = len(x)
    f_smooth = np.sin(7.0 * x[0]) * np.cos(5.0 * x[dim - 1]) + x[0] ** 2
    f_linear = 0.5 + 2.0 * x[0]  # exact along x for any neighbour arrangement
    return {"smooth": f_smooth, "linear": f_linear}


def _check(ctx, x, radius, h, lo=(0, 0, 0), hi=(1, 1, 1), periodic=(0, 0, 0)):
    import paper_2401_08586_b200 as P
    dim = len(x)
    orc = O.Oracle()
    og = orc.grid(dim, radius, lo, hi, periodic)
    rel, cell, _, start, items = orc.build_rel(og, x)
    table = orc.rcll(og, rel, cell, items, start, 2)
    g = P.grid_init(dim, lo, hi, radius, periodic)
    out = {}
    for name, f in _fields(x).items():
        want, wdeg = orc.grad_normalized(dim, x, f, table.offsets, table.items, h)
        got, gdeg = ctx.rcll_grad_normalized(g, rel, cell, items, start, 2, x, f, h)
        for k in range(dim):
            assert np.array_equal(got[k], want[k]), f"{name}: axis {k} differs"
        assert gdeg == wdeg
        out[name] = got
    return out, table


def test_gradient_2d_lattice(ctx):
    ds = 0.01
    x = O.Oracle().lattice(2, ds, 0.3, 1)
    out, _ = _check(ctx, x, 2.4 * ds, 1.2 * ds)
    # exact on linear fields (gradient.hpp:24-25) away from degenerate rows
    gx = out["linear"][0]
    assert np.max(np.abs(gx[gx != 0.0] - 2.0)) < 1e-9


def test_gradient_3d_lattice(ctx):
    ds = 0.05
    x = O.Oracle().lattice(3, ds, 0.3, 1)
    _check(ctx, x, 2.4 * ds, 1.2 * ds)


def test_gradient_dam_break_column(ctx):
    ds = 0.04
    x = O.Oracle().lattice(3, ds, 0.3, 1, (0, 0, 0), (0.5, 1.0, 0.5))
    _check(ctx, x, 2.4 * ds, 1.2 * ds)


def test_gradient_periodic(ctx):
    ds = 0.02
    x = O.Oracle().lattice(2, ds, 0.25, 3)
    _check(ctx, x, 2.4 * ds, 1.2 * ds, periodic=(1, 1, 0))


def test_gradient_long_rows(ctx):
    """kh = 4 ds: ~50 neighbours per row, beyond the 24-slot row buffer, so rows
    are walked in id order by minimum search."""
    ds = 0.02
    x = O.Oracle().lattice(2, ds, 0.3, 2)
    _, table = _check(ctx, x, 4.0 * ds, 2.0 * ds)
    assert np.diff(table.offsets).max() > 24


def test_gradient_rejects_non_fp16(ctx):
    import paper_2401_08586_b200 as P
    x = O.Oracle().lattice(2, 0.1, 0.0, 1)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 0.24)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    with pytest.raises(ValueError):
        ctx.rcll_grad_normalized(g, rel, cell, items, start, 0, x, x[0], 0.12)


@pytest.mark.parametrize("order", ["shuffled", "reversed"])
def test_gradient_2d_particle_orders(ctx, order):
    """Incoherent id orders: the windowed gradient's tiles without a window."""
    x = O.Oracle().lattice(2, 0.01, 0.3, 4)
    rs = np.random.default_rng(11)
    perm = rs.permutation(len(x[0])) if order == "shuffled" else np.arange(len(x[0]))[::-1]
    x = [np.ascontiguousarray(a[perm]) for a in x]
    _check(ctx, x, 0.024, 0.012)


def test_gradient_2d_dense_cluster(ctx):
    """A dense blob: segments beyond 32 records and tiles whose rows do not fit the
    shared-memory row buffer (the selection walk)."""
    rs = np.random.default_rng(6)
    x = np.concatenate([0.45 + 0.012 * rs.standard_normal((2, 2500)), rs.random((2, 500))], axis=1)
    x = [np.ascontiguousarray(a) for a in np.clip(x, 0.0, 1.0 - 1e-12)]
    _check(ctx, x, 0.048, 0.024)


def test_gradient_2d_matches_encode_path(ctx):
    """The windowed fused gradient equals the encode + k_r16_grad one (SPHX_W2=0)."""
    import os

    import paper_2401_08586_b200 as P
    x = O.Oracle().lattice(2, 1.0 / 317, 0.3, 8)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 / 317)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    f = np.sin(9.0 * x[0]) + x[1]
    a = ctx.rcll_grad_normalized(g, rel, cell, items, start, 2, x, f, 1.2 / 317)
    os.environ["SPHX_W2"] = "0"
    try:
        b = ctx.rcll_grad_normalized(g, rel, cell, items, start, 2, x, f, 1.2 / 317)
    finally:
        del os.environ["SPHX_W2"]
    assert all(np.array_equal(a[0][k], b[0][k]) for k in range(2)) and a[1] == b[1]
