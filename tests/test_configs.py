"""The large BASELINE configurations at test scale, full tables against the oracle.

C4 (dam-break column: a jittered lattice filling [0,.5]x[0,1]x[0,.5] of the unit
cube, 75 % of the cells empty -- SURVEY 8(d)) and C5 (un-jittered 3-D lattice,
SURVEY 8(d)) are benchmarked at 16M / 262M particles with sampled-row parity
(bench.py); here the same constructions at a size the oracle finishes in seconds
are compared table for table, at every precision, through the C ABI.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

PREC = {"fp64": 0, "fp32": 1, "fp16": 2}


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _check(ctx, x, ds, prec):
    import paper_2401_08586_b200 as P
    orc = O.Oracle()
    og = orc.grid(3, 2.4 * ds)
    orel, ocell, _, ostart, oitems = orc.build_rel(og, x)
    want = orc.rcll(og, orel, ocell, oitems, ostart, prec)
    g = P.grid_init(3, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    assert np.array_equal(start, ostart) and np.array_equal(items, oitems)
    off, it = ctx.rcll(g, rel, cell, items, start, prec)
    assert np.array_equal(off, want.offsets), "offsets differ"
    assert np.array_equal(it, want.items), "items differ"
    return off, it


@pytest.mark.parametrize("prec", ["fp64", "fp32", "fp16"])
def test_dam_break_column(ctx, prec):
    ds = 0.02  # 25 x 50 x 25 = 31,250 particles in a 21^3-cell unit-cube grid
    x = O.Oracle().lattice(3, ds, 0.3, 1, (0, 0, 0), (0.5, 1.0, 0.5))
    assert len(x[0]) == 25 * 50 * 25
    off, it = _check(ctx, x, ds, PREC[prec])
    assert it.size > 0


def test_unjittered_lattice_closed_form(ctx):
    side = 40
    ds = 1.0 / side
    x = O.Oracle().lattice(3, ds, 0.0, 1)
    off, it = _check(ctx, x, ds, PREC["fp16"])
    offs = [(a, b, c) for a in range(-2, 3) for b in range(-2, 3) for c in range(-2, 3)
            if 0 < a * a + b * b + c * c < 5.76]
    assert len(offs) == 56
    total = sum(int(np.prod([side - abs(v) for v in vv])) for vv in offs)
    assert off[-1] == total
    rows = np.diff(off)
    interior = [(a + side * (b + side * c)) for a in (5, 20) for b in (5, 33) for c in (9, 30)]
    assert all(rows[i] == 56 for i in interior)
