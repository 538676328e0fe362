"""Dense clusters: the capacity fallbacks of the encode and sweep kernels.

The small cases hold at most a few dozen particles per cell, so every encode CTA
stages its member window and its chunk range in shared memory and every sweep
tile fits its packed rows. Clustered SPH states (a splash, a collapsing column)
break those assumptions. Here a Gaussian blob puts hundreds to thousands of
particles in a cell, so that, at every precision and for both cell-based
backends:
- encode windows exceed shared memory (2-D WCAP 768 members, 3-D 1,024; xy
  encode 1,024) and so do chunk ranges (2-D OCAP 384, 3-D 512, xy 640), which
  takes the global-memory paths of k_encode_rows / k_encode_xy;
- rows exceed the kept hit words (2-D 4 words, 3-D 16), which takes the re-test
  path, and tiles exceed their packed-row capacity, which takes the direct
  global-memory row build.
Tables must equal the C oracle's (pinned to the reference in test_oracle.py) bit
for bit.
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


def _blob(dim, n_blob, sigma, n_back, seed, centre=0.45):
    rs = np.random.default_rng(seed)
    blob = centre + sigma * rs.standard_normal((dim, n_blob))
    back = rs.random((dim, n_back))
    x = np.clip(np.concatenate([blob, back], axis=1), 0.0, 1.0 - 1e-12)
    return [np.ascontiguousarray(a) for a in x]


CASES = [
    # dim, n_blob, sigma, n_back, ds
    (2, 3000, 0.012, 600, 0.02),
    (3, 3000, 0.03, 400, 0.05),
]


@pytest.mark.parametrize("prec", ["fp16", "fp32", "fp64"])
@pytest.mark.parametrize("dim,n_blob,sigma,n_back,ds", CASES)
def test_dense_cluster_tables(ctx, dim, n_blob, sigma, n_back, ds, prec):
    import paper_2401_08586_b200 as P
    x = _blob(dim, n_blob, sigma, n_back, seed=11 + dim)
    h = 1.2 * ds
    orc = O.Oracle()
    og = orc.grid(dim, 2.0 * h)
    orel, ocell, ocell_of, ostart, oitems = orc.build_rel(og, x)
    counts = np.diff(ostart)
    assert counts.max() > 300, "the blob must overfill cells"
    p = PREC[prec]
    g = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.0 * h)
    rel, cell, cell_of, start, items = ctx.build_rel_coords(g, x)
    assert np.array_equal(start, ostart) and np.array_equal(items, oitems)
    want = orc.rcll(og, orel, ocell, oitems, ostart, p)
    off, it = ctx.rcll(g, rel, cell, items, start, p)
    assert np.array_equal(off, want.offsets), "rcll offsets"
    assert np.array_equal(it, want.items), "rcll items"
    assert np.diff(off).max() > 1000, "rows must overflow the kept hit words"
    want = orc.cll(og, x, h, ocell_of, oitems, ostart, p)
    off, it = ctx.cell_link_list(g, x, h, items, start, cell_of, p)
    assert np.array_equal(off, want.offsets), "cll offsets"
    assert np.array_equal(it, want.items), "cll items"
