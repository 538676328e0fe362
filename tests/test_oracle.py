"""Pin the CPU checker before trusting it (CPU-only).

The plain-C restatement (oracle/sphx_oracle.c) must reproduce, bit for bit, the
golden vectors generated from the reference itself (tests/golden/), and -- where
the compiled reference (oracle/_ref) is present -- the reference's own outputs.
"""
import os

import numpy as np
import pytest

import oracle as O
from golden_cases import PREC_NAMES, load_cases, load_configs

PREC = {"fp64": O.FP64, "fp32": O.FP32, "fp16": O.FP16}


@pytest.fixture(scope="module")
def orc():
    return O.Oracle()


def _regen_positions(orc, c):
    m = c.meta
    if m["kind"] == "random":
        xs, _ = orc.random(m["dim"], m["n"], m["seed"], m["lo"], m["hi"])
        return xs
    if m["kind"] == "lattice":
        return orc.lattice(m["dim"], m["ds"], m["jitter"], m["seed"], m["lo"], m["hi"])
    return c.x


# ---- binary16 (test_binary16.cpp:13-61) --------------------------------------------------
def test_known_encodings(orc):
    lib = orc.lib
    assert lib.so_f16_from_f64(1.0) == 0x3C00
    assert lib.so_f16_from_f64(2.0) == 0x4000
    assert lib.so_f16_from_f64(-1.0) == 0xBC00
    assert lib.so_f16_from_f64(0.0) == 0x0000
    assert lib.so_f16_from_f64(-0.0) == 0x8000
    assert lib.so_f16_from_f64(65504.0) == 0x7BFF
    assert lib.so_f16_from_f64(2.0 ** -24) == 0x0001
    assert lib.so_f16_from_f64(1023.0 * 2.0 ** -24) == 0x03FF
    assert lib.so_f16_to_f64(lib.so_f16_from_f64(2049.0)) == 2048.0
    assert lib.so_f16_to_f64(lib.so_f16_from_f64(2051.0)) == 2052.0
    assert lib.so_f16_from_f64(65520.0) == 0x7C00
    assert lib.so_f16_from_f64(np.nextafter(65520.0, 0.0)) == 0x7BFF
    assert lib.so_f16_from_f64(2.0 ** -25) == 0x0000
    assert lib.so_f16_from_f64(2.0 ** -25 * 1.0000001) == 0x0001
    assert lib.so_f16_from_f64(float("nan")) == 0x7E00
    assert lib.so_f16_from_f64(float("inf")) == 0x7C00


def test_exhaustive_round_trip(orc):
    lib = orc.lib
    finite = 0
    for b in range(0x10000):
        if (b & 0x7C00) == 0x7C00:
            continue
        finite += 1
        assert lib.so_f16_from_f64(lib.so_f16_to_f64(b)) == b
    assert finite == 65536 - 2048


def test_f16_agrees_with_numpy_on_random_doubles(orc):
    # numpy's float64->float16 cast is a single correctly rounded conversion
    rs = np.random.default_rng(3)
    vals = np.concatenate([rs.standard_normal(20000) * 10.0 ** rs.integers(-9, 5, 20000),
                           rs.uniform(-1, 1, 5000) * 2.0 ** -14])
    want = vals.astype(np.float16).view(np.uint16)
    got = np.array([orc.lib.so_f16_from_f64(float(v)) for v in vals], np.uint16)
    assert np.array_equal(got, want)


@pytest.mark.skipif(not os.path.exists(O.REF_SO), reason="reference not built")
def test_f16_agrees_with_reference(orc):
    ref = O.ref_lib()
    rs = np.random.default_rng(4)
    vals = rs.standard_normal(5000) * 10.0 ** rs.integers(-9, 5, 5000)
    for v in vals:
        assert orc.lib.so_f16_from_f64(float(v)) == ref.ref_f16_from_f64(float(v))


# ---- generators (test_model.cpp:12-56) --------------------------------------------------
def test_lattice_examples(orc):
    x = orc.lattice(2, 0.5, 0.0, 1)
    assert len(x[0]) == 4
    assert x[0][0] == 0.25 and x[1][0] == 0.25 and x[0][3] == 0.75 and x[1][3] == 0.75
    assert len(orc.lattice(2, 0.01, 0.0, 1)[0]) == 10000
    with pytest.raises(ValueError):
        orc.lattice(2, 1.5, 0.0, 1)
    with pytest.raises(ValueError):
        orc.lattice(2, 0.1, 0.5, 1)


def test_random_ds_rule(orc):
    assert orc.random(2, 10000, 7)[1] == pytest.approx(0.01)
    assert orc.random(3, 1000, 7)[1] == pytest.approx(0.1)


# ---- small cases against the reference-generated fixtures -------------------------------
@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c.name)
def test_oracle_matches_reference_fixture(orc, case):
    m = case.meta
    x = _regen_positions(orc, case)
    for a, b in zip(x, case.x):
        assert np.array_equal(a, b), "generator drifted from the reference"
    g = orc.grid(m["dim"], 2.0 * m["h"], m["lo"], m["hi"], m["periodic"])
    assert list(g.counts)[: m["dim"]] == m["grid"]["counts"][: m["dim"]]
    assert g.cutoff_norm == m["grid"]["cutoff_norm"]
    cell_of, start, items = orc.rebin(g, x)
    assert np.array_equal(items, case.items) and np.array_equal(start, case.start)
    assert np.array_equal(cell_of, case.cell_of)
    rel, cell, cell_of2, start2, items2 = orc.build_rel(g, x)
    for a in range(m["dim"]):
        assert np.array_equal(rel[a], case.rel[a]) and np.array_equal(cell[a], case.cell[a])
    assert np.array_equal(items2, case.items)
    for p in PREC_NAMES:
        t = orc.rcll(g, rel, cell, items, start, PREC[p])
        off, it = case.table("rcll", p)
        assert np.array_equal(t.offsets, off) and np.array_equal(t.items, it), f"rcll {p}"
        t = orc.cll(g, x, m["h"], cell_of, items, start, PREC[p])
        off, it = case.table("cll", p)
        assert np.array_equal(t.offsets, off) and np.array_equal(t.items, it), f"cll {p}"
        t = orc.all_list(x, m["h"], PREC[p])
        off, it = case.table("all", p)
        assert np.array_equal(t.offsets, off) and np.array_equal(t.items, it), f"all {p}"


def test_rebin_outside_grid_names_particle(orc):
    # test_grid.cpp:173-190
    x, _ = orc.random(2, 500, 31)
    g = orc.grid(2, 2.0 * 1.2 * (1.0 / 500) ** 0.5)
    x[0][17] = 2.5
    with pytest.raises(IndexError, match="17"):
        orc.rebin(g, x)


# ---- full configs against the golden hashes ---------------------------------------------
def _config(orc, name):
    c = load_configs()[name]
    x = orc.lattice(c["dim"], c["ds"], c["jitter"], c["seed"])
    h = 1.2 * c["ds"]
    g = orc.grid(c["dim"], 2.0 * h)
    rel, cell, cell_of, start, items = orc.build_rel(g, x)
    return c, x, h, g, rel, cell, cell_of, start, items


@pytest.mark.parametrize("prec", PREC_NAMES)
def test_oracle_c1_golden(orc, prec):
    c, x, h, g, rel, cell, cell_of, start, items = _config(orc, "C1")
    assert len(x[0]) == c["n"] and g.total == c["cells"]
    t = orc.rcll(g, rel, cell, items, start, PREC[prec])
    assert f"{t.hash():016x}" == c["tables"][f"rcll_{prec}"]["hash"]
    t = orc.cll(g, x, h, cell_of, items, start, PREC[prec])
    assert f"{t.hash():016x}" == c["tables"][f"cll_{prec}"]["hash"]


@pytest.mark.parametrize("be_prec", ["rcll_fp64", "rcll_fp32", "cll_fp32", "rcll_fp16"])
def test_oracle_c2_golden(orc, be_prec):
    c, x, h, g, rel, cell, cell_of, start, items = _config(orc, "C2")
    be, prec = be_prec.split("_")
    if be == "rcll":
        t = orc.rcll(g, rel, cell, items, start, PREC[prec])
    else:
        t = orc.cll(g, x, h, cell_of, items, start, PREC[prec])
    assert t.total == c["tables"][be_prec]["total"]
    assert f"{t.hash():016x}" == c["tables"][be_prec]["hash"]


@pytest.mark.parametrize("dim,ds,jitter", [(2, 0.02, 0.3), (3, 0.1, 0.3), (2, 0.05, 0.0)])
def test_oracle_grad_normalized_matches_reference(dim, ds, jitter):
    """The oracle's grad_normalized restatement == the reference's gradient.cpp on the
    reference's own FP16 RCLL table (the mixed step, dynamics.cpp:145-155)."""
    if not os.path.exists(O.REF_SO):
        pytest.skip("reference library not built")
    r = O.RefSystem.lattice(dim, ds, jitter, 1).make_grid()
    x = [r.x(k) for k in range(dim)]
    h = 1.2 * ds
    for f in (np.sin(3 * x[0]) + x[dim - 1] ** 2, 1.0 + 2.0 * x[0]):
        gr, dr = r.grad_normalized_rcll(2, f, h)
        t = r.rcll(2)
        go, do = O.Oracle().grad_normalized(dim, x, f, t.offsets, t.items, h)
        assert dr == do
        for a, b in zip(gr, go):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 1, 0)])
def test_oracle_update_relative_matches_reference(prec, periodic):
    """so_update_relative == the reference's update_relative, including where it
    throws (the particles before the throw updated, the rest untouched)."""
    if not os.path.exists(O.REF_SO):
        pytest.skip("reference library not built")
    ds = 0.02
    r = O.RefSystem.lattice(2, ds, 0.3, 1).make_grid(periodic=tuple(bool(p) for p in periodic))
    orc = O.Oracle()
    og = orc.grid(2, 2.4 * ds, periodic=periodic)
    rel, cell = [np.array(a) for a in r.rel_coords()[0]], [np.array(a) for a in r.rel_coords()[1]]
    rng = np.random.default_rng(11)
    dx = [rng.uniform(-0.45, 0.45, r.n) * og.edge[k] for k in range(2)]
    e_ref = r.update_relative(dx, prec)
    e_or = orc.update_relative(og, rel, cell, dx, prec)
    assert (e_ref == 0) == (e_or == 0)
    if e_ref:
        assert e_ref - 1 == (e_or - 1) >> 3
    rr, rc = r.rel_coords()
    for k in range(2):
        assert np.array_equal(rr[k], rel[k]) and np.array_equal(rc[k], cell[k])
