"""The C++ drop-in API (`_core`, include/sphx/*.hpp) restating the reference's own
tests (test_model.cpp, test_grid.cpp, test_nnps.cpp, test_binary16.cpp).

CPU-only tests exercise the host pieces (generators, grid construction, the
scalar per-point helpers, binary16); tests marked gpu drive the neighbour
search and the device binning on the B200."""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2401_08586_b200 import _core as c

F64, F32, F16 = c.Precision.fp64, c.Precision.fp32, c.Precision.fp16


# ---- generators (test_model.cpp:12-63) --------------------------------------------------
def test_lattice_examples():
    ps = c.build_lattice(c.Domain.unit(2), 0.5, 0.0, 1)
    assert ps.size() == 4
    assert ps.x(0)[0] == 0.25 and ps.x(1)[0] == 0.25 and ps.x(0)[3] == 0.75 and ps.x(1)[3] == 0.75
    assert c.build_lattice(c.Domain.unit(2), 0.01, 0.0, 1).size() == 10000
    with pytest.raises(ValueError):
        c.build_lattice(c.Domain.unit(2), 1.5, 0.0, 1)
    with pytest.raises(ValueError):
        c.build_lattice(c.Domain.unit(2), 0.1, 0.5, 1)


def test_lattice_determinism_and_bounds():
    d = c.Domain.unit(2)
    a, b, cc = (c.build_lattice(d, 0.05, 0.25, s) for s in (42, 42, 43))
    for k in range(2):
        assert np.array_equal(a.x(k), b.x(k))
        assert 0.0 < a.x(k).min() and a.x(k).max() < 1.0
    assert not all(np.array_equal(a.x(k), cc.x(k)) for k in range(2))


def test_random_spacing_rule_and_mass():
    assert c.build_random_uniform(c.Domain.unit(2), 10000, 7).ds() == pytest.approx(0.01)
    assert c.build_random_uniform(c.Domain.unit(3), 1000000, 7).ds() == pytest.approx(0.01)
    ps = c.build_lattice(c.Domain.unit(2), 0.1, 0.0, 1, 1000.0)
    assert ps.h() == pytest.approx(0.12)
    assert ps.mass_total() == pytest.approx(1000.0 * 0.01 * 100)


def test_generators_match_reference_generators():
    orc = O.Oracle()
    for dim, ds, jit, seed in [(2, 0.02, 0.3, 3), (3, 0.1, 0.2, 9), (1, 0.01, 0.1, 2)]:
        ps = c.build_lattice(c.Domain.unit(dim), ds, jit, seed)
        for a, b in zip([ps.x(k) for k in range(dim)], orc.lattice(dim, ds, jit, seed)):
            assert np.array_equal(a, b)


def test_csv_round_trip(tmp_path):
    ps = c.build_lattice(c.Domain.unit(2), 0.26, 0.3, 5)
    path = str(tmp_path / "snap.csv")
    c.write_csv(ps, path)
    lines = open(path).read().splitlines()
    assert lines[0] == "id,x,y,vx,vy,rho,p"
    for i, line in enumerate(lines[1:]):
        f = line.split(",")
        assert int(f[0]) == i and float(f[1]) == ps.x(0)[i] and float(f[2]) == ps.x(1)[i]


# ---- binary16 (test_binary16.cpp) --------------------------------------------------------
def test_binary16_exhaustive_against_numpy():
    b = np.arange(0x10000, dtype=np.uint16)
    finite = (b & 0x7C00) != 0x7C00
    vals = b[finite].view(np.float16).astype(np.float64)
    assert np.array_equal(c.f16_bits(vals), b[finite])
    rs = np.random.default_rng(2)
    v = rs.standard_normal(200000) * 10.0 ** rs.integers(-9, 5, 200000)
    assert np.array_equal(c.f16_bits(v), v.astype(np.float16).view(np.uint16))
    assert c.f16_bits([65520.0])[0] == 0x7C00 and c.f16_bits([2.0 ** -25])[0] == 0


# ---- grid (test_grid.cpp) ------------------------------------------------------------------
def test_normalization_examples():
    assert c.normalize_domain([0.5, 0.5, 0.0], c.Domain.unit(2))[:2] == [0.0, 0.0]
    assert c.normalize_domain([1.0, 0.0, 0.0], c.Domain.unit(2))[:2] == [1.0, -1.0]
    rect = c.Domain.box(2, [0.0, 0.0, 0.0], [2.0, 1.0, 0.0])
    assert c.normalize_domain([2.0, 1.0, 0.0], rect)[:2] == [1.0, 0.5]
    box = c.Domain.box(3, [-0.3, 0.1, 2.0], [0.9, 4.0, 2.5])
    rs = np.random.default_rng(5)
    for _ in range(200):
        x = [rs.uniform(-0.3, 0.9), rs.uniform(0.1, 4.0), rs.uniform(2.0, 2.5)]
        back = c.denormalize_domain(c.normalize_domain(x, box), box)
        assert np.allclose(back, x, rtol=1e-14, atol=0)


def test_grid_constants_match_reference():
    if not os.path.exists(O.REF_SO):
        pytest.skip("reference not built")
    for dim, ds, per in [(2, 0.01, (0, 0, 0)), (3, 0.013, (1, 0, 1)), (2, 0.0007, (0, 1, 0))]:
        r = O.RefSystem.lattice(dim, ds, 0.0, 1).make_grid(periodic=per, rebin=False, rel=False)
        want = r.grid_desc()
        g = c.CellGrid(c.Domain.unit(dim), 2.0 * r.h, [bool(p) for p in per])
        assert [g.count(k) for k in range(dim)] == want["counts"][:dim]
        assert g.cutoff_norm() == want["cutoff_norm"]
        for k in range(dim):
            assert g.hc(k) == want["hc"][k] and g.origin_norm(k) == want["origin"][k]
            assert g.edge_phys(k) == want["edge"][k]


def test_locate_tie_break():
    ps = c.build_lattice(c.Domain.unit(2), 0.1, 0.0, 1)
    g = c.make_grid_for(ps)
    cell, rel = g.locate([g.center_norm(0, 1), g.center_norm(1, 2), 0.0])
    assert cell[:2] == [1, 2] and rel[:2] == [0.0, 0.0]
    cell, rel = g.locate([g.origin_norm(0) + 2.0 * g.hc(0), g.center_norm(1, 2), 0.0])
    assert cell[0] == 1 and rel[0] == 1.0


def test_locate_matches_reference_bitwise():
    if not os.path.exists(O.REF_SO):
        pytest.skip("reference not built")
    import ctypes as C
    r = O.RefSystem.random(2, 3000, 17).make_grid(rebin=False, rel=False)
    g = c.CellGrid(c.Domain.unit(2), 2.0 * r.h, [False, False, False])
    rs = np.random.default_rng(1)
    for _ in range(3000):
        xn = [float(rs.uniform(-1, 1)), float(rs.uniform(-1, 1)), 0.0]
        cell, rel = g.locate(xn)
        cw = (C.c_int32 * 3)()
        rw = (C.c_double * 3)()
        r.lib.ref_grid_locate(r.grid, (C.c_double * 3)(*xn), cw, rw)
        assert list(cw)[:2] == cell[:2] and list(rw)[:2] == rel[:2]


def _rc(rel, cell):
    rc = c.RelCoords()
    for k, (r, cc) in enumerate(zip(rel, cell)):
        rc.set_rel(k, np.asarray(r, np.float64))
        rc.set_cell(k, np.asarray(cc, np.int32))
    return rc


def test_rel_distance_adjacent_centres():
    g = c.make_grid_for(c.build_lattice(c.Domain.unit(2), 0.1, 0.0, 1))
    rc = _rc([[0.0, 0.0], [0.0, 0.0]], [[1, 2], [1, 1]])
    assert c.rel_distance(rc, 0, 1, g, F64) == pytest.approx(g.hc(0), rel=1e-15)
    assert c.rel_distance(rc, 0, 0, g, F64) == 0.0


def test_update_relative_migration_and_fp16_exact():
    g = c.make_grid_for(c.build_lattice(c.Domain.unit(1), 0.1, 0.0, 1))
    edge = g.edge_phys(0)
    rc = _rc([[0.9] * 10], [[1] * 10])
    c.update_relative(rc, 0, [0.15 * edge, 0.0, 0.0], g, F64)
    assert rc.rel(0)[0] == pytest.approx(-0.8, rel=1e-12) and rc.cell(0)[0] == 2
    before = rc.rel(0)[0]
    c.update_relative(rc, 0, [0.0, 0.0, 0.0], g, F64)
    assert rc.rel(0)[0] == before
    with pytest.raises(RuntimeError, match="skips a cell"):
        c.update_relative(rc, 0, [1.5 * edge, 0.0, 0.0], g, F64)
    rc = _rc([[c.round16(0.9)] * 10], [[3] * 10])
    c.update_relative(rc, 0, [0.2 * edge, 0.0, 0.0], g, F16)
    assert rc.rel(0)[0] == c.round16(c.round16(0.9) + c.round16(0.4)) - 2.0
    assert rc.cell(0)[0] == 4


def test_update_relative_random_walk_drift():
    ps = c.build_lattice(c.Domain.unit(2), 0.2, 0.0, 1)
    g = c.make_grid_for(ps)
    x = [ps.x(0).copy(), ps.x(1).copy()]
    rel, cell = [[], []], [[], []]
    for i in range(ps.size()):
        cl, r = g.locate(c.normalize_domain([x[0][i], x[1][i], 0.0], ps.domain()))
        for k in range(2):
            rel[k].append(r[k])
            cell[k].append(cl[k])
    rc = _rc(rel, cell)
    rs = np.random.default_rng(23)
    span = 0.2 * g.edge_phys(0)
    for _ in range(300):
        for i in range(ps.size()):
            dx = [0.0, 0.0, 0.0]
            for k in range(2):
                st = rs.uniform(-span, span)
                if not 0.02 < x[k][i] + st < 0.98:
                    st = -st
                dx[k] = st
                x[k][i] += st
            c.update_relative(rc, i, dx, g, F64)
    for i in range(ps.size()):
        rec = c.reconstruct_norm(rc, i, g)
        want = c.normalize_domain([x[0][i], x[1][i], 0.0], ps.domain())
        assert abs(rec[0] - want[0]) < 1e-10 and abs(rec[1] - want[1]) < 1e-10


def test_spatial_sort_permutation_examples():
    ps = c.ParticleSystem(c.Domain.unit(2), 0.3, 3, 1.0)
    ps.set_x(0, [0.1, 0.5, 0.9])
    ps.set_x(1, [0.5, 0.5, 0.5])
    assert list(c.spatial_sort_permutation(ps)) == [0, 1, 2]
    ps.set_x(0, [0.9, 0.5, 0.1])
    assert list(c.spatial_sort_permutation(ps)) == [2, 1, 0]


# ---- neighbour search on the B200 (test_nnps.cpp) ---------------------------------------
def brute_force(ps):
    x = np.stack([ps.x(k) for k in range(ps.dim())], axis=1)
    d = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    n = len(x)
    rows = [np.flatnonzero((d[i] < 2.0 * ps.h()) & (np.arange(n) != i)) for i in range(n)]
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return off, np.concatenate(rows).astype(np.int32) if rows else np.empty(0, np.int32)


def same(t, off, items):
    return np.array_equal(t.offsets(), off) and np.array_equal(t.items(), items)


@pytest.mark.gpu
def test_single_particle_and_collinear():
    ps = c.ParticleSystem(c.Domain.unit(2), 0.1, 1, 1.0)
    ps.set_x(0, [0.5])
    ps.set_x(1, [0.5])
    t = c.all_list(ps, F64)
    assert t.size() == 1 and len(t.row(0)) == 0
    ps = c.ParticleSystem(c.Domain.unit(1), 0.1, 3, 1.0)
    ps.set_x(0, [0.4, 0.5, 0.6])
    t = c.all_list(ps, F64)
    assert all(len(t.row(i)) == 2 for i in range(3))


@pytest.mark.gpu
def test_strict_cutoff():
    ps = c.ParticleSystem(c.Domain.unit(2), 0.1, 2, 1.0)
    cut = 2.0 * ps.h()
    ps.set_x(0, [0.3, 0.3 + cut * (1.0 + 1e-9)])
    ps.set_x(1, [0.5, 0.5])
    assert len(c.all_list(ps, F64).row(0)) == 0
    ps.set_x(0, [0.3, 0.3 + cut * (1.0 - 1e-9)])
    assert len(c.all_list(ps, F64).row(0)) == 1


@pytest.mark.gpu
def test_backend_equivalence_fp64():
    from tests_rng import Rng
    rng = Rng(101)
    for dim in (1, 2, 3):
        for _ in range(3):
            n = 50 + rng.below(400)
            ps = c.build_random_uniform(c.Domain.unit(dim), n, rng.next_u64())
            g = c.make_grid_for(ps)
            g.rebin(ps)
            rc = c.build_rel_coords(ps, g)
            off, items = brute_force(ps)
            assert same(c.all_list(ps, F64), off, items)
            assert same(c.cell_link_list(ps, g, F64), off, items)
            assert same(c.rcll(rc, g, F64), off, items)


@pytest.mark.gpu
def test_symmetry_no_self_all_precisions():
    ps = c.build_random_uniform(c.Domain.unit(2), 300, 7)
    for p in (F64, F32, F16):
        t = c.all_list(ps, p)
        for i in range(t.size()):
            row = t.row(i)
            assert i not in row
            for j in row:
                assert i in t.row(int(j))


@pytest.mark.gpu
def test_fp16_matches_scalar_binary16_and_cell_equals_all():
    from tests_rng import Rng
    rng = Rng(313)
    for rep in range(4):
        n = 200 + rng.below(600)
        seed = rng.next_u64()
        ps = (c.build_random_uniform(c.Domain.unit(2), n, seed) if rep % 2 == 0 else
              c.build_lattice(c.Domain.unit(2), 0.97 / math.sqrt(n), 0.3, seed))
        g = c.make_grid_for(ps)
        g.rebin(ps)
        batch = c.all_list(ps, F16)
        # scalar binary16: float16 ops round once (24 >= 2*11+2: innocuous)
        xs = ps.x(0).astype(np.float16)
        ys = ps.x(1).astype(np.float16)
        cut = np.float16(2.0 * ps.h())
        rows = []
        for i in range(ps.size()):
            dx = (xs[i] - xs).astype(np.float16)
            dy = (ys[i] - ys).astype(np.float16)
            acc = ((dx * dx).astype(np.float16) + (dy * dy).astype(np.float16)).astype(np.float16)
            r = np.sqrt(acc.astype(np.float32)).astype(np.float16)
            hit = r < cut
            hit[i] = False
            rows.append(np.flatnonzero(hit))
        off = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
        assert same(batch, off, np.concatenate(rows))
        assert c.tables_equal(c.cell_link_list(ps, g, F16), batch)


@pytest.mark.gpu
def test_rcll_fp16_equals_rel_distance_classification():
    ps = c.build_random_uniform(c.Domain.unit(2), 400, 99)
    g = c.make_grid_for(ps)
    g.rebin(ps)
    rc = c.build_rel_coords(ps, g)
    t = c.rcll(rc, g, F16)
    cutoff = c.round16(g.cutoff_norm())
    rc16 = c.RelCoords()
    for k in range(2):
        rc16.set_rel(k, [c.round16(v) for v in rc.rel(k)])
        rc16.set_cell(k, rc.cell(k))
    cx, cy = rc.cell(0), rc.cell(1)
    for i in range(ps.size()):
        listed = set(t.row(i).tolist())
        cand = np.flatnonzero((np.abs(cx - cx[i]) <= 1) & (np.abs(cy - cy[i]) <= 1))
        for j in cand:
            if j == i:
                continue
            assert (c.rel_distance(rc16, i, int(j), g, F16) < cutoff) == (int(j) in listed)


@pytest.mark.gpu
def test_permutation_equivariance():
    for p in (F64, F16):
        ps = c.build_random_uniform(c.Domain.unit(2), 500, 1234)
        before = c.all_list(ps, p)
        perm = c.spatial_sort_permutation(ps)
        c.apply_permutation(ps, perm)
        after = c.all_list(ps, p)
        assert c.tables_equal(after, c.remap_table(before, perm))


@pytest.mark.gpu
def test_mismatch_report_counting():
    ps = c.build_random_uniform(c.Domain.unit(2), 200, 55)
    t = c.all_list(ps, F64)
    rep = c.mismatch_report(t, t)
    assert rep.incorrect_count == 0 and rep.incorrect_percent == 0.0
    r16 = c.mismatch_report(c.all_list(ps, F16), t)
    assert r16.incorrect_count % 2 == 0


@pytest.mark.gpu
def test_periodic_seam():
    ps = c.ParticleSystem(c.Domain.unit(2), 0.05, 2, 1.0)
    ps.set_x(0, [0.01, 0.99])
    ps.set_x(1, [0.5, 0.5])
    g = c.CellGrid(c.Domain.unit(2), 2.0 * ps.h(), [True, False, False])
    g.rebin(ps)
    t = c.cell_link_list(ps, g, F64)
    assert list(t.row(0)) == [1]
    rc = c.build_rel_coords(ps, g)
    assert c.tables_equal(t, c.rcll(rc, g, F64))


@pytest.mark.gpu
def test_rebin_invariants_and_errors():
    ps = c.build_random_uniform(c.Domain.unit(2), 500, 31)
    g = c.make_grid_for(ps)
    g.rebin(ps)
    start, items, cell_of = g.cell_start(), g.items(), g.cell_of()
    assert sorted(items.tolist()) == list(range(500))
    for cl in range(g.cell_total()):
        for i in items[start[cl]:start[cl + 1]]:
            assert cell_of[i] == cl
    x0 = ps.x(0)
    x0[17] = 2.5
    ps.set_x(0, x0)
    with pytest.raises(IndexError, match="17"):
        g.rebin(ps)
    empty = c.ParticleSystem(c.Domain.unit(2), 0.1, 0, 1.0)
    g2 = c.CellGrid(c.Domain.unit(2), 0.24, [False, False, False])
    g2.rebin(empty)
    assert not g2.cell_start().any()


@pytest.mark.gpu
def test_build_rel_coords_round_trip():
    ps = c.build_lattice(c.Domain.unit(2), 0.1, 0.0, 1)
    g = c.make_grid_for(ps)
    g.rebin(ps)
    rc = c.build_rel_coords(ps, g)
    for i in range(ps.size()):
        xn = c.normalize_domain([ps.x(0)[i], ps.x(1)[i], 0.0], ps.domain())
        rec = c.reconstruct_norm(rc, i, g)
        assert rec[0] == pytest.approx(xn[0], rel=1e-13) and rec[1] == pytest.approx(xn[1], rel=1e-13)
        assert -1.0 <= rc.rel(0)[i] <= 1.0 and -1.0 <= rc.rel(1)[i] <= 1.0


@pytest.mark.gpu
def test_stale_membership_messages():
    ps = c.build_random_uniform(c.Domain.unit(2), 100, 3)
    g = c.make_grid_for(ps)
    g.rebin(ps)
    other = c.build_random_uniform(c.Domain.unit(2), 101, 3)
    with pytest.raises(ValueError, match="grid membership is stale; rebin first"):
        c.cell_link_list(other, g, F16)
    with pytest.raises(ValueError, match="all_list needs at least one particle"):
        c.all_list(c.ParticleSystem(c.Domain.unit(2), 0.1, 0, 1.0), F16)


# ---- the literal drop-in: reference library with our nnps.cpp ----------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(kind="lattice", dim=2, ds=0.01, jitter=0.3, seed=1),
    dict(kind="lattice", dim=3, ds=0.04, jitter=0.3, seed=2),
    dict(kind="random", dim=2, n=3000, seed=5, periodic=(1, 1, 0)),
    dict(kind="random", dim=1, n=500, seed=6, periodic=(1, 0, 0)),
], ids=["lat2d", "lat3d", "rand2d_periodic", "rand1d_periodic"])
def test_dropin_reference_library_gives_identical_tables(case):
    if not os.path.exists(O.DROPIN_SO):
        pytest.skip("drop-in library not built")
    drop = O.dropin_lib()
    per = case.get("periodic", (0, 0, 0))
    systems = []
    for lib in (O.ref_lib(), drop):
        if case["kind"] == "lattice":
            s = O.RefSystem.lattice(case["dim"], case["ds"], case["jitter"], case["seed"], lib=lib)
        else:
            s = O.RefSystem.random(case["dim"], case["n"], case["seed"], lib=lib)
        systems.append(s.make_grid(periodic=per))
    ref, dr = systems
    for p in (O.FP64, O.FP32, O.FP16):
        for be in ("rcll", "cll"):
            a = getattr(ref, be)(p)
            b = getattr(dr, be)(p)
            assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.items, b.items), (be, p)


@pytest.mark.gpu
def test_concurrent_calls_from_threads():
    """The drop-in releases the GIL; concurrent rcll / cell_link_list / rebin calls
    from several threads share one library context and must each return their own
    table (the session lock holds the context through the table copy)."""
    from concurrent.futures import ThreadPoolExecutor
    systems = []
    for s in range(6):
        ps = c.build_lattice(c.Domain.unit(2), 0.01 + 0.002 * s, 0.3, 40 + s)
        g = c.make_grid_for(ps)
        rc = c.build_rel_coords(ps, g)
        systems.append((ps, g, rc))
    want = [(c.rcll(rc, g, F16), c.cell_link_list(ps, g, F32)) for ps, g, rc in systems]

    def work(k):
        ps, g, rc = systems[k % len(systems)]
        g2 = c.make_grid_for(ps)
        g2.rebin(ps)
        a, b = c.rcll(rc, g, F16), c.cell_link_list(ps, g2, F32)
        wa, wb = want[k % len(systems)]
        return c.tables_equal(a, wa) and c.tables_equal(b, wb)

    with ThreadPoolExecutor(max_workers=6) as ex:
        assert all(ex.map(work, range(36)))
