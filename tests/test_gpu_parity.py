"""GPU parity: the sm_100a path through the C ABI vs the reference.

Every table must be bit-identical (offsets and items) to the reference's own
output at the same precision: small cases against the full reference tables in
tests/golden/small_cases.npz, BASELINE configs C1..C3 against the reference's
table hashes in tests/golden/golden.json.
"""
import numpy as np
import pytest

import oracle as O
from golden_cases import PREC_NAMES, load_cases, load_configs

pytestmark = pytest.mark.gpu

PREC = {"fp64": 0, "fp32": 1, "fp16": 2}


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


@pytest.fixture(scope="module")
def P():
    import paper_2401_08586_b200 as P
    return P


def _grid(P, meta):
    return P.grid_init(meta["dim"], meta["lo"], meta["hi"], 2.0 * meta["h"], meta["periodic"])


def _eq(got, want, what):
    off, it = got
    woff, wit = want
    assert np.array_equal(off, woff), f"{what}: offsets differ"
    assert np.array_equal(it, wit), f"{what}: items differ"


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c.name)
def test_small_case_binning(ctx, P, case):
    g = _grid(P, case.meta)
    assert list(g.counts)[: case.dim] == case.meta["grid"]["counts"][: case.dim]
    assert g.cutoff_norm == case.meta["grid"]["cutoff_norm"]
    cell_of, start, items = ctx.rebin(g, case.x)
    assert np.array_equal(cell_of, case.cell_of)
    assert np.array_equal(start, case.start)
    assert np.array_equal(items, case.items)
    rel, cell, cell_of2, start2, items2 = ctx.build_rel_coords(g, case.x)
    for k in range(case.dim):
        assert np.array_equal(rel[k], case.rel[k]), f"rel axis {k}"
        assert np.array_equal(cell[k], case.cell[k]), f"cell axis {k}"
    assert np.array_equal(items2, case.items) and np.array_equal(start2, case.start)
    cell_of3, start3, items3 = ctx.rebuild_members(g, case.cell)
    assert np.array_equal(items3, case.items) and np.array_equal(cell_of3, case.cell_of)


@pytest.mark.parametrize("prec", PREC_NAMES)
@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c.name)
def test_small_case_tables(ctx, P, case, prec):
    g = _grid(P, case.meta)
    p = PREC[prec]
    got = ctx.rcll(g, case.rel, case.cell, case.items, case.start, p)
    _eq(got, case.table("rcll", prec), f"rcll {prec}")
    got = ctx.cell_link_list(g, case.x, case.meta["h"], case.items, case.start, case.cell_of, p)
    _eq(got, case.table("cll", prec), f"cll {prec}")
    got = ctx.all_list(case.x, case.meta["h"], p)
    _eq(got, case.table("all", prec), f"all {prec}")


def _config_inputs(name):
    c = load_configs()[name]
    orc = O.Oracle()
    x = orc.lattice(c["dim"], c["ds"], c["jitter"], c["seed"])
    return c, x, 1.2 * c["ds"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_config_golden_hashes(ctx, P, name):
    c, x, h = _config_inputs(name)
    g = P.grid_init(c["dim"], (0, 0, 0), (1, 1, 1), 2.0 * h)
    assert g.cell_total == c["cells"]
    rel, cell, cell_of, start, items = ctx.build_rel_coords(g, x)
    for prec in PREC_NAMES:
        t = ctx.rcll(g, rel, cell, items, start, PREC[prec])
        want = c["tables"][f"rcll_{prec}"]
        assert int(t[0][-1]) == want["total"], f"rcll {prec} total"
        assert f"{O.fnv_hash(*t):016x}" == want["hash"], f"rcll {prec} hash"
        t = ctx.cell_link_list(g, x, h, items, start, cell_of, PREC[prec])
        want = c["tables"][f"cll_{prec}"]
        assert int(t[0][-1]) == want["total"], f"cll {prec} total"
        assert f"{O.fnv_hash(*t):016x}" == want["hash"], f"cll {prec} hash"


def test_table_stream_matches_golden_c2(ctx, P):
    """sphx_table_stream (the drop-in's hand-off, sphx_cuda.h) delivers the offsets
    then the items in whole-element chunks (C2's 78 MB table: several 16 MB
    stage chunks) that concatenate to the golden table; a failing sink stops the
    copy with an error, and the table stays available afterwards."""
    c, x, h = _config_inputs("C2")
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h)
    rel, cell, cell_of, start, items = ctx.build_rel_coords(g, x)
    off, it = ctx.rcll(g, rel, cell, items, start, PREC["fp16"])
    parts, seen = {0: [], 1: []}, []
    ctx.table_stream(lambda part, b: (seen.append(part), parts[part].append(b)) and None)
    assert seen == sorted(seen) and seen.count(1) > 1
    assert all(len(b) % 8 == 0 for b in parts[0]) and all(len(b) % 4 == 0 for b in parts[1])
    s_off = np.frombuffer(b"".join(parts[0]), np.int64)
    s_it = np.frombuffer(b"".join(parts[1]), np.int32)
    assert np.array_equal(s_off, off) and np.array_equal(s_it, it)
    want = c["tables"]["rcll_fp16"]
    assert f"{O.fnv_hash(s_off, s_it):016x}" == want["hash"]
    calls = []
    with pytest.raises(RuntimeError, match="sink"):
        ctx.table_stream(lambda part, b: calls.append(part) or False)
    assert calls == [0]
    again = []
    ctx.table_stream(lambda part, b: again.append(len(b)) and None)
    assert sum(again) == 8 * len(off) + 4 * len(it)


def test_binning_matches_oracle_c2(ctx, P):
    c, x, h = _config_inputs("C2")
    orc = O.Oracle()
    og = orc.grid(2, 2.0 * h)
    orel, ocell, ocell_of, ostart, oitems = orc.build_rel(og, x)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h)
    rel, cell, cell_of, start, items = ctx.build_rel_coords(g, x)
    for k in range(2):
        assert np.array_equal(rel[k], orel[k]) and np.array_equal(cell[k], ocell[k])
    assert np.array_equal(items, oitems) and np.array_equal(start, ostart)
    assert np.array_equal(cell_of, ocell_of)


def test_device_resident_rcll_matches_host_api(ctx, P):
    import torch
    c, x, h = _config_inputs("C2")
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h)
    dev = torch.device("cuda:0")
    xd = [torch.from_numpy(a).to(dev) for a in x]
    n = len(x[0])
    rel = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    cell = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
    cell_of = torch.empty(n, dtype=torch.int32, device=dev)
    start = torch.empty(g.cell_total + 1, dtype=torch.int32, device=dev)
    items = torch.empty(n, dtype=torch.int32, device=dev)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        ctx.build_rel_coords_device(g, xd, rel, cell, cell_of, start, items)
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        out = torch.empty(20 * n, dtype=torch.int32, device=dev)
        ctx.rcll_device(g, rel, cell, items, start, 2, off, out)
        torch.cuda.synchronize()
    finally:
        ctx.set_stream(None)
    total = int(off[-1])
    want = load_configs()["C2"]["tables"]["rcll_fp16"]
    assert total == want["total"]
    assert total <= out.numel()
    h_ = O.fnv_hash(off.cpu().numpy(), out[:total].cpu().numpy())
    assert f"{h_:016x}" == want["hash"]


def test_capacity_overflow_is_reported(ctx, P):
    import torch
    c, x, h = _config_inputs("C1")
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h)
    rel, cell, cell_of, start, items = ctx.build_rel_coords(g, x)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    n = len(x[0])
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.full((1000,), -7, dtype=torch.int32, device=dev)
    ctx.rcll_device(g, [t(r) for r in rel], [t(cc) for cc in cell], t(items), t(start), 2, off,
                    out)
    torch.cuda.synchronize()
    assert int(off[-1]) == load_configs()["C1"]["tables"]["rcll_fp16"]["total"]


# ---- error behaviour mirrors the reference's exceptions ---------------------------------
def test_stale_membership_errors(ctx, P):
    case = load_cases()[0]
    g = _grid(P, case.meta)
    with pytest.raises(ValueError, match="^grid membership is stale$"):
        ctx.rcll(g, case.rel, case.cell, case.items[:-1], case.start, 2)
    with pytest.raises(ValueError, match="^grid membership is stale; rebin first$"):
        ctx.cell_link_list(g, case.x, case.meta["h"], case.items[:-1], case.start, case.cell_of, 2)


def test_rebin_out_of_grid_names_particle(ctx, P):
    orc = O.Oracle()
    x, ds = orc.random(2, 500, 31)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    x[0][17] = 2.5
    x[1][300] = -1.0
    with pytest.raises(IndexError, match="^particle 17 lies outside the grid$"):
        ctx.rebin(g, x)


def test_all_list_needs_a_particle(ctx):
    with pytest.raises(ValueError, match="at least one particle"):
        ctx.all_list([np.empty(0), np.empty(0)], 0.1, 2)


def test_empty_system(ctx, P):
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 0.24)
    cell_of, start, items = ctx.rebin(g, [np.empty(0), np.empty(0)])
    assert len(items) == 0 and not start.any()
    off, it = ctx.rcll(g, [np.empty(0)] * 2, [np.empty(0, np.int32)] * 2, items, start, 2)
    assert list(off) == [0] and len(it) == 0


# ---- properties (test_nnps.cpp:91-103, :158-184) ------------------------------------------
def test_symmetry_no_self(ctx, P):
    case = [c for c in load_cases() if c.name == "symmetry_300"][0]
    for p in (0, 1, 2):
        off, it = ctx.all_list(case.x, case.meta["h"], p)
        for i in range(case.n):
            row = it[off[i]:off[i + 1]]
            assert i not in row
            for j in row:
                back = it[off[j]:off[j + 1]]
                assert i in back


def test_rcll_fp16_matches_rel_distance(ctx, P):
    case = [c for c in load_cases() if c.name == "rcll16_400"][0]
    orc = O.Oracle()
    og = orc.grid(2, 2.0 * case.meta["h"])
    g = _grid(P, case.meta)
    off, it = ctx.rcll(g, case.rel, case.cell, case.items, case.start, 2)
    rel16 = [np.array([orc.round_to(2, v) for v in r]) for r in case.rel]
    cutoff = orc.round_to(2, og.cutoff_norm)
    for i in range(case.n):
        listed = set(it[off[i]:off[i + 1]].tolist())
        for j in range(case.n):
            if i == j or any(abs(int(case.cell[k][i]) - int(case.cell[k][j])) > 1 for k in range(2)):
                continue
            d = orc.rel_distance(og, rel16, case.cell, i, j, 2)
            assert (d < cutoff) == (j in listed)
