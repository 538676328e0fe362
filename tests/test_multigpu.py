"""Slab decomposition (paper_2401_08586_b200/multigpu.py).

CPU: the partition rules, and the halo exchange over torch.distributed (gloo,
world_size 2 and 3) with each rank's local sweep emulated by the oracle: the
per-rank rows, mapped to global ids, must equal the global reference rows.
GPU: two and three slabs swept on one device through the C ABI (window binning
+ row-range RCLL); the reassembled table must be the one-GPU table bit for bit.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

import oracle as O
from paper_2401_08586_b200.multigpu import SlabPlan, exchange_halo, pack, unpack


# ---------------------------------------------------------------------------------------
# partition rules (CPU)
# ---------------------------------------------------------------------------------------
def test_plan_bounds_cover_axis():
    p = SlabPlan(3, (10, 11, 37), (0, 0, 0), 4)
    assert p.axis == 2 and p.G == 37
    assert p.bounds[0][0] == 0 and p.bounds[-1][1] == 37
    assert all(a[1] == b[0] for a, b in zip(p.bounds, p.bounds[1:]))
    assert sum(hi - lo for lo, hi in p.bounds) == 37
    assert max(p.nlayers(r) for r in range(4)) - min(p.nlayers(r) for r in range(4)) <= 1
    assert list(p.owner_of_layer(np.arange(37))) == sum(
        ([r] * p.nlayers(r) for r in range(4)), [])


def test_plan_neighbours_wall_and_wrap():
    wall = SlabPlan(2, (8, 20, 1), (1, 0, 0), 3)
    assert [wall.prev(r) for r in range(3)] == [None, 0, 1]
    assert [wall.next(r) for r in range(3)] == [1, 2, None]
    assert wall.layer0(0) == -1 and wall.local_layer_counts(1) == wall.nlayers(1) + 2
    ring = SlabPlan(2, (8, 20, 1), (0, 1, 0), 3)
    assert [ring.prev(r) for r in range(3)] == [2, 0, 1]
    assert [ring.next(r) for r in range(3)] == [1, 2, 0]
    # the reference does not wrap an axis of <= 2 cells (nnps.cpp:223)
    short = SlabPlan(2, (8, 2, 1), (0, 1, 0), 2)
    assert not short.wrap and short.prev(0) is None and short.next(1) is None
    one = SlabPlan(2, (8, 20, 1), (0, 1, 0), 1)
    assert one.prev(0) is None and one.next(0) is None and one.local_layer_counts(0) == 20


def test_plan_rejects_bad_splits():
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 3, 1), (0, 0, 0), 4)   # fewer layers than ranks
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 3, 1), (0, 1, 0), 2)   # periodic: both halos the same layer
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 8, 1), (0, 0, 0), 0)


def test_pack_roundtrip():
    x = [torch.arange(6, dtype=torch.float64) * 0.5, torch.arange(6, dtype=torch.float64)]
    ids = torch.tensor([3, 7, 9, 11, 20, 2**30], dtype=torch.int32)
    sel = torch.tensor([True, False, True, False, True, True])
    xs, i2 = unpack(pack(x, ids, sel), 2)
    assert torch.equal(i2, ids[sel])
    assert torch.equal(xs[0], x[0][sel]) and torch.equal(xs[1], x[1][sel])
    xs, i2 = unpack(pack(x, ids, torch.zeros(6, dtype=torch.bool)), 2)
    assert i2.numel() == 0 and xs[0].numel() == 0


# ---------------------------------------------------------------------------------------
# halo exchange over gloo, local sweeps emulated by the oracle (CPU)
# ---------------------------------------------------------------------------------------
CASES = [  # dim, ds, jitter, periodic, precision
    (2, 0.02, 0.3, (1, 1, 0), 2),
    (2, 0.02, 0.3, (0, 0, 0), 2),
    (3, 0.08, 0.3, (1, 1, 1), 1),
    (1, 0.01, 0.3, (1, 0, 0), 0),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, outdir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc = O.Oracle()
    for ci, (dim, ds, jit, per, prec) in enumerate(CASES):
        x = orc.lattice(dim, ds, jit, 7 + ci)
        g = orc.grid(dim, 2.4 * ds, periodic=per)
        plan = SlabPlan(dim, list(g.counts), list(g.periodic), world)
        _, cell, _, _, _ = orc.build_rel(g, x)
        layer = cell[plan.axis]
        L0, L1 = plan.owned(rank)
        own = np.nonzero((layer >= L0) & (layer < L1))[0]
        xo = [torch.from_numpy(np.ascontiguousarray(a[own])) for a in x]
        io = torch.from_numpy(own.astype(np.int32))
        lay = torch.from_numpy(layer[own])
        down = pack(xo, io, lay == L0)
        up = pack(xo, io, lay == L1 - 1)
        below, above = exchange_halo(plan, rank, down, up)
        xb, ib = unpack(below, dim)
        xa, ia = unpack(above, dim)
        # the halos are exactly the neighbouring layers of the global system
        for msg_ids, want_layer in ((ib, L0 - 1), (ia, L1)):
            if plan.world > 1 and (plan.wrap or 0 <= want_layer < plan.G):
                want = np.nonzero(layer == want_layer % plan.G)[0]
                assert np.array_equal(msg_ids.numpy(), want), (ci, rank, want_layer)
            else:
                assert msg_ids.numel() == 0
        # local sweep (emulated): owned + halo binned on the global grid
        xl = [torch.cat([o, b, a]).numpy() for o, b, a in zip(xo, xb, xa)]
        ids = torch.cat([io, ib, ia]).numpy()
        rel, cl, _, st, it = orc.build_rel(g, xl)
        t = orc.rcll(g, rel, cl, it, st, prec)
        rows = {}
        for r in range(len(own)):
            rows[int(ids[r])] = np.sort(ids[t.items[t.offsets[r]:t.offsets[r + 1]]])
        np.save(os.path.join(outdir, f"case{ci}_rank{rank}.npy"),
                np.array([(k, v) for k, v in rows.items()], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_exchange_matches_global(world):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True)
        orc = O.Oracle()
        for ci, (dim, ds, jit, per, prec) in enumerate(CASES):
            x = orc.lattice(dim, ds, jit, 7 + ci)
            g = orc.grid(dim, 2.4 * ds, periodic=per)
            rel, cell, _, st, it = orc.build_rel(g, x)
            want = orc.rcll(g, rel, cell, it, st, prec)
            seen = np.zeros(len(x[0]), np.int64)
            for r in range(world):
                for i, row in np.load(os.path.join(d, f"case{ci}_rank{r}.npy"),
                                      allow_pickle=True):
                    seen[i] += 1
                    assert np.array_equal(row, want.row(i)), (ci, r, i)
            assert (seen == 1).all(), f"case {ci}: every particle owned exactly once"


# ---------------------------------------------------------------------------------------
# GPU: several slabs on one device == the one-GPU table
# ---------------------------------------------------------------------------------------
GPU_CASES = [  # dim, ds, jitter, periodic, world
    (2, 0.01, 0.3, (1, 1, 0), 2),
    (2, 0.01, 0.3, (0, 0, 0), 3),
    (2, 0.004, 0.0, (0, 1, 0), 4),
    (3, 0.04, 0.3, (1, 1, 1), 2),
    (3, 0.04, 0.2, (0, 0, 0), 3),
    (1, 0.001, 0.3, (1, 0, 0), 2),
]


def _split_tables(P, ctx, dim, ds, jit, per, world, prec):
    from paper_2401_08586_b200 import multigpu as M
    dev = torch.device("cuda", 0)
    x = P.build_lattice(dim, ds, jit, 5)
    n = len(x[0])
    g = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.4 * ds, per)
    # one-GPU table (itself pinned to the reference by test_gpu_parity.py)
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    off1, it1 = ctx.rcll(g, rel, cell, items, start, prec)
    plan = M.SlabPlan.for_grid(g, world)
    slabs, downs, ups = [], [], []
    for r in range(world):
        xo, io, lay = M.owned_from_global(ctx, g, plan, r, x, dev, chunk=max(n // 3, 1))
        s = M.Slab(ctx, g, plan, r, xo, io)
        d, u = s.boundary(layer_global=lay)
        slabs.append(s)
        downs.append(d)
        ups.append(u)
    for s, (below, above) in zip(slabs, M.exchange_local(plan, downs, ups)):
        s.assemble(below, above)
        s.bin()
        s.rows_sized(prec)
    torch.cuda.synchronize()
    off, it = M.global_table(slabs, n)
    return (off1, it1), (off, it), slabs


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: f"{c[0]}d_w{c[4]}_p{''.join(map(str, c[3]))}")
@pytest.mark.parametrize("prec", [0, 1, 2])
def test_slabs_on_one_gpu_equal_global(case, prec):
    import paper_2401_08586_b200 as P
    dim, ds, jit, per, world = case
    ctx = P.Context(0)
    (off1, it1), (off, it), slabs = _split_tables(P, ctx, dim, ds, jit, per, world, prec)
    assert np.array_equal(off, off1)
    assert np.array_equal(it, it1)
    assert sum(s.n_owned for s in slabs) == len(off1) - 1
    # refresh(): the halo re-exchanged from the binned layers gives the same rows
    from paper_2401_08586_b200 import multigpu as M
    plan = slabs[0].plan
    downs, ups = zip(*[s.boundary() for s in slabs])
    for s, (b, a) in zip(slabs, M.exchange_local(plan, list(downs), list(ups))):
        s.assemble(b, a)
        s.bin()
        s.rows_sized(prec)
    off2, it2 = M.global_table(slabs, len(off1) - 1)
    assert np.array_equal(off2, off1) and np.array_equal(it2, it1)


@pytest.mark.gpu
def test_row_range_matches_table_slice():
    import paper_2401_08586_b200 as P
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    x = P.build_lattice(2, 0.01, 0.3, 3)
    n = len(x[0])
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 0.024, (1, 0, 0))
    rel, cell, _, start, items = ctx.build_rel_coords(g, x)
    off, it = ctx.rcll(g, rel, cell, items, start, 2)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rel_d, cell_d = [d(a) for a in rel], [d(a) for a in cell]
    ids = d((np.arange(n) * 3 + 1).astype(np.int32))
    for row0, nrows in ((0, n), (17, 1000), (n - 5, 5), (100, 0)):
        o = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
        out = torch.empty(max(int(off[-1]), 1), dtype=torch.int32, device=dev)
        ctx.rcll_rows_device(g, rel_d, cell_d, d(items), d(start), 2, ids, row0, nrows, o, out)
        oh = o.cpu().numpy()
        assert np.array_equal(oh, off[row0: row0 + nrows + 1] - off[row0])
        want = it[off[row0]: off[row0 + nrows]] * 3 + 1
        assert np.array_equal(out[: int(oh[-1])].cpu().numpy(), want)
    with pytest.raises(ValueError):
        o = torch.empty(2, dtype=torch.int64, device=dev)
        ctx.rcll_rows_device(g, rel_d, cell_d, d(items), d(start), 2, None, n - 1, 2, o, out)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_lattice_device_matches_generator(dim):
    import paper_2401_08586_b200 as P
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    ds = {1: 0.001, 2: 0.01, 3: 0.05}[dim]
    lo, hi = (-0.5, 0.25, 1.0), (0.75, 1.5, 2.0)
    x = P.build_lattice(dim, ds, 0.0, 1, lo=lo, hi=hi)
    n = len(x[0])
    for id0, cnt in ((0, n), (n // 3, n // 2), (n - 1, 1)):
        xd = [torch.empty(cnt, dtype=torch.float64, device=dev) for _ in range(dim)]
        ctx.lattice_device(dim, lo, hi, ds, id0, xd)
        for k in range(dim):
            assert np.array_equal(xd[k].cpu().numpy(), x[k][id0: id0 + cnt])
    with pytest.raises(ValueError):
        ctx.lattice_device(dim, lo, hi, ds, n, [torch.empty(1, dtype=torch.float64,
                                                            device=dev)] * dim)
