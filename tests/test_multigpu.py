"""Slab decomposition (paper_2401_08586_b200/multigpu.py).

CPU: the partition rules, and the whole per-call protocol over torch.distributed
(gloo, world_size 2 and 3): each rank's owned RelCoords in CSR order, the
fixed-capacity boundary-layer messages (exchange_gloo), the local CellGrid
assembly (a numpy restatement of k_slab_assemble) and the rows of the owned
particles (the oracle on the local system) -- mapped to global ids, they must
equal the global reference rows, every particle owned exactly once.
GPU: several slabs on one device through the C ABI (window binning, CSR-order
owned state, exchange_local, sphx_slab_assemble_device, row-range RCLL); the
reassembled table must be the one-GPU table bit for bit. And bench.py at
--gpus 2 --share-gpu: two ranks on one GPU, host-staged gloo halo inside the
timed step, rows checked in-run against the lattice closed form.
"""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

import oracle as O
from paper_2401_08586_b200.multigpu import SlabPlan, exchange_gloo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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
    assert wall.layer0(0) == -1
    ring = SlabPlan(2, (8, 20, 1), (0, 1, 0), 3)
    assert [ring.prev(r) for r in range(3)] == [2, 0, 1]
    assert [ring.next(r) for r in range(3)] == [1, 2, 0]
    # the reference does not wrap an axis of <= 2 cells (nnps.cpp:223)
    short = SlabPlan(2, (8, 2, 1), (0, 1, 0), 2)
    assert not short.wrap and short.prev(0) is None and short.next(1) is None
    one = SlabPlan(2, (8, 20, 1), (0, 1, 0), 1)  # one slab on a ring: its own neighbour
    assert one.prev(0) == 0 and one.next(0) == 0


def test_plan_rejects_bad_splits():
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 3, 1), (0, 0, 0), 4)   # fewer layers than ranks
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 3, 1), (0, 1, 0), 2)   # periodic: both halos the same layer
    with pytest.raises(ValueError):
        SlabPlan(2, (8, 8, 1), (0, 0, 0), 0)


# ---------------------------------------------------------------------------------------
# the per-call protocol over gloo, local sweep by the oracle (CPU)
# ---------------------------------------------------------------------------------------
CASES = [  # dim, ds, jitter, periodic, precision
    (2, 0.02, 0.3, (1, 1, 0), 2),
    (2, 0.02, 0.3, (0, 0, 0), 2),
    (3, 0.08, 0.3, (1, 1, 1), 1),
    (1, 0.01, 0.3, (1, 0, 0), 0),
]


class HostSlab:
    """SlabState's layout and messages on host tensors (the oracle bins)."""

    def __init__(self, plan, rank, g, rel, cell, items, start):
        self.plan, self.rank, self.dim = plan, rank, g.dim
        ax = plan.axis
        L0, L1 = plan.owned(rank)
        self.nl = L1 - L0
        self.CL = int(np.prod([g.counts[k] for k in range(g.dim) if k != ax]))
        CL = self.CL
        cs = start[L0 * CL: L1 * CL + 1]
        own = items[cs[0]: cs[-1]]  # CSR order: owned layers are a contiguous range
        self.n_own = len(own)
        self.owned_start = torch.from_numpy((cs - cs[0]).astype(np.int32))
        self.first_count = int(self.owned_start[CL])
        self.last_begin = int(self.owned_start[(self.nl - 1) * CL])
        self.rel_o = [r[own] for r in rel]
        self.cell_o = [c[own].copy() for c in cell]
        self.cell_o[ax] -= L0 - 1  # local layer: 1 .. nl
        self.ids_o = own.astype(np.int32)

    def boundary_max(self):
        return max(self.first_count, self.n_own - self.last_begin, 1)

    def allocate(self, cap):
        n = self.n_own
        self.cap = cap
        self.slot_below, self.slot_above, self.n_slots = n + cap, n + 2 * cap, n + 3 * cap
        self.rel = [torch.zeros(self.n_slots, dtype=torch.float64) for _ in range(self.dim)]
        self.cell = [torch.zeros(self.n_slots, dtype=torch.int32) for _ in range(self.dim)]
        self.ids = torch.zeros(self.n_slots, dtype=torch.int32)
        for k in range(self.dim):
            self.rel[k][:n] = torch.from_numpy(self.rel_o[k])
            self.cell[k][:n] = torch.from_numpy(self.cell_o[k])
        self.ids[:n] = torch.from_numpy(self.ids_o)
        self.recv_start = [torch.zeros(self.CL + 1, dtype=torch.int32) for _ in range(2)]

    def send(self, side):
        b = 0 if side == 0 else self.last_begin
        s0 = 0 if side == 0 else (self.nl - 1) * self.CL
        return ([r[b: b + self.cap] for r in self.rel] + [self.ids[b: b + self.cap]]
                + [self.owned_start[s0: s0 + self.CL + 1]])

    def recv(self, side):
        b = self.slot_below if side == 0 else self.slot_above
        return ([r[b: b + self.cap] for r in self.rel] + [self.ids[b: b + self.cap]]
                + [self.recv_start[side]])

    def has(self, side):
        return (self.plan.prev(self.rank) if side == 0 else self.plan.next(self.rank)) is not None

    def assemble(self, counts):
        """numpy restatement of k_slab_start / k_slab_items (slab.cu)."""
        ax, CL, nl, n = self.plan.axis, self.CL, self.nl, self.n_own
        rB = self.recv_start[0].numpy().astype(np.int64) if self.has(0) else np.zeros(CL + 1, np.int64)
        rA = self.recv_start[1].numpy().astype(np.int64) if self.has(1) else np.zeros(CL + 1, np.int64)
        rB, rA = rB - rB[0], rA - rA[0]
        mB, mA = int(rB[-1]), int(rA[-1])
        ocs = self.owned_start.numpy().astype(np.int64)
        start = np.concatenate([rB[:-1], mB + ocs[:-1], mB + n + rA]).astype(np.int32)
        items = np.concatenate([self.slot_below + np.arange(mB), np.arange(n),
                                self.slot_above + np.arange(mA)]).astype(np.int32)
        cell = [c.numpy().copy() for c in self.cell]
        for r, slot0, layer in ((rB, self.slot_below, 0), (rA, self.slot_above, nl + 1)):
            for c in range(CL):
                rem, cc = c, [0, 0, 0]
                for k in range(self.dim):
                    if k != ax:
                        cc[k] = rem % counts[k]
                        rem //= counts[k]
                cc[ax] = layer
                for m in range(r[c], r[c + 1]):
                    for k in range(self.dim):
                        cell[k][slot0 + m] = cc[k]
        return start, items, cell


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
        rel, cell, _, start, items = orc.build_rel(g, x)
        s = HostSlab(plan, rank, g, rel, cell, items, start)
        cap = torch.tensor([s.boundary_max()], dtype=torch.int64)
        dist.all_reduce(cap, op=dist.ReduceOp.MAX)
        s.allocate(int(cap))
        exchange_gloo(s)
        lstart, litems, lcell = s.assemble(list(g.counts))
        lg = orc.grid(dim, 2.4 * ds, periodic=per)  # the local grid: nl + 2 layers, walled
        lg.counts[plan.axis] = s.nl + 2
        lg.periodic[plan.axis] = 0
        lg.total = int(np.prod([lg.counts[k] for k in range(dim)]))
        relh = [r.numpy() for r in s.rel]
        t = orc.rcll(lg, relh, lcell, litems, lstart, prec)
        ids = s.ids.numpy()
        rows = {}
        for r in range(s.n_own):
            rows[int(ids[r])] = np.sort(ids[t.items[t.offsets[r]:t.offsets[r + 1]]])
        np.save(os.path.join(outdir, f"case{ci}_rank{rank}.npy"),
                np.array([(k, v) for k, v in rows.items()], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_protocol_matches_global(world):
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
    (2, 0.01, 0.3, (0, 0, 0), 1),
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
    states = []
    for r in range(world):
        xo, io = M.owned_from_host(ctx, g, plan, r, x, dev, chunk=max(n // 3, 1))
        states.append(M.SlabState(ctx, g, plan, r, xo, io))
    cap = max(s.boundary_max() for s in states)
    for s in states:
        s.allocate(cap)
    M.exchange_local(states)
    for s in states:
        s.assemble()
        s.rows(prec)
        torch.cuda.synchronize()
        s.size_output(prec)
    torch.cuda.synchronize()
    off, it = M.global_table(states, n)
    return (off1, it1), (off, it), states


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: f"{c[0]}d_w{c[4]}_p{''.join(map(str, c[3]))}")
@pytest.mark.parametrize("prec", [0, 1, 2])
def test_slabs_on_one_gpu_equal_global(case, prec):
    import paper_2401_08586_b200 as P
    from paper_2401_08586_b200 import multigpu as M
    dim, ds, jit, per, world = case
    ctx = P.Context(0)
    (off1, it1), (off, it), states = _split_tables(P, ctx, dim, ds, jit, per, world, prec)
    assert np.array_equal(off, off1)
    assert np.array_equal(it, it1)
    assert sum(s.n_own for s in states) == len(off1) - 1
    # a second call on the resident state (exchange -> assembly -> rows) is the same
    M.exchange_local(states)
    for s in states:
        s.assemble()
        s.rows(prec)
    torch.cuda.synchronize()
    off2, it2 = M.global_table(states, len(off1) - 1)
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


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_share_gpu(scaling):
    """bench.py --gpus 2 --share-gpu: the N > 1 path end to end on one GPU."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--share-gpu", "--config", "C5s", "--scaling", scaling, "--steps", "3",
                        "--warmup", "1", "--e2e-steps", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([s for s in r.stdout.splitlines() if s.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    p = line["parity"]
    assert p["checked"] and p["bit_exact"] and p["rows_differing"] == 0
    assert p["total"] == p["total_expected"]
    sites = line["config"]["sites"]
    assert sites == ([96, 96, 48] if scaling == "weak" else [96, 96, 96])
    assert line["config"]["halo_bytes_per_step"] > 0
    assert line["ms_per_step"] >= line["breakdown_ms"]["rows"]
