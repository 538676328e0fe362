"""Slab decomposition of the NNPS path: one process per GPU.

The reference is single-process (nnps.cpp has no distributed path); this module
is the B200 scale-out of the same call. Rows are independent per particle, so
the global neighbour table is partitioned by owner:

* The global CellGrid's slowest axis (y in 2-D, z in 3-D, x in 1-D) is cut into
  ``world`` contiguous ranges of whole cell layers (``SlabPlan``). Rank r owns
  the particles whose cell lies in its layers.
* Each rank keeps its owned particles' RelCoords (on the GLOBAL grid: global
  normalisation, cell choice and Eq. 6 rel bit-identical to one GPU) resident in
  CSR order. The linear cell index is x-fastest (cell_grid.hpp:74-78), so a cell
  layer is a contiguous range of CSR positions: the first and the last owned
  layer are a prefix and a suffix of the rank's arrays.
* A call exchanges those two layers with the neighbouring ranks (rank +- 1,
  wrapping when the axis is periodic with > 2 layers, the reference's wrap rule
  nnps.cpp:223): the rel slice of each axis (FP64, the drop-in's RelCoords), the
  global ids and the layer's slice of cell_start. Messages have a fixed capacity
  agreed once (the largest boundary layer), so no size round trip and no host
  synchronisation: NCCL point-to-point on GPUs (``exchange_nccl``), host-staged
  gloo when several ranks share one GPU (``exchange_gloo``).
* ``sphx_slab_assemble_device`` writes the local CellGrid of nl + 2 layers
  (lower halo, owned, upper halo) from device-side sizes, and
  ``sphx_rcll_rows_device`` produces the rows of the owned particles with global
  ids as neighbour ids. The rows come out sorted exactly as the reference's
  (nnps.cpp:54): every cell's members are ascending in global id.

The union of the per-rank tables, rows placed by global id, is the one-GPU
table bit for bit (tests/test_multigpu.py: several slabs on one GPU, and ranks
over gloo sharing a GPU); the exchange protocol is also checked on CPU (gloo,
world_size 2 and 3).
"""
from __future__ import annotations

import json
import os
import statistics

import numpy as np
import torch
import torch.distributed as dist

from . import capi


# ---------------------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------------------
class SlabPlan:
    """Contiguous cell-layer ranges of the slab axis, one per rank."""

    def __init__(self, dim: int, counts, periodic, world: int):
        if world < 1:
            raise ValueError("world size must be >= 1")
        self.dim = int(dim)
        self.axis = self.dim - 1
        self.G = int(counts[self.axis])
        self.world = int(world)
        # the reference wraps an axis only when it is periodic with > 2 cells
        self.wrap = bool(periodic[self.axis]) and self.G > 2
        if self.G < self.world:
            raise ValueError(f"{self.G} cell layers cannot be split over {world} ranks")
        self.bounds = [(r * self.G // world, (r + 1) * self.G // world) for r in range(world)]
        if world > 1 and self.wrap:
            for lo, hi in self.bounds:
                if hi - lo + 2 > self.G:  # both halos would be the same layer
                    raise ValueError("periodic slab axis too short for this many ranks")

    @classmethod
    def for_grid(cls, grid, world: int) -> "SlabPlan":
        return cls(grid.dim, list(grid.counts), list(grid.periodic), world)

    def owned(self, r: int):
        return self.bounds[r]

    def nlayers(self, r: int) -> int:
        lo, hi = self.bounds[r]
        return hi - lo

    def prev(self, r: int):
        """Rank holding the layer just below rank r's slab (None at a wall; r itself
        for one rank on a periodic axis)."""
        if r > 0:
            return r - 1
        return self.world - 1 if self.wrap else None

    def next(self, r: int):
        if r < self.world - 1:
            return r + 1
        return 0 if self.wrap else None

    def layer0(self, r: int) -> int:
        """Global layer of local layer 0 (the lower halo; -1 = below a wall)."""
        return self.bounds[r][0] - 1

    def local_grid(self, grid, r: int):
        """The rank's CellGrid descriptor: the global one with nl + 2 layers along
        the slab axis, not periodic there (the halos carry the wrap)."""
        g = type(grid).from_buffer_copy(grid)
        g.counts[self.axis] = self.nlayers(r) + 2
        g.periodic[self.axis] = 0
        return g

    def owner_of_layer(self, layer: np.ndarray) -> np.ndarray:
        """Rank owning each global layer."""
        edges = np.array([hi for _, hi in self.bounds])
        return np.searchsorted(edges, np.asarray(layer), side="right")


def cells_per_layer(grid, axis: int) -> int:
    return int(np.prod([grid.counts[k] for k in range(grid.dim) if k != axis]))


# ---------------------------------------------------------------------------------------
# one rank's slab
# ---------------------------------------------------------------------------------------
class SlabState:
    """A rank's resident slab: owned RelCoords in CSR order + reserved halo slots.

    Slots: [owned (n_own) | pad (cap) | lower halo (cap) | upper halo (cap)]. The pad
    lets the last-layer message be a fixed-size slice starting inside the owned part.
    """

    def __init__(self, ctx: capi.Context, grid, plan: SlabPlan, rank: int, x_owned, ids_owned):
        if plan.world == 1 and plan.wrap:
            raise ValueError("one slab on a periodic axis: use the one-GPU path")
        self.ctx, self.grid, self.plan, self.rank = ctx, grid, plan, rank
        self.dim = grid.dim
        self.axis = plan.axis
        self.local = plan.local_grid(grid, rank)
        self.CL = cells_per_layer(grid, self.axis)
        self.nl = plan.nlayers(rank)
        self.device = ids_owned.device
        dev = self.device
        n = int(ids_owned.numel())
        self.n_own = n
        # owned particles on the global grid, binned into the local window (layers 1..nl)
        rel = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(self.dim)]
        cell = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(self.dim)]
        cell_of = torch.empty(n, dtype=torch.int32, device=dev)
        start = torch.empty(self.local.cell_total + 1, dtype=torch.int32, device=dev)
        items = torch.empty(n, dtype=torch.int32, device=dev)
        if n:
            ctx.build_rel_coords_window_device(grid, self.local, self.axis, plan.layer0(rank),
                                               [a.contiguous() for a in x_owned], rel, cell,
                                               cell_of, start, items)
        else:
            start.zero_()
        perm = items.long()  # CSR order: the boundary layers become a prefix and a suffix
        self._rel_o = [r[perm] for r in rel]
        self._cell_o = [c[perm] for c in cell]
        self._ids_o = ids_owned[perm].contiguous()
        CL, nl = self.CL, self.nl
        st = start.cpu().numpy().astype(np.int64)
        if st[CL] != 0 or st[(nl + 1) * CL] != n:
            raise RuntimeError("owned particles outside the rank's layers")
        self.owned_start = start[CL: (nl + 1) * CL + 1].contiguous()
        self.first_count = int(st[2 * CL] - st[CL])           # layer 1
        self.last_begin = int(st[nl * CL] - st[CL])            # layer nl
        self.last_count = n - self.last_begin
        self.cap = None

    def boundary_max(self) -> int:
        return max(self.first_count, self.last_count, 1)

    def allocate(self, cap: int):
        """Slot arrays for a fixed message capacity (the largest boundary layer)."""
        dev, n, d = self.device, self.n_own, self.dim
        self.cap = int(cap)
        self.slot_below = n + self.cap
        self.slot_above = n + 2 * self.cap
        self.n_slots = n + 3 * self.cap
        self.rel = [torch.zeros(self.n_slots, dtype=torch.float64, device=dev) for _ in range(d)]
        self.cell = [torch.zeros(self.n_slots, dtype=torch.int32, device=dev) for _ in range(d)]
        self.ids = torch.zeros(self.n_slots, dtype=torch.int32, device=dev)
        for k in range(d):
            self.rel[k][:n] = self._rel_o[k]
            self.cell[k][:n] = self._cell_o[k]
        self.ids[:n] = self._ids_o
        del self._rel_o, self._cell_o, self._ids_o
        self.recv_start = [torch.zeros(self.CL + 1, dtype=torch.int32, device=dev)
                           for _ in range(2)]
        self.start = torch.empty(self.local.cell_total + 1, dtype=torch.int32, device=dev)
        self.items = torch.empty(self.n_slots, dtype=torch.int32, device=dev)
        self.offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        per = {1: 8, 2: 24, 3: 64}[self.dim]
        self.out = torch.empty(max(n * per, 1), dtype=torch.int32, device=dev)

    # -- messages -------------------------------------------------------------------------
    def send(self, side: int):
        """Side 0: the first owned layer (to prev); side 1: the last (to next). Fixed
        sizes: rel[k] (cap), ids (cap), cell_start slice (CL + 1)."""
        b = 0 if side == 0 else self.last_begin
        s0 = 0 if side == 0 else (self.nl - 1) * self.CL
        return ([r[b: b + self.cap] for r in self.rel] + [self.ids[b: b + self.cap]]
                + [self.owned_start[s0: s0 + self.CL + 1]])

    def recv(self, side: int):
        """Side 0: the lower halo (from prev); side 1: the upper halo (from next)."""
        b = self.slot_below if side == 0 else self.slot_above
        return ([r[b: b + self.cap] for r in self.rel] + [self.ids[b: b + self.cap]]
                + [self.recv_start[side]])

    def has(self, side: int) -> bool:
        return (self.plan.prev(self.rank) if side == 0 else self.plan.next(self.rank)) is not None

    # -- per call ------------------------------------------------------------------------
    def assemble(self):
        self.ctx.slab_assemble_device(
            self.local, self.axis, self.n_own, self.slot_below, self.slot_above, self.n_slots,
            self.owned_start, self.recv_start[0] if self.has(0) else None,
            self.recv_start[1] if self.has(1) else None, self.start, self.items, self.cell)

    def rows(self, prec: int):
        self.ctx.rcll_rows_device(self.local, self.rel, self.cell, self.items, self.start, prec,
                                  self.ids, 0, self.n_own, self.offsets, self.out)

    def step(self, prec: int, exchange):
        """One NNPS call of the rank: halo exchange -> local CellGrid -> owned rows."""
        exchange(self)
        self.assemble()
        self.rows(prec)

    def size_output(self, prec: int) -> int:
        """Grow the row buffer to the exact total (one host sync, setup only)."""
        total = int(self.offsets[-1].item())
        if total > self.out.numel():
            self.out = torch.empty(total + total // 16 + 1024, dtype=torch.int32,
                                   device=self.device)
            self.rows(prec)
        return total


# ---------------------------------------------------------------------------------------
# halo exchange (the only collective on the path)
# ---------------------------------------------------------------------------------------
def _coll_device(device):
    """Collectives run on the device under NCCL, on the host under gloo."""
    return device if dist.get_backend() == "nccl" else torch.device("cpu")


def agree_capacity(state: SlabState, group=None) -> int:
    """Largest boundary layer over all ranks (once per setup)."""
    t = torch.tensor([state.boundary_max()], dtype=torch.int64,
                     device=_coll_device(state.device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def _nvtx(name):
    """NVTX range (Nsight) around a host-side phase; a no-op without CUDA."""
    import contextlib
    if torch.cuda.is_available():
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


def exchange_nccl(st: SlabState, group=None):
    with _nvtx("sphx.halo"):
        _exchange_nccl(st, group)


def _exchange_nccl(st: SlabState, group=None):
    """First layer -> prev, last layer -> next, halos <- both, in one NCCL group.
    Operations are posted in the same order on every rank, so NCCL's in-order
    matching of point-to-point pairs is right even when prev == next (world 2,
    periodic). Stream-ordered: the waits make the current stream wait."""
    prv, nxt = st.plan.prev(st.rank), st.plan.next(st.rank)
    if prv == st.rank:  # one rank on a periodic axis: its own opposite layers
        return exchange_local([st])
    ops = []
    if prv is not None:
        ops += [dist.P2POp(dist.isend, t, prv, group=group) for t in st.send(0)]
    if nxt is not None:
        ops += [dist.P2POp(dist.isend, t, nxt, group=group) for t in st.send(1)]
    if nxt is not None:
        ops += [dist.P2POp(dist.irecv, t, nxt, group=group) for t in st.recv(1)]
    if prv is not None:
        ops += [dist.P2POp(dist.irecv, t, prv, group=group) for t in st.recv(0)]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def exchange_gloo(st: SlabState, group=None):
    with _nvtx("sphx.halo"):
        _exchange_gloo(st, group)


def _exchange_gloo(st: SlabState, group=None):
    """The same exchange staged through host memory over gloo (ranks sharing a
    GPU, where NCCL cannot run): device -> host, tagged send/recv, host -> device."""
    prv, nxt = st.plan.prev(st.rank), st.plan.next(st.rank)
    if prv == st.rank:
        return exchange_local([st])
    works, inbox = [], []
    for side, peer, tag in ((0, prv, 0), (1, nxt, 1)):
        if peer is None:
            continue
        for i, t in enumerate(st.send(side)):
            works.append(dist.isend(t.cpu(), peer, group=group, tag=16 * tag + i))
    for side, peer, tag in ((1, nxt, 0), (0, prv, 1)):
        if peer is None:
            continue
        for i, t in enumerate(st.recv(side)):
            h = torch.empty(t.shape, dtype=t.dtype)
            works.append(dist.irecv(h, peer, group=group, tag=16 * tag + i))
            inbox.append((t, h))
    for w in works:
        w.wait()
    for t, h in inbox:
        t.copy_(h, non_blocking=False)


def exchange_local(states):
    """The same exchange between slabs held by one process (single-GPU tests)."""
    by_rank = {st.rank: st for st in states}
    for st in states:
        plan, r = st.plan, st.rank
        for side, peer, their in ((0, plan.prev(r), 1), (1, plan.next(r), 0)):
            if peer is None:
                continue
            for dst, src in zip(st.recv(side), by_rank[peer].send(their)):
                dst.copy_(src)


# ---------------------------------------------------------------------------------------
# owned particles of a rank
# ---------------------------------------------------------------------------------------
def _layers(ctx, grid, axis, pts, device):
    """Global cell layer of each point (device binning on the global grid)."""
    m = pts[0].numel()
    rel = [torch.empty(m, dtype=torch.float64, device=device) for _ in range(grid.dim)]
    cell = [torch.empty(m, dtype=torch.int32, device=device) for _ in range(grid.dim)]
    cell_of = torch.empty(m, dtype=torch.int32, device=device)
    start = torch.empty(grid.cell_total + 1, dtype=torch.int32, device=device)
    items = torch.empty(m, dtype=torch.int32, device=device)
    ctx.build_rel_coords_device(grid, pts, rel, cell, cell_of, start, items)
    return cell[axis]


def owned_from_host(ctx, grid, plan: SlabPlan, rank: int, x_host, device, chunk: int = 1 << 22):
    """Owned particles of `rank` out of a host-resident global system (ascending ids)."""
    L0, L1 = plan.owned(rank)
    n = len(x_host[0])
    xs, ids = [[] for _ in range(grid.dim)], []
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        xd = [torch.from_numpy(np.ascontiguousarray(a[c0:c1])).to(device) for a in x_host]
        lay = _layers(ctx, grid, plan.axis, xd, device)
        keep = (lay >= L0) & (lay < L1)
        for k in range(grid.dim):
            xs[k].append(xd[k][keep])
        ids.append(torch.arange(c0, c1, dtype=torch.int32, device=device)[keep])
    return [torch.cat(a) for a in xs], torch.cat(ids)


def owned_lattice_device(ctx, grid, plan: SlabPlan, rank: int, sites, ds, lo, hi, device):
    """Owned sites of an un-jittered lattice generated on the device
    (sphx_lattice_device, bit-identical to build_lattice): only the planes around
    the rank's layers are generated, then kept by their cell layer."""
    dim, axis = grid.dim, plan.axis
    L0, L1 = plan.owned(rank)
    plane = int(np.prod([sites[k] for k in range(dim) if k != axis]))
    per_layer = float(grid.hc[axis]) / (2.0 * ds / max(hi[k] - lo[k] for k in range(dim)))
    p0 = max(int(np.floor(L0 * per_layer)) - 2, 0)
    p1 = min(int(np.ceil(L1 * per_layer)) + 2, sites[axis])
    xd = [torch.empty((p1 - p0) * plane, dtype=torch.float64, device=device) for _ in range(dim)]
    ctx.lattice_device(dim, lo, hi, ds, p0 * plane, xd)
    lay = _layers(ctx, grid, axis, xd, device)
    keep = (lay >= L0) & (lay < L1)
    ids = torch.arange(p0 * plane, p1 * plane, dtype=torch.int32, device=device)[keep]
    if ids.numel():
        first, last = int(ids[0]) // plane, int(ids[-1]) // plane
        if (first == p0 and p0 > 0) or (last == p1 - 1 and p1 < sites[axis]):
            raise RuntimeError("plane window too narrow for the rank's layers")
    return [a[keep] for a in xd], ids


def global_table(states, n_global: int):
    """Host CSR of the whole system from per-slab rows (rows placed by global id)."""
    lens = np.zeros(n_global, np.int64)
    parts = []
    for s in states:
        off = s.offsets.cpu().numpy()
        ids = s.ids[: s.n_own].cpu().numpy()
        lens[ids] = np.diff(off)
        parts.append((ids, off, s.out[: int(off[-1])].cpu().numpy()))
    offsets = np.zeros(n_global + 1, np.int64)
    np.cumsum(lens, out=offsets[1:])
    items = np.empty(int(offsets[-1]), np.int32)
    for ids, off, it in parts:
        for r, i in enumerate(ids):
            items[offsets[i]: offsets[i + 1]] = it[off[r]: off[r + 1]]
    return offsets, items


# ---------------------------------------------------------------------------------------
# parity (in the bench)
# ---------------------------------------------------------------------------------------
LATTICE_OFFSETS3 = [(a, b, c) for a in range(-2, 3) for b in range(-2, 3) for c in range(-2, 3)
                    if 0 < a * a + b * b + c * c < 5.76]  # |v| < kh = 2.4 ds: 56 sites
LATTICE_OFFSETS2 = [(a, b, 0) for a in range(-2, 3) for b in range(-2, 3)
                    if 0 < a * a + b * b < 5.76]


def lattice_total(sites) -> int:
    offs = LATTICE_OFFSETS3 if len(sites) == 3 else LATTICE_OFFSETS2
    return int(sum(np.prod([max(sites[k] - abs(v[k]), 0) for k in range(len(sites))],
                           dtype=np.int64) for v in offs))


def sampled_rows(st: SlabState, samples: int, seed: int):
    n = st.n_own
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(samples, n), replace=False)) if n else np.zeros(0, int)
    off = st.offsets.cpu().numpy()
    out = st.out[: int(off[-1])].cpu().numpy()
    return idx, [out[off[i]: off[i + 1]] for i in idx]


def parity_lattice(st: SlabState, sites, samples=1000, seed=1):
    """Sampled owned rows against the un-jittered lattice's closed form (the sites
    within 2.4 ds, global ids)."""
    dim = len(sites)
    offs = LATTICE_OFFSETS3 if dim == 3 else LATTICE_OFFSETS2
    idx, rows = sampled_rows(st, samples, seed + st.rank)
    gid = st.ids[: st.n_own].cpu().numpy()
    bad = 0
    for i, row in zip(idx, rows):
        g = int(gid[i])
        c = [g % sites[0], (g // sites[0]) % sites[1] if dim > 1 else 0,
             g // (sites[0] * sites[1]) if dim > 2 else 0]
        exp = []
        for v in offs:
            q = [c[k] + v[k] for k in range(dim)]
            if all(0 <= q[k] < sites[k] for k in range(dim)):
                exp.append(q[0] + sites[0] * (q[1] + (sites[1] * q[2] if dim > 2 else 0)))
        bad += int(not np.array_equal(row, np.array(sorted(exp), dtype=np.int32)))
    return len(idx), bad


def parity_oracle(st: SlabState, prec: int, samples=500, seed=1):
    """Sampled owned rows against the oracle's rel_distance classification of every
    CSR member of the 3^d local neighbour cells (rel_distance(...) < round_to(prec,
    cutoff) <=> listed, test_nnps.cpp:158-184)."""
    import oracle as O
    orc = O.Oracle()
    dim = st.dim
    og = orc.grid(dim, st.grid.radius_phys, lo=list(st.grid.lo), hi=list(st.grid.hi),
                  periodic=list(st.grid.periodic))
    relh = [t.cpu().numpy() for t in st.rel]
    cellh = [t.cpu().numpy() for t in st.cell]
    start = st.start.cpu().numpy()
    items = st.items.cpu().numpy()
    ids = st.ids.cpu().numpy()
    cnt = list(st.local.counts)[:dim]
    per = [bool(st.local.periodic[k]) and cnt[k] > 2 for k in range(dim)]
    cutoff = orc.round_to(prec, og.cutoff_norm)
    idx, rows = sampled_rows(st, samples, seed + st.rank)
    bad = 0
    rng3 = [(-1, 0, 1) if k < dim else (0,) for k in range(3)]
    for i, row in zip(idx, rows):
        ci = [int(cellh[k][i]) for k in range(dim)]
        exp = []
        for dz in rng3[2]:
            for dy in rng3[1]:
                for dx in rng3[0]:
                    c = [ci[k] + (dx, dy, dz)[k] for k in range(dim)]
                    ok = True
                    for k in range(dim):
                        if not 0 <= c[k] < cnt[k]:
                            if not per[k]:
                                ok = False
                            c[k] %= cnt[k]
                    if not ok:
                        continue
                    lin = c[0] + (cnt[0] * (c[1] + (cnt[1] * c[2] if dim > 2 else 0)) if dim > 1 else 0)
                    for p in range(start[lin], start[lin + 1]):
                        j = int(items[p])
                        if j != i and orc.rel_distance(og, relh, cellh, int(i), j, prec) < cutoff:
                            exp.append(int(ids[j]))
        bad += int(not np.array_equal(row, np.array(sorted(exp), dtype=np.int32)))
    return len(idx), bad


# ---------------------------------------------------------------------------------------
# bench (N > 1 under torchrun)
# ---------------------------------------------------------------------------------------
def _env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_sites(w, world: int, scaling: str):
    """Global lattice sites per axis and the domain [0, hi] for `world` ranks. Weak
    scaling stacks the per-GPU lattice (w["weak_sites"], else the whole config)
    `world` times along the slab axis; strong splits the whole config."""
    dim, ds = w["dim"], w["ds"]
    side = [int(round(1.0 / ds))] * dim
    if scaling == "weak" and "weak_sites" in w:
        side = list(w["weak_sites"])
    hi = [s * ds for s in side]
    if scaling == "weak":
        side[dim - 1] *= world
        hi[dim - 1] *= world
    return side, hi


def bench(args, workloads, metric, clock_sampler=None, peaks=(6650.0, "fallback")):
    """N ranks, one slab each. A step is one NNPS call per rank: the halo exchange
    (NCCL, or host-staged gloo with --share-gpu), the slab assembly and the owned
    rows, on resident owned RelCoords -- timed with CUDA events on the rank's
    stream, the reported time the max over ranks of the median step."""
    world, rank, local = _env()
    share = bool(getattr(args, "share_gpu", False))
    dev_index = 0 if share else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if share:
        dist.init_process_group("gloo")
        exchange = exchange_gloo
    else:
        dist.init_process_group("nccl", device_id=dev)
        exchange = exchange_nccl
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    w = workloads[args.config]
    scaling = args.scaling
    prec = {"fp64": 0, "fp32": 1, "fp16": 2}[args.precision]
    dim, ds = w["dim"], w["ds"]
    h = 1.2 * ds
    sites, hi = workload_sites(w, world, scaling)
    lo = [0.0] * dim
    grid = capi.grid_init(dim, (0, 0, 0), hi + [1.0] * (3 - dim), 2.0 * h)
    plan = SlabPlan.for_grid(grid, world)
    ctx = capi.Context(dev_index)
    ctx.set_stream(stream.cuda_stream)

    if w.get("device_lattice"):
        xo, io = owned_lattice_device(ctx, grid, plan, rank, sites, ds, lo, hi, dev)
    else:
        x_host = capi.build_lattice(dim, ds, w["jitter"], w["seed"], lo=(0, 0, 0),
                                    hi=tuple(hi) + (1.0,) * (3 - dim))
        xo, io = owned_from_host(ctx, grid, plan, rank, x_host, dev)
        del x_host
    n_global = int(np.prod(sites))
    st = SlabState(ctx, grid, plan, rank, xo, io)
    del xo, io
    st.allocate(agree_capacity(st) if world > 1 else st.boundary_max())
    st.step(prec, exchange)
    torch.cuda.synchronize()
    total = st.size_output(prec)
    torch.cuda.synchronize()

    # parity of this run: sampled rows (closed form / oracle) and the global total
    if w.get("device_lattice") or w["jitter"] == 0.0:
        checked, bad = parity_lattice(st, sites)
        method = "sampled rows vs lattice closed form; total vs closed form"
    else:
        checked, bad = parity_oracle(st, prec)
        method = "sampled rows vs oracle rel_distance classification of the 3^d cells"

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        flush.zero_()
        st.step(prec, exchange)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = clock_sampler(dev_index) if clock_sampler else None
    if sampler:
        sampler.__enter__()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    dist.barrier()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        st.step(prec, exchange)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches - launches0
    t_local = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e-3
    # the rows alone (no exchange, no assembly), for the kernel's share of the step
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(max(args.steps // 2, 3))]
    for a, b in ev2:
        flush.zero_()
        a.record(stream)
        st.rows(prec)
        b.record(stream)
    torch.cuda.synchronize()
    t_rows_local = statistics.median(a.elapsed_time(b) for a, b in ev2) * 1e-3

    # e2e: the owned inputs from pinned host memory, the exchange, rows, the table back
    h_in = [t[: st.n_own].cpu().pin_memory() for t in st.rel + st.cell] + [
        st.ids[: st.n_own].cpu().pin_memory()]
    d_in = [t[: st.n_own] for t in st.rel + st.cell] + [st.ids[: st.n_own]]
    h_off = torch.empty(st.n_own + 1, dtype=torch.int64).pin_memory()
    h_out = torch.empty(max(total, 1), dtype=torch.int32).pin_memory()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(max(args.e2e_steps, 1))]
    dist.barrier()
    for a, b in e2e_ev:
        a.record(stream)
        for hsrc, ddst in zip(h_in, d_in):
            ddst.copy_(hsrc, non_blocking=True)
        st.step(prec, exchange)
        h_off.copy_(st.offsets, non_blocking=True)
        h_out[:total].copy_(st.out[:total], non_blocking=True)
        b.record(stream)
    torch.cuda.synchronize()
    t_e2e_local = statistics.median(a.elapsed_time(b) for a, b in e2e_ev) * 1e-3
    if sampler:
        sampler.__exit__(None, None, None)

    cdev = _coll_device(dev)
    red = torch.tensor([t_local, t_rows_local, t_e2e_local], dtype=torch.float64, device=cdev)
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    h2d_local = sum(t.numel() * t.element_size() for t in h_in)
    halo_local = (st.cap * (8 * dim + 4) + 4 * (st.CL + 1)) * (int(st.has(0)) + int(st.has(1)))
    cnt = torch.tensor([st.n_own, total, launches, checked, bad, h2d_local, halo_local],
                       dtype=torch.int64, device=cdev)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    t_max, t_rows, t_e2e = red.tolist()
    owned, pairs, launches_all, checked, bad, h2d, halo_bytes = [int(v) for v in cnt.tolist()]
    closed = lattice_total(sites) if (w.get("device_lattice") or w["jitter"] == 0.0) else None
    if rank == 0:
        assert owned == n_global, (owned, n_global)
        s_pos = {0: 8, 1: 4, 2: 2}[prec] * dim
        C = grid.cell_total
        b_sweep = (n_global * s_pos + 4 * n_global + 4 * (C + world) + 8 * (n_global + world)
                   + 4 * pairs)
        peak, peak_kind = peaks
        achieved = b_sweep / world / t_rows / 1e9
        parity = {"checked": True, "rows_checked": checked, "rows_differing": bad,
                  "method": method,
                  "bit_exact": bool(bad == 0 and (closed is None or closed == pairs))}
        if closed is not None:
            parity.update(total=pairs, total_expected=closed)
        line = {
            "metric": metric, "value": owned / t_max, "unit": "particles/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": {0: "f64", 1: "f32", 2: "f16"}[prec],
            "data": ("synthetic (lattice generated on the device per rank)"
                     if w.get("device_lattice") else
                     "synthetic (reference build_lattice generator, seed 1)"),
            "config": {"workload": f"{w['desc']}, {scaling} scaling over {world} slab(s)",
                       "sites": sites, "n_particles": owned, "pairs": pairs,
                       "precision": args.precision, "backend": "rcll",
                       "parallelism": f"slab{world} (cell layers along axis {plan.axis})",
                       "exchange": ("host-staged gloo, ranks sharing one GPU" if share else
                                    "NCCL p2p (grouped send/recv of the boundary layers)"),
                       "halo_bytes_per_step": halo_bytes,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)"},
            "parity": parity,
            "breakdown_ms": {"step": t_max * 1e3, "rows": t_rows * 1e3,
                             "exchange_and_assembly": (t_max - t_rows) * 1e3},
            "roofline": {"bound": "hbm", "kernel": "the rows of one rank (max over ranks)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes_per_rank": b_sweep / world},
            "e2e": {"value": owned / t_e2e, "unit": "particles/s", "ms_per_step": t_e2e * 1e3,
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * (owned + world) + 4 * pairs,
                    "api": "pinned host owned RelCoords -> exchange + assembly + rows -> "
                           "pinned table"},
            "gpu_launches": launches_all,
            "clocks": sampler.summary() if sampler else None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()
