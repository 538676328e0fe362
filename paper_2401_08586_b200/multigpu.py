"""Slab decomposition of the NNPS path: one process per GPU.

The reference is single-process (nnps.cpp has no distributed path); this module
is the B200 scale-out of the same call. Rows are independent per particle, so
the global neighbour table is partitioned by owner:

* The global CellGrid's slowest axis (y in 2-D, z in 3-D, x in 1-D) is cut into
  ``world`` contiguous ranges of whole cell layers (``SlabPlan``). Rank r owns
  the particles whose cell lies in its layers.
* Each rank receives one halo layer from each neighbour (rank +- 1, wrapping when
  the axis is periodic with > 2 layers, the reference's wrap rule nnps.cpp:223)
  over ``torch.distributed`` point-to-point (NCCL on GPUs, gloo in the CPU tests).
* The rank bins owned + halo particles on the GLOBAL grid
  (``sphx_build_rel_coords_window_device``: global normalisation, cell choice
  and Eq. 6 rel bit-identical to the one-GPU run) into a local grid of
  ``nl + 2`` layers with the axis non-periodic, then produces the rows of its
  owned particles only (``sphx_rcll_rows_device``) with global ids as neighbour
  ids. Local arrays are [owned | halo below | halo above], each part in
  ascending global id, so every candidate run is in global-id order and the
  rows come out exactly as the reference's (sorted ascending, nnps.cpp:54).

The union of the per-rank tables, rows placed by global id, is the one-GPU
table bit for bit (tests/test_multigpu.py checks it on one GPU with two slabs,
and the partition + exchange logic on CPU with gloo, world_size 2).
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
        """Rank holding the layer just below rank r's slab (None at a wall)."""
        if self.world == 1:
            return None
        if r > 0:
            return r - 1
        return self.world - 1 if self.wrap else None

    def next(self, r: int):
        if self.world == 1:
            return None
        if r < self.world - 1:
            return r + 1
        return 0 if self.wrap else None

    def layer0(self, r: int) -> int:
        """Global layer of local layer 0 (the lower halo; -1 = below a wall)."""
        return self.bounds[r][0] - 1 if self.world > 1 else 0

    def local_layer_counts(self, r: int) -> int:
        return self.nlayers(r) + 2 if self.world > 1 else self.G

    def local_grid(self, grid, r: int):
        """The rank's CellGrid descriptor: the global one with nl + 2 layers along
        the slab axis, not periodic there (the halos carry the wrap)."""
        if self.world == 1:
            return grid
        g = type(grid).from_buffer_copy(grid)
        g.counts[self.axis] = self.local_layer_counts(r)
        g.periodic[self.axis] = 0
        return g

    def owner_of_layer(self, layer: np.ndarray) -> np.ndarray:
        """Rank owning each global layer."""
        edges = np.array([hi for _, hi in self.bounds])
        return np.searchsorted(edges, np.asarray(layer), side="right")


# ---------------------------------------------------------------------------------------
# halo exchange (the only collective on the path)
# ---------------------------------------------------------------------------------------
def pack(x, ids, sel) -> torch.Tensor:
    """[dim + 1, m] float64 message: positions, then global ids (exact in fp64)."""
    rows = [a[sel] for a in x] + [ids[sel].to(torch.float64)]
    return torch.stack(rows) if rows[0].numel() else torch.empty(
        (len(rows), 0), dtype=torch.float64, device=ids.device)


def unpack(buf: torch.Tensor, dim: int):
    x = [buf[k].contiguous() for k in range(dim)]
    ids = buf[dim].to(torch.int32)
    return x, ids


def exchange_halo(plan: SlabPlan, rank: int, send_down: torch.Tensor, send_up: torch.Tensor,
                  group=None):
    """Send the first owned layer to prev (its upper halo) and the last owned layer
    to next (its lower halo); returns (halo_below, halo_above) messages.

    Operations are posted in the same order on every rank, so the in-order
    matching of NCCL point-to-point pairs them correctly even when prev == next
    (world 2, periodic); gloo matches on the tags.
    """
    prv, nxt = plan.prev(rank), plan.next(rank)
    dev = send_down.device
    rows = send_down.shape[0]

    def ops_for(down, up, from_next, from_prev):
        ops = []
        if prv is not None:
            ops.append(dist.P2POp(dist.isend, down, prv, group=group, tag=0))
        if nxt is not None:
            ops.append(dist.P2POp(dist.isend, up, nxt, group=group, tag=1))
        if nxt is not None:
            ops.append(dist.P2POp(dist.irecv, from_next, nxt, group=group, tag=0))
        if prv is not None:
            ops.append(dist.P2POp(dist.irecv, from_prev, prv, group=group, tag=1))
        return ops

    def run(ops):
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    # sizes, then payloads (at least one column so no zero-byte messages)
    sz_down = torch.tensor([send_down.shape[1]], dtype=torch.int64, device=dev)
    sz_up = torch.tensor([send_up.shape[1]], dtype=torch.int64, device=dev)
    sz_next = torch.zeros(1, dtype=torch.int64, device=dev)
    sz_prev = torch.zeros(1, dtype=torch.int64, device=dev)
    run(ops_for(sz_down, sz_up, sz_next, sz_prev))
    m_next, m_prev = int(sz_next.item()), int(sz_prev.item())

    def padded(buf):
        if buf.shape[1] > 0:
            return buf.contiguous()
        return torch.zeros((rows, 1), dtype=torch.float64, device=dev)

    r_next = torch.empty((rows, max(m_next, 1)), dtype=torch.float64, device=dev)
    r_prev = torch.empty((rows, max(m_prev, 1)), dtype=torch.float64, device=dev)
    run(ops_for(padded(send_down), padded(send_up), r_next, r_prev))
    return r_prev[:, :m_prev], r_next[:, :m_next]


def exchange_local(plan: SlabPlan, downs, ups):
    """The same exchange between slabs held by one process (single-GPU tests)."""
    out = []
    for r in range(plan.world):
        prv, nxt = plan.prev(r), plan.next(r)
        below = ups[prv] if prv is not None else downs[r][:, :0]
        above = downs[nxt] if nxt is not None else downs[r][:, :0]
        out.append((below, above))
    return out


# ---------------------------------------------------------------------------------------
# one rank's slab on its GPU
# ---------------------------------------------------------------------------------------
class Slab:
    """Owned particles (ascending global ids) + halos, binned and swept on one GPU."""

    def __init__(self, ctx: capi.Context, grid, plan: SlabPlan, rank: int, x_owned, ids_owned):
        self.ctx, self.grid, self.plan, self.rank = ctx, grid, plan, rank
        self.local = plan.local_grid(grid, rank)
        self.dim = grid.dim
        self.x_owned = [a.contiguous() for a in x_owned]
        self.ids_owned = ids_owned.contiguous()
        self.n_owned = int(ids_owned.numel())
        self.device = ids_owned.device
        self.layer = None  # local slab-axis layer of each owned particle (after bin())
        self.n = 0

    # -- halo ---------------------------------------------------------------------------
    def boundary(self, layer_global=None):
        """(first-layer message, last-layer message) of the owned particles."""
        if self.plan.world == 1:
            e = torch.empty((self.dim + 1, 0), dtype=torch.float64, device=self.device)
            return e, e
        if layer_global is not None:
            L0, L1 = self.plan.owned(self.rank)
            first, last = layer_global == L0, layer_global == L1 - 1
        else:
            first, last = self.layer == 1, self.layer == self.plan.nlayers(self.rank)
        return pack(self.x_owned, self.ids_owned, first), pack(self.x_owned, self.ids_owned, last)

    def assemble(self, below: torch.Tensor, above: torch.Tensor):
        """Local arrays [owned | halo below | halo above] (each ascending in id)."""
        xb, ib = unpack(below, self.dim)
        xa, ia = unpack(above, self.dim)
        self.x = [torch.cat([o, b, a]).contiguous()
                  for o, b, a in zip(self.x_owned, xb, xa)]
        self.ids = torch.cat([self.ids_owned, ib, ia]).contiguous()
        self.n = int(self.ids.numel())
        self._alloc()

    def _alloc(self):
        """Grow-only device buffers (re-used across refresh() calls)."""
        dev = self.device
        if getattr(self, "_cap", -1) < self.n:
            self._cap = n = max(self.n + self.n // 8, 1)
            self.rel = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(self.dim)]
            self.cell = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(self.dim)]
            self.cell_of = torch.empty(n, dtype=torch.int32, device=dev)
            self.items = torch.empty(n, dtype=torch.int32, device=dev)
        if not hasattr(self, "start"):
            self.start = torch.empty(self.local.cell_total + 1, dtype=torch.int32, device=dev)
            self.offsets = torch.empty(self.n_owned + 1, dtype=torch.int64, device=dev)
            per = {1: 8, 2: 24, 3: 80}[self.dim]
            self.out = torch.empty(max(self.n_owned * per, 1), dtype=torch.int32, device=dev)

    def _view(self, ts):
        return [t[: self.n] for t in ts]

    # -- binning + rows -----------------------------------------------------------------
    def bin(self):
        """Window binning of the local particles on the global grid."""
        x, rel, cell = self._view(self.x), self._view(self.rel), self._view(self.cell)
        if self.plan.world == 1:
            self.ctx.build_rel_coords_device(self.grid, x, rel, cell, self.cell_of[: self.n],
                                             self.start, self.items[: self.n])
        else:
            self.ctx.build_rel_coords_window_device(
                self.grid, self.local, self.plan.axis, self.plan.layer0(self.rank), x, rel, cell,
                self.cell_of[: self.n], self.start, self.items[: self.n])
        self.layer = self.cell[self.plan.axis][: self.n_owned]

    def rows(self, prec: int):
        """Rows of the owned particles into self.offsets / self.out (device API:
        no synchronisation; returns nothing)."""
        self.ctx.rcll_rows_device(self.local, self._view(self.rel), self._view(self.cell),
                                  self.items[: self.n], self.start, prec, self.ids[: self.n], 0,
                                  self.n_owned, self.offsets, self.out)

    def rows_sized(self, prec: int) -> int:
        """rows() growing the output to the exact total (one host sync)."""
        self.rows(prec)
        total = int(self.offsets[-1].item())
        if total > self.out.numel():
            self.out = torch.empty(total + total // 16 + 1024, dtype=torch.int32,
                                   device=self.device)
            self.rows(prec)
        return total

    def refresh(self, prec: int, exchange):
        """Full per-call pipeline: halo exchange -> window binning -> rows."""
        down, up = self.boundary()
        below, above = exchange(down, up)
        self.assemble(below, above)
        self.bin()
        self.rows(prec)


def owned_from_global(ctx: capi.Context, grid, plan: SlabPlan, rank: int, x_host, device,
                      chunk: int = 1 << 22):
    """Owned particles of `rank` out of a host-resident global system: locate every
    particle on the device (global grid), keep those in the rank's layers.
    Returns (x list, global ids, global layer), ascending in id."""
    L0, L1 = plan.owned(rank)
    n = len(x_host[0])
    xs, ids, lays = [[] for _ in range(grid.dim)], [], []
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        m = c1 - c0
        xd = [torch.from_numpy(np.ascontiguousarray(a[c0:c1])).to(device) for a in x_host]
        rel = [torch.empty(m, dtype=torch.float64, device=device) for _ in range(grid.dim)]
        cell = [torch.empty(m, dtype=torch.int32, device=device) for _ in range(grid.dim)]
        cell_of = torch.empty(m, dtype=torch.int32, device=device)
        start = torch.empty(grid.cell_total + 1, dtype=torch.int32, device=device)
        items = torch.empty(m, dtype=torch.int32, device=device)
        ctx.build_rel_coords_device(grid, xd, rel, cell, cell_of, start, items)
        lay = cell[plan.axis]
        keep = (lay >= L0) & (lay < L1)
        for k in range(grid.dim):
            xs[k].append(xd[k][keep])
        ids.append(torch.arange(c0, c1, dtype=torch.int32, device=device)[keep])
        lays.append(lay[keep])
    return [torch.cat(a) for a in xs], torch.cat(ids), torch.cat(lays)


def global_table(slabs, n_global: int):
    """Host CSR of the whole system from per-slab rows (rows placed by global id)."""
    lens = np.zeros(n_global, np.int64)
    parts = []
    for s in slabs:
        off = s.offsets.cpu().numpy()
        ids = s.ids_owned.cpu().numpy()
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
# bench (N > 1 under torchrun)
# ---------------------------------------------------------------------------------------
def _env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def bench(args, workloads, metric, clock_sampler=None, peaks=(6650.0, "fallback"), golden=None):
    """Weak scaling: the config's lattice stacked `world` times along the slab axis
    (rank r owns about one config's worth of particles). A step is one rows() call
    per rank on resident slab inputs (owned + halo RelCoords + local CSR), the
    multi-GPU counterpart of the one-GPU step; the full per-call pipeline
    (halo exchange + window binning + rows) is timed separately under "pipeline"."""
    world, rank, local = _env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if "RANK" not in os.environ:  # `bench.py --slab` without torchrun: a world of one
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    w = workloads[args.config]
    prec = {"fp64": 0, "fp32": 1, "fp16": 2}[args.precision]
    dim, ds = w["dim"], w["ds"]
    h = 1.2 * ds
    hi = [1.0, 1.0, 1.0]
    hi[dim - 1] = float(world)
    x_host = capi.build_lattice(dim, ds, w["jitter"], w["seed"], lo=(0, 0, 0), hi=hi)
    n_global = len(x_host[0])
    grid = capi.grid_init(dim, (0, 0, 0), hi, 2.0 * h)
    plan = SlabPlan.for_grid(grid, world)
    ctx = capi.Context(local)
    ctx.set_stream(stream.cuda_stream)

    xo, io, lay = owned_from_global(ctx, grid, plan, rank, x_host, dev)
    del x_host
    slab = Slab(ctx, grid, plan, rank, xo, io)
    ex = lambda d, u: exchange_halo(plan, rank, d, u)  # noqa: E731
    down, up = slab.boundary(layer_global=lay)
    below, above = ex(down, up)
    slab.assemble(below, above)
    slab.bin()
    total = slab.rows_sized(prec)
    torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    ctx.enable_timing(True)
    for _ in range(args.warmup):
        flush.zero_()
        slab.rows(prec)
    torch.cuda.synchronize()
    dist.barrier()

    sampler = clock_sampler(local) if clock_sampler else None
    if sampler:
        sampler.__enter__()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sweep_ms = []
    torch.cuda.synchronize()
    dist.barrier()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        slab.rows(prec)
        ev[k][1].record(stream)
        sweep_ms.append(ctx.last_timing()[1])
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches - launches0
    t_local = statistics.mean(a.elapsed_time(b) for a, b in ev) * 1e-3

    # full per-call pipeline: exchange + window binning + rows
    pipe_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    ctx.enable_timing(False)
    for _ in range(args.warmup):
        slab.refresh(prec, ex)
    torch.cuda.synchronize()
    dist.barrier()
    for k in range(args.steps):
        flush.zero_()
        pipe_ev[k][0].record(stream)
        slab.refresh(prec, ex)
        pipe_ev[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t_pipe_local = statistics.mean(a.elapsed_time(b) for a, b in pipe_ev) * 1e-3

    # e2e: pinned host inputs -> H2D -> rows -> D2H of the table, per rank
    h_in = [t[: slab.n].cpu().pin_memory() for t in slab.rel + slab.cell] + [
        slab.items[: slab.n].cpu().pin_memory(), slab.start.cpu().pin_memory(),
        slab.ids.cpu().pin_memory()]
    d_in = [t[: slab.n] for t in slab.rel + slab.cell] + [slab.items[: slab.n], slab.start,
                                                         slab.ids]
    h_off = torch.empty(slab.n_owned + 1, dtype=torch.int64).pin_memory()
    h_out = torch.empty(max(total, 1), dtype=torch.int32).pin_memory()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.e2e_steps)]
    for k in range(args.e2e_steps):
        e2e_ev[k][0].record(stream)
        for hsrc, ddst in zip(h_in, d_in):
            ddst.copy_(hsrc, non_blocking=True)
        slab.rows(prec)
        h_off.copy_(slab.offsets, non_blocking=True)
        h_out[:total].copy_(slab.out[:total], non_blocking=True)
        e2e_ev[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t_e2e_local = statistics.mean(a.elapsed_time(b) for a, b in e2e_ev) * 1e-3
    if sampler:
        sampler.__exit__(None, None, None)

    red = torch.tensor([t_local, t_pipe_local, t_e2e_local], dtype=torch.float64, device=dev)
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    cnt = torch.tensor([slab.n_owned, total, launches, slab.n - slab.n_owned,
                        sum(t.numel() * t.element_size() for t in h_in)],
                       dtype=torch.int64, device=dev)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    t_max, t_pipe, t_e2e = red.tolist()
    owned, pairs, launches_all, halo, h2d = [int(v) for v in cnt.tolist()]
    # parity: one slab is the whole system, so its table must carry the reference's
    # golden hash; with more slabs the stacked lattices have no reference table and
    # tests/test_multigpu.py checks slab rows = one-GPU rows bit for bit
    parity = {"checked": False,
              "covered_by": "tests/test_multigpu.py (2/3/4 slabs, every precision: "
                            "reassembled slab tables = the one-GPU table)"}
    if world == 1 and golden is not None and args.config in ("C1", "C2", "C3"):
        from .capi import table_hash
        g = golden(args.config, args.precision)
        h = table_hash(slab.offsets.cpu().numpy(), slab.out[:total].cpu().numpy())
        parity = {"checked": True,
                  "bit_exact_vs_reference_hash": total == g["total"] and f"{h:016x}" == g["hash"],
                  "hash": f"{h:016x}", "golden": g["hash"]}
    if rank == 0:
        assert owned == n_global, (owned, n_global)
        t_sweep = statistics.mean(sweep_ms) * 1e-3
        s_pos = {0: 8, 1: 4, 2: 2}[prec] * dim
        n_l, C_l = slab.n, slab.local.cell_total
        b_sweep = (n_l * s_pos + 4 * n_l + 4 * (C_l + 1) + 8 * (slab.n_owned + 1)
                   + 4 * total)
        peak, peak_kind = peaks
        achieved = b_sweep / t_sweep / 1e9
        line = {
            "metric": metric, "value": owned / t_max, "unit": "particles/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {0: "f64", 1: "f32", 2: "f16"}[prec],
            "data": "synthetic (reference build_lattice generator, seed 1, stacked per rank)",
            "config": {"workload": f"{w['desc']} x{world} stacked along the slab axis",
                       "n_particles": owned, "pairs": pairs, "halo_particles": halo,
                       "precision": args.precision, "backend": "rcll",
                       "parallelism": f"slab{world} (cell layers along axis {plan.axis})",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)"},
            "parity": parity,
            "pipeline": {"ms_per_step": t_pipe * 1e3, "value": owned / t_pipe,
                         "what": "halo exchange (NCCL p2p) + window binning + rows"},
            "roofline": {"bound": "hbm", "kernel": "k_rcll16 (2-D) / k_r16_test + k_r16_emit (3-D), rank 0",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes": b_sweep},
            "e2e": {"value": owned / t_e2e, "unit": "particles/s", "ms_per_step": t_e2e * 1e3,
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * (owned + world) + 4 * pairs,
                    "api": "pinned host slab inputs -> sphx_rcll_rows_device -> pinned table"},
            "gpu_launches": launches_all,
            "clocks": sampler.summary() if sampler else None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()
