#!/usr/bin/env python
"""Per-step device time of sphx_rcll_device without the library's internal
encode/sweep events (they sit between the two kernels and would serialise a
programmatic dependent launch).   python tools/step_time.py [C2|C3] [steps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_2401_08586_b200 as P
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    w = bench.WORKLOADS[cfg]
    dim, ds = w["dim"], w["ds"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = P.Context(0)
    ctx.set_stream(stream.cuda_stream)
    grid = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    x = P.build_lattice(dim, ds, w["jitter"], w["seed"], (0, 0, 0), w.get("box_hi", (1, 1, 1)))
    n = len(x[0])
    xd = [torch.from_numpy(a).to(dev) for a in x]
    rel = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(dim)]
    cell = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(dim)]
    cell_of = torch.empty(n, dtype=torch.int32, device=dev)
    start = torch.empty(grid.cell_total + 1, dtype=torch.int32, device=dev)
    items = torch.empty(n, dtype=torch.int32, device=dev)
    ctx.build_rel_coords_device(grid, xd, rel, cell, cell_of, start, items)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.empty(n * (24 if dim == 2 else 64), dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    ctx.enable_timing(False)
    for _ in range(5):
        flush.zero_()
        ctx.rcll_device(grid, rel, cell, items, start, 2, off, out)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        ev[k][0].record(stream)
        ctx.rcll_device(grid, rel, cell, items, start, 2, off, out)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    t = statistics.mean(a.elapsed_time(b) for a, b in ev)
    h = P.capi.table_hash(off.cpu().numpy(), out[:int(off[-1])].cpu().numpy())
    lib = os.path.basename(os.environ.get("SPHX_CUDA_LIB", "in-tree libsphx_cuda.so"))
    print(f"{cfg} [{lib}] step {t * 1e3:.1f} us (no internal events), hash {h:016x}")


if __name__ == "__main__":
    main()
