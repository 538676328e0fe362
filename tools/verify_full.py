#!/usr/bin/env python
"""Full-table parity of a large configuration ("C4 (16M): full oracle
run on the host"): the reference library's own rcll() (oracle/_ref, all host
threads) and the device table, compared by total and FNV-1a table hash.

    python tools/verify_full.py C4 [--precision fp16]

Prints one JSON line. Test infrastructure: the reference is the checker only.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402  (WORKLOADS, PREC)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["C2", "C3", "C4"])
    ap.add_argument("--precision", default="fp16", choices=sorted(bench.PREC))
    args = ap.parse_args()
    import torch

    import oracle as O
    import paper_2401_08586_b200 as P
    w = bench.WORKLOADS[args.config]
    prec = bench.PREC[args.precision]
    dim, ds = w["dim"], w["ds"]
    x = P.build_lattice(dim, ds, w["jitter"], w["seed"], (0, 0, 0), w.get("box_hi", (1, 1, 1)))
    n = len(x[0])

    # the device table
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    grid = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.4 * ds)
    xd = [torch.from_numpy(a).to(dev) for a in x]
    rel = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(dim)]
    cell = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(dim)]
    cell_of = torch.empty(n, dtype=torch.int32, device=dev)
    start = torch.empty(grid.cell_total + 1, dtype=torch.int32, device=dev)
    items = torch.empty(n, dtype=torch.int32, device=dev)
    ctx.build_rel_coords_device(grid, xd, rel, cell, cell_of, start, items)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.empty(n * 64, dtype=torch.int32, device=dev)
    ctx.rcll_device(grid, rel, cell, items, start, prec, off, out)
    torch.cuda.synchronize()
    total = int(off[-1])
    if total > out.numel():
        out = torch.empty(total, dtype=torch.int32, device=dev)
        ctx.rcll_device(grid, rel, cell, items, start, prec, off, out)
        torch.cuda.synchronize()
    gpu_hash = P.capi.table_hash(off.cpu().numpy(), out[:total].cpu().numpy())
    del xd, rel, cell, cell_of, start, items, off, out

    # the reference's own rcll on the host (domain = the unit cube, like the grid)
    lib = O.ref_lib()
    lib.ref_set_threads(os.cpu_count() or 1)
    r = O.RefSystem.from_arrays(x, ds, lo=(0, 0, 0), hi=(1, 1, 1)).make_grid()
    t0 = time.perf_counter()
    t = lib.ref_rcll(r.rel, r.grid, prec)
    t_ref = time.perf_counter() - t0
    if not t:
        raise O.RefError(lib.ref_last_error().decode())
    ref_total = int(lib.ref_table_total(t))
    ref_hash = int(lib.ref_table_hash(t))
    lib.ref_free_table(t)
    print(json.dumps({
        "check": "full-table parity (SURVEY 8c)", "config": args.config,
        "workload": w["desc"], "precision": args.precision, "n_particles": n,
        "total_gpu": total, "total_reference": ref_total,
        "hash_gpu": f"{gpu_hash:016x}", "hash_reference": f"{ref_hash:016x}",
        "bit_exact": total == ref_total and gpu_hash == ref_hash,
        "reference_seconds": t_ref, "reference_threads": int(lib.ref_max_threads())}))


if __name__ == "__main__":
    main()
