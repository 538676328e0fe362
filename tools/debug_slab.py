"""Diagnostics for the slab path on one GPU (developer tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2401_08586_b200 as P  # noqa: E402
from paper_2401_08586_b200 import multigpu as M  # noqa: E402

dim, ds, jit, per, world, prec = 2, 0.01, 0.3, (0, 0, 0), 3, 0
dev = torch.device("cuda", 0)
ctx = P.Context(0)
x = P.build_lattice(dim, ds, jit, 5)
n = len(x[0])
g = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.4 * ds, per)
plan = M.SlabPlan.for_grid(g, world)
print("G", plan.G, "bounds", plan.bounds)
rel, cell, _, start, items = ctx.build_rel_coords(g, x)
off1, it1 = ctx.rcll(g, rel, cell, items, start, prec)
print("full total", off1[-1])
slabs, downs, ups = [], [], []
for r in range(world):
    xo, io, lay = M.owned_from_global(ctx, g, plan, r, x, dev, chunk=max(n // 3, 1))
    print("rank", r, "owned", io.numel(), "layers", int(lay.min()), int(lay.max()))
    s = M.Slab(ctx, g, plan, r, xo, io)
    d, u = s.boundary(layer_global=lay)
    print("  down", d.shape, "up", u.shape)
    slabs.append(s)
    downs.append(d)
    ups.append(u)
for r, (s, (below, above)) in enumerate(zip(slabs, M.exchange_local(plan, downs, ups))):
    s.assemble(below, above)
    s.bin()
    torch.cuda.synchronize()
    it = s.items[: s.n].cpu().numpy()
    st = s.start.cpu().numpy()
    cl = [c[: s.n].cpu().numpy() for c in s.cell]
    print("rank", r, "n", s.n, "local counts", list(s.local.counts), "start[-1]", st[-1],
          "perm ok", np.array_equal(np.sort(it), np.arange(s.n)),
          "layer range", cl[1].min(), cl[1].max(),
          "owned layers", cl[1][: s.n_owned].min(), cl[1][: s.n_owned].max())
    s.rows(prec)
    torch.cuda.synchronize()
    off = s.offsets.cpu().numpy()
    print("  offsets head", off[:5], "tail", off[-3:], "diff min/max", np.diff(off).min(),
          np.diff(off).max())
