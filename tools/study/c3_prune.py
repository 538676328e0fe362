"""Study (CPU, float64 estimate): how many of the 3-D FP16 RCLL test groups (32
records of one xy-plane run, k_r16_test's hit word) could a per-group bounding
box skip at C3, per lane and per warp (a group is only skipped when all 32 lanes
of the warp skip it: the lanes are CSR-order particles of 2-3 cells sharing their
runs). Bound: y (per dcy class) and z ranges of the group vs the target."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/../..")
import paper_2401_08586_b200 as P  # noqa: E402

x = P.build_lattice(3, 0.01, 0.3, 1, (0, 0, 0), (1, 1, 1))
n = len(x[0])
h = 1.2 * 0.01
cut = 2 * h
nc = int(np.floor(1.0 / cut))
edge = 1.0 / nc
c = [np.minimum((x[k] / edge).astype(np.int64), nc - 1) for k in range(3)]
cell = (c[2] * nc + c[1]) * nc + c[0]
order = np.lexsort((np.arange(n), cell))        # CSR order: cell, then id
starts = np.searchsorted(cell[order], np.arange(nc ** 3 + 1))
rng = np.random.default_rng(0)
warps = rng.choice(n // 32, 400, replace=False)
GS = int(sys.argv[1]) if len(sys.argv) > 1 else 32   # records per group
AX = sys.argv[2] if len(sys.argv) > 2 else "yz"       # axes of the bounding box
tot = lane_skip = warp_skip = 0
for w in warps:
    lanes = order[32 * w: 32 * w + 32]
    # runs are shared by lanes of one cell; evaluate per distinct cell of the warp
    for cc in np.unique(cell[lanes]):
        L = lanes[cell[lanes] == cc]
        cx, cy, cz = cc % nc, (cc // nc) % nc, cc // nc // nc
        for dz in (-1, 0, 1):
            z = cz + dz
            if z < 0 or z >= nc:
                continue
            mem = []
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    yy, xx = cy + dy, cx + dx
                    if 0 <= yy < nc and 0 <= xx < nc:
                        q = (z * nc + yy) * nc + xx
                        mem.append(order[starts[q]:starts[q + 1]])
            run = np.sort(np.concatenate(mem))          # id-merged run
            for g in range(0, len(run), GS):
                grp = run[g:g + GS]
                # per lane: minimum possible distance to the group's bounding box
                d2 = 0.0
                for k in range(3):
                    if "xyz"[k] not in AX:
                        continue
                    lo, hi = x[k][grp].min(), x[k][grp].max()
                    d2 = d2 + np.maximum(0, np.maximum(lo - x[k][L], x[k][L] - hi)) ** 2
                skip = d2 >= cut ** 2
                tot += len(L)
                lane_skip += skip.sum()
                # the warp runs this cell's lanes' loop together with the other cells' lanes
                warp_skip += len(L) if skip.all() else 0
print(f"group {GS} box {AX}: C3 groups x lanes {tot}: per-lane skippable {lane_skip / tot:.1%}, "
      f"warp-uniform skippable {warp_skip / tot:.1%}")
