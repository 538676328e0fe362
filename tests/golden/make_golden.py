"""Generate the golden vectors from the reference itself (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref can be
built):  ``python tests/golden/make_golden.py``.  Outputs, committed:

* ``tests/golden/golden.json`` -- per BASELINE config (C1..C3) and backend x
  precision: particle count, cell count, total pairs, max row, FNV-1a table hash
  (SURVEY.md 8(c) hash definition) computed from the reference's own tables.
* ``tests/golden/small_cases.npz`` + ``small_cases.json`` -- small systems with
  their positions, grid CSR and the full reference tables for every backend and
  precision: the cases restate the reference tests' inputs (test_nnps.cpp:71-89,
  :105-156, :91-103, :158-184, :241-257) plus periodic, non-unit-domain, tiny and
  clustered edge cases.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

PRECS = (O.FP64, O.FP32, O.FP16)


def table_summary(t: O.Table) -> dict:
    rows = np.diff(t.offsets)
    return {"total": int(t.total), "hash": f"{t.hash():016x}",
            "max_row": int(rows.max()) if len(rows) else 0,
            "min_row": int(rows.min()) if len(rows) else 0}


def config_goldens() -> dict:
    cfgs = {
        "C1": dict(dim=2, ds=0.01, jitter=0.0, seed=1),
        "C2": dict(dim=2, ds=0.001, jitter=0.3, seed=1),
        "C3": dict(dim=3, ds=0.01, jitter=0.3, seed=1),
    }
    out = {}
    for name, c in cfgs.items():
        r = O.RefSystem.lattice(c["dim"], c["ds"], c["jitter"], c["seed"]).make_grid()
        entry = dict(c, n=r.n, cells=r.cell_total(), grid=r.grid_desc(), tables={})
        for p in PRECS:
            for be in ("rcll", "cll"):
                t = r.rcll(p) if be == "rcll" else r.cll(p)
                entry["tables"][f"{be}_{O.PREC_NAMES[p]}"] = table_summary(t)
                print(name, be, O.PREC_NAMES[p], entry["tables"][f"{be}_{O.PREC_NAMES[p]}"],
                      flush=True)
        out[name] = entry
    return out


class Rng:
    """Drives the C restatement's mt19937_64 to reproduce the reference tests'
    parameter draws (rng.hpp)."""

    def __init__(self, seed):
        import ctypes as C
        self.lib = O._oracle_lib()
        self.lib.so_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        self.lib.so_rng_next.restype = C.c_uint64
        self.lib.so_rng_next.argtypes = [C.c_void_p]
        self.lib.so_rng_below.restype = C.c_uint64
        self.lib.so_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        self.buf = C.create_string_buffer(312 * 8 + 8)
        self.lib.so_rng_seed(self.buf, seed)

    def next_u64(self):
        return int(self.lib.so_rng_next(self.buf))

    def below(self, n):
        return int(self.lib.so_rng_below(self.buf, n))


def small_cases():
    cases = []
    # test_nnps.cpp:71-89 -- backend equivalence draws
    rng = Rng(101)
    for dim in (1, 2, 3):
        for _ in range(3):
            n = 50 + rng.below(400)
            seed = rng.next_u64()
            cases.append(dict(name=f"equiv_d{dim}_n{n}", kind="random", dim=dim, n=n, seed=seed))
    # test_nnps.cpp:105-156 -- batch vs scalar draws
    rng = Rng(313)
    for rep in range(4):
        n = 200 + rng.below(600)
        seed = rng.next_u64()
        if rep % 2 == 0:
            cases.append(dict(name=f"batch_rand_n{n}", kind="random", dim=2, n=n, seed=seed))
        else:
            cases.append(dict(name=f"batch_lat_n{n}", kind="lattice", dim=2,
                              ds=0.97 / np.sqrt(float(n)), jitter=0.3, seed=seed))
    cases.append(dict(name="symmetry_300", kind="random", dim=2, n=300, seed=7))
    cases.append(dict(name="rcll16_400", kind="random", dim=2, n=400, seed=99))
    cases.append(dict(name="perm_500", kind="random", dim=2, n=500, seed=1234))
    # periodic seam (test_nnps.cpp:241-257)
    cases.append(dict(name="seam", kind="arrays", dim=2, ds=0.05,
                      x=[[0.01, 0.99], [0.5, 0.5]], periodic=[1, 0, 0]))
    # periodic / domain / shape edge cases
    cases.append(dict(name="periodic_xy_d2", kind="random", dim=2, n=700, seed=5,
                      periodic=[1, 1, 0]))
    cases.append(dict(name="periodic_y_d2", kind="lattice", dim=2, ds=0.04, jitter=0.3, seed=3,
                      periodic=[0, 1, 0]))
    cases.append(dict(name="periodic_xyz_d3", kind="random", dim=3, n=900, seed=8,
                      periodic=[1, 1, 1]))
    cases.append(dict(name="periodic_z_d3", kind="lattice", dim=3, ds=0.1, jitter=0.25, seed=4,
                      periodic=[0, 0, 1]))
    cases.append(dict(name="periodic_x_d1", kind="random", dim=1, n=200, seed=6,
                      periodic=[1, 0, 0]))
    cases.append(dict(name="box_d2", kind="random", dim=2, n=600, seed=21,
                      lo=[-0.5, 0.25, 0.0], hi=[1.5, 1.0, 1.0]))
    cases.append(dict(name="box_d3", kind="lattice", dim=3, ds=0.05, jitter=0.2, seed=22,
                      lo=[0.0, 0.0, 0.0], hi=[1.0, 0.5, 0.35]))
    cases.append(dict(name="lattice_exact_d2", kind="lattice", dim=2, ds=0.05, jitter=0.0, seed=1))
    cases.append(dict(name="lattice_exact_d3", kind="lattice", dim=3, ds=0.1, jitter=0.0, seed=1))
    cases.append(dict(name="single", kind="arrays", dim=2, ds=0.1, x=[[0.5], [0.5]]))
    cases.append(dict(name="collinear_d1", kind="arrays", dim=1, ds=0.1, x=[[0.4, 0.5, 0.6]]))
    # clustered: dense blob + sparse background (long rows, empty cells)
    rs = np.random.default_rng(77)
    blob = 0.5 + 0.03 * rs.standard_normal((2, 400))
    back = rs.random((2, 200))
    xy = np.clip(np.concatenate([blob, back], axis=1), 0.0, 1.0)
    cases.append(dict(name="cluster_d2", kind="arrays", dim=2, ds=0.02, x=xy.tolist()))
    blob3 = np.clip(0.4 + 0.07 * rs.standard_normal((3, 500)), 0.0, 1.0)
    cases.append(dict(name="cluster_d3", kind="arrays", dim=3, ds=0.05, x=blob3.tolist()))
    return cases


def build_case(c):
    lo = c.get("lo", [0.0, 0.0, 0.0])
    hi = c.get("hi", [1.0, 1.0, 1.0])
    if c["kind"] == "random":
        r = O.RefSystem.random(c["dim"], c["n"], c["seed"], lo, hi)
    elif c["kind"] == "lattice":
        r = O.RefSystem.lattice(c["dim"], c["ds"], c["jitter"], c["seed"], lo, hi)
    else:
        r = O.RefSystem.from_arrays([np.array(a) for a in c["x"]], c["ds"], lo, hi)
    r.make_grid(periodic=c.get("periodic", [0, 0, 0]))
    return r, lo, hi


def main():
    goldens = {"hash": "FNV-1a 64: x=1469598103934665603; for o in offsets: x^=u64(o), "
                       "x*=1099511628211; for j in items: x^=u32(j), x*=1099511628211",
               "generator": "reference sphx built in place by oracle/Makefile (oracle/_ref)",
               "configs": config_goldens()}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(goldens, f, indent=1)

    arrays = {}
    index = []
    for k, c in enumerate(small_cases()):
        r, lo, hi = build_case(c)
        key = f"c{k}"
        meta = dict(c)
        meta.pop("x", None)
        meta.update(key=key, lo=lo, hi=hi, n=r.n, h=r.h, grid=r.grid_desc(),
                    periodic=c.get("periodic", [0, 0, 0]))
        for d, xd in enumerate(r.positions()):
            arrays[f"{key}_x{d}"] = xd
        rel, cell = r.rel_coords()
        for d in range(c["dim"]):
            arrays[f"{key}_rel{d}"] = rel[d]
            arrays[f"{key}_cell{d}"] = cell[d]
        arrays[f"{key}_items"] = r.items()
        arrays[f"{key}_start"] = r.cell_start()
        arrays[f"{key}_cellof"] = r.cell_of()
        meta["tables"] = {}
        for p in PRECS:
            for be in ("rcll", "cll", "all"):
                t = {"rcll": r.rcll, "cll": r.cll, "all": r.all_list}[be](p)
                tk = f"{be}_{O.PREC_NAMES[p]}"
                arrays[f"{key}_{tk}_off"] = t.offsets
                arrays[f"{key}_{tk}_items"] = t.items
                meta["tables"][tk] = table_summary(t)
        index.append(meta)
        print(key, c["name"], r.n, meta["tables"]["rcll_fp16"], flush=True)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
