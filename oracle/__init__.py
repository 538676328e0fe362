"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

* ``ref``    -- the unmodified reference sphx NNPS path, compiled in place from
               /root/reference/proj by ``oracle/Makefile`` into ``oracle/_ref``.
* ``oracle`` -- our plain-C restatement (``oracle/sphx_oracle.c``) in
               ``oracle/_build``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline -- never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsphx_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SRC = "/root/reference/proj"

FP64, FP32, FP16 = 0, 1, 2
PREC_NAMES = {FP64: "fp64", FP32: "fp32", FP16: "fp16"}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Build the checkers (the reference one only where its sources exist)."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets += ["ref", "dropin"]
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def fnv_hash(offsets: np.ndarray, items: np.ndarray) -> int:
    """Table hash used by the golden vectors: FNV-1a 64 over
    offsets (as u64) then items (as u32)."""
    x = 1469598103934665603
    mask = (1 << 64) - 1
    # vectorised FNV is not associative; do it in C via the oracle library
    lib = _oracle_lib()
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    it = np.ascontiguousarray(items, dtype=np.int32)
    t = _SoTable(int(len(o) - 1), int(len(it)), o.ctypes.data_as(C.POINTER(C.c_int64)),
                 it.ctypes.data_as(C.POINTER(C.c_int32)))
    x = lib.so_table_hash(C.byref(t)) & mask
    return int(x)


# --------------------------------------------------------------------------------------
# Reference library
# --------------------------------------------------------------------------------------
_ref = None
_dropin = None
DROPIN_SO = os.path.join(HERE, "_ref", "libsphx_dropin.so")


def dropin_lib():
    """The reference library with its nnps.cpp replaced by our drop-in
    (paper_2401_08586_b200/csrc/host/nnps_cuda.cpp): same ctypes face as ref_lib()."""
    global _dropin
    if _dropin is None:
        _dropin = _bind_ref(C.CDLL(DROPIN_SO))
    return _dropin


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        _ref = _bind_ref(C.CDLL(REF_SO))
    return _ref


def _bind_ref(lib):
    if True:
        vp = C.c_void_p
        d3 = C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_batch_kernels_available": (C.c_int, []),
            "ref_set_threads": (None, [C.c_int]),
            "ref_max_threads": (C.c_int, []),
            "ref_f16_from_f64": (C.c_uint16, [C.c_double]),
            "ref_f16_to_f64": (C.c_double, [C.c_uint16]),
            "ref_round_to": (C.c_double, [C.c_int, C.c_double]),
            "ref_sqrt16": (C.c_uint16, [C.c_uint16]),
            "ref_ps_lattice": (vp, [C.c_int, d3, d3, C.c_double, C.c_double, C.c_uint64]),
            "ref_ps_random": (vp, [C.c_int, d3, d3, C.c_uint64, C.c_uint64]),
            "ref_ps_from_arrays": (vp, [C.c_int, d3, d3, C.c_double, C.c_uint64, vp, vp, vp]),
            "ref_ps_size": (C.c_uint64, [vp]),
            "ref_ps_h": (C.c_double, [vp]),
            "ref_ps_set_h": (None, [vp, C.c_double]),
            "ref_ps_get_x": (None, [vp, C.c_int, _f64p]),
            "ref_ps_set_x": (None, [vp, C.c_int, _f64p]),
            "ref_ps_spatial_sort": (None, [vp, vp]),
            "ref_free_ps": (None, [vp]),
            "ref_grid_make": (vp, [vp, C.POINTER(C.c_int)]),
            "ref_grid_desc": (None, [vp, C.POINTER(C.c_int), d3]),
            "ref_grid_cell_total": (C.c_int64, [vp]),
            "ref_grid_rebin": (C.c_int, [vp, vp]),
            "ref_grid_items_size": (C.c_uint64, [vp]),
            "ref_grid_items": (None, [vp, _i32p]),
            "ref_grid_cell_start": (None, [vp, _i32p]),
            "ref_grid_cell_of": (None, [vp, C.c_uint64, _i32p]),
            "ref_grid_locate": (None, [vp, d3, C.POINTER(C.c_int32), d3]),
            "ref_free_grid": (None, [vp]),
            "ref_rel_build": (vp, [vp, vp]),
            "ref_rel_get": (None, [vp, C.c_int, vp, vp]),
            "ref_rel_distance": (C.c_double, [vp, vp, C.c_uint64, C.c_uint64, C.c_int]),
            "ref_free_rel": (None, [vp]),
            "ref_rcll": (vp, [vp, vp, C.c_int]),
            "ref_cll": (vp, [vp, vp, C.c_int]),
            "ref_all_list": (vp, [vp, C.c_int]),
            "ref_table_size": (C.c_uint64, [vp]),
            "ref_table_total": (C.c_int64, [vp]),
            "ref_table_radius": (C.c_double, [vp]),
            "ref_table_copy": (None, [vp, vp, vp]),
            "ref_table_hash": (C.c_uint64, [vp]),
            "ref_free_table": (None, [vp]),
            "ref_grad_normalized": (C.c_int64, [vp, vp, vp, C.c_double, vp, vp, vp]),
            "ref_update_relative": (C.c_int64, [vp, vp, C.c_uint64, vp, vp, vp, C.c_int]),
            "ref_time_nnps": (C.c_double, [C.c_int, vp, vp, vp, C.c_int, C.c_int]),
            "ref_mixed_new": (vp, [vp, C.POINTER(C.c_int), C.c_int]),
            "ref_mixed_free": (None, [vp]),
            "ref_mixed_get": (None, [vp, C.c_int, C.c_int, vp]),
            "ref_mixed_set": (None, [vp, C.c_int, C.c_int, vp]),
            "ref_mixed_grid": (None, [vp, vp, vp, vp]),
            "ref_mixed_step": (C.c_int, [vp, d3, d3, C.c_uint64, C.c_int, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
            "ref_mixed_table": (None, [vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
    return lib


def _d3(v):
    a = (C.c_double * 3)(*[float(x) for x in v])
    return a


class RefError(RuntimeError):
    pass


@dataclass
class Table:
    offsets: np.ndarray
    items: np.ndarray
    radius: float = 0.0

    @property
    def total(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def row(self, i: int) -> np.ndarray:
        return self.items[self.offsets[i]:self.offsets[i + 1]]

    def hash(self) -> int:
        return fnv_hash(self.offsets, self.items)


def _ref_table(ptr, lib=None) -> Table:
    lib = lib or ref_lib()
    if not ptr:
        raise RefError(lib.ref_last_error().decode())
    n = lib.ref_table_size(ptr)
    tot = lib.ref_table_total(ptr)
    off = np.empty(n + 1, np.int64)
    it = np.empty(max(tot, 1), np.int32)
    lib.ref_table_copy(ptr, off.ctypes.data, it.ctypes.data)
    rad = lib.ref_table_radius(ptr)
    lib.ref_free_table(ptr)
    return Table(off, it[:tot], rad)


class RefSystem:
    """A reference ParticleSystem + CellGrid + RelCoords triple."""

    def __init__(self, ps_ptr, dim: int, lib=None):
        self.lib = lib or ref_lib()
        if not ps_ptr:
            raise RefError(self.lib.ref_last_error().decode())
        self.ps = ps_ptr
        self.dim = dim
        self.grid = None
        self.rel = None

    # constructors (lib=dropin_lib() drives the reference with our NNPS) -----------
    @classmethod
    def lattice(cls, dim, ds, jitter, seed, lo=(0, 0, 0), hi=(1, 1, 1), lib=None):
        lib = lib or ref_lib()
        return cls(lib.ref_ps_lattice(dim, _d3(lo), _d3(hi), ds, jitter, seed), dim, lib)

    @classmethod
    def random(cls, dim, n, seed, lo=(0, 0, 0), hi=(1, 1, 1), lib=None):
        lib = lib or ref_lib()
        return cls(lib.ref_ps_random(dim, _d3(lo), _d3(hi), n, seed), dim, lib)

    @classmethod
    def from_arrays(cls, x, ds, lo=(0, 0, 0), hi=(1, 1, 1), h=None, lib=None):
        lib = lib or ref_lib()
        dim = len(x)
        xs = [np.ascontiguousarray(a, np.float64) for a in x]
        ptrs = [a.ctypes.data for a in xs] + [None] * (3 - dim)
        n = len(xs[0])
        self = cls(lib.ref_ps_from_arrays(dim, _d3(lo), _d3(hi), ds, n, *ptrs), dim, lib)
        if h is not None:
            lib.ref_ps_set_h(self.ps, h)
        return self

    def __del__(self):
        try:
            if self.rel:
                self.lib.ref_free_rel(self.rel)
            if self.grid:
                self.lib.ref_free_grid(self.grid)
            if self.ps:
                self.lib.ref_free_ps(self.ps)
        except Exception:
            pass

    # state -------------------------------------------------------------------------
    @property
    def n(self) -> int:
        return int(self.lib.ref_ps_size(self.ps))

    @property
    def h(self) -> float:
        return float(self.lib.ref_ps_h(self.ps))

    def x(self, k: int) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        self.lib.ref_ps_get_x(self.ps, k, out)
        return out

    def positions(self):
        return [self.x(k) for k in range(self.dim)]

    def spatial_sort(self) -> np.ndarray:
        perm = np.empty(self.n, np.uint32)
        self.lib.ref_ps_spatial_sort(self.ps, perm.ctypes.data)
        return perm

    def make_grid(self, periodic=(False, False, False), rebin=True, rel=True):
        if self.grid:
            self.lib.ref_free_grid(self.grid)
        p = (C.c_int * 3)(*[int(bool(v)) for v in periodic])
        self.grid = self.lib.ref_grid_make(self.ps, p)
        if not self.grid:
            raise RefError(self.lib.ref_last_error().decode())
        if rebin:
            rc = self.lib.ref_grid_rebin(self.grid, self.ps)
            if rc != 0:
                raise RefError(self.lib.ref_last_error().decode())
        if rel:
            self.rel = self.lib.ref_rel_build(self.ps, self.grid)
        return self

    def grid_desc(self) -> dict:
        ints = (C.c_int * 7)()
        d = (C.c_double * 14)()
        self.lib.ref_grid_desc(self.grid, ints, d)
        return {
            "dim": ints[0], "counts": list(ints[1:4]), "periodic": list(ints[4:7]),
            "hc": list(d[0:3]), "cutoff_norm": d[3], "radius": d[4], "span": list(d[5:8]),
            "origin": list(d[8:11]), "edge": list(d[11:14]),
        }

    def cell_total(self) -> int:
        return int(self.lib.ref_grid_cell_total(self.grid))

    def items(self) -> np.ndarray:
        out = np.empty(self.lib.ref_grid_items_size(self.grid), np.int32)
        self.lib.ref_grid_items(self.grid, out)
        return out

    def cell_start(self) -> np.ndarray:
        out = np.empty(self.cell_total() + 1, np.int32)
        self.lib.ref_grid_cell_start(self.grid, out)
        return out

    def cell_of(self) -> np.ndarray:
        out = np.empty(self.n, np.int32)
        self.lib.ref_grid_cell_of(self.grid, self.n, out)
        return out

    def rel_coords(self):
        rel, cell = [], []
        for k in range(self.dim):
            r = np.empty(self.n, np.float64)
            c = np.empty(self.n, np.int32)
            self.lib.ref_rel_get(self.rel, k, r.ctypes.data, c.ctypes.data)
            rel.append(r)
            cell.append(c)
        return rel, cell

    def rel_distance(self, i, j, prec) -> float:
        return float(self.lib.ref_rel_distance(self.rel, self.grid, i, j, prec))

    # backends ----------------------------------------------------------------------
    def update_relative(self, dx, prec):
        """update_relative(rel, i, dx[:, i], grid, prec) for every particle in index
        order (cell_grid.cpp:180-212); returns 0 or 1 + the particle that threw."""
        dx = [np.ascontiguousarray(a, np.float64) for a in dx]
        ptrs = [a.ctypes.data for a in dx] + [None] * (3 - len(dx))
        return int(self.lib.ref_update_relative(self.rel, self.grid, self.n, *ptrs, prec))

    def grad_normalized_rcll(self, prec, f, h):
        """The reference's mixed step core: grad_normalized(f, ps, rcll(rel, grid, prec),
        make_kernel(h, dim)) (dynamics.cpp:145-155, gradient.cpp:44-82)."""
        t = self.lib.ref_rcll(self.rel, self.grid, prec)
        if not t:
            raise RefError(self.lib.ref_last_error().decode())
        f = np.ascontiguousarray(f, np.float64)
        g = [np.zeros(self.n, np.float64) for _ in range(3)]
        deg = self.lib.ref_grad_normalized(self.ps, t, f.ctypes.data, h,
                                           *[a.ctypes.data for a in g])
        self.lib.ref_free_table(t)
        return g[:self.dim], int(deg)

    def rcll(self, prec) -> Table:
        return _ref_table(self.lib.ref_rcll(self.rel, self.grid, prec), self.lib)

    def cll(self, prec) -> Table:
        return _ref_table(self.lib.ref_cll(self.ps, self.grid, prec), self.lib)

    def all_list(self, prec) -> Table:
        return _ref_table(self.lib.ref_all_list(self.ps, prec), self.lib)

    def time_nnps(self, backend: str, prec: int, repeats: int = 5) -> float:
        which = 0 if backend == "rcll" else 1
        return float(self.lib.ref_time_nnps(which, self.ps, self.rel, self.grid, prec, repeats))


class RefMixed:
    """The reference's MixedState (dynamics.hpp:71-82) and step_mixed
    (dynamics.cpp:136-203), through the compiled reference library."""

    FIELDS = {"x": 0, "v": 1, "rho": 2, "p": 3, "e": 4, "m": 5, "rel": 6}

    def __init__(self, system: "RefSystem", periodic, approach: int):
        self.lib = system.lib
        per = (C.c_int * 3)(*[int(bool(p)) for p in list(periodic) + [0] * 3][:3])
        self.st = self.lib.ref_mixed_new(system.ps, per, approach)
        if not self.st:
            raise RefError(self.lib.ref_last_error().decode())
        self.n, self.dim = system.n, system.dim

    def __del__(self):
        try:
            if self.st:
                self.lib.ref_mixed_free(self.st)
        except Exception:
            pass

    def get(self, name: str, k: int = 0) -> np.ndarray:
        if name == "cell":
            out = np.empty(self.n, np.int32)
            self.lib.ref_mixed_get(self.st, 7, k, out.ctypes.data)
            return out
        out = np.empty(self.n, np.float64)
        self.lib.ref_mixed_get(self.st, self.FIELDS[name], k, out.ctypes.data)
        return out

    def set(self, name: str, k: int, values) -> None:
        a = np.ascontiguousarray(values, np.float64)
        assert a.size == self.n
        self.lib.ref_mixed_set(self.st, self.FIELDS[name], k, a.ctypes.data)

    def grid_members(self, cells: int):
        cell_of = np.empty(self.n, np.int32)
        start = np.empty(cells + 1, np.int32)
        items = np.empty(self.n, np.int32)
        self.lib.ref_mixed_grid(self.st, cell_of.ctypes.data, start.ctypes.data, items.ctypes.data)
        return cell_of, start, items

    def step(self, dt, c_sound, rho0=1.0, mu=0.0, body_force=(0, 0, 0), n_moving=0,
             evolve_density=True, compute_energy=False):
        """One step_mixed; returns (max_dx, table total). Raises RefError with the
        reference's message when it throws."""
        mx = C.c_double()
        tot = C.c_int64()
        rc = self.lib.ref_mixed_step(self.st, (C.c_double * 4)(dt, c_sound, rho0, mu),
                                     _d3(list(body_force) + [0] * (3 - len(body_force))),
                                     n_moving, int(evolve_density), int(compute_energy),
                                     C.byref(mx), C.byref(tot))
        if rc != 0:
            raise RefError(self.lib.ref_last_error().decode())
        return mx.value, tot.value

    def table(self, total: int):
        off = np.empty(self.n + 1, np.int64)
        it = np.empty(total, np.int32)
        self.lib.ref_mixed_table(self.st, off.ctypes.data, it.ctypes.data)
        return off, it


# --------------------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------------------
class _SoTable(C.Structure):
    _fields_ = [("n", C.c_int64), ("total", C.c_int64),
                ("offsets", C.POINTER(C.c_int64)), ("items", C.POINTER(C.c_int32))]


class SoGrid(C.Structure):
    _fields_ = [("dim", C.c_int), ("counts", C.c_int * 3), ("periodic", C.c_int * 3),
                ("total", C.c_int64), ("radius", C.c_double), ("cutoff_norm", C.c_double),
                ("hd", C.c_double), ("edge", C.c_double * 3), ("hc", C.c_double * 3),
                ("origin", C.c_double * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3)]


_oracle = None


def _oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        vp = C.c_void_p
        d3 = C.POINTER(C.c_double)
        sig = {
            "so_f16_from_f64": (C.c_uint16, [C.c_double]),
            "so_f16_to_f64": (C.c_double, [C.c_uint16]),
            "so_round_to": (C.c_double, [C.c_int, C.c_double]),
            "so_lattice_count": (C.c_int64, [C.c_int, d3, d3, C.c_double]),
            "so_build_gapped_random": (C.c_int, [d3, d3, C.c_int64, C.c_double, C.c_double,
                                                 C.c_uint64, vp, vp]),
            "so_build_lattice": (C.c_int, [C.c_int, d3, d3, C.c_double, C.c_double, C.c_uint64,
                                           vp, vp, vp]),
            "so_build_random": (C.c_double, [C.c_int, d3, d3, C.c_int64, C.c_uint64, vp, vp, vp]),
            "so_grid_init": (C.c_int, [C.POINTER(SoGrid), C.c_int, d3, d3, C.c_double,
                                       C.POINTER(C.c_int)]),
            "so_locate": (None, [C.POINTER(SoGrid), d3, C.POINTER(C.c_int32), d3]),
            "so_rebin": (C.c_int, [C.POINTER(SoGrid), C.c_int64, C.POINTER(vp), _i32p, _i32p,
                                   _i32p, C.POINTER(C.c_int64)]),
            "so_build_rel": (None, [C.POINTER(SoGrid), C.c_int64, C.POINTER(vp), C.POINTER(vp),
                                    C.POINTER(vp), _i32p, _i32p, _i32p]),
            "so_rcll": (C.c_int, [C.POINTER(SoGrid), C.c_int64, C.POINTER(vp), C.POINTER(vp),
                                  _i32p, _i32p, C.c_int, C.POINTER(_SoTable)]),
            "so_cll": (C.c_int, [C.POINTER(SoGrid), C.c_int64, C.POINTER(vp), C.c_double, _i32p,
                                 _i32p, _i32p, C.c_int, C.POINTER(_SoTable)]),
            "so_all_list": (C.c_int, [C.c_int, C.c_int64, C.POINTER(vp), C.c_double, C.c_int,
                                      C.POINTER(_SoTable)]),
            "so_rel_distance": (C.c_double, [C.POINTER(SoGrid), C.POINTER(vp), C.POINTER(vp),
                                             C.c_int64, C.c_int64, C.c_int]),
            "so_table_free": (None, [C.POINTER(_SoTable)]),
            "so_update_relative": (C.c_int64, [C.POINTER(SoGrid), C.c_int64, C.POINTER(vp),
                                               C.POINTER(vp), C.POINTER(vp), C.c_int]),
            "so_grad_normalized": (C.c_int64, [C.c_int, C.c_int64, C.POINTER(vp), vp, vp, vp,
                                               C.c_double, C.POINTER(vp)]),
            "so_table_hash": (C.c_uint64, [C.POINTER(_SoTable)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _oracle = lib
    return _oracle


def _ptrs(arrs):
    a = (C.c_void_p * 3)(*([x.ctypes.data for x in arrs] + [None] * (3 - len(arrs))))
    return a


def _take_table(t: _SoTable) -> Table:
    lib = _oracle_lib()
    off = np.ctypeslib.as_array(t.offsets, shape=(t.n + 1,)).copy()
    it = (np.ctypeslib.as_array(t.items, shape=(t.total,)).copy() if t.total
          else np.empty(0, np.int32))
    lib.so_table_free(C.byref(t))
    return Table(off, it)


class Oracle:
    """Plain-C restatement driven from numpy arrays (all in particle order)."""

    def __init__(self):
        self.lib = _oracle_lib()

    def round_to(self, prec, x):
        return self.lib.so_round_to(prec, x)

    def f16_bits(self, x):
        return self.lib.so_f16_from_f64(x)

    def lattice(self, dim, ds, jitter, seed, lo=(0, 0, 0), hi=(1, 1, 1)):
        n = self.lib.so_lattice_count(dim, _d3(lo), _d3(hi), ds)
        xs = [np.empty(n, np.float64) for _ in range(dim)]
        rc = self.lib.so_build_lattice(dim, _d3(lo), _d3(hi), ds, jitter, seed,
                                       *([x.ctypes.data for x in xs] + [None] * (3 - dim)))
        if rc != 0:
            raise ValueError("invalid lattice parameters")
        return xs

    def gapped_random(self, n, cutoff, width, seed, lo=(0, 0, 0), hi=(1, 1, 1)):
        """build_gapped_random (experiments.cpp:55-112) positions, 2-D."""
        xs = [np.empty(n, np.float64) for _ in range(2)]
        rc = self.lib.so_build_gapped_random(_d3(lo), _d3(hi), n, cutoff, width, seed,
                                             xs[0].ctypes.data, xs[1].ctypes.data)
        if rc != 0:
            raise RuntimeError("guard-annulus sampling stalled; widen the budget")
        return xs

    def random(self, dim, n, seed, lo=(0, 0, 0), hi=(1, 1, 1)):
        xs = [np.empty(n, np.float64) for _ in range(dim)]
        ds = self.lib.so_build_random(dim, _d3(lo), _d3(hi), n, seed,
                                      *([x.ctypes.data for x in xs] + [None] * (3 - dim)))
        return xs, ds

    def grid(self, dim, radius, lo=(0, 0, 0), hi=(1, 1, 1), periodic=(0, 0, 0)) -> SoGrid:
        g = SoGrid()
        p = (C.c_int * 3)(*[int(bool(v)) for v in periodic])
        if self.lib.so_grid_init(C.byref(g), dim, _d3(lo), _d3(hi), radius, p) != 0:
            raise ValueError("invalid grid")
        return g

    def rebin(self, g: SoGrid, x):
        n = len(x[0])
        cell_of = np.empty(n, np.int32)
        start = np.empty(g.total + 1, np.int32)
        items = np.empty(max(n, 1), np.int32)
        bad = C.c_int64(-1)
        xs = [np.ascontiguousarray(a, np.float64) for a in x]
        rc = self.lib.so_rebin(C.byref(g), n, _ptrs(xs), cell_of, start, items, C.byref(bad))
        if rc != 0:
            raise IndexError(f"particle {bad.value} lies outside the grid")
        return cell_of, start, items[:n]

    def build_rel(self, g: SoGrid, x):
        n = len(x[0])
        xs = [np.ascontiguousarray(a, np.float64) for a in x]
        rel = [np.empty(n, np.float64) for _ in range(g.dim)]
        cell = [np.empty(n, np.int32) for _ in range(g.dim)]
        cell_of = np.empty(n, np.int32)
        start = np.empty(g.total + 1, np.int32)
        items = np.empty(max(n, 1), np.int32)
        self.lib.so_build_rel(C.byref(g), n, _ptrs(xs), _ptrs(rel), _ptrs(cell), cell_of,
                              start, items)
        return rel, cell, cell_of, start, items[:n]

    def rcll(self, g: SoGrid, rel, cell, items, start, prec) -> Table:
        t = _SoTable()
        rel = [np.ascontiguousarray(a, np.float64) for a in rel]
        cell = [np.ascontiguousarray(a, np.int32) for a in cell]
        self.lib.so_rcll(C.byref(g), len(rel[0]), _ptrs(rel), _ptrs(cell),
                         np.ascontiguousarray(items, np.int32),
                         np.ascontiguousarray(start, np.int32), prec, C.byref(t))
        return _take_table(t)

    def cll(self, g: SoGrid, x, h, cell_of, items, start, prec) -> Table:
        t = _SoTable()
        xs = [np.ascontiguousarray(a, np.float64) for a in x]
        self.lib.so_cll(C.byref(g), len(xs[0]), _ptrs(xs), h,
                        np.ascontiguousarray(cell_of, np.int32),
                        np.ascontiguousarray(items, np.int32),
                        np.ascontiguousarray(start, np.int32), prec, C.byref(t))
        return _take_table(t)

    def all_list(self, x, h, prec) -> Table:
        t = _SoTable()
        xs = [np.ascontiguousarray(a, np.float64) for a in x]
        if self.lib.so_all_list(len(xs), len(xs[0]), _ptrs(xs), h, prec, C.byref(t)) != 0:
            raise ValueError("all_list needs at least one particle")
        return _take_table(t)

    def update_relative(self, g: SoGrid, rel, cell, dx, prec) -> int:
        """In place on rel/cell (numpy); 0 or 1 + ((i << 3) | (axis << 1) | kind)."""
        dx = [np.ascontiguousarray(a, np.float64) for a in dx]
        return int(self.lib.so_update_relative(C.byref(g), len(rel[0]), _ptrs(rel), _ptrs(cell),
                                               _ptrs(dx), prec))

    def grad_normalized(self, dim, x, f, offsets, items, h):
        """grad_normalized on a table (gradient.cpp:44-82): (g[dim], degenerate)."""
        n = len(offsets) - 1
        x = [np.ascontiguousarray(a, np.float64) for a in x]
        f = np.ascontiguousarray(f, np.float64)
        off = np.ascontiguousarray(offsets, np.int64)
        it = np.ascontiguousarray(items, np.int32)
        g = [np.zeros(n, np.float64) for _ in range(dim)]
        gp = (C.c_void_p * 3)(*([a.ctypes.data for a in g] + [None] * (3 - dim)))
        deg = self.lib.so_grad_normalized(dim, n, _ptrs(x), f.ctypes.data, off.ctypes.data,
                                          it.ctypes.data, h, gp)
        return g, int(deg)

    def rel_distance(self, g: SoGrid, rel, cell, i, j, prec) -> float:
        rel = [np.ascontiguousarray(a, np.float64) for a in rel]
        cell = [np.ascontiguousarray(a, np.int32) for a in cell]
        return self.lib.so_rel_distance(C.byref(g), _ptrs(rel), _ptrs(cell), i, j, prec)
