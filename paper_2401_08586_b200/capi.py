"""ctypes binding of the C ABI (include/sphx_cuda.h) -> lib/libsphx_cuda.so.

This is the Python-side view of the drop-in boundary. There is no CPU path:
if the library or an sm_100 device is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPHX_CUDA_LIB") or os.path.join(PKG, "lib", "libsphx_cuda.so")

FP64, FP32, FP16 = 0, 1, 2
PRECISIONS = {"fp64": FP64, "fp32": FP32, "fp16": FP16}

OK = 0
ERR_GENERIC, ERR_INVALID_ARGUMENT, ERR_OUT_OF_RANGE = -1, -2, -3
ERR_RUNTIME, ERR_CUDA, ERR_CAPACITY = -4, -5, -6


class SphxCudaError(RuntimeError):
    """CUDA / device failure (SPHX_ERR_CUDA)."""


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("counts", C.c_int32 * 3), ("periodic", C.c_int32 * 3),
                ("reserved", C.c_int32), ("hc", C.c_double * 3), ("origin", C.c_double * 3),
                ("cutoff_norm", C.c_double), ("radius_phys", C.c_double),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3)]

    @property
    def cell_total(self) -> int:
        t = 1
        for k in range(self.dim):
            t *= self.counts[k]
        return t

    def as_dict(self) -> dict:
        return {"dim": self.dim, "counts": list(self.counts), "periodic": list(self.periodic),
                "hc": list(self.hc), "origin": list(self.origin), "cutoff_norm": self.cutoff_norm,
                "radius_phys": self.radius_phys, "lo": list(self.lo), "hi": list(self.hi)}


_lib = None
# int sink(void* user, int32_t part, const void* data, int64_t bytes)  (sphx_cuda.h)
TABLE_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64)


def lib():
    """Load libsphx_cuda.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the NNPS path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    p3 = C.c_void_p * 3
    G = C.POINTER(GridDesc)
    sigs = {
        "sphx_last_error": (C.c_char_p, []),
        "sphx_grid_init": (C.c_int, [G, i32, C.POINTER(dbl), C.POINTER(dbl), dbl, C.POINTER(i32)]),
        "sphx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "sphx_destroy": (None, [vp]),
        "sphx_set_stream": (C.c_int, [vp, vp]),
        "sphx_launch_count": (i64, [vp]),
        "sphx_rcll": (C.c_int, [vp, G, i64, p3, p3, i64, vp, vp, i32, C.POINTER(i64)]),
        "sphx_cell_link_list": (C.c_int, [vp, G, i64, p3, dbl, i64, vp, vp, vp, i32,
                                          C.POINTER(i64)]),
        "sphx_all_list": (C.c_int, [vp, i32, i64, p3, dbl, i32, C.POINTER(i64)]),
        "sphx_table_copy": (C.c_int, [vp, vp, vp]),
        "sphx_table_stream": (C.c_int, [vp, TABLE_SINK, vp]),
        "sphx_rebin": (C.c_int, [vp, G, i64, p3, vp, vp, vp]),
        "sphx_build_rel_coords": (C.c_int, [vp, G, i64, p3, p3, p3, vp, vp, vp]),
        "sphx_rebuild_members": (C.c_int, [vp, G, i64, p3, vp, vp, vp]),
        "sphx_rcll_device": (C.c_int, [vp, G, i64, p3, p3, vp, vp, i32, vp, vp, i64]),
        "sphx_cell_link_list_device": (C.c_int, [vp, G, i64, p3, dbl, vp, vp, vp, i32, vp, vp,
                                                 i64]),
        "sphx_build_rel_coords_device": (C.c_int, [vp, G, i64, p3, p3, p3, vp, vp, vp]),
        "sphx_rebin_device": (C.c_int, [vp, G, i64, p3, vp, vp, vp, vp]),
        "sphx_enable_timing": (C.c_int, [vp, C.c_int]),
        "sphx_build_lattice": (C.c_int, [i32, C.POINTER(dbl), C.POINTER(dbl), dbl, dbl,
                                         C.c_uint64, C.POINTER(i64), vp, vp, vp]),
        "sphx_build_random_uniform": (C.c_int, [i32, C.POINTER(dbl), C.POINTER(dbl), i64,
                                                C.c_uint64, C.POINTER(dbl), vp, vp, vp]),
        "sphx_last_timing": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "sphx_table_hash": (C.c_uint64, [vp, i64, vp, i64]),
        "sphx_build_rel_coords_window_device": (C.c_int, [vp, G, G, i32, i32, i64, p3, p3, p3,
                                                          vp, vp, vp]),
        "sphx_rcll_rows_device": (C.c_int, [vp, G, i64, p3, p3, vp, vp, i32, vp, i64, i64, vp,
                                            vp, i64]),
        "sphx_lattice_device": (C.c_int, [vp, i32, C.POINTER(dbl), C.POINTER(dbl), dbl, i64, i64,
                                          p3]),
        "sphx_slab_assemble_device": (C.c_int, [vp, G, i32, i64, i64, i64, i64, vp, vp, vp, vp,
                                                vp, p3]),
        "sphx_rcll_distances_device": (C.c_int, [vp, G, i64, p3, p3, i32, vp, vp, vp]),
        "sphx_table_distances": (C.c_int, [vp, G, i32, vp]),
        "sphx_update_relative": (C.c_int, [vp, G, i64, p3, p3, p3, i32]),
        "sphx_update_relative_device": (C.c_int, [vp, G, i64, p3, p3, p3, i32, vp]),
        "sphx_rebuild_members_device": (C.c_int, [vp, G, i64, p3, vp, vp, vp]),
        "sphx_rcll_grad_normalized": (C.c_int, [vp, G, i64, p3, p3, i64, vp, vp, i32, p3, vp, dbl,
                                                p3, C.POINTER(i64)]),
        "sphx_rcll_grad_normalized_device": (C.c_int, [vp, G, i64, p3, p3, vp, vp, i32, p3, vp,
                                                       dbl, p3, vp]),
        "sphx_step_mixed_device": (C.c_int, [vp, G, i32, C.POINTER(MixedStateDevice),
                                             C.POINTER(StepConfig), vp, vp, i64,
                                             C.POINTER(dbl), C.POINTER(i64)]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ("sphx_last_error", "sphx_grid_init", "sphx_create", "sphx_destroy",
            "sphx_set_stream", "sphx_launch_count", "sphx_rcll", "sphx_cell_link_list",
            "sphx_all_list", "sphx_table_copy", "sphx_table_stream", "sphx_rebin", "sphx_build_rel_coords",
            "sphx_rebuild_members", "sphx_rcll_device", "sphx_cell_link_list_device",
            "sphx_build_rel_coords_device", "sphx_rebin_device", "sphx_enable_timing",
            "sphx_last_timing", "sphx_build_lattice", "sphx_build_random_uniform",
            "sphx_table_hash", "sphx_build_rel_coords_window_device", "sphx_rcll_rows_device",
            "sphx_lattice_device", "sphx_rcll_distances_device", "sphx_table_distances",
            "sphx_rcll_grad_normalized", "sphx_rcll_grad_normalized_device",
            "sphx_update_relative", "sphx_update_relative_device", "sphx_rebuild_members_device",
            "sphx_step_mixed_device", "sphx_slab_assemble_device")

APPROACH_I, APPROACH_II, APPROACH_III = 0, 1, 2


class StepConfig(C.Structure):
    """sphx_step_config = StepConfig (dynamics.hpp:84-96) without pre_force."""
    _fields_ = [("dt", C.c_double), ("c_sound", C.c_double), ("rho0", C.c_double),
                ("mu", C.c_double), ("body_force", C.c_double * 3), ("n_moving", C.c_int64),
                ("evolve_density", C.c_int32), ("compute_energy", C.c_int32)]


class MixedStateDevice(C.Structure):
    """sphx_mixed_state_device = MixedState (dynamics.hpp:71-82) in device memory."""
    _fields_ = [("n", C.c_int64), ("h", C.c_double), ("x", C.c_void_p * 3),
                ("v", C.c_void_p * 3), ("m", C.c_void_p), ("rho", C.c_void_p),
                ("p", C.c_void_p), ("e", C.c_void_p), ("rel", C.c_void_p * 3),
                ("cell", C.c_void_p * 3), ("cell_of", C.c_void_p), ("cell_start", C.c_void_p),
                ("items", C.c_void_p)]


def table_hash(offsets: np.ndarray, items: np.ndarray) -> int:
    """FNV-1a 64 table digest (the golden-vector hash)."""
    o = np.ascontiguousarray(offsets, np.int64)
    it = np.ascontiguousarray(items, np.int32)
    return int(lib().sphx_table_hash(o.ctypes.data, len(o) - 1, it.ctypes.data, len(it)))


def check(rc: int) -> None:
    """Map a C-ABI status to the exception class the reference throws."""
    if rc == OK:
        return
    msg = lib().sphx_last_error().decode()
    if rc == ERR_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if rc == ERR_OUT_OF_RANGE:
        raise IndexError(msg)          # std::out_of_range
    if rc == ERR_CUDA:
        raise SphxCudaError(msg)
    raise RuntimeError(msg)            # std::runtime_error / generic


def _d3(v) -> "C.Array":
    v = list(v) + [0.0] * (3 - len(v))
    return (C.c_double * 3)(*[float(a) for a in v])


def grid_init(dim: int, lo, hi, radius: float, periodic=(0, 0, 0)) -> GridDesc:
    """CellGrid(Domain::box(dim, lo, hi), radius, periodic) as a descriptor."""
    g = GridDesc()
    p = (C.c_int32 * 3)(*[int(bool(x)) for x in list(periodic) + [0] * (3 - len(periodic))])
    check(lib().sphx_grid_init(C.byref(g), dim, _d3(lo), _d3(hi), float(radius), p))
    return g


def build_lattice(dim: int, ds: float, jitter: float, seed: int, lo=(0, 0, 0), hi=(1, 1, 1)):
    """ParticleSystem positions of build_lattice (particle_system.cpp:31-62)."""
    n = C.c_int64()
    check(lib().sphx_build_lattice(dim, _d3(lo), _d3(hi), ds, jitter, seed, C.byref(n),
                                   None, None, None))
    xs = [np.empty(n.value, np.float64) for _ in range(dim)]
    check(lib().sphx_build_lattice(dim, _d3(lo), _d3(hi), ds, jitter, seed, C.byref(n),
                                   *[x.ctypes.data for x in xs], *([None] * (3 - dim))))
    return xs


def build_random_uniform(dim: int, n: int, seed: int, lo=(0, 0, 0), hi=(1, 1, 1)):
    """Positions and ds of build_random_uniform (particle_system.cpp:64-77)."""
    xs = [np.empty(n, np.float64) for _ in range(dim)]
    ds = C.c_double()
    check(lib().sphx_build_random_uniform(dim, _d3(lo), _d3(hi), n, seed, C.byref(ds),
                                          *[x.ctypes.data for x in xs], *([None] * (3 - dim))))
    return xs, ds.value


def _ptr3(arrs):
    ptrs = [a.ctypes.data if a is not None else None for a in arrs] + [None] * (3 - len(arrs))
    return (C.c_void_p * 3)(*ptrs)


def _dptr3(tensors):
    ptrs = [t.data_ptr() if t is not None else None for t in tensors]
    ptrs += [None] * (3 - len(ptrs))
    return (C.c_void_p * 3)(*ptrs)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Context:
    """One sphx_context: a CUDA stream plus grow-only device buffers."""

    _last_total = 0

    def __init__(self, device: int = -1):
        h = C.c_void_p()
        check(lib().sphx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().sphx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().sphx_launch_count(self.h))

    def set_stream(self, stream_handle: int | None):
        """Pin the context to a CUDA stream (None: back to following torch)."""
        check(lib().sphx_set_stream(self.h, stream_handle))
        self._pinned = stream_handle is not None

    def _bind(self, t):
        """Device API calls are ordered on torch's current stream of the tensors'
        device unless a stream was pinned with set_stream()."""
        if getattr(self, "_pinned", False):
            return
        import torch
        # torch's default stream has handle 0, which the ABI reads as "own stream":
        # pass cudaStreamLegacy (0x1) for it instead
        h = torch.cuda.current_stream(t.device).cuda_stream or 0x1
        check(lib().sphx_set_stream(self.h, h))

    def enable_timing(self, on: bool = True):
        check(lib().sphx_enable_timing(self.h, int(on)))

    def last_timing(self):
        e, s = C.c_float(), C.c_float()
        check(lib().sphx_last_timing(self.h, C.byref(e), C.byref(s)))
        return e.value, s.value

    # ---- drop-in host API -------------------------------------------------------------
    def _fetch(self, n: int, total: int):
        off = np.empty(n + 1, np.int64)
        items = np.empty(max(total, 1), np.int32)
        check(lib().sphx_table_copy(self.h, off.ctypes.data, items.ctypes.data))
        return off, items[:total]

    def table_stream(self, sink):
        """sphx_table_stream: sink(part, bytes) gets the offsets (part 0) and then
        the items (part 1) chunk by chunk; a falsy/raising sink stops the copy."""
        def cb(_user, part, data, nbytes):
            try:
                return 0 if sink(part, C.string_at(data, nbytes)) is not False else 1
            except Exception:  # noqa: BLE001 - reported through the C ABI
                return 1
        fn = TABLE_SINK(cb)
        check(lib().sphx_table_stream(self.h, fn, None))

    def rcll(self, grid: GridDesc, rel, cell, items, cell_start, prec: int):
        rel = [_c64(a) for a in rel]
        cell = [_c32(a) for a in cell]
        items = _c32(items)
        cell_start = _c32(cell_start)
        n = len(rel[0]) if rel else 0
        tot = C.c_int64()
        check(lib().sphx_rcll(self.h, C.byref(grid), n, _ptr3(rel), _ptr3(cell), len(items),
                              items.ctypes.data, cell_start.ctypes.data, prec, C.byref(tot)))
        self._last_total = tot.value
        return self._fetch(n, tot.value)

    def update_relative(self, grid: GridDesc, rel, cell, dx, prec: int):
        """update_relative for every particle (host arrays are updated in place)."""
        for a in list(rel) + list(cell):
            assert a.flags["C_CONTIGUOUS"]
        dx = [_c64(a) for a in dx]
        check(lib().sphx_update_relative(self.h, C.byref(grid), len(rel[0]), _ptr3(rel),
                                         _ptr3(cell), _ptr3(dx), prec))

    def update_relative_device(self, grid, rel, cell, dx, prec, status):
        self._bind(status)
        check(lib().sphx_update_relative_device(self.h, C.byref(grid), rel[0].numel(), _dptr3(rel),
                                                _dptr3(cell), _dptr3(dx), prec,
                                                status.data_ptr()))

    def rebuild_members_device(self, grid, cell, cell_of, cell_start, items):
        self._bind(items)
        check(lib().sphx_rebuild_members_device(self.h, C.byref(grid), cell[0].numel(),
                                                _dptr3(cell), cell_of.data_ptr(),
                                                cell_start.data_ptr(), items.data_ptr()))

    def step_mixed_device(self, grid: GridDesc, approach: int, state: dict, cfg: dict,
                          offsets, items_out):
        """step_mixed (dynamics.cpp:136-203) on device tensors. `state` holds torch
        tensors x, v (lists per axis), m, rho, p, e, rel, cell (lists), cell_of,
        cell_start, items, and the float h; they are updated in place. Returns
        (max_dx, table total); the step's table is in offsets / items_out."""
        self._bind(state["rho"])
        st = MixedStateDevice()
        st.n = state["rho"].numel()
        st.h = float(state["h"])
        for k in range(3):
            for name in ("x", "v", "rel", "cell"):
                arr = state.get(name)
                getattr(st, name)[k] = arr[k].data_ptr() if arr is not None and k < len(arr) else None
        for name in ("m", "rho", "p", "e", "cell_of", "cell_start", "items"):
            setattr(st, name, state[name].data_ptr())
        c = StepConfig()
        c.dt, c.c_sound = float(cfg["dt"]), float(cfg["c_sound"])
        c.rho0, c.mu = float(cfg.get("rho0", 1.0)), float(cfg.get("mu", 0.0))
        bf = list(cfg.get("body_force", (0.0, 0.0, 0.0))) + [0.0] * 3
        for k in range(3):
            c.body_force[k] = float(bf[k])
        c.n_moving = int(cfg.get("n_moving", 0))
        c.evolve_density = int(bool(cfg.get("evolve_density", True)))
        c.compute_energy = int(bool(cfg.get("compute_energy", False)))
        mx = C.c_double()
        tot = C.c_int64()
        check(lib().sphx_step_mixed_device(self.h, C.byref(grid), approach, C.byref(st), C.byref(c),
                                           offsets.data_ptr(), items_out.data_ptr(),
                                           items_out.numel(), C.byref(mx), C.byref(tot)))
        return mx.value, tot.value

    def rcll_grad_normalized(self, grid: GridDesc, rel, cell, items, cell_start, prec: int, x, f,
                             h: float):
        """Fused grad_normalized(f, ps, rcll(rel, grid, prec), make_kernel(h, dim))."""
        rel = [_c64(a) for a in rel]
        cell = [_c32(a) for a in cell]
        x = [_c64(a) for a in x]
        f = _c64(f)
        items = _c32(items)
        cell_start = _c32(cell_start)
        n = len(rel[0])
        g = [np.empty(n, np.float64) for _ in range(len(rel))]
        deg = C.c_int64()
        check(lib().sphx_rcll_grad_normalized(self.h, C.byref(grid), n, _ptr3(rel), _ptr3(cell),
                                              len(items), items.ctypes.data, cell_start.ctypes.data,
                                              prec, _ptr3(x), f.ctypes.data, float(h), _ptr3(g),
                                              C.byref(deg)))
        return g, deg.value

    def rcll_grad_normalized_device(self, grid, rel, cell, items, cell_start, prec, x, f, h, g,
                                    deg):
        self._bind(f)
        check(lib().sphx_rcll_grad_normalized_device(
            self.h, C.byref(grid), rel[0].numel(), _dptr3(rel), _dptr3(cell), items.data_ptr(),
            cell_start.data_ptr(), prec, _dptr3(x), f.data_ptr(), float(h), _dptr3(g),
            deg.data_ptr()))

    def table_distances(self, grid: GridDesc, prec: int) -> np.ndarray:
        """Per-pair distances of the last rcll() table (rel_distance per entry)."""
        d = np.empty(max(self._last_total, 1), dtype=np.float64)
        check(lib().sphx_table_distances(self.h, C.byref(grid), prec, d.ctypes.data))
        return d[:self._last_total]

    def rcll_distances_device(self, grid, rel, cell, prec, offsets, items, dist):
        self._bind(offsets)
        check(lib().sphx_rcll_distances_device(self.h, C.byref(grid), rel[0].numel(), _dptr3(rel),
                                               _dptr3(cell), prec, offsets.data_ptr(),
                                               items.data_ptr(), dist.data_ptr()))

    def cell_link_list(self, grid: GridDesc, x, h: float, items, cell_start, cell_of, prec: int):
        x = [_c64(a) for a in x]
        items, cell_start, cell_of = _c32(items), _c32(cell_start), _c32(cell_of)
        n = len(x[0])
        tot = C.c_int64()
        check(lib().sphx_cell_link_list(self.h, C.byref(grid), n, _ptr3(x), float(h), len(items),
                                        items.ctypes.data, cell_start.ctypes.data,
                                        cell_of.ctypes.data, prec, C.byref(tot)))
        return self._fetch(n, tot.value)

    def all_list(self, x, h: float, prec: int):
        x = [_c64(a) for a in x]
        n = len(x[0])
        tot = C.c_int64()
        check(lib().sphx_all_list(self.h, len(x), n, _ptr3(x), float(h), prec, C.byref(tot)))
        return self._fetch(n, tot.value)

    def rebin(self, grid: GridDesc, x):
        x = [_c64(a) for a in x]
        n = len(x[0])
        cell_of = np.empty(max(n, 1), np.int32)
        start = np.empty(grid.cell_total + 1, np.int32)
        items = np.empty(max(n, 1), np.int32)
        check(lib().sphx_rebin(self.h, C.byref(grid), n, _ptr3(x), cell_of.ctypes.data,
                               start.ctypes.data, items.ctypes.data))
        return cell_of[:n], start, items[:n]

    def build_rel_coords(self, grid: GridDesc, x):
        x = [_c64(a) for a in x]
        n = len(x[0])
        d = grid.dim
        rel = [np.empty(max(n, 1), np.float64) for _ in range(d)]
        cell = [np.empty(max(n, 1), np.int32) for _ in range(d)]
        cell_of = np.empty(max(n, 1), np.int32)
        start = np.empty(grid.cell_total + 1, np.int32)
        items = np.empty(max(n, 1), np.int32)
        check(lib().sphx_build_rel_coords(self.h, C.byref(grid), n, _ptr3(x), _ptr3(rel),
                                          _ptr3(cell), cell_of.ctypes.data, start.ctypes.data,
                                          items.ctypes.data))
        return [r[:n] for r in rel], [c[:n] for c in cell], cell_of[:n], start, items[:n]

    def rebuild_members(self, grid: GridDesc, cell):
        cell = [_c32(a) for a in cell]
        n = len(cell[0])
        cell_of = np.empty(max(n, 1), np.int32)
        start = np.empty(grid.cell_total + 1, np.int32)
        items = np.empty(max(n, 1), np.int32)
        check(lib().sphx_rebuild_members(self.h, C.byref(grid), n, _ptr3(cell),
                                         cell_of.ctypes.data, start.ctypes.data,
                                         items.ctypes.data))
        return cell_of[:n], start, items[:n]

    # ---- raw host pointers (e.g. pinned torch CPU tensors) ------------------------------
    def rcll_ptr(self, grid: GridDesc, n: int, rel_ptrs, cell_ptrs, items_ptr: int,
                 start_ptr: int, prec: int) -> int:
        tot = C.c_int64()
        r = (C.c_void_p * 3)(*(list(rel_ptrs) + [None] * (3 - len(rel_ptrs))))
        c = (C.c_void_p * 3)(*(list(cell_ptrs) + [None] * (3 - len(cell_ptrs))))
        check(lib().sphx_rcll(self.h, C.byref(grid), n, r, c, n, items_ptr, start_ptr, prec,
                              C.byref(tot)))
        return tot.value

    def table_copy_ptr(self, offsets_ptr: int, items_ptr: int) -> None:
        check(lib().sphx_table_copy(self.h, offsets_ptr, items_ptr))

    # ---- device-resident API (torch tensors as device memory) ---------------------------
    def rcll_device(self, grid, rel, cell, items, cell_start, prec, offsets, items_out):
        self._bind(offsets)
        check(lib().sphx_rcll_device(self.h, C.byref(grid), rel[0].numel(), _dptr3(rel),
                                     _dptr3(cell), items.data_ptr(), cell_start.data_ptr(), prec,
                                     offsets.data_ptr(), items_out.data_ptr(), items_out.numel()))

    def cell_link_list_device(self, grid, x, h, items, cell_start, cell_of, prec, offsets,
                              items_out):
        self._bind(offsets)
        check(lib().sphx_cell_link_list_device(self.h, C.byref(grid), x[0].numel(), _dptr3(x),
                                               float(h), items.data_ptr(), cell_start.data_ptr(),
                                               cell_of.data_ptr(), prec, offsets.data_ptr(),
                                               items_out.data_ptr(), items_out.numel()))

    def build_rel_coords_device(self, grid, x, rel, cell, cell_of, cell_start, items):
        self._bind(items)
        check(lib().sphx_build_rel_coords_device(self.h, C.byref(grid), x[0].numel(), _dptr3(x),
                                                 _dptr3(rel), _dptr3(cell), cell_of.data_ptr(),
                                                 cell_start.data_ptr(), items.data_ptr()))

    # ---- slab decomposition (multigpu.py) -----------------------------------------------
    def build_rel_coords_window_device(self, global_grid, local_grid, axis, layer0, x, rel, cell,
                                       cell_of, cell_start, items):
        self._bind(items)
        check(lib().sphx_build_rel_coords_window_device(
            self.h, C.byref(global_grid), C.byref(local_grid), axis, layer0, x[0].numel(),
            _dptr3(x), _dptr3(rel), _dptr3(cell), cell_of.data_ptr(), cell_start.data_ptr(),
            items.data_ptr()))

    def rcll_rows_device(self, grid, rel, cell, items, cell_start, prec, ids, row0, nrows,
                         offsets, items_out):
        self._bind(offsets)
        check(lib().sphx_rcll_rows_device(
            self.h, C.byref(grid), rel[0].numel(), _dptr3(rel), _dptr3(cell), items.data_ptr(),
            cell_start.data_ptr(), prec, ids.data_ptr() if ids is not None else None, row0, nrows,
            offsets.data_ptr(), items_out.data_ptr(), items_out.numel()))

    def slab_assemble_device(self, local_grid, axis, n_own, slot_below, slot_above, n_slots,
                             owned_start, recv_below, recv_above, cell_start, items, cell):
        """Local CellGrid of a slab after its halo exchange (sphx_slab_assemble_device)."""
        self._bind(cell_start)
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        check(lib().sphx_slab_assemble_device(
            self.h, C.byref(local_grid), axis, n_own, slot_below, slot_above, n_slots,
            owned_start.data_ptr(), ptr(recv_below), ptr(recv_above), cell_start.data_ptr(),
            items.data_ptr(), _dptr3(cell)))

    def lattice_device(self, dim, lo, hi, ds, id0, x):
        self._bind(x[0])
        check(lib().sphx_lattice_device(self.h, dim, _d3(lo), _d3(hi), float(ds), id0,
                                        x[0].numel(), _dptr3(x)))
