// C ABI of libsphx_cuda.so (include/sphx_cuda.h): context, device buffers,
// precision constants, and the host/device entry points of the NNPS path.
// No CPU fallback anywhere: every neighbour decision is made on the device.

#include <nvtx3/nvToolsExt.h>
#include <thread>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <random>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "sphx/binary16.hpp"
#include "sphx_cuda.h"

namespace sphx_dev {
// sweep.cu
int launch_encode(int dim, int prec, int mode, int n, int64_t C, int nx, int wrapx,
                  const PrecConsts& pc, const double* const x[3], const int32_t* items,
                  const int32_t* start, const SweepArgs& a, cudaStream_t st);
int64_t launch_sweep(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st);
size_t coord_bytes(int dim, int prec);
size_t chunk_bytes(int dim, int prec, int mode);
int64_t chunk_capacity(int dim, int prec, int mode, int64_t n, int64_t C);
int sweep_tile(int dim, int prec, int mode);
int hit_words(int dim, int prec, int mode);
// binning.cu
int64_t scan_tiles(int64_t C);
void launch_locate(int mode, const LocateArgs& a, cudaStream_t st);
void launch_scan_counts(const int32_t* in, int32_t* out, int64_t C, unsigned long long* tiles,
                        int* counter, cudaStream_t st);
void launch_scatter_sort(int n, int64_t C, const int32_t* cell_of, const int32_t* slot,
                         const int32_t* start, int32_t* items, cudaStream_t st);
int launch_rcll_grad(int dim, const SweepArgs& a, cudaStream_t st);
int launch_update_relative(int64_t n, int dim, int prec, double* const rel[3],
                           int32_t* const cell[3], const double* const dx[3],
                           const double edge[3], const int counts[3], const int periodic[3],
                           unsigned long long* status, cudaStream_t st);
int launch_rcll_distances(int dim, int prec, int64_t nrows, const GridConsts& g,
                          const PrecConsts& pc, const double hc[3], const double* const rel[3],
                          const int32_t* const cell[3], const int64_t* off,
                          const int32_t* items, double* dist, cudaStream_t st);
void launch_lattice(int dim, const double lo[3], double ds, const int64_t counts[3], int64_t id0,
                    int64_t count, double* const x[3], cudaStream_t st);
int launch_step_rates(int dim, const StepArgs& a, cudaStream_t st);
int launch_kick_drift(int dim, const StepArgs& a, cudaStream_t st);
// window.cu
int64_t win2_tiles(int64_t nrows);
size_t win2_desc_bytes(int64_t nrows);
int launch_win2(const Win2Args& a, bool grad, cudaStream_t st, cudaEvent_t mid);
// slab.cu
int launch_slab_assemble(const SlabArgs& a, cudaStream_t st);
}  // namespace sphx_dev

using namespace sphx_dev;

// ----------------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------------
namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e__ = (call);                                                             \
    if (e__ != cudaSuccess)                                                               \
      return fail(SPHX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__));    \
  } while (0)

#define CKL()                                                                             \
  do {                                                                                    \
    cudaError_t e__ = cudaGetLastError();                                                 \
    if (e__ != cudaSuccess)                                                               \
      return fail(SPHX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e__)); \
  } while (0)

#define TRY(x)              \
  do {                      \
    int r__ = (x);          \
    if (r__ != SPHX_OK) return r__; \
  } while (0)

// ----------------------------------------------------------------------------------
// device buffers (grow-only)
// ----------------------------------------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return SPHX_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t want = std::max<size_t>(need, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(SPHX_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(want) +
                                     "): " + cudaGetErrorString(e));
    }
    bytes = want;
    return SPHX_OK;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

struct sphx_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  bool timing = false;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  float t_encode = 0.f, t_sweep = 0.f;
  // inputs staged from host
  Buf in_x[3], in_cell[3], in_items, in_start, in_cellof;
  // encode / sweep scratch
  Buf pos_own, tri, qc, qtag, selfpos, xy_nch, xy_cstart, xy_tiles;
  // single-pass sweep: look-back words (epoch-tagged) and the tile ticket
  Buf sw_tiles, sw_ticket, sw_rowk, sw_hitw;
  unsigned long long sw_tick = 0;
  unsigned sw_epoch = 0;
  int64_t sw_ntiles = 0;
  // table of the last host-API call
  Buf t_offsets, t_items, t_dist;
  // fused gradient (host API staging)
  Buf g_x[3], g_f, g_out[3], g_deg;
  int64_t t_n = -1, t_total = 0, t_capacity = 0;
  bool t_rcll = false;  // the last host table came from sphx_rcll (inputs still staged)
  // binning scratch
  Buf b_counts, b_slot, b_bad, b_tiles, b_out_cellof, b_out_start, b_out_items, b_rel[3], b_cell[3];
  // device time step: stress (sigma, tau, eps), rates, displacement, max |dx|, status
  Buf s_stress, s_rates, s_dx, s_flags;
  // windowed 2-D FP16 RCLL: CSR-order binary16 x/y pairs, cell x, ids, run lists
  Buf w_xy, w_u, w_id, w_run, w_desc, w_cb, w_self;
  // pinned staging for pageable host buffers (two chunks) and their events
  void* h_stage = nullptr;
  cudaEvent_t h_ev[2] = {nullptr, nullptr};
};

namespace {

// NVTX range over one phase of a call (bin / encode / sweep / pack+sweep / halo),
// visible to Nsight Systems / Compute; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ----------------------------------------------------------------------------------
// precision constants (host, exact)
// ----------------------------------------------------------------------------------
double r16(double x) { return sphx::round16(x); }
uint16_t b16(double x) { return sphx::Binary16::encode(x); }

uint16_t thr16(double cutoff16) {
  // smallest binary16 a >= 0 with round16(sqrt(a)) >= cutoff16 (nnps.cpp:344, :409);
  // the predicate is monotone in a, so bisect over the finite patterns + inf.
  if (std::isnan(cutoff16)) return 0;
  auto pred = [&](uint32_t b) {
    return r16(std::sqrt(sphx::Binary16::decode((uint16_t)b))) >= cutoff16;
  };
  if (pred(0)) return 0;
  uint32_t lo = 0, hi = 0x7C00u;  // pred(inf) holds
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    (pred(mid) ? hi : lo) = mid;
  }
  return (uint16_t)hi;
}

float thr32(float cutoff) {
  if (std::isnan(cutoff)) return 0.0f;
  uint32_t lo = 0, hi = 0x7F800000u;  // predicate true at +inf
  auto pred = [&](uint32_t b) {
    float a;
    std::memcpy(&a, &b, 4);
    return std::sqrt(a) >= cutoff;
  };
  if (pred(lo)) return 0.0f;
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    (pred(mid) ? hi : lo) = mid;
  }
  float t;
  std::memcpy(&t, &hi, 4);
  return t;
}

double thr64(double cutoff) {
  if (std::isnan(cutoff)) return 0.0;
  uint64_t lo = 0, hi = 0x7FF0000000000000ull;
  auto pred = [&](uint64_t b) {
    double a;
    std::memcpy(&a, &b, 8);
    return std::sqrt(a) >= cutoff;
  };
  if (pred(lo)) return 0.0;
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    (pred(mid) ? hi : lo) = mid;
  }
  double t;
  std::memcpy(&t, &hi, 8);
  return t;
}

double span_of(const sphx_grid_desc& g, int k) { return g.hi[k] - g.lo[k]; }

// mode RCLL: cutoff = round_to(prec, cutoff_norm), hh/cc from hc (nnps.cpp:289-295)
// mode CLL/ALL: cutoff = round_to(prec, 2h), shifts = round_to(prec, span) (:177-197)
PrecConsts make_consts(int mode, int prec, const sphx_grid_desc& g, double h) {
  PrecConsts c;
  std::memset(&c, 0, sizeof(c));
  const double cut = mode == MODE_RCLL ? g.cutoff_norm : 2.0 * h;
  for (int k = 0; k < 3; ++k) {
    const double hc = k < g.dim ? g.hc[k] : 0.0;
    const double sp = k < g.dim ? span_of(g, k) : 0.0;
    c.h_hh[k] = b16(0.5 * hc);
    c.h_cc[k] = b16(hc);
    c.h_sh[k] = b16(sp);
    c.f_hh[k] = (float)(0.5 * hc);
    c.f_cc[k] = (float)hc;
    c.f_sh[k] = (float)sp;
    c.d_hh[k] = 0.5 * hc;
    c.d_cc[k] = hc;
    c.d_sh[k] = sp;
  }
  c.h_thr = thr16(r16(cut));
  c.f_thr = thr32((float)cut);
  c.d_thr = thr64(cut);
  return c;
}

int check_prec_dim(int32_t prec, int32_t dim) {
  if (prec < SPHX_FP64 || prec > SPHX_FP16) return fail(SPHX_ERR_INVALID_ARGUMENT, "unknown precision");
  if (dim < 1 || dim > 3) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain dimension must be 1, 2 or 3");
  return SPHX_OK;
}

int64_t cell_total(const sphx_grid_desc& g) {
  int64_t t = 1;
  for (int k = 0; k < g.dim; ++k) t *= g.counts[k];
  return t;
}

GridConsts grid_consts(const sphx_grid_desc& g) {
  GridConsts gc;
  gc.dim = g.dim;
  for (int k = 0; k < 3; ++k) {
    gc.counts[k] = k < g.dim ? g.counts[k] : 1;
    gc.wrap[k] = (k < g.dim && g.periodic[k] && g.counts[k] > 2) ? 1 : 0;
  }
  return gc;
}

BinConsts bin_consts(const sphx_grid_desc& g) {
  BinConsts b;
  std::memset(&b, 0, sizeof(b));
  b.dim = g.dim;
  double hd = 0.0;
  for (int k = 0; k < g.dim; ++k) hd = std::max(hd, span_of(g, k));  // Domain::h_d
  b.hd = hd;
  for (int k = 0; k < 3; ++k) {
    b.counts[k] = k < g.dim ? g.counts[k] : 1;
    b.loc_counts[k] = b.counts[k];
    b.hc[k] = g.hc[k];
    b.origin[k] = g.origin[k];
    b.lo[k] = g.lo[k];
    b.hi[k] = g.hi[k];
  }
  b.win_axis = -1;
  return b;
}

// Slab window: locate on the global grid (its normalisation, origin and
// counts), keep layers [layer0, layer0 + local.counts[axis]) (mod the global
// count) along `axis`, CSR over the local grid.
BinConsts window_consts(const sphx_grid_desc& global, const sphx_grid_desc& local, int axis,
                        int layer0) {
  BinConsts b = bin_consts(global);
  for (int k = 0; k < 3; ++k) b.counts[k] = k < local.dim ? local.counts[k] : 1;
  b.win_axis = axis;
  b.win_lo = layer0;
  b.win_global = global.counts[axis];
  return b;
}

// Device -> pageable host memory (the drop-in's std::vectors) goes through two
// pinned staging chunks: chunk c+1's DMA is in flight while chunk c is handed to
// the consumer (an 8-thread memcpy, or the caller's sink). The driver's own
// pageable D2H copies single-threaded (~16 GB/s, measured).
// Host -> device stays on the driver's pageable path: measured on the box it
// beats a staged copy for the drop-in's 4-8 MB inputs (2.9 vs 3.7 ms at C2).
constexpr size_t kStage = size_t(16) << 20;
constexpr int kCopyThreads = 8;

bool host_is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(void* dst, const void* src, size_t n) {
  if (n < (size_t(2) << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  std::thread th[kCopyThreads - 1];
  auto part = [&](int k) {
    const size_t a = n * k / kCopyThreads, b = n * (k + 1) / kCopyThreads;
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  };
  for (int k = 1; k < kCopyThreads; ++k) th[k - 1] = std::thread(part, k);
  part(0);
  for (auto& t : th) t.join();
}

int stage_ensure(sphx_context* ctx) {
  if (ctx->h_stage) return SPHX_OK;
  CK(cudaMallocHost(&ctx->h_stage, 2 * kStage));
  for (auto& e : ctx->h_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SPHX_OK;
}

// Streams `bytes` of device memory through the pinned stage; take(chunk, offset,
// length) consumes each chunk in order and returns SPHX_OK or an error code.
template <class Take>
int d2h_staged(sphx_context* ctx, const void* dsrc, size_t bytes, Take&& take) {
  TRY(stage_ensure(ctx));
  char* st[2] = {static_cast<char*>(ctx->h_stage), static_cast<char*>(ctx->h_stage) + kStage};
  const size_t nch = (bytes + kStage - 1) / kStage;
  auto issue = [&](size_t c) -> int {
    const size_t o = c * kStage, l = std::min(kStage, bytes - o);
    CK(cudaMemcpyAsync(st[c & 1], static_cast<const char*>(dsrc) + o, l, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaEventRecord(ctx->h_ev[c & 1], ctx->stream));
    return SPHX_OK;
  };
  for (size_t c = 0; c < nch && c < 2; ++c) TRY(issue(c));
  int rc = SPHX_OK;
  for (size_t c = 0; c < nch; ++c) {
    CK(cudaEventSynchronize(ctx->h_ev[c & 1]));
    const size_t o = c * kStage, l = std::min(kStage, bytes - o);
    if (rc == SPHX_OK) rc = take(st[c & 1], o, l);
    if (rc == SPHX_OK && c + 2 < nch) TRY(issue(c + 2));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return rc;
}

// device -> host; returns once the data is in `dst`
int copy_d2h(sphx_context* ctx, void* dst, const void* dsrc, size_t bytes) {
  if (!bytes) return SPHX_OK;
  if (bytes < (size_t(4) << 20) || !host_is_pageable(dst)) {
    CK(cudaMemcpyAsync(dst, dsrc, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SPHX_OK;
  }
  return d2h_staged(ctx, dsrc, bytes, [&](const char* chunk, size_t o, size_t l) {
    par_memcpy(static_cast<char*>(dst) + o, chunk, l);
    return SPHX_OK;
  });
}

// host -> device, stream-ordered (the host buffer may be reused on return)
int copy_h2d(sphx_context* ctx, void* ddst, const void* src, size_t bytes) {
  if (!bytes) return SPHX_OK;
  CK(cudaMemcpyAsync(ddst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return SPHX_OK;
}

int upload(sphx_context* ctx, Buf& b, const void* src, size_t bytes) {
  TRY(b.ensure(bytes));
  return copy_h2d(ctx, b.p, src, bytes);
}

// Encode on device pointers (src = rel for RCLL, positions for CLL/ALL): the
// candidate runs and own-particle data the sweep reads; fills *out for it.
// Rows to produce: particles [row0, row0 + nrows); ids = output id of each
// particle (null: its index). The multi-GPU slab path asks for the owned rows
// of a slab-local system with global ids.
struct RowSel {
  int64_t row0 = 0, nrows = -1;  // nrows < 0: all
  const int32_t* ids = nullptr;
};

// The windowed 2-D FP16 RCLL path (window.cu) is the default; SPHX_W2=0 selects
// the encode + k_rcll16 path.
bool win2_enabled() {
  const char* e = std::getenv("SPHX_W2");
  return !(e && e[0] == '0');
}

int run_prepare(sphx_context* ctx, int mode, const sphx_grid_desc& g, int64_t n64,
                const double* const src[3], const int32_t* const cellk[3], const int32_t* items,
                const int32_t* start, const int32_t* cell_of, int prec, double h, int64_t* d_off,
                SweepArgs* out, const RowSel& sel = RowSel(), bool allow_window = true) {
  if (n64 > INT32_MAX - 64)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "too many particles for one context (int32 ids)");
  const int n = (int)n64;
  const int64_t nrows = sel.nrows < 0 ? n64 : sel.nrows;
  if (sel.row0 < 0 || sel.row0 + nrows > n64)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "row range outside the system");
  cudaStream_t st = ctx->stream;
  std::memset(out, 0, sizeof(*out));
  out->n = n;
  out->row0 = (int)sel.row0;
  out->nrows = (int)nrows;
  out->ids = sel.ids;
  out->order = items;
  out->offsets = d_off;
  if (n == 0 || nrows == 0) {
    CK(cudaMemsetAsync(d_off, 0, sizeof(int64_t), st));
    return SPHX_OK;
  }
  const int64_t C = mode == MODE_ALL ? 0 : cell_total(g);
  if (allow_window && g.dim == 2 && prec == SPHX_FP16 && mode == MODE_RCLL &&
      g.counts[0] <= 2048 && win2_enabled()) {
    const PrecConsts pc = make_consts(mode, prec, g, h);
    if (pc.h_thr != 0) {  // (thr == 0: no pair can hit; the generic path handles it)
      // windowed path (window.cu): pack + sweep in run_sweep, no encode
      const size_t np = (size_t)n + 64;
      // lanes past their segment read up to 32 records beyond it (masked out):
      // fresh buffers are zeroed once so that the padding past n is defined
      for (Buf* b : {&ctx->w_xy, &ctx->w_u, &ctx->w_id}) {
        const size_t want = (b == &ctx->w_u ? 2 : 4) * np;
        const void* old = b->p;
        TRY(b->ensure(want));
        if (b->p != old) CK(cudaMemsetAsync(b->p, 0, b->bytes, st));
      }
      TRY(ctx->w_run.ensure(32 * (size_t)C));
      TRY(ctx->w_desc.ensure(win2_desc_bytes(nrows)));
      TRY(ctx->w_cb.ensure(16 * (size_t)C));
      TRY(ctx->w_self.ensure(4 * (size_t)n));
      SweepArgs& a = *out;
      a.g = grid_consts(g);
      a.c = pc;
      a.win2 = 1;
      for (int k = 0; k < 3; ++k) {
        a.src[k] = k < g.dim ? src[k] : nullptr;
        a.cellk[k] = cellk ? cellk[k] : nullptr;
      }
      a.start = start;
      a.cell_of = cell_of;
      if (ctx->timing) CK(cudaEventRecord(ctx->ev[0], st));  // ev[1]: after the pack
      return SPHX_OK;
    }
  }
  const int64_t chunks = chunk_capacity(g.dim, prec, mode, n, C);
  // record indices (selfpos) are 32-bit and chunk starts (xy_cstart) 31-bit
  if (4 * chunks >= (int64_t(1) << 32) || chunks >= INT32_MAX)
    return fail(SPHX_ERR_INVALID_ARGUMENT,
                "too many candidate records for one context (split the system into slabs)");
  TRY(ctx->pos_own.ensure(coord_bytes(g.dim, prec) * (size_t)n));
  TRY(ctx->qc.ensure(chunk_bytes(g.dim, prec, mode) * (size_t)chunks));
  TRY(ctx->qtag.ensure(16 * (size_t)chunks));
  if (mode != MODE_ALL) {
    TRY(ctx->tri.ensure(sizeof(int2) * std::max<int64_t>(C, 1)));
    if (g.dim == 3 && prec == SPHX_FP16 && mode == MODE_RCLL) {  // xy-plane runs
      TRY(ctx->xy_nch.ensure(sizeof(int32_t) * std::max<int64_t>(C, 1)));
      TRY(ctx->xy_cstart.ensure(sizeof(int32_t) * (C + 1)));
      TRY(ctx->xy_tiles.ensure(sizeof(unsigned long long) * (scan_tiles(C) + 2)));
    }
    TRY(ctx->selfpos.ensure(sizeof(int32_t) * (size_t)n));
  }

  SweepArgs& a = *out;
  a.g = grid_consts(g);
  a.c = make_consts(mode, prec, g, h);
  a.tri = ctx->tri.as<int2>();
  a.qc = ctx->qc.p;
  a.nchunks = chunks;
  a.qtag = ctx->qtag.p;
  a.selfpos = ctx->selfpos.as<uint32_t>();
  a.xy_nch = ctx->xy_nch.as<int32_t>();
  a.xy_cstart = ctx->xy_cstart.as<int32_t>();
  a.xy_tiles = ctx->xy_tiles.as<unsigned long long>();
  a.pos_own = ctx->pos_own.p;
  for (int k = 0; k < 3; ++k) a.cellk[k] = cellk ? cellk[k] : nullptr;
  a.cell_of = cell_of;

  if (ctx->timing) CK(cudaEventRecord(ctx->ev[0], st));
  NvtxRange nvtx_encode("sphx.encode");
  ctx->launches += launch_encode(g.dim, prec, mode, n, C, a.g.counts[0], a.g.wrap[0], a.c, src,
                                 items, start, a, st);
  CKL();
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[1], st));
  return SPHX_OK;
}

// The windowed 2-D FP16 RCLL kernels' arguments (window.cu) from a prepared call.
Win2Args win2_args(sphx_context* ctx, const SweepArgs& a) {
  Win2Args w;
  std::memset(&w, 0, sizeof(w));
  w.n = a.n;
  w.row0 = a.row0;
  w.nrows = a.nrows;
  w.g = a.g;
  w.c = a.c;
  for (int k = 0; k < 2; ++k) {
    w.rel[k] = a.src[k];
    w.cellk[k] = a.cellk[k];
  }
  w.items = a.order;
  w.start = a.start;
  w.wxy = ctx->w_xy.as<__half>();
  w.wu = ctx->w_u.as<__half>();
  w.wid = ctx->w_id.as<int32_t>();
  w.wrun = ctx->w_run.as<uint8_t>();
  w.desc = ctx->w_desc.p;
  w.ids = a.ids;
  w.wcb = ctx->w_cb.as<int4>();
  w.wself = ctx->w_self.as<int32_t>();
  return w;
}

// The single-pass sweep: offsets (always) and the rows (where they fit in
// `capacity`; the exact total is d_off[nrows] either way).
int run_sweep(sphx_context* ctx, int dim, int prec, int mode, SweepArgs& a, int32_t* d_items,
              int64_t capacity) {
  if (a.n == 0 || a.nrows == 0) return SPHX_OK;
  cudaStream_t st = ctx->stream;
  const int64_t nt = a.win2    ? win2_tiles(a.nrows)
                               : (a.nrows + sweep_tile(dim, prec, mode) - 1) / sweep_tile(dim, prec, mode);
  if (nt > ctx->sw_ntiles || ctx->sw_epoch >= 0xFFFFu) {
    // fresh (or recycled) look-back words: epoch 0 marks them unpublished
    TRY(ctx->sw_tiles.ensure(sizeof(unsigned long long) * std::max<int64_t>(nt, ctx->sw_ntiles)));
    ctx->sw_ntiles = std::max<int64_t>(nt, ctx->sw_ntiles);
    CK(cudaMemsetAsync(ctx->sw_tiles.p, 0, sizeof(unsigned long long) * ctx->sw_ntiles, st));
    ctx->sw_epoch = 0;
  }
  if (!ctx->sw_ticket.p) {
    TRY(ctx->sw_ticket.ensure(sizeof(unsigned long long)));
    CK(cudaMemsetAsync(ctx->sw_ticket.p, 0, sizeof(unsigned long long), st));
    ctx->sw_tick = 0;
  }
  if (a.win2) {
    Win2Args w = win2_args(ctx, a);
    w.offsets = a.offsets;
    w.out = d_items;
    w.capacity = capacity;
    w.tiles = ctx->sw_tiles.as<unsigned long long>();
    w.epoch = ++ctx->sw_epoch;
    NvtxRange nvtx_sweep("sphx.pack+sweep");
    ctx->launches += launch_win2(w, false, st, ctx->timing ? ctx->ev[1] : nullptr);
    CKL();
    if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], st));
    return SPHX_OK;
  }
  const int hw = hit_words(dim, prec, mode);
  if (hw > 0) {
    TRY(ctx->sw_rowk.ensure(sizeof(int32_t) * (size_t)a.nrows));
    TRY(ctx->sw_hitw.ensure(sizeof(unsigned) * (size_t)hw * (size_t)a.nrows));
    a.rowk = ctx->sw_rowk.as<int32_t>();
    a.hitw = ctx->sw_hitw.as<unsigned>();
  }
  a.items = d_items;
  a.capacity = capacity;
  a.tiles = ctx->sw_tiles.as<unsigned long long>();
  a.ticket = ctx->sw_ticket.as<unsigned long long>();
  a.tick0 = ctx->sw_tick;
  a.epoch = ++ctx->sw_epoch;
  NvtxRange nvtx_sweep("sphx.sweep");
  const int64_t used = launch_sweep(dim, prec, mode, a, st);
  CKL();
  ctx->sw_tick += (unsigned long long)used;
  ctx->launches += hw > 0 ? 2 : 1;  // test + emit kernels, or the single-pass sweep
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], st));
  return SPHX_OK;
}

// Device API: encode + sweep, no synchronisation (capacity overflow is
// detectable by the caller through d_off[n]).
int run_nnps(sphx_context* ctx, int mode, const sphx_grid_desc& g, int64_t n,
             const double* const src[3], const int32_t* const cellk[3], const int32_t* items,
             const int32_t* start, const int32_t* cell_of, int prec, double h, int64_t* d_off,
             int32_t* d_items, int64_t capacity) {
  SweepArgs a;
  TRY(run_prepare(ctx, mode, g, n, src, cellk, items, start, cell_of, prec, h, d_off, &a));
  return run_sweep(ctx, g.dim, prec, mode, a, d_items, capacity);
}

// Host-API driver: encode, sweep into the context's table, read the exact total;
// if the table was too small, grow it and sweep again (the encode is reused).
int run_host_table(sphx_context* ctx, int mode, const sphx_grid_desc& g, int64_t n,
                   const double* const d_src[3], const int32_t* const d_cellk[3],
                   const int32_t* d_items, const int32_t* d_start, const int32_t* d_cellof,
                   int prec, double h, int64_t* total) {
  TRY(ctx->t_offsets.ensure(sizeof(int64_t) * (n + 1)));
  SweepArgs a;
  TRY(run_prepare(ctx, mode, g, n, d_src, d_cellk, d_items, d_start, d_cellof, prec, h,
                  ctx->t_offsets.as<int64_t>(), &a));
  if (ctx->t_capacity == 0) {
    // first table on this context: room for the typical row lengths of a
    // uniform distribution at kh = 2.4 ds (2-D ~18, 3-D ~57)
    const int64_t per = g.dim == 3 ? 64 : (g.dim == 2 ? 24 : 6);
    ctx->t_capacity = std::max<int64_t>(per * n, 1024);
    TRY(ctx->t_items.ensure(sizeof(int32_t) * ctx->t_capacity));
  }
  int64_t tot = 0;
  for (int pass = 0; pass < 2; ++pass) {
    TRY(run_sweep(ctx, g.dim, prec, mode, a, ctx->t_items.as<int32_t>(), ctx->t_capacity));
    CK(cudaMemcpyAsync(&tot, ctx->t_offsets.as<int64_t>() + n, sizeof(int64_t),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (tot <= ctx->t_capacity) break;
    ctx->t_capacity = tot + tot / 16 + 1024;
    TRY(ctx->t_items.ensure(sizeof(int32_t) * ctx->t_capacity));
  }
  ctx->t_n = n;
  ctx->t_total = tot;
  *total = tot;
  return SPHX_OK;
}

int check_ctx(sphx_context* ctx) {
  if (!ctx) return fail(SPHX_ERR_INVALID_ARGUMENT, "null context");
  CK(cudaSetDevice(ctx->device));
  return SPHX_OK;
}

// Binning on device pointers (locate -> counts -> scan -> scatter -> per-cell sort).
int run_binning(sphx_context* ctx, int bmode, const sphx_grid_desc& g, int64_t n64,
                const double* const d_x[3], const int32_t* const d_cell_in[3],
                double* const d_rel[3], int32_t* const d_cell[3], int32_t* d_cell_of,
                int32_t* d_start, int32_t* d_items, unsigned long long* d_bad,
                const BinConsts* window = nullptr) {
  const int n = (int)n64;
  const int64_t C = cell_total(g);
  cudaStream_t st = ctx->stream;
  TRY(ctx->b_counts.ensure(sizeof(int32_t) * std::max<int64_t>(C, 1)));
  TRY(ctx->b_slot.ensure(sizeof(int32_t) * std::max(n, 1)));
  const int64_t nt = std::max<int64_t>(scan_tiles(C), 1);
  TRY(ctx->b_tiles.ensure(sizeof(unsigned long long) * nt + 16));
  CK(cudaMemsetAsync(ctx->b_counts.p, 0, sizeof(int32_t) * C, st));
  CK(cudaMemsetAsync(ctx->b_tiles.p, 0, sizeof(unsigned long long) * nt + 16, st));
  LocateArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = n;
  a.g = window ? *window : bin_consts(g);
  for (int k = 0; k < 3; ++k) {
    a.x[k] = d_x ? d_x[k] : nullptr;
    a.cell_in[k] = d_cell_in ? d_cell_in[k] : nullptr;
    a.rel_out[k] = d_rel ? d_rel[k] : nullptr;
    a.cell_out[k] = d_cell ? d_cell[k] : nullptr;
  }
  a.cell_of = d_cell_of;
  a.counts = ctx->b_counts.as<int32_t>();
  a.slot = ctx->b_slot.as<int32_t>();
  a.bad = d_bad;
  NvtxRange nvtx_bin("sphx.bin");
  launch_locate(bmode, a, st);
  CKL();
  ++ctx->launches;
  unsigned long long* tiles = ctx->b_tiles.as<unsigned long long>();
  launch_scan_counts(a.counts, d_start, C, tiles, reinterpret_cast<int*>(tiles + nt), st);
  CKL();
  ++ctx->launches;
  launch_scatter_sort(n, C, d_cell_of, a.slot, d_start, d_items, st);
  CKL();
  ctx->launches += 2;
  return SPHX_OK;
}

}  // namespace

// ==================================================================================
// C ABI
// ==================================================================================
extern "C" {

const char* sphx_last_error(void) { return g_err.c_str(); }

int sphx_grid_init(sphx_grid_desc* g, int32_t dim, const double lo[3], const double hi[3],
                   double radius, const int32_t periodic[3]) {
  // CellGrid::CellGrid (cell_grid.cpp:9-34) and Domain::validate (domain.hpp:29-34)
  if (!g) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  std::memset(g, 0, sizeof(*g));
  if (dim < 1 || dim > 3) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain dimension must be 1, 2 or 3");
  for (int k = 0; k < dim; ++k)
    if (!(lo[k] < hi[k])) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain bounds must satisfy lo < hi");
  if (!(radius > 0.0)) return fail(SPHX_ERR_INVALID_ARGUMENT, "search radius must be positive");
  g->dim = dim;
  double hd = 0.0;
  for (int k = 0; k < dim; ++k) hd = std::max(hd, hi[k] - lo[k]);
  g->cutoff_norm = 2.0 * radius / hd;
  g->radius_phys = radius;
  for (int k = 0; k < 3; ++k) {
    g->counts[k] = 1;
    g->lo[k] = lo[k];
    g->hi[k] = hi[k];
    g->periodic[k] = periodic ? (periodic[k] != 0) : 0;
  }
  for (int k = 0; k < dim; ++k) {
    const double span = hi[k] - lo[k];
    double edge;
    if (g->periodic[k]) {
      const int c = static_cast<int>(std::floor(span / radius + 1e-12));
      g->counts[k] = c > 0 ? c : 1;
      edge = span / g->counts[k];
      if (g->counts[k] < 3) return fail(SPHX_ERR_INVALID_ARGUMENT, "periodic axis needs at least 3 cells");
    } else {
      g->counts[k] = static_cast<int>(std::ceil(span / radius - 1e-12));
      if (g->counts[k] < 1) g->counts[k] = 1;
      edge = radius;
    }
    g->hc[k] = 2.0 * edge / hd;
    g->origin[k] = (2.0 * lo[k] - (hi[k] + lo[k])) / hd;
  }
  return SPHX_OK;
}

int sphx_create(int device, sphx_context** out) {
  if (!out) return fail(SPHX_ERR_INVALID_ARGUMENT, "null output");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(SPHX_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0) CK(cudaGetDevice(&device));
  if (device >= ndev) return fail(SPHX_ERR_CUDA, "device index out of range");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(SPHX_ERR_CUDA, std::string("libsphx_cuda is built for sm_100a (B200); device is ") +
                                   prop.name + " sm_" + std::to_string(prop.major) +
                                   std::to_string(prop.minor));
  CK(cudaSetDevice(device));
  auto* ctx = new sphx_context();
  ctx->device = device;
  e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return fail(SPHX_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  *out = ctx;
  return SPHX_OK;
}

void sphx_destroy(sphx_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  Buf* all[] = {&ctx->in_x[0], &ctx->in_x[1], &ctx->in_x[2], &ctx->in_cell[0], &ctx->in_cell[1],
                &ctx->in_cell[2], &ctx->in_items, &ctx->in_start, &ctx->in_cellof, &ctx->pos_own,
                &ctx->tri, &ctx->qc, &ctx->xy_nch, &ctx->xy_cstart, &ctx->xy_tiles,
                &ctx->qtag, &ctx->selfpos, &ctx->sw_tiles, &ctx->sw_ticket, &ctx->sw_rowk, &ctx->sw_hitw, &ctx->t_offsets, &ctx->t_items, &ctx->t_dist, &ctx->g_x[0], &ctx->g_x[1], &ctx->g_x[2],
                &ctx->g_f, &ctx->g_out[0], &ctx->g_out[1], &ctx->g_out[2], &ctx->g_deg,
                &ctx->b_counts, &ctx->b_slot, &ctx->b_bad, &ctx->b_tiles, &ctx->b_out_cellof,
                &ctx->b_out_start, &ctx->b_out_items, &ctx->b_rel[0], &ctx->b_rel[1],
                &ctx->b_rel[2], &ctx->b_cell[0], &ctx->b_cell[1], &ctx->b_cell[2],
                &ctx->s_stress, &ctx->s_rates, &ctx->s_dx, &ctx->s_flags,
                &ctx->w_xy, &ctx->w_u, &ctx->w_id, &ctx->w_run, &ctx->w_desc, &ctx->w_cb, &ctx->w_self};
  for (Buf* b : all) b->release();
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  for (auto& e : ctx->h_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

int sphx_set_stream(sphx_context* ctx, void* stream) {
  TRY(check_ctx(ctx));
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return SPHX_OK;
}

int64_t sphx_launch_count(const sphx_context* ctx) { return ctx ? ctx->launches : 0; }

int sphx_enable_timing(sphx_context* ctx, int on) {
  TRY(check_ctx(ctx));
  ctx->timing = on != 0;
  return SPHX_OK;
}

int sphx_last_timing(sphx_context* ctx, float* encode_ms, float* sweep_ms) {
  TRY(check_ctx(ctx));
  if (!ctx->timing) return fail(SPHX_ERR_INVALID_ARGUMENT, "timing not enabled");
  CK(cudaEventSynchronize(ctx->ev[2]));
  float e = 0.f, s = 0.f;
  CK(cudaEventElapsedTime(&e, ctx->ev[0], ctx->ev[1]));
  CK(cudaEventElapsedTime(&s, ctx->ev[1], ctx->ev[2]));
  if (encode_ms) *encode_ms = e;
  if (sweep_ms) *sweep_ms = s;
  return SPHX_OK;
}

// ---------------- drop-in host API ----------------

int sphx_rcll(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
              const double* const rel[3], const int32_t* const cell[3], int64_t n_items,
              const int32_t* items, const int32_t* cell_start, int32_t precision,
              int64_t* total) {
  TRY(check_ctx(ctx));
  if (!grid || !total) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(precision, grid->dim));
  if (n_items != n) return fail(SPHX_ERR_INVALID_ARGUMENT, "grid membership is stale");  // nnps.cpp:298
  const int64_t C = cell_total(*grid);
  const double* d_rel[3] = {nullptr, nullptr, nullptr};
  const int32_t* d_cell[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < grid->dim; ++k) {
    TRY(upload(ctx, ctx->in_x[k], rel[k], sizeof(double) * n));
    TRY(upload(ctx, ctx->in_cell[k], cell[k], sizeof(int32_t) * n));
    d_rel[k] = ctx->in_x[k].as<double>();
    d_cell[k] = ctx->in_cell[k].as<int32_t>();
  }
  TRY(upload(ctx, ctx->in_items, items, sizeof(int32_t) * n));
  TRY(upload(ctx, ctx->in_start, cell_start, sizeof(int32_t) * (C + 1)));
  const int rc = run_host_table(ctx, MODE_RCLL, *grid, n, d_rel, d_cell,
                                ctx->in_items.as<int32_t>(), ctx->in_start.as<int32_t>(), nullptr,
                                precision, 0.0, total);
  ctx->t_rcll = rc == SPHX_OK;
  return rc;
}

int sphx_cell_link_list(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                        const double* const x[3], double h, int64_t n_items,
                        const int32_t* items, const int32_t* cell_start,
                        const int32_t* cell_of, int32_t precision, int64_t* total) {
  TRY(check_ctx(ctx));
  if (!grid || !total) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(precision, grid->dim));
  if (n_items != n)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "grid membership is stale; rebin first");  // nnps.cpp:184
  const int64_t C = cell_total(*grid);
  const double* d_x[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < grid->dim; ++k) {
    TRY(upload(ctx, ctx->in_x[k], x[k], sizeof(double) * n));
    d_x[k] = ctx->in_x[k].as<double>();
  }
  TRY(upload(ctx, ctx->in_items, items, sizeof(int32_t) * n));
  TRY(upload(ctx, ctx->in_start, cell_start, sizeof(int32_t) * (C + 1)));
  TRY(upload(ctx, ctx->in_cellof, cell_of, sizeof(int32_t) * n));
  ctx->t_rcll = false;
  return run_host_table(ctx, MODE_CLL, *grid, n, d_x, nullptr, ctx->in_items.as<int32_t>(),
                        ctx->in_start.as<int32_t>(), ctx->in_cellof.as<int32_t>(), precision, h,
                        total);
}

int sphx_all_list(sphx_context* ctx, int32_t dim, int64_t n, const double* const x[3], double h,
                  int32_t precision, int64_t* total) {
  TRY(check_ctx(ctx));
  if (!total) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(precision, dim));
  if (n == 0) return fail(SPHX_ERR_INVALID_ARGUMENT, "all_list needs at least one particle");
  sphx_grid_desc g;
  std::memset(&g, 0, sizeof(g));
  g.dim = dim;
  for (int k = 0; k < 3; ++k) g.counts[k] = 1;
  const double* d_x[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < dim; ++k) {
    TRY(upload(ctx, ctx->in_x[k], x[k], sizeof(double) * n));
    d_x[k] = ctx->in_x[k].as<double>();
  }
  ctx->t_rcll = false;
  return run_host_table(ctx, MODE_ALL, g, n, d_x, nullptr, nullptr, nullptr, nullptr, precision,
                        h, total);
}

int sphx_table_stream(sphx_context* ctx, sphx_table_sink sink, void* user) {
  TRY(check_ctx(ctx));
  if (!sink) return fail(SPHX_ERR_INVALID_ARGUMENT, "null sink");
  if (ctx->t_n < 0) return fail(SPHX_ERR_INVALID_ARGUMENT, "no table computed on this context");
  const void* src[2] = {ctx->t_offsets.p, ctx->t_items.p};
  const size_t bytes[2] = {sizeof(int64_t) * size_t(ctx->t_n + 1),
                           sizeof(int32_t) * size_t(ctx->t_total)};
  for (int part = 0; part < 2; ++part) {
    if (!bytes[part]) continue;
    TRY(d2h_staged(ctx, src[part], bytes[part], [&](const char* chunk, size_t, size_t l) {
      return sink(user, part, chunk, int64_t(l)) == 0
                 ? SPHX_OK
                 : fail(SPHX_ERR_RUNTIME, "table sink failed");
    }));
  }
  return SPHX_OK;
}

int sphx_table_copy(sphx_context* ctx, int64_t* offsets, int32_t* items) {
  TRY(check_ctx(ctx));
  if (ctx->t_n < 0) return fail(SPHX_ERR_INVALID_ARGUMENT, "no table computed on this context");
  if (offsets) TRY(copy_d2h(ctx, offsets, ctx->t_offsets.p, sizeof(int64_t) * (ctx->t_n + 1)));
  if (items && ctx->t_total)
    TRY(copy_d2h(ctx, items, ctx->t_items.p, sizeof(int32_t) * ctx->t_total));
  CK(cudaStreamSynchronize(ctx->stream));
  return SPHX_OK;
}

static int binning_host(sphx_context* ctx, int bmode, const sphx_grid_desc* grid, int64_t n,
                        const double* const x[3], const int32_t* const cell_in[3],
                        double* const rel[3], int32_t* const cell[3], int32_t* cell_of,
                        int32_t* cell_start, int32_t* items) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(SPHX_FP64, grid->dim));
  if (n > INT32_MAX - 1024) return fail(SPHX_ERR_INVALID_ARGUMENT, "too many particles");
  const int dim = grid->dim;
  const int64_t C = cell_total(*grid);
  const double* d_x[3] = {nullptr, nullptr, nullptr};
  const int32_t* d_cin[3] = {nullptr, nullptr, nullptr};
  double* d_rel[3] = {nullptr, nullptr, nullptr};
  int32_t* d_cell[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < dim; ++k) {
    if (bmode == 2) {
      TRY(upload(ctx, ctx->in_cell[k], cell_in[k], sizeof(int32_t) * n));
      d_cin[k] = ctx->in_cell[k].as<int32_t>();
    } else {
      TRY(upload(ctx, ctx->in_x[k], x[k], sizeof(double) * n));
      d_x[k] = ctx->in_x[k].as<double>();
    }
    if (bmode == 1) {
      TRY(ctx->b_rel[k].ensure(sizeof(double) * std::max<int64_t>(n, 1)));
      TRY(ctx->b_cell[k].ensure(sizeof(int32_t) * std::max<int64_t>(n, 1)));
      d_rel[k] = ctx->b_rel[k].as<double>();
      d_cell[k] = ctx->b_cell[k].as<int32_t>();
    }
  }
  TRY(ctx->b_out_cellof.ensure(sizeof(int32_t) * std::max<int64_t>(n, 1)));
  TRY(ctx->b_out_start.ensure(sizeof(int32_t) * (C + 1)));
  TRY(ctx->b_out_items.ensure(sizeof(int32_t) * std::max<int64_t>(n, 1)));
  TRY(ctx->b_bad.ensure(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(ctx->b_bad.p, 0xFF, sizeof(unsigned long long), ctx->stream));
  TRY(run_binning(ctx, bmode, *grid, n, d_x, d_cin, d_rel, d_cell, ctx->b_out_cellof.as<int32_t>(),
                  ctx->b_out_start.as<int32_t>(), ctx->b_out_items.as<int32_t>(),
                  ctx->b_bad.as<unsigned long long>()));
  unsigned long long bad = ~0ull;
  CK(cudaMemcpyAsync(&bad, ctx->b_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad != ~0ull)
    return fail(SPHX_ERR_OUT_OF_RANGE, "particle " + std::to_string(bad) + " lies outside the grid");
  auto d2h = [&](void* dst, const void* src, size_t bytes) -> int {
    if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    return SPHX_OK;
  };
  TRY(d2h(cell_of, ctx->b_out_cellof.p, sizeof(int32_t) * n));
  TRY(d2h(cell_start, ctx->b_out_start.p, sizeof(int32_t) * (C + 1)));
  TRY(d2h(items, ctx->b_out_items.p, sizeof(int32_t) * n));
  if (bmode == 1) {
    for (int k = 0; k < dim; ++k) {
      TRY(d2h(rel[k], d_rel[k], sizeof(double) * n));
      TRY(d2h(cell[k], d_cell[k], sizeof(int32_t) * n));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SPHX_OK;
}

int sphx_rebin(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n, const double* const x[3],
               int32_t* cell_of, int32_t* cell_start, int32_t* items) {
  return binning_host(ctx, 0, grid, n, x, nullptr, nullptr, nullptr, cell_of, cell_start, items);
}

int sphx_build_rel_coords(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                          const double* const x[3], double* const rel[3], int32_t* const cell[3],
                          int32_t* cell_of, int32_t* cell_start, int32_t* items) {
  return binning_host(ctx, 1, grid, n, x, nullptr, rel, cell, cell_of, cell_start, items);
}

int sphx_rebuild_members(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                         const int32_t* const cell[3], int32_t* cell_of, int32_t* cell_start,
                         int32_t* items) {
  return binning_host(ctx, 2, grid, n, nullptr, cell, nullptr, nullptr, cell_of, cell_start,
                      items);
}

// ---------------- device-resident API ----------------

int sphx_rcll_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                     const double* const d_rel[3], const int32_t* const d_cell[3],
                     const int32_t* d_items, const int32_t* d_cell_start, int32_t precision,
                     int64_t* d_offsets, int32_t* d_items_out, int64_t capacity) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  return run_nnps(ctx, MODE_RCLL, *grid, n, d_rel, d_cell, d_items, d_cell_start, nullptr,
                  precision, 0.0, d_offsets, d_items_out, capacity);
}

int sphx_cell_link_list_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                               const double* const d_x[3], double h, const int32_t* d_items,
                               const int32_t* d_cell_start, const int32_t* d_cell_of,
                               int32_t precision, int64_t* d_offsets, int32_t* d_items_out,
                               int64_t capacity) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  return run_nnps(ctx, MODE_CLL, *grid, n, d_x, nullptr, d_items, d_cell_start, d_cell_of,
                  precision, h, d_offsets, d_items_out, capacity);
}

int sphx_build_rel_coords_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                 const double* const d_x[3], double* const d_rel[3],
                                 int32_t* const d_cell[3], int32_t* d_cell_of,
                                 int32_t* d_cell_start, int32_t* d_items) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(SPHX_FP64, grid->dim));
  TRY(ctx->b_bad.ensure(sizeof(unsigned long long)));
  return run_binning(ctx, 1, *grid, n, d_x, nullptr, d_rel, d_cell, d_cell_of, d_cell_start,
                     d_items, ctx->b_bad.as<unsigned long long>());
}

int sphx_rebin_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                      const double* const d_x[3], int32_t* d_cell_of, int32_t* d_cell_start,
                      int32_t* d_items, int64_t* d_bad) {
  TRY(check_ctx(ctx));
  if (!grid || !d_bad) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(SPHX_FP64, grid->dim));
  CK(cudaMemsetAsync(d_bad, 0xFF, sizeof(int64_t), ctx->stream));
  return run_binning(ctx, 0, *grid, n, d_x, nullptr, nullptr, nullptr, d_cell_of, d_cell_start,
                     d_items, reinterpret_cast<unsigned long long*>(d_bad));
}

// ---------------- RCLL maintenance (update_relative + rebuild_members) ----------------

int sphx_update_relative_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                double* const d_rel[3], int32_t* const d_cell[3],
                                const double* const d_dx[3], int32_t precision,
                                unsigned long long* d_status) {
  TRY(check_ctx(ctx));
  if (!grid || !d_status) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(precision, grid->dim));
  double edge[3] = {0.0, 0.0, 0.0};
  int counts[3] = {1, 1, 1}, periodic[3] = {0, 0, 0};
  double* rel[3] = {nullptr, nullptr, nullptr};
  int32_t* cell[3] = {nullptr, nullptr, nullptr};
  const double* dx[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < grid->dim; ++k) {
    // CellGrid::edge_phys (cell_grid.cpp:9-34): span / count on a periodic axis, else 2h
    edge[k] = grid->periodic[k] ? (grid->hi[k] - grid->lo[k]) / grid->counts[k] : grid->radius_phys;
    counts[k] = grid->counts[k];
    periodic[k] = grid->periodic[k] != 0;
    rel[k] = d_rel[k];
    cell[k] = d_cell[k];
    dx[k] = d_dx[k];
  }
  CK(cudaMemsetAsync(d_status, 0xFF, sizeof(unsigned long long), ctx->stream));
  ctx->launches += launch_update_relative(n, grid->dim, precision, rel, cell, dx, edge, counts,
                                          periodic, d_status, ctx->stream);
  CKL();
  return SPHX_OK;
}

int sphx_update_relative(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                         double* const rel[3], int32_t* const cell[3], const double* const dx[3],
                         int32_t precision) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  const int dim = grid->dim;
  double* d_rel[3] = {nullptr, nullptr, nullptr};
  int32_t* d_cell[3] = {nullptr, nullptr, nullptr};
  const double* d_dx[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < dim; ++k) {
    TRY(upload(ctx, ctx->b_rel[k], rel[k], sizeof(double) * n));
    TRY(upload(ctx, ctx->b_cell[k], cell[k], sizeof(int32_t) * n));
    TRY(upload(ctx, ctx->g_x[k], dx[k], sizeof(double) * n));
    d_rel[k] = ctx->b_rel[k].as<double>();
    d_cell[k] = ctx->b_cell[k].as<int32_t>();
    d_dx[k] = ctx->g_x[k].as<double>();
  }
  TRY(ctx->b_bad.ensure(sizeof(unsigned long long)));
  TRY(sphx_update_relative_device(ctx, grid, n, d_rel, d_cell, d_dx, precision,
                                  ctx->b_bad.as<unsigned long long>()));
  unsigned long long st = ~0ull;
  CK(cudaMemcpyAsync(&st, ctx->b_bad.p, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
  for (int k = 0; k < dim && n; ++k) {
    CK(cudaMemcpyAsync(rel[k], d_rel[k], sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(cell[k], d_cell[k], sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (st != ~0ull) {  // the message std::runtime_error carries (cell_grid.cpp:185, 196, 205)
    const int axis = (int)((st >> 1) & 3);
    return fail(SPHX_ERR_RUNTIME, (st & 1) ? "particle leaves the grid on axis " + std::to_string(axis)
                                           : "displacement skips a cell on axis " + std::to_string(axis));
  }
  return SPHX_OK;
}

int sphx_rebuild_members_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                const int32_t* const d_cell[3], int32_t* d_cell_of,
                                int32_t* d_cell_start, int32_t* d_items) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(SPHX_FP64, grid->dim));
  TRY(ctx->b_bad.ensure(sizeof(unsigned long long)));
  return run_binning(ctx, 2, *grid, n, nullptr, d_cell, nullptr, nullptr, d_cell_of, d_cell_start,
                     d_items, ctx->b_bad.as<unsigned long long>());
}


// ---------------- the mixed time step on device ----------------

int sphx_step_mixed_device(sphx_context* ctx, const sphx_grid_desc* grid, int32_t approach,
                           const sphx_mixed_state_device* state, const sphx_step_config* cfg,
                           int64_t* d_offsets, int32_t* d_items_out, int64_t capacity,
                           double* max_dx, int64_t* total) {
  TRY(check_ctx(ctx));
  if (!grid || !state || !cfg || !max_dx || !total)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(SPHX_FP64, grid->dim));
  if (approach < SPHX_APPROACH_I || approach > SPHX_APPROACH_III)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "unknown approach");
  // make_kernel (kernel.hpp:17-29): the step builds its KernelParams from ps.h()
  if (!(state->h > 0.0)) return fail(SPHX_ERR_INVALID_ARGUMENT, "smoothing length must be positive");
  const int64_t n = state->n;
  const int dim = grid->dim;
  if (cfg->n_moving < 0 || cfg->n_moving > n)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "n_moving exceeds the particle count");
  const int64_t n_mov = cfg->n_moving == 0 ? n : cfg->n_moving;
  *max_dx = 0.0;
  *total = 0;
  // (1) neighbour search per approach (dynamics.cpp:145-155)
  if (approach == SPHX_APPROACH_III)
    TRY(sphx_rcll_device(ctx, grid, n, state->rel, state->cell, state->items, state->cell_start,
                         SPHX_FP16, d_offsets, d_items_out, capacity));
  else
    TRY(sphx_cell_link_list_device(ctx, grid, n, state->x, state->h, state->items,
                                   state->cell_start, state->cell_of,
                                   approach == SPHX_APPROACH_I ? SPHX_FP64 : SPHX_FP16, d_offsets,
                                   d_items_out, capacity));
  int64_t tot = 0;
  if (n > 0) {
    CK(cudaMemcpyAsync(&tot, d_offsets + n, sizeof(tot), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  *total = tot;
  if (tot > capacity)  // nothing of the state has changed yet
    return fail(SPHX_ERR_CAPACITY, "neighbour table needs " + std::to_string(tot) +
                                       " entries, capacity " + std::to_string(capacity));
  if (n == 0) return SPHX_OK;

  // (2) EOS and FP64 rates (dynamics.cpp:157-164)
  StepArgs a;
  a.n = n;
  a.n_mov = n_mov;
  a.off = d_offsets;
  a.nb = d_items_out;
  TRY(ctx->s_stress.ensure(sizeof(double) * 18 * n));
  TRY(ctx->s_rates.ensure(sizeof(double) * 6 * n));
  TRY(ctx->s_dx.ensure(sizeof(double) * 3 * n));
  TRY(ctx->s_flags.ensure(2 * sizeof(unsigned long long)));
  double* sb = ctx->s_stress.as<double>();
  double* rb = ctx->s_rates.as<double>();
  for (int s = 0; s < 6; ++s) {
    a.sig[s] = sb + (size_t)s * n;
    a.tau[s] = sb + (size_t)(6 + s) * n;
    a.eps[s] = sb + (size_t)(12 + s) * n;
  }
  a.drho = rb;
  a.de = rb + n;
  a.inv_r2 = rb + (size_t)5 * n;
  for (int k = 0; k < 3; ++k) {
    a.x[k] = k < dim ? state->x[k] : nullptr;
    a.v[k] = k < dim ? state->v[k] : nullptr;
    a.dv[k] = rb + (size_t)(2 + k) * n;
    a.dx[k] = ctx->s_dx.as<double>() + (size_t)k * n;
    a.bf[k] = cfg->body_force[k];
    a.lo[k] = grid->lo[k];
    a.hi[k] = grid->hi[k];
    a.span[k] = grid->hi[k] - grid->lo[k];  // Domain::span (domain.hpp:32)
    a.per[k] = k < dim && grid->periodic[k];
  }
  a.m = state->m;
  a.rho = state->rho;
  a.p = state->p;
  a.e = state->e;
  a.h = state->h;
  const double pi = 3.141592653589793;
  const double h = state->h;
  a.alpha = dim == 1 ? 1.0 / h : (dim == 2 ? 15.0 / (7.0 * pi * h * h) : 3.0 / (2.0 * pi * h * h * h));
  a.mu = cfg->mu;
  a.c2 = cfg->c_sound * cfg->c_sound;
  a.rho0 = cfg->rho0;
  a.dt = cfg->dt;
  a.evolve_density = cfg->evolve_density != 0;
  a.compute_energy = cfg->compute_energy != 0;
  unsigned long long* flags = ctx->s_flags.as<unsigned long long>();
  a.maxdx = flags;
  CK(cudaMemsetAsync(flags, 0, sizeof(unsigned long long), ctx->stream));
  ctx->launches += launch_step_rates(dim, a, ctx->stream);
  CKL();
  // (3)-(4) kick, drift (dynamics.cpp:166-187)
  ctx->launches += launch_kick_drift(dim, a, ctx->stream);
  CKL();
  // (5) coordinate maintenance (dynamics.cpp:188-201)
  unsigned long long st = ~0ull;
  if (approach == SPHX_APPROACH_III) {
    double* dxp[3] = {a.dx[0], a.dx[1], a.dx[2]};
    TRY(sphx_update_relative_device(ctx, grid, n_mov, state->rel, state->cell, dxp, SPHX_FP64,
                                    flags + 1));
    TRY(sphx_rebuild_members_device(ctx, grid, n, state->cell, state->cell_of, state->cell_start,
                                    state->items));
  } else {
    TRY(sphx_rebin_device(ctx, grid, n, state->x, state->cell_of, state->cell_start, state->items,
                          reinterpret_cast<int64_t*>(flags + 1)));
  }
  unsigned long long hf[2] = {0, ~0ull};
  CK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::memcpy(max_dx, &hf[0], sizeof(double));
  st = hf[1];
  if (st != ~0ull) {
    if (approach == SPHX_APPROACH_III) {  // update_relative's runtime_error (cell_grid.cpp:185-205)
      const int axis = (int)((st >> 1) & 3);
      return fail(SPHX_ERR_RUNTIME, (st & 1) ? "particle leaves the grid on axis " + std::to_string(axis)
                                             : "displacement skips a cell on axis " + std::to_string(axis));
    }
    return fail(SPHX_ERR_OUT_OF_RANGE, "particle " + std::to_string(st) + " lies outside the grid");
  }
  return SPHX_OK;
}

// ---------------- multi-GPU slab path ----------------

int sphx_rcll_grad_normalized_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                     const double* const d_rel[3], const int32_t* const d_cell[3],
                                     const int32_t* d_items, const int32_t* d_cell_start,
                                     int32_t precision, const double* const d_x[3],
                                     const double* d_f, double h, double* const d_g[3],
                                     unsigned long long* d_degenerate) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  if (precision != SPHX_FP16 || grid->dim < 2)
    return fail(SPHX_ERR_INVALID_ARGUMENT,
                "the fused gradient runs on the FP16 RCLL search in 2-D or 3-D");
  if (!(h > 0.0)) return fail(SPHX_ERR_INVALID_ARGUMENT, "smoothing length must be positive");
  if (!d_degenerate) return fail(SPHX_ERR_INVALID_ARGUMENT, "null degenerate counter");
  // GradField::degenerate_count is always written, 0 for an empty system (gradient.cpp:44-50)
  CK(cudaMemsetAsync(d_degenerate, 0, sizeof(unsigned long long), ctx->stream));
  if (n == 0) return SPHX_OK;
  SweepArgs a;
  // the fused search reuses the table scratch: a later sphx_table_copy /
  // sphx_table_distances must not read it as the last rcll's table
  ctx->t_n = -1;
  ctx->t_rcll = false;
  TRY(ctx->t_offsets.ensure(sizeof(int64_t) * (n + 1)));
  // 2-D: the windowed kernels (window.cu) with the gradient in place of the
  // table; 3-D (and grids the window does not cover): encode + k_r16_grad
  TRY(run_prepare(ctx, MODE_RCLL, *grid, n, d_rel, d_cell, d_items, d_cell_start, nullptr,
                  precision, 0.0, ctx->t_offsets.as<int64_t>(), &a, RowSel(), grid->dim == 2));
  const double pi_ = 3.141592653589793;
  if (a.win2) {
    Win2Args w = win2_args(ctx, a);
    for (int k = 0; k < 2; ++k) {
      w.gx[k] = d_x[k];
      w.gout[k] = d_g[k];
    }
    w.gf = d_f;
    w.gdeg = d_degenerate;
    w.gh = h;
    w.galpha = 15.0 / (7.0 * pi_ * h * h);  // make_kernel (kernel.hpp:17-29), dim 2
    NvtxRange nvtx_grad("sphx.pack+grad");
    ctx->launches += launch_win2(w, true, ctx->stream, ctx->timing ? ctx->ev[1] : nullptr);
    CKL();
    if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    return SPHX_OK;
  }
  for (int k = 0; k < 3; ++k) {
    a.gx[k] = k < grid->dim ? d_x[k] : nullptr;
    a.gout[k] = k < grid->dim ? d_g[k] : nullptr;
  }
  a.gf = d_f;
  a.gdeg = d_degenerate;
  a.gh = h;
  // make_kernel (kernel.hpp:17-29), evaluated as the reference writes it
  const double pi = 3.141592653589793;
  a.galpha = grid->dim == 2 ? 15.0 / (7.0 * pi * h * h) : 3.0 / (2.0 * pi * h * h * h);
  ctx->launches += launch_rcll_grad(grid->dim, a, ctx->stream);
  CKL();
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  return SPHX_OK;
}

int sphx_rcll_grad_normalized(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                              const double* const rel[3], const int32_t* const cell[3],
                              int64_t n_items, const int32_t* items, const int32_t* cell_start,
                              int32_t precision, const double* const x[3], const double* f,
                              double h, double* const g[3], int64_t* degenerate) {
  TRY(check_ctx(ctx));
  if (!grid || !degenerate) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(precision, grid->dim));
  if (n_items != n) return fail(SPHX_ERR_INVALID_ARGUMENT, "grid membership is stale");
  const int dim = grid->dim;
  const int64_t C = cell_total(*grid);
  const double* d_rel[3] = {nullptr, nullptr, nullptr};
  const int32_t* d_cell[3] = {nullptr, nullptr, nullptr};
  const double* d_x[3] = {nullptr, nullptr, nullptr};
  double* d_g[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < dim; ++k) {
    TRY(upload(ctx, ctx->in_x[k], rel[k], sizeof(double) * n));
    TRY(upload(ctx, ctx->in_cell[k], cell[k], sizeof(int32_t) * n));
    TRY(upload(ctx, ctx->g_x[k], x[k], sizeof(double) * n));
    TRY(ctx->g_out[k].ensure(sizeof(double) * std::max<int64_t>(n, 1)));
    d_rel[k] = ctx->in_x[k].as<double>();
    d_cell[k] = ctx->in_cell[k].as<int32_t>();
    d_x[k] = ctx->g_x[k].as<double>();
    d_g[k] = ctx->g_out[k].as<double>();
  }
  TRY(upload(ctx, ctx->in_items, items, sizeof(int32_t) * n));
  TRY(upload(ctx, ctx->in_start, cell_start, sizeof(int32_t) * (C + 1)));
  TRY(upload(ctx, ctx->g_f, f, sizeof(double) * n));
  TRY(ctx->g_deg.ensure(sizeof(unsigned long long)));
  TRY(sphx_rcll_grad_normalized_device(ctx, grid, n, d_rel, d_cell, ctx->in_items.as<int32_t>(),
                                       ctx->in_start.as<int32_t>(), precision, d_x,
                                       ctx->g_f.as<double>(), h, d_g,
                                       ctx->g_deg.as<unsigned long long>()));
  for (int k = 0; k < dim; ++k)
    if (n) CK(cudaMemcpyAsync(g[k], d_g[k], sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  unsigned long long deg = 0;
  if (n) CK(cudaMemcpyAsync(&deg, ctx->g_deg.p, sizeof(deg), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *degenerate = (int64_t)deg;
  return SPHX_OK;
}

int sphx_rcll_distances_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                               const double* const d_rel[3], const int32_t* const d_cell[3],
                               int32_t precision, const int64_t* d_offsets,
                               const int32_t* d_items, double* d_dist) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  const GridConsts gc = grid_consts(*grid);
  const PrecConsts pc = make_consts(MODE_RCLL, precision, *grid, 0.0);
  double hc[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < grid->dim; ++k) hc[k] = grid->hc[k];
  ctx->launches += launch_rcll_distances(grid->dim, precision, n, gc, pc, hc, d_rel, d_cell,
                                         d_offsets, d_items, d_dist, ctx->stream);
  CKL();
  return SPHX_OK;
}

int sphx_table_distances(sphx_context* ctx, const sphx_grid_desc* grid, int32_t precision,
                         double* dist) {
  TRY(check_ctx(ctx));
  if (!grid || !dist) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  if (ctx->t_n < 0 || !ctx->t_rcll)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "no rcll table computed on this context");
  TRY(ctx->t_dist.ensure(sizeof(double) * std::max<int64_t>(ctx->t_total, 1)));
  const double* d_rel[3] = {nullptr, nullptr, nullptr};
  const int32_t* d_cell[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k < grid->dim; ++k) {
    d_rel[k] = ctx->in_x[k].as<double>();
    d_cell[k] = ctx->in_cell[k].as<int32_t>();
  }
  TRY(sphx_rcll_distances_device(ctx, grid, ctx->t_n, d_rel, d_cell, precision,
                                 ctx->t_offsets.as<int64_t>(), ctx->t_items.as<int32_t>(),
                                 ctx->t_dist.as<double>()));
  if (ctx->t_total)
    CK(cudaMemcpyAsync(dist, ctx->t_dist.p, sizeof(double) * ctx->t_total, cudaMemcpyDeviceToHost,
                       ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SPHX_OK;
}

int sphx_rcll_rows_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                          const double* const d_rel[3], const int32_t* const d_cell[3],
                          const int32_t* d_items, const int32_t* d_cell_start, int32_t precision,
                          const int32_t* d_ids, int64_t row0, int64_t nrows, int64_t* d_offsets,
                          int32_t* d_items_out, int64_t capacity) {
  TRY(check_ctx(ctx));
  if (!grid) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(precision, grid->dim));
  RowSel sel;
  sel.row0 = row0;
  sel.nrows = nrows;
  sel.ids = d_ids;
  SweepArgs a;
  TRY(run_prepare(ctx, MODE_RCLL, *grid, n, d_rel, d_cell, d_items, d_cell_start, nullptr,
                  precision, 0.0, d_offsets, &a, sel));
  return run_sweep(ctx, grid->dim, precision, MODE_RCLL, a, d_items_out, capacity);
}

int sphx_slab_assemble_device(sphx_context* ctx, const sphx_grid_desc* local, int32_t axis,
                              int64_t n_own, int64_t slot_below, int64_t slot_above,
                              int64_t n_slots, const int32_t* d_owned_start,
                              const int32_t* d_recv_below, const int32_t* d_recv_above,
                              int32_t* d_cell_start, int32_t* d_items, int32_t* const d_cell[3]) {
  TRY(check_ctx(ctx));
  if (!local || !d_owned_start || !d_cell_start || !d_items || !d_cell)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_prec_dim(SPHX_FP64, local->dim));
  if (axis < 0 || axis >= local->dim || local->counts[axis] < 3)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "bad slab axis");
  if (n_own < 0 || slot_below < n_own || slot_above < slot_below || n_slots < slot_above ||
      n_slots > INT32_MAX)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "bad slab slots");
  SlabArgs a;
  std::memset(&a, 0, sizeof(a));
  a.dim = local->dim;
  a.axis = axis;
  a.CL = 1;
  for (int k = 0; k < local->dim; ++k) {
    a.cnt[k] = local->counts[k];
    if (k != axis) a.CL *= local->counts[k];
  }
  a.nl = local->counts[axis] - 2;
  a.n_own = (int)n_own;
  a.slotB = (int)slot_below;
  a.slotA = (int)slot_above;
  a.n_slots = (int)n_slots;
  a.haveB = d_recv_below != nullptr;
  a.haveA = d_recv_above != nullptr;
  a.ocs = d_owned_start;
  a.rB = d_recv_below;
  a.rA = d_recv_above;
  a.start = d_cell_start;
  a.items = d_items;
  for (int k = 0; k < 3; ++k) a.cell[k] = k < local->dim ? d_cell[k] : nullptr;
  NvtxRange nvtx_slab("sphx.slab_assemble");
  ctx->launches += launch_slab_assemble(a, ctx->stream);
  CKL();
  return SPHX_OK;
}

int sphx_build_rel_coords_window_device(sphx_context* ctx, const sphx_grid_desc* global,
                                        const sphx_grid_desc* local, int32_t axis, int32_t layer0,
                                        int64_t n, const double* const d_x[3],
                                        double* const d_rel[3], int32_t* const d_cell[3],
                                        int32_t* d_cell_of, int32_t* d_cell_start,
                                        int32_t* d_items) {
  TRY(check_ctx(ctx));
  if (!global || !local) return fail(SPHX_ERR_INVALID_ARGUMENT, "null grid");
  TRY(check_prec_dim(SPHX_FP64, global->dim));
  if (axis < 0 || axis >= global->dim || local->dim != global->dim)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "bad slab window");
  for (int k = 0; k < global->dim; ++k)
    if (k != axis && local->counts[k] != global->counts[k])
      return fail(SPHX_ERR_INVALID_ARGUMENT, "slab grid differs from the global grid off the slab axis");
  if (local->counts[axis] < 1 || local->counts[axis] > global->counts[axis] + 2 || layer0 < -1 ||
      layer0 >= global->counts[axis])
    return fail(SPHX_ERR_INVALID_ARGUMENT, "slab window outside the global grid");
  TRY(ctx->b_bad.ensure(sizeof(unsigned long long)));
  const BinConsts w = window_consts(*global, *local, axis, layer0);
  return run_binning(ctx, 1, *local, n, d_x, nullptr, d_rel, d_cell, d_cell_of, d_cell_start,
                     d_items, ctx->b_bad.as<unsigned long long>(), &w);
}

int sphx_lattice_device(sphx_context* ctx, int32_t dim, const double lo[3], const double hi[3],
                        double ds, int64_t id0, int64_t count, double* const d_x[3]) {
  TRY(check_ctx(ctx));
  TRY(check_prec_dim(SPHX_FP64, dim));
  int64_t counts[3] = {1, 1, 1};
  for (int k = 0; k < dim; ++k) counts[k] = static_cast<int64_t>(std::floor((hi[k] - lo[k]) / ds + 0.5));
  const int64_t total = counts[0] * counts[1] * counts[2];
  if (id0 < 0 || count < 0 || id0 + count > total)
    return fail(SPHX_ERR_INVALID_ARGUMENT, "lattice id range outside the lattice");
  if (count == 0) return SPHX_OK;
  launch_lattice(dim, lo, ds, counts, id0, count, d_x, ctx->stream);
  CKL();
  ++ctx->launches;
  return SPHX_OK;
}

// ---------------- synthetic inputs (particle_system.cpp:31-77) ----------------

int sphx_build_lattice(int32_t dim, const double lo[3], const double hi[3], double ds,
                       double jitter, uint64_t seed, int64_t* n_out, double* x0, double* x1,
                       double* x2) {
  if (!n_out) return fail(SPHX_ERR_INVALID_ARGUMENT, "null argument");
  if (dim < 1 || dim > 3) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain dimension must be 1, 2 or 3");
  for (int k = 0; k < dim; ++k)
    if (!(lo[k] < hi[k])) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain bounds must satisfy lo < hi");
  if (!(ds > 0.0)) return fail(SPHX_ERR_INVALID_ARGUMENT, "ds must be positive");
  if (jitter < 0.0 || jitter >= 0.5) return fail(SPHX_ERR_INVALID_ARGUMENT, "jitter must be in [0, 0.5)");
  int64_t counts[3] = {1, 1, 1}, n = 1;
  for (int k = 0; k < dim; ++k) {
    if (ds > hi[k] - lo[k]) return fail(SPHX_ERR_INVALID_ARGUMENT, "ds exceeds the smallest domain span");
    counts[k] = static_cast<int64_t>(std::floor((hi[k] - lo[k]) / ds + 0.5));
    n *= counts[k];
  }
  *n_out = n;
  if (!x0) return SPHX_OK;  // size query
  double* xs[3] = {x0, x1, x2};
  std::mt19937_64 gen(seed);
  auto u01 = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };  // rng.hpp:15
  int64_t idx = 0;
  int64_t c[3];
  for (c[2] = 0; c[2] < counts[2]; ++c[2])
    for (c[1] = 0; c[1] < counts[1]; ++c[1])
      for (c[0] = 0; c[0] < counts[0]; ++c[0]) {
        for (int k = 0; k < dim; ++k) {
          double v = lo[k] + (static_cast<double>(c[k]) + 0.5) * ds;
          if (jitter > 0.0) v += jitter * ds * (2.0 * u01() - 1.0);
          xs[k][idx] = v;
        }
        ++idx;
      }
  return SPHX_OK;
}

uint64_t sphx_table_hash(const int64_t* offsets, int64_t n, const int32_t* items, int64_t total) {
  uint64_t x = 1469598103934665603ull;  // FNV-1a 64 over offsets (u64) then items (u32)
  for (int64_t i = 0; i <= n; ++i) {
    x ^= static_cast<uint64_t>(offsets[i]);
    x *= 1099511628211ull;
  }
  for (int64_t q = 0; q < total; ++q) {
    x ^= static_cast<uint32_t>(items[q]);
    x *= 1099511628211ull;
  }
  return x;
}

int sphx_build_random_uniform(int32_t dim, const double lo[3], const double hi[3], int64_t n,
                              uint64_t seed, double* ds_out, double* x0, double* x1, double* x2) {
  if (dim < 1 || dim > 3) return fail(SPHX_ERR_INVALID_ARGUMENT, "domain dimension must be 1, 2 or 3");
  if (n < 1) return fail(SPHX_ERR_INVALID_ARGUMENT, "n must be at least 1");
  double vol = 1.0;
  for (int k = 0; k < dim; ++k) vol *= hi[k] - lo[k];
  if (ds_out) *ds_out = std::pow(vol / static_cast<double>(n), 1.0 / dim);
  double* xs[3] = {x0, x1, x2};
  std::mt19937_64 gen(seed);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < dim; ++k)
      xs[k][i] = lo[k] + (hi[k] - lo[k]) * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
  return SPHX_OK;
}

}  // extern "C"
