// Shared device-side definitions for the sm_100a NNPS kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sphx_dev {

enum { FP64 = 0, FP32 = 1, FP16 = 2 };
enum { MODE_RCLL = 0, MODE_CLL = 1, MODE_ALL = 2 };

// Precision constants of one NNPS call, computed on the host so that they are
// exactly the values the reference forms (nnps.cpp:287-295, :177-197):
//   hh[k]  = round_to(prec, 0.5*hc[k])          (RCLL half cell edge)
//   cc[k]  = round_to(prec, hc[k])              (RCLL centre difference, dc=+1;
//                                                dc=-1 is its negation, dc=0 is 0)
//   sh[k]  = round_to(prec, span[k])            (CLL periodic shift magnitude)
//   thr    = smallest acc with finish(acc) >= round_to(prec, cutoff): the
//            reference's sqrt-then-compare is replaced by the exact, monotone
//            test acc < thr (SURVEY.md 8(c) "threshold trick").
struct PrecConsts {
  uint16_t h_hh[3], h_cc[3], h_sh[3], h_thr;
  float f_hh[3], f_cc[3], f_sh[3], f_thr;
  double d_hh[3], d_cc[3], d_sh[3], d_thr;
};

struct GridConsts {
  int dim;
  int counts[3];
  int wrap[3];  // periodic(k) && count(k) > 2  (nnps.cpp:223, :364)
};

// Arguments of the sweep kernels (encode writes the candidate arrays, the
// single-pass sweep reads them).
struct SweepArgs {
  int n;
  GridConsts g;
  PrecConsts c;
  int2* tri;                  // [C] chunk run [x, y) of each cell's x-triple
  void* qc;                   // [chunks] records: coordinate quads per axis (x pre-shifted
                              // for CLL), then the RCLL x offset quad dc = cx_i - cx_j
  void* qtag;                 // [chunks] uint4 particle ids (~0 = sentinel)
  int64_t nchunks;            // chunks allocated for qc / qtag
  uint32_t* selfpos;          // [n] record index of particle i in its own-cell run (< 2^32)
  const void* pos_own;        // packed coords in particle order
  const int32_t* cellk[3];    // RCLL: RelCoords::cell[k] (particle order)
  const int32_t* cell_of;     // CLL:  CellGrid::cell_of  (particle order)
  int64_t* offsets;           // [nrows+1]
  int32_t* items;             // [capacity]
  int64_t capacity;
  int row0, nrows;            // rows produced: particles [row0, row0 + nrows)
  const int32_t* ids;         // output id of particle j (null: j) -- global ids of a slab
  const int32_t* order;       // CellGrid::items: the test kernel visits rows in cell order
  // fused NNPS -> grad_normalized (gradient.cpp:44-82)
  const double* gx[3];        // ParticleSystem::x(k)
  const double* gf;           // the field f
  double* gout[3];            // GradField::g[k]
  unsigned long long* gdeg;   // GradField::degenerate_count (accumulated)
  double gh, galpha;          // KernelParams h, alpha (make_kernel, kernel.hpp:17-29)
  unsigned long long* tiles;  // [tiles] look-back words (epoch-tagged, never cleared)
  unsigned long long* ticket; // tile ticket counter (monotone across calls)
  unsigned long long tick0;   // ticket value at this call's first tile
  unsigned epoch;             // this call's look-back epoch (1..65535)
  int32_t* xy_nch;            // 3-D FP16 RCLL encode: [C] chunks per xy run
  int32_t* xy_cstart;         //   [C+1] first chunk of each run (scan of xy_nch)
  unsigned long long* xy_tiles;  // scan look-back words + counter (zeroed per call)
  int32_t* rowk;              // [nrows] row lengths of the test pass (bit 31: words overflowed)
  unsigned* hitw;             // [W][nrows] hit words of the test pass
  int win2;                   // 2-D FP16 RCLL: the windowed path (window.cu), no encode
  const double* src[3];       // windowed path: RelCoords::rel[k]
  const int32_t* start;       // windowed path: CellGrid::cell_start
};

// Arguments of the windowed 2-D FP16 RCLL (capi.cu fills them).
struct Win2Args {
  int n;                      // particles (CSR size)
  int row0, nrows;            // rows produced: particles [row0, row0 + nrows)
  GridConsts g;
  PrecConsts c;
  const double* rel[2];       // RelCoords::rel[k] (particle order)
  const int32_t* cellk[2];    // RelCoords::cell[k]
  const int32_t* items;       // CellGrid::items (CSR)
 const int32_t* start;       // CellGrid::cell_start [C+1]
  __half* wxy;                // [n + 16] pair-interleaved binary16 x / y (CSR order)
  __half* wu;                 // [n + 16] CSR cell x of each record (binary16)
  int32_t* wid;               // [n + 16] candidate ids (CSR order; global ids of a slab)
  const int32_t* ids;         // output id of local particle j (null: j) -- a slab's global ids
  uint8_t* wrun;              // [C][32] run lists: positions of each x-triple in id order
  int32_t* wself;             // [n] CSR position of each particle (the inverse of items)
  int4* wcb;                  // [C] CSR boundaries of each x-triple: L | C | R | end (x = -1:
                              //     the triple wraps a periodic x axis)
  void* desc;                 // [tiles] W2Desc: each tile's bands and window rows (pack -> sweep)
  int bt, wcap, cscap, runcap;  // the sweep's tile size and shared-memory capacities
  // fused NNPS -> grad_normalized (gradient.cpp:44-82): no table, g per particle
  const double* gx[2];        // ParticleSystem::x(k)
  const double* gf;           // the field f
  double* gout[2];            // GradField::g[k]
  unsigned long long* gdeg;   // GradField::degenerate_count (accumulated)
  double gh, galpha;          // KernelParams h, alpha (make_kernel, kernel.hpp:17-29)
  int64_t* offsets;           // [nrows + 1]
  int32_t* out;               // [capacity]
  int64_t capacity;
  unsigned long long* tiles;  // look-back words (epoch-tagged, never cleared)
  unsigned epoch;
};

// Slab assembly after a halo exchange (slab.cu)
struct SlabArgs {
  int dim, axis, CL, nl;       // CL = cells per layer; nl = owned layers
  int cnt[3];                  // local grid counts (axis: nl + 2)
  int n_own, slotB, slotA;     // first slot of the lower / upper halo
  int haveB, haveA;            // 0: a wall, no halo on that side
  const int32_t* ocs;          // owned CSR start over layers 1..nl [nl*CL + 1], from 0
  const int32_t* rB;           // received cell_start slice of the lower halo [CL + 1]
  const int32_t* rA;           // ... of the upper halo
  int32_t* start;              // local cell_start [(nl + 2) * CL + 1]
  int32_t* items;              // local CSR -> slot [n_slots]
  int32_t* cell[3];            // RelCoords::cell of the halo slots (written)
  int n_slots;
};

// Look-back words carry flag and value in one 64-bit word, so relaxed gpu-scope
// accesses suffice. (An acquire load would compile to CCTL.IVALL -- an L1
// invalidation per spin iteration that evicts every warp's cached candidates.)
// RN(r / h) for a launch-constant h from y = RN(1/h) (__drcp_rn): two FMA
// residual corrections. After the first, q is within one ulp of r/h, so the
// second is Markstein's correctly rounded step (Handbook of Floating-Point
// Arithmetic, Markstein's theorem: y within half an ulp of 1/h, q within one ulp,
// the residual r - hq exact by FMA => RN(q + (r - hq) y) = RN(r/h)): the bits of
// __ddiv_rn(r, h) for normal operands, in five FP64 ops instead of its ~20.
__device__ __forceinline__ double div_by(double r, double h, double y) {
  double q = __dmul_rn(r, y);
  q = __fma_rn(__fma_rn(-q, h, r), y, q);
  return __fma_rn(__fma_rn(-q, h, r), y, q);
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int warp_inclusive_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Decoupled look-back (single-pass prefix over blocks in dynamic launch order).
// Called by all 32 lanes of one warp; returns the exclusive prefix of block `bid`.
// Tile word: [63:62] flag (1 = aggregate, 2 = inclusive prefix), [61:0] value.
__device__ __forceinline__ long long lookback_exclusive(unsigned long long* tiles, int bid,
                                                        long long block_total) {
  const unsigned long long AGG = 1ull << 62, PRE = 2ull << 62, VAL = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (bid == 0) {
    if (lane == 0) st_relaxed_u64(&tiles[0], PRE | (unsigned long long)block_total);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&tiles[bid], AGG | (unsigned long long)block_total);
  long long excl = 0;
  int p = bid - 1;
  unsigned backoff = 32;
  // windows of 32 predecessors; a window that is not fully published is re-polled
  // after a short sleep so that waiting warps do not steal issue slots
  while (true) {
    const int idx = p - lane;
    const unsigned long long st = idx >= 0 ? ld_relaxed_u64(&tiles[idx]) : PRE;
    const unsigned flag = (unsigned)(st >> 62);
    const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == 2u);
    const unsigned zero_mask = __ballot_sync(0xffffffffu, flag == 0u);
    const int first = pre_mask ? __ffs(pre_mask) - 1 : 32;
    const unsigned need = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (zero_mask & need) {
      __nanosleep(backoff);
      backoff = backoff < 1024 ? backoff * 2 : 1024;
      continue;
    }
    const long long v = lane <= first ? (long long)(st & VAL) : 0ll;
    excl += warp_sum_ll(v);
    if (first < 32) break;
    p -= 32;
  }
  if (lane == 0) st_relaxed_u64(&tiles[bid], PRE | (unsigned long long)(excl + block_total));
  return excl;
}

// Binning (binning.cu)
struct BinConsts {
  int dim;
  int counts[3];  // cell counts of the (local) CSR grid
  double hc[3], origin[3], lo[3], hi[3];
  double hd;
  // slab window (multi-GPU): cells are located on the global grid, then the
  // window axis coordinate becomes (c - win_lo) mod win_global
  int win_axis;  // -1: no window
  int win_lo, win_global;
  int loc_counts[3];  // counts used by locate (global grid)
};

struct LocateArgs {
  int n;
  BinConsts g;
  const double* x[3];
  const int32_t* cell_in[3];  // BIN_MEMBERS
  double* rel_out[3];         // BIN_REL
  int32_t* cell_out[3];       // BIN_REL
  int32_t* cell_of;
  int32_t* counts;  // [C], zeroed
  int32_t* slot;    // [n]
  unsigned long long* bad;  // BIN_REBIN: min out-of-grid index
};

// device time step (step.cu): the state, the step's table and its scratch
struct StepArgs {
  int64_t n = 0, n_mov = 0;
  const int64_t* off = nullptr;  // the step's neighbour table
  const int32_t* nb = nullptr;
  double* x[3] = {nullptr, nullptr, nullptr};
  double* v[3] = {nullptr, nullptr, nullptr};
  const double* m = nullptr;
  double* rho = nullptr;
  double* p = nullptr;
  double* e = nullptr;
  double* sig[6] = {};  // StressState (dynamics.hpp:33-37), sym_index order
  double* tau[6] = {};
  double* eps[6] = {};
  double* drho = nullptr;  // rates
  double* dv[3] = {nullptr, nullptr, nullptr};
  double* de = nullptr;
  double* dx[3] = {nullptr, nullptr, nullptr};  // Eq. 9 displacement of the step
  double h = 0, alpha = 0, mu = 0, c2 = 0, rho0 = 0, dt = 0;
  double bf[3] = {0, 0, 0};
  int evolve_density = 1, compute_energy = 0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, span[3] = {0, 0, 0};
  int per[3] = {0, 0, 0};
  unsigned long long* maxdx = nullptr;  // bits of the non-negative max |dx|
  double* inv_r2 = nullptr;  // 1 / (rho rho) per particle (rhs_momentum / rhs_energy)
};

}  // namespace sphx_dev
