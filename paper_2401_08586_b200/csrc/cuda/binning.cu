// Device cell binning and RCLL encoding for sm_100a.
//
// Replaces the reference's serial host loops (paths relative to proj/):
//   normalize_domain  cell_grid.hpp:16-24      (Eq. 5)
//   CellGrid::locate  cell_grid.cpp:36-64      (cell choice, Eq. 6 rel, tie break)
//   CellGrid::rebin   cell_grid.cpp:66-84      (+ out-of-grid check naming i)
//   build_rel_coords  cell_grid.cpp:114-133
//   rebuild_members   cell_grid.cpp:86-95
//   build_csr         cell_grid.cpp:97-108     (stable counting sort)
//
// Pipeline: k_locate (FP64 cell + rel per particle, histogram via atomics that
// also hand out a slot inside the cell) -> k_scan_counts (single-pass
// decoupled look-back exclusive scan -> cell_start) -> k_scatter -> k_cell_sort
// (restores ascending particle ids inside each cell, which is exactly the order
// the reference's stable serial counting sort produces).
//
// Every FP64 operation is an explicit round-to-nearest intrinsic so no FMA is
// formed: the cell choice decides the candidate set, so it must match bit for bit.

#include <climits>

#include "common.cuh"

namespace sphx_dev {

enum { BIN_REBIN = 0, BIN_REL = 1, BIN_MEMBERS = 2 };

// static_cast<int32_t>(double) as g++ emits it on x86-64 (cvttsd2si): NaN and
// out-of-range values give INT_MIN.
__device__ __forceinline__ int x86_cvt_i32(double q) {
  if (!(q >= -2147483648.0 && q < 2147483648.0)) return INT_MIN;
  return (int)q;
}

__device__ __forceinline__ double center_norm(const BinConsts& g, int k, int c) {
  return __dadd_rn(g.origin[k], __dmul_rn(__dadd_rn((double)c, 0.5), g.hc[k]));
}

__device__ __forceinline__ void locate_axis(const BinConsts& g, int k, double xn, int& cell,
                                            double& rel) {
  const double off = __dsub_rn(xn, g.origin[k]);
  int c = x86_cvt_i32(floor(__ddiv_rn(off, g.hc[k])));
  if (c < 0) c = 0;
  if (c >= g.loc_counts[k]) c = g.loc_counts[k] - 1;
  double r = __ddiv_rn(__dmul_rn(2.0, __dsub_rn(xn, center_norm(g, k, c))), g.hc[k]);
  if (r < -1.0 && c > 0) {
    --c;
    r = __ddiv_rn(__dmul_rn(2.0, __dsub_rn(xn, center_norm(g, k, c))), g.hc[k]);
  } else if (r > 1.0 && c + 1 < g.loc_counts[k]) {
    ++c;
    r = __ddiv_rn(__dmul_rn(2.0, __dsub_rn(xn, center_norm(g, k, c))), g.hc[k]);
  }
  if (r == -1.0 && c > 0) {  // shared face -> lower cell, rel = +1
    --c;
    r = 1.0;
  }
  cell = c;
  rel = r;
}

template <int MODE>
__global__ void k_locate(LocateArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const BinConsts& g = a.g;
  int c[3] = {0, 0, 0};
  if (MODE == BIN_MEMBERS) {
    for (int k = 0; k < g.dim; ++k) c[k] = a.cell_in[k][i];
  } else {
    bool outside = false;
    for (int k = 0; k < g.dim; ++k) {
      const double xn =
          __ddiv_rn(__dsub_rn(__dmul_rn(2.0, a.x[k][i]), __dadd_rn(g.hi[k], g.lo[k])), g.hd);
      if (MODE == BIN_REBIN) {
        const double off = __dsub_rn(xn, g.origin[k]);
        const double top = __dmul_rn((double)g.loc_counts[k], g.hc[k]);
        if (off < __dmul_rn(-1e-9, g.hc[k]) || off > __dadd_rn(top, __dmul_rn(1e-9, g.hc[k])))
          outside = true;
      }
      double r;
      locate_axis(g, k, xn, c[k], r);
      if (k == g.win_axis) {  // global layer -> slab-local layer (periodic wrap)
        int d = c[k] - g.win_lo;
        if (d < 0) d += g.win_global;
        else if (d >= g.counts[k]) d -= g.win_global;  // a window longer than the axis
        if (d < 0 || d >= g.counts[k]) d = g.counts[k] - 1;  // outside the window: malformed
        c[k] = d;
      }
      if (MODE == BIN_REL) {
        a.rel_out[k][i] = r;
        a.cell_out[k][i] = c[k];
      }
    }
    if (outside) {
      atomicMin(a.bad, (unsigned long long)i);
      a.cell_of[i] = -1;  // excluded from the scatter; the call reports the error
      return;
    }
  }
  long long lin = c[g.dim - 1];
  for (int k = g.dim - 2; k >= 0; --k) lin = lin * g.counts[k] + c[k];
  a.cell_of[i] = (int32_t)lin;
  a.slot[i] = atomicAdd(a.counts + lin, 1);
}

// Exclusive scan of C int32 counts into out[0..C] (out[C] = total).
constexpr int SCAN_BT = 256, SCAN_IT = 8;

__global__ void __launch_bounds__(SCAN_BT) k_scan_counts(const int32_t* __restrict__ in,
                                                         int32_t* __restrict__ out, int64_t C,
                                                         unsigned long long* tiles,
                                                         int* counter) {
  __shared__ int s_bid;
  __shared__ int s_woff[SCAN_BT / 32];
  __shared__ long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(counter, 1);
  __syncthreads();
  const int bid = s_bid;
  const int64_t b0 = (int64_t)bid * SCAN_BT * SCAN_IT + (int64_t)tid * SCAN_IT;
  int v[SCAN_IT];
  int sum = 0;
#pragma unroll
  for (int q = 0; q < SCAN_IT; ++q) {
    v[q] = b0 + q < C ? in[b0 + q] : 0;
    sum += v[q];
  }
  const int incl = warp_inclusive_scan(sum);
  if (lane == 31) s_woff[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < SCAN_BT / 32 ? s_woff[lane] : 0;
    const int wi = warp_inclusive_scan(w);
    if (lane < SCAN_BT / 32) s_woff[lane] = wi - w;
    const int btot = __shfl_sync(0xffffffffu, wi, SCAN_BT / 32 - 1);
    const long long base = lookback_exclusive(tiles, bid, btot);
    if (lane == 0) s_base = base;
  }
  __syncthreads();
  long long run = s_base + s_woff[warp] + incl - sum;
#pragma unroll
  for (int q = 0; q < SCAN_IT; ++q) {
    if (b0 + q < C) out[b0 + q] = (int32_t)run;
    run += v[q];
    if (b0 + q == C - 1) out[C] = (int32_t)run;
  }
  if (C == 0 && bid == 0 && tid == 0) out[0] = 0;
}

__global__ void k_scatter(int n, const int32_t* __restrict__ cell_of, const int32_t* __restrict__ slot,
                          const int32_t* __restrict__ start, int32_t* __restrict__ items) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && cell_of[i] >= 0) items[start[cell_of[i]] + slot[i]] = i;
}

// Ascending ids inside each cell (the serial stable counting sort's order).
__global__ void k_cell_sort(int64_t C, const int32_t* __restrict__ start, int32_t* items) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int b = start[c], e = start[c + 1];
  for (int p = b + 1; p < e; ++p) {
    const int x = items[p];
    int q = p;
    while (q > b && items[q - 1] > x) {
      items[q] = items[q - 1];
      --q;
    }
    items[q] = x;
  }
}

// Un-jittered lattice sites [id0, id0 + count) of build_lattice
// (particle_system.cpp:49-56): x_k = lo_k + (c_k + 0.5) * ds, x fastest.
// Lets each rank of a slab run create its own slab of a lattice directly in HBM.
struct LatticeArgs {
  int dim;
  double lo[3], ds;
  long long counts[3];
  long long id0, count;
  double* x[3];
};

__global__ void k_lattice(LatticeArgs a) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.count) return;
  long long id = a.id0 + t;
  for (int k = 0; k < a.dim; ++k) {
    const long long c = id % a.counts[k];
    id /= a.counts[k];
    a.x[k][t] = __dadd_rn(a.lo[k], __dmul_rn(__dadd_rn((double)c, 0.5), a.ds));
  }
}

// ------------------------------------------------------------------------------
// Host launchers
// ------------------------------------------------------------------------------
int64_t scan_tiles(int64_t C) { return (C + SCAN_BT * SCAN_IT - 1) / (SCAN_BT * SCAN_IT); }

void launch_locate(int mode, const LocateArgs& a, cudaStream_t st) {
  const int blocks = (a.n + 255) / 256;
  if (blocks == 0) return;
  if (mode == BIN_REBIN) k_locate<BIN_REBIN><<<blocks, 256, 0, st>>>(a);
  else if (mode == BIN_REL) k_locate<BIN_REL><<<blocks, 256, 0, st>>>(a);
  else k_locate<BIN_MEMBERS><<<blocks, 256, 0, st>>>(a);
}

// tiles/counter must be zeroed before (they are: the caller memsets them).
void launch_scan_counts(const int32_t* in, int32_t* out, int64_t C, unsigned long long* tiles,
                        int* counter, cudaStream_t st) {
  int64_t blocks = scan_tiles(C);
  if (blocks == 0) blocks = 1;
  k_scan_counts<<<(unsigned)blocks, SCAN_BT, 0, st>>>(in, out, C, tiles, counter);
}

void launch_scatter_sort(int n, int64_t C, const int32_t* cell_of, const int32_t* slot,
                         const int32_t* start, int32_t* items, cudaStream_t st) {
  if (n > 0) k_scatter<<<(n + 255) / 256, 256, 0, st>>>(n, cell_of, slot, start, items);
  if (C > 0) k_cell_sort<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(C, start, items);
}

void launch_lattice(int dim, const double lo[3], double ds, const int64_t counts[3], int64_t id0,
                    int64_t count, double* const x[3], cudaStream_t st) {
  LatticeArgs a;
  a.dim = dim;
  a.ds = ds;
  a.id0 = id0;
  a.count = count;
  for (int k = 0; k < 3; ++k) {
    a.lo[k] = k < dim ? lo[k] : 0.0;
    a.counts[k] = counts[k];
    a.x[k] = k < dim ? x[k] : nullptr;
  }
  k_lattice<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(a);
}

}  // namespace sphx_dev
