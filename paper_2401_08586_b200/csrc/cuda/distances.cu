// Per-pair distances of an RCLL neighbour table: for every entry (i, j) the value
// the reference's rcll compares against the cutoff, finish(acc) at the precision
// (nnps.cpp:321-346, :395-409), with the minimum-image cell offset the search used
// (dc = -off, nnps.cpp:359-362). For pairs that do not wrap a periodic axis this is
// exactly rel_distance(rc, i, j, grid, prec) (cell_grid.cpp:135-178).
//
// FP64: d = (ri - rj) * (0.5 hc) + dc * hc; acc += d * d; sqrt(acc).
// FP32: every step in float; cc = (float)(dc * hc); sqrtf.
// FP16: s = r16(ri - rj); t = r16(s * r16(hc/2)); d = r16(t + r16(dc hc));
//       acc = r16(acc + r16(d * d)); r16(sqrt(acc)) -- the square root is taken in
//       double and rounded once to binary16, as round16(std::sqrt(acc)) does.
// One thread per row; the distances are written in the table's entry order.

#include "common.cuh"

namespace sphx_dev {

template <int D, int P>
__global__ void k_rcll_distances(int64_t nrows, GridConsts g, PrecConsts pc, double hc0,
                                 double hc1, double hc2, const double* __restrict__ r0,
                                 const double* __restrict__ r1, const double* __restrict__ r2,
                                 const int32_t* __restrict__ c0, const int32_t* __restrict__ c1,
                                 const int32_t* __restrict__ c2, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ items, double* __restrict__ dist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const double* rel[3] = {r0, r1, r2};
  const int32_t* cel[3] = {c0, c1, c2};
  const double hc[3] = {hc0, hc1, hc2};
  double ri[3];
  int ci[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    ri[k] = __ldg(rel[k] + i);
    ci[k] = __ldg(cel[k] + i);
  }
  const int64_t e0 = __ldg(off + i), e1 = __ldg(off + i + 1);
  for (int64_t e = e0; e < e1; ++e) {
    const int j = __ldg(items + e);
    double accd = 0.0;
    float accf = 0.0f;
    __half acch = __ushort_as_half(0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int dc = ci[k] - __ldg(cel[k] + j);  // minimum image on a wrapping axis
      if (g.wrap[k]) {
        if (dc > 1) dc -= g.counts[k];
        else if (dc < -1) dc += g.counts[k];
      }
      const double rj = __ldg(rel[k] + j);
      if constexpr (P == FP64) {
        const double d = __dadd_rn(__dmul_rn(__dsub_rn(ri[k], rj), 0.5 * hc[k]),
                                   __dmul_rn((double)dc, hc[k]));
        accd = __dadd_rn(accd, __dmul_rn(d, d));
      } else if constexpr (P == FP32) {
        const float s = __fsub_rn(__double2float_rn(ri[k]), __double2float_rn(rj));
        const float t = __fmul_rn(s, pc.f_hh[k]);
        const float d = __fadd_rn(t, __double2float_rn(__dmul_rn((double)dc, hc[k])));
        accf = __fadd_rn(accf, __fmul_rn(d, d));
      } else {
        const __half s = __hsub_rn(__double2half(ri[k]), __double2half(rj));
        const __half t = __hmul_rn(s, __ushort_as_half(pc.h_hh[k]));
        const __half d = __hadd_rn(t, __double2half(__dmul_rn((double)dc, hc[k])));
        acch = __hadd_rn(acch, __hmul_rn(d, d));
      }
    }
    double r;
    if constexpr (P == FP64) r = __dsqrt_rn(accd);
    else if constexpr (P == FP32) r = (double)__fsqrt_rn(accf);
    else r = (double)__half2float(__double2half(__dsqrt_rn((double)__half2float(acch))));
    dist[e] = r;
  }
}

int launch_rcll_distances(int dim, int prec, int64_t nrows, const GridConsts& g,
                          const PrecConsts& pc, const double hc[3], const double* const rel[3],
                          const int32_t* const cell[3], const int64_t* off,
                          const int32_t* items, double* dist, cudaStream_t st) {
  if (nrows == 0) return 0;
  const unsigned nb = (unsigned)((nrows + 127) / 128);
#define LD(D, P)                                                                          \
  if (dim == D && prec == P) {                                                            \
    k_rcll_distances<D, P><<<nb, 128, 0, st>>>(nrows, g, pc, hc[0], hc[1], hc[2], rel[0],  \
                                                rel[1], rel[2], cell[0], cell[1], cell[2], \
                                                off, items, dist);                         \
    return 1;                                                                             \
  }
  LD(1, FP64) LD(2, FP64) LD(3, FP64) LD(1, FP32) LD(2, FP32) LD(3, FP32)
  LD(1, FP16) LD(2, FP16) LD(3, FP16)
#undef LD
  return 0;
}

}  // namespace sphx_dev
