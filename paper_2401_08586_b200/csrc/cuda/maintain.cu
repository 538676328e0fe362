// Device RCLL maintenance: the per-step Eq. 8 migration of
// the relative coordinates, update_relative (cell_grid.cpp:180-212), for every
// particle of a step at once, so that RelCoords stay resident in HBM across
// steps (step_mixed, dynamics.cpp:191-198; the paper's "no re-normalisation").
//
// Per particle and axis, exactly as the reference:
//   |dx| < edge_phys, else "displacement skips a cell on axis k";
//   inc = round_to(prec, 2 dx / edge); r = round_to(prec, rel + inc);
//   r > 1: r -= 2, cell + 1;  r < -1: r += 2, cell - 1 (exact in every precision);
//   leaving a non-periodic axis: "particle leaves the grid on axis k".
// The reference throws at the first offending (particle, axis) in index order;
// here every particle is processed and the lowest (particle, axis, kind) key is
// reported through *status (~0: none).

#include "common.cuh"

namespace sphx_dev {

__device__ __forceinline__ double round_prec(int prec, double x) {
  if (prec == FP64) return x;
  if (prec == FP32) return (double)__double2float_rn(x);
  return (double)__half2float(__double2half(x));  // RNE to binary16, subnormals kept
}

__global__ void k_update_relative(int64_t n, int dim, int prec, double* r0, double* r1, double* r2,
                                  int32_t* c0, int32_t* c1, int32_t* c2, const double* dx0,
                                  const double* dx1, const double* dx2, double e0, double e1,
                                  double e2, int n0, int n1, int n2, int p0, int p1, int p2,
                                  unsigned long long* status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* rel[3] = {r0, r1, r2};
  int32_t* cel[3] = {c0, c1, c2};
  const double* dxs[3] = {dx0, dx1, dx2};
  const double edge[3] = {e0, e1, e2};
  const int cnt[3] = {n0, n1, n2}, per[3] = {p0, p1, p2};
  for (int k = 0; k < dim; ++k) {
    const double dx = dxs[k][i];
    if (!(fabs(dx) < edge[k])) {  // kind 0: skips a cell
      atomicMin(status, ((unsigned long long)i << 3) | ((unsigned long long)k << 1));
      return;
    }
    const double inc = round_prec(prec, __ddiv_rn(__dmul_rn(2.0, dx), edge[k]));
    double r = round_prec(prec, __dadd_rn(rel[k][i], inc));
    int c = cel[k][i];
    if (r > 1.0) {
      r = __dsub_rn(r, 2.0);
      if (++c >= cnt[k]) {
        if (per[k]) {
          c = 0;
        } else {  // kind 1: leaves the grid
          atomicMin(status, ((unsigned long long)i << 3) | ((unsigned long long)k << 1) | 1ull);
          return;
        }
      }
    } else if (r < -1.0) {
      r = __dadd_rn(r, 2.0);
      if (--c < 0) {
        if (per[k]) {
          c = cnt[k] - 1;
        } else {
          atomicMin(status, ((unsigned long long)i << 3) | ((unsigned long long)k << 1) | 1ull);
          return;
        }
      }
    }
    rel[k][i] = r;
    cel[k][i] = c;
  }
}

int launch_update_relative(int64_t n, int dim, int prec, double* const rel[3],
                           int32_t* const cell[3], const double* const dx[3],
                           const double edge[3], const int counts[3], const int periodic[3],
                           unsigned long long* status, cudaStream_t st) {
  if (n == 0) return 0;
  k_update_relative<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      n, dim, prec, rel[0], rel[1], rel[2], cell[0], cell[1], cell[2], dx[0], dx[1], dx[2],
      edge[0], edge[1], edge[2], counts[0], counts[1], counts[2], periodic[0], periodic[1],
      periodic[2], status);
  return 1;
}

}  // namespace sphx_dev
