// The mixed-precision time step on device: step_mixed
// (dynamics.cpp:136-203) after its neighbour search, with the state resident in
// HBM. Every kernel restates the reference's FP64 loops with explicit
// round-to-nearest operations in the reference's evaluation order (the library is
// built with --fmad=false), so every field is bit-identical to the reference:
//   k_eos         apply_eos                        dynamics.cpp:125-130
//   k_stress      assemble_newtonian_stress        dynamics.cpp:8-32, its three
//                 grad_normalized(v_a) calls (gradient.cpp:44-82) in one pass: the
//                 denominators and scales do not depend on the field
//   k_rates       rhs_density + rhs_momentum + rhs_energy over one walk of the row
//                 (dynamics.cpp:34-123); each sum keeps its own order
//   k_kick_drift  symplectic Euler kick, drift, periodic wrap, Eq. 9 displacement
//                 and the max-|dx| reduction (dynamics.cpp:166-187)
// kernel_grad / kernel_dwdr / make_kernel: kernel.hpp:17-64.

#include "common.cuh"

namespace sphx_dev {


// sym_index (dynamics.hpp:39-45)
__host__ __device__ constexpr int sym(int a, int b) {
  return a == b ? a : ((a < b ? a : b) == 0 ? ((a < b ? b : a) == 1 ? 3 : 4) : 5);
}

__device__ __forceinline__ double dwdr(double R, double alpha) {
  if (R < 1.0) return __dmul_rn(alpha, __dadd_rn(__dmul_rn(-2.0, R), __dmul_rn(__dmul_rn(1.5, R), R)));
  if (R < 2.0) {
    const double t = __dsub_rn(2.0, R);
    return __dmul_rn(-alpha, __dmul_rn(__dmul_rn(0.5, t), t));
  }
  return 0.0;
}

// kernel_grad(dx, kp) for dx = x_i - x_j
template <int D>
__device__ __forceinline__ void kgrad(const double (&dx)[3], double h, double ih, double alpha,
                                      double (&gw)[3]) {
  double r2 = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) r2 = __dadd_rn(r2, __dmul_rn(dx[k], dx[k]));
  const double r = __dsqrt_rn(r2);
#pragma unroll
  for (int k = 0; k < 3; ++k) gw[k] = 0.0;
  if (r == 0.0) return;
  const double R = div_by(r, h, ih);  // ih = RN(1/h)
  const double sc = __ddiv_rn(dwdr(R, alpha), __dmul_rn(h, r));
#pragma unroll
  for (int k = 0; k < D; ++k) gw[k] = __dmul_rn(sc, dx[k]);
}

// apply_eos, and 1/(rho rho) once per particle: rhs_momentum / rhs_energy evaluate
// the same expression for every pair (dynamics.cpp:74, :79, :103, :108)
__global__ void k_eos(int64_t n, const double* __restrict__ rho, double* __restrict__ p, double c2,
                      double rho0, double* __restrict__ inv_r2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = rho[i];
  p[i] = __dmul_rn(c2, __dsub_rn(r, rho0));
  inv_r2[i] = __ddiv_rn(1.0, __dmul_rn(r, r));
}

template <int D>
__global__ void __launch_bounds__(128) k_stress(StepArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double ih = __drcp_rn(a.h);
  double xi[3], vi[3];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    xi[k] = a.x[k][i];
    vi[k] = a.v[k][i];
  }
  double num[3][3] = {}, den[3] = {0.0, 0.0, 0.0}, scale[3] = {0.0, 0.0, 0.0};
  const int64_t e0 = a.off[i], e1 = a.off[i + 1];
  for (int64_t q = e0; q < e1; ++q) {
    const int j = __ldg(a.nb + q);
    double dx[3] = {0.0, 0.0, 0.0}, gw[3];
#pragma unroll
    for (int k = 0; k < D; ++k) dx[k] = __dsub_rn(xi[k], __ldg(a.x[k] + j));
    kgrad<D>(dx, a.h, ih, a.alpha, gw);
#pragma unroll
    for (int c = 0; c < D; ++c) {  // grad_normalized(v_c): num += (f_j - f_i) gw
      const double df = __dsub_rn(__ldg(a.v[c] + j), vi[c]);
#pragma unroll
      for (int k = 0; k < D; ++k) num[c][k] = __dadd_rn(num[c][k], __dmul_rn(df, gw[k]));
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      den[k] = __dadd_rn(den[k], __dmul_rn(-dx[k], gw[k]));
      scale[k] = __dadd_rn(scale[k], fabs(__dmul_rn(dx[k], gw[k])));
    }
  }
  double gv[3][3];  // gv[c][k] = d v_c / d x_k
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const bool degenerate = fabs(den[k]) < __dmul_rn(1e-14, scale[k] > 0.0 ? scale[k] : 1.0);
#pragma unroll
    for (int c = 0; c < D; ++c) gv[c][k] = degenerate ? 0.0 : __ddiv_rn(num[c][k], den[k]);
  }
  const double pi = a.p[i];
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int b = c; b < D; ++b) {
      const int s = sym(c, b);
      const double sum = __dadd_rn(gv[c][b], gv[b][c]);
      a.eps[s][i] = __dmul_rn(0.5, sum);
      const double t = __dmul_rn(a.mu, sum);
      a.tau[s][i] = t;
      a.sig[s][i] = __dsub_rn(t, c == b ? pi : 0.0);
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_rates(StepArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double ih = __drcp_rn(a.h);
  double xi[3], vi[3], si[6];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    xi[k] = a.x[k][i];
    vi[k] = a.v[k][i];
  }
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int b = c; b < D; ++b) si[sym(c, b)] = a.sig[sym(c, b)][i];
  const double rhoi = a.rho[i], pi = a.p[i];
  const double inv_i = a.inv_r2[i];
  double acc_rho = 0.0, acc_e = 0.0, acc_v[3] = {0.0, 0.0, 0.0};
  const int64_t e0 = a.off[i], e1 = a.off[i + 1];
  for (int64_t q = e0; q < e1; ++q) {
    const int j = __ldg(a.nb + q);
    double dx[3] = {0.0, 0.0, 0.0}, gw[3];
#pragma unroll
    for (int k = 0; k < D; ++k) dx[k] = __dsub_rn(xi[k], __ldg(a.x[k] + j));
    kgrad<D>(dx, a.h, ih, a.alpha, gw);
    const double mj = __ldg(a.m + j);
    double dv_dot = 0.0;  // rhs_density / rhs_energy
#pragma unroll
    for (int k = 0; k < D; ++k)
      dv_dot = __dadd_rn(dv_dot, __dmul_rn(__dsub_rn(vi[k], __ldg(a.v[k] + j)), gw[k]));
    acc_rho = __dadd_rn(acc_rho, __dmul_rn(mj, dv_dot));
    const double inv_j = __ldg(a.inv_r2 + j);
#pragma unroll
    for (int c = 0; c < D; ++c) {  // rhs_momentum
      double term = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) {
        const int s = sym(c, b);
        term = __dadd_rn(term, __dmul_rn(__dadd_rn(__dmul_rn(si[s], inv_i),
                                                   __dmul_rn(__ldg(a.sig[s] + j), inv_j)),
                                         gw[b]));
      }
      acc_v[c] = __dadd_rn(acc_v[c], __dmul_rn(mj, term));
    }
    if (a.compute_energy) {  // rhs_energy
      const double pj = __ldg(a.p + j);
      acc_e = __dadd_rn(acc_e, __dmul_rn(__dmul_rn(__dmul_rn(0.5, mj),
                                                   __dadd_rn(__dmul_rn(pi, inv_i), __dmul_rn(pj, inv_j))),
                                         dv_dot));
    }
  }
  if (a.evolve_density) a.drho[i] = acc_rho;
#pragma unroll
  for (int c = 0; c < D; ++c) a.dv[c][i] = __dadd_rn(acc_v[c], a.bf[c]);
  if (a.compute_energy) {
    double work = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        const int s = sym(c, b);
        work = __dadd_rn(work, __dmul_rn(a.tau[s][i], a.eps[s][i]));
      }
    a.de[i] = __dadd_rn(acc_e, __ddiv_rn(work, rhoi));
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_kick_drift(StepArgs a) {
  __shared__ double wmax[8];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0;
  if (i < a.n_mov) {
#pragma unroll
    for (int k = 0; k < D; ++k) a.v[k][i] = __dadd_rn(a.v[k][i], __dmul_rn(a.dv[k][i], a.dt));
    if (a.evolve_density) a.rho[i] = __dadd_rn(a.rho[i], __dmul_rn(a.drho[i], a.dt));
    if (a.compute_energy) a.e[i] = __dadd_rn(a.e[i], __dmul_rn(a.de[i], a.dt));
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double d = __dmul_rn(a.v[k][i], a.dt);
      mx = fmax(mx, fabs(d));
      double xk = __dadd_rn(a.x[k][i], d);
      if (a.per[k]) {
        if (xk >= a.hi[k]) xk = __dsub_rn(xk, a.span[k]);
        if (xk < a.lo[k]) xk = __dadd_rn(xk, a.span[k]);
      }
      a.x[k][i] = xk;
      a.dx[k][i] = d;
    }
  }
  // max |dx| over the block, then one atomic per block (|dx| >= 0: the IEEE bit
  // pattern orders like the value)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, wmax[w]);
    atomicMax(a.maxdx, (unsigned long long)__double_as_longlong(mx));
  }
}

// Launches the rates part of the step on `st`; returns the number of kernels.
int launch_step_rates(int dim, const StepArgs& a, cudaStream_t st) {
  if (a.n == 0) return 0;
  const unsigned g256 = (unsigned)((a.n + 255) / 256), g128 = (unsigned)((a.n + 127) / 128);
  k_eos<<<g256, 256, 0, st>>>(a.n, a.rho, a.p, a.c2, a.rho0, a.inv_r2);
#define RATES(D)                              \
  if (dim == D) {                             \
    k_stress<D><<<g128, 128, 0, st>>>(a);     \
    k_rates<D><<<g128, 128, 0, st>>>(a);      \
  }
  RATES(1) RATES(2) RATES(3)
#undef RATES
  return 3;
}

int launch_kick_drift(int dim, const StepArgs& a, cudaStream_t st) {
  if (a.n_mov == 0) return 0;
  const unsigned g = (unsigned)((a.n_mov + 255) / 256);
  if (dim == 1) k_kick_drift<1><<<g, 256, 0, st>>>(a);
  if (dim == 2) k_kick_drift<2><<<g, 256, 0, st>>>(a);
  if (dim == 3) k_kick_drift<3><<<g, 256, 0, st>>>(a);
  return 1;
}

}  // namespace sphx_dev
