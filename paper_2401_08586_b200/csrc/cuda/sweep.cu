// Fused NNPS sweep for sm_100a: candidate enumeration over the 3^d neighbour
// cells, exact reduced-precision distance test, per-row sort, single-pass CSR
// offsets (decoupled look-back) and the neighbour-list write -- one kernel.
//
// Reference semantics (paths relative to the reference's proj/):
//   rcll            nnps.cpp:283-416 (axis_term/finish :321-346, 2-D batch
//                   detail::range_f16_rel_2d nnps_batch.cpp:203-261)
//   cell_link_list  nnps.cpp:174-281 (dist_prec :91-124, batch range_*_abs_2d
//                   nnps_batch.cpp:119-201)
//   all_list        nnps.cpp:128-172
//   build_table     nnps.cpp:26-66 (rows ascending, int64 offsets)
//
// Thread <-> particle in particle (row) order, so the CSR rows a block produces
// are one contiguous run and the global offsets come from a single-pass
// decoupled look-back instead of a count/scan/fill triple. Hits are inserted
// in order into a per-thread row in shared memory (XOR-swizzled so both the
// per-thread insertions and the per-row warp copy-out are bank-conflict-free),
// then each warp streams its 32 rows to HBM with contiguous stores. Rows longer
// than CAP are recomputed straight into global memory (clustered inputs only).
//
// Bit-exactness: every arithmetic step uses an explicit round-to-nearest
// intrinsic (no FMA contraction; the reference is built without -march), FP16
// uses native binary16 ALU ops which keep subnormals, and sqrt(acc) < cutoff is
// replaced by the exact threshold test acc < thr (PrecConsts).

#include "common.cuh"

namespace sphx_dev {

// ------------------------------------------------------------------------------
// Packed coordinate layouts (HBM): FP16 2-D = half2 (4 B), FP16 3-D = half4 (8 B),
// FP32 = float/float2/float4, FP64 = double/double2/double4.
// ------------------------------------------------------------------------------
template <int D, int P>
struct Coord;
template <>
struct Coord<1, FP16> { using T = __half2; };
template <>
struct Coord<2, FP16> { using T = __half2; };
template <>
struct Coord<3, FP16> { using T = uint2; };
template <>
struct Coord<1, FP32> { using T = float; };
template <>
struct Coord<2, FP32> { using T = float2; };
template <>
struct Coord<3, FP32> { using T = float4; };
template <>
struct Coord<1, FP64> { using T = double; };
template <>
struct Coord<2, FP64> { using T = double2; };
template <>
struct Coord<3, FP64> { using T = double4; };

template <int D, int P>
__device__ __forceinline__ typename Coord<D, P>::T pack(const double v[3]);

template <>
__device__ __forceinline__ __half2 pack<1, FP16>(const double v[3]) {
  return __halves2half2(__double2half(v[0]), __ushort_as_half(0));
}
template <>
__device__ __forceinline__ __half2 pack<2, FP16>(const double v[3]) {
  return __halves2half2(__double2half(v[0]), __double2half(v[1]));
}
template <>
__device__ __forceinline__ uint2 pack<3, FP16>(const double v[3]) {
  const __half2 xy = __halves2half2(__double2half(v[0]), __double2half(v[1]));
  const __half2 z0 = __halves2half2(__double2half(v[2]), __ushort_as_half(0));
  return make_uint2(*reinterpret_cast<const unsigned*>(&xy), *reinterpret_cast<const unsigned*>(&z0));
}
template <>
__device__ __forceinline__ float pack<1, FP32>(const double v[3]) { return __double2float_rn(v[0]); }
template <>
__device__ __forceinline__ float2 pack<2, FP32>(const double v[3]) {
  return make_float2(__double2float_rn(v[0]), __double2float_rn(v[1]));
}
template <>
__device__ __forceinline__ float4 pack<3, FP32>(const double v[3]) {
  return make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]), 0.f);
}
template <>
__device__ __forceinline__ double pack<1, FP64>(const double v[3]) { return v[0]; }
template <>
__device__ __forceinline__ double2 pack<2, FP64>(const double v[3]) { return make_double2(v[0], v[1]); }
template <>
__device__ __forceinline__ double4 pack<3, FP64>(const double v[3]) {
  return make_double4(v[0], v[1], v[2], 0.0);
}

template <class T>
__device__ __forceinline__ T ldg(const void* base, int64_t s) {
  return __ldg(reinterpret_cast<const T*>(base) + s);
}
template <>
__device__ __forceinline__ double4 ldg<double4>(const void* base, int64_t s) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * s;
  const double2 a = __ldg(p), b = __ldg(p + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Generic per-axis access for the FP32/FP64 testers.
__device__ __forceinline__ float ax(float v, int) { return v; }
__device__ __forceinline__ float ax(float2 v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ float ax(float4 v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); }
__device__ __forceinline__ double ax(double v, int) { return v; }
__device__ __forceinline__ double ax(double2 v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ double ax(double4 v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); }

__device__ __forceinline__ float f_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float f_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float f_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double f_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double f_mul(double a, double b) { return __dmul_rn(a, b); }

template <int P>
struct Scalar;
template <>
struct Scalar<FP32> {
  using T = float;
  static __device__ __forceinline__ T hh(const PrecConsts& c, int k) { return c.f_hh[k]; }
  static __device__ __forceinline__ T cc(const PrecConsts& c, int k) { return c.f_cc[k]; }
  static __device__ __forceinline__ T sh(const PrecConsts& c, int k) { return c.f_sh[k]; }
  static __device__ __forceinline__ T thr(const PrecConsts& c) { return c.f_thr; }
};
template <>
struct Scalar<FP64> {
  using T = double;
  static __device__ __forceinline__ T hh(const PrecConsts& c, int k) { return c.d_hh[k]; }
  static __device__ __forceinline__ T cc(const PrecConsts& c, int k) { return c.d_cc[k]; }
  static __device__ __forceinline__ T sh(const PrecConsts& c, int k) { return c.d_sh[k]; }
  static __device__ __forceinline__ T thr(const PrecConsts& c) { return c.d_thr; }
};

__device__ __forceinline__ __half hbits(uint16_t b) { return __ushort_as_half(b); }

// ------------------------------------------------------------------------------
// Distance testers. Row = constants of one (dy, dz) row of neighbour cells; the
// x offset enters per candidate through the cell boundaries m1/m2 of the
// contiguous x-range (RCLL: dc_x = +1 for s < m1, 0 for s < m2, -1 after) or
// through the range's wrap direction wx (CLL shift).
// ------------------------------------------------------------------------------
template <int D, int P, int MODE>
struct Tester;

// ---- RCLL, FP16 (nnps.cpp:332-337, :406, :344; nnps_batch.cpp:238-258) ----
template <int D>
struct RcllHalfBase {
  __half2 ri_xy, hh_xy;
  __half ri_z, hh_z, ccp_x;
  uint16_t thr;
  struct Row {
    __half ccy, ccz;
  };
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    Row r;
    // cc = round16(dc * hc) with dc = -off (minimum image): +-round16(hc) or +0
    r.ccy = dy == 0 ? __ushort_as_half(0) : (dy < 0 ? hbits(a.c.h_cc[1]) : __hneg(hbits(a.c.h_cc[1])));
    r.ccz = dz == 0 ? __ushort_as_half(0) : (dz < 0 ? hbits(a.c.h_cc[2]) : __hneg(hbits(a.c.h_cc[2])));
    return r;
  }
  __device__ __forceinline__ __half ccx(int64_t s, int64_t m1, int64_t m2) const {
    const __half z = __ushort_as_half(0);
    return s < m1 ? ccp_x : (s < m2 ? z : __hneg(ccp_x));
  }
};

template <>
struct Tester<2, FP16, MODE_RCLL> : RcllHalfBase<2> {
  using C = __half2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    ri_xy = ldg<__half2>(a.pos_own, i);
    hh_xy = __halves2half2(hbits(a.c.h_hh[0]), hbits(a.c.h_hh[1]));
    ccp_x = hbits(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row& r, C rj, int64_t s, int64_t m1, int64_t m2, int) const {
    const __half2 sd = __hsub2_rn(ri_xy, rj);
    const __half2 t = __hmul2_rn(sd, hh_xy);
    const __half2 d = __hadd2_rn(t, __halves2half2(ccx(s, m1, m2), r.ccy));
    const __half2 q = __hmul2_rn(d, d);
    const __half acc = __hadd_rn(__low2half(q), __high2half(q));
    return __half_as_ushort(acc) < thr;
  }
};

template <>
struct Tester<1, FP16, MODE_RCLL> : RcllHalfBase<1> {
  using C = __half2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    ri_xy = ldg<__half2>(a.pos_own, i);
    hh_xy = __halves2half2(hbits(a.c.h_hh[0]), __ushort_as_half(0));
    ccp_x = hbits(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row&, C rj, int64_t s, int64_t m1, int64_t m2, int) const {
    const __half sd = __hsub_rn(__low2half(ri_xy), __low2half(rj));
    const __half t = __hmul_rn(sd, __low2half(hh_xy));
    const __half d = __hadd_rn(t, ccx(s, m1, m2));
    const __half q = __hmul_rn(d, d);
    return __half_as_ushort(q) < thr;
  }
};

template <>
struct Tester<3, FP16, MODE_RCLL> : RcllHalfBase<3> {
  using C = uint2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const uint2 o = ldg<uint2>(a.pos_own, i);
    ri_xy = *reinterpret_cast<const __half2*>(&o.x);
    ri_z = __low2half(*reinterpret_cast<const __half2*>(&o.y));
    hh_xy = __halves2half2(hbits(a.c.h_hh[0]), hbits(a.c.h_hh[1]));
    hh_z = hbits(a.c.h_hh[2]);
    ccp_x = hbits(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row& r, C c, int64_t s, int64_t m1, int64_t m2, int) const {
    const __half2 rj = *reinterpret_cast<const __half2*>(&c.x);
    const __half rz = __low2half(*reinterpret_cast<const __half2*>(&c.y));
    const __half2 sd = __hsub2_rn(ri_xy, rj);
    const __half2 t = __hmul2_rn(sd, hh_xy);
    const __half2 d = __hadd2_rn(t, __halves2half2(ccx(s, m1, m2), r.ccy));
    const __half2 q = __hmul2_rn(d, d);
    const __half sz = __hsub_rn(ri_z, rz);
    const __half tz = __hmul_rn(sz, hh_z);
    const __half dz = __hadd_rn(tz, r.ccz);
    const __half qz = __hmul_rn(dz, dz);
    const __half acc = __hadd_rn(__hadd_rn(__low2half(q), __high2half(q)), qz);
    return __half_as_ushort(acc) < thr;
  }
};

// ---- CLL / all_list, FP16 (dist_prec nnps.cpp:112-121; nnps_batch.cpp:145-157) ----
struct CllHalfRow {
  __half shy, shz;
  bool any;  // any nonzero shift on y/z in this row
};

__device__ __forceinline__ __half shift_half(const SweepArgs& a, int k, int w) {
  return w == 0 ? __ushort_as_half(0) : (w > 0 ? hbits(a.c.h_sh[k]) : __hneg(hbits(a.c.h_sh[k])));
}

template <int D>
struct CllHalfBase {
  __half2 xi_xy;
  __half xi_z;
  __half shx_p;
  uint16_t thr;
  using Row = CllHalfRow;
  __device__ __forceinline__ Row row(const SweepArgs& a, int, int, int wy, int wz) const {
    Row r;
    r.shy = shift_half(a, 1, wy);
    r.shz = shift_half(a, 2, wz);
    r.any = (wy != 0) || (wz != 0);
    return r;
  }
};

template <int M>
struct Tester2HalfCll : CllHalfBase<2> {
  using C = __half2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    xi_xy = ldg<__half2>(a.pos_own, i);
    shx_p = hbits(a.c.h_sh[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row& r, C xj, int64_t, int64_t, int64_t, int wx) const {
    if (r.any || wx != 0) {  // xj = round16(xj + shift) on the shifted axes
      const __half sx = wx == 0 ? __ushort_as_half(0) : (wx > 0 ? shx_p : __hneg(shx_p));
      xj = __hadd2_rn(xj, __halves2half2(sx, r.shy));
    }
    const __half2 d = __hsub2_rn(xi_xy, xj);
    const __half2 q = __hmul2_rn(d, d);
    const __half acc = __hadd_rn(__low2half(q), __high2half(q));
    return __half_as_ushort(acc) < thr;
  }
};
template <>
struct Tester<2, FP16, MODE_CLL> : Tester2HalfCll<MODE_CLL> {};
template <>
struct Tester<2, FP16, MODE_ALL> : Tester2HalfCll<MODE_ALL> {};

template <int M>
struct Tester1HalfCll : CllHalfBase<1> {
  using C = __half2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    xi_xy = ldg<__half2>(a.pos_own, i);
    shx_p = hbits(a.c.h_sh[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row&, C c, int64_t, int64_t, int64_t, int wx) const {
    __half xj = __low2half(c);
    if (wx != 0) xj = __hadd_rn(xj, wx > 0 ? shx_p : __hneg(shx_p));
    const __half d = __hsub_rn(__low2half(xi_xy), xj);
    const __half q = __hmul_rn(d, d);
    return __half_as_ushort(q) < thr;
  }
};
template <>
struct Tester<1, FP16, MODE_CLL> : Tester1HalfCll<MODE_CLL> {};
template <>
struct Tester<1, FP16, MODE_ALL> : Tester1HalfCll<MODE_ALL> {};

template <int M>
struct Tester3HalfCll : CllHalfBase<3> {
  using C = uint2;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const uint2 o = ldg<uint2>(a.pos_own, i);
    xi_xy = *reinterpret_cast<const __half2*>(&o.x);
    xi_z = __low2half(*reinterpret_cast<const __half2*>(&o.y));
    shx_p = hbits(a.c.h_sh[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ bool test(const Row& r, C c, int64_t, int64_t, int64_t, int wx) const {
    __half2 xj = *reinterpret_cast<const __half2*>(&c.x);
    __half zj = __low2half(*reinterpret_cast<const __half2*>(&c.y));
    if (r.any || wx != 0) {
      const __half sx = wx == 0 ? __ushort_as_half(0) : (wx > 0 ? shx_p : __hneg(shx_p));
      xj = __hadd2_rn(xj, __halves2half2(sx, r.shy));
      zj = __hadd_rn(zj, r.shz);
    }
    const __half2 d = __hsub2_rn(xi_xy, xj);
    const __half2 q = __hmul2_rn(d, d);
    const __half dz = __hsub_rn(xi_z, zj);
    const __half qz = __hmul_rn(dz, dz);
    const __half acc = __hadd_rn(__hadd_rn(__low2half(q), __high2half(q)), qz);
    return __half_as_ushort(acc) < thr;
  }
};
template <>
struct Tester<3, FP16, MODE_CLL> : Tester3HalfCll<MODE_CLL> {};
template <>
struct Tester<3, FP16, MODE_ALL> : Tester3HalfCll<MODE_ALL> {};

// ---- RCLL, FP32 / FP64 (nnps.cpp:324-331, :401-405, :342-343) ----
template <int D, int P>
struct TesterRcllScalar {
  using S = Scalar<P>;
  using T = typename S::T;
  using C = typename Coord<D, P>::T;
  T ri[3], hh[3], ccp_x, thr;
  struct Row {
    T ccy, ccz;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const C o = ldg<C>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      ri[k] = ax(o, k);
      hh[k] = S::hh(a.c, k);
    }
    ccp_x = S::cc(a.c, 0);
    thr = S::thr(a.c);
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    Row r;
    r.ccy = dy == 0 ? T(0) : (dy < 0 ? S::cc(a.c, 1) : -S::cc(a.c, 1));
    r.ccz = dz == 0 ? T(0) : (dz < 0 ? S::cc(a.c, 2) : -S::cc(a.c, 2));
    return r;
  }
  __device__ __forceinline__ bool test(const Row& r, C c, int64_t s, int64_t m1, int64_t m2, int) const {
    const T cc[3] = {s < m1 ? ccp_x : (s < m2 ? T(0) : -ccp_x), r.ccy, r.ccz};
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const T d = f_add(f_mul(f_sub(ri[k], ax(c, k)), hh[k]), cc[k]);
      const T q = f_mul(d, d);
      acc = k == 0 ? q : f_add(acc, q);  // 0 + q == q exactly (q >= +0)
    }
    return acc < thr;
  }
};

// ---- CLL / all_list, FP32 / FP64 (dist_prec nnps.cpp:94-111) ----
template <int D, int P>
struct TesterCllScalar {
  using S = Scalar<P>;
  using T = typename S::T;
  using C = typename Coord<D, P>::T;
  T xi[3], shx, thr;
  struct Row {
    T shy, shz;
    bool any;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const C o = ldg<C>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) xi[k] = ax(o, k);
    shx = S::sh(a.c, 0);
    thr = S::thr(a.c);
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int, int, int wy, int wz) const {
    Row r;
    r.shy = wy == 0 ? T(0) : (wy > 0 ? S::sh(a.c, 1) : -S::sh(a.c, 1));
    r.shz = wz == 0 ? T(0) : (wz > 0 ? S::sh(a.c, 2) : -S::sh(a.c, 2));
    r.any = wy != 0 || wz != 0;
    return r;
  }
  __device__ __forceinline__ bool test(const Row& r, C c, int64_t, int64_t, int64_t, int wx) const {
    const T sh[3] = {wx == 0 ? T(0) : (wx > 0 ? shx : -shx), r.shy, r.shz};
    const bool shifted = r.any || wx != 0;
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      T xj = ax(c, k);
      // FP64 adds the shift unconditionally (x + 0.0 is exact); FP32 only when
      // nonzero (nnps.cpp:97, :106) -- adding +0 is harmless for both.
      if (shifted) xj = f_add(xj, sh[k]);
      const T d = f_sub(xi[k], xj);
      const T q = f_mul(d, d);
      acc = k == 0 ? q : f_add(acc, q);
    }
    return acc < thr;
  }
};

template <int D>
struct Tester<D, FP32, MODE_RCLL> : TesterRcllScalar<D, FP32> {};
template <int D>
struct Tester<D, FP64, MODE_RCLL> : TesterRcllScalar<D, FP64> {};
template <int D>
struct Tester<D, FP32, MODE_CLL> : TesterCllScalar<D, FP32> {};
template <int D>
struct Tester<D, FP64, MODE_CLL> : TesterCllScalar<D, FP64> {};
template <int D>
struct Tester<D, FP32, MODE_ALL> : TesterCllScalar<D, FP32> {};
template <int D>
struct Tester<D, FP64, MODE_ALL> : TesterCllScalar<D, FP64> {};

// ------------------------------------------------------------------------------
// Candidate enumeration: the 3^d neighbour cells of the particle's cell, in rows
// of up to three x-adjacent cells that are contiguous in the CSR arrays
// (linear cell index is x-fastest, cell_grid.hpp:74-78). Periodic x wraps split
// a row into two ranges. Emits every j != i that passes the distance test.
// ------------------------------------------------------------------------------
template <int D, int P, int MODE, class Emit>
__device__ __forceinline__ void enumerate(const SweepArgs& a, int i, Emit& emit) {
  using Tst = Tester<D, P, MODE>;
  using C = typename Tst::C;
  Tst tst;
  tst.init(a, i);

  auto scan = [&](const typename Tst::Row& row, int64_t b, int64_t e, int64_t m1, int64_t m2,
                  int wx) {
    for (int64_t s = b; s < e; ++s) {
      const C cand = ldg<C>(a.pos_s, s);
      if (tst.test(row, cand, s, m1, m2, wx)) {
        const int j = MODE == MODE_ALL ? (int)s : __ldg(a.pid_s + s);
        if (j != i) emit(j);
      }
    }
  };

  if (MODE == MODE_ALL) {
    const typename Tst::Row row = tst.row(a, 0, 0, 0, 0);
    scan(row, 0, a.n, 0, 0, 0);
    return;
  }

  int ci[3] = {0, 0, 0};
  if (MODE == MODE_RCLL) {
#pragma unroll
    for (int k = 0; k < D; ++k) ci[k] = __ldg(a.cellk[k] + i);
  } else {
    int lin = __ldg(a.cell_of + i);  // nnps.cpp:205-209
#pragma unroll
    for (int k = 0; k < D; ++k) {
      ci[k] = lin % a.g.counts[k];
      lin /= a.g.counts[k];
    }
  }
  const int nx = a.g.counts[0], ny = a.g.counts[1], nz = a.g.counts[2];
  const int32_t* st = a.cell_start;
  const int dz_lo = D > 2 ? -1 : 0, dz_hi = D > 2 ? 1 : 0;
  const int dy_lo = D > 1 ? -1 : 0, dy_hi = D > 1 ? 1 : 0;
  for (int dz = dz_lo; dz <= dz_hi; ++dz) {
    int cz = ci[2] + dz, wz = 0;
    if (D > 2) {
      if (cz < 0) {
        if (!a.g.wrap[2]) continue;
        cz += nz;
        wz = -1;
      } else if (cz >= nz) {
        if (!a.g.wrap[2]) continue;
        cz -= nz;
        wz = 1;
      }
    }
    for (int dy = dy_lo; dy <= dy_hi; ++dy) {
      int cy = ci[1] + dy, wy = 0;
      if (D > 1) {
        if (cy < 0) {
          if (!a.g.wrap[1]) continue;
          cy += ny;
          wy = -1;
        } else if (cy >= ny) {
          if (!a.g.wrap[1]) continue;
          cy -= ny;
          wy = 1;
        }
      }
      const typename Tst::Row row = tst.row(a, dy, dz, wy, wz);
      const int64_t rb = (int64_t)(D > 2 ? cz : 0) * ny * nx + (int64_t)(D > 1 ? cy : 0) * nx;
      const int cx = ci[0];
      if (!a.g.wrap[0] || (cx > 0 && cx < nx - 1)) {
        const int lo = cx > 0 ? cx - 1 : 0, hi = cx + 1 < nx ? cx + 1 : nx - 1;
        scan(row, __ldg(st + rb + lo), __ldg(st + rb + hi + 1), __ldg(st + rb + cx),
             __ldg(st + rb + cx + 1), 0);
      } else if (cx == 0) {
        // cell nx-1 seen one period below (dc_x = +1 / shift -span), then cells 0..1
        const int64_t b0 = __ldg(st + rb + nx - 1), e0 = __ldg(st + rb + nx);
        scan(row, b0, e0, e0, e0, -1);
        const int64_t b1 = __ldg(st + rb);
        scan(row, b1, __ldg(st + rb + 2), b1, __ldg(st + rb + 1), 0);
      } else {
        // cells nx-2..nx-1, then cell 0 one period above (dc_x = -1 / shift +span)
        const int64_t e1 = __ldg(st + rb + nx);
        scan(row, __ldg(st + rb + nx - 2), e1, __ldg(st + rb + nx - 1), e1, 0);
        const int64_t b0 = __ldg(st + rb);
        scan(row, b0, __ldg(st + rb + 1), b0, b0, 1);
      }
    }
  }
}

// Per-thread sorted row in shared memory; element q of thread t lives at
// t*CAP + (q & ~31) + ((q ^ t) & 31).
template <int CAP>
__device__ __forceinline__ int sidx(int t, int q) {
  return t * CAP + (q & ~31) + ((q ^ t) & 31);
}

template <int CAP>
struct SmemEmit {
  int32_t* S;
  int t;
  int k;
  __device__ __forceinline__ void operator()(int j) {
    if (k < CAP) {
      int q = k;
      while (q > 0) {
        const int v = S[sidx<CAP>(t, q - 1)];
        if (v <= j) break;
        S[sidx<CAP>(t, q)] = v;
        --q;
      }
      S[sidx<CAP>(t, q)] = j;
    }
    ++k;
  }
};

struct GlobalEmit {  // long rows: sorted insertion directly into the output row
  int32_t* row;
  int k;
  __device__ __forceinline__ void operator()(int j) {
    int q = k;
    while (q > 0) {
      const int v = row[q - 1];
      if (v <= j) break;
      row[q] = v;
      --q;
    }
    row[q] = j;
    ++k;
  }
};

template <int D, int P, int MODE, int BT, int CAP>
__global__ void __launch_bounds__(BT) k_sweep(SweepArgs a) {
  static_assert(BT % 32 == 0 && BT <= 1024 && CAP % 32 == 0, "shape");
  __shared__ int32_t S[BT * CAP];
  __shared__ int s_bid;
  __shared__ int s_woff[BT / 32];
  __shared__ long long s_base;
  __shared__ int s_btot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(a.block_counter, 1);
  __syncthreads();
  const int bid = s_bid;
  const int i = bid * BT + tid;

  SmemEmit<CAP> em{S, tid, 0};
  if (i < a.n) enumerate<D, P, MODE>(a, i, em);
  const int k = em.k;

  // block-wide exclusive scan of row lengths + single-pass global prefix
  const int incl = warp_inclusive_scan(k);
  if (lane == 31) s_woff[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < BT / 32 ? s_woff[lane] : 0;
    const int wi = warp_inclusive_scan(w);
    if (lane < BT / 32) s_woff[lane] = wi - w;
    const int btot = __shfl_sync(0xffffffffu, wi, BT / 32 - 1);
    const long long base = lookback_exclusive(a.tiles, bid, btot);
    if (lane == 0) {
      s_base = base;
      s_btot = btot;
    }
  }
  __syncthreads();
  const long long grow = s_base + s_woff[warp] + incl - k;
  if (i < a.n) {
    a.offsets[i] = grow;
    if (i == a.n - 1) a.offsets[a.n] = grow + k;
  }
  if (s_base + s_btot > a.capacity) return;  // caller grows the table and re-runs

  // each warp streams its 32 rows with contiguous stores
  __syncwarp();
  for (int r = 0; r < 32; ++r) {
    const int len = __shfl_sync(0xffffffffu, k, r);
    const long long rbase = __shfl_sync(0xffffffffu, grow, r);
    if (len > CAP) continue;
    const int t = warp * 32 + r;
    for (int q = lane; q < len; q += 32) a.items[rbase + q] = S[sidx<CAP>(t, q)];
  }
  if (k > CAP) {
    GlobalEmit ge{a.items + grow, 0};
    enumerate<D, P, MODE>(a, i, ge);
  }
}

// Encode: round coordinates into the precision and pack them, in particle order
// (own) and in CSR order (candidates). Also resets the look-back state.
// RCLL: src = RelCoords::rel (nnps.cpp:304-315). CLL/all: src = positions
// (round_coords nnps.cpp:75-89, packing :185-194).
template <int D, int P>
__global__ void k_encode(int n, const double* __restrict__ x0, const double* __restrict__ x1,
                         const double* __restrict__ x2, const int32_t* __restrict__ items,
                         void* pos_own, void* pos_s, unsigned long long* tiles, int ntiles,
                         int* counter) {
  using C = typename Coord<D, P>::T;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    double v[3] = {x0[t], D > 1 ? x1[t] : 0.0, D > 2 ? x2[t] : 0.0};
    reinterpret_cast<C*>(pos_own)[t] = pack<D, P>(v);
    if (items) {
      int j = items[t];
      if (j < 0 || j >= n) j = t;  // malformed membership: keep memory-safe
      double w[3] = {x0[j], D > 1 ? x1[j] : 0.0, D > 2 ? x2[j] : 0.0};
      reinterpret_cast<C*>(pos_s)[t] = pack<D, P>(w);
    }
  }
  if (t < ntiles) tiles[t] = 0ull;
  if (t == 0) *counter = 0;
}

template <int D>
struct Shape {
  static constexpr int BT = D == 3 ? 64 : 128;
  static constexpr int CAP = D == 3 ? 96 : 32;
};

// ------------------------------------------------------------------------------
// Host-side launchers (called from capi.cu)
// ------------------------------------------------------------------------------
int sweep_block_threads(int dim) { return dim == 3 ? Shape<3>::BT : Shape<2>::BT; }

template <int D, int P>
static void launch_encode_t(int n, const double* const x[3], const int32_t* items, void* own,
                            void* pos_s, unsigned long long* tiles, int ntiles, int* counter,
                            cudaStream_t st) {
  const int work = n > ntiles ? n : ntiles;
  const int blocks = (work + 255) / 256 > 0 ? (work + 255) / 256 : 1;
  k_encode<D, P><<<blocks, 256, 0, st>>>(n, x[0], x[1], x[2], items, own, pos_s, tiles, ntiles,
                                         counter);
}

void launch_encode(int dim, int prec, int n, const double* const x[3], const int32_t* items,
                   void* own, void* pos_s, unsigned long long* tiles, int ntiles, int* counter,
                   cudaStream_t st) {
#define ENC(D, P)                                                                      \
  if (dim == D && prec == P) {                                                         \
    launch_encode_t<D, P>(n, x, items, own, pos_s, tiles, ntiles, counter, st);        \
    return;                                                                            \
  }
  ENC(1, FP16) ENC(2, FP16) ENC(3, FP16) ENC(1, FP32) ENC(2, FP32) ENC(3, FP32)
  ENC(1, FP64) ENC(2, FP64) ENC(3, FP64)
#undef ENC
}

size_t coord_bytes(int dim, int prec) {
  if (prec == FP16) return dim == 3 ? 8 : 4;
  if (prec == FP32) return dim == 1 ? 4 : (dim == 2 ? 8 : 16);
  return dim == 1 ? 8 : (dim == 2 ? 16 : 32);
}

template <int D, int P, int M>
static void launch_sweep_t(const SweepArgs& a, cudaStream_t st) {
  const int blocks = (a.n + Shape<D>::BT - 1) / Shape<D>::BT;
  k_sweep<D, P, M, Shape<D>::BT, Shape<D>::CAP><<<blocks, Shape<D>::BT, 0, st>>>(a);
}

void launch_sweep(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) {
#define SW(D, P, M)                       \
  if (dim == D && prec == P && mode == M) { \
    launch_sweep_t<D, P, M>(a, st);       \
    return;                               \
  }
#define SWP(D, M) SW(D, FP16, M) SW(D, FP32, M) SW(D, FP64, M)
  SWP(1, MODE_RCLL) SWP(2, MODE_RCLL) SWP(3, MODE_RCLL)
  SWP(1, MODE_CLL) SWP(2, MODE_CLL) SWP(3, MODE_CLL)
  SWP(1, MODE_ALL) SWP(2, MODE_ALL) SWP(3, MODE_ALL)
#undef SWP
#undef SW
}

}  // namespace sphx_dev
