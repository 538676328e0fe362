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
// Candidate layout ("x-triples"). k_encode_tri builds, for every cell c, one
// record run holding the members of the x-neighbour cells (cx-1, cx, cx+1) --
// wrapped on a periodic x axis -- merged by particle id. Each record carries the
// packed coordinates and a tag = id << 2 | code, code = x cell offset + 1 (RCLL:
// dc_x = cx_i - cx_j; CLL: the periodic wrap direction). A particle's candidates
// are then 3 (2-D) or 9 (3-D) id-ascending runs, one per (dy, dz) row, which for
// spatially coherent particle numberings are already nearly in global id order.
//
// Thread <-> particle in particle (row) order, so the CSR rows of a block are one
// contiguous run and the global offsets come from a single-pass decoupled
// look-back instead of a count/scan/fill triple. Hits are inserted in order into
// a per-thread row in shared memory (append fast path), each warp packs its 32
// rows contiguously and streams them to HBM with coalesced stores. Rows longer
// than CAP are recomputed straight into global memory (clustered inputs only).
//
// Bit-exactness: every arithmetic step uses an explicit round-to-nearest
// intrinsic (no FMA contraction; the reference is built without -march), FP16
// uses native binary16 ALU ops which keep subnormals, and sqrt(acc) < cutoff is
// replaced by the exact threshold test acc < thr (PrecConsts).

#include <climits>

#include "common.cuh"

namespace sphx_dev {

// ------------------------------------------------------------------------------
// Packed coordinates: FP16 2-D = half2 (4 B), FP16 3-D = half4 (8 B), FP32 =
// float/float2/float4, FP64 = double/double2/double4.
// ------------------------------------------------------------------------------
template <int D, int P>
struct Coord;
template <> struct Coord<1, FP16> { using T = __half2; };
template <> struct Coord<2, FP16> { using T = __half2; };
template <> struct Coord<3, FP16> { using T = uint2; };
template <> struct Coord<1, FP32> { using T = float; };
template <> struct Coord<2, FP32> { using T = float2; };
template <> struct Coord<3, FP32> { using T = float4; };
template <> struct Coord<1, FP64> { using T = double; };
template <> struct Coord<2, FP64> { using T = double2; };
template <> struct Coord<3, FP64> { using T = double4; };

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
__device__ __forceinline__ T ldg(const void* base, int s) {
  return __ldg(reinterpret_cast<const T*>(base) + s);
}
template <>
__device__ __forceinline__ double4 ldg<double4>(const void* base, int s) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * s;
  const double2 a = __ldg(p), b = __ldg(p + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// ------------------------------------------------------------------------------
// Candidate records: coordinates + tag (id << 2 | code), one vector load each.
// ------------------------------------------------------------------------------
struct alignas(16) U4x2 {
  ulonglong2 a, b;
};

template <int D, int P>
struct Rec;
template <int D>
struct RecHalfLo {  // FP16, 1-D/2-D: {half2, tag} = 8 B
  using R = uint2;
  using C = __half2;
  static __device__ __forceinline__ R make(C c, unsigned tag) {
    return make_uint2(*reinterpret_cast<const unsigned*>(&c), tag);
  }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = *reinterpret_cast<const __half2*>(&r.x);
    tag = r.y;
  }
};
template <> struct Rec<1, FP16> : RecHalfLo<1> {};
template <> struct Rec<2, FP16> : RecHalfLo<2> {};
template <>
struct Rec<3, FP16> {  // {half2 xy, half2 z0, tag, 0} = 16 B
  using R = uint4;
  using C = uint2;
  static __device__ __forceinline__ R make(C c, unsigned tag) { return make_uint4(c.x, c.y, tag, 0u); }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = make_uint2(r.x, r.y);
    tag = r.z;
  }
};
template <>
struct Rec<1, FP32> {
  using R = uint2;
  using C = float;
  static __device__ __forceinline__ R make(C c, unsigned tag) { return make_uint2(__float_as_uint(c), tag); }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = __uint_as_float(r.x);
    tag = r.y;
  }
};
template <>
struct Rec<2, FP32> {
  using R = uint4;
  using C = float2;
  static __device__ __forceinline__ R make(C c, unsigned tag) {
    return make_uint4(__float_as_uint(c.x), __float_as_uint(c.y), tag, 0u);
  }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = make_float2(__uint_as_float(r.x), __uint_as_float(r.y));
    tag = r.z;
  }
};
template <>
struct Rec<3, FP32> {
  using R = uint4;
  using C = float4;
  static __device__ __forceinline__ R make(C c, unsigned tag) {
    return make_uint4(__float_as_uint(c.x), __float_as_uint(c.y), __float_as_uint(c.z), tag);
  }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z), 0.f);
    tag = r.w;
  }
};
template <>
struct Rec<1, FP64> {
  using R = ulonglong2;
  using C = double;
  static __device__ __forceinline__ R make(C c, unsigned tag) {
    return make_ulonglong2((unsigned long long)__double_as_longlong(c), tag);
  }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c = __longlong_as_double((long long)r.x);
    tag = (unsigned)r.y;
  }
};
template <int D>
struct RecF64Wide {  // {x, y, z|tag, tag|0} = 32 B
  using R = U4x2;
  using C = typename Coord<D, FP64>::T;
  static __device__ __forceinline__ R make(C c, unsigned tag) {
    R r;
    const double x = c.x, y = c.y;
    r.a = make_ulonglong2((unsigned long long)__double_as_longlong(x),
                          (unsigned long long)__double_as_longlong(y));
    if constexpr (D == 3)
      r.b = make_ulonglong2((unsigned long long)__double_as_longlong(c.z), tag);
    else
      r.b = make_ulonglong2(tag, 0ull);
    return r;
  }
  static __device__ __forceinline__ void split(const R& r, C& c, unsigned& tag) {
    c.x = __longlong_as_double((long long)r.a.x);
    c.y = __longlong_as_double((long long)r.a.y);
    if constexpr (D == 3) {
      c.z = __longlong_as_double((long long)r.b.x);
      tag = (unsigned)r.b.y;
    } else {
      tag = (unsigned)r.b.x;
    }
  }
};
template <> struct Rec<2, FP64> : RecF64Wide<2> {};
template <> struct Rec<3, FP64> : RecF64Wide<3> {};

template <class R>
__device__ __forceinline__ R ldr(const void* base, int s) {
  return __ldg(reinterpret_cast<const R*>(base) + s);
}
template <>
__device__ __forceinline__ U4x2 ldr<U4x2>(const void* base, int s) {
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(base) + 2 * s;
  U4x2 r;
  r.a = __ldg(p);
  r.b = __ldg(p + 1);
  return r;
}

// ------------------------------------------------------------------------------
// Scalar helpers
// ------------------------------------------------------------------------------
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

__device__ __forceinline__ __half hbits(unsigned b) { return __ushort_as_half((unsigned short)b); }
__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<const unsigned*>(&h); }
__device__ __forceinline__ __half2 u2h(unsigned u) { return *reinterpret_cast<const __half2*>(&u); }

// 16-bit value selected by a record code (0, 1, 2) from a 3-entry table packed
// in a 64-bit word: [-v, 0, +v] for dc/wrap = -1, 0, +1.
__device__ __forceinline__ unsigned lut16(unsigned long long lut, unsigned code) {
  return (unsigned)(lut >> (code * 16u)) & 0xFFFFu;
}
__device__ __forceinline__ unsigned long long make_lut16(unsigned v) {
  return (unsigned long long)(v ^ 0x8000u) | ((unsigned long long)v << 32);
}

// ------------------------------------------------------------------------------
// Distance testers: test(row, cand, code) -> hit. Row = constants of one (dy, dz)
// row of neighbour cells; code = the record's x offset + 1.
// ------------------------------------------------------------------------------
template <int D, int P, int MODE>
struct Tester;

// ---- RCLL, FP16 (nnps.cpp:332-337, :406, :344; nnps_batch.cpp:238-258) ----
// cc = round16(dc * hc), dc = -off (minimum image): +-round16(hc) or +0.
__device__ __forceinline__ __half cc_row_half(unsigned cc_bits, int d) {
  return d == 0 ? __ushort_as_half(0) : (d < 0 ? hbits(cc_bits) : hbits(cc_bits ^ 0x8000u));
}

template <>
struct Tester<2, FP16, MODE_RCLL> {
  using C = __half2;
  static constexpr bool kPair = true;
  __half2 ri, hh, rix2, riy2, hhx2, hhy2, thr2;
  unsigned long long cclut;
  unsigned thr;
  struct Row {
    __half2 ccy2;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    thr2 = __half2half2(hbits(a.c.h_thr));
    ri = ldg<__half2>(a.pos_own, i);
    hh = __halves2half2(hbits(a.c.h_hh[0]), hbits(a.c.h_hh[1]));
    rix2 = __low2half2(ri);
    riy2 = __high2half2(ri);
    hhx2 = __low2half2(hh);
    hhy2 = __high2half2(hh);
    cclut = make_lut16(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int, int, int) const {
    return Row{__half2half2(cc_row_half(a.c.h_cc[1], dy))};
  }
  __device__ __forceinline__ bool test(const Row& r, C rj, unsigned code) const {
    const __half2 t = __hmul2_rn(__hsub2_rn(ri, rj), hh);
    const __half2 cc = __halves2half2(hbits(lut16(cclut, code)), __low2half(r.ccy2));
    const __half2 d = __hadd2_rn(t, cc);
    const __half2 q = __hmul2_rn(d, d);
    return __half_as_ushort(__hadd_rn(__low2half(q), __high2half(q))) < thr;
  }
  // Two candidates per binary16x2 instruction (lanes = candidates); same op
  // sequence per candidate, x and y squares summed in axis order. The pair's
  // centre differences come from one byte permute of [-cc, 0 | +cc] indexed by
  // the record codes; the cutoff test is one packed compare (acc >= 0, NaN fails).
  __device__ __forceinline__ unsigned test2(const Row& r, C c0, C c1, unsigned k0,
                                            unsigned k1) const {
    const __half2 X = __lows2half2(c0, c1), Y = __highs2half2(c0, c1);
    const __half2 tx = __hmul2_rn(__hsub2_rn(rix2, X), hhx2);
    const __half2 ty = __hmul2_rn(__hsub2_rn(riy2, Y), hhy2);
    const unsigned sel = 0x1010u + 0x22u * k0 + 0x2200u * k1;
    const __half2 dx = __hadd2_rn(tx, u2h(__byte_perm((unsigned)cclut, (unsigned)(cclut >> 32), sel)));
    const __half2 dy = __hadd2_rn(ty, r.ccy2);
    const __half2 acc = __hadd2_rn(__hmul2_rn(dx, dx), __hmul2_rn(dy, dy));
    const unsigned mk = __hlt2_mask(acc, thr2);
    return (mk & 1u) | ((mk >> 15) & 2u);
  }
};

template <>
struct Tester<1, FP16, MODE_RCLL> {
  using C = __half2;
  __half ri, hh;
  unsigned long long cclut;
  unsigned thr;
  struct Row {};
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    ri = __low2half(ldg<__half2>(a.pos_own, i));
    hh = hbits(a.c.h_hh[0]);
    cclut = make_lut16(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ Row row(const SweepArgs&, int, int, int, int) const { return Row{}; }
  __device__ __forceinline__ bool test(const Row&, C rj, unsigned code) const {
    const __half t = __hmul_rn(__hsub_rn(ri, __low2half(rj)), hh);
    const __half d = __hadd_rn(t, hbits(lut16(cclut, code)));
    return __half_as_ushort(__hmul_rn(d, d)) < thr;
  }
};

template <>
struct Tester<3, FP16, MODE_RCLL> {
  using C = uint2;
  __half2 rxy, hxy;
  __half rz, hz;
  unsigned long long cclut;
  unsigned thr;
  struct Row {
    __half ccy, ccz;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const uint2 o = ldg<uint2>(a.pos_own, i);
    rxy = u2h(o.x);
    rz = __low2half(u2h(o.y));
    hxy = __halves2half2(hbits(a.c.h_hh[0]), hbits(a.c.h_hh[1]));
    hz = hbits(a.c.h_hh[2]);
    cclut = make_lut16(a.c.h_cc[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    return Row{cc_row_half(a.c.h_cc[1], dy), cc_row_half(a.c.h_cc[2], dz)};
  }
  __device__ __forceinline__ bool test(const Row& r, C c, unsigned code) const {
    const __half2 t = __hmul2_rn(__hsub2_rn(rxy, u2h(c.x)), hxy);
    const __half2 d = __hadd2_rn(t, __halves2half2(hbits(lut16(cclut, code)), r.ccy));
    const __half2 q = __hmul2_rn(d, d);
    const __half tz = __hmul_rn(__hsub_rn(rz, __low2half(u2h(c.y))), hz);
    const __half dz = __hadd_rn(tz, r.ccz);
    const __half acc = __hadd_rn(__hadd_rn(__low2half(q), __high2half(q)), __hmul_rn(dz, dz));
    return __half_as_ushort(acc) < thr;
  }
};

// ---- CLL / all_list, FP16 (dist_prec nnps.cpp:112-121; nnps_batch.cpp:145-157) ----
// xj = round16(xj + shift) on shifted axes; adding +0 elsewhere is harmless.
__device__ __forceinline__ __half sh_row_half(unsigned sh_bits, int w) {
  return w == 0 ? __ushort_as_half(0) : (w > 0 ? hbits(sh_bits) : hbits(sh_bits ^ 0x8000u));
}

template <int D>
struct TesterHalfCll {
  using C = typename Coord<D, FP16>::T;
  __half2 xi;
  __half xz;
  unsigned long long shlut;
  unsigned thr;
  struct Row {
    __half shy, shz;
    bool any;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    if constexpr (D == 3) {
      const uint2 o = ldg<uint2>(a.pos_own, i);
      xi = u2h(o.x);
      xz = __low2half(u2h(o.y));
    } else {
      xi = ldg<__half2>(a.pos_own, i);
    }
    shlut = make_lut16(a.c.h_sh[0]);
    thr = a.c.h_thr;
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int, int, int wy, int wz) const {
    return Row{sh_row_half(a.c.h_sh[1], wy), sh_row_half(a.c.h_sh[2], wz), wy != 0 || wz != 0};
  }
  __device__ __forceinline__ bool test(const Row& r, C c, unsigned code) const {
    const bool shifted = r.any || code != 1u;
    if constexpr (D == 1) {
      __half xj = __low2half(c);
      if (shifted) xj = __hadd_rn(xj, hbits(lut16(shlut, code)));
      const __half d = __hsub_rn(__low2half(xi), xj);
      return __half_as_ushort(__hmul_rn(d, d)) < thr;
    } else {
      __half2 xj;
      if constexpr (D == 3) xj = u2h(c.x); else xj = c;
      if (shifted) xj = __hadd2_rn(xj, __halves2half2(hbits(lut16(shlut, code)), r.shy));
      const __half2 d = __hsub2_rn(xi, xj);
      const __half2 q = __hmul2_rn(d, d);
      __half acc = __hadd_rn(__low2half(q), __high2half(q));
      if constexpr (D == 3) {
        __half zj = __low2half(u2h(c.y));
        if (shifted) zj = __hadd_rn(zj, r.shz);
        const __half dz = __hsub_rn(xz, zj);
        acc = __hadd_rn(acc, __hmul_rn(dz, dz));
      }
      return __half_as_ushort(acc) < thr;
    }
  }
};
template <int D> struct Tester<D, FP16, MODE_CLL> : TesterHalfCll<D> {};
template <int D> struct Tester<D, FP16, MODE_ALL> : TesterHalfCll<D> {};

// ---- RCLL, FP32 / FP64 (nnps.cpp:324-331, :401-405, :342-343) ----
template <int D, int P>
struct TesterRcllScalar {
  using S = Scalar<P>;
  using T = typename S::T;
  using C = typename Coord<D, P>::T;
  T ri[3], hh[3], ccp, thr;
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
    ccp = S::cc(a.c, 0);
    thr = S::thr(a.c);
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    Row r;
    r.ccy = dy == 0 ? T(0) : (dy < 0 ? S::cc(a.c, 1) : -S::cc(a.c, 1));
    r.ccz = dz == 0 ? T(0) : (dz < 0 ? S::cc(a.c, 2) : -S::cc(a.c, 2));
    return r;
  }
  __device__ __forceinline__ bool test(const Row& r, C c, unsigned code) const {
    const T cc[3] = {code == 2u ? ccp : (code == 0u ? -ccp : T(0)), r.ccy, r.ccz};
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
  __device__ __forceinline__ bool test(const Row& r, C c, unsigned code) const {
    const T sh[3] = {code == 2u ? shx : (code == 0u ? -shx : T(0)), r.shy, r.shz};
    const bool shifted = r.any || code != 1u;
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

template <int D> struct Tester<D, FP32, MODE_RCLL> : TesterRcllScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_RCLL> : TesterRcllScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_CLL> : TesterCllScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_CLL> : TesterCllScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_ALL> : TesterCllScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_ALL> : TesterCllScalar<D, FP64> {};

template <class T, class = void>
struct PairTraits {
  static constexpr bool value = false;
};
template <class T>
struct PairTraits<T, decltype((void)T::kPair)> {
  static constexpr bool value = T::kPair;
};

// ------------------------------------------------------------------------------
// Candidate enumeration. visit_rows calls fn(dy, dz, wy, wz, b, e) for each
// (dy, dz) row of the 3^d neighbourhood, wrapped or skipped per periodic(k)
// (nnps.cpp:359-372), with [b, e) the row's x-triple run of records.
// ------------------------------------------------------------------------------
template <int D, int MODE, class Fn>
__device__ __forceinline__ void visit_rows(const SweepArgs& a, int i, Fn&& fn) {
  if constexpr (MODE == MODE_ALL) {  // all_list: one "row" of every particle
    fn(0, 0, 0, 0, 0, a.n);
    return;
  } else {
    int ci[3] = {0, 0, 0};
    if constexpr (MODE == MODE_RCLL) {
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
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (ci[k] < 0 || ci[k] >= a.g.counts[k]) return;  // malformed cell: no candidates
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
        const int2 r = __ldg(a.tri + ((int64_t)cz * ny + cy) * nx + ci[0]);
        fn(dy, dz, wy, wz, r.x, r.y);
      }
    }
  }
}

// Candidate j of a chunk: the record s (RCLL/CLL) or particle s itself (all_list).
template <int D, int P, int MODE>
__device__ __forceinline__ void load_cand(const SweepArgs& a, int s,
                                          typename Tester<D, P, MODE>::C& c, unsigned& tg) {
  if constexpr (MODE == MODE_ALL) {
    c = ldg<typename Tester<D, P, MODE>::C>(a.pos_own, s);
    tg = ((unsigned)s << 2) | 1u;
  } else {
    using RT = Rec<D, P>;
    RT::split(ldr<typename RT::R>(a.rec, s), c, tg);
  }
}

// Distance tests of particle i against all its candidates, four records per
// chunk (arrays are padded so a chunk may run past its row end). For every chunk
// fn(m, tg, s) receives the hit mask m (bit u: record s+u is a neighbour j != i)
// and the four tags (j = tg >> 2).
template <int D, int P, int MODE, class ChunkFn>
__device__ __forceinline__ void scan_particle(const SweepArgs& a, int i, ChunkFn&& fn) {
  using Tst = Tester<D, P, MODE>;
  using C = typename Tst::C;
  Tst tst;
  tst.init(a, i);
  const unsigned selftag = (unsigned)i << 2;
  visit_rows<D, MODE>(a, i, [&](int dy, int dz, int wy, int wz, int b, int e) {
    const typename Tst::Row row = tst.row(a, dy, dz, wy, wz);
#pragma unroll 2
    for (int s = b; s < e; s += 4) {
      C c[4];
      unsigned tg[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_cand<D, P, MODE>(a, s + u, c[u], tg[u]);
      unsigned m;
      if constexpr (PairTraits<Tst>::value) {
        m = tst.test2(row, c[0], c[1], tg[0] & 3u, tg[1] & 3u) |
            (tst.test2(row, c[2], c[3], tg[2] & 3u, tg[3] & 3u) << 2);
      } else {
        m = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) m |= (unsigned)tst.test(row, c[u], tg[u] & 3u) << u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) m &= ~((unsigned)((tg[u] ^ selftag) < 4u) << u);  // j == i
      const int left = e - s;
      if (left < 4) m &= (1u << left) - 1u;
      fn(m, tg, s);
    }
  });
}

// ------------------------------------------------------------------------------
// Row assembly
// ------------------------------------------------------------------------------
template <int CAP>
struct SmemEmit {  // per-thread sorted row in shared memory, element q at row[q ^ x]
  int32_t* row;    // S + t*CAP
  int x;           // t & 31 (XOR swizzle: every warp-wide access hits 32 banks)
  int k;
  int last;        // largest id so far
  __device__ __forceinline__ void operator()(int j) {
    if (k < CAP) {
      if (j >= last) {  // append fast path (runs arrive id-ascending)
        row[k ^ x] = j;
        last = j;
      } else {  // shift the larger tail up by one
        int q = k, v;
        while (q > 0 && (v = row[(q - 1) ^ x]) > j) {
          row[q ^ x] = v;
          --q;
        }
        row[q ^ x] = j;
      }
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

template <class Emit>
__device__ __forceinline__ void emit_mask(Emit& em, unsigned m, const unsigned tg[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (m >> u & 1u) em((int)(tg[u] >> 2));
}

template <int D>
struct MaskWords {  // 32-bit words of 4-bit hit nibbles per particle (0: no masks)
  static constexpr int W = D == 3 ? 16 : (D == 2 ? 4 : 2);
};
constexpr unsigned kOverflow = 0x80000000u;  // counts[i] flag: masks did not fit

// Pass 1: row lengths k_i, per-block sums, and the hit nibbles of every chunk so
// that pass 3 never repeats a distance test.
template <int D, int P, int MODE, int BT>
__global__ void __launch_bounds__(BT) k_count(SweepArgs a) {
  __shared__ int s_w[BT / 32];
  constexpr int W = MODE == MODE_ALL ? 0 : MaskWords<D>::W;
  const int i = blockIdx.x * BT + threadIdx.x;
  int k = 0;
  if (i < a.n) {
    unsigned acc = 0, over = 0;
    int bits = 0, words = 0;
    scan_particle<D, P, MODE>(a, i, [&](unsigned m, const unsigned*, int) {
      k += __popc(m);
      if constexpr (W > 0) {
        acc |= m << bits;
        bits += 4;
        if (bits == 32) {
          if (words < W) a.masks[(int64_t)words * a.n + i] = acc;
          ++words;
          acc = 0;
          bits = 0;
        }
      }
    });
    if constexpr (W > 0) {
      if (bits) {
        if (words < W) a.masks[(int64_t)words * a.n + i] = acc;
        ++words;
      }
      over = words > W ? kOverflow : 0u;
    } else {
      over = kOverflow;  // all_list: pass 3 re-tests
    }
    a.counts[i] = (int)((unsigned)k | over);
  }
  int v = k;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
#pragma unroll
    for (int w = 0; w < BT / 32; ++w) t += s_w[w];
    a.block_sum[blockIdx.x] = t;
  }
}

// Pass 2: exclusive scan of the block sums in place (one block); offsets[n] = total.
__global__ void __launch_bounds__(1024) k_scan_blocks(long long* sums, int nb, int64_t* offsets,
                                                      int n) {
  __shared__ long long s_w[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = min(b0 + per, nb);
  long long local = 0;
  for (int b = b0; b < b1; ++b) local += sums[b];
  long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const long long w = s_w[lane];
    long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    s_w[lane] = wi - w;
    if (lane == 31) offsets[n] = wi;
  }
  __syncthreads();
  long long run = s_w[warp] + incl - local;
  for (int b = b0; b < b1; ++b) {
    const long long s = sums[b];
    sums[b] = run;
    run += s;
  }
}

// Pass 3: rows. The block's base comes from pass 2, the rows' offsets from a
// block scan of the pass-1 counts. Each thread replays its hit nibbles (one id
// load per hit, no distance test) into a sorted row in shared memory and each
// warp streams its rows to HBM. Rows whose masks did not fit are re-tested;
// rows longer than CAP are written straight into global memory.
template <int D, int P, int MODE, int BT, int CAP>
__global__ void __launch_bounds__(BT) k_fill(SweepArgs a) {
  static_assert(BT % 32 == 0 && CAP % 32 == 0, "shape");
  __shared__ int32_t S[BT * CAP];
  __shared__ int s_w[BT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = blockIdx.x * BT + tid;
  const unsigned kw = i < a.n ? (unsigned)__ldg(a.counts + i) : 0u;
  const int k = (int)(kw & ~kOverflow);
  const bool retest = (kw & kOverflow) != 0u;
  const int incl = warp_inclusive_scan(k);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int wbase = 0;
  long long btot = 0;
#pragma unroll
  for (int w = 0; w < BT / 32; ++w) {
    wbase += w < warp ? s_w[w] : 0;
    btot += s_w[w];
  }
  const long long bbase = a.block_sum[blockIdx.x];  // scanned in place by pass 2
  const int wrel = incl - k;
  const long long grow = bbase + wbase + wrel;
  if (i < a.n) a.offsets[i] = grow;
  if (bbase + btot > a.capacity) return;  // device API: caller grows the table

  int32_t* wS = S + warp * 32 * CAP;
  if (i < a.n && k <= CAP) {
    SmemEmit<CAP> em{wS + lane * CAP, lane, 0, INT_MIN};
    if (!retest) {
      constexpr int W = MaskWords<D>::W;
      unsigned acc = 0;
      int bits = 32, words = 0;
      visit_rows<D, MODE>(a, i, [&](int, int, int, int, int b, int e) {
        for (int s = b; s < e; s += 4) {
          if (bits == 32) {
            acc = words < W ? __ldg(a.masks + (int64_t)words * a.n + i) : 0u;
            ++words;
            bits = 0;
          }
          const unsigned m = (acc >> bits) & 0xFu;
          bits += 4;
          if (m) {
            typename Tester<D, P, MODE>::C c[4];
            unsigned tg[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (m >> u & 1u) load_cand<D, P, MODE>(a, s + u, c[u], tg[u]);
            emit_mask(em, m, tg);
          }
        }
      });
    } else {
      scan_particle<D, P, MODE>(a, i, [&](unsigned m, const unsigned* tg, int) {
        emit_mask(em, m, tg);
      });
    }
  }

  // rows that fit were sorted in shared memory: one warp-wide store per row;
  // longer rows are recomputed straight into global memory
  __syncwarp();
  int32_t* __restrict__ out = a.items + bbase + wbase;
#pragma unroll 4
  for (int r = 0; r < 32; ++r) {
    const int len = __shfl_sync(0xffffffffu, k, r);
    const int ro = __shfl_sync(0xffffffffu, wrel, r);
    if (len > CAP) continue;
#pragma unroll
    for (int p = 0; p < CAP / 32; ++p) {
      const int q = lane + 32 * p;
      if (q < len) out[ro + q] = wS[r * CAP + (q ^ r)];
    }
  }
  if (i < a.n && k > CAP) {
    GlobalEmit ge{a.items + grow, 0};
    scan_particle<D, P, MODE>(a, i, [&](unsigned m, const unsigned* tg, int) {
      emit_mask(ge, m, tg);
    });
  }
}
// ------------------------------------------------------------------------------
// Encode: round coordinates into the precision and pack them.
// RCLL: src = RelCoords::rel (nnps.cpp:304-315); CLL/all: src = positions
// (round_coords nnps.cpp:75-89, packing :185-194).
// ------------------------------------------------------------------------------
// Own coordinates (particle order) + reset of the look-back state.
template <int D, int P>
__global__ void k_encode_own(int n, const double* __restrict__ x0, const double* __restrict__ x1,
                             const double* __restrict__ x2, void* pos_own) {
  using C = typename Coord<D, P>::T;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    const double v[3] = {x0[t], D > 1 ? x1[t] : 0.0, D > 2 ? x2[t] : 0.0};
    reinterpret_cast<C*>(pos_own)[t] = pack<D, P>(v);
  }
}

// One thread per cell c: merge the members of cells (cx-1, cx, cx+1) by id into
// the run tri[c] = [slot, slot+len). The slot is a closed form of cell_start so
// no scan is needed: with st(x) = cell_start[row + x] and n_x the cell counts,
//   open x axis:     slot = st(max(cx-1,0)) + st(cx) + st(min(cx+1,X))
//   periodic x axis: slot = st(cx-1) + st(cx) + st(cx+1) + n_{X-1} - n_0,
//                    st(-1) = st(0) - n_{X-1};
// consecutive slots then differ by exactly the triple length and every x row of
// cells occupies a sub-range of [3*st(0), 3*st(X)), so all runs fit in 3n.
template <int D, int P, int MODE>
__global__ void k_encode_tri(int64_t C, int nx, int wrapx, const int32_t* __restrict__ start,
                             const int32_t* __restrict__ items, int n,
                             const double* __restrict__ x0, const double* __restrict__ x1,
                             const double* __restrict__ x2, int2* __restrict__ tri,
                             void* __restrict__ rec) {
  using RT = Rec<D, P>;
  using R = typename RT::R;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int cx = (int)(c % nx);
  const int32_t* st = start + (c - cx);
  const int n0 = st[1] - st[0], nl = st[nx] - st[nx - 1];
  int lo[3], hi[3];
  unsigned code[3];
  // list 0: cell cx-1 (dc_x = +1 -> code 2; CLL: wrapped from below -> code 0)
  if (cx > 0) {
    lo[0] = st[cx - 1];
    hi[0] = st[cx];
    code[0] = MODE == MODE_RCLL ? 2u : 1u;
  } else if (wrapx) {
    lo[0] = st[nx - 1];
    hi[0] = st[nx];
    code[0] = MODE == MODE_RCLL ? 2u : 0u;
  } else {
    lo[0] = hi[0] = 0;
    code[0] = 1u;
  }
  lo[1] = st[cx];
  hi[1] = st[cx + 1];
  code[1] = 1u;
  // list 2: cell cx+1 (dc_x = -1 -> code 0; CLL: wrapped from above -> code 2)
  if (cx + 1 < nx) {
    lo[2] = st[cx + 1];
    hi[2] = st[cx + 2];
    code[2] = MODE == MODE_RCLL ? 0u : 1u;
  } else if (wrapx) {
    lo[2] = st[0];
    hi[2] = st[1];
    code[2] = MODE == MODE_RCLL ? 0u : 2u;
  } else {
    lo[2] = hi[2] = 0;
    code[2] = 1u;
  }
  int slot;
  if (!wrapx) {
    slot = st[cx > 0 ? cx - 1 : 0] + st[cx] + st[cx + 1 < nx ? cx + 1 : nx];
  } else {
    const int stm1 = cx > 0 ? st[cx - 1] : st[0] - nl;
    slot = stm1 + st[cx] + st[cx + 1] + nl - n0;
  }
  const int len = (hi[0] - lo[0]) + (hi[1] - lo[1]) + (hi[2] - lo[2]);
  tri[c] = make_int2(slot, slot + len);
  R* out = reinterpret_cast<R*>(rec) + slot;
  int p0 = lo[0], p1 = lo[1], p2 = lo[2];
  int v0 = p0 < hi[0] ? items[p0] : INT_MAX;
  int v1 = p1 < hi[1] ? items[p1] : INT_MAX;
  int v2 = p2 < hi[2] ? items[p2] : INT_MAX;
  for (int q = 0; q < len; ++q) {
    int j;
    unsigned cd;
    if (v0 <= v1 && v0 <= v2 && p0 < hi[0]) {
      j = v0;
      cd = code[0];
      v0 = ++p0 < hi[0] ? items[p0] : INT_MAX;
    } else if (v1 <= v2 && p1 < hi[1]) {
      j = v1;
      cd = code[1];
      v1 = ++p1 < hi[1] ? items[p1] : INT_MAX;
    } else {
      j = v2;
      cd = code[2];
      v2 = ++p2 < hi[2] ? items[p2] : INT_MAX;
    }
    const int js = (j >= 0 && j < n) ? j : 0;  // malformed membership: stay memory-safe
    const double v[3] = {x0[js], D > 1 ? x1[js] : 0.0, D > 2 ? x2[js] : 0.0};
    out[q] = RT::make(pack<D, P>(v), ((unsigned)j << 2) | cd);
  }
}

template <int D>
struct Shape {
  static constexpr int BT = D == 3 ? 64 : 128;  // rows per block (count and fill)
  static constexpr int CAP = D == 3 ? 96 : 32;  // rows sorted in shared memory up to CAP
};

// ------------------------------------------------------------------------------
// Host-side launchers (called from capi.cu)
// ------------------------------------------------------------------------------
int sweep_block_rows(int dim) { return dim == 3 ? Shape<3>::BT : Shape<2>::BT; }
int mask_words(int dim) {
  return dim == 3 ? MaskWords<3>::W : (dim == 2 ? MaskWords<2>::W : MaskWords<1>::W);
}

size_t coord_bytes(int dim, int prec) {
  if (prec == FP16) return dim == 3 ? 8 : 4;
  if (prec == FP32) return dim == 1 ? 4 : (dim == 2 ? 8 : 16);
  return dim == 1 ? 8 : (dim == 2 ? 16 : 32);
}

size_t record_bytes(int dim, int prec) {
  if (prec == FP16) return dim == 3 ? 16 : 8;
  if (prec == FP32) return dim == 1 ? 8 : 16;
  return dim == 1 ? 16 : 32;
}

template <int D, int P>
static int encode_t(int mode, int n, int64_t C, int nx, int wrapx, const double* const x[3],
                    const int32_t* items, const int32_t* start, void* own, int2* tri, void* rec,
                    cudaStream_t st) {
  k_encode_own<D, P><<<(n + 255) / 256, 256, 0, st>>>(n, x[0], x[1], x[2], own);
  if (mode == MODE_ALL || C == 0) return 1;
  const unsigned cb = (unsigned)((C + 127) / 128);
  if (mode == MODE_RCLL)
    k_encode_tri<D, P, MODE_RCLL><<<cb, 128, 0, st>>>(C, nx, wrapx, start, items, n, x[0], x[1],
                                                       x[2], tri, rec);
  else
    k_encode_tri<D, P, MODE_CLL><<<cb, 128, 0, st>>>(C, nx, wrapx, start, items, n, x[0], x[1],
                                                      x[2], tri, rec);
  return 2;
}

// Returns the number of kernel launches issued (n > 0).
int launch_encode(int dim, int prec, int mode, int n, int64_t C, int nx, int wrapx,
                  const double* const x[3], const int32_t* items, const int32_t* start,
                  void* own, int2* tri, void* rec, cudaStream_t st) {
#define ENC(D, P) \
  if (dim == D && prec == P) return encode_t<D, P>(mode, n, C, nx, wrapx, x, items, start, own, tri, rec, st);
  ENC(1, FP16) ENC(2, FP16) ENC(3, FP16) ENC(1, FP32) ENC(2, FP32) ENC(3, FP32)
  ENC(1, FP64) ENC(2, FP64) ENC(3, FP64)
#undef ENC
  return 0;
}

template <int D, int P, int M>
static void count_t(const SweepArgs& a, cudaStream_t st) {
  constexpr int BT = Shape<D>::BT;
  const int nb = (a.n + BT - 1) / BT;
  k_count<D, P, M, BT><<<nb, BT, 0, st>>>(a);
  k_scan_blocks<<<1, 1024, 0, st>>>(a.block_sum, nb, a.offsets, a.n);
}

template <int D, int P, int M>
static void fill_t(const SweepArgs& a, cudaStream_t st) {
  constexpr int BT = Shape<D>::BT;
  k_fill<D, P, M, BT, Shape<D>::CAP><<<(a.n + BT - 1) / BT, BT, 0, st>>>(a);
}

#define SW(FN, D, P, M) \
  if (dim == D && prec == P && mode == M) return FN<D, P, M>(a, st);
#define SWP(FN, D, M) SW(FN, D, FP16, M) SW(FN, D, FP32, M) SW(FN, D, FP64, M)
#define SWA(FN)                                                                \
  SWP(FN, 1, MODE_RCLL) SWP(FN, 2, MODE_RCLL) SWP(FN, 3, MODE_RCLL)            \
  SWP(FN, 1, MODE_CLL) SWP(FN, 2, MODE_CLL) SWP(FN, 3, MODE_CLL)              \
  SWP(FN, 1, MODE_ALL) SWP(FN, 2, MODE_ALL) SWP(FN, 3, MODE_ALL)

// Pass 1 + 2: counts, block sums, scanned block bases, offsets[n] = total.
void launch_count(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) { SWA(count_t) }
// Pass 3: offsets[0..n) and the rows.
void launch_fill(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) { SWA(fill_t) }

#undef SWA
#undef SWP
#undef SW

}  // namespace sphx_dev
