// NNPS sweep for sm_100a: candidate enumeration over the 3^d neighbour cells,
// the exact reduced-precision distance test, per-row sort and the CSR table.
//
// Reference semantics (paths relative to the reference's proj/):
//   rcll            nnps.cpp:283-416 (axis_term/finish :321-346, 2-D batch
//                   detail::range_f16_rel_2d nnps_batch.cpp:203-261)
//   cell_link_list  nnps.cpp:174-281 (dist_prec :91-124, batch range_*_abs_2d
//                   nnps_batch.cpp:119-201)
//   all_list        nnps.cpp:128-172
//   build_table     nnps.cpp:26-66 (rows ascending, int64 offsets)
//
// Candidate layout ("x-triple runs" in 4-record chunks). For every cell c the
// encode (k_encode_rows) merges, by particle id, the members of the x-neighbour
// cells (cx-1, cx, cx+1) -- wrapped on a periodic x axis -- into one run of
// records, padded with NaN sentinels to whole chunks of 4. A chunk is one record
// of quads (array of structures, 32 bytes at FP16): a quad of coordinates per
// axis, then for RCLL the quad of x offsets dc = cx_i - cx_j in {-1,0,1}; the 4
// ids of a chunk are a separate uint4. CLL records carry the periodic x shift
// already applied (round_to(prec, xj + shift), nnps.cpp:116). A particle's
// candidates are the 3 (2-D) / 9 (3-D) runs of its (dz, dy) rows.
//
// Kernels (each a tile of consecutive rows in particle order, a decoupled
// look-back for the row offsets, sorted rows packed in shared memory, 16-byte
// stores of the tile):
//   k_rcll16<2>            FP16 RCLL 2-D, one fused pass;
//   k_r16_test/k_r16_emit  FP16 RCLL 3-D, tests (cell order) and ordered emission;
//   k_sweep<D,P,MODE>      every other precision / mode (one pass);
//   k_r16_grad<D>          fused FP16 RCLL -> grad_normalized (no table).
//
// Bit-exactness: every step is an explicit round-to-nearest op in the
// precision (no contraction; the reference is built without -march). The x term
// t + cc (cc = round_to(prec, dc*hc), dc*hc exact) is one fused dc*hc + t -- a
// single rounding of the same exact sum. FP16 uses native binary16 ALU ops, which
// keep subnormals, and sqrt(acc) < cutoff is the exact monotone test acc < thr.

#include <climits>
#include <type_traits>

#ifndef SPHX_UNROLL
#define SPHX_UNROLL 4
#endif
#ifndef SPHX_MINB2
#define SPHX_MINB2 12
#endif
#ifndef SPHX_TICKET
#define SPHX_TICKET 0  // k_rcll16 tiles from blockIdx (1: from the ticket counter)
#endif

#include "common.cuh"

namespace sphx_dev {

// binning.cu
int64_t scan_tiles(int64_t C);
void launch_scan_counts(const int32_t* in, int32_t* out, int64_t C, unsigned long long* tiles,
                        int* counter, cudaStream_t st);

constexpr int kPhaseAUnroll = SPHX_UNROLL;  // chunk loads issued together in phase A

// ------------------------------------------------------------------------------
// Own-particle coordinates (particle order): FP16 half2 / half4, FP32/FP64 vectors.
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

__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<const unsigned*>(&h); }
__device__ __forceinline__ __half2 u2h(unsigned u) { return *reinterpret_cast<const __half2*>(&u); }
__device__ __forceinline__ __half hbits(unsigned b) { return __ushort_as_half((unsigned short)b); }

template <int P>
struct Prec;
template <>
struct Prec<FP16> {
  using T = __half;
  using Quad = uint2;  // 4 binary16
  static __device__ __forceinline__ T cvt(double v) { return __double2half(v); }
};
template <>
struct Prec<FP32> {
  using T = float;
  using Quad = float4;
  static __device__ __forceinline__ T cvt(double v) { return __double2float_rn(v); }
};
struct alignas(16) DQuad {
  double2 a, b;
};
template <>
struct Prec<FP64> {
  using T = double;
  using Quad = DQuad;
  static __device__ __forceinline__ T cvt(double v) { return v; }
};

template <int D, int P>
__device__ __forceinline__ typename Coord<D, P>::T pack(const double v[3]) {
  using T = typename Prec<P>::T;
  if constexpr (P == FP16) {
    const __half2 xy = __halves2half2(__double2half(v[0]), D > 1 ? __double2half(v[1]) : hbits(0));
    if constexpr (D == 3) {
      const __half2 z0 = __halves2half2(__double2half(v[2]), hbits(0));
      return make_uint2(h2u(xy), h2u(z0));
    } else {
      return xy;
    }
  } else if constexpr (D == 1) {
    return Prec<P>::cvt(v[0]);
  } else if constexpr (D == 2) {
    typename Coord<D, P>::T c;
    c.x = Prec<P>::cvt(v[0]);
    c.y = Prec<P>::cvt(v[1]);
    return c;
  } else {
    typename Coord<D, P>::T c;
    c.x = Prec<P>::cvt(v[0]);
    c.y = Prec<P>::cvt(v[1]);
    c.z = Prec<P>::cvt(v[2]);
    c.w = T(0);
    return c;
  }
}

// axis k of a packed coordinate as the precision's scalar type
template <int D, int P>
__device__ __forceinline__ typename Prec<P>::T axis_of(const typename Coord<D, P>::T& c, int k) {
  if constexpr (P == FP16) {
    if constexpr (D == 3) {
      return k == 0 ? __low2half(u2h(c.x)) : (k == 1 ? __high2half(u2h(c.x)) : __low2half(u2h(c.y)));
    } else {
      return k == 0 ? __low2half(c) : __high2half(c);
    }
  } else if constexpr (D == 1) {
    return c;
  } else if constexpr (D == 2) {
    return k == 0 ? c.x : c.y;
  } else {
    return k == 0 ? c.x : (k == 1 ? c.y : c.z);
  }
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
template <>
__device__ __forceinline__ DQuad ldg<DQuad>(const void* base, int64_t s) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * s;
  DQuad q;
  q.a = __ldg(p);
  q.b = __ldg(p + 1);
  return q;
}

// element u of a quad
__device__ __forceinline__ float qel(const float4& q, int u) {
  return u == 0 ? q.x : (u == 1 ? q.y : (u == 2 ? q.z : q.w));
}
__device__ __forceinline__ double qel(const DQuad& q, int u) {
  return u == 0 ? q.a.x : (u == 1 ? q.a.y : (u == 2 ? q.b.x : q.b.y));
}
__device__ __forceinline__ void qset(float4& q, int u, float v) {
  if (u == 0) q.x = v; else if (u == 1) q.y = v; else if (u == 2) q.z = v; else q.w = v;
}
__device__ __forceinline__ void qset(DQuad& q, int u, double v) {
  if (u == 0) q.a.x = v; else if (u == 1) q.a.y = v; else if (u == 2) q.b.x = v; else q.b.y = v;
}
__device__ __forceinline__ void qset(uint2& q, int u, __half v) {
  const unsigned b = __half_as_ushort(v);
  if (u == 0) q.x = (q.x & 0xFFFF0000u) | b;
  else if (u == 1) q.x = (q.x & 0xFFFFu) | (b << 16);
  else if (u == 2) q.y = (q.y & 0xFFFF0000u) | b;
  else q.y = (q.y & 0xFFFFu) | (b << 16);
}

__device__ __forceinline__ float f_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float f_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float f_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float f_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double f_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double f_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double f_fma(double a, double b, double c) { return __fma_rn(a, b, c); }

template <int P>
struct Consts;
template <>
struct Consts<FP32> {
  static __device__ __forceinline__ float hh(const PrecConsts& c, int k) { return c.f_hh[k]; }
  static __device__ __forceinline__ float cc(const PrecConsts& c, int k) { return c.f_cc[k]; }
  static __device__ __forceinline__ float sh(const PrecConsts& c, int k) { return c.f_sh[k]; }
  static __device__ __forceinline__ float thr(const PrecConsts& c) { return c.f_thr; }
};
template <>
struct Consts<FP64> {
  static __device__ __forceinline__ double hh(const PrecConsts& c, int k) { return c.d_hh[k]; }
  static __device__ __forceinline__ double cc(const PrecConsts& c, int k) { return c.d_cc[k]; }
  static __device__ __forceinline__ double sh(const PrecConsts& c, int k) { return c.d_sh[k]; }
  static __device__ __forceinline__ double thr(const PrecConsts& c) { return c.d_thr; }
};

// Chunk of 4 candidate records as loaded by the testers.
template <int D, int P>
struct Chunk {
  typename Prec<P>::Quad x[D];
  typename Prec<P>::Quad dc;
};

// Chunks are stored array-of-structures: one record of NQ quads (the D
// coordinate quads, then the RCLL dc quad), padded to a power of two, so a
// chunk is one 32-byte sector at FP16 and is fetched with 16-byte loads.
template <int D, int P, int MODE>
struct ChunkLay {
  static constexpr int QB = P == FP16 ? 8 : (P == FP32 ? 16 : 32);  // bytes per quad
  static constexpr int NQ = D + (MODE == MODE_RCLL ? 1 : 0);
  static constexpr int NQP = NQ <= 1 ? 1 : (NQ <= 2 ? 2 : 4);
  static constexpr int BYTES = QB * NQP;
};
// 3-D FP16 RCLL uses xy-plane runs (k_encode_xy). A chunk is 32 bytes (one
// 256-bit load): the x, y, z quads, then for each of dcx and dcy one word of PRMT
// selector nibbles, (s1 << 12 | s0 << 4) per record pair, s = 0 / 1 / 2 for an
// offset of 0 / +1 / -1 (dc_half2 turns a pair's selector into its half2).
template <>
struct ChunkLay<3, FP16, MODE_RCLL> {
  static constexpr int QB = 8, NQ = 3, NQP = 4, BYTES = 32;
  static constexpr int SELX = 24, SELY = 28;  // byte offsets of the selector words
};

// selector nibble of record l (0..3) for a cell offset code s (0: 0, 1: +1, 2: -1)
__device__ __forceinline__ uint32_t dc_nibble(int l, uint32_t s) {
  return s << (16 * (l >> 1) + ((l & 1) ? 12 : 4));
}

// half2 {dc_l0, dc_l1} of a record pair from its 16 selector bits:
// bytes 00 3C BC pick the high byte of 0, +1.0, -1.0
__device__ __forceinline__ __half2 dc_half2(uint32_t sel16) {
  return u2h(__byte_perm(0x00BC3C00u, 0u, sel16));
}

// element u (0..3) of quad q of chunk ch
template <int D, int P, int MODE>
__device__ __forceinline__ typename Prec<P>::T* rec_el(void* qc, int64_t ch, int q, int u) {
  using L = ChunkLay<D, P, MODE>;
  return reinterpret_cast<typename Prec<P>::T*>(static_cast<char*>(qc) + ch * L::BYTES +
                                                q * L::QB) + u;
}

// 4 lane masks of a pair of HSET2 results -> 4-bit hit nibble (record order)
__device__ __forceinline__ unsigned nibble(unsigned mk01, unsigned mk23) {
  const unsigned w = __byte_perm(mk01, mk23, 0x6420) & 0x08040201u;
  return (w * 0x01010101u) >> 24;
}

// acc = acc >> 4 | nibble << 28, the nibble being the 4 tests acc_u < thr of two
// binary16x2 accumulators (records 0,1 in a01, 2,3 in a23); NaN never hits.
__device__ __forceinline__ void acc_nibble(unsigned& acc, __half2 a01, __half2 a23, __half2 thr2) {
  asm("{\n\t.reg .pred p0, p1, p2, p3;\n\t"
      "setp.lt.f16x2 p0|p1, %1, %3;\n\t"
      "setp.lt.f16x2 p2|p3, %2, %3;\n\t"
      "shr.b32 %0, %0, 4;\n\t"
      "@p0 or.b32 %0, %0, 0x10000000;\n\t"
      "@p1 or.b32 %0, %0, 0x20000000;\n\t"
      "@p2 or.b32 %0, %0, 0x40000000;\n\t"
      "@p3 or.b32 %0, %0, 0x80000000;\n\t}"
      : "+r"(acc)
      : "r"(h2u(a01)), "r"(h2u(a23)), "r"(h2u(thr2)));
}

// row constant: +-v for a -1/+1 row offset (as dc = -off), +0 for the centre row
__device__ __forceinline__ __half2 row_half2(unsigned v_bits, int off, bool neg_is_pos) {
  if (off == 0) return u2h(0u);
  const bool pos = neg_is_pos ? off < 0 : off > 0;
  const unsigned b = pos ? v_bits : (v_bits ^ 0x8000u);
  return u2h(b | (b << 16));
}

// ------------------------------------------------------------------------------
// Distance testers: test4(row, chunk) -> 4-bit hit mask.
// ------------------------------------------------------------------------------
template <int D, int P, int MODE>
struct Tester;

// ---- RCLL, FP16 (nnps.cpp:332-337, :406, :344; nnps_batch.cpp:238-258) -------
// Two candidates per binary16x2 instruction; per candidate and axis
//   s = r16(ri - rj); t = r16(s * r16(hc/2)); d = r16(t + r16(dc*hc)); q = r16(d*d)
// and acc sums the axes in order. The x offset is the fused dc*hc16 + t.
template <int D>
struct Tester<D, FP16, MODE_RCLL> {
  __half2 r2[3], hh2[3], hc2, thr2;
  struct Row {
    __half2 cc[3];  // y, z centre differences (index 1, 2)
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const typename Coord<D, FP16>::T o = ldg<typename Coord<D, FP16>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      r2[k] = __half2half2(axis_of<D, FP16>(o, k));
      hh2[k] = __half2half2(hbits(a.c.h_hh[k]));
    }
    hc2 = __half2half2(hbits(a.c.h_cc[0]));
    thr2 = __half2half2(hbits(a.c.h_thr));
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    Row r;
    r.cc[0] = u2h(0u);
    r.cc[1] = row_half2(a.c.h_cc[1], dy, true);  // dc = -dy: cc = +hc for dy = -1
    r.cc[2] = row_half2(a.c.h_cc[2], dz, true);
    return r;
  }
  __device__ __forceinline__ __half2 pair_acc(const Row& r, const Chunk<D, FP16>& ch, bool hi) const {
    __half2 acc;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const __half2 xj = u2h(hi ? ch.x[k].y : ch.x[k].x);
      const __half2 t = __hmul2_rn(__hsub2_rn(r2[k], xj), hh2[k]);
      const __half2 d = k == 0 ? __hfma2(u2h(hi ? ch.dc.y : ch.dc.x), hc2, t) : __hadd2_rn(t, r.cc[k]);
      const __half2 q = __hmul2_rn(d, d);
      acc = k == 0 ? q : __hadd2_rn(acc, q);
    }
    return acc;
  }
  __device__ __forceinline__ unsigned test4(const Row& r, const Chunk<D, FP16>& ch) const {
    return nibble(__hlt2_mask(pair_acc(r, ch, false), thr2), __hlt2_mask(pair_acc(r, ch, true), thr2));
  }
  __device__ __forceinline__ void acc4(const Row& r, const Chunk<D, FP16>& ch, unsigned& acc) const {
    acc_nibble(acc, pair_acc(r, ch, false), pair_acc(r, ch, true), thr2);
  }
};

// ---- CLL / all_list, FP16 (dist_prec nnps.cpp:112-121; nnps_batch.cpp:145-157) ----
// x carries its periodic shift already; y/z shifts are per row (wrapped rows).
template <int D, int MODE>
struct TesterHalfAbs {
  __half2 x2[3], sh2[3], thr2;
  struct Row {
    __half2 sh[3];
    bool any;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const typename Coord<D, FP16>::T o = ldg<typename Coord<D, FP16>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) x2[k] = __half2half2(axis_of<D, FP16>(o, k));
    thr2 = __half2half2(hbits(a.c.h_thr));
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int, int, int wy, int wz) const {
    Row r;
    r.sh[0] = u2h(0u);
    r.sh[1] = row_half2(a.c.h_sh[1], wy, false);
    r.sh[2] = row_half2(a.c.h_sh[2], wz, false);
    r.any = wy != 0 || wz != 0;
    return r;
  }
  __device__ __forceinline__ __half2 pair_acc(const Row& r, const Chunk<D, FP16>& ch, bool hi) const {
    __half2 acc;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      __half2 xj = u2h(hi ? ch.x[k].y : ch.x[k].x);
      if (k > 0 && r.any) xj = __hadd2_rn(xj, r.sh[k]);  // round16(xj + shift)
      const __half2 d = __hsub2_rn(x2[k], xj);
      const __half2 q = __hmul2_rn(d, d);
      acc = k == 0 ? q : __hadd2_rn(acc, q);
    }
    return acc;
  }
  __device__ __forceinline__ unsigned test4(const Row& r, const Chunk<D, FP16>& ch) const {
    return nibble(__hlt2_mask(pair_acc(r, ch, false), thr2), __hlt2_mask(pair_acc(r, ch, true), thr2));
  }
  __device__ __forceinline__ void acc4(const Row& r, const Chunk<D, FP16>& ch, unsigned& acc) const {
    acc_nibble(acc, pair_acc(r, ch, false), pair_acc(r, ch, true), thr2);
  }
};
template <int D> struct Tester<D, FP16, MODE_CLL> : TesterHalfAbs<D, MODE_CLL> {};
template <int D> struct Tester<D, FP16, MODE_ALL> : TesterHalfAbs<D, MODE_ALL> {};

// ---- RCLL, FP32 / FP64 (nnps.cpp:324-331, :401-405, :342-343) ----
template <int D, int P>
struct TesterRcllScalar {
  using T = typename Prec<P>::T;
  using S = Consts<P>;
  T ri[3], hh[3], hcx, thr;
  struct Row {
    T cc[3];
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const typename Coord<D, P>::T o = ldg<typename Coord<D, P>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      ri[k] = axis_of<D, P>(o, k);
      hh[k] = S::hh(a.c, k);
    }
    hcx = S::cc(a.c, 0);
    thr = S::thr(a.c);
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int dy, int dz, int, int) const {
    Row r;
    r.cc[0] = T(0);
    r.cc[1] = dy == 0 ? T(0) : (dy < 0 ? S::cc(a.c, 1) : -S::cc(a.c, 1));
    r.cc[2] = dz == 0 ? T(0) : (dz < 0 ? S::cc(a.c, 2) : -S::cc(a.c, 2));
    return r;
  }
  __device__ __forceinline__ unsigned test4(const Row& r, const Chunk<D, P>& ch) const {
    unsigned m = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const T t = f_mul(f_sub(ri[k], qel(ch.x[k], u)), hh[k]);
        const T d = k == 0 ? f_fma(qel(ch.dc, u), hcx, t) : f_add(t, r.cc[k]);
        const T q = f_mul(d, d);
        acc = k == 0 ? q : f_add(acc, q);  // 0 + q == q exactly (q >= +0)
      }
      m |= (unsigned)(acc < thr) << u;
    }
    return m;
  }
  __device__ __forceinline__ void acc4(const Row& r, const Chunk<D, P>& ch, unsigned& acc) const {
    acc = (acc >> 4) | (test4(r, ch) << 28);
  }
};

// ---- CLL / all_list, FP32 / FP64 (dist_prec nnps.cpp:94-111) ----
template <int D, int P>
struct TesterAbsScalar {
  using T = typename Prec<P>::T;
  using S = Consts<P>;
  T xi[3], thr;
  struct Row {
    T sh[3];
    bool any;
  };
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const typename Coord<D, P>::T o = ldg<typename Coord<D, P>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < D; ++k) xi[k] = axis_of<D, P>(o, k);
    thr = S::thr(a.c);
  }
  __device__ __forceinline__ Row row(const SweepArgs& a, int, int, int wy, int wz) const {
    Row r;
    r.sh[0] = T(0);
    r.sh[1] = wy == 0 ? T(0) : (wy > 0 ? S::sh(a.c, 1) : -S::sh(a.c, 1));
    r.sh[2] = wz == 0 ? T(0) : (wz > 0 ? S::sh(a.c, 2) : -S::sh(a.c, 2));
    r.any = wy != 0 || wz != 0;
    return r;
  }
  __device__ __forceinline__ unsigned test4(const Row& r, const Chunk<D, P>& ch) const {
    unsigned m = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        T xj = qel(ch.x[k], u);
        // the shift is added only on shifted axes (FP32, nnps.cpp:106); FP64 adds
        // it always (:97), where + 0.0 is exact
        if (k > 0 && r.any) xj = f_add(xj, r.sh[k]);
        const T d = f_sub(xi[k], xj);
        const T q = f_mul(d, d);
        acc = k == 0 ? q : f_add(acc, q);
      }
      m |= (unsigned)(acc < thr) << u;
    }
    return m;
  }
  __device__ __forceinline__ void acc4(const Row& r, const Chunk<D, P>& ch, unsigned& acc) const {
    acc = (acc >> 4) | (test4(r, ch) << 28);
  }
};

template <int D> struct Tester<D, FP32, MODE_RCLL> : TesterRcllScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_RCLL> : TesterRcllScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_CLL> : TesterAbsScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_CLL> : TesterAbsScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_ALL> : TesterAbsScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_ALL> : TesterAbsScalar<D, FP64> {};

template <int D, int P, int MODE>
__device__ __forceinline__ void load_chunk(const SweepArgs& a, int64_t ch, Chunk<D, P>& c) {
  using L = ChunkLay<D, P, MODE>;
  using Q = typename Prec<P>::Quad;
  if constexpr (L::BYTES >= 16) {
    constexpr int NV = L::BYTES / 16;
    union {
      uint4 v[NV];
      Q q[L::NQP];
    } u;
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const char*>(a.qc) + ch * L::BYTES);
#pragma unroll
    for (int v = 0; v < NV; ++v) u.v[v] = __ldg(p + v);
#pragma unroll
    for (int k = 0; k < D; ++k) c.x[k] = u.q[k];
    if constexpr (MODE == MODE_RCLL) c.dc = u.q[D];
  } else {  // FP16 1-D CLL/all: one 8-byte quad
    c.x[0] = __ldg(reinterpret_cast<const Q*>(a.qc) + ch);
  }
}

// ------------------------------------------------------------------------------
// Candidate enumeration. visit_rows calls fn(dy, dz, wy, wz, cb, ce) for each
// (dy, dz) row of the 3^d neighbourhood of particle i, wrapped or skipped per
// periodic(k) (nnps.cpp:359-372); [cb, ce) is the row's run of chunks.
// ------------------------------------------------------------------------------
template <int D, int MODE, class Fn>
__device__ __forceinline__ void visit_rows(const SweepArgs& a, int i, Fn&& fn) {
  if constexpr (MODE == MODE_ALL) {  // all_list: one "row" holding every particle
    fn(0, 0, 0, 0, 0, (a.n + 3) / 4);
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

// Hit words. The chunks of each run are tested in groups of up to 8; the 4-bit
// hit nibbles of a group form one 32-bit word, chunk g at bits 0-3 (bit u of a
// nibble: record u is a neighbour j != i). The own record (particle i) sits in
// its own-cell run at selfpos[i] and is masked out there.
template <int D, int P, int MODE>
__device__ __forceinline__ unsigned group_word(const SweepArgs& a, const Tester<D, P, MODE>& tst,
                                               const typename Tester<D, P, MODE>::Row& row,
                                               bool own, int selfch, unsigned selfmask, int g,
                                               int e) {
  unsigned acc = 0;
#pragma unroll 4
  for (int ch = g; ch < e; ++ch) {
    Chunk<D, P> c;
    load_chunk<D, P, MODE>(a, ch, c);
    tst.acc4(row, c, acc);
    if (own && ch == selfch) acc &= selfmask;
  }
  return acc >> (4 * (8 - (e - g)));
}

// Calls fn(row, own, g, e) for every group [g, e) of chunks of particle i, in
// row order ((dz, dy) ascending; runs are id-merged, so hits come out sorted
// inside each run).
template <int D, int P, int MODE, class Fn>
__device__ __forceinline__ void walk_groups(const SweepArgs& a, int i, const Tester<D, P, MODE>& tst,
                                            Fn&& fn) {
  visit_rows<D, MODE>(a, i, [&](int dy, int dz, int wy, int wz, int cb, int ce) {
    const typename Tester<D, P, MODE>::Row row = tst.row(a, dy, dz, wy, wz);
    const bool own = dy == 0 && dz == 0;
    for (int g = cb; g < ce; g += 8) fn(row, own, g, min(g + 8, ce));
  });
}

// Row sinks: a row being built in shared memory (32-bit shared address, so each
// store is one STS) or straight in HBM (tiles whose rows exceed the tile buffer).
struct SharedRow {
  uint32_t base;  // shared-space byte address of element 0
  __device__ __forceinline__ void st(int e, int v) const {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + 4u * (uint32_t)e), "r"(v) : "memory");
  }
  // predicated store (no branch)
  __device__ __forceinline__ void st_if(bool c, int e, int v) const {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.shared.b32 [%0], %1;\n\t}"
                 ::"r"(base + 4u * (uint32_t)e), "r"(v), "r"((int)c) : "memory");
  }
  __device__ __forceinline__ int ld(int e) const {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (uint32_t)e) : "memory");
    return v;
  }
};
struct GlobalRow {
  int32_t* p;
  __device__ __forceinline__ void st(int e, int v) const { p[e] = v; }
  __device__ __forceinline__ void st_if(bool c, int e, int v) const {
    if (c) p[e] = v;
  }
  __device__ __forceinline__ int ld(int e) const { return p[e]; }
};

// Appends the hits of one chunk (nibble m, ids tq) to dst[k..]: predicated
// stores at the prefix positions, no branches.
template <class Row>
__device__ __forceinline__ void append4(const Row& dst, int& k, unsigned m, const uint4& tq) {
  const int p1 = k + (int)(m & 1u);
  const int p2 = p1 + (int)((m >> 1) & 1u);
  const int p3 = p2 + (int)((m >> 2) & 1u);
  dst.st_if(m & 1u, k, (int)tq.x);
  dst.st_if(m & 2u, p1, (int)tq.y);
  dst.st_if(m & 4u, p2, (int)tq.z);
  dst.st_if(m & 8u, p3, (int)tq.w);
  k = p3 + (int)(m >> 3);
}

// dst[0, gs) and dst[gs, k) are each sorted: insert the tail into the head. Once
// a tail element is already above everything before it, the rest are too.
template <class Row>
__device__ __forceinline__ void merge_tail(const Row& dst, int gs, int k) {
  for (int e = gs; e < k; ++e) {
    const int v = dst.ld(e);
    int w = dst.ld(e - 1);
    if (w < v) break;
    int q = e;
    do {
      dst.st(q, w);
      --q;
    } while (q > 0 && (w = dst.ld(q - 1)) > v);
    dst.st(q, v);
  }
}

// Streams the packed tile pk[0, n) to gout: 16-byte stores on the aligned
// vectors of gout, element stores at the two ragged ends.
template <int BT>
__device__ __forceinline__ void stream_tile(int32_t* gout, const SharedRow& pk, int n, int tid) {
  const int ph = (int)(((uintptr_t)gout & 15u) >> 2);
  int4* g4 = reinterpret_cast<int4*>(gout - ph);
  const int nv = (ph + n + 3) >> 2;
  for (int q = tid; q < nv; q += BT) {
    const int e0 = 4 * q - ph;  // tile index of the vector's first element
    if (e0 >= 0 && e0 + 4 <= n) {
      g4[q] = make_int4(pk.ld(e0), pk.ld(e0 + 1), pk.ld(e0 + 2), pk.ld(e0 + 3));
    } else {
      for (int e = max(e0, 0); e < min(e0 + 4, n); ++e) gout[e] = pk.ld(e);
    }
  }
}

// Decoupled look-back over the tiles of one call. Tile words carry the call's
// epoch, so the array is never cleared between calls:
//   [63:48] epoch, [47:46] flag (1 = aggregate, 2 = inclusive prefix), [45:0] value.
// Publishing (one lane) and resolving (one warp) are separate so that a tile can
// build its rows while its predecessors finish.
__device__ __forceinline__ void lookback_publish(unsigned long long* tiles, int bid, long long total,
                                                 unsigned epoch) {
  const unsigned long long E = (unsigned long long)epoch << 48;
  st_relaxed_u64(&tiles[bid], E | ((bid == 0 ? 2ull : 1ull) << 46) | (unsigned long long)total);
}

__device__ __forceinline__ long long lookback_resolve(unsigned long long* tiles, int bid,
                                                      long long total, unsigned epoch) {
  if (bid == 0) return 0;
  const unsigned long long E = (unsigned long long)epoch << 48, PRE = 2ull << 46,
                           VAL = (1ull << 46) - 1;
  const int lane = threadIdx.x & 31;
  long long excl = 0;
  int p = bid - 1;
  unsigned backoff = 64, spins = 0;
  while (true) {
    const int idx = p - lane;
    const unsigned long long st = idx >= 0 ? ld_relaxed_u64(&tiles[idx]) : (E | PRE);
    const unsigned flag = (st >> 48) == epoch ? (unsigned)(st >> 46) & 3u : 0u;
    const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == 2u);
    const unsigned zero_mask = __ballot_sync(0xffffffffu, flag == 0u);
    const int first = pre_mask ? __ffs(pre_mask) - 1 : 32;
    const unsigned need = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (zero_mask & need) {
      // a predecessor that never publishes is a bug: fail the launch (~4 s)
      // instead of hanging the device
      if (++spins > (1u << 22)) __trap();
      __nanosleep(backoff);
      backoff = backoff < 1024 ? backoff * 2 : 1024;
      continue;
    }
    const long long v = lane <= first ? (long long)(st & VAL) : 0ll;
    excl += warp_sum_ll(v);
    if (first < 32) break;
    p -= 32;
  }
  if (lane == 0) st_relaxed_u64(&tiles[bid], E | PRE | (unsigned long long)(excl + total));
  return excl;
}

// ------------------------------------------------------------------------------
// FP16 RCLL, 2-D / 3-D: the hot path, written out without the generic walk.
// Per particle the 3^(d-1) runs (dz, dy ascending) are resolved once into
// registers; each chunk is one 32-byte record {x quad, y quad, (z quad,) dc quad}.
// Per pair of candidates and axis: s = r16(ri - rj); t = r16(s * r16(hc/2));
// d = r16(t + r16(dc*hc)) (x: one fused dc*hc16 + t, dc*hc16 exact) or
// r16(t + cc_row) (y, z; skipped for the centre row, where cc = 0 and t + 0 == t);
// acc = r16(acc + r16(d*d)); hit: acc < thr (nnps.cpp:332-346, nnps_batch.cpp:238-258).
// ------------------------------------------------------------------------------
template <int D>
struct R16 {
  // runs per particle: 2-D x-triples of rows dy = -1, 0, 1; 3-D xy-plane runs of
  // planes dz = -1, 0, 1 (k_encode_xy)
  static constexpr int NR = 3;
};

// Programmatic dependent launch (sm_90+): the kernel may start while the previous
// kernel on the stream finishes its last wave; it must execute
// griddepcontrol.wait before reading that kernel's output (the previous kernel
// executes griddepcontrol.launch_dependents at its start).
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// One chunk (4 candidates) against particle i: the 4-bit hit nibble is shifted
// into acc from the top (acc = acc >> 4 | nibble << 28). ZC: the run's last
// centre difference (z in 3-D, y in 2-D) is zero (the dz = 0 / dy = 0 run), so
// its add is skipped: r16(t + 0) only turns -0 into +0, which is then squared.
template <int D, bool ZC = false>
__device__ __forceinline__ void r16_chunk(const char* __restrict__ qc, int ch, const __half2 (&r2)[3],
                                          const __half2 (&hh2)[3], __half2 hc2, __half2 thr2,
                                          __half2 ccy, __half2 ccz, unsigned& acc) {
  __half2 a[2];
  if constexpr (D == 3) {
    // xy-plane run chunk (32 B, one 256-bit load): x, y | z quads, dcx, dcy
    // selector words; ccy is the y cell edge (dcy per record), ccz the run's z
    // centre difference
    uint4 v0, v1;
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w), "=r"(v1.x), "=r"(v1.y), "=r"(v1.z),
          "=r"(v1.w)
        : "l"(qc + (size_t)ch * 32));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned xj = h ? v0.y : v0.x, yj = h ? v0.w : v0.z, zj = h ? v1.y : v1.x;
      __half2 t = __hmul2_rn(__hsub2_rn(r2[0], u2h(xj)), hh2[0]);
      __half2 d = __hfma2(dc_half2(h ? v1.z >> 16 : v1.z), hc2, t);
      __half2 acc2 = __hmul2_rn(d, d);
      t = __hmul2_rn(__hsub2_rn(r2[1], u2h(yj)), hh2[1]);
      d = __hfma2(dc_half2(h ? v1.w >> 16 : v1.w), ccy, t);
      acc2 = __hadd2_rn(acc2, __hmul2_rn(d, d));
      t = __hmul2_rn(__hsub2_rn(r2[2], u2h(zj)), hh2[2]);
      if constexpr (!ZC) t = __hadd2_rn(t, ccz);
      acc2 = __hadd2_rn(acc2, __hmul2_rn(t, t));
      a[h] = acc2;
    }
  } else {
    // the 32-byte record is one sector: one 256-bit load (LDG.256, sm_100)
    uint4 v0;
    uint2 v1;
    unsigned pad0, pad1;
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w), "=r"(v1.x), "=r"(v1.y), "=r"(pad0),
          "=r"(pad1)
        : "l"(qc + (size_t)ch * 32));
    (void)pad0;
    (void)pad1;
    // quads: x = (v0.x, v0.y), y = (v0.z, v0.w), dc = (v1.x, v1.y)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned xj = h ? v0.y : v0.x, yj = h ? v0.w : v0.z;
      __half2 t = __hmul2_rn(__hsub2_rn(r2[0], u2h(xj)), hh2[0]);
      const __half2 d = __hfma2(u2h(h ? v1.y : v1.x), hc2, t);
      __half2 acc2 = __hmul2_rn(d, d);
      t = __hmul2_rn(__hsub2_rn(r2[1], u2h(yj)), hh2[1]);
      if constexpr (!ZC) t = __hadd2_rn(t, ccy);
      acc2 = __hadd2_rn(acc2, __hmul2_rn(t, t));
      a[h] = acc2;
    }
  }
  acc_nibble(acc, a[0], a[1], thr2);
}

// Cursor over a particle's runs, flattened into one chunk sequence. The run
// table holds the non-empty runs of the particle as {first chunk | row << 27,
// end chunk}; the row (dz, dy) gives the y / z centre differences.
struct RunCursor {
  int r, ch, end;
  __half2 ccy, ccz;
};

// row constants: cc(-1) = +hc16 (dc = -dy), cc(0) = 0, cc(+1) = -hc16, as half2 bits
__device__ __forceinline__ __half2 cc_of(unsigned hc16, int off) {
  const unsigned b = off < 0 ? hc16 : (hc16 ^ 0x8000u);
  return u2h(off == 0 ? 0u : (b | (b << 16)));
}

template <int D, int BT>
__device__ __forceinline__ void run_open(const int2* runs, int tid, int r, RunCursor& c,
                                         unsigned hcy, unsigned hcz) {
  const int2 e = runs[r * BT + tid];
  const int q = (unsigned)e.x >> 27;  // 0..8: dy = q % 3 - 1, dz = q / 3 - 1
  c.r = r;
  c.ch = e.x & ((1 << 27) - 1);
  c.end = e.y;
  c.ccy = cc_of(hcy, q % 3 - 1);
  c.ccz = cc_of(hcz, q / 3 - 1);
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Tiles of BT consecutive rows (one block each): A (hit words) -> block scan ->
// publish -> B (sorted rows into the packed tile) -> resolve -> offsets, stream.
template <int D>
struct R16Shape {
  static constexpr int BT = D == 3 ? 64 : 128;
  static constexpr int PCAP = D == 3 ? 64 * 60 : 128 * 20;  // packed rows per tile
  static constexpr int WMAX = D == 3 ? 20 : 4;              // hit words kept per row
  static constexpr int MINB = D == 3 ? 14 : SPHX_MINB2;     // CTAs per SM (register budget)
};

template <int D, int BT, int PCAP, int WMAX>
__global__ void __launch_bounds__(BT, R16Shape<D>::MINB) k_rcll16(SweepArgs a) {
  constexpr int NR = R16<D>::NR;
  __shared__ __align__(16) int32_t PK[PCAP + 4];
  __shared__ unsigned NIB[WMAX * BT];
  __shared__ int2 RUNS[NR * BT];
  __shared__ int s_w[BT / 32];
  __shared__ long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();  // programmatic launch behind the encode: its runs are complete
#if SPHX_TICKET
  __shared__ int s_tile;
  if (tid == 0) s_tile = (int)(atomicAdd(a.ticket, 1ull) - a.tick0);
  __syncthreads();
  const int tile = s_tile;
#else
  // blocks are dispatched in index order, so tile = blockIdx.x never waits on a
  // tile that has not started (a predecessor that never publishes traps)
  const int tile = blockIdx.x;
#endif
  const int r = tile * BT + tid;
  const bool valid = r < a.nrows;
  const int i = a.row0 + (valid ? r : 0);
  const char* __restrict__ qc = static_cast<const char*>(a.qc);
  const uint4* __restrict__ tags = reinterpret_cast<const uint4*>(a.qtag);

  // own particle: coordinates, constants, self record
  __half2 r2[3], hh2[3];
  const unsigned hcy = a.c.h_cc[1], hcz = a.c.h_cc[2];
  const __half2 hc2 = __half2half2(hbits(a.c.h_cc[0])), thr2 = __half2half2(hbits(a.c.h_thr));
  {
    const typename Coord<D, FP16>::T o = ldg<typename Coord<D, FP16>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r2[k] = k < D ? __half2half2(axis_of<D, FP16>(o, k)) : u2h(0u);
      hh2[k] = __half2half2(hbits(a.c.h_hh[k]));
    }
  }
  const unsigned self = __ldg(a.selfpos + i);  // record index (may exceed 2^31)
  const int selfch = (int)(self >> 2);
  const unsigned selfmask = ~(1u << (28 + (self & 3u)));

  // the particle's non-empty runs, (dz, dy) ascending
  int nruns = 0;
  {
    const int nx = a.g.counts[0], ny = a.g.counts[1], nz = a.g.counts[2];
    const int cx = __ldg(a.cellk[0] + i), cy = __ldg(a.cellk[1] + i);
    const int cz = D == 3 ? __ldg(a.cellk[2] + i) : 0;
    const bool ok = valid && cx >= 0 && cx < nx && cy >= 0 && cy < ny && cz >= 0 && cz < nz;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int dy = (q % 3) - 1, dz = D == 3 ? (q / 3) - 1 : 0;
      int y = cy + dy, z = cz + dz;
      bool in = ok;
      if (y < 0) { y += ny; in = in && a.g.wrap[1]; }
      else if (y >= ny) { y -= ny; in = in && a.g.wrap[1]; }
      if (D == 3) {
        if (z < 0) { z += nz; in = in && a.g.wrap[2]; }
        else if (z >= nz) { z -= nz; in = in && a.g.wrap[2]; }
      }
      if (in) {
        const int2 t = __ldg(a.tri + ((int64_t)z * ny + y) * nx + cx);
        if (t.y > t.x) {
          RUNS[nruns * BT + tid] = make_int2(t.x | ((D == 3 ? q : q + 3) << 27), t.y);
          ++nruns;
        }
      }
    }
  }

  // A: hit words. Each run is tested in groups of up to 8 chunks (one word); the
  // id quads of chunks with hits are prefetched into L1 for B.
  int k = 0, w = 0;
  for (int q = 0; q < nruns; ++q) {
    RunCursor c;
    run_open<D, BT>(RUNS, tid, q, c, hcy, hcz);
    for (int g = c.ch; g < c.end; g += 8) {
      const int e = min(g + 8, c.end);
      unsigned acc = 0;
#pragma unroll(kPhaseAUnroll)
      for (int ch = g; ch < e; ++ch) {
        r16_chunk<D>(qc, ch, r2, hh2, hc2, thr2, c.ccy, c.ccz, acc);
        if (ch == selfch) acc &= selfmask;
        if (acc >> 28) prefetch_l1(tags + ch);
      }
      acc >>= 4 * (8 - (e - g));
      k += __popc(acc);
      if (w < WMAX) NIB[w * BT + tid] = acc;
      ++w;
    }
  }

  const int incl = warp_inclusive_scan(k);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int wbase = 0, btot = 0;
#pragma unroll
  for (int u = 0; u < BT / 32; ++u) {
    wbase += u < warp ? s_w[u] : 0;
    btot += s_w[u];
  }
  const int excl = wbase + incl - k;
  if (tid == 0) lookback_publish(a.tiles, tile, btot, a.epoch);

  // B: sorted rows, hits appended with predicated stores; a run whose first id
  // is below the row's last is merged in (runs interleave only where two cell
  // rows share id ranges).
  auto build = [&](const auto& dst) {
    int kk = 0, wq = 0;
    for (int q = 0; q < nruns; ++q) {
      RunCursor c;
      run_open<D, BT>(RUNS, tid, q, c, hcy, hcz);
      const int gs = kk;
      for (int g = c.ch; g < c.end; g += 8) {
        unsigned word;
        if (wq < WMAX) {
          word = NIB[wq * BT + tid];
        } else {  // not kept: test again
          const int e = min(g + 8, c.end);
          word = 0;
          for (int ch = g; ch < e; ++ch) {
            r16_chunk<D>(qc, ch, r2, hh2, hc2, thr2, c.ccy, c.ccz, word);
            if (ch == selfch) word &= selfmask;
          }
          word >>= 4 * (8 - (e - g));
        }
        ++wq;
        while (word) {  // next chunk with hits
          const int sh = (__ffs(word) - 1) & ~3;
          const unsigned m = (word >> sh) & 15u;
          word &= ~(15u << sh);
          append4(dst, kk, m, __ldg(tags + g + (sh >> 2)));
        }
      }
      if (gs > 0 && kk > gs && dst.ld(gs) < dst.ld(gs - 1)) merge_tail(dst, gs, kk);
    }
  };
  const bool fits = btot <= PCAP;
  if (fits && valid && k > 0)
    build(SharedRow{(uint32_t)__cvta_generic_to_shared(PK) + 4u * (uint32_t)excl});

  if (warp == 0) {
    const long long b = lookback_resolve(a.tiles, tile, btot, a.epoch);
    if (lane == 0) s_base = b;
  }
  __syncthreads();
  const long long base = s_base;
  if (valid) a.offsets[r] = base + excl;
  if (r == a.nrows - 1) a.offsets[a.nrows] = base + excl + k;
  if (base + btot > a.capacity) return;

  int32_t* gout = a.items + base;
  if (!fits) {
    if (valid && k > 0) build(GlobalRow{gout + excl});
    return;
  }
  stream_tile<BT>(gout, SharedRow{(uint32_t)__cvta_generic_to_shared(PK)}, btot, tid);
}

// ------------------------------------------------------------------------------
// FP16 RCLL in two kernels. The candidate tests are latency-bound and want every
// resident warp they can get, while the ordered part (scan, look-back, sorted rows,
// coalesced stores) is light; splitting them keeps the look-back off the tests.
//   k_r16_test: one thread per row, no shared memory, no inter-block dependency:
//     hit words (groups of <= 8 chunks of a run, in (dz, dy) run order) -> hitw,
//     row length -> rowk (bit 31: more than W words).
//   k_r16_emit: tiles of BT rows: block scan of rowk, look-back, sorted rows into a
//     packed shared tile from the hit words and the id quads, 16-byte stores.
// ------------------------------------------------------------------------------
template <int D>
struct R16Two {
  static constexpr int W = D == 3 ? 16 : 4;          // hit words per row
  static constexpr int TB = 256, TMINB = D == 3 ? 4 : 5;   // test kernel: threads, CTAs/SM
  // emit tiles: 128 rows up to 8M rows, 64 above (measured: C3 457 vs 465 us,
  // C5 117 vs 124 ms); the look-back buffer is sized for the smaller tile
  static constexpr int BT = 128, BT_LARGE = 64;
  static constexpr int64_t LARGE_ROWS = 8 << 20;
  static constexpr int PCAP_ROW = D == 3 ? 60 : 20;   // packed entries per row of a tile
  static constexpr int EMINB = D == 3 ? 7 : 10, EMINB_LARGE = 12;
};

// the row's run in each (dz, dy) slot q (empty: cb == ce), RCLL cell of particle i
template <int D>
__device__ __forceinline__ void r16_runs(const SweepArgs& a, int i, bool valid, int (&cb)[R16<D>::NR],
                                         int (&ce)[R16<D>::NR]) {
  constexpr int NR = R16<D>::NR;
  const int nx = a.g.counts[0], ny = a.g.counts[1], nz = a.g.counts[2];
  const int cx = __ldg(a.cellk[0] + i), cy = __ldg(a.cellk[1] + i);
  const int cz = D == 3 ? __ldg(a.cellk[2] + i) : 0;
  const bool ok = valid && cx >= 0 && cx < nx && cy >= 0 && cy < ny && cz >= 0 && cz < nz;
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    // 2-D: the x-triple of row cy + q - 1; 3-D: the xy run of plane cz + q - 1
    int y = D == 3 ? cy : cy + q - 1, z = D == 3 ? cz + q - 1 : 0;
    bool in = ok;
    if (D == 2) {
      if (y < 0) { y += ny; in = in && a.g.wrap[1]; }
      else if (y >= ny) { y -= ny; in = in && a.g.wrap[1]; }
    } else {
      if (z < 0) { z += nz; in = in && a.g.wrap[2]; }
      else if (z >= nz) { z -= nz; in = in && a.g.wrap[2]; }
    }
    int2 t = make_int2(0, 0);
    if (in) t = __ldg(a.tri + ((int64_t)z * ny + y) * nx + cx);
    cb[q] = t.x;
    ce[q] = t.y;
  }
}

// everything the tests of one particle need
template <int D>
struct R16Own {
  __half2 r2[3], hh2[3], hc2, thr2;
  unsigned hcy, hcz;
  int selfch;
  unsigned selfmask;
  __device__ __forceinline__ void init(const SweepArgs& a, int i) {
    const typename Coord<D, FP16>::T o = ldg<typename Coord<D, FP16>::T>(a.pos_own, i);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r2[k] = k < D ? __half2half2(axis_of<D, FP16>(o, k)) : u2h(0u);
      hh2[k] = __half2half2(hbits(a.c.h_hh[k]));
    }
    hc2 = __half2half2(hbits(a.c.h_cc[0]));
    thr2 = __half2half2(hbits(a.c.h_thr));
    hcy = a.c.h_cc[1];
    hcz = a.c.h_cc[2];
    const unsigned self = __ldg(a.selfpos + i);  // record index (may exceed 2^31)
    selfch = (int)(self >> 2);
    selfmask = ~(1u << (28 + (self & 3u)));
  }
  // hit word of chunks [g, e) of the run in slot q
  template <int Q>
  __device__ __forceinline__ unsigned group(const char* __restrict__ qc, int g, int e) const {
    // 2-D: the run's y centre difference; 3-D: per-record dcy times the y edge,
    // and the run's z centre difference
    const __half2 ccy = D == 3 ? __half2half2(hbits(hcy)) : cc_of(hcy, Q - 1);
    const __half2 ccz = D == 3 ? cc_of(hcz, Q - 1) : u2h(0u);
    unsigned acc = 0;
#pragma unroll 4
    for (int ch = g; ch < e; ++ch) {
      r16_chunk<D, (Q == R16<D>::NR / 2)>(qc, ch, r2, hh2, hc2, thr2, ccy, ccz, acc);
      if (Q == R16<D>::NR / 2 && ch == selfch) acc &= selfmask;
    }
    return acc >> (4 * (8 - (e - g)));
  }
};

template <int D, int Q, class F>
__device__ __forceinline__ void r16_for_slots(F&& f) {
  if constexpr (Q < R16<D>::NR) {
    f(std::integral_constant<int, Q>());
    r16_for_slots<D, Q + 1>(f);
  }
}

// Rows are visited in cell (CSR) order, so the lanes of a warp are particles of
// two or three cells that share their runs: the candidate loads of those lanes
// coalesce and their loops run in step.
template <int D>
__global__ void __launch_bounds__(R16Two<D>::TB, R16Two<D>::TMINB) k_r16_test(SweepArgs a) {
  pdl_trigger();  // the emit may launch once every test CTA has started
  pdl_wait();     // the xy encode has completed
  constexpr int NR = R16<D>::NR, W = R16Two<D>::W;
  const int t = blockIdx.x * R16Two<D>::TB + threadIdx.x;
  if (t >= a.n) return;
  const int i = a.order ? __ldg(a.order + t) : t;
  const int r = i - a.row0;
  if (r < 0 || r >= a.nrows) return;  // not a requested row (or malformed membership)
  const char* __restrict__ qc = static_cast<const char*>(a.qc);
  R16Own<D> own;
  own.init(a, i);
  int cb[NR], ce[NR];
  r16_runs<D>(a, i, true, cb, ce);
  int k = 0, w = 0;
  r16_for_slots<D, 0>([&](auto qv) {
    constexpr int Q = decltype(qv)::value;
    for (int g = cb[Q]; g < ce[Q]; g += 8) {
      const unsigned word = own.template group<Q>(qc, g, min(g + 8, ce[Q]));
      k += __popc(word);
      if (w < W) a.hitw[(int64_t)w * a.nrows + r] = word;
      ++w;
    }
  });
  a.rowk[r] = (int)((unsigned)k | (w > W ? 0x80000000u : 0u));
}

template <int D, int BT, int PCAP>
__global__ void __launch_bounds__(BT, BT == R16Two<D>::BT ? R16Two<D>::EMINB : R16Two<D>::EMINB_LARGE)
    k_r16_emit(SweepArgs a) {
  pdl_wait();  // the tests have completed
  constexpr int NR = R16<D>::NR, W = R16Two<D>::W;
  __shared__ __align__(16) int32_t PK[PCAP + 4];
  __shared__ int s_w[BT / 32];
  __shared__ int s_tile;
  __shared__ long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int)(atomicAdd(a.ticket, 1ull) - a.tick0);
  __syncthreads();
  const int tile = s_tile;
  const int r = tile * BT + tid;
  const bool valid = r < a.nrows;
  const int i = a.row0 + (valid ? r : 0);
  const unsigned kw = valid ? (unsigned)__ldg(a.rowk + r) : 0u;
  const int k = (int)(kw & 0x7FFFFFFFu);
  const bool ovf = kw >> 31;

  const int incl = warp_inclusive_scan(k);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int wbase = 0, btot = 0;
#pragma unroll
  for (int u = 0; u < BT / 32; ++u) {
    wbase += u < warp ? s_w[u] : 0;
    btot += s_w[u];
  }
  const int excl = wbase + incl - k;
  if (tid == 0) lookback_publish(a.tiles, tile, btot, a.epoch);

  const char* __restrict__ qc = static_cast<const char*>(a.qc);
  const uint4* __restrict__ tags = reinterpret_cast<const uint4*>(a.qtag);
  // the sorted row: runs in (dz, dy) order, hits appended with predicated stores;
  // a run whose first id is below the row's last is merged in (runs interleave
  // only where two cell rows / planes share id ranges)
  auto build = [&](const auto& dst) {
    int cb[NR], ce[NR];
    r16_runs<D>(a, i, true, cb, ce);
    R16Own<D> own;
    if (ovf) own.init(a, i);
    int kk = 0, w = 0, ng = 0;
#pragma unroll
    for (int q = 0; q < NR; ++q) ng += (ce[q] - cb[q] + 7) >> 3;
    ng = min(ng, W);
    // hit words six groups ahead of their use (independent loads in flight)
    auto ldw = [&](int v) { return v < ng ? __ldg(a.hitw + (int64_t)v * a.nrows + r) : 0u; };
    unsigned h0 = ldw(0), h1 = ldw(1), h2 = ldw(2), h3 = ldw(3), h4 = ldw(4), h5 = ldw(5);
    r16_for_slots<D, 0>([&](auto qv) {
      constexpr int Q = decltype(qv)::value;
      const int gs = kk;
      for (int g = cb[Q]; g < ce[Q]; g += 8) {
        unsigned word = w < W ? h0 : own.template group<Q>(qc, g, min(g + 8, ce[Q]));
        h0 = h1;
        h1 = h2;
        h2 = h3;
        h3 = h4;
        h4 = h5;
        h5 = ldw(w + 6);
        ++w;
        while (word) {  // next chunk with hits
          const int sh = (__ffs(word) - 1) & ~3;
          const unsigned m = (word >> sh) & 15u;
          word &= ~(15u << sh);
          append4(dst, kk, m, __ldg(tags + g + (sh >> 2)));
        }
      }
      if (gs > 0 && kk > gs && dst.ld(gs) < dst.ld(gs - 1)) merge_tail(dst, gs, kk);
    });
  };
  const bool fits = btot <= PCAP;
  if (fits && valid && k > 0)
    build(SharedRow{(uint32_t)__cvta_generic_to_shared(PK) + 4u * (uint32_t)excl});

  if (warp == 0) {
    const long long b = lookback_resolve(a.tiles, tile, btot, a.epoch);
    if (lane == 0) s_base = b;
  }
  __syncthreads();
  const long long base = s_base;
  if (valid) a.offsets[r] = base + excl;
  if (r == a.nrows - 1) a.offsets[a.nrows] = base + excl + k;
  if (base + btot > a.capacity) return;
  int32_t* gout = a.items + base;
  if (!fits) {
    if (valid && k > 0) build(GlobalRow{gout + excl});
    return;
  }
  stream_tile<BT>(gout, SharedRow{(uint32_t)__cvta_generic_to_shared(PK)}, btot, tid);
}

// ------------------------------------------------------------------------------
// Fused FP16 RCLL -> grad_normalized (the mixed step's core,
// dynamics.cpp:145-155): the neighbour rows never reach HBM. Rows are visited in
// cell order (lanes of a warp share runs); each row is built sorted in a per-thread
// shared-memory slot exactly as the table would hold it, and the FP64 gradient is
// accumulated over it in that order with explicit round-to-nearest operations, so
// the result is bit-identical to grad_normalized(f, ps, rcll(rel, grid, fp16), kp):
//   dx = x_i - x_j; r = sqrt(sum dx^2); R = r/h; dW/dR (kernel.hpp:41-49);
//   gw = dW/dR / (h r) * dx (kernel.hpp:53-64); num += (f_j - f_i) gw;
//   den += (-dx) gw; scale += |dx gw|; g = num/den, or 0 (degenerate) when
//   |den| < 1e-14 * (scale > 0 ? scale : 1) (gradient.cpp:56-79).
// A row longer than the slot is walked in id order by repeated minimum search.
// ------------------------------------------------------------------------------
template <int D>
struct R16Grad {
  static constexpr int BT = D == 3 ? 64 : 128;
  static constexpr int CAP = D == 3 ? 80 : 24;  // row slot
  static constexpr int W = D == 3 ? 16 : 4;     // hit words kept
};

__device__ __forceinline__ double kdwdr(double R, double alpha) {
  if (R < 1.0) return __dmul_rn(alpha, __dadd_rn(__dmul_rn(-2.0, R), __dmul_rn(__dmul_rn(1.5, R), R)));
  if (R < 2.0) {
    const double t = __dsub_rn(2.0, R);
    return __dmul_rn(-alpha, __dmul_rn(__dmul_rn(0.5, t), t));
  }
  return 0.0;
}

template <int D>
struct GradTerm {
  double num[3], den[3], scale[3];
};

template <int D>
struct GradAcc {
  double num[3] = {0.0, 0.0, 0.0}, den[3] = {0.0, 0.0, 0.0}, scale[3] = {0.0, 0.0, 0.0};
  double xi[3], fi, ih;  // ih = RN(1/h)
  struct Nb {  // neighbour j's inputs (positions, field value)
    double x[3], f;
  };
  __device__ __forceinline__ static Nb load(const SweepArgs& a, int j) {
    Nb nb;
#pragma unroll
    for (int k = 0; k < 3; ++k) nb.x[k] = k < D ? __ldg(a.gx[k] + j) : 0.0;
    nb.f = __ldg(a.gf + j);
    return nb;
  }
  __device__ __forceinline__ GradTerm<D> term(const SweepArgs& a, int j) const {
    return term(a, load(a, j));
  }
  __device__ __forceinline__ GradTerm<D> term(const SweepArgs& a, const Nb& nb) const {
    double dx[3], gw[3] = {0.0, 0.0, 0.0}, r2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      dx[k] = __dsub_rn(xi[k], nb.x[k]);
      r2 = __dadd_rn(r2, __dmul_rn(dx[k], dx[k]));
    }
    const double r = __dsqrt_rn(r2);
    if (r != 0.0) {
      const double R = div_by(r, a.gh, ih);
      const double sc = __ddiv_rn(kdwdr(R, a.galpha), __dmul_rn(a.gh, r));
#pragma unroll
      for (int k = 0; k < D; ++k) gw[k] = __dmul_rn(sc, dx[k]);
    }
    const double df = __dsub_rn(nb.f, fi);
    GradTerm<D> t;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      t.num[k] = __dmul_rn(df, gw[k]);
      t.den[k] = __dmul_rn(-dx[k], gw[k]);
      t.scale[k] = fabs(__dmul_rn(dx[k], gw[k]));
    }
    return t;
  }
  __device__ __forceinline__ void acc(const GradTerm<D>& t) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      num[k] = __dadd_rn(num[k], t.num[k]);
      den[k] = __dadd_rn(den[k], t.den[k]);
      scale[k] = __dadd_rn(scale[k], t.scale[k]);
    }
  }
  __device__ __forceinline__ void add(const SweepArgs& a, int j) { acc(term(a, j)); }
};

template <int D, int BT, int CAP, int W>
__global__ void __launch_bounds__(BT) k_r16_grad(SweepArgs a) {
  pdl_wait();  // the encode has completed
  constexpr int NR = R16<D>::NR;
  __shared__ __align__(16) int32_t ROWS[BT * CAP];
  __shared__ unsigned NIB[W * BT];
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = blockIdx.x * BT + tid;
  const bool active = t < a.n;
  const int i = active ? (a.order ? __ldg(a.order + t) : t) : 0;
  const char* __restrict__ qc = static_cast<const char*>(a.qc);
  const uint4* __restrict__ tags = reinterpret_cast<const uint4*>(a.qtag);
  const int32_t* __restrict__ tag1 = reinterpret_cast<const int32_t*>(a.qtag);
  unsigned long long deg = 0;
  if (active) {
    R16Own<D> own;
    own.init(a, i);
    int cb[NR], ce[NR];
    r16_runs<D>(a, i, true, cb, ce);
    // A: hit words
    int k = 0, w = 0;
    r16_for_slots<D, 0>([&](auto qv) {
      constexpr int Q = decltype(qv)::value;
      for (int g = cb[Q]; g < ce[Q]; g += 8) {
        const unsigned word = own.template group<Q>(qc, g, min(g + 8, ce[Q]));
        k += __popc(word);
        if (w < W) NIB[w * BT + tid] = word;
        ++w;
      }
    });
    auto word_at = [&](int wi, auto qv, int g) -> unsigned {
      constexpr int Q = decltype(qv)::value;
      return wi < W ? NIB[wi * BT + tid] : own.template group<Q>(qc, g, min(g + 8, ce[Q]));
    };
    GradAcc<D> acc;
#pragma unroll
    for (int kk = 0; kk < D; ++kk) acc.xi[kk] = __ldg(a.gx[kk] + i);
    acc.fi = __ldg(a.gf + i);
    acc.ih = __drcp_rn(a.gh);
    if (k <= CAP) {
      // B: the sorted row in this thread's slot, then the gradient over it
      const SharedRow row{(uint32_t)__cvta_generic_to_shared(ROWS) + 4u * (uint32_t)(tid * CAP)};
      int kk = 0, wq = 0;
      r16_for_slots<D, 0>([&](auto qv) {
        constexpr int Q = decltype(qv)::value;
        const int gs = kk;
        for (int g = cb[Q]; g < ce[Q]; g += 8) {
          unsigned word = word_at(wq, qv, g);
          ++wq;
          while (word) {  // next chunk with hits
            const int sh = (__ffs(word) - 1) & ~3;
            const unsigned m = (word >> sh) & 15u;
            word &= ~(15u << sh);
            append4(row, kk, m, __ldg(tags + g + (sh >> 2)));
          }
        }
        if (gs > 0 && kk > gs && row.ld(gs) < row.ld(gs - 1)) merge_tail(row, gs, kk);
      });
      if (k > 0) {  // the next neighbour's inputs load while this term is computed
        typename GradAcc<D>::Nb cur = GradAcc<D>::load(a, row.ld(0));
        for (int e = 0; e < k; ++e) {
          const typename GradAcc<D>::Nb nxt = GradAcc<D>::load(a, row.ld(e + 1 < k ? e + 1 : e));
          acc.acc(acc.term(a, cur));
          cur = nxt;
        }
      }
    } else {
      // long row: ids in ascending order by repeated minimum search over the hits
      int last = INT_MIN;
      for (int e = 0; e < k; ++e) {
        int best = INT_MAX, wq = 0;
        r16_for_slots<D, 0>([&](auto qv) {
          constexpr int Q = decltype(qv)::value;
          for (int g = cb[Q]; g < ce[Q]; g += 8) {
            unsigned word = word_at(wq, qv, g);
            ++wq;
            while (word) {
              const int b = __ffs(word) - 1;
              word &= word - 1;
              const int id = __ldg(tag1 + 4 * (int64_t)g + b);
              if (id > last && id < best) best = id;
            }
          }
        });
        acc.add(a, best);
        last = best;
      }
    }
#pragma unroll
    for (int kk = 0; kk < D; ++kk) {
      const double lim = __dmul_rn(1e-14, acc.scale[kk] > 0.0 ? acc.scale[kk] : 1.0);
      double g = 0.0;
      if (fabs(acc.den[kk]) < lim) ++deg;
      else g = __ddiv_rn(acc.num[kk], acc.den[kk]);
      a.gout[kk][i] = g;
    }
  }
  // degenerate pairs: warp sum, one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) deg += __shfl_xor_sync(0xffffffffu, deg, o);
  if (lane == 0 && deg) atomicAdd(a.gdeg, deg);
}

int launch_rcll_grad(int dim, const SweepArgs& a, cudaStream_t st) {
  if (dim == 2) {
    using G = R16Grad<2>;
    launch_pdl(k_r16_grad<2, G::BT, G::CAP, G::W>, (unsigned)((a.n + G::BT - 1) / G::BT), G::BT,
               st, a);
    return 1;
  }
  if (dim == 3) {
    using G = R16Grad<3>;
    launch_pdl(k_r16_grad<3, G::BT, G::CAP, G::W>, (unsigned)((a.n + G::BT - 1) / G::BT), G::BT,
               st, a);
    return 1;
  }
  return 0;
}

// The whole table in one pass over tiles of BT consecutive rows (particle order).
//   A. each thread tests its particle's candidates; the hit words go to shared
//      memory (WMAX per thread; later groups are re-tested in B) and the row
//      length k counts every hit;
//   block scan of k; the tile publishes its aggregate;
//   B. rows are built sorted, packed at their final places in a shared tile
//      (rows longer than the tile buffer go straight to HBM after the look-back);
//   the look-back resolves the tile's base: offsets[] are written and the tile is
//      streamed out with 16-byte stores.
// Tiles are taken in launch order from a ticket counter, so the look-back never
// waits on a tile that has not started.
template <int D, int P, int MODE, int BT, int PCAP, int WMAX>
__global__ void __launch_bounds__(BT) k_sweep(SweepArgs a) {
  static_assert(BT % 32 == 0 && BT <= 1024, "shape");
  __shared__ __align__(16) int32_t PK[PCAP + 4];
  __shared__ unsigned NIB[WMAX * BT];
  __shared__ int s_w[BT / 32];
  __shared__ int s_tile;
  __shared__ long long s_base;
  using Tst = Tester<D, P, MODE>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int)(atomicAdd(a.ticket, 1ull) - a.tick0);
  __syncthreads();
  const int tile = s_tile;
  const int r = tile * BT + tid;
  const bool valid = r < a.nrows;
  const int i = a.row0 + r;

  Tst tst;
  int selfch = -1;
  unsigned selfmask = ~0u;
  int k = 0;
  if (valid) {
    tst.init(a, i);
    const unsigned self = MODE == MODE_ALL ? (unsigned)i : __ldg(a.selfpos + i);
    selfch = (int)(self >> 2);
    selfmask = ~(1u << (28 + (self & 3u)));
    int w = 0;
    walk_groups<D, P, MODE>(a, i, tst, [&](const typename Tst::Row& row, bool own, int g, int e) {
      const unsigned word = group_word<D, P, MODE>(a, tst, row, own, selfch, selfmask, g, e);
      k += __popc(word);
      if (w < WMAX) NIB[w * BT + tid] = word;
      ++w;
    });
  }

  const int incl = warp_inclusive_scan(k);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int wbase = 0, btot = 0;
#pragma unroll
  for (int w = 0; w < BT / 32; ++w) {
    wbase += w < warp ? s_w[w] : 0;
    btot += s_w[w];
  }
  const int excl = wbase + incl - k;
  if (tid == 0) lookback_publish(a.tiles, tile, btot, a.epoch);

  // B: the sorted row of particle i into dst. Chunks are walked in lockstep and
  // their hits appended with predicated stores; a group (run) whose first id is
  // below the row's last one is merged in (rows interleave only where two runs
  // of different cell rows share id ranges).
  auto build = [&](const auto& dst) {
    int kk = 0, w = 0;
    const uint4* tags = reinterpret_cast<const uint4*>(a.qtag);
    walk_groups<D, P, MODE>(a, i, tst, [&](const typename Tst::Row& row, bool own, int g, int e) {
      unsigned word = w < WMAX ? NIB[w * BT + tid]
                               : group_word<D, P, MODE>(a, tst, row, own, selfch, selfmask, g, e);
      ++w;
      const int gs = kk;
      while (word) {  // next chunk with hits
        const int sh = (__ffs(word) - 1) & ~3;
        const unsigned m = (word >> sh) & 15u;
        word &= ~(15u << sh);
        append4(dst, kk, m, __ldg(tags + g + (sh >> 2)));
      }
      if (gs > 0 && kk > gs && dst.ld(gs) < dst.ld(gs - 1)) merge_tail(dst, gs, kk);
    });
  };
  const bool fits = btot <= PCAP;
  if (fits && valid && k > 0)
    build(SharedRow{(uint32_t)__cvta_generic_to_shared(PK) + 4u * (uint32_t)excl});

  if (warp == 0) {
    const long long b = lookback_resolve(a.tiles, tile, btot, a.epoch);
    if (lane == 0) s_base = b;
  }
  __syncthreads();
  const long long base = s_base;
  if (valid) a.offsets[r] = base + excl;
  if (r == a.nrows - 1) a.offsets[a.nrows] = base + excl + k;
  if (base + btot > a.capacity) return;  // device API: the caller grows the table

  int32_t* gout = a.items + base;  // the tile's rows, contiguous
  if (!fits) {
    if (valid && k > 0) build(GlobalRow{gout + excl});
    return;
  }
  stream_tile<BT>(gout, SharedRow{(uint32_t)__cvta_generic_to_shared(PK)}, btot, tid);
}

// ------------------------------------------------------------------------------
// Encode
// ------------------------------------------------------------------------------
// Own coordinates at storage precision, particle order (all_list: round_to,
// nnps.cpp:75-89; the cell modes get theirs from k_encode_rows).
template <int D, int P>
__global__ void k_pack_own(int n, const double* __restrict__ x0, const double* __restrict__ x1,
                           const double* __restrict__ x2, void* __restrict__ pos_own) {
  using C = typename Coord<D, P>::T;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double v[3] = {x0[t], D > 1 ? x1[t] : 0.0, D > 2 ? x2[t] : 0.0};
  reinterpret_cast<C*>(pos_own)[t] = pack<D, P>(v);
}

// Chunk start of cell c's run: with st(x) = cell_start[row + x], n_x the cell
// counts and A(c) = st(cx-1) + st(cx) + st(cx+1) (clamped to the row on an open
// x axis; on a periodic one st(-1) = st(0) - n_{X-1} and A += n_{X-1} - n_0),
// consecutive A differ by exactly the triple length and each x row of cells
// stays inside [3 st(0), 3 st(X)). Rounding A + 6c up to a multiple of 4 leaves
// room to pad every run to whole chunks; all runs fit in 3n + 6C records.
__device__ __forceinline__ int64_t run_record_slot(const int32_t* st, int cx, int nx, int wrapx,
                                                   int64_t c) {
  int64_t A;
  if (!wrapx) {
    A = (int64_t)st[cx > 0 ? cx - 1 : 0] + st[cx] + st[cx + 1 < nx ? cx + 1 : nx];
  } else {
    const int n0 = st[1] - st[0], nl = st[nx] - st[nx - 1];
    const int stm1 = cx > 0 ? st[cx - 1] : st[0] - nl;
    A = (int64_t)stm1 + st[cx] + st[cx + 1] + nl - n0;
  }
  return (A + 6 * c + 3) & ~int64_t(3);
}

// record r (chunk r/4, element r%4), quad q
template <int D, int P, int MODE>
__device__ __forceinline__ void store_el(void* qc, int64_t r, int q, typename Prec<P>::T v) {
  *rec_el<D, P, MODE>(qc, r >> 2, q, (int)(r & 3)) = v;
}

// all_list: chunks of 4 consecutive particles (one run over everything).
template <int D, int P>
__global__ void k_encode_all(int n, const void* __restrict__ pos_own, SweepArgs a) {
  using T = typename Prec<P>::T;
  using Q = typename Prec<P>::Quad;
  using CT = typename Coord<D, P>::T;
  const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch * 4 >= n) return;
  Q qx[3];
  uint4 qt;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t j = ch * 4 + u;
    T xs[3];
    unsigned tag = 0xFFFFFFFFu;
    if (j < n) {
      const CT cj = ldg<CT>(pos_own, j);
#pragma unroll
      for (int k = 0; k < D; ++k) xs[k] = axis_of<D, P>(cj, k);
      tag = (unsigned)j;
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if constexpr (P == FP16) xs[k] = hbits(0x7E00u); else xs[k] = T(NAN);
      }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) qset(qx[k], u, xs[k]);
    if (u == 0) qt.x = tag; else if (u == 1) qt.y = tag; else if (u == 2) qt.z = tag; else qt.w = tag;
  }
#pragma unroll
  for (int k = 0; k < D; ++k)
    *reinterpret_cast<Q*>(rec_el<D, P, MODE_ALL>(a.qc, ch, k, 0)) = qx[k];
  reinterpret_cast<uint4*>(a.qtag)[ch] = qt;
}

template <int D>
struct Shape {
  static constexpr int BT = D == 3 ? 64 : 128;                     // rows per tile
  static constexpr int PCAP = D == 3 ? 64 * 64 : (D == 2 ? 128 * 24 : 128 * 8);  // packed tile
  static constexpr int WMAX = D == 3 ? 24 : (D == 2 ? 8 : 4);      // hit words kept per row
};

// ------------------------------------------------------------------------------
// Host-side launchers (called from capi.cu)
// ------------------------------------------------------------------------------
int sweep_tile(int dim, int prec, int mode) {
  if (prec == FP16 && mode == MODE_RCLL && dim >= 2)
    return dim == 3 ? R16Two<3>::BT_LARGE : R16Shape<2>::BT;  // the smaller 3-D tile
  return dim == 3 ? Shape<3>::BT : Shape<2>::BT;
}
size_t coord_bytes(int dim, int prec) {
  if (prec == FP16) return dim == 3 ? 8 : 4;
  if (prec == FP32) return dim == 1 ? 4 : (dim == 2 ? 8 : 16);
  return dim == 1 ? 8 : (dim == 2 ? 16 : 32);
}
// hit words per row the two-kernel FP16 RCLL sweep keeps (0: single kernel)
int hit_words(int dim, int prec, int mode) {
  if (prec == FP16 && mode == MODE_RCLL && dim == 3) return R16Two<3>::W;
  return 0;
}
size_t chunk_bytes(int dim, int prec, int mode) {
#define CB(D, P, M) if (dim == D && prec == P && mode == M) return ChunkLay<D, P, M>::BYTES;
  CB(1, FP16, MODE_RCLL) CB(2, FP16, MODE_RCLL) CB(3, FP16, MODE_RCLL)
  CB(1, FP32, MODE_RCLL) CB(2, FP32, MODE_RCLL) CB(3, FP32, MODE_RCLL)
  CB(1, FP64, MODE_RCLL) CB(2, FP64, MODE_RCLL) CB(3, FP64, MODE_RCLL)
  CB(1, FP16, MODE_CLL) CB(2, FP16, MODE_CLL) CB(3, FP16, MODE_CLL)
  CB(1, FP32, MODE_CLL) CB(2, FP32, MODE_CLL) CB(3, FP32, MODE_CLL)
  CB(1, FP64, MODE_CLL) CB(2, FP64, MODE_CLL) CB(3, FP64, MODE_CLL)
  CB(1, FP16, MODE_ALL) CB(2, FP16, MODE_ALL) CB(3, FP16, MODE_ALL)
  CB(1, FP32, MODE_ALL) CB(2, FP32, MODE_ALL) CB(3, FP32, MODE_ALL)
  CB(1, FP64, MODE_ALL) CB(2, FP64, MODE_ALL) CB(3, FP64, MODE_ALL)
#undef CB
  return 0;
}
// chunks the candidate arrays need
int64_t chunk_capacity(int dim, int prec, int mode, int64_t n, int64_t C) {
  if (mode == MODE_ALL) return (n + 3) / 4 + 1;
  if (dim == 3 && prec == FP16 && mode == MODE_RCLL) return (9 * n) / 4 + C + 2;  // xy runs
  return (3 * n + 6 * C) / 4 + 2;
}

// ------------------------------------------------------------------------------
// Row-tiled encode (RCLL / CLL): one CTA per XB consecutive cells of one cell row
// (the x-fastest linear cell index makes the row's slots and its runs contiguous).
//   1. the member window -- cells [x0-2, x1+2) -- is staged in shared memory: merge
//      key (id, or global id of a slab), CSR id and coordinates at storage precision
//      (RelCoords::rel for RCLL, positions for CLL; round_to, nnps.cpp:304-315/75-89);
//   2. each member of cells [x0-1, x1] is placed in the runs centred at x-1, x, x+1
//      that this CTA owns: its position is its index in its cell plus the number of
//      smaller keys in the run's two other cells (binary search; cells hold ascending
//      keys), i.e. its place in the id-merge of the three cells;
//   3. the CTA's runs -- a contiguous chunk range -- are assembled in shared memory
//      (sentinels: NaN coordinates, id ~0) and written out with 16-byte stores.
// Own-cell members also get pos_own (particle order) and selfpos. The candidate's
// cell is its CSR cell and its x offset dc = 1 - list (nnps.cpp:359-362); CLL
// records of a wrapped list carry round_to(prec, x + shift) (nnps.cpp:116).
// ------------------------------------------------------------------------------
struct EncArgs {
  int nx, nxb, wrapx;
  int ny, wrapy;               // xy-plane runs (3-D FP16 RCLL)
  const int32_t* cstart;       // xy runs: first chunk of each cell's run (scan), [C+1]
  int64_t nrows;               // cell rows (ny * nz)
  const int32_t* start;        // CellGrid::cell_start
  const int32_t* items;        // CellGrid::items
  const double* x[3];          // rel (RCLL) or positions (CLL)
  PrecConsts pc;
};

template <int D, int P>
struct EncShape {
  // 2-D: 32-cell rows of 128 threads (9 waves at C2 instead of 3.3 with 64-cell
  // rows of 256: 47.6 vs 50.7 us)
  static constexpr int XB = 32;                     // cells per CTA
  static constexpr int BT = D == 3 ? 256 : 128;
  static constexpr int WCAP = D == 3 ? 1024 : 512;  // staged window members
  static constexpr int OCAP = D == 3 ? 512 : 256;   // staged chunks
};

// window: key, id (int32), coordinates; then the chunks and their ids
template <int D, int P, int MODE>
constexpr size_t enc_smem_bytes() {
  using E = EncShape<D, P>;
  using L = ChunkLay<D, P, MODE>;
  return (size_t)E::WCAP * (8 + D * sizeof(typename Prec<P>::T)) + (size_t)E::OCAP * (L::BYTES + 16);
}

template <int D, int P, int MODE>
__global__ void __launch_bounds__(EncShape<D, P>::BT) k_encode_rows(EncArgs e, SweepArgs a) {
  // programmatic dependent launch of the 2-D sweep: each CTA triggers after its
  // stores (triggering at the start measured 149 vs 137 us at C2; at the end 136.5)
  using E = EncShape<D, P>;
  using L = ChunkLay<D, P, MODE>;
  using T = typename Prec<P>::T;
  constexpr int XB = E::XB, BT = E::BT, NW = XB + 4;
  extern __shared__ __align__(16) unsigned char sm[];
  int32_t* skey = reinterpret_cast<int32_t*>(sm);
  int32_t* sid = skey + E::WCAP;
  T* scrd = reinterpret_cast<T*>(sid + E::WCAP);                 // [D][WCAP]
  unsigned char* sch = sm + (size_t)E::WCAP * (8 + D * sizeof(T));  // [OCAP][BYTES]
  uint32_t* stag = reinterpret_cast<uint32_t*>(sch + (size_t)E::OCAP * L::BYTES);  // [OCAP*4]
  __shared__ int wst[NW + 1];   // window member offset of local cell u
  __shared__ int wgs[NW];       // CSR slot of local cell u's first member
  __shared__ int wraw[NW];      // unwrapped x of local cell u
  __shared__ int64_t s_ch0;     // first chunk of the CTA's runs
  __shared__ int s_nch;         // chunks of the CTA's runs

  const int tid = threadIdx.x;
  const int64_t row = blockIdx.x / e.nxb;
  const int x0 = (int)(blockIdx.x % e.nxb) * XB;
  const int x1 = min(x0 + XB, e.nx);
  const int nx = e.nx;
  const int32_t* st = e.start + row * nx;  // st[nx] is the next row's first slot
  const int64_t crow = row * nx;

  // window cells (count and first slot), prefix over them by warp 0
  __shared__ int64_t rslot[XB];  // first record of each run owned here
  if (tid < 32) {
    int tot = 0;
    for (int u0 = 0; u0 < NW; u0 += 32) {
      const int u = u0 + tid;
      int cnt = 0;
      if (u < NW) {
        int gx = x0 - 2 + u, gs = 0;
        wraw[u] = gx;
        bool ok = gx >= 0 && gx < nx;
        if (!ok && e.wrapx) {
          gx = ((gx % nx) + nx) % nx;
          ok = true;
        }
        if (ok) {
          gs = st[gx];
          cnt = st[gx + 1] - gs;
        }
        wgs[u] = gs;
      }
      const int incl = warp_inclusive_scan(cnt);
      if (u < NW) wst[u + 1] = tot + incl;
      tot += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) wst[0] = 0;
  }
  for (int v = tid; v < x1 - x0; v += BT)
    rslot[v] = run_record_slot(st, x0 + v, nx, e.wrapx, crow + x0 + v);
  __syncthreads();
  const int W = wst[NW];
  const bool win_sm = W <= E::WCAP;

  // member window: key, id, coordinates
  auto cell_of_member = [&](int m) {  // last u with wst[u] <= m (binary lifting)
    static_assert(NW < 128, "window cells");
    int w = 0;
#pragma unroll
    for (int st = 64; st > 0; st >>= 1)
      if (w + st < NW && wst[w + st] <= m) w += st;
    return w;
  };
  auto member = [&](int m, int& u) {
    u = cell_of_member(m);
    return __ldg(e.items + wgs[u] + (m - wst[u]));
  };
  if (win_sm) {
    for (int m = tid; m < W; m += BT) {
      int u;
      const int j = member(m, u);
      sid[m] = j;
      skey[m] = a.ids ? __ldg(a.ids + j) : j;
#pragma unroll
      for (int k = 0; k < D; ++k) scrd[k * E::WCAP + m] = Prec<P>::cvt(__ldg(e.x[k] + j));
    }
  }
  auto key_of = [&](int m) -> int {
    if (win_sm) return skey[m];
    int u;
    const int j = member(m, u);
    return a.ids ? __ldg(a.ids + j) : j;
  };
  auto id_of = [&](int m) -> int {
    int u;
    return win_sm ? sid[m] : member(m, u);
  };
  auto crd_of = [&](int m, int k) -> T {
    if (win_sm) return scrd[k * E::WCAP + m];
    int u;
    return Prec<P>::cvt(__ldg(e.x[k] + member(m, u)));
  };

  // runs: chunk ranges (tri) and the CTA's chunk span
  if (tid < x1 - x0) {
    const int t = x0 + tid, u = t - x0 + 2;
    const int len = (wst[u + 2] - wst[u - 1]);
    const int64_t slot = rslot[tid];
    const int nch = (len + 3) >> 2;
    a.tri[crow + t] = make_int2((int)(slot >> 2), (int)((slot >> 2) + nch));
    if (tid == 0) s_ch0 = slot >> 2;
    if (t == x1 - 1) s_nch = (int)((slot >> 2) + nch - (rslot[0] >> 2));
  }
  __syncthreads();
  const int64_t ch0 = s_ch0;
  const int nch = s_nch;
  const bool out_sm = nch <= E::OCAP;

  T nanv;
  if constexpr (P == FP16) nanv = hbits(0x7E00u); else nanv = T(NAN);
  // sentinel fill of the CTA's chunks (records past each run's end stay sentinels)
  if (out_sm) {
    for (int q = tid; q < nch * 4; q += BT) {
      const int c = q >> 2, l = q & 3;
#pragma unroll
      for (int k = 0; k < D; ++k) *rec_el<D, P, MODE>(sch, c, k, l) = nanv;
      if constexpr (MODE == MODE_RCLL) *rec_el<D, P, MODE>(sch, c, D, l) = T(0.0f);
      stag[q] = 0xFFFFFFFFu;
    }
  } else {
    // direct: pad records of each run
    for (int t = x0 + tid; t < x1; t += BT) {
      const int u = t - x0 + 2;
      const int len = wst[u + 2] - wst[u - 1];
      const int64_t slot = rslot[t - x0];
      for (int q = len; q < ((len + 3) & ~3); ++q) {
#pragma unroll
        for (int k = 0; k < D; ++k) store_el<D, P, MODE>(a.qc, slot + q, k, nanv);
        if constexpr (MODE == MODE_RCLL) store_el<D, P, MODE>(a.qc, slot + q, D, T(0.0f));
        reinterpret_cast<unsigned*>(a.qtag)[slot + q] = 0xFFFFFFFFu;
      }
    }
  }
  __syncthreads();

  // number of keys < key in window cell u
  auto less_in = [&](int u, int key) {
    int lo = wst[u], hi = wst[u + 1];
    if (win_sm && hi - lo <= 16) {  // branch-free for the first 8 keys
      int c = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) c += (lo + q < hi) & (skey[min(lo + q, hi - 1)] < key);
      for (int q = lo + 8; q < hi; ++q) c += skey[q] < key;
      return c;
    }
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (key_of(mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo - wst[u];
  };

  // records: members of window cells 1 .. XB+2 (x0-1 .. x1)
  const int mlo = wst[1], mhi = wst[min(x1 - x0 + 3, NW)];
  for (int m = mlo + tid; m < mhi; m += BT) {
    const int u = cell_of_member(m);  // >= 1: m >= wst[1]
    const int idx = m - wst[u];
    const int key = key_of(m), j = id_of(m);
    T c[3];
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = crd_of(m, k);
    // runs centred at local u-1, u, u+1 owned by this CTA (local 2 .. x1-x0+1)
    int lt[3];
    lt[0] = u > 1 ? less_in(u - 2, key) : 0;
    lt[1] = less_in(u - 1, key);
    lt[2] = u + 1 < NW ? less_in(u + 1, key) : 0;
    const int lt3 = u + 2 < NW ? less_in(u + 2, key) : 0;
#pragma unroll
    for (int Lr = 0; Lr < 3; ++Lr) {  // member is list Lr of the run centred at local v
      const int v = u + 1 - Lr;
      if (v < 2 || v >= x1 - x0 + 2) continue;
      // other lists of run v: cells v-1, v, v+1 except u
      int pos = idx;
      if (Lr == 0) pos += lt[2] + lt3;              // cells u+1, u+2
      else if (Lr == 1) pos += lt[1] + lt[2];       // cells u-1, u+1
      else pos += lt[0] + lt[1];                    // cells u-2, u-1
      const int64_t rec = rslot[v - 2] + pos;
      T cx = c[0];
      if constexpr (MODE == MODE_CLL) {
        const int raw = wraw[u];
        const int w = raw < 0 ? -1 : (raw >= nx ? 1 : 0);
        if (w != 0) {  // round_to(prec, x + shift), nnps.cpp:116
          T sh;
          if constexpr (P == FP16) sh = hbits(e.pc.h_sh[0]);
          else if constexpr (P == FP32) sh = e.pc.f_sh[0];
          else sh = e.pc.d_sh[0];
          if constexpr (P == FP16) cx = __hadd_rn(cx, w > 0 ? sh : __hneg(sh));
          else cx = f_add(cx, w > 0 ? sh : -sh);
        }
      }
      const uint32_t tag = a.ids ? (uint32_t)key : (uint32_t)j;
      if (out_sm) {
        const int lr = (int)(rec - 4 * ch0);
        *rec_el<D, P, MODE>(sch, lr >> 2, 0, lr & 3) = cx;
#pragma unroll
        for (int k = 1; k < D; ++k) *rec_el<D, P, MODE>(sch, lr >> 2, k, lr & 3) = c[k];
        if constexpr (MODE == MODE_RCLL) *rec_el<D, P, MODE>(sch, lr >> 2, D, lr & 3) = (T)(float)(1 - Lr);
        stag[lr] = tag;
      } else {
        store_el<D, P, MODE>(a.qc, rec, 0, cx);
#pragma unroll
        for (int k = 1; k < D; ++k) store_el<D, P, MODE>(a.qc, rec, k, c[k]);
        if constexpr (MODE == MODE_RCLL) store_el<D, P, MODE>(a.qc, rec, D, (T)(float)(1 - Lr));
        reinterpret_cast<uint32_t*>(a.qtag)[rec] = tag;
      }
      if (Lr == 1) {  // own cell: pos_own and the self record
        a.selfpos[j] = (uint32_t)rec;
        T own[3] = {c[0], D > 1 ? c[1] : T(0.0f), D > 2 ? c[2] : T(0.0f)};
        typename Coord<D, P>::T pk;
        if constexpr (P == FP16) {
          const __half2 xy = __halves2half2(own[0], D > 1 ? own[1] : hbits(0));
          if constexpr (D == 3) pk = make_uint2(h2u(xy), h2u(__halves2half2(own[2], hbits(0))));
          else pk = xy;
        } else if constexpr (D == 1) {
          pk = own[0];
        } else if constexpr (D == 2) {
          pk.x = own[0];
          pk.y = own[1];
        } else {
          pk.x = own[0];
          pk.y = own[1];
          pk.z = own[2];
          pk.w = T(0);
        }
        reinterpret_cast<typename Coord<D, P>::T*>(const_cast<void*>(a.pos_own))[j] = pk;
      }
    }
  }
  __syncthreads();
  if (out_sm) {  // stream the CTA's chunks and id quads
    const uint4* src = reinterpret_cast<const uint4*>(sch);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(a.qc) + ch0 * L::BYTES);
    if constexpr (L::BYTES >= 16) {
      for (int q = tid; q < nch * (L::BYTES / 16); q += BT) dst[q] = src[q];
    } else {
      const uint2* s2 = reinterpret_cast<const uint2*>(sch);
      uint2* d2 = reinterpret_cast<uint2*>(static_cast<char*>(a.qc) + ch0 * L::BYTES);
      for (int q = tid; q < nch; q += BT) d2[q] = s2[q];
    }
    const uint4* ts = reinterpret_cast<const uint4*>(stag);
    uint4* td = reinterpret_cast<uint4*>(a.qtag) + ch0;
    for (int q = tid; q < nch; q += BT) td[q] = ts[q];
  }
  pdl_trigger();  // after this CTA's stores: the sweep launches behind the last CTAs
}

// ------------------------------------------------------------------------------
// 3-D FP16 RCLL: xy-plane runs. The run of cell (x, y, z) is the id-merge of the
// nine cells (x-1..x+1, y-1..y+1, z) (wrapped on periodic x / y, absent beyond a
// wall); each record carries dcx and dcy (= -offset, the minimum image, nnps.cpp:
// 359-362). A particle then has 3 runs (dz = -1, 0, 1) whose hits interleave only
// where a lattice plane straddles two cell planes, so its row is built with few
// merges. Run slots are a scan of the run lengths (k_xy_runlen + k_scan_counts).
// ------------------------------------------------------------------------------
__global__ void k_xy_runlen(int64_t C, int nx, int ny, int wrapx, int wrapy,
                            const int32_t* __restrict__ start, int32_t* __restrict__ nch) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int x = (int)(c % nx), y = (int)((c / nx) % ny);
  const int64_t plane = c - x - (int64_t)y * nx;
  int len = 0;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    int yy = y + dy;
    if (yy < 0 || yy >= ny) {
      if (!wrapy) continue;
      yy = yy < 0 ? yy + ny : yy - ny;
    }
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      int xx = x + dx;
      if (xx < 0 || xx >= nx) {
        if (!wrapx) continue;
        xx = xx < 0 ? xx + nx : xx - nx;
      }
      const int64_t cc = plane + (int64_t)yy * nx + xx;
      len += __ldg(start + cc + 1) - __ldg(start + cc);
    }
  }
  nch[c] = (len + 3) >> 2;
}

struct XYShape {
  static constexpr int XB = 16, BT = 256;
  static constexpr int NW = XB + 4;      // window cells per row (x0-2 .. x1+1)
  static constexpr int WCAP = 1024;      // staged window members
  static constexpr int OCAP = 640;       // staged chunks (48 B + 16 B ids each)
};

constexpr size_t xy_smem_bytes() {
  return (size_t)XYShape::WCAP * (4 + 4 + 4 + 2 + 1) +
         (size_t)XYShape::OCAP * (ChunkLay<3, FP16, MODE_RCLL>::BYTES + 16);
}

__global__ void __launch_bounds__(XYShape::BT) k_encode_xy(EncArgs e, SweepArgs a) {
  pdl_trigger();  // the tests may launch once every encode CTA has started
  using S = XYShape;
  using L = ChunkLay<3, FP16, MODE_RCLL>;
  constexpr int XB = S::XB, BT = S::BT, NW = S::NW, NWC = 3 * NW;
  extern __shared__ __align__(16) unsigned char sm[];
  int32_t* skey = reinterpret_cast<int32_t*>(sm);              // merge key, window order
  int32_t* sid = skey + S::WCAP;                                // particle id
  int32_t* sstrip = sid + S::WCAP;                              // keys of each column strip, sorted
  int16_t* srank = reinterpret_cast<int16_t*>(sstrip + S::WCAP); // rank in the member's strip
  uint8_t* sw = reinterpret_cast<uint8_t*>(srank + S::WCAP);     // window cell of the member
  unsigned char* sch = sm + (size_t)S::WCAP * 15;               // [OCAP][48]
  uint32_t* stag = reinterpret_cast<uint32_t*>(sch + (size_t)S::OCAP * L::BYTES);
  __shared__ int wst[NWC + 1];   // window member offset of window cell w = r * NW + u
  __shared__ int wgs[NWC];       // CSR slot of window cell w's first member
  __shared__ int sst[NW + 1];    // strip member offset of window column u (its 3 cells)
  __shared__ int64_t s_ch0;
  __shared__ int s_nch;

  const int tid = threadIdx.x;
  const int nx = e.nx, ny = e.ny;
  const int64_t row = blockIdx.x / e.nxb;        // (y, z) row of the centre cells
  const int x0 = (int)(blockIdx.x % e.nxb) * XB;
  const int x1 = min(x0 + XB, nx);
  const int y = (int)(row % ny);
  const int64_t plane = (row - y) * nx;         // first cell of plane z
  const int nrun = x1 - x0;

  // empty runs only (a run holds its own cell, so the CTA's cells are empty too):
  // the chunk ranges are all that is written (dam-break C4: 3/4 of the grid)
  {
    const int64_t c0 = plane + (int64_t)y * nx + x0;
    if (e.cstart[c0 + nrun] == e.cstart[c0]) {
      for (int v = tid; v < nrun; v += BT) a.tri[c0 + v] = make_int2(e.cstart[c0], e.cstart[c0]);
      return;
    }
  }

  // window cells: rows y-1, y, y+1 (r = 0, 1, 2), columns x0-2 .. x1+1
  if (tid < 32) {
    int tot = 0;
    for (int w0 = 0; w0 < NWC; w0 += 32) {
      const int w = w0 + tid;
      int cnt = 0;
      if (w < NWC) {
        const int r = w / NW, u = w % NW;
        int gx = x0 - 2 + u, gy = y - 1 + r, gs = 0;
        bool ok = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
        if (ok || ((gx >= 0 && gx < nx) || e.wrapx) && ((gy >= 0 && gy < ny) || e.wrapy)) {
          gx = ((gx % nx) + nx) % nx;
          gy = ((gy % ny) + ny) % ny;
          const int64_t cc = plane + (int64_t)gy * nx + gx;
          gs = e.start[cc];
          cnt = e.start[cc + 1] - gs;
        }
        wgs[w] = gs;
      }
      const int incl = warp_inclusive_scan(cnt);
      if (w < NWC) wst[w + 1] = tot + incl;
      tot += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) wst[0] = 0;
    __syncwarp();
    int scnt = 0;  // strips: NW <= 32 columns, one lane each
    if (tid < NW)
      for (int r = 0; r < 3; ++r) scnt += wst[r * NW + tid + 1] - wst[r * NW + tid];
    const int sincl = warp_inclusive_scan(scnt);
    if (tid < NW) sst[tid + 1] = sincl;
    if (tid == 0) sst[0] = 0;
  }
  __syncthreads();
  const int W = wst[NWC];
  const bool win_sm = W <= S::WCAP;

  auto find_cell = [&](int m) {  // last w with wst[w] <= m (binary lifting, NWC < 64)
    static_assert(NWC < 64, "window cells");
    int w = 0;
#pragma unroll
    for (int st = 32; st > 0; st >>= 1)
      if (w + st < NWC && wst[w + st] <= m) w += st;
    return w;
  };
  auto member_id = [&](int m, int w) { return __ldg(e.items + wgs[w] + (m - wst[w])); };
  if (win_sm) {
    for (int m = tid; m < W; m += BT) {
      const int w = find_cell(m);
      const int j = member_id(m, w);
      sid[m] = j;
      skey[m] = a.ids ? __ldg(a.ids + j) : j;
      sw[m] = (uint8_t)w;
    }
  }
  auto key_of = [&](int m) -> int {
    if (win_sm) return skey[m];
    const int j = member_id(m, find_cell(m));
    return a.ids ? __ldg(a.ids + j) : j;
  };

  // the CTA's runs: chunk span from the scanned run starts
  if (tid == 0) {
    s_ch0 = e.cstart[plane + (int64_t)y * nx + x0];
    s_nch = (int)(e.cstart[plane + (int64_t)y * nx + x1] - s_ch0);
  }
  for (int v = tid; v < nrun; v += BT) {
    const int64_t c = plane + (int64_t)y * nx + x0 + v;
    a.tri[c] = make_int2(e.cstart[c], e.cstart[c + 1]);
  }
  __syncthreads();
  const int64_t ch0 = s_ch0;
  const int nch = s_nch;
  const bool out_sm = nch <= S::OCAP;
  const __half nanv = hbits(0x7E00u);
  if (out_sm) {  // NaN coordinates, zero selectors, ~0 ids
    const uint32_t nan2 = 0x7E007E00u;
    for (int c = tid; c < nch; c += BT) {
      uint4* ck = reinterpret_cast<uint4*>(sch + (size_t)c * L::BYTES);
      ck[0] = make_uint4(nan2, nan2, nan2, nan2);
      ck[1] = make_uint4(nan2, nan2, 0u, 0u);
      reinterpret_cast<uint4*>(stag)[c] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
  } else {
    for (int v = tid; v < nrun; v += BT) {  // pad records of each run
      const int64_t c = plane + (int64_t)y * nx + x0 + v;
      const int64_t r0 = 4 * (int64_t)e.cstart[c], r1 = 4 * (int64_t)e.cstart[c + 1];
      int len = 0;
      for (int rr = 0; rr < 3; ++rr)
        for (int uu = v + 1; uu <= v + 3; ++uu) len += wst[rr * NW + uu + 1] - wst[rr * NW + uu];
      for (int64_t q = r0 + len; q < r1; ++q) {
#pragma unroll
        for (int k = 0; k < 3; ++k) store_el<3, FP16, MODE_RCLL>(a.qc, q, k, nanv);
        reinterpret_cast<unsigned*>(a.qtag)[q] = 0xFFFFFFFFu;
      }
      for (int64_t ch = r0 >> 2; ch < (r1 >> 2); ++ch)  // selectors are OR-ed in below
        *reinterpret_cast<uint2*>(static_cast<char*>(a.qc) + ch * L::BYTES + L::SELX) =
            make_uint2(0u, 0u);
    }
  }

  auto less_in = [&](int w, int key) {  // keys below `key` in window cell w (lower bound)
    const int lo = wst[w];
    int base = lo, len = wst[w + 1] - lo;
    if (win_sm && len < 32) {  // branch-free binary lifting
      int b = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (b + st <= len && skey[lo + b + st - 1] < key) b += st;
      return b;
    }
    if (win_sm) {
      while (len > 0) {
        const int half = len >> 1;
        const bool go = skey[base + half] < key;
        base = go ? base + half + 1 : base;
        len = go ? len - half - 1 : half;
      }
    } else {
      while (len > 0) {
        const int half = len >> 1;
        const bool go = key_of(base + half) < key;
        base = go ? base + half + 1 : base;
        len = go ? len - half - 1 : half;
      }
    }
    return base - lo;
  };

  // place member m (window cell w, merge key `key`, id j) in the runs centred at
  // window columns u-1 .. u+1; col[du] = keys below `key` in window column u-2+du
  auto place = [&](int m, int w, int key, int j, const int (&col)[5]) {
    const int r = w / NW, u = w - r * NW;
    __half c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = __double2half(__ldg(e.x[k] + j));
#pragma unroll
    for (int dv = -1; dv <= 1; ++dv) {  // runs centred at window column v = u + dv
      const int v = u + dv;
      if (v < 2 || v >= nrun + 2) continue;
      const int pos = col[1 + dv] + col[2 + dv] + col[3 + dv];
      const int64_t cidx = plane + (int64_t)y * nx + (x0 + v - 2);
      const int64_t rec = 4 * (int64_t)e.cstart[cidx] + pos;
      const uint32_t sx = dv == 1 ? 1u : (dv == -1 ? 2u : 0u);  // dcx = v - u
      const uint32_t sy = r == 0 ? 1u : (r == 2 ? 2u : 0u);     // dcy = 1 - r
      const uint32_t tag = a.ids ? (uint32_t)key : (uint32_t)j;
      const int l = (int)(rec & 3);
      if (out_sm) {
        const int lr = (int)(rec - 4 * ch0);
#pragma unroll
        for (int k = 0; k < 3; ++k) *rec_el<3, FP16, MODE_RCLL>(sch, lr >> 2, k, l) = c[k];
        unsigned char* ck = sch + (size_t)(lr >> 2) * L::BYTES;
        if (sx) atomicOr(reinterpret_cast<unsigned*>(ck + L::SELX), dc_nibble(l, sx));
        if (sy) atomicOr(reinterpret_cast<unsigned*>(ck + L::SELY), dc_nibble(l, sy));
        stag[lr] = tag;
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) store_el<3, FP16, MODE_RCLL>(a.qc, rec, k, c[k]);
        char* ck = static_cast<char*>(a.qc) + (rec >> 2) * L::BYTES;
        if (sx) atomicOr(reinterpret_cast<unsigned*>(ck + L::SELX), dc_nibble(l, sx));
        if (sy) atomicOr(reinterpret_cast<unsigned*>(ck + L::SELY), dc_nibble(l, sy));
        reinterpret_cast<uint32_t*>(a.qtag)[rec] = tag;
      }
      if (dv == 0 && r == 1) {  // own cell: pos_own and the self record
        a.selfpos[j] = (uint32_t)rec;
        reinterpret_cast<uint2*>(const_cast<void*>(a.pos_own))[j] =
            make_uint2(h2u(__halves2half2(c[0], c[1])), h2u(__halves2half2(c[2], hbits(0))));
      }
    }
    (void)m;
  };

  if (win_sm) {
    // strips: the three cells of each window column id-merged (rank = index in own
    // cell + keys below in the column's two other cells)
    for (int m = tid; m < W; m += BT) {
      const int w = sw[m];
      const int r = w / NW, u = w - r * NW;
      const int key = skey[m];
      int sr = m - wst[w];
#pragma unroll
      for (int rr = 0; rr < 3; ++rr)
        if (rr != r) sr += less_in(rr * NW + u, key);
      sstrip[sst[u] + sr] = key;
      srank[m] = (int16_t)sr;
    }
    __syncthreads();
    auto strip_less = [&](int u, int key) {  // keys below `key` in strip u
      const int lo = sst[u], len = sst[u + 1] - lo;
      int base = 0;
      if (len < 64) {
#pragma unroll
        for (int st = 32; st > 0; st >>= 1) {
          const int t = base + st;
          if (t <= len && sstrip[lo + t - 1] < key) base = t;
        }
      } else {
        int n = len;
        while (n > 0) {
          const int half = n >> 1;
          const bool go = sstrip[lo + base + half] < key;
          base = go ? base + half + 1 : base;
          n = go ? n - half - 1 : half;
        }
      }
      return base;
    };
    // records: members of window columns 1 .. nrun+2 (x0-1 .. x1)
    for (int m = tid; m < W; m += BT) {
      const int w = sw[m];
      const int u = w % NW;
      if (u < 1 || u > nrun + 2) continue;
      const int key = skey[m];
      int col[5];
#pragma unroll
      for (int du = 0; du < 5; ++du) {
        const int uu = u - 2 + du;
        col[du] = du == 2 ? (int)srank[m] : ((uu >= 0 && uu < NW) ? strip_less(uu, key) : 0);
      }
      place(m, w, key, sid[m], col);
    }
  } else {
    __syncthreads();
    for (int m = tid; m < W; m += BT) {
      const int w = find_cell(m);
      const int r = w / NW, u = w % NW;
      if (u < 1 || u > nrun + 2) continue;
      const int idx = m - wst[w];
      const int key = key_of(m);
      int col[5];
#pragma unroll
      for (int du = 0; du < 5; ++du) {
        const int uu = u - 2 + du;
        int s = 0;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
          s += (rr == r && du == 2) ? idx : ((uu >= 0 && uu < NW) ? less_in(rr * NW + uu, key) : 0);
        col[du] = s;
      }
      place(m, w, key, member_id(m, w), col);
    }
  }
  __syncthreads();
  if (out_sm) {
    const uint4* src = reinterpret_cast<const uint4*>(sch);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(a.qc) + ch0 * L::BYTES);
    for (int q = tid; q < nch * (L::BYTES / 16); q += BT) dst[q] = src[q];
    const uint4* ts = reinterpret_cast<const uint4*>(stag);
    uint4* td = reinterpret_cast<uint4*>(a.qtag) + ch0;
    for (int q = tid; q < nch; q += BT) td[q] = ts[q];
  }
}

template <int D, int P, int M>
static int encode_cells(int64_t C, int nx, int wrapx, const PrecConsts& pc,
                        const double* const x[3], const int32_t* items, const int32_t* start,
                        const SweepArgs& a, cudaStream_t st) {
  using E = EncShape<D, P>;
  EncArgs e;
  e.nx = nx;
  e.nxb = (nx + E::XB - 1) / E::XB;
  e.wrapx = wrapx;
  e.nrows = C / nx;
  e.start = start;
  e.items = items;
  for (int k = 0; k < 3; ++k) e.x[k] = x[k];
  e.pc = pc;
  constexpr size_t smem = enc_smem_bytes<D, P, M>();
  cudaFuncSetAttribute(k_encode_rows<D, P, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  k_encode_rows<D, P, M><<<(unsigned)(e.nrows * e.nxb), E::BT, smem, st>>>(e, a);
  return 1;
}

template <int D, int P>
static int encode_t(int mode, int n, int64_t C, int nx, int wrapx, const PrecConsts& pc,
                    const double* const x[3], const int32_t* items, const int32_t* start,
                    const SweepArgs& a, cudaStream_t st) {
  if (mode == MODE_ALL) {
    k_pack_own<D, P><<<(n + 255) / 256, 256, 0, st>>>(n, x[0], x[1], x[2],
                                                       const_cast<void*>(a.pos_own));
    const int64_t nch = (n + 3) / 4;
    k_encode_all<D, P><<<(unsigned)((nch + 127) / 128), 128, 0, st>>>(n, a.pos_own, a);
    return 2;
  }
  if (C == 0) return 0;
  if constexpr (D == 3 && P == FP16) {
    if (mode == MODE_RCLL) {  // xy-plane runs: lengths -> scan -> records
      const int ny = a.g.counts[1];
      k_xy_runlen<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(C, nx, ny, wrapx, a.g.wrap[1], start,
                                                                 a.xy_nch);
      const int64_t nt = scan_tiles(C);
      cudaMemsetAsync(a.xy_tiles, 0, sizeof(unsigned long long) * (nt + 2), st);
      launch_scan_counts(a.xy_nch, a.xy_cstart, C, a.xy_tiles,
                         reinterpret_cast<int*>(a.xy_tiles + nt + 1), st);
      EncArgs e;
      e.nx = nx;
      e.nxb = (nx + XYShape::XB - 1) / XYShape::XB;
      e.wrapx = wrapx;
      e.ny = ny;
      e.wrapy = a.g.wrap[1];
      e.nrows = C / nx;
      e.start = start;
      e.items = items;
      for (int k = 0; k < 3; ++k) e.x[k] = x[k];
      e.pc = pc;
      e.cstart = a.xy_cstart;
      constexpr size_t smem = xy_smem_bytes();
      cudaFuncSetAttribute(k_encode_xy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_encode_xy<<<(unsigned)(e.nrows * e.nxb), XYShape::BT, smem, st>>>(e, a);
      return 3;
    }
  }
  if (mode == MODE_RCLL) return encode_cells<D, P, MODE_RCLL>(C, nx, wrapx, pc, x, items, start, a, st);
  return encode_cells<D, P, MODE_CLL>(C, nx, wrapx, pc, x, items, start, a, st);
}

// Returns the number of kernel launches issued (n > 0).
int launch_encode(int dim, int prec, int mode, int n, int64_t C, int nx, int wrapx,
                  const PrecConsts& pc, const double* const x[3], const int32_t* items,
                  const int32_t* start, const SweepArgs& a, cudaStream_t st) {
#define ENC(D, P) \
  if (dim == D && prec == P) return encode_t<D, P>(mode, n, C, nx, wrapx, pc, x, items, start, a, st);
  ENC(1, FP16) ENC(2, FP16) ENC(3, FP16) ENC(1, FP32) ENC(2, FP32) ENC(3, FP32)
  ENC(1, FP64) ENC(2, FP64) ENC(3, FP64)
#undef ENC
  return 0;
}

template <int D, int P, int M>
static int64_t sweep_t(const SweepArgs& a, cudaStream_t st) {
  using S = Shape<D>;
  if constexpr (P == FP16 && M == MODE_RCLL && D == 3) {
    // 3-D: tests and ordered emission in separate kernels (R16Two)
    using R = R16Two<D>;
    launch_pdl(k_r16_test<D>, (unsigned)((a.n + R::TB - 1) / R::TB), R::TB, st, a);
    if (a.nrows > R::LARGE_ROWS) {
      const int64_t nb = (a.nrows + R::BT_LARGE - 1) / R::BT_LARGE;
      launch_pdl(k_r16_emit<D, R::BT_LARGE, R::BT_LARGE * R::PCAP_ROW>, (unsigned)nb,
                 R::BT_LARGE, st, a);
      return nb;
    }
    const int64_t nb = (a.nrows + R::BT - 1) / R::BT;
    launch_pdl(k_r16_emit<D, R::BT, R::BT * R::PCAP_ROW>, (unsigned)nb, R::BT, st, a);
    return nb;
  } else if constexpr (P == FP16 && M == MODE_RCLL && D == 2) {
    // 2-D: one fused kernel (the look-back wait hides the emission)
    using R = R16Shape<D>;
    const int64_t nb = (a.nrows + R::BT - 1) / R::BT;
    launch_pdl(k_rcll16<D, R::BT, R::PCAP, R::WMAX>, (unsigned)nb, R::BT, st, a);
    return SPHX_TICKET ? nb : 0;  // tiles from blockIdx take no tickets
  } else {
    const int64_t nb = (a.nrows + S::BT - 1) / S::BT;
    k_sweep<D, P, M, S::BT, S::PCAP, S::WMAX><<<(unsigned)nb, S::BT, 0, st>>>(a);
    return nb;
  }
}

#define SW(FN, D, P, M) \
  if (dim == D && prec == P && mode == M) return FN<D, P, M>(a, st);
#define SWP(FN, D, M) SW(FN, D, FP16, M) SW(FN, D, FP32, M) SW(FN, D, FP64, M)
#define SWA(FN)                                                     \
  SWP(FN, 1, MODE_RCLL) SWP(FN, 2, MODE_RCLL) SWP(FN, 3, MODE_RCLL) \
  SWP(FN, 1, MODE_CLL) SWP(FN, 2, MODE_CLL) SWP(FN, 3, MODE_CLL)    \
  SWP(FN, 1, MODE_ALL) SWP(FN, 2, MODE_ALL) SWP(FN, 3, MODE_ALL)

// The single-pass sweep: offsets[0..nrows] and the rows. Returns the tickets used.
int64_t launch_sweep(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) {
  SWA(sweep_t)
  return 0;
}

#undef SWA
#undef SWP
#undef SW

}  // namespace sphx_dev
