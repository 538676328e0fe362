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
// Candidate layout ("x-triples" in 4-record chunks). For every cell c the encode
// step merges, by particle id, the members of the x-neighbour cells (cx-1, cx,
// cx+1) -- wrapped on a periodic x axis -- into one run of records, padded with
// NaN sentinels to whole chunks of 4. Chunks are stored structure-of-arrays: one
// quad of coordinates per axis (binary16 quad = 8 B), one quad of x offsets dc
// (RCLL; dc = cx_i - cx_j in {-1,0,1}) and one quad of ids. CLL records carry the
// periodic x shift already applied (round_to(prec, xj + shift), nnps.cpp:116).
// A particle's candidates are the 3 (2-D) / 9 (3-D) runs of its (dy, dz) rows.
//
// Passes:  count (distance tests, one per candidate; hit nibbles + row lengths)
//          -> tile sums -> scan -> fill (hit ids from the nibbles into sorted,
//          warp-packed rows in shared memory, coalesced stores to HBM).
// Count runs in cell (CSR) order so the lanes of one cell share every record;
// fill runs in particle order so the 32 rows of a warp are one contiguous run.
//
// Bit-exactness: every step is an explicit round-to-nearest op in the
// precision (no contraction; the reference is built without -march). The x term
// t + cc (cc = round_to(prec, dc*hc), dc*hc exact) is one fused dc*hc + t -- a
// single rounding of the same exact sum. FP16 uses native binary16 ALU ops, which
// keep subnormals, and sqrt(acc) < cutoff is the exact monotone test acc < thr.

#include <climits>

#include "common.cuh"

namespace sphx_dev {

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

// 4 lane masks of a pair of HSET2 results -> 4-bit hit nibble (record order)
__device__ __forceinline__ unsigned nibble(unsigned mk01, unsigned mk23) {
  const unsigned w = __byte_perm(mk01, mk23, 0x6420) & 0x08040201u;
  return (w * 0x01010101u) >> 24;
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
};

template <int D> struct Tester<D, FP32, MODE_RCLL> : TesterRcllScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_RCLL> : TesterRcllScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_CLL> : TesterAbsScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_CLL> : TesterAbsScalar<D, FP64> {};
template <int D> struct Tester<D, FP32, MODE_ALL> : TesterAbsScalar<D, FP32> {};
template <int D> struct Tester<D, FP64, MODE_ALL> : TesterAbsScalar<D, FP64> {};

template <int D, int P, int MODE>
__device__ __forceinline__ void load_chunk(const SweepArgs& a, int64_t ch, Chunk<D, P>& c) {
  using Q = typename Prec<P>::Quad;
#pragma unroll
  for (int k = 0; k < D; ++k) c.x[k] = ldg<Q>(a.qx[k], ch);
  if constexpr (MODE == MODE_RCLL) c.dc = ldg<Q>(a.qdc, ch);
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

// Distance tests of particle i against every candidate chunk. fn(m, ch) gets the
// hit nibble of chunk ch (bit u: record 4ch+u is a neighbour j != i). The own
// record (id i) sits in the own-cell run at selfpos[i] and is masked out there.
template <int D, int P, int MODE, class ChunkFn>
__device__ __forceinline__ void scan_particle(const SweepArgs& a, int i, ChunkFn&& fn) {
  using Tst = Tester<D, P, MODE>;
  Tst tst;
  tst.init(a, i);
  const int64_t self = MODE == MODE_ALL ? (int64_t)i : (int64_t)__ldg(a.selfpos + i);
  visit_rows<D, MODE>(a, i, [&](int dy, int dz, int wy, int wz, int cb, int ce) {
    const typename Tst::Row row = tst.row(a, dy, dz, wy, wz);
    const bool own = dy == 0 && dz == 0;
#pragma unroll 4
    for (int ch = cb; ch < ce; ++ch) {
      Chunk<D, P> c;
      load_chunk<D, P, MODE>(a, ch, c);
      unsigned m = tst.test4(row, c);
      if (own) {
        const int64_t d = self - 4 * (int64_t)ch;
        if (d >= 0 && d < 4) m &= ~(1u << d);
      }
      if (MODE == MODE_ALL) {  // the single run ends exactly at n
        const int64_t left = a.n - 4 * (int64_t)ch;
        if (left < 4) m &= (1u << left) - 1u;
      }
      fn(m, ch);
    }
  });
}

template <int D>
struct MaskWords {  // 32-bit words of 4-bit hit nibbles per particle
  static constexpr int W = D == 3 ? 16 : (D == 2 ? 4 : 2);
};
constexpr unsigned kOverflow = 0x80000000u;  // counts[i] flag: nibbles did not fit

// Pass 1 (cell order): row lengths k_i and the hit nibbles of every chunk.
template <int D, int P, int MODE, int BT>
__global__ void __launch_bounds__(BT) k_count(SweepArgs a) {
  constexpr int W = MaskWords<D>::W;
  const int s = blockIdx.x * BT + threadIdx.x;
  if (s >= a.n) return;
  const int i = a.order ? __ldg(a.order + s) : s;
  if (i < a.row0 || i >= a.row0 + a.nrows) return;  // not a requested row (or malformed)
  int k = 0, bits = 0, words = 0;
  unsigned acc = 0;
  scan_particle<D, P, MODE>(a, i, [&](unsigned m, int64_t) {
    k += __popc(m);
    acc |= m << bits;
    bits += 4;
    if (bits == 32) {
      if (words < W) a.masks[(int64_t)words * a.n + s] = acc;
      ++words;
      acc = 0;
      bits = 0;
    }
  });
  if (bits) {
    if (words < W) a.masks[(int64_t)words * a.n + s] = acc;
    ++words;
  }
  a.counts[i] = (int)((unsigned)k | (words > W ? kOverflow : 0u));
}

// Pass 2a: row-length sums of tiles of `tile` consecutive particles.
__global__ void __launch_bounds__(256) k_tile_sums(const int32_t* __restrict__ counts, int n, int tile,
                                                   long long* __restrict__ sums) {
  __shared__ long long s_w[8];
  const int64_t base = (int64_t)blockIdx.x * tile;
  long long v = 0;
  for (int q = threadIdx.x; q < tile; q += 256) {
    const int64_t i = base + q;
    if (i < n) v += (int)((unsigned)__ldg(counts + i) & ~kOverflow);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_w[w];
    sums[blockIdx.x] = t;
  }
}

// Pass 2b: exclusive scan of the tile sums in place (one block); offsets[n] = total.
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

// ------------------------------------------------------------------------------
// Row assembly (pass 3)
// ------------------------------------------------------------------------------
// Sorted insertion of a chunk's hits (ids ascending within the chunk, since runs
// are id-sorted). Fast path: the chunk's first hit is >= the row's last id, so
// the hits are appended as they are.
template <class Row>
__device__ __forceinline__ void emit4(Row& row, int& k, int& last, unsigned m, const uint4& tq) {
  const int j[4] = {(int)tq.x, (int)tq.y, (int)tq.z, (int)tq.w};
  const int first = (m & 1u) ? j[0] : ((m & 2u) ? j[1] : ((m & 4u) ? j[2] : j[3]));
  if (first >= last) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (m >> u & 1u) {
        row[k] = j[u];
        ++k;
        last = j[u];
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (m >> u & 1u) {
        const int v = j[u];
        int q = k;
        int w;
        while (q > 0 && (w = row[q - 1]) > v) {
          row[q] = w;
          --q;
        }
        row[q] = v;
        ++k;
        last = max(last, v);
      }
    }
  }
}

// Replays particle i's hits into row[0..k): from its nibbles (masks at slot s),
// or by re-testing when they did not fit.
template <int D, int P, int MODE, class Row>
__device__ __forceinline__ void build_row(const SweepArgs& a, int i, int64_t s, bool retest,
                                          Row& row) {
  int k = 0, last = INT_MIN;
  const uint4* qtag = reinterpret_cast<const uint4*>(a.qtag);
  if (!retest) {
    constexpr int W = MaskWords<D>::W;
    unsigned acc = 0;
    int bits = 32, words = 0;
    auto next = [&]() {
      if (bits == 32) {
        acc = words < W ? __ldg(a.masks + (int64_t)words * a.n + s) : 0u;
        ++words;
        bits = 0;
      }
      const unsigned m = (acc >> bits) & 0xFu;
      bits += 4;
      return m;
    };
    visit_rows<D, MODE>(a, i, [&](int, int, int, int, int cb, int ce) {
      // groups of 4 chunks: the id quads of all hit chunks are loaded together
      for (int ch = cb; ch < ce; ch += 4) {
        unsigned m[4];
        uint4 tq[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          m[g] = ch + g < ce ? next() : 0u;
          if (m[g]) tq[g] = __ldg(qtag + ch + g);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
          if (m[g]) emit4(row, k, last, m[g], tq[g]);
      }
    });
  } else {
    scan_particle<D, P, MODE>(a, i, [&](unsigned m, int64_t ch) {
      if (m) emit4(row, k, last, m, __ldg(qtag + ch));
    });
  }
}

// Pass 3 (particle order): offsets[i] and the rows. A warp's 32 rows are one
// contiguous run of the table: they are built directly at their packed places
// in shared memory and streamed out with coalesced stores. Rows longer than CAP
// are built straight in global memory.
template <int D, int P, int MODE, int BT, int CAP>
__global__ void __launch_bounds__(BT) k_fill(SweepArgs a) {
  static_assert(BT % 32 == 0, "shape");
  __shared__ int32_t S[BT * CAP];
  __shared__ int s_w[BT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = blockIdx.x * BT + tid;  // row index (particle row0 + r)
  const bool valid = r < a.nrows;
  const int i = a.row0 + r;
  const unsigned kw = valid ? (unsigned)__ldg(a.counts + i) : 0u;
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
  const long long grow = bbase + wbase + incl - k;
  if (valid) a.offsets[r] = grow;
  if (bbase + btot > a.capacity) return;  // device API: the caller grows the table

  const int64_t s = MODE == MODE_ALL ? i : (valid ? (int64_t)__ldg(a.rank + i) : 0);
  const unsigned over = __ballot_sync(0xffffffffu, k > CAP);
  int32_t* wS = S + warp * 32 * CAP;
  int32_t* __restrict__ out = a.items + bbase + wbase;
  if (!over) {
    const int wrel = incl - k;
    if (k > 0) {
      int32_t* row = wS + wrel;
      build_row<D, P, MODE>(a, i, s, retest, row);
    }
    __syncwarp();
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    for (int e = lane; e < wtot; e += 32) out[e] = wS[e];  // coalesced
    return;
  }
  // warp with an over-long row: short rows via per-thread slots in shared memory
  // (one warp-wide store per row), long rows straight into global memory
  const int wrel = incl - k;
  if (k > 0) {
    if (k <= CAP) {
      int32_t* row = wS + lane * CAP;
      build_row<D, P, MODE>(a, i, s, retest, row);
    } else {
      int32_t* row = out + wrel;
      build_row<D, P, MODE>(a, i, s, retest, row);
    }
  }
  __syncwarp();
  for (int w = 0; w < 32; ++w) {
    const int len = __shfl_sync(0xffffffffu, k, w);
    const int ro = __shfl_sync(0xffffffffu, wrel, w);
    if (len > CAP) continue;
    for (int q = lane; q < len; q += 32) out[ro + q] = wS[w * CAP + q];
  }
}

// ------------------------------------------------------------------------------
// Encode
// ------------------------------------------------------------------------------
// Own coordinates (particle order); for the cell modes also rank[items[t]] = t
// and the members' packed coordinates in CSR order. RCLL: src = RelCoords::rel
// (nnps.cpp:304-315); CLL/all: src = positions (round_coords nnps.cpp:75-89).
template <int D, int P, int MODE>
__global__ void k_encode_own(int n, const double* __restrict__ x0, const double* __restrict__ x1,
                             const double* __restrict__ x2, const int32_t* __restrict__ items,
                             void* __restrict__ pos_csr, int32_t* __restrict__ cell_slot,
                             SweepArgs a) {
  using C = typename Coord<D, P>::T;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double v[3] = {x0[t], D > 1 ? x1[t] : 0.0, D > 2 ? x2[t] : 0.0};
  reinterpret_cast<C*>(const_cast<void*>(a.pos_own))[t] = pack<D, P>(v);
  if constexpr (MODE != MODE_ALL) {
    int j = items[t];
    if (j < 0 || j >= n) j = 0;  // malformed membership: stay memory-safe
    a.rank[j] = t;
    const double w[3] = {x0[j], D > 1 ? x1[j] : 0.0, D > 2 ? x2[j] : 0.0};
    reinterpret_cast<C*>(pos_csr)[t] = pack<D, P>(w);
    // the cell holding slot t: the member's own cell (RelCoords::cell for RCLL,
    // CellGrid::cell_of for CLL), clamped to stay memory-safe
    int c;
    if constexpr (MODE == MODE_RCLL) {
      int ck[3] = {0, 0, 0};
#pragma unroll
      for (int k = 0; k < D; ++k) ck[k] = min(max(a.cellk[k][j], 0), a.g.counts[k] - 1);
      c = (ck[2] * a.g.counts[1] + ck[1]) * a.g.counts[0] + ck[0];
    } else {
      c = a.cell_of[j];
    }
    cell_slot[t] = c;
  }
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

// x-neighbour list l (0: cx-1, 1: cx, 2: cx+1) of the run centred at tx: its cell
// range in the row, and the periodic wrap direction (-1: seen one period below).
__device__ __forceinline__ int list_range(const int32_t* st, int tx, int l, int nx, int wrapx,
                                          int& lo, int& hi) {
  int x = tx - 1 + l, w = 0;
  if (x < 0) {
    if (!wrapx) return lo = hi = 0, 0;
    x += nx;
    w = -1;
  } else if (x >= nx) {
    if (!wrapx) return lo = hi = 0, 0;
    x -= nx;
    w = 1;
  }
  lo = st[x];
  hi = st[x + 1];
  return w;
}

template <int P>
__device__ __forceinline__ void store_el(void* q, int64_t r, typename Prec<P>::T v) {
  reinterpret_cast<typename Prec<P>::T*>(q)[r] = v;
}

// One thread per cell c: the run's chunk range and the sentinel records (NaN
// coordinates, id ~0) that pad it to whole chunks.
template <int D, int P, int MODE>
__global__ void k_encode_runs(int64_t C, int nx, int wrapx, const int32_t* __restrict__ start,
                              SweepArgs a) {
  using T = typename Prec<P>::T;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int cx = (int)(c % nx);
  const int32_t* st = start + (c - cx);
  int len = 0;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    int lo, hi;
    list_range(st, cx, l, nx, wrapx, lo, hi);
    len += hi - lo;
  }
  const int64_t slot = run_record_slot(st, cx, nx, wrapx, c);
  const int nch = (len + 3) >> 2;
  a.tri[c] = make_int2((int)(slot >> 2), (int)((slot >> 2) + nch));
  T nan;
  if constexpr (P == FP16) nan = hbits(0x7E00u); else nan = T(NAN);
  for (int q = len; q < 4 * nch; ++q) {
#pragma unroll
    for (int k = 0; k < D; ++k) store_el<P>(a.qx[k], slot + q, nan);
    if constexpr (MODE == MODE_RCLL) store_el<P>(a.qdc, slot + q, T(0.0f));
    reinterpret_cast<unsigned*>(a.qtag)[slot + q] = 0xFFFFFFFFu;
  }
}

// One thread per CSR slot s (particle j = items[s] in cell c): its record in
// each of the three runs that contain cell c (runs centred at cx+1, cx, cx-1,
// where c is list 0, 1, 2). The record's place in a run is its index in c plus
// the number of smaller ids in the run's two other cells (cells hold ascending
// ids), i.e. the position in the id-merge of the three cells. With slab ids the
// merge key is the output id (each cell is one id-ascending class there).
template <int D, int P, int MODE>
__global__ void k_encode_members(int n, int nx, int wrapx, PrecConsts pc,
                                 const int32_t* __restrict__ start,
                                 const int32_t* __restrict__ items,
                                 const int32_t* __restrict__ cell_of_slot,
                                 const void* __restrict__ pos_csr, SweepArgs a) {
  using T = typename Prec<P>::T;
  using CT = typename Coord<D, P>::T;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int j = __ldg(items + s);
  const int c = __ldg(cell_of_slot + s);
  const int cx = c % nx;
  const int32_t* st = start + (c - cx);
  const int idx = s - __ldg(st + cx);
  const CT cj = ldg<CT>(pos_csr, s);
#pragma unroll
  for (int L = 0; L < 3; ++L) {  // c is list L of the run centred at tx
    int tx = cx + 1 - L;
    if (tx < 0 || tx >= nx) {
      if (!wrapx) continue;
      tx = tx < 0 ? tx + nx : tx - nx;
    }
    int pos = idx, w = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      int lo, hi;
      const int wl = list_range(st, tx, l, nx, wrapx, lo, hi);
      if (l == L) {
        w = wl;
        continue;
      }
      int cnt = 0;
      if (a.ids) {  // slab: merge by output (global) id -- in 1-D a run can mix
        const int gj = __ldg(a.ids + j);  // owned and halo cells
        for (int q = lo; q < hi; ++q) cnt += __ldg(a.ids + __ldg(items + q)) < gj;
      } else {
        for (int q = lo; q < hi; ++q) cnt += __ldg(items + q) < j;
      }
      pos += cnt;
    }
    const int64_t r = run_record_slot(st, tx, nx, wrapx, (c - cx) + tx) + pos;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      T v = axis_of<D, P>(cj, k);
      if (MODE == MODE_CLL && k == 0 && w != 0) {  // round_to(prec, xj + shift), nnps.cpp:116
        T sh;
        if constexpr (P == FP16) sh = hbits(pc.h_sh[0]);
        else if constexpr (P == FP32) sh = pc.f_sh[0];
        else sh = pc.d_sh[0];
        if constexpr (P == FP16) v = __hadd_rn(v, w > 0 ? sh : __hneg(sh));
        else v = f_add(v, w > 0 ? sh : -sh);
      }
      store_el<P>(a.qx[k], r, v);
    }
    if constexpr (MODE == MODE_RCLL) store_el<P>(a.qdc, r, (T)(float)(1 - L));  // dc_x
    // output id: the particle index, or its global id for a multi-GPU slab
    reinterpret_cast<unsigned*>(a.qtag)[r] = a.ids ? (unsigned)__ldg(a.ids + j) : (unsigned)j;
    if (L == 1) a.selfpos[j] = (int)r;
  }
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
  for (int k = 0; k < D; ++k) reinterpret_cast<Q*>(a.qx[k])[ch] = qx[k];
  reinterpret_cast<uint4*>(a.qtag)[ch] = qt;
}

template <int D>
struct Shape {
  static constexpr int CBT = 128;               // count: threads per block
  static constexpr int BT = D == 3 ? 64 : 128;  // fill: rows per block (= scan tile)
  static constexpr int CAP = D == 3 ? 96 : 32;  // fill: shared-memory slots per row
};

// ------------------------------------------------------------------------------
// Host-side launchers (called from capi.cu)
// ------------------------------------------------------------------------------
int fill_tile(int dim) { return dim == 3 ? Shape<3>::BT : Shape<2>::BT; }
int mask_words(int dim) {
  return dim == 3 ? MaskWords<3>::W : (dim == 2 ? MaskWords<2>::W : MaskWords<1>::W);
}
size_t coord_bytes(int dim, int prec) {
  if (prec == FP16) return dim == 3 ? 8 : 4;
  if (prec == FP32) return dim == 1 ? 4 : (dim == 2 ? 8 : 16);
  return dim == 1 ? 8 : (dim == 2 ? 16 : 32);
}
size_t quad_bytes(int prec) { return prec == FP16 ? 8 : (prec == FP32 ? 16 : 32); }
// chunks the candidate arrays need
int64_t chunk_capacity(int mode, int64_t n, int64_t C) {
  return mode == MODE_ALL ? (n + 3) / 4 + 1 : (3 * n + 6 * C) / 4 + 2;
}

template <int D, int P, int M>
static void encode_cells(int n, int64_t C, int nx, int wrapx, const PrecConsts& pc,
                         const double* const x[3], const int32_t* items, const int32_t* start,
                         void* pos_csr, int32_t* cell_slot, const SweepArgs& a, cudaStream_t st) {
  k_encode_own<D, P, M><<<(n + 255) / 256, 256, 0, st>>>(n, x[0], x[1], x[2], items, pos_csr,
                                                         cell_slot, a);
  k_encode_runs<D, P, M><<<(unsigned)((C + 255) / 256), 256, 0, st>>>(C, nx, wrapx, start, a);
  k_encode_members<D, P, M><<<(n + 255) / 256, 256, 0, st>>>(n, nx, wrapx, pc, start, items,
                                                             cell_slot, pos_csr, a);
}

template <int D, int P>
static int encode_t(int mode, int n, int64_t C, int nx, int wrapx, const PrecConsts& pc,
                    const double* const x[3], const int32_t* items, const int32_t* start,
                    void* pos_csr, int32_t* cell_slot, const SweepArgs& a, cudaStream_t st) {
  if (mode == MODE_ALL) {
    k_encode_own<D, P, MODE_ALL><<<(n + 255) / 256, 256, 0, st>>>(n, x[0], x[1], x[2], nullptr,
                                                                   nullptr, nullptr, a);
    const int64_t nch = (n + 3) / 4;
    k_encode_all<D, P><<<(unsigned)((nch + 127) / 128), 128, 0, st>>>(n, a.pos_own, a);
    return 2;
  }
  if (C == 0) return 0;
  if (mode == MODE_RCLL)
    encode_cells<D, P, MODE_RCLL>(n, C, nx, wrapx, pc, x, items, start, pos_csr, cell_slot, a, st);
  else
    encode_cells<D, P, MODE_CLL>(n, C, nx, wrapx, pc, x, items, start, pos_csr, cell_slot, a, st);
  return 3;
}

// Returns the number of kernel launches issued (n > 0).
int launch_encode(int dim, int prec, int mode, int n, int64_t C, int nx, int wrapx,
                  const PrecConsts& pc, const double* const x[3], const int32_t* items,
                  const int32_t* start, void* pos_csr, int32_t* cell_slot, const SweepArgs& a,
                  cudaStream_t st) {
#define ENC(D, P) \
  if (dim == D && prec == P) return encode_t<D, P>(mode, n, C, nx, wrapx, pc, x, items, start, pos_csr, cell_slot, a, st);
  ENC(1, FP16) ENC(2, FP16) ENC(3, FP16) ENC(1, FP32) ENC(2, FP32) ENC(3, FP32)
  ENC(1, FP64) ENC(2, FP64) ENC(3, FP64)
#undef ENC
  return 0;
}

template <int D, int P, int M>
static void count_t(const SweepArgs& a, cudaStream_t st) {
  constexpr int CBT = Shape<D>::CBT;
  k_count<D, P, M, CBT><<<(a.n + CBT - 1) / CBT, CBT, 0, st>>>(a);
  const int tile = Shape<D>::BT;
  const int nt = (a.nrows + tile - 1) / tile;
  k_tile_sums<<<nt, 256, 0, st>>>(a.counts + a.row0, a.nrows, tile, a.block_sum);
  k_scan_blocks<<<1, 1024, 0, st>>>(a.block_sum, nt, a.offsets, a.nrows);
}

template <int D, int P, int M>
static void fill_t(const SweepArgs& a, cudaStream_t st) {
  constexpr int BT = Shape<D>::BT;
  k_fill<D, P, M, BT, Shape<D>::CAP><<<(a.nrows + BT - 1) / BT, BT, 0, st>>>(a);
}

#define SW(FN, D, P, M) \
  if (dim == D && prec == P && mode == M) return FN<D, P, M>(a, st);
#define SWP(FN, D, M) SW(FN, D, FP16, M) SW(FN, D, FP32, M) SW(FN, D, FP64, M)
#define SWA(FN)                                                     \
  SWP(FN, 1, MODE_RCLL) SWP(FN, 2, MODE_RCLL) SWP(FN, 3, MODE_RCLL) \
  SWP(FN, 1, MODE_CLL) SWP(FN, 2, MODE_CLL) SWP(FN, 3, MODE_CLL)    \
  SWP(FN, 1, MODE_ALL) SWP(FN, 2, MODE_ALL) SWP(FN, 3, MODE_ALL)

// Pass 1 + 2: counts and hit nibbles, tile sums, scanned tile bases, offsets[n].
void launch_count(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) { SWA(count_t) }
// Pass 3: offsets[0..n) and the rows.
void launch_fill(int dim, int prec, int mode, const SweepArgs& a, cudaStream_t st) { SWA(fill_t) }

#undef SWA
#undef SWP
#undef SW

}  // namespace sphx_dev
