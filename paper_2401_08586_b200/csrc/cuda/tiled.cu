// Cell-tiled FP16 RCLL for 2-D (the BASELINE metric path): rcll(rel, grid, fp16)
// of nnps.cpp:283-416 with the 2-D batch kernel detail::range_f16_rel_2d
// (nnps_batch.cpp:203-261) and build_table's sorted rows (nnps.cpp:26-66).
//
// The reference packs the rel coordinates into CSR order once per call
// (nnps.cpp:304-315) and streams, for every particle, the contiguous CSR range
// of each of its 9 neighbour cells. Here a CTA owns a *tile*: `tw` consecutive
// cells of one cell row. Every target of the tile (a member of one of its
// cells) draws its candidates from the same three cell-row segments -- rows
// cy-1, cy, cy+1, cells x0-1 .. x0+w -- which are contiguous CSR ranges
// (linear cell = cx + nx*cy, x fastest, cell_grid.hpp:74-78) plus at most one
// wrapped halo cell per side. The CTA stages them in shared memory once,
// converting FP64 rel to binary16 on the way (round16, nnps.cpp:306), as
// id-merged x-triple runs (cells c-1, c, c+1 of a row), so a target's hits come
// out in ascending id order run by run (build_table sorts rows, nnps.cpp:54).
//
// Four kernels, chained with programmatic dependent launch:
//   k_t2_rank   per cell row, each record's place in the three x-triples it
//               belongs to (its index + the members below it in the two other
//               cells, from merges of neighbouring cells), 3 bytes per record;
//   k_t2_count  stage + scatter by rank into the runs; per target its 3 runs
//               (contiguous) are tested two candidates per binary16x2 op; hit
//               bits over run positions -> mw/mx (by CSR position of the
//               target), the row length -> cnt[i] (particle order);
//   k_t2_scan   offsets = exclusive scan of cnt (int64, decoupled look-back);
//   k_t2_fill   stage ids into the runs by rank, hit bits -> ids -> the sorted
//               row in shared memory (runs of different rows merged where they
//               interleave), rows streamed to items[offsets[i]...] coalesced.
// Tiles whose stage exceeds shared memory, or whose runs exceed 255 records,
// are split (sub-tiles down to one cell). Targets whose RelCoords cell
// disagrees with their CSR cell (a stale grid), whose one-cell sub-tile still
// overflows, or whose 3 runs hold more than 128 records take a per-row
// global-memory path with the same arithmetic.
//
// Exactness (per candidate, nnps.cpp:332-346): s = r16(ri - rj); t = r16(s*hh);
// x: d = r16(t + dc*hc16) as one HFMA2 (dc in {-1,0,1}, dc*hc16 exact); y:
// d = r16(t + cc) (cc = round16(-dy*hc) in {+hc16, 0, -hc16}; +0 for the centre
// row only turns -0 into +0, which squares the same); acc = r16(r16(dx^2) +
// r16(dy^2)); hit iff acc < thr (the exact threshold of r16(sqrt(acc)) <
// cutoff16, capi.cu thr16).

#include <utility>

#include "common.cuh"

namespace sphx_dev {

namespace {

#ifndef SPHX_T2BT
#define SPHX_T2BT 128
#endif
constexpr int kBT = SPHX_T2BT;           // threads per CTA (rank, count, fill)
constexpr int kTWMax = kBT / 2;          // widest tile (cells)
constexpr int kNQ = 3 * (kTWMax + 2);    // staged cells per tile
constexpr int kNR = 3 * kTWMax;          // runs per tile
constexpr int kSCap = 6 * kBT;           // staged records per (sub-)tile
constexpr int kRCap = 18 * kBT;          // run records per (sub-)tile
constexpr int kPCap = 24 * kBT;          // fill: row buffer entries per chunk of kBT targets
constexpr int kScanBT = 512, kScanIPT = 16;  // scan: threads, counts per thread

__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<const unsigned*>(&h); }
__device__ __forceinline__ __half2 u2h(unsigned u) { return *reinterpret_cast<const __half2*>(&u); }
__device__ __forceinline__ __half2 hb2(unsigned short b) {
  return u2h((unsigned)b | ((unsigned)b << 16));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ int warp_incl(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// ---------------------------------------------------------------------------
// Tile geometry and the per-cell tables
// ---------------------------------------------------------------------------
// Staged cells q = r*(w+2) + u: row r (dy = r - R0), cell x = x0-1+u (u =
// 0..w+1), wrapped on a periodic x axis or empty outside a walled one; rows
// outside a walled y axis are empty. NROW = 3 (count, fill: rows cy-1..cy+1,
// R0 = 1) or 1 (rank: row cy). Per cell: SB[q] = stage offset (SB[nq] = stage
// size), CSRB[q] = CSR position of stage record 0 of the cell's range (csr =
// CSRB[q] + e), SLOT[q] = run base of the record's place in the runs centred at
// u-1, u, u+1 (-1 outside the sub-tile) and (r << 8 | u). CELLQ[e] = the cell
// of stage record e. Runs p = 3*(c-1) + r (c = 1..w) hold the id-merged members
// of cells c-1, c, c+1 of row r, padded to an even length, so the three runs
// of a target in cell c are contiguous; RB[p] = offset of run p.
struct Geo {
  int cy, x0, w, nq;
  int rowc[3];      // linear index of cell (0, y) of row r, -1 if the row is absent
  int kt, t0, T;    // first target's CSR position and stage offset; targets
  int total, rtotal;
  int over;         // the stage or the runs exceed shared memory / rank bytes
};

struct Tables {
  int SB[kNQ + 1];
  int CSRB[kNQ];
  int RB[kNR + 1];
  int4 SLOT[kNQ];
  uint16_t CELLQ[kSCap];
};

// Warp 0 only.
template <int NROW>
__device__ void geo_build(const TileArgs& a, int cy, int x0, int w, Geo& G, Tables& Tb) {
  constexpr int R0 = NROW == 3 ? 1 : 0;
  const int lane = threadIdx.x & 31;
  const int nx = a.g.counts[0], ny = a.g.counts[1];
  int rowc[3] = {-1, -1, -1};
#pragma unroll
  for (int r = 0; r < NROW; ++r) {
    int y = cy + r - R0;
    bool in = true;
    if (y < 0) { y += ny; in = a.g.wrap[1] != 0; }
    else if (y >= ny) { y -= ny; in = a.g.wrap[1] != 0; }
    rowc[r] = in ? y * nx : -1;
  }
  const int nq = NROW * (w + 2);
  int run = 0;
  for (int q0 = 0; q0 < nq; q0 += 32) {
    const int q = q0 + lane;
    int len = 0, cs = 0;
    if (q < nq) {
      const int r = q / (w + 2), u = q - r * (w + 2);
      int x = x0 - 1 + u;
      bool in = rowc[r] >= 0;
      if (x < 0) { x += nx; in = in && a.g.wrap[0]; }
      else if (x >= nx) { x -= nx; in = in && a.g.wrap[0]; }
      if (in) {
        const int c = rowc[r] + x;
        cs = __ldg(a.start + c);
        len = __ldg(a.start + c + 1) - cs;
      }
    }
    const int incl = warp_incl(len, lane);
    if (q < nq) {
      Tb.SB[q] = run + incl - len;
      Tb.CSRB[q] = cs - (run + incl - len);
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) Tb.SB[nq] = run;
  __syncwarp();
  int rrun = 0, rmax = 0;
  if (NROW == 3) {
    const int nr = 3 * w;
    for (int p0 = 0; p0 < nr; p0 += 32) {
      const int p = p0 + lane;
      int plen = 0;
      if (p < nr) {
        const int c = p / 3 + 1, r = p - 3 * (c - 1), q = r * (w + 2) + c;
        const int len = Tb.SB[q + 2] - Tb.SB[q - 1];
        plen = len + (len & 1);
      }
      rmax = max(rmax, plen);
      const int incl = warp_incl(plen, lane);
      if (p < nr) Tb.RB[p] = rrun + incl - plen;
      rrun += __shfl_sync(0xffffffffu, incl, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    if (lane == 0) Tb.RB[nr] = rrun;
    __syncwarp();
    for (int q = lane; q < nq; q += 32) {
      const int r = q / (w + 2), u = q - r * (w + 2);
      int b[3];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int c = u + s - 1;  // runs centred at c hold cell u at place s
        b[s] = (c >= 1 && c <= w) ? Tb.RB[3 * (c - 1) + r] : -1;
      }
      Tb.SLOT[q] = make_int4(b[0], b[1], b[2], (r << 8) | u);
    }
  }
  if (lane == 0) {
    G.cy = cy;
    G.x0 = x0;
    G.w = w;
    G.nq = nq;
#pragma unroll
    for (int r = 0; r < 3; ++r) G.rowc[r] = rowc[r];
    const int q1 = R0 * (w + 2) + 1;  // the targets' row, cell u = 1 (x = x0)
    G.t0 = Tb.SB[q1];
    G.kt = Tb.CSRB[q1] + G.t0;
    G.T = Tb.SB[q1 + w] - G.t0;
    G.total = run;
    G.rtotal = rrun;
    G.over = run > kSCap || rrun > kRCap || rmax > 256;
  }
}

// Splits the tile (cy, [tx0, tx1)) into sub-tiles that fit shared memory and
// calls body() for each (all threads; G and the tables valid inside, CELLQ set
// unless G.over).
template <int NROW, class Body>
__device__ __forceinline__ void for_subtiles(const TileArgs& a, Geo& G, Tables& Tb, Body&& body) {
  const int nx = a.g.counts[0];
  const int tile = (int)blockIdx.x;
  const int cy = tile / a.tpr, b = tile - cy * a.tpr;
  const int tx0 = b * a.tw, tx1 = min(tx0 + a.tw, nx);
  int x0 = tx0;
  while (x0 < tx1) {
    int w = tx1 - x0;
    while (true) {
      if (threadIdx.x < 32) geo_build<NROW>(a, cy, x0, w, G, Tb);
      __syncthreads();
      if (!G.over || w == 1) break;
      w = (w + 1) >> 1;
      __syncthreads();
    }
    if (!G.over) {
      for (int q = threadIdx.x; q < G.nq; q += kBT)
        for (int e = Tb.SB[q]; e < Tb.SB[q + 1]; ++e) Tb.CELLQ[e] = (uint16_t)q;
      __syncthreads();
    }
    body();
    x0 += w;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Global-memory path for one row (stale cell, overflow, long runs): the
// reference's own enumeration (nnps.cpp:351-372) over the CSR, the same
// binary16 arithmetic, j != i.
// ---------------------------------------------------------------------------
struct Consts2 {
  __half2 hh0, hh1, hc0, thr;
  unsigned short hcy;
};

__device__ __forceinline__ Consts2 consts2(const TileArgs& a) {
  Consts2 k;
  k.hh0 = hb2(a.c.h_hh[0]);
  k.hh1 = hb2(a.c.h_hh[1]);
  k.hc0 = hb2(a.c.h_cc[0]);
  k.thr = hb2(a.c.h_thr);
  k.hcy = a.c.h_cc[1];
  return k;
}

// cc for a row offset: dc = -dy, cc = round16(dc * hc) = +hc16 (dy = -1), 0, -hc16 (dy = +1)
__device__ __forceinline__ unsigned short cc_bits(unsigned short hc16, int dy) {
  return dy == 0 ? 0 : (dy < 0 ? hc16 : (unsigned short)(hc16 ^ 0x8000u));
}

__device__ __forceinline__ bool hit1(const Consts2& K, __half2 rx, __half2 ry, __half xj, __half yj,
                                     int dcx, __half2 ccy) {
  __half2 t = __hmul2_rn(__hsub2_rn(rx, __half2half2(xj)), K.hh0);
  __half2 d = __hfma2(__half2half2(__int2half_rn(dcx)), K.hc0, t);
  __half2 acc = __hmul2_rn(d, d);
  t = __hmul2_rn(__hsub2_rn(ry, __half2half2(yj)), K.hh1);
  d = __hadd2_rn(t, ccy);
  acc = __hadd2_rn(acc, __hmul2_rn(d, d));
  return (__hlt2_mask(acc, K.thr) & 1u) != 0;
}

// Calls fn(j) for every neighbour j != i of particle i (cells from
// RelCoords::cell), cell by cell in the reference's order.
template <class Fn>
__device__ void slow_row(const TileArgs& a, const Consts2& K, int i, Fn&& fn) {
  const int nx = a.g.counts[0], ny = a.g.counts[1];
  const int cx = __ldg(a.cellk[0] + i), cy = __ldg(a.cellk[1] + i);
  if (cx < 0 || cx >= nx || cy < 0 || cy >= ny) return;  // malformed cell: no candidates
  const __half2 rx = __half2half2(__double2half(__ldg(a.rel[0] + i)));
  const __half2 ry = __half2half2(__double2half(__ldg(a.rel[1] + i)));
  for (int oy = -1; oy <= 1; ++oy) {
    int y = cy + oy;
    if (y < 0 || y >= ny) {
      if (!a.g.wrap[1]) continue;
      y = (y + ny) % ny;
    }
    const __half2 ccy = hb2(cc_bits(K.hcy, oy));
    for (int ox = -1; ox <= 1; ++ox) {
      int x = cx + ox;
      if (x < 0 || x >= nx) {
        if (!a.g.wrap[0]) continue;
        x = (x + nx) % nx;
      }
      const int c = y * nx + x;
      const int b = __ldg(a.start + c), e = __ldg(a.start + c + 1);
      for (int s = b; s < e; ++s) {
        const int j = __ldg(a.items + s);
        if (j == i) continue;
        const __half xj = __double2half(__ldg(a.rel[0] + j));
        const __half yj = __double2half(__ldg(a.rel[1] + j));
        if (hit1(K, rx, ry, xj, yj, -ox, ccy)) fn(j);
      }
    }
  }
}

// in-place heap sort of p[0, n) (the global-memory path's rows can be long)
__device__ void heap_sort(int32_t* p, int64_t n) {
  auto sift = [&](int64_t root, int64_t end) {
    while (true) {
      int64_t c = 2 * root + 1;
      if (c >= end) return;
      if (c + 1 < end && p[c + 1] > p[c]) ++c;
      if (p[root] >= p[c]) return;
      const int32_t t = p[root];
      p[root] = p[c];
      p[c] = t;
      root = c;
    }
  };
  for (int64_t s = n / 2 - 1; s >= 0; --s) sift(s, n);
  for (int64_t e = n - 1; e > 0; --e) {
    const int32_t t = p[0];
    p[0] = p[e];
    p[e] = t;
    sift(0, e);
  }
}

// p[0, gs) and p[gs, k) are each sorted: insert the tail into the head. Once a
// tail element is above everything before it, the rest are too.
__device__ __forceinline__ void merge_tail(int32_t* p, int gs, int k) {
  for (int e = gs; e < k; ++e) {
    const int v = p[e];
    int w = p[e - 1];
    if (w < v) break;
    int q = e;
    do {
      p[q] = w;
      --q;
    } while (q > 0 && (w = p[q - 1]) > v);
    p[q] = v;
  }
}

// ---------------------------------------------------------------------------
// Rank pass: one cell row per tile (cells x0-1 .. x0+w of row cy, ids only)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBT) k_t2_rank(TileArgs a) {
  __shared__ Geo G;
  __shared__ Tables Tb;
  __shared__ int SID[kSCap];
  __shared__ uint16_t LB[4][kSCap];  // members below the record in cells u-2, u-1, u+1, u+2
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  uint8_t* rank_b = reinterpret_cast<uint8_t*>(a.rank);
  for_subtiles<1>(a, G, Tb, [&]() {
    if (G.over) return;  // a cell of > 255 records: its runs take the global path
    const int w = G.w, nq = G.nq, total = G.total;
    for (int e = tid; e < total; e += kBT) {
      const int j = __ldg(a.items + Tb.CSRB[Tb.CELLQ[e]] + e);
      SID[e] = a.ids ? __ldg(a.ids + j) : j;
    }
    __syncthreads();
    // merges of cell u with u + d (d = 1, 2): each side learns its members' lower
    // bound in the other
    for (int m = tid; m < 2 * nq; m += kBT) {
      const int d = m < nq ? 1 : 2, ua = m < nq ? m : m - nq, ub = ua + d;
      if (ub >= nq) continue;
      int i = Tb.SB[ua];
      const int ie = Tb.SB[ua + 1];
      int j = Tb.SB[ub];
      const int jb = j, ib = i, je = Tb.SB[ub + 1];
      uint16_t* lba = LB[d == 1 ? 2 : 3];  // for cell ua: below in ua + d
      uint16_t* lbb = LB[d == 1 ? 1 : 0];  // for cell ub: below in ub - d
      while (i < ie && j < je) {
        const int vi = SID[i], vj = SID[j];
        if (vi < vj) { lba[i] = (uint16_t)(j - jb); ++i; }
        else { lbb[j] = (uint16_t)(i - ib); ++j; }
      }
      for (; i < ie; ++i) lba[i] = (uint16_t)(je - jb);
      for (; j < je; ++j) lbb[j] = (uint16_t)(ie - ib);
    }
    __syncthreads();
    for (int e = tid; e < total; e += kBT) {
      const int u = Tb.CELLQ[e];
      const int idx = e - Tb.SB[u];
      const int lm2 = u >= 2 ? LB[0][e] : 0, lm1 = u >= 1 ? LB[1][e] : 0;
      const int lp1 = u <= w ? LB[2][e] : 0, lp2 = u + 2 <= w + 1 ? LB[3][e] : 0;
      // byte s: place in the run centred at the record's cell + s - 1
      const uint32_t r0 = (uint32_t)min(idx + lm2 + lm1, 255),
                     r1 = (uint32_t)min(idx + lm1 + lp1, 255),
                     r2 = (uint32_t)min(idx + lp1 + lp2, 255);
      const int csr = Tb.CSRB[u] + e;
      if (u >= 2 && u <= w - 1) {  // all three runs centred in this sub-tile
        a.rank[csr] = r0 | (r1 << 8) | (r2 << 16);
      } else {
        uint8_t* p = rank_b + 4 * (int64_t)csr;
        if (u - 1 >= 1 && u - 1 <= w) p[0] = (uint8_t)r0;
        if (u >= 1 && u <= w) p[1] = (uint8_t)r1;
        if (u + 1 >= 1 && u + 1 <= w) p[2] = (uint8_t)r2;
      }
    }
  });
}

// ---------------------------------------------------------------------------
// Count pass
// ---------------------------------------------------------------------------
// Run record pair (records 2p, 2p+1 of the run storage): x pair, y pair, dc pair
// (dc = c - cell of the record, in {-1, 0, 1}), cc pair (the run's row). Pads:
// x = NaN (never a hit).
__device__ __forceinline__ void pair_bits(unsigned& acc, const uint4 rec, __half2 rx, __half2 ry,
                                          const Consts2& K) {
  __half2 t = __hmul2_rn(__hsub2_rn(rx, u2h(rec.x)), K.hh0);
  const __half2 d = __hfma2(u2h(rec.z), K.hc0, t);
  __half2 q = __hmul2_rn(d, d);
  t = __hadd2_rn(__hmul2_rn(__hsub2_rn(ry, u2h(rec.y)), K.hh1), u2h(rec.w));
  q = __hadd2_rn(q, __hmul2_rn(t, t));
  asm("{\n\t.reg .pred p0, p1;\n\t"
      "setp.lt.f16x2 p0|p1, %1, %2;\n\t"
      "shr.b32 %0, %0, 2;\n\t"
      "@p0 or.b32 %0, %0, 0x40000000;\n\t"
      "@p1 or.b32 %0, %0, 0x80000000;\n\t}"
      : "+r"(acc)
      : "r"(h2u(q)), "r"(h2u(K.thr)));
}

// dynamic shared memory of the count kernel: run record pairs
constexpr size_t kCountSmem = (size_t)kRCap * 8;

__global__ void __launch_bounds__(kBT) k_t2_count(TileArgs a) {
  __shared__ Geo G;
  __shared__ Tables Tb;
  __shared__ uint8_t TU[kSCap];
  __shared__ uint8_t SELF[kSCap];
  __shared__ __half2 TXY[kSCap];
  extern __shared__ __align__(16) uint4 REC[];  // [kRCap / 2] run record pairs
  __half* RH = reinterpret_cast<__half*>(REC);
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const Consts2 K = consts2(a);
  const __half cc0 = __ushort_as_half(cc_bits(K.hcy, -1)), cc2 = __ushort_as_half(cc_bits(K.hcy, 1));
  const __half dcm = __ushort_as_half(0xBC00u), dcz = __ushort_as_half(0), dcp = __ushort_as_half(0x3C00u);
  for_subtiles<3>(a, G, Tb, [&]() {
    const int T = G.T;
    if (T == 0) return;
    const bool over = G.over;
    const int t0 = G.t0, kt = G.kt;
    if (!over) {
      const int total = G.total;
      for (int e = tid; e < total; e += kBT) {
        const int q = Tb.CELLQ[e];
        const int4 sl = Tb.SLOT[q];
        const int csr = Tb.CSRB[q] + e;
        const int j = __ldg(a.items + csr);
        const uint32_t rk = __ldg(a.rank + csr);
        const __half x = __double2half(__ldg(a.rel[0] + j)), y = __double2half(__ldg(a.rel[1] + j));
        const int r = sl.w >> 8;
        const __half cc = r == 0 ? cc0 : (r == 1 ? dcz : cc2);
        auto put = [&](int base, int s, __half dc) {  // dc = c - u = s - 1
          const int pos = base + (int)((rk >> (8 * s)) & 255u);
          const int ph = 8 * (pos >> 1) + (pos & 1);
          RH[ph] = x;
          RH[ph + 2] = y;
          RH[ph + 4] = dc;
          RH[ph + 6] = cc;
        };
        if (sl.x >= 0) put(sl.x, 0, dcm);
        if (sl.y >= 0) put(sl.y, 1, dcz);
        if (sl.z >= 0) put(sl.z, 2, dcp);
        if (r == 1 && sl.y >= 0) {  // a target (row dy = 0, cell inside the sub-tile)
          TU[e - t0] = (uint8_t)(sl.w & 255);
          SELF[e - t0] = (uint8_t)((rk >> 8) & 255u);
          TXY[e - t0] = __halves2half2(x, y);
        }
      }
      const int w = G.w;
      for (int p = tid; p < 3 * w; p += kBT) {  // pad odd runs with a NaN record
        const int c = p / 3 + 1, r = p - 3 * (c - 1), q = r * (w + 2) + c;
        const int len = Tb.SB[q + 2] - Tb.SB[q - 1];
        if (len & 1) {
          const int ph = 8 * ((Tb.RB[p] + len) >> 1) + 1;
          RH[ph] = __ushort_as_half(0x7E00u);
          RH[ph + 2] = __ushort_as_half(0u);
          RH[ph + 4] = __ushort_as_half(0u);
          RH[ph + 6] = __ushort_as_half(0u);
        }
      }
      __syncthreads();
    }
    const int x0m1 = G.x0 - 1, cy = G.cy;
    for (int t = tid; t < T; t += kBT) {
      const int k = kt + t;
      const int i = __ldg(a.items + k);
      if (i < a.row0 || i >= a.row0 + a.nrows) continue;
      bool slow = over;
      int cnt = 0;
      if (!slow) {
        const int ut = TU[t];
        const int p0 = 3 * (ut - 1);
        const int base = Tb.RB[p0], len = Tb.RB[p0 + 3] - base;  // the target's 3 runs
        slow = len > 128 || __ldg(a.cellk[0] + i) != x0m1 + ut || __ldg(a.cellk[1] + i) != cy;
        if (!slow) {
          const __half2 xy = TXY[t];
          const __half2 rx = __low2half2(xy), ry = __high2half2(xy);
          const uint4* R = REC + (base >> 1);
          const int np = len >> 1;
          unsigned wv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            unsigned acc = 0;
            const int m = min(16, np - 16 * q);
            if (m > 0) {
#pragma unroll 4
              for (int p = 0; p < m; ++p) pair_bits(acc, R[16 * q + p], rx, ry, K);
              acc >>= 2 * (16 - m);
            }
            wv[q] = acc;
          }
          const int sb = Tb.RB[p0 + 1] - base + SELF[t];  // the own record is not a neighbour
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if ((sb >> 5) == q) wv[q] &= ~(1u << (sb & 31));
          cnt = __popc(wv[0]) + __popc(wv[1]) + __popc(wv[2]) + __popc(wv[3]);
          a.mw[k] = wv[0];
          a.mw[(int64_t)a.n + k] = wv[1];
          if (len > 64) {
            a.mx[k] = wv[2];
            a.mx[(int64_t)a.n + k] = wv[3];
          }
        }
      }
      if (slow) {
        cnt = 0;
        slow_row(a, K, i, [&](int) { ++cnt; });
      }
      a.flag[k] = slow ? 1 : 0;
      a.cnt[i - a.row0] = cnt;
    }
  });
}

// ---------------------------------------------------------------------------
// Scan: offsets[r] = sum of cnt[0, r), offsets[nrows] = total
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lb_publish(unsigned long long* tiles, int bid, long long total,
                                           unsigned epoch) {
  const unsigned long long E = (unsigned long long)epoch << 48;
  st_release_u64(&tiles[bid], E | ((bid == 0 ? 2ull : 1ull) << 46) | (unsigned long long)total);
}

__device__ __forceinline__ long long lb_resolve(unsigned long long* tiles, int bid, long long total,
                                                unsigned epoch) {
  if (bid == 0) return 0;
  const unsigned long long E = (unsigned long long)epoch << 48, PRE = 2ull << 46,
                           VAL = (1ull << 46) - 1;
  const int lane = threadIdx.x & 31;
  long long excl = 0;
  int p = bid - 1;
  unsigned backoff = 32, spins = 0;
  while (true) {
    const int idx = p - lane;
    const unsigned long long st = idx >= 0 ? ld_relaxed_u64(&tiles[idx]) : (E | PRE);
    const unsigned flag = (st >> 48) == epoch ? (unsigned)(st >> 46) & 3u : 0u;
    const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == 2u);
    const unsigned zero_mask = __ballot_sync(0xffffffffu, flag == 0u);
    const int first = pre_mask ? __ffs(pre_mask) - 1 : 32;
    const unsigned need = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (zero_mask & need) {
      if (++spins > (1u << 22)) __trap();
      __nanosleep(backoff);
      backoff = backoff < 256 ? backoff * 2 : 256;
      continue;
    }
    const long long v = lane <= first ? (long long)(st & VAL) : 0ll;
    excl += warp_sum_ll(v);
    if (first < 32) break;
    p -= 32;
  }
  if (lane == 0) st_release_u64(&tiles[bid], E | PRE | (unsigned long long)(excl + total));
  return excl;
}

// Tiles of kScanBT * kScanIPT counts; tile = blockIdx.x (blocks are dispatched
// in index order, so a tile never waits on one that has not started -- the
// assumption single-pass scans make; a predecessor that never publishes traps).
__global__ void __launch_bounds__(kScanBT) k_t2_scan(const int32_t* __restrict__ cnt, int nrows,
                                                     int64_t* __restrict__ off,
                                                     unsigned long long* tiles, unsigned epoch) {
  __shared__ long long s_w[kScanBT / 32];
  __shared__ long long s_base;
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanBT * kScanIPT + (int64_t)tid * kScanIPT;
  int v[kScanIPT];
  if (base + kScanIPT <= nrows) {
    const int4* p = reinterpret_cast<const int4*>(cnt + base);
#pragma unroll
    for (int q = 0; q < kScanIPT / 4; ++q) {
      const int4 x = __ldg(p + q);
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanIPT; ++q) v[q] = base + q < nrows ? __ldg(cnt + base + q) : 0;
  }
  long long s = 0;
#pragma unroll
  for (int q = 0; q < kScanIPT; ++q) s += v[q];
  long long x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  long long wb = 0, tot = 0;
#pragma unroll
  for (int u = 0; u < kScanBT / 32; ++u) {
    wb += u < warp ? s_w[u] : 0;
    tot += s_w[u];
  }
  if (tid == 0) lb_publish(tiles, blockIdx.x, tot, epoch);
  if (warp == 0) {
    const long long b = lb_resolve(tiles, blockIdx.x, tot, epoch);
    if (lane == 0) s_base = b;
  }
  __syncthreads();
  long long run = s_base + wb + x - s;
  const bool al = (reinterpret_cast<uintptr_t>(off) & 15u) == 0;
  if (base + kScanIPT <= nrows && al) {
    longlong2* p = reinterpret_cast<longlong2*>(off + base);
#pragma unroll
    for (int q = 0; q < kScanIPT / 2; ++q) {
      const long long a0 = run;
      run += v[2 * q];
      const long long a1 = run;
      run += v[2 * q + 1];
      p[q] = make_longlong2(a0, a1);
    }
    if (base + kScanIPT == nrows) off[nrows] = run;
  } else {
#pragma unroll
    for (int q = 0; q < kScanIPT; ++q) {
      if (base + q < nrows) off[base + q] = run;
      run += v[q];
      if (base + q == nrows - 1) off[nrows] = run;
    }
  }
}

// ---------------------------------------------------------------------------
// Fill pass
// ---------------------------------------------------------------------------
// dynamic shared memory: rows, run ids, the row tag of each row entry
constexpr size_t kFillSmem = (size_t)kPCap * 4 + (size_t)kRCap * 4 + (size_t)kPCap;

__global__ void __launch_bounds__(kBT, 1024 / kBT) k_t2_fill(TileArgs a) {
  __shared__ Geo G;
  __shared__ Tables Tb;
  __shared__ uint8_t TU[kSCap];
  __shared__ long long DST[kBT];  // offsets[i] - the row's position in ROWS
  __shared__ int s_w[kBT / 32];
  __shared__ int s_fit;
  extern __shared__ __align__(16) int32_t ROWS[];  // [kPCap]
  int32_t* RID = ROWS + kPCap;                     // [kRCap] run ids
  uint8_t* TAG = reinterpret_cast<uint8_t*>(RID + kRCap);  // [kPCap] row of each entry
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Consts2 K = consts2(a);
  const int64_t cap = a.capacity;
  for_subtiles<3>(a, G, Tb, [&]() {
    const int T = G.T;
    if (T == 0) return;
    const bool over = G.over;
    const int t0 = G.t0, kt = G.kt;
    if (!over) {
      const int total = G.total;
      for (int e = tid; e < total; e += kBT) {  // ids into the runs at their ranks
        const int q = Tb.CELLQ[e];
        const int4 sl = Tb.SLOT[q];
        const int csr = Tb.CSRB[q] + e;
        const int j = __ldg(a.items + csr);
        const uint32_t rk = __ldg(a.rank + csr);
        const int id = a.ids ? __ldg(a.ids + j) : j;
        if (sl.x >= 0) RID[sl.x + (int)(rk & 255u)] = id;
        if (sl.y >= 0) RID[sl.y + (int)((rk >> 8) & 255u)] = id;
        if (sl.z >= 0) RID[sl.z + (int)((rk >> 16) & 255u)] = id;
        if ((sl.w >> 8) == 1 && sl.y >= 0) TU[e - t0] = (uint8_t)(sl.w & 255);
      }
      __syncthreads();
    }
    for (int c0 = 0; c0 < T; c0 += kBT) {
      const int t = c0 + tid;
      const int k = kt + t;
      int i = -1;
      long long o0 = 0;
      int L = 0;
      bool fast = false;
      if (t < T) {
        const int ii = __ldg(a.items + k);
        if (ii >= a.row0 && ii < a.row0 + a.nrows) {
          i = ii;
          o0 = a.offsets[i - a.row0];
          L = (int)(a.offsets[i - a.row0 + 1] - o0);
          fast = !over && __ldg(a.flag + k) == 0;
        }
      }
      // tile-local row positions (block scan of the fast rows' lengths)
      const int x = fast ? L : 0;
      const int incl = warp_incl(x, lane);
      if (lane == 31) s_w[warp] = incl;
      if (tid == 0) s_fit = 0;
      __syncthreads();
      int pos = incl - x;
#pragma unroll
      for (int u = 0; u < kBT / 32; ++u) pos += u < warp ? s_w[u] : 0;
      const bool fits = fast && pos + L <= kPCap;
      if (fits) atomicMax(&s_fit, pos + L);
      DST[tid] = o0 - pos;
      if (fast && (fits || o0 + L <= cap)) {
        int32_t* row = fits ? ROWS + pos : a.out + o0;
        const int ut = TU[t];
        const int p0 = 3 * (ut - 1);
        const int base = Tb.RB[p0], len = Tb.RB[p0 + 3] - base;
        const int b1 = Tb.RB[p0 + 1] - base, b2 = Tb.RB[p0 + 2] - base;
        unsigned long long v0 = (unsigned long long)__ldg(a.mw + k) |
                                ((unsigned long long)__ldg(a.mw + (int64_t)a.n + k) << 32);
        unsigned long long v1 = 0;
        if (len > 64)
          v1 = (unsigned long long)__ldg(a.mx + k) | ((unsigned long long)__ldg(a.mx + (int64_t)a.n + k) << 32);
        // hits before the 2nd / 3rd run (b1, b2 < 128): the runs (rows dy = -1,
        // 0, 1) are each sorted and interleave only where cell rows share ids
        auto below = [&](int b) {
          return b >= 64 ? __popcll(v0) + __popcll(v1 & ((1ull << (b - 64)) - 1ull))
                         : __popcll(v0 & ((1ull << b) - 1ull));
        };
        const int m1 = below(b1), m2 = below(b2);
        const int32_t* rid = RID + base;
        for (int m = 0; m < L; ++m) {  // next hit, lowest bit first
          const bool lo = v0 != 0;
          const unsigned long long v = lo ? v0 : v1;
          const int b = __ffsll((long long)v) - 1 + (lo ? 0 : 64);
          const unsigned long long cl = v & (v - 1);
          v0 = lo ? cl : v0;
          v1 = lo ? v1 : cl;
          row[m] = rid[b];
          if (fits) TAG[pos + m] = (uint8_t)tid;
        }
        if (m1 > 0 && m1 < m2 && row[m1] < row[m1 - 1]) merge_tail(row, m1, m2);
        if (m2 > 0 && m2 < L && row[m2] < row[m2 - 1]) merge_tail(row, m2, L);
      } else if (i >= 0 && !fast && o0 + L <= cap) {
        int32_t* row = a.out + o0;
        int m = 0;
        slow_row(a, K, i, [&](int j) { row[m++] = a.ids ? __ldg(a.ids + j) : j; });
        heap_sort(row, m);
      }
      __syncthreads();
      const int nf = s_fit;  // rows -> items, 32 consecutive entries per warp store
      for (int f = tid; f < nf; f += kBT) {
        const long long d = DST[TAG[f]] + f;
        if (d < cap) a.out[d] = ROWS[f];
      }
      __syncthreads();
    }
  });
}

}  // namespace

// Host-side shape of a call: tile width from the mean occupancy (about 0.9
// targets per thread), spread evenly over each cell row.
void tiled2_shape(int nx, int ny, int64_t n, int* tw, int* tpr, int64_t* ntiles) {
  const double occ = (double)n / ((double)nx * (double)ny);
  int want = (int)(0.9 * kBT / (occ > 1e-9 ? occ : 1e-9));
  want = want < 1 ? 1 : (want > kTWMax ? kTWMax : want);
  int p = (nx + want - 1) / want;
  int w = (nx + p - 1) / p;
  p = (nx + w - 1) / w;
  *tw = w;
  *tpr = p;
  *ntiles = (int64_t)p * ny;
}

int64_t tiled2_scan_tiles(int64_t nrows) {
  return (nrows + kScanBT * kScanIPT - 1) / (kScanBT * kScanIPT);
}

// rank -> count -> scan -> fill; returns the launches issued.
int launch_tiled2(const TileArgs& a, bool count, cudaStream_t st) {
  if (a.nrows == 0 || a.ntiles == 0) return 0;
  static int attr_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_dev[dev]) {
    cudaFuncSetAttribute(k_t2_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCountSmem);
    cudaFuncSetAttribute(k_t2_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFillSmem);
    attr_dev[dev] = 1;
  }
  int launches = 0;
  if (count) {
    launch_pdl(k_t2_rank, (unsigned)a.ntiles, kBT, 0, st, a);
    launch_pdl(k_t2_count, (unsigned)a.ntiles, kBT, kCountSmem, st, a);
    launch_pdl(k_t2_scan, (unsigned)tiled2_scan_tiles(a.nrows), kScanBT, 0, st,
               (const int32_t*)a.cnt, a.nrows, a.offsets, a.tiles, a.epoch);
    launches += 3;
  }
  launch_pdl(k_t2_fill, (unsigned)a.ntiles, kBT, kFillSmem, st, a);
  return launches + 1;
}

}  // namespace sphx_dev
