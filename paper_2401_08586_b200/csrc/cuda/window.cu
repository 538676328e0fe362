// Windowed FP16 RCLL for 2-D -- the BASELINE metric path: rcll(rel, grid, fp16)
// of nnps.cpp:283-416 (2-D FP16: the batch kernel detail::range_f16_rel_2d,
// nnps_batch.cpp:203-261) with build_table's sorted rows (nnps.cpp:26-66).
//
// Two kernels per call, chained with programmatic dependent launch:
//
//   k_w2_pack   the reference's per-call preparation (nnps.cpp:300-315), in CSR
//               order. Record blocks: xy[4p + (s&1)] = r16(rel_x[items[s]]),
//               xy[4p + 2 + (s&1)] = r16(rel_y[...]) (p = s/2: one 8-byte load
//               is the x pair and the y pair of two neighbouring records) and
//               id[s] = items[s]. Cell blocks (one thread per cell v):
//               u[s] = x(v) as binary16 for v's members (the CSR cell, so
//               u_i - u_j is the reference's minimum-image dc = -off,
//               nnps.cpp:359-362; exact: the path needs nx <= 2048), and the
//               *run list* of the x-triple centred at v: the positions of cells
//               v-1, v, v+1 (one contiguous CSR span) in ascending id order, by a
//               3-way merge of the cells' ascending ids (32 bytes, 0xFF-padded).
//
//   k_w2<BT>    one CTA per tile of BT consecutive rows (particle order). The
//               tile's targets are split at id-order jumps of more than two
//               cells into at most two *bands*; each band's window -- cell rows
//               ymin-1 .. ymax+1, cells xmin-1 .. xmax+1 -- is one contiguous CSR
//               range per cell row (linear cell = cx + nx*cy, x fastest,
//               cell_grid.hpp:74-78), staged in shared memory with TMA bulk
//               copies (cp.async.bulk, one mbarrier, one lane of warp 0 per window
//               row issuing that row's copies) together with the run lists
//               of its centre cells. A target's candidates in stencil row oy are
//               one contiguous window segment (cells cx-1, cx, cx+1):
//               A  tested two per binary16x2 op straight from shared memory
//                  (warp-uniform trip count, dc = u_i - u_j as one HSUB2) into a
//                  32-bit hit word per segment; the target's own record is found
//                  by id in its cell and cleared; block scan; decoupled look-back
//                  publish;
//               B  the centre cell's run list walks the segment in id order, so
//                  hits are appended already sorted (a segment whose ids
//                  interleave with the previous row's is merged in); rows packed
//                  in shared memory (over the dead coordinates), 16-byte stores.
//
// Tiles whose targets do not form <= 2 compact bands (a shuffled particle order),
// whose window exceeds shared memory or wraps a periodic x axis run the same A
// and B on the pack's CSR-order arrays in global memory. Targets whose segment
// exceeds 32 positions, wraps a periodic x axis there, or whose RelCoords cell is
// not their CSR cell take an exact per-row path that walks the 9 cells like the
// reference (nnps.cpp:354-410) and sorts the row.
//
// Exactness (per candidate, nnps.cpp:332-346, nnps_batch.cpp:238-258):
// s = r16(ri - rj); t = r16(s*hh); x: d = r16(t + r16(dc*hc)) as one HFMA2 (dc in
// {-1,0,1}, dc*hc16 exact); y: d = r16(t + cc) (cc = r16(-oy*hc); skipped in the
// centre row, where t + 0 only turns -0 into +0, which squares the same);
// acc = r16(r16(dx^2) + r16(dy^2)); hit iff acc < thr, the exact threshold of
// r16(sqrt(acc)) < cutoff16 (capi.cu thr16).

#include <climits>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace sphx_dev {

namespace {

constexpr int kSegMax = 32;   // positions per segment (one hit word, one run list)
constexpr int kRowsMax = 12;  // window rows (both bands)
constexpr int kBandRows = 6;  // rows of one band: ymax - ymin <= 3
constexpr int kPackR = 2;     // records per pack thread

// A tile's window, computed by the pack (one warp per tile) and brought into
// the sweep's shared memory with one bulk copy. fast = 0: no window (the tile's
// targets do not form <= 2 compact bands, or the window does not fit).
struct W2Desc {
  int fast, nb, split, total;  // bands; first row of band 1; window records
  int bx[2][4];                // band: xmin, xmax, ymin, ymax
  int rbase[kRowsMax];         // window row: window position of its first record
  int ra8[kRowsMax];           //   aligned CSR start (-1: no row)
  int rn[kRowsMax];            //   records (8-aligned)
  int rgy[kRowsMax];           //   grid row
};
static_assert(sizeof(W2Desc) % 16 == 0, "bulk-copied");

template <int BT>
struct W2Cfg {
  static constexpr int WCap = 12 * BT + BT / 4;  // window records
  static constexpr int PCap = WCap * 3 / 2 + 48;  // packed row entries (alias the coordinates)
  static constexpr int CSCap = 3 * BT;            // window cell boundaries
  static constexpr int RunCap = 7 * BT / 4;      // run lists
  static constexpr int MinB = BT == 128 ? 9 : 4;  // CTAs per SM (register budget: <= 56 at 9)
};

__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<const unsigned*>(&h); }
__device__ __forceinline__ __half2 u2h(unsigned u) { return *reinterpret_cast<const __half2*>(&u); }
__device__ __forceinline__ __half hb(unsigned b) { return __ushort_as_half((unsigned short)b); }

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// bits [q, 32) set
__device__ __forceinline__ unsigned above(int q) { return q >= 32 ? 0u : ~0u << q; }

// y centre difference of stencil row oy: cc = r16(dc*hc) with dc = -oy
__device__ __forceinline__ __half cc_half(unsigned hc16, int oy) {
  return oy == 0 ? hb(0) : hb(oy < 0 ? hc16 : (hc16 ^ 0x8000u));
}

struct SharedRow {
  uint32_t base;
  __device__ __forceinline__ void st(int e, int v) const {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + 4u * (uint32_t)e), "r"(v) : "memory");
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
  __device__ __forceinline__ int ld(int e) const { return p[e]; }
};

// dst[0, gs) and dst[gs, k) are each sorted: insert the tail into the head
// (stops at the first tail element already above everything before it).
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

template <class Row>
__device__ __forceinline__ void insertion_sort(const Row& dst, int k) {
  for (int e = 1; e < k; ++e) {
    const int v = dst.ld(e);
    int q = e;
    int w;
    while (q > 0 && (w = dst.ld(q - 1)) > v) {
      dst.st(q, w);
      --q;
    }
    dst.st(q, v);
  }
}

// look-back words: [63:48] epoch, [47:46] flag (1 aggregate, 2 inclusive), [45:0] value
__device__ __forceinline__ void lb_publish(unsigned long long* tiles, int bid, long long total,
                                           unsigned epoch) {
  const unsigned long long E = (unsigned long long)epoch << 48;
  st_relaxed_u64(&tiles[bid], E | ((bid == 0 ? 2ull : 1ull) << 46) | (unsigned long long)total);
}

__device__ __forceinline__ long long lb_resolve(unsigned long long* tiles, int bid, long long total,
                                                unsigned epoch) {
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
      // tiles run in blockIdx order, so a predecessor that never publishes is a
      // bug: fail the launch (~4 s) instead of hanging the device
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

template <int BT>
__device__ __forceinline__ void stream_tile(int32_t* gout, const SharedRow& pk, int n, int tid) {
  const int ph = (int)(((uintptr_t)gout & 15u) >> 2);
  int4* g4 = reinterpret_cast<int4*>(gout - ph);
  const int nv = (ph + n + 3) >> 2;
  for (int q = tid; q < nv; q += BT) {
    const int e0 = 4 * q - ph;
    if (e0 >= 0 && e0 + 4 <= n) {
      g4[q] = make_int4(pk.ld(e0), pk.ld(e0 + 1), pk.ld(e0 + 2), pk.ld(e0 + 3));
    } else {
      for (int e = max(e0, 0); e < min(e0 + 4, n); ++e) gout[e] = pk.ld(e);
    }
  }
}

// One candidate pair (positions 2t, 2t+1 of a segment): hits set the bits
// `bit` and `bit << 1` of H.
__device__ __forceinline__ void pair_test(unsigned X2, unsigned Y2, unsigned U2, __half2 rx2,
                                          __half2 ry2, __half2 ut2, __half2 hhx, __half2 hhy,
                                          __half2 hc2, __half2 ccy, bool ycc, __half2 thr2,
                                          unsigned bit, unsigned& H) {
  const __half2 tx = __hmul2_rn(__hsub2_rn(rx2, u2h(X2)), hhx);
  const __half2 dx = __hfma2(__hsub2_rn(ut2, u2h(U2)), hc2, tx);
  __half2 ty = __hmul2_rn(__hsub2_rn(ry2, u2h(Y2)), hhy);
  if (ycc) ty = __hadd2_rn(ty, ccy);
  const __half2 acc = __hadd2_rn(__hmul2_rn(dx, dx), __hmul2_rn(ty, ty));
  asm("{\n\t.reg .pred p0, p1;\n\t"
      ".reg .b32 b1;\n\t"
      "setp.lt.f16x2 p0|p1, %1, %2;\n\t"
      "shl.b32 b1, %3, 1;\n\t"
      "@p0 or.b32 %0, %0, %3;\n\t"
      "@p1 or.b32 %0, %0, b1;\n\t}"
      : "+r"(H)
      : "r"(h2u(acc)), "r"(h2u(thr2)), "r"(bit));
}

template <int BT>
struct W2Smem {
  using C = W2Cfg<BT>;
  union {
    struct {
      uint2 xy[C::WCap / 2 + 16];  // pair p: {x pair, y pair} of positions 2p, 2p+1 (+ pad:
      __half u[C::WCap + 32];      //   idle lanes read up to 32 positions past a segment)
    } c;
    int pk[C::PCap];               // phase B: the tile's packed rows (the coordinates are dead)
  };
  int id[C::WCap];                 // candidate particle ids
  uint4 run[C::RunCap * 2];        // run lists of the window's centre cells (32 bytes each)
  short cs[C::CSCap];              // window cell boundaries, relative to the row's CSR start
  alignas(16) W2Desc d;            // the tile's bands and window rows (from the pack)
  int wsum[BT / 32];
  long long base;
  unsigned long long bar;
};
static_assert(sizeof(W2Smem<128>::pk) <= sizeof(W2Smem<128>::c), "packed rows alias the coordinates");
static_assert(W2Cfg<256>::WCap < (1 << 12) && W2Cfg<256>::RunCap < (1 << 14) && kSegMax < (1 << 6),
              "segment words: window position 12 bits, length 6 bits, run list 14 bits");

// Where a segment's records are read from: the staged window (shared memory,
// window positions) or the pack's CSR-order arrays (global memory, CSR
// positions; tiles without a window). Positions keep their parity in both, so
// pair p/2 is the same record pair.
struct SmemSrc {  // 32-bit shared addresses of the window's arrays
  // a segment's first pair load starts at a multiple of 4 positions, so a group of
  // 4 pairs is two 16-byte loads of coordinates and two 8-byte loads of cell x
  static constexpr int kAlign = 4;
  uint32_t xy, u, id;
  __device__ __forceinline__ void quad(int q, uint2 (&v)[4], unsigned (&w)[4]) const {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
          : "=r"(v[2 * h].x), "=r"(v[2 * h].y), "=r"(v[2 * h + 1].x), "=r"(v[2 * h + 1].y)
          : "r"(xy + 8u * (uint32_t)(q + 2 * h)));
      asm("ld.shared.v2.b32 {%0, %1}, [%2];"
          : "=r"(w[2 * h]), "=r"(w[2 * h + 1])
          : "r"(u + 4u * (uint32_t)(q + 2 * h)));
    }
  }
  __device__ __forceinline__ int ident(int p) const {
    int v;
    asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(id + 4u * (uint32_t)p));
    return v;
  }
};
struct GlobSrc {
  static constexpr int kAlign = 8;  // positions per 4-pair vector load
  const uint2* xy;
  const unsigned* u;
  const int* id;
  // pairs q .. q+3 (q a multiple of 4): one 256-bit and one 128-bit load
  __device__ __forceinline__ void quad(int q, uint2 (&v)[4], unsigned (&w)[4]) const {
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v[0].x), "=r"(v[0].y), "=r"(v[1].x), "=r"(v[1].y), "=r"(v[2].x), "=r"(v[2].y),
          "=r"(v[3].x), "=r"(v[3].y)
        : "l"(xy + q));
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(u + q));
    w[0] = t.x;
    w[1] = t.y;
    w[2] = t.z;
    w[3] = t.w;
  }
  __device__ __forceinline__ int ident(int p) const { return __ldg(id + p); }
};

// Band geometry (identical in every thread: computed from the descriptor).
struct Geo {
  int rows[2], ncs[2], nrun[2];
  __device__ __forceinline__ int row0(int q) const { return q ? rows[0] : 0; }
  __device__ __forceinline__ int ncs_of(int q) const { return q ? ncs[1] : ncs[0]; }
  __device__ __forceinline__ int nrun_of(int q) const { return q ? nrun[1] : nrun[0]; }
  __device__ __forceinline__ int cs0(int rr) const {
    return rr < rows[0] ? rr * ncs[0] : rows[0] * ncs[0] + (rr - rows[0]) * ncs[1];
  }
  __device__ __forceinline__ int run0(int rr) const {
    return rr < rows[0] ? rr * nrun[0] : rows[0] * nrun[0] + (rr - rows[0]) * nrun[1];
  }
};

__device__ __forceinline__ Geo geo_of(const int (&bx)[2][4], int nb) {
  Geo G;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool on = q < nb;
    G.rows[q] = on ? bx[q][3] - bx[q][2] + 3 : 0;
    G.ncs[q] = on ? bx[q][1] - bx[q][0] + 4 : 0;
    G.nrun[q] = on ? bx[q][1] - bx[q][0] + 1 : 0;
  }
  return G;
}

// Segment of target (cx, cy) in stencil row oy = s - 1: window positions of the
// cell boundaries L | C | R | end, and the window row.
struct Seg {
  int pL, pC, pR, pE, r;
};
template <int BT>
__device__ __forceinline__ Seg seg_of(const W2Smem<BT>& S, const Geo& G, int b, int cx, int cy,
                                      int s) {
  Seg g;
  g.r = G.row0(b) + (cy + s - S.d.bx[b][2]);  // window row (ymin-1 is the band's row 0)
  const short* cs = S.cs + G.cs0(g.r) + (cx - S.d.bx[b][0]);
  const int base = S.d.rbase[g.r];
  g.pL = base + cs[0];
  g.pC = base + cs[1];
  g.pR = base + cs[2];
  g.pE = base + cs[3];
  return g;
}

// Segment of target (cx, cy) in stencil row oy = s - 1 from the CSR (tiles
// without a window): CSR positions of the cell boundaries L | C | R | end and
// the centre cell (its run list). ok = false: the segment wraps a periodic x
// axis (the exact path); an absent row (walled y) is an empty segment.
__device__ __forceinline__ Seg seg_glob(const Win2Args& a, int cx, int cy, int s, bool& ok) {
  Seg g{0, 0, 0, 0, -1};
  const int nx = a.g.counts[0], ny = a.g.counts[1];
  if (a.g.wrap[0] && (cx == 0 || cx == nx - 1)) {
    ok = false;
    return g;
  }
  int y = cy + s - 1;
  if (y < 0 || y >= ny) {
    if (!a.g.wrap[1]) return g;
    y = (y + ny) % ny;
  }
  const int64_t row = (int64_t)y * nx;
  const int4 b = __ldg(a.wcb + row + cx);  // the pack's boundaries of the triple
  if (b.x < 0) {
    ok = false;
    return g;
  }
  g.pL = b.x;
  g.pC = b.y;
  g.pR = b.z;
  g.pE = b.w;
  g.r = (int)(row + cx);  // the centre cell
  return g;
}

// Cell blocks [0, ncb): one cell v per thread (see the file comment; first in
// the grid: their merge is the longest dependency chain). Record blocks
// [ncb, ...): kPackR records per thread (strided by the block size). The
// block's cells and their x-neighbours are one CSR span, staged in shared
// memory. Triples whose span exceeds 32 or that need a wrapped cell get no run
// list (the sweep takes those rows on the exact path).
// One warp per sweep tile (blocks [0, ntb)): the tile's bands and window rows
// (the sweep's prologue, moved here where issue slots are idle). Targets are the
// tile's a.bt consecutive rows, bt/32 per lane; a band split is a jump of more
// than two cells between consecutive targets.
__device__ void w2_tile_desc(const Win2Args& a, int tile) {
  const int lane = threadIdx.x & 31, per = a.bt >> 5;
  const int nx = a.g.counts[0], ny = a.g.counts[1];
  const int r0 = tile * a.bt + lane * per;
  auto cell = [&](int j, int& x, int& y) {  // target r0 + j (false past the rows)
    if (r0 + j >= a.nrows) return false;
    const int i = a.row0 + r0 + j;
    x = __ldg(a.cellk[0] + i);
    y = __ldg(a.cellk[1] + i);
    return true;
  };
  // breaks between consecutive targets (the previous lane's last for j = 0)
  int lx = 0, ly = 0;
  cell(per - 1, lx, ly);
  int qx = __shfl_up_sync(0xffffffffu, lx, 1), qy = __shfl_up_sync(0xffffffffu, ly, 1);
  int nbrk = 0, first = INT_MAX;
  for (int j = 0; j < per; ++j) {
    int x, y;
    if (!cell(j, x, y)) break;
    if ((lane > 0 || j > 0) && (abs(x - qx) > 2 || abs(y - qy) > 2)) {
      ++nbrk;
      first = min(first, lane * per + j);
    }
    qx = x;
    qy = y;
  }
  nbrk = __reduce_add_sync(0xffffffffu, nbrk);
  first = __reduce_min_sync(0xffffffffu, first);
  W2Desc* D = static_cast<W2Desc*>(a.desc) + tile;
  int fast = nbrk <= 1;
  const int nb = nbrk + 1, split = nbrk == 1 ? first : a.bt;
  int bx[2][4];
  {
    int x0[2] = {INT_MAX, INT_MAX}, x1[2] = {INT_MIN, INT_MIN};
    int y0[2] = {INT_MAX, INT_MAX}, y1[2] = {INT_MIN, INT_MIN};
    for (int j = 0; j < per; ++j) {  // (the cells are L1 hits now)
      int x, y;
      if (!cell(j, x, y)) break;
      const bool q1 = lane * per + j >= split;
      x0[0] = q1 ? x0[0] : min(x0[0], x);
      x1[0] = q1 ? x1[0] : max(x1[0], x);
      y0[0] = q1 ? y0[0] : min(y0[0], y);
      y1[0] = q1 ? y1[0] : max(y1[0], y);
      x0[1] = q1 ? min(x0[1], x) : x0[1];
      x1[1] = q1 ? max(x1[1], x) : x1[1];
      y0[1] = q1 ? min(y0[1], y) : y0[1];
      y1[1] = q1 ? max(y1[1], y) : y1[1];
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      bx[q][0] = __reduce_min_sync(0xffffffffu, x0[q]);
      bx[q][1] = __reduce_max_sync(0xffffffffu, x1[q]);
      bx[q][2] = __reduce_min_sync(0xffffffffu, y0[q]);
      bx[q][3] = __reduce_max_sync(0xffffffffu, y1[q]);
    }
  }
  const Geo G = geo_of(bx, fast ? nb : 0);
  if (fast) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q >= nb) continue;
      // rows/cells of the band inside the grid; columns xmin-1 .. xmax+1 must not
      // wrap a periodic x axis
      if (bx[q][0] < 0 || bx[q][1] >= nx || bx[q][2] < 0 || bx[q][3] >= ny) fast = 0;
      if (a.g.wrap[0] && (bx[q][0] == 0 || bx[q][1] == nx - 1)) fast = 0;
      if (G.rows[q] > kBandRows) fast = 0;
    }
    const int nr = G.rows[0] + G.rows[1];
    if (G.cs0(nr) > a.cscap || G.run0(nr) > a.runcap) fast = 0;
  }
  // window rows: one lane per row
  const int nrw = fast ? G.rows[0] + G.rows[1] : 0;
  int gy = -1, a8 = -1, n8 = 0;
  if (lane < nrw) {
    const int q = lane < G.rows[0] ? 0 : 1;
    const int bx0 = q ? bx[1][0] : bx[0][0], bx1 = q ? bx[1][1] : bx[0][1];
    const int y = (q ? bx[1][2] : bx[0][2]) - 1 + (lane - G.row0(q));
    gy = y;
    if (y < 0 || y >= ny) gy = a.g.wrap[1] ? (y + ny) % ny : -1;
    if (gy >= 0) {
      const int64_t row = (int64_t)gy * nx;
      const int s0 = __ldg(a.start + row + max(bx0 - 1, 0));
      const int s1 = __ldg(a.start + row + min(bx1 + 1, nx - 1) + 1);
      a8 = s0 & ~7;
      n8 = s1 > s0 ? ((s1 + 7) & ~7) - a8 : 0;
    }
  }
  int incl = n8;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total > a.wcap) fast = 0;
  if (lane < kRowsMax) {
    D->rbase[lane] = incl - n8;
    D->ra8[lane] = a8;
    D->rn[lane] = n8;
    D->rgy[lane] = gy;
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) D->bx[q][e] = bx[q][e];
  }
  if (lane == 0) {
    D->fast = fast;
    D->nb = nb;
    D->split = split;
    D->total = total;
  }
}

__global__ void __launch_bounds__(256) k_w2_pack(Win2Args a, int ntb, int ncb) {
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < ntb) {
    const int tile = blockIdx.x * 8 + (tid >> 5);
    if (tile * a.bt < a.nrows) w2_tile_desc(a, tile);
    pdl_trigger();
    return;
  }
  if ((int)blockIdx.x < ntb + ncb) {
    constexpr int kSpan = 2048;
    __shared__ int sid[kSpan];
    __shared__ int sst[256 + 3];
    const int64_t C = (int64_t)a.g.counts[0] * a.g.counts[1];
    const int64_t v0 = (int64_t)(blockIdx.x - ntb) * 256;
    for (int e = tid; e < 256 + 3; e += 256)
      sst[e] = __ldg(a.start + min(max(v0 - 1 + e, (int64_t)0), C));
    __syncthreads();
    const int lo = sst[0], hi = sst[256 + 2];
    const bool staged = hi - lo <= kSpan;
    if (staged)
      for (int e = tid; e < hi - lo; e += 256) {
        const int j = __ldg(a.items + lo + e);
        sid[e] = a.ids ? __ldg(a.ids + j) : j;  // merged by output id
      }
    __syncthreads();
    const int* sids = sid - lo;
    auto key = [&](int p) {  // the output id at CSR position p
      if (staged) return sids[p];
      const int j = __ldg(a.items + p);
      return a.ids ? __ldg(a.ids + j) : j;
    };
    const int64_t v = v0 + tid;
    const int nx = a.g.counts[0];
    const int x = (int)(v % nx);
    if (v < C) {
      const int m1 = sst[tid + 1], m2 = sst[tid + 2];
      const __half hx = __int2half_rn(x);
      for (int s = m1; s < m2; ++s) a.wu[s] = hx;
      const int s0 = x > 0 ? sst[tid] : m1;
      const int e = x + 1 < nx ? sst[tid + 3] : m2;
      const bool wraps = a.g.wrap[0] && (x == 0 || x == nx - 1);
      a.wcb[v] = wraps ? make_int4(-1, -1, -1, -1) : make_int4(s0, m1, m2, e);
      if (e - s0 <= kSegMax && !wraps) {
        int iL = s0, iC = m1, iR = m2;
        int vL = iL < m1 ? key(iL) : INT_MAX;
        int vC = iC < m2 ? key(iC) : INT_MAX;
        int vR = iR < e ? key(iR) : INT_MAX;
        unsigned w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = 0xFFFFFFFFu;
#pragma unroll
        for (int t = 0; t < kSegMax; ++t) {
          if (t >= e - s0) break;
          const int mn = min(vL, min(vC, vR));
          const bool tl = mn == vL, tc = !tl && mn == vC;
          const int pos = tl ? iL : (tc ? iC : iR);
          if (tl) ++iL;
          else if (tc) ++iC;
          else ++iR;
          const int nxt = pos + 1;
          const int nv = (tl ? nxt < m1 : (tc ? nxt < m2 : nxt < e)) ? key(nxt) : INT_MAX;
          vL = tl ? nv : vL;
          vC = tc ? nv : vC;
          vR = (!tl && !tc) ? nv : vR;
          const unsigned sh = 8 * (t & 3);
          w[t >> 2] = (w[t >> 2] & ~(0xFFu << sh)) | ((unsigned)(pos - s0) << sh);
        }
        uint4* dst = reinterpret_cast<uint4*>(a.wrun + v * kSegMax);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    pdl_trigger();
    return;
  }
  int id[kPackR];
  double rx[kPackR], ry[kPackR];
  const int s0 = (blockIdx.x - ntb - ncb) * 256 * kPackR + tid;
  // the CSR's records (a slab's arrays have spare capacity past them)
  const int nrec = __ldg(a.start + (int64_t)a.g.counts[0] * a.g.counts[1]);
#pragma unroll
  for (int q = 0; q < kPackR; ++q) {
    const int s = s0 + 256 * q;
    id[q] = s < nrec ? __ldg(a.items + s) : 0;
  }
#pragma unroll
  for (int q = 0; q < kPackR; ++q) {
    rx[q] = __ldg(a.rel[0] + id[q]);
    ry[q] = __ldg(a.rel[1] + id[q]);
  }
#pragma unroll
  for (int q = 0; q < kPackR; ++q) {
    const int s = s0 + 256 * q;
    if (s >= nrec) break;
    const int p = s >> 1, h = s & 1;
    a.wxy[4 * p + h] = __double2half(rx[q]);
    a.wxy[4 * p + 2 + h] = __double2half(ry[q]);
    a.wid[s] = a.ids ? __ldg(a.ids + id[q]) : id[q];
    a.wself[id[q]] = s;
  }
  pdl_trigger();
}

__device__ __forceinline__ __half w2_x(const Win2Args& a, int64_t s) {
  return a.wxy[4 * (s >> 1) + (s & 1)];
}
__device__ __forceinline__ __half w2_y(const Win2Args& a, int64_t s) {
  return a.wxy[4 * (s >> 1) + 2 + (s & 1)];
}

// The exact per-row path (any input): the reference's 9-cell walk
// (nnps.cpp:354-410) with its minimum-image offsets dc = -off (:359-362).
// EMIT: the row is written to dst[0, k) and sorted.
template <bool EMIT, class Row, bool SORT = true>
__device__ int w2_slow_row(const Win2Args& a, int i, int cxi, int cyi, __half rx, __half ry,
                           const Row& dst) {
  const int nx = a.g.counts[0], ny = a.g.counts[1];
  const __half hhx = hb(a.c.h_hh[0]), hhy = hb(a.c.h_hh[1]);
  const __half thr = hb(a.c.h_thr);
  const int gi = a.ids ? __ldg(a.ids + i) : i;  // the target's output id
  int k = 0;
  for (int oy = -1; oy <= 1; ++oy) {
    int cy = cyi + oy;
    if (cy < 0 || cy >= ny) {
      if (!a.g.wrap[1] || cy < -ny || cy >= 2 * ny) continue;
      cy = (cy + ny) % ny;
    }
    const __half ccy = cc_half(a.c.h_cc[1], oy);
    for (int ox = -1; ox <= 1; ++ox) {
      int cx = cxi + ox;
      if (cx < 0 || cx >= nx) {
        if (!a.g.wrap[0] || cx < -nx || cx >= 2 * nx) continue;
        cx = (cx + nx) % nx;
      }
      const int64_t c = (int64_t)cy * nx + cx;
      const int b = __ldg(a.start + c), e = __ldg(a.start + c + 1);
      const __half ccx = cc_half(a.c.h_cc[0], ox);  // r16(dc*hc), dc = -ox
      for (int s = b; s < e; ++s) {
        const int j = __ldg(a.wid + s);
        if (j == gi) continue;
        const __half dx = __hadd_rn(__hmul_rn(__hsub_rn(rx, w2_x(a, s)), hhx), ccx);
        const __half dy = __hadd_rn(__hmul_rn(__hsub_rn(ry, w2_y(a, s)), hhy), ccy);
        const __half acc = __hadd_rn(__hmul_rn(dx, dx), __hmul_rn(dy, dy));
        if (__hlt(acc, thr)) {
          if (EMIT) dst.st(k, j);
          ++k;
        }
      }
    }
  }
  if (EMIT && SORT) insertion_sort(dst, k);
  return k;
}

// grad_normalized's per-row sums (gradient.cpp:57-72, kernel_grad kernel.hpp:
// 53-64, kernel_dwdr :40-47) in the reference's operation order, every FP64 op
// rounded once (no contraction), over the row's neighbours in ascending id order.
__device__ __forceinline__ double w2_dwdr(double R, double alpha) {
  if (R < 1.0) return __dmul_rn(alpha, __dadd_rn(__dmul_rn(-2.0, R), __dmul_rn(__dmul_rn(1.5, R), R)));
  if (R < 2.0) {
    const double t = __dsub_rn(2.0, R);
    return __dmul_rn(-alpha, __dmul_rn(__dmul_rn(0.5, t), t));
  }
  return 0.0;
}
// One neighbour's contributions to the three sums (the same for (i,j) and (j,i)).
struct W2Term {
  double num[2], den[2], scale[2];
};

struct W2Grad {
  double num[2] = {0.0, 0.0}, den[2] = {0.0, 0.0}, scale[2] = {0.0, 0.0};
  double xi[2], fi, ih;  // ih = RN(1/h)
  // neighbour j's inputs (positions, field value)
  struct Nb {
    double x[2], f;
  };
  __device__ __forceinline__ static Nb load(const Win2Args& a, int j) {
    return Nb{{__ldg(a.gx[0] + j), __ldg(a.gx[1] + j)}, __ldg(a.gf + j)};
  }
  __device__ __forceinline__ W2Term term(const Win2Args& a, int j) const { return term(a, load(a, j)); }
  __device__ __forceinline__ W2Term term(const Win2Args& a, const Nb& nb) const {
    double dx[2], gw[2] = {0.0, 0.0}, r2 = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      dx[k] = __dsub_rn(xi[k], nb.x[k]);
      r2 = __dadd_rn(r2, __dmul_rn(dx[k], dx[k]));
    }
    const double r = __dsqrt_rn(r2);
    if (r != 0.0) {
      const double R = div_by(r, a.gh, ih);
      const double sc = __ddiv_rn(w2_dwdr(R, a.galpha), __dmul_rn(a.gh, r));
#pragma unroll
      for (int k = 0; k < 2; ++k) gw[k] = __dmul_rn(sc, dx[k]);
    }
    const double df = __dsub_rn(nb.f, fi);
    W2Term t;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      t.num[k] = __dmul_rn(df, gw[k]);
      t.den[k] = __dmul_rn(-dx[k], gw[k]);
      t.scale[k] = fabs(__dmul_rn(dx[k], gw[k]));
    }
    return t;
  }
  __device__ __forceinline__ void acc(const W2Term& t) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      num[k] = __dadd_rn(num[k], t.num[k]);
      den[k] = __dadd_rn(den[k], t.den[k]);
      scale[k] = __dadd_rn(scale[k], t.scale[k]);
    }
  }
  __device__ __forceinline__ void add(const Win2Args& a, int j) { acc(term(a, j)); }
  // g_k = num/den, or 0 and a degenerate count (gradient.cpp:73-80)
  __device__ __forceinline__ unsigned long long finish(const Win2Args& a, int i) const {
    unsigned long long deg = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double lim = __dmul_rn(1e-14, scale[k] > 0.0 ? scale[k] : 1.0);
      double g = 0.0;
      if (fabs(den[k]) < lim) ++deg;
      else g = __ddiv_rn(num[k], den[k]);
      a.gout[k][i] = g;
    }
    return deg;
  }
};

// The gradient of a row that is not packed in shared memory: its neighbours in
// ascending id order by repeated selection over the exact 9-cell walk.
__device__ void w2_slow_grad(const Win2Args& a, int i, int cxi, int cyi, __half rx, __half ry,
                             W2Grad& acc) {
  int last = INT_MIN;
  while (true) {
    int best = INT_MAX;
    const struct Sel {
      int* best;
      int last;
      __device__ void st(int, int v) const {
        if (v > last && v < *best) *best = v;
      }
      __device__ int ld(int) const { return 0; }
    } sel{&best, last};
    w2_slow_row<true, Sel, false>(a, i, cxi, cyi, rx, ry, sel);
    if (best == INT_MAX) break;
    acc.add(a, best);
    last = best;
  }
}

// GRAD: the fused NNPS -> grad_normalized (no table): each packed row is walked
// in id order into the FP64 sums of its particle.
template <int BT, bool GRAD>
__global__ void __launch_bounds__(BT, GRAD ? 1024 / BT : W2Cfg<BT>::MinB) k_w2(Win2Args a) {
  using Cfg = W2Cfg<BT>;
  extern __shared__ __align__(128) unsigned char smraw[];
  W2Smem<BT>& S = *reinterpret_cast<W2Smem<BT>*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;  // tiles are dispatched in blockIdx order (look-back)
  const int r = tile * BT + tid;
  const bool valid = r < a.nrows;
  const int i = a.row0 + (valid ? r : 0);
  const int nx = a.g.counts[0];
  // the shared window's base, kept in a register (otherwise re-derived from the
  // CTA id at every shared access)
  uint32_t smb = smem_u32(smraw);
  asm volatile("" : "+r"(smb));
  auto sa = [&](const void* p) {
    return smb + (uint32_t)(reinterpret_cast<const unsigned char*>(p) - smraw);
  };
  const uint32_t bar = sa(&S.bar);

  // ---- targets (inputs: issued before the pack is waited for) ----
  const int cx = __ldg(a.cellk[0] + i), cy = __ldg(a.cellk[1] + i);
  const __half rxh = __double2half(__ldg(a.rel[0] + i));
  const __half ryh = __double2half(__ldg(a.rel[1] + i));

  // one warp polls the barrier (phase `ph`); the others wait at __syncthreads
  auto wait_bar = [&](unsigned ph) {
    if (warp == 0)
      asm volatile(
          "{\n\t.reg .pred P;\n"
          "W2WAIT%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
          "@!P bra W2WAIT%=;\n\t}" ::"r"(bar),
          "r"(ph)
          : "memory");
    __syncthreads();
  };
  // warp 0: stage the window (TMA bulk copies) -- one lane per window row issues
  // its row's copies after lane 0 has armed the barrier with the window's bytes
  auto issue_window = [&](const Geo& G, int nrw) {
    const int rr = lane;
    const int gy = rr < nrw ? S.d.rgy[rr] : -1;
    const int q = rr < G.rows[0] ? 0 : 1;
    const unsigned rb = gy >= 0 ? 32u * (unsigned)G.nrun_of(q) : 0u;
    const unsigned tx = (unsigned)S.d.total * 10u + __reduce_add_sync(0xffffffffu, rb);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx)
                   : "memory");
    __syncwarp();
    if (gy >= 0) {
      const int n8 = S.d.rn[rr], a8 = S.d.ra8[rr], wb = S.d.rbase[rr];
      const void* src[4] = {a.wxy + 2 * (int64_t)a8, a.wu + a8, a.wid + a8,
                            a.wrun + ((int64_t)gy * nx + S.d.bx[q][0]) * kSegMax};
      const uint32_t dst[4] = {sa(&S.c.xy[wb >> 1]), sa(&S.c.u[wb]), sa(&S.id[wb]),
                               sa(&S.run[2 * G.run0(rr)])};
      const unsigned bytes[4] = {4u * n8, 2u * n8, 4u * n8, rb};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (bytes[c] == 0) continue;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dst[c]),
            "l"(src[c]), "r"(bytes[c]), "r"(bar)
            : "memory");
      }
    }
  };
  // ---- the tile's descriptor (bands, window rows: the pack's tile warps) ----
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pdl_wait();  // the pack's arrays are complete
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((unsigned)sizeof(W2Desc))
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sa(&S.d)),
        "l"(static_cast<const W2Desc*>(a.desc) + tile), "r"((unsigned)sizeof(W2Desc)), "r"(bar)
        : "memory");
  }
  wait_bar(0);
  bool fast = S.d.fast;
  const int b = (S.d.nb == 2 && tid >= S.d.split) ? 1 : 0;
  const Geo G = geo_of(S.d.bx, fast ? S.d.nb : 0);
  const int nrw = G.rows[0] + G.rows[1];

  // ---- the window's cell boundaries (cell_start is an input) while the copies
  // fly: a warp per row ----
  if (fast) {
    if (warp == 0) issue_window(G, nrw);
    for (int rr = warp; rr < nrw; rr += BT / 32) {
      const int q = rr < G.rows[0] ? 0 : 1;
      const int ncs = G.ncs_of(q), cs0 = G.cs0(rr);
      const int gy = S.d.rgy[rr], a8 = S.d.ra8[rr];
      const int64_t row = (int64_t)gy * nx;
      for (int e = lane; e < ncs; e += 32)
        S.cs[cs0 + e] =
            gy < 0 ? (short)0
                   : (short)(__ldg(a.start + row + min(max(S.d.bx[q][0] - 1 + e, 0), nx)) - a8);
    }
    wait_bar(1);
  }
  pdl_wait();  // (the exact path reads the pack's arrays from global memory)

  // ---- A: hit words, row length ----
  const __half2 hhx = __half2half2(hb(a.c.h_hh[0])), hhy = __half2half2(hb(a.c.h_hh[1]));
  const __half2 hc2 = __half2half2(hb(a.c.h_cc[0])), thr2 = __half2half2(hb(a.c.h_thr));
  const __half2 rx2 = __half2half2(rxh), ry2 = __half2half2(ryh);
  const __half2 ut2 = __half2half2(__int2half_rn(cx));
  bool slow = !valid;
  int k = 0;
  const SmemSrc ssrc{sa(S.c.xy), sa(S.c.u), sa(S.id)};
  const GlobSrc gsrc{reinterpret_cast<const uint2*>(a.wxy), reinterpret_cast<const unsigned*>(a.wu),
                     a.wid};
  // segment s of this lane's target: window positions (fast tile) or CSR
  // positions (tile without a window)
  auto seg = [&](int s) -> Seg {
    Seg g{0, 0, 0, 0, -1};
    if (!valid || slow) return g;
    if (fast) return seg_of(S, G, b, cx, cy, s);
    bool ok = true;
    g = seg_glob(a, cx, cy, s, ok);
    if (!ok) slow = true;
    return g;
  };
  const int selfcsr = valid ? __ldg(a.wself + i) : 0;
  unsigned hw[3];  // phase A hit words of the 3 segments (registers: s is unrolled there)
  // window tiles: each segment's start, length and run-list slot, packed by phase A
  // (pL | len << 12 | run << 18) so that phase B does not derive them again
  unsigned sg[3] = {0u, 0u, 0u};
  auto phase_a = [&](const auto& src) {  // every lane: warp-uniform loops
    int tot = 0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const Seg g = seg(s);
      constexpr int kA = std::decay_t<decltype(src)>::kAlign;
      const int p0 = g.pL & ~(kA - 1);
      if (g.pE - p0 > kSegMax) slow = true;
      // pairs of this lane; the loop runs the warp's maximum (lanes past their
      // segment test the records that follow it, masked out below)
      const int np = slow ? 0 : (g.pE - p0 + 1) >> 1;
      const int npmax = __reduce_max_sync(0xffffffffu, np);
      const __half2 ccy = __half2half2(cc_half(a.c.h_cc[1], s - 1));
      const int q0 = p0 >> 1;
      unsigned H = 0;
      // groups of 4 pairs with no branch between them, so the 4 dependent
      // binary16 chains interleave
#pragma unroll
      for (int t0 = 0; t0 < kSegMax / 2; t0 += 4) {
        if (t0 >= npmax) break;
        uint2 xy[4];
        unsigned u2[4];
        src.quad(q0 + t0, xy, u2);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          pair_test(xy[t].x, xy[t].y, u2[t], rx2, ry2, ut2, hhx, hhy, hc2, ccy, s != 1, thr2,
                    1u << (2 * (t0 + t)), H);
      }
      H &= above(g.pL - p0) & ~above(g.pE - p0);  // bit q = position p0 + q
      if (s == 1 && !slow) {
        // the target's own record (its CSR position from the pack), which must
        // lie in its centre cell
        const int sp = fast ? S.d.rbase[g.r] + (selfcsr - S.d.ra8[g.r]) : selfcsr;
        if (sp >= g.pC && sp < g.pR) H &= ~(1u << (sp - p0));
        else slow = true;  // RelCoords cell is not the CSR cell (a stale grid)
      }
      hw[s] = H;
      if constexpr (std::is_same_v<std::decay_t<decltype(src)>, SmemSrc>)
        sg[s] = (unsigned)g.pL | ((unsigned)(g.pE - g.pL) << 12) |
                ((unsigned)(G.run0(g.r) + cx - S.d.bx[b][0]) << 18);
      tot += __popc(H);
    }
    k = tot;
  };
  if (fast) phase_a(ssrc);  // (CTA-uniform)
  else phase_a(gsrc);
  if (valid && slow) k = w2_slow_row<false>(a, i, cx, cy, rxh, ryh, GlobalRow{nullptr});

  // ---- block scan, publish ----
  const int incl = warp_inclusive_scan(k);
  if (lane == 31) S.wsum[warp] = incl;
  __syncthreads();
  int wbase = 0, btot = 0;
#pragma unroll
  for (int u = 0; u < BT / 32; ++u) {
    wbase += u < warp ? S.wsum[u] : 0;
    btot += S.wsum[u];
  }
  const int excl = wbase + incl - k;
  if (!GRAD && tid == 0) lb_publish(a.tiles, tile, btot, a.epoch);

  // ---- B: sorted rows ----
  // The run list of the target's centre cell walks each segment in id order, so
  // hits are appended sorted: a warp-uniform walk, four positions per step.
  auto build_src = [&](const auto& dst, bool part, const auto& src) {
    int kk = 0;
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
      const unsigned H = part ? (s == 0 ? hw[0] : (s == 1 ? hw[1] : hw[2])) : 0u;
      constexpr bool kSg = std::is_same_v<std::decay_t<decltype(src)>, SmemSrc>;
      Seg g{0, 0, 0, 0, -1};
      unsigned sgw = 0;
      if constexpr (kSg) sgw = H ? (s == 0 ? sg[0] : (s == 1 ? sg[1] : sg[2])) : 0u;
      else if (H) g = seg(s);
      const int pL = kSg ? (int)(sgw & 0xFFFu) : g.pL;
      const int len = kSg ? (int)((sgw >> 12) & 0x3Fu) : g.pE - g.pL;
      const int lmax = __reduce_max_sync(0xffffffffu, len);
      if (lmax == 0) continue;
      constexpr int kA = std::decay_t<decltype(src)>::kAlign;
      const unsigned hrel = H >> (pL & (kA - 1));  // bit o = position pL + o
      uint4 w[2];
      if (fast) {
        const uint4* rl =
            kSg ? &S.run[2 * (sgw >> 18)] : &S.run[2 * (H ? G.run0(g.r) + cx - S.d.bx[b][0] : 0)];
        w[0] = rl[0];
        w[1] = rl[1];
      } else {
        const uint4* rl = reinterpret_cast<const uint4*>(a.wrun) + 2 * (int64_t)(H ? g.r : 0);
        w[0] = __ldg(rl);
        w[1] = __ldg(rl + 1);
      }
      const int gs = kk;
      if constexpr (std::is_same_v<std::decay_t<decltype(src)>, SmemSrc> &&
                    std::is_same_v<std::decay_t<decltype(dst)>, SharedRow>) {
        // shared addresses carried in bytes: the segment's ids from idb, the row's
        // next slot at da (advanced by 4 per hit); one PRMT per run-list offset
        const uint32_t idb = src.id + 4u * (uint32_t)pL;
        uint32_t da = dst.base + 4u * (uint32_t)kk;
#pragma unroll
        for (int t4 = 0; t4 < 8; ++t4) {
          if (4 * t4 >= lmax) break;
          const unsigned word = t4 < 4 ? (&w[0].x)[t4] : (&w[1].x)[t4 - 4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned off = __byte_perm(word, 0u, 0x4440u | u);  // 0xFF past the run
            unsigned sh;
            asm("shr.b32 %0, %1, %2;" : "=r"(sh) : "r"(hrel), "r"(off));  // (0 for off >= 32)
            const unsigned hit = sh & 1u;
            if (hit) {
              int v;
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(idb + 4u * off) : "memory");
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(da), "r"(v) : "memory");
            }
            da += hit << 2;
          }
        }
        kk = (int)((da - dst.base) >> 2);
      } else {
#pragma unroll
        for (int t4 = 0; t4 < 8; ++t4) {
          if (4 * t4 >= lmax) break;
          const unsigned word = t4 < 4 ? (&w[0].x)[t4] : (&w[1].x)[t4 - 4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned off = (word >> (8 * u)) & 0xFFu;  // 0xFF past the run
            unsigned sh;
            asm("shr.b32 %0, %1, %2;" : "=r"(sh) : "r"(hrel), "r"(off));  // (0 for off >= 32)
            const bool hit = sh & 1u;
            if (hit) dst.st(kk, src.ident(pL + (int)off));
            kk += hit;
          }
        }
      }
      if (gs > 0 && kk > gs && dst.ld(gs) < dst.ld(gs - 1)) merge_tail(dst, gs, kk);
    }
  };
  auto build = [&](const auto& dst, bool part) {
    if (fast) build_src(dst, part, ssrc);
    else build_src(dst, part, gsrc);
  };
  const bool fits = btot <= Cfg::PCap;
  if (fits) {
    const SharedRow row{sa(S.pk) + 4u * (uint32_t)excl};
    build(row, valid && !slow);
    if (valid && slow && k > 0) w2_slow_row<true>(a, i, cx, cy, rxh, ryh, row);
  }
  if constexpr (GRAD) {
    unsigned long long deg = 0;
    if (valid) {
      W2Grad acc;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) acc.xi[kk] = __ldg(a.gx[kk] + i);
      acc.fi = __ldg(a.gf + i);
      acc.ih = __drcp_rn(a.gh);
      if (fits && k > 0) {  // the thread's own sorted row; the next neighbour's
                            // inputs are loaded while this one's term is computed
        const SharedRow row{sa(S.pk) + 4u * (uint32_t)excl};
        W2Grad::Nb cur = W2Grad::load(a, row.ld(0));
        for (int e = 0; e < k; ++e) {
          const W2Grad::Nb nxt = W2Grad::load(a, row.ld(e + 1 < k ? e + 1 : e));
          acc.acc(acc.term(a, cur));
          cur = nxt;
        }
      } else if (!fits) {
        w2_slow_grad(a, i, cx, cy, rxh, ryh, acc);
      }
      deg = acc.finish(a, i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) deg += __shfl_xor_sync(0xffffffffu, deg, o);
    if (lane == 0 && deg) atomicAdd(a.gdeg, deg);
    return;
  }

  if (warp == 0) {
    const long long bse = lb_resolve(a.tiles, tile, btot, a.epoch);
    if (lane == 0) S.base = bse;
  }
  __syncthreads();
  const long long base = S.base;
  if (valid) a.offsets[r] = base + excl;
  if (r == a.nrows - 1) a.offsets[a.nrows] = base + excl + k;
  if (base + btot > a.capacity) return;
  int32_t* gout = a.out + base;
  if (!fits) {
    const GlobalRow row{gout + excl};
    build(row, valid && !slow);
    if (valid && slow && k > 0) w2_slow_row<true>(a, i, cx, cy, rxh, ryh, row);
    return;
  }
  stream_tile<BT>(gout, SharedRow{sa(S.pk)}, btot, tid);
}

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

// rows per tile: SPHX_W2BT=128|256 (default 128; read per call)
int w2_bt() {
  const char* e = std::getenv("SPHX_W2BT");
  return (e && std::atoi(e) == 256) ? 256 : 128;
}

template <int BT, bool GRAD>
void launch_sweep_bt(const Win2Args& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_w2<BT, GRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(W2Smem<BT>));
    attr = true;
  }
  launch_pdl(k_w2<BT, GRAD>, (unsigned)((a.nrows + BT - 1) / BT), BT, sizeof(W2Smem<BT>), st, a);
}

}  // namespace

int64_t win2_tiles(int64_t nrows) { return (nrows + w2_bt() - 1) / w2_bt(); }
size_t win2_desc_bytes(int64_t nrows) { return sizeof(W2Desc) * (size_t)win2_tiles(nrows); }

// pack + sweep (grad: pack + fused gradient); returns the number of kernels launched.
// mid: an event recorded between the two (timing breakdown only), or null.
int launch_win2(const Win2Args& args, bool grad, cudaStream_t st, cudaEvent_t mid) {
  Win2Args a = args;
  a.bt = w2_bt();
  a.wcap = a.bt == 256 ? W2Cfg<256>::WCap : W2Cfg<128>::WCap;
  a.cscap = a.bt == 256 ? W2Cfg<256>::CSCap : W2Cfg<128>::CSCap;
  a.runcap = a.bt == 256 ? W2Cfg<256>::RunCap : W2Cfg<128>::RunCap;
  const int nbr = (a.n + 256 * kPackR - 1) / (256 * kPackR);
  const int64_t C = (int64_t)a.g.counts[0] * a.g.counts[1];
  const int ncb = (int)((C + 255) / 256);
  const int64_t ntiles = (a.nrows + a.bt - 1) / a.bt;
  const int ntb = (int)((ntiles + 7) / 8);
  k_w2_pack<<<(unsigned)(ntb + ncb + nbr), 256, 0, st>>>(a, ntb, ncb);
  if (mid) cudaEventRecord(mid, st);
  if (grad) {
    if (a.bt == 256) launch_sweep_bt<256, true>(a, st);
    else launch_sweep_bt<128, true>(a, st);
  } else {
    if (a.bt == 256) launch_sweep_bt<256, false>(a, st);
    else launch_sweep_bt<128, false>(a, st);
  }
  return 2;
}

}  // namespace sphx_dev
