/* TEST INFRASTRUCTURE ONLY -- see sphx_oracle.h.
 *
 * Plain-C restatement of the reference NNPS path. Compiled with
 * -ffp-contract=off so no multiply-add is fused (the reference is built with no
 * -march and therefore never contracts). */
#include "sphx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* binary16: binary16.cpp:12-57 (from_f64) and :59-74 (to_f64).              */
/* ------------------------------------------------------------------------ */
uint16_t so_f16_from_f64(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
  const int ef = (int)((b >> 52) & 0x7FF);
  const uint64_t frac = b & 0x000FFFFFFFFFFFFFull;
  if (ef == 0x7FF) return frac ? 0x7E00u : (uint16_t)(sign | 0x7C00u); /* NaN canonical */
  if ((b & 0x7FFFFFFFFFFFFFFFull) == 0) return sign;
  const int e = ef - 1023;
  if (e >= 16) return (uint16_t)(sign | 0x7C00u);
  uint64_t sig = frac | (ef ? (1ull << 52) : 0);
  int he = e + 15, shift = 42;
  if (he < 1) {
    shift += 1 - he;
    he = 0;
    if (shift >= 54) return sign;
  }
  uint64_t hs = sig >> shift;
  const uint64_t rem = sig & ((1ull << shift) - 1), half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (hs & 1))) ++hs; /* round to nearest even */
  if (he == 0) return (uint16_t)(sign | hs);       /* subnormal (carry -> min normal) */
  const uint32_t packed = ((uint32_t)he << 10) + (uint32_t)(hs - 0x400);
  if (packed >= 0x7C00u) return (uint16_t)(sign | 0x7C00u);
  return (uint16_t)(sign | packed);
}

double so_f16_to_f64(uint16_t b) {
  const int ef = (b >> 10) & 0x1F, fr = b & 0x3FF;
  double m;
  if (ef == 0x1F) {
    if (fr) return NAN;
    m = INFINITY;
  } else if (ef == 0) {
    m = (double)fr * 0x1.0p-24; /* ldexp(fr, -24), exact */
  } else {                      /* ldexp(fr|0x400, ef-25) built directly */
    const uint64_t bits = ((uint64_t)(ef - 15 + 1023) << 52) | ((uint64_t)fr << 42);
    memcpy(&m, &bits, 8);
  }
  return (b & 0x8000u) ? -m : m;
}

double so_round16(double x) { return so_f16_to_f64(so_f16_from_f64(x)); }

/* binary16.hpp:97-103 */
double so_round_to(int prec, double x) {
  if (prec == SO_FP64) return x;
  if (prec == SO_FP32) return (double)(float)x;
  return so_round16(x);
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (std::mt19937_64 is pinned by the C++ standard) + rng.hpp.     */
/* ------------------------------------------------------------------------ */
void so_rng_seed(so_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t so_rng_next(so_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:15 */
double so_rng_uniform01(so_rng* r) { return (double)(so_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:22-29 */
uint64_t so_rng_below(so_rng* r, uint64_t n) {
  const uint64_t limit = ~(uint64_t)0 - (~(uint64_t)0 % n);
  uint64_t v;
  do v = so_rng_next(r);
  while (v >= limit);
  return v % n;
}

/* ------------------------------------------------------------------------ */
/* build_gapped_random (experiments.cpp:55-112), restated by brute force: a    */
/* draw is rejected when any placed particle lies at squared distance in      */
/* (lo2, hi2). The reference searches only the 3x3 buckets of edge            */
/* cutoff + width around the draw; every particle closer than cutoff + width  */
/* lies in them, so scanning all placed particles takes the same decisions.   */
/* Returns 0, or -4 (the reference's runtime_error) after 4000 rejections.    */
/* ------------------------------------------------------------------------ */
int so_build_gapped_random(const double* lo, const double* hi, int64_t n, double cutoff,
                           double width, uint64_t seed, double* x0, double* x1) {
  so_rng rng;
  so_rng_seed(&rng, seed);
  const double lo2 = (cutoff - width) * (cutoff - width);
  const double hi2 = (cutoff + width) * (cutoff + width);
  for (int64_t i = 0; i < n; ++i) {
    int attempt = 0;
    for (;; ++attempt) {
      if (attempt > 4000) return -4;
      const double x = lo[0] + (hi[0] - lo[0]) * so_rng_uniform01(&rng); /* rng.hpp:17 */
      const double y = lo[1] + (hi[1] - lo[1]) * so_rng_uniform01(&rng);
      int ok = 1;
      for (int64_t j = 0; j < i && ok; ++j) {
        const double dx = x - x0[j], dy = y - x1[j];
        const double d2 = dx * dx + dy * dy;
        if (d2 > lo2 && d2 < hi2) ok = 0;
      }
      if (ok) {
        x0[i] = x;
        x1[i] = y;
        break;
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Generators: particle_system.cpp:31-62 (lattice), :64-77 (uniform).        */
/* ------------------------------------------------------------------------ */
int64_t so_lattice_count(int dim, const double* lo, const double* hi, double ds) {
  int64_t n = 1;
  for (int k = 0; k < dim; ++k) n *= (int64_t)floor((hi[k] - lo[k]) / ds + 0.5);
  return n;
}

int so_build_lattice(int dim, const double* lo, const double* hi, double ds, double jitter,
                     uint64_t seed, double* x0, double* x1, double* x2) {
  if (!(ds > 0.0) || jitter < 0.0 || jitter >= 0.5) return -2;
  int64_t counts[3] = {1, 1, 1};
  for (int k = 0; k < dim; ++k) {
    if (ds > hi[k] - lo[k]) return -2;
    counts[k] = (int64_t)floor((hi[k] - lo[k]) / ds + 0.5);
  }
  double* xs[3] = {x0, x1, x2};
  so_rng rng;
  so_rng_seed(&rng, seed);
  int64_t idx = 0;
  for (int64_t c2 = 0; c2 < counts[2]; ++c2)
    for (int64_t c1 = 0; c1 < counts[1]; ++c1)
      for (int64_t c0 = 0; c0 < counts[0]; ++c0) {
        const int64_t c[3] = {c0, c1, c2};
        for (int k = 0; k < dim; ++k) {
          double xk = lo[k] + ((double)c[k] + 0.5) * ds;
          if (jitter > 0.0) xk += jitter * ds * (2.0 * so_rng_uniform01(&rng) - 1.0);
          xs[k][idx] = xk;
        }
        ++idx;
      }
  return 0;
}

double so_build_random(int dim, const double* lo, const double* hi, int64_t n, uint64_t seed,
                       double* x0, double* x1, double* x2) {
  double vol = 1.0;
  for (int k = 0; k < dim; ++k) vol *= hi[k] - lo[k];
  const double ds = pow(vol / (double)n, 1.0 / dim);
  double* xs[3] = {x0, x1, x2};
  so_rng rng;
  so_rng_seed(&rng, seed);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < dim; ++k) xs[k][i] = lo[k] + (hi[k] - lo[k]) * so_rng_uniform01(&rng);
  return ds;
}

/* ------------------------------------------------------------------------ */
/* Grid: cell_grid.cpp:9-34; normalize_domain cell_grid.hpp:16-24.           */
/* ------------------------------------------------------------------------ */
int so_grid_init(so_grid* g, int dim, const double* lo, const double* hi, double radius,
                 const int* periodic) {
  memset(g, 0, sizeof(*g));
  if (!(radius > 0.0)) return -2;
  g->dim = dim;
  g->radius = radius;
  double hd = 0.0;
  for (int k = 0; k < dim; ++k) hd = fmax(hd, hi[k] - lo[k]);
  g->hd = hd;
  g->cutoff_norm = 2.0 * radius / hd;
  g->total = 1;
  for (int k = 0; k < 3; ++k) {
    g->counts[k] = 1;
    g->lo[k] = lo[k];
    g->hi[k] = hi[k];
    g->periodic[k] = periodic ? periodic[k] : 0;
  }
  for (int k = 0; k < dim; ++k) {
    const double span = hi[k] - lo[k];
    if (g->periodic[k]) {
      const int c = (int)floor(span / radius + 1e-12);
      g->counts[k] = c > 0 ? c : 1;
      g->edge[k] = span / g->counts[k];
      if (g->counts[k] < 3) return -2;
    } else {
      g->counts[k] = (int)ceil(span / radius - 1e-12);
      if (g->counts[k] < 1) g->counts[k] = 1;
      g->edge[k] = radius;
    }
    g->hc[k] = 2.0 * g->edge[k] / hd;
    g->total *= g->counts[k];
    g->origin[k] = (2.0 * lo[k] - (hi[k] + lo[k])) / hd;
  }
  return 0;
}

static double center_norm(const so_grid* g, int k, int32_t c) {
  return g->origin[k] + ((double)c + 0.5) * g->hc[k]; /* cell_grid.hpp:70-72 */
}

static int64_t linear_cell(const so_grid* g, const int32_t* c) { /* cell_grid.hpp:74-78 */
  int64_t idx = c[g->dim - 1];
  for (int k = g->dim - 2; k >= 0; --k) idx = idx * g->counts[k] + c[k];
  return idx;
}

static void normalize(const so_grid* g, const double* const* x, int64_t i, double* xn) {
  for (int k = 0; k < 3; ++k) xn[k] = 0.0;
  for (int k = 0; k < g->dim; ++k) xn[k] = (2.0 * x[k][i] - (g->hi[k] + g->lo[k])) / g->hd;
}

/* cell_grid.cpp:36-64 */
void so_locate(const so_grid* g, const double* xn, int32_t* cell, double* rel) {
  for (int k = 0; k < g->dim; ++k) {
    const double off = xn[k] - g->origin[k];
    int32_t c = (int32_t)floor(off / g->hc[k]);
    if (c < 0) c = 0;
    if (c >= g->counts[k]) c = g->counts[k] - 1;
    double r = 2.0 * (xn[k] - center_norm(g, k, c)) / g->hc[k];
    if (r < -1.0 && c > 0) {
      --c;
      r = 2.0 * (xn[k] - center_norm(g, k, c)) / g->hc[k];
    } else if (r > 1.0 && c + 1 < g->counts[k]) {
      ++c;
      r = 2.0 * (xn[k] - center_norm(g, k, c)) / g->hc[k];
    }
    if (r == -1.0 && c > 0) {
      --c;
      r = 1.0;
    }
    cell[k] = c;
    rel[k] = r;
  }
  for (int k = g->dim; k < 3; ++k) {
    cell[k] = 0;
    rel[k] = 0.0;
  }
}

/* build_csr: cell_grid.cpp:97-108 (serial stable counting sort). */
static void build_csr(const so_grid* g, int64_t n, const int32_t* cell_of, int32_t* start,
                      int32_t* items) {
  memset(start, 0, sizeof(int32_t) * (size_t)(g->total + 1));
  for (int64_t i = 0; i < n; ++i) ++start[cell_of[i] + 1];
  for (int64_t c = 0; c < g->total; ++c) start[c + 1] += start[c];
  int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->total + 1));
  memcpy(cursor, start, sizeof(int32_t) * (size_t)g->total);
  for (int64_t i = 0; i < n; ++i) items[cursor[cell_of[i]]++] = (int32_t)i;
  free(cursor);
}

/* cell_grid.cpp:66-84 */
int so_rebin(const so_grid* g, int64_t n, const double* const* x, int32_t* cell_of,
             int32_t* start, int32_t* items, int64_t* bad) {
  double xn[3], r[3];
  int32_t c[3];
  for (int64_t i = 0; i < n; ++i) {
    normalize(g, x, i, xn);
    for (int k = 0; k < g->dim; ++k) {
      const double off = xn[k] - g->origin[k];
      const double top = g->counts[k] * g->hc[k];
      if (off < -1e-9 * g->hc[k] || off > top + 1e-9 * g->hc[k]) {
        if (bad) *bad = i;
        return -3;
      }
    }
    so_locate(g, xn, c, r);
    cell_of[i] = (int32_t)linear_cell(g, c);
  }
  build_csr(g, n, cell_of, start, items);
  return 0;
}

/* cell_grid.cpp:114-133 and rebuild_members :86-95 */
void so_build_rel(const so_grid* g, int64_t n, const double* const* x, double** rel,
                  int32_t** cell, int32_t* cell_of, int32_t* start, int32_t* items) {
  double xn[3], r[3];
  int32_t c[3];
  for (int64_t i = 0; i < n; ++i) {
    normalize(g, x, i, xn);
    so_locate(g, xn, c, r);
    for (int k = 0; k < g->dim; ++k) {
      rel[k][i] = r[k];
      cell[k][i] = c[k];
    }
    cell_of[i] = (int32_t)linear_cell(g, c);
  }
  build_csr(g, n, cell_of, start, items);
}

/* ------------------------------------------------------------------------ */
/* Table building: nnps.cpp:26-66 (rows ascending, offsets int64).           */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t* v;
  int64_t len, cap;
} vec32;

static void vpush(vec32* a, int32_t x) {
  if (a->len == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 1024;
    a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
  }
  a->v[a->len++] = x;
}

static void sort_tail(int32_t* v, int64_t len) { /* insertion sort: rows are short */
  for (int64_t a = 1; a < len; ++a) {
    const int32_t x = v[a];
    int64_t b = a;
    while (b > 0 && v[b - 1] > x) {
      v[b] = v[b - 1];
      --b;
    }
    v[b] = x;
  }
}

static void table_begin(so_table* t, int64_t n) {
  t->n = n;
  t->total = 0;
  t->offsets = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  t->items = NULL;
}

static void table_end_row(so_table* t, vec32* buf, int64_t i, int64_t row_begin) {
  sort_tail(buf->v + row_begin, buf->len - row_begin);
  t->offsets[i + 1] = buf->len;
}

static void table_finish(so_table* t, vec32* buf) {
  t->total = buf->len;
  t->items = buf->v ? buf->v : (int32_t*)malloc(4);
}

void so_table_free(so_table* t) {
  free(t->offsets);
  free(t->items);
  t->offsets = NULL;
  t->items = NULL;
}

uint64_t so_table_hash(const so_table* t) {
  uint64_t x = 1469598103934665603ull;
  for (int64_t i = 0; i <= t->n; ++i) {
    x ^= (uint64_t)t->offsets[i];
    x *= 1099511628211ull;
  }
  for (int64_t q = 0; q < t->total; ++q) {
    x ^= (uint32_t)t->items[q];
    x *= 1099511628211ull;
  }
  return x;
}

/* ------------------------------------------------------------------------ */
/* Absolute-coordinate distance: dist_prec, nnps.cpp:91-124.                 */
/* xd holds coordinates already rounded into prec (round_coords :75-89).     */
/* ------------------------------------------------------------------------ */
static double dist_prec(double* const* xd, int dim, int64_t i, int64_t j, const double* shift,
                        int prec) {
  if (prec == SO_FP64) {
    double acc = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double d = xd[k][i] - (xd[k][j] + shift[k]);
      acc += d * d;
    }
    return sqrt(acc);
  }
  if (prec == SO_FP32) {
    float acc = 0.0f;
    for (int k = 0; k < dim; ++k) {
      float xj = (float)xd[k][j];
      if (shift[k] != 0.0) xj += (float)shift[k];
      const float d = (float)xd[k][i] - xj;
      acc += d * d;
    }
    return (double)sqrtf(acc);
  }
  double acc16 = 0.0;
  for (int k = 0; k < dim; ++k) {
    double xj = xd[k][j];
    if (shift[k] != 0.0) xj = so_round16(xj + shift[k]);
    const double d = so_round16(xd[k][i] - xj);
    const double sq = so_round16(d * d);
    acc16 = so_round16(acc16 + sq);
  }
  return so_round16(sqrt(acc16));
}

static double** round_coords(int dim, int64_t n, const double* const* x, int prec) {
  double** xd = (double**)calloc(3, sizeof(double*));
  for (int k = 0; k < dim; ++k) {
    xd[k] = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) xd[k][i] = so_round_to(prec, x[k][i]);
  }
  return xd;
}

static void free_coords(double** xd) {
  for (int k = 0; k < 3; ++k) free(xd[k]);
  free(xd);
}

/* nnps.cpp:128-172 */
int so_all_list(int dim, int64_t n, const double* const* x, double h, int prec, so_table* out) {
  if (n == 0) return -2; /* "all_list needs at least one particle" */
  const double cutoff = so_round_to(prec, 2.0 * h);
  double** xd = round_coords(dim, n, x, prec);
  const double noshift[3] = {0.0, 0.0, 0.0};
  vec32 buf = {0};
  table_begin(out, n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rb = buf.len;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      if (dist_prec(xd, dim, i, j, noshift, prec) < cutoff) vpush(&buf, (int32_t)j);
    }
    table_end_row(out, &buf, i, rb);
  }
  table_finish(out, &buf);
  free_coords(xd);
  return 0;
}

/* nnps.cpp:174-281 */
int so_cll(const so_grid* g, int64_t n, const double* const* x, double h,
           const int32_t* cell_of, const int32_t* items, const int32_t* start, int prec,
           so_table* out) {
  const int dim = g->dim;
  const double cutoff = so_round_to(prec, 2.0 * h);
  double** xd = round_coords(dim, n, x, prec);
  double span_prec[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < dim; ++k) span_prec[k] = so_round_to(prec, g->hi[k] - g->lo[k]);
  vec32 buf = {0};
  table_begin(out, n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rb = buf.len;
    int32_t ci[3] = {0, 0, 0};
    int32_t lin = cell_of[i];
    for (int k = 0; k < dim; ++k) {
      ci[k] = lin % g->counts[k];
      lin /= g->counts[k];
    }
    const int oy_lo = dim > 1 ? -1 : 0, oy_hi = dim > 1 ? 1 : 0;
    const int oz_lo = dim > 2 ? -1 : 0, oz_hi = dim > 2 ? 1 : 0;
    for (int oz = oz_lo; oz <= oz_hi; ++oz)
      for (int oy = oy_lo; oy <= oy_hi; ++oy)
        for (int ox = -1; ox <= 1; ++ox) {
          const int off[3] = {ox, oy, oz};
          int32_t c[3] = {0, 0, 0};
          double shift[3] = {0.0, 0.0, 0.0};
          int skip = 0;
          for (int k = 0; k < dim && !skip; ++k) {
            int32_t ck = ci[k] + off[k];
            if (ck < 0) {
              if (g->periodic[k] && g->counts[k] > 2) {
                ck += g->counts[k];
                shift[k] = -span_prec[k];
              } else {
                skip = 1;
              }
            } else if (ck >= g->counts[k]) {
              if (g->periodic[k] && g->counts[k] > 2) {
                ck -= g->counts[k];
                shift[k] = span_prec[k];
              } else {
                skip = 1;
              }
            }
            c[k] = ck;
          }
          if (skip) continue;
          const int64_t cell = linear_cell(g, c);
          for (int64_t s = start[cell]; s < start[cell + 1]; ++s) {
            const int32_t j = items[s];
            if (j == i) continue;
            if (dist_prec(xd, dim, i, j, shift, prec) < cutoff) vpush(&buf, j);
          }
        }
    table_end_row(out, &buf, i, rb);
  }
  table_finish(out, &buf);
  free_coords(xd);
  return 0;
}

/* rcll axis_term (nnps.cpp:321-339): one axis of the relative distance. */
static double axis_term(int prec, double reli, double relj, int dc, double hc, double half_hc) {
  if (prec == SO_FP64) return (reli - relj) * (0.5 * hc) + (double)dc * hc;
  if (prec == SO_FP32) {
    const float s = (float)reli - (float)relj;
    const float t = s * (float)half_hc;
    const float cc = (float)so_round_to(prec, dc * hc);
    return (double)(t + cc);
  }
  const double s = so_round16(reli - relj);
  const double t = so_round16(s * half_hc);
  const double cc = so_round16((double)dc * hc);
  return so_round16(t + cc);
}

static double finish(int prec, double acc) { /* nnps.cpp:340-346 */
  if (prec == SO_FP64) return sqrt(acc);
  if (prec == SO_FP32) return (double)sqrtf((float)acc);
  return so_round16(sqrt(acc));
}

/* nnps.cpp:283-416 */
int so_rcll(const so_grid* g, int64_t n, const double* const* rel, const int32_t* const* cell,
            const int32_t* items, const int32_t* start, int prec, so_table* out) {
  const int dim = g->dim;
  const double cutoff = so_round_to(prec, g->cutoff_norm);
  double half_hc[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < dim; ++k) half_hc[k] = so_round_to(prec, 0.5 * g->hc[k]);
  double** rp = round_coords(dim, n, rel, prec); /* rel_prec, :303-306 */
  vec32 buf = {0};
  table_begin(out, n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rb = buf.len;
    int32_t ci[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) ci[k] = cell[k][i];
    const int oy_lo = dim > 1 ? -1 : 0, oy_hi = dim > 1 ? 1 : 0;
    const int oz_lo = dim > 2 ? -1 : 0, oz_hi = dim > 2 ? 1 : 0;
    for (int oz = oz_lo; oz <= oz_hi; ++oz)
      for (int oy = oy_lo; oy <= oy_hi; ++oy)
        for (int ox = -1; ox <= 1; ++ox) {
          const int off[3] = {ox, oy, oz};
          int32_t c[3] = {0, 0, 0};
          int dc[3] = {0, 0, 0};
          int skip = 0;
          for (int k = 0; k < dim && !skip; ++k) {
            int32_t ck = ci[k] + off[k];
            dc[k] = -off[k]; /* minimum image, :359-362 */
            if (ck < 0 || ck >= g->counts[k]) {
              if (g->periodic[k] && g->counts[k] > 2)
                ck = (ck + g->counts[k]) % g->counts[k];
              else
                skip = 1;
            }
            c[k] = ck;
          }
          if (skip) continue;
          const int64_t cl = linear_cell(g, c);
          for (int64_t s = start[cl]; s < start[cl + 1]; ++s) {
            const int32_t j = items[s];
            if (j == i) continue;
            double acc = 0.0;
            for (int k = 0; k < dim; ++k) {
              const double d = axis_term(prec, rp[k][i], rp[k][j], dc[k], g->hc[k], half_hc[k]);
              if (prec == SO_FP64)
                acc += d * d;
              else if (prec == SO_FP32)
                acc = (double)((float)acc + (float)d * (float)d);
              else
                acc = so_round16(acc + so_round16(d * d));
            }
            if (finish(prec, acc) < cutoff) vpush(&buf, j);
          }
        }
    table_end_row(out, &buf, i, rb);
  }
  table_finish(out, &buf);
  free_coords(rp);
  return 0;
}

/* cell_grid.cpp:135-178 */
double so_rel_distance(const so_grid* g, const double* const* rel, const int32_t* const* cell,
                       int64_t i, int64_t j, int prec) {
  if (prec == SO_FP64) {
    double acc = 0.0;
    for (int k = 0; k < g->dim; ++k) {
      const double hc = g->hc[k];
      const double cc = (double)(cell[k][i] - cell[k][j]) * hc;
      const double d = (rel[k][i] - rel[k][j]) * (0.5 * hc) + cc;
      acc += d * d;
    }
    return sqrt(acc);
  }
  if (prec == SO_FP32) {
    float acc = 0.0f;
    for (int k = 0; k < g->dim; ++k) {
      const double hc = g->hc[k];
      const float ri = (float)rel[k][i];
      const float rj = (float)rel[k][j];
      const float half_hc = (float)(0.5 * hc);
      const float cc = (float)((double)(cell[k][i] - cell[k][j]) * hc);
      const float d = (ri - rj) * half_hc + cc;
      acc += d * d;
    }
    return (double)sqrtf(acc);
  }
  double acc = 0.0;
  for (int k = 0; k < g->dim; ++k) {
    const double hc = g->hc[k];
    const double ri = so_round16(rel[k][i]);
    const double rj = so_round16(rel[k][j]);
    const double half_hc = so_round16(0.5 * hc);
    const double cc = so_round16((double)(cell[k][i] - cell[k][j]) * hc);
    const double s = so_round16(ri - rj);
    const double t = so_round16(s * half_hc);
    const double d = so_round16(t + cc);
    acc = so_round16(acc + so_round16(d * d));
  }
  return so_round16(sqrt(acc));
}

/* ---- SPH gradient on a neighbour table (test infrastructure) --------------------
 * make_kernel (kernel.hpp:17-29), kernel_dwdr (kernel.hpp:41-49), kernel_grad
 * (kernel.hpp:53-64) and grad_normalized (gradient.cpp:44-82): FP64, each row
 * summed in table order, built without contraction like the reference. */
static double so_kernel_alpha(int dim, double h) {
  const double pi = 3.14159265358979323846; /* std::numbers::pi */
  if (dim == 1) return 1.0 / h;
  if (dim == 2) return 15.0 / (7.0 * pi * h * h);
  return 3.0 / (2.0 * pi * h * h * h);
}

static double so_kernel_dwdr(double R, double alpha) {
  if (R < 1.0) return alpha * (-2.0 * R + 1.5 * R * R);
  if (R < 2.0) {
    const double t = 2.0 - R;
    return -alpha * (0.5 * t * t);
  }
  return 0.0;
}

int64_t so_grad_normalized(int dim, int64_t n, const double* const* x, const double* f,
                           const int64_t* offsets, const int32_t* items, double h,
                           double** g) {
  const double alpha = so_kernel_alpha(dim, h);
  int64_t degenerate = 0;
  for (int64_t i = 0; i < n; ++i) {
    double num[3] = {0.0, 0.0, 0.0}, den[3] = {0.0, 0.0, 0.0}, scale[3] = {0.0, 0.0, 0.0};
    for (int64_t e = offsets[i]; e < offsets[i + 1]; ++e) {
      const int32_t j = items[e];
      double dx[3] = {0.0, 0.0, 0.0};
      for (int k = 0; k < dim; ++k) dx[k] = x[k][i] - x[k][j];
      double gw[3] = {0.0, 0.0, 0.0};
      double r2 = 0.0;
      for (int k = 0; k < dim; ++k) r2 += dx[k] * dx[k];
      const double r = sqrt(r2);
      if (r != 0.0) {
        const double R = r / h;
        const double sc = so_kernel_dwdr(R, alpha) / (h * r);
        for (int k = 0; k < dim; ++k) gw[k] = sc * dx[k];
      }
      const double df = f[j] - f[i];
      for (int k = 0; k < dim; ++k) {
        num[k] += df * gw[k];
        den[k] += -dx[k] * gw[k];
        scale[k] += fabs(dx[k] * gw[k]);
      }
    }
    for (int k = 0; k < dim; ++k) {
      if (fabs(den[k]) < 1e-14 * (scale[k] > 0.0 ? scale[k] : 1.0)) {
        g[k][i] = 0.0;
        ++degenerate;
      } else {
        g[k][i] = num[k] / den[k];
      }
    }
  }
  return degenerate;
}

/* update_relative (cell_grid.cpp:180-212) for particles [0, n): returns 0, or
 * 1 + ((i << 3) | (k << 1) | kind) for the first (particle, axis) that throws
 * (kind 0: displacement skips a cell, 1: particle leaves the grid), with the
 * particles before it updated, as the reference leaves them. */
int64_t so_update_relative(const so_grid* g, int64_t n, double** rel, int32_t** cell,
                           const double* const* dx, int prec) {
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < g->dim; ++k) {
      const double edge = g->edge[k];
      if (!(fabs(dx[k][i]) < edge)) return 1 + ((i << 3) | ((int64_t)k << 1));
      const double inc = so_round_to(prec, 2.0 * dx[k][i] / edge);
      double r = so_round_to(prec, rel[k][i] + inc);
      int32_t c = cell[k][i];
      if (r > 1.0) {
        r -= 2.0;
        ++c;
        if (c >= g->counts[k]) {
          if (g->periodic[k]) c = 0;
          else return 1 + ((i << 3) | ((int64_t)k << 1) | 1);
        }
      } else if (r < -1.0) {
        r += 2.0;
        --c;
        if (c < 0) {
          if (g->periodic[k]) c = g->counts[k] - 1;
          else return 1 + ((i << 3) | ((int64_t)k << 1) | 1);
        }
      }
      rel[k][i] = r;
      cell[k][i] = c;
    }
  }
  return 0;
}
