/* TEST INFRASTRUCTURE ONLY -- the CPU checker for the NNPS hot path.
 *
 * Plain-C restatement of the reference sphx NNPS algorithm (CLL and RCLL at
 * FP64/FP32/FP16, dim 1..3, periodic axes) plus the inputs it consumes (lattice
 * and uniform generators, cell grid, locate, CSR binning, RCLL encoding). Each
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj). Single-threaded, scalar, no intrinsics.
 *
 * Parity: pinned against the reference compiled in place (oracle/_ref, see
 * oracle/Makefile) and the golden vectors in tests/golden/ produced from it.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker / the CPU baseline. */
#ifndef SPHX_ORACLE_H
#define SPHX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SO_FP64 = 0, SO_FP32 = 1, SO_FP16 = 2 };

/* binary16 (binary16.cpp:12-74) and the rounding model (binary16.hpp:85-103). */
uint16_t so_f16_from_f64(double x);
double so_f16_to_f64(uint16_t b);
double so_round16(double x);
double so_round_to(int prec, double x);

/* mt19937_64 with the reference's hand-rolled U[0,1) (rng.hpp:11-33). */
typedef struct so_rng {
  uint64_t mt[312];
  int idx;
} so_rng;
void so_rng_seed(so_rng* r, uint64_t seed);
uint64_t so_rng_next(so_rng* r);
double so_rng_uniform01(so_rng* r);
uint64_t so_rng_below(so_rng* r, uint64_t n);

/* Generators (particle_system.cpp:31-77). x0/x1/x2 hold n doubles each
 * (unused axes may be NULL). so_lattice_count gives n for the lattice. */
int64_t so_lattice_count(int dim, const double* lo, const double* hi, double ds);
int so_build_lattice(int dim, const double* lo, const double* hi, double ds, double jitter,
                     uint64_t seed, double* x0, double* x1, double* x2);
/* returns ds = (volume/n)^(1/dim) */
double so_build_random(int dim, const double* lo, const double* hi, int64_t n, uint64_t seed,
                       double* x0, double* x1, double* x2);

/* build_gapped_random (experiments.cpp:55-112), 2-D: 0 or -4 (stalled). */
int so_build_gapped_random(const double* lo, const double* hi, int64_t n, double cutoff,
                           double width, uint64_t seed, double* x0, double* x1);

/* Uniform cell grid (cell_grid.cpp:9-34). */
typedef struct so_grid {
  int dim;
  int counts[3];
  int periodic[3];
  int64_t total;
  double radius, cutoff_norm, hd;
  double edge[3], hc[3], origin[3], lo[3], hi[3];
} so_grid;
int so_grid_init(so_grid* g, int dim, const double* lo, const double* hi, double radius,
                 const int* periodic);
void so_locate(const so_grid* g, const double* xn, int32_t* cell, double* rel);
/* rebin (cell_grid.cpp:66-108): fills cell_of[n], start[total+1], items[n].
 * Returns 0, or -3 with *bad = first particle outside the grid. */
int so_rebin(const so_grid* g, int64_t n, const double* const* x, int32_t* cell_of,
             int32_t* start, int32_t* items, int64_t* bad);
/* build_rel_coords + rebuild_members (cell_grid.cpp:86-133). */
void so_build_rel(const so_grid* g, int64_t n, const double* const* x, double** rel,
                  int32_t** cell, int32_t* cell_of, int32_t* start, int32_t* items);

/* CSR neighbour table (nnps.hpp:16-26). */
typedef struct so_table {
  int64_t n;
  int64_t total;
  int64_t* offsets; /* n+1 */
  int32_t* items;   /* total */
} so_table;
void so_table_free(so_table* t);
uint64_t so_table_hash(const so_table* t);

/* rcll (nnps.cpp:283-416). rel/cell in particle order, items/start = grid CSR. */
int so_rcll(const so_grid* g, int64_t n, const double* const* rel, const int32_t* const* cell,
            const int32_t* items, const int32_t* start, int prec, so_table* out);
/* cell_link_list (nnps.cpp:174-281). own cell from cell_of (grid.cell_of). */
int so_cll(const so_grid* g, int64_t n, const double* const* x, double h,
           const int32_t* cell_of, const int32_t* items, const int32_t* start, int prec,
           so_table* out);
/* all_list (nnps.cpp:128-172). */
int so_all_list(int dim, int64_t n, const double* const* x, double h, int prec, so_table* out);
/* rel_distance (cell_grid.cpp:135-178). */
double so_rel_distance(const so_grid* g, const double* const* rel, const int32_t* const* cell,
                       int64_t i, int64_t j, int prec);

/* update_relative (cell_grid.cpp:180-212) over particles [0, n); 0 or
 * 1 + ((i << 3) | (axis << 1) | kind) for the first throw. */
int64_t so_update_relative(const so_grid* g, int64_t n, double** rel, int32_t** cell,
                           const double* const* dx, int prec);

/* grad_normalized (gradient.cpp:44-82) with the cubic B-spline gradient
 * (kernel.hpp:17-64): g[k][i] for every row of the table; returns the number of
 * degenerate (particle, axis) pairs. */
int64_t so_grad_normalized(int dim, int64_t n, const double* const* x, const double* f,
                           const int64_t* offsets, const int32_t* items, double h,
                           double** g);

#ifdef __cplusplus
}
#endif
#endif
