/*
 * sphx_cuda.h -- the C ABI of the B200 (sm_100a) NNPS library (libsphx_cuda.so).
 *
 * This is the drop-in boundary for the reference's neighbour-search hot path.
 * Plain C types only: pointers, sizes, a POD grid descriptor. No torch, no C++.
 * Each entry point names the reference interface it replaces (paths relative to
 * the reference's proj/ tree):
 *
 *   sphx_rcll            <- NeighborTable rcll(const RelCoords&, const CellGrid&,
 *                                              Precision)           nnps.hpp:41, nnps.cpp:283-416
 *   sphx_cell_link_list  <- NeighborTable cell_link_list(const ParticleSystem&,
 *                                              const CellGrid&, Precision)
 *                                                                   nnps.hpp:36, nnps.cpp:174-281
 *   sphx_all_list        <- NeighborTable all_list(const ParticleSystem&, Precision)
 *                                                                   nnps.hpp:31, nnps.cpp:128-172
 *   sphx_rebin           <- void CellGrid::rebin(const ParticleSystem&)
 *                                                                   cell_grid.hpp:86, cell_grid.cpp:66-108
 *   sphx_build_rel_coords<- RelCoords build_rel_coords(const ParticleSystem&, CellGrid&)
 *                                                                   cell_grid.hpp:120, cell_grid.cpp:114-133
 *   sphx_rebuild_members <- void CellGrid::rebuild_members(const RelCoords&)
 *                                                                   cell_grid.hpp:89, cell_grid.cpp:86-108
 *   sphx_table_copy / sphx_table_stream
 *                        <- (ownership hand-off of the returned NeighborTable, nnps.hpp:16-26)
 *   sphx_update_relative(_device)
 *                        <- void update_relative(RelCoords&, size_t i, const std::array<double,3>&,
 *                                                const CellGrid&, Precision) for all i
 *                                                                   cell_grid.hpp:134, cell_grid.cpp:180-212
 *   sphx_rebuild_members_device <- CellGrid::rebuild_members on device memory
 *   sphx_rcll_grad_normalized(_device)
 *                        <- grad_normalized(f, ps, rcll(rc, grid, fp16), kp) fused
 *                                                                   gradient.cpp:44-82, dynamics.cpp:145-155
 *   sphx_step_mixed_device <- StepResult step_mixed(MixedState&, const StepConfig&)
 *                                                                   dynamics.cpp:136-203
 *   sphx_table_distances / sphx_rcll_distances_device
 *                        <- double rel_distance(const RelCoords&, size_t i, size_t j,
 *                                               const CellGrid&, Precision) for every entry
 *                                                                   cell_grid.hpp:128, cell_grid.cpp:135-178
 *   sphx_last_error      <- the what() of the exception the reference would throw
 *   (the reference's own C-style template is detail::range_f16_rel_2d & co,
 *    detail/nnps_batch.hpp:13-41)
 *
 * Output contract (nnps.hpp:13-26): CSR with int64 offsets[n+1], int32 items,
 * rows in original particle order, each row ascending, no self entries;
 * bit-identical to the reference CPU implementation at the same precision.
 *
 * Error convention: every function returns SPHX_OK (0) or a negative code whose
 * class mirrors the C++ exception the reference throws (the C++ shim rethrows the
 * same type with sphx_last_error() as the message). There is no CPU fallback: a
 * missing CUDA device or a device that is not sm_100 is SPHX_ERR_CUDA.
 *
 * Host-memory entry points are synchronous. *_device entry points take device
 * pointers and are ordered on the context's stream (sphx_set_stream).
 */
#ifndef SPHX_CUDA_H
#define SPHX_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHX_OK 0
#define SPHX_ERR_GENERIC (-1)          /* std::exception */
#define SPHX_ERR_INVALID_ARGUMENT (-2) /* std::invalid_argument */
#define SPHX_ERR_OUT_OF_RANGE (-3)     /* std::out_of_range */
#define SPHX_ERR_RUNTIME (-4)          /* std::runtime_error */
#define SPHX_ERR_CUDA (-5)             /* no usable sm_100 device / CUDA failure */
#define SPHX_ERR_CAPACITY (-6)         /* device table capacity too small (device API) */

/* Precision (binary16.hpp:87): arithmetic precision of the distance pipeline. */
#define SPHX_FP64 0
#define SPHX_FP32 1
#define SPHX_FP16 2

/* POD image of the CellGrid/Domain state the NNPS path consumes
 * (cell_grid.hpp:55-96, domain.hpp:36-43). Axes >= dim are ignored. */
typedef struct sphx_grid_desc {
  int32_t dim;          /* 1..3 */
  int32_t counts[3];    /* CellGrid::count(k) */
  int32_t periodic[3];  /* CellGrid::periodic(k) */
  int32_t reserved;
  double hc[3];         /* CellGrid::hc(k): normalised cell edge 2*edge/h_d */
  double origin[3];     /* CellGrid::origin_norm(k) */
  double cutoff_norm;   /* CellGrid::cutoff_norm(): 2*radius/h_d */
  double radius_phys;   /* CellGrid::radius_phys(): 2h */
  double lo[3];         /* Domain::lo */
  double hi[3];         /* Domain::hi */
} sphx_grid_desc;

/* Fill a descriptor exactly as CellGrid's constructor would (cell_grid.cpp:9-34).
 * Returns SPHX_ERR_INVALID_ARGUMENT for radius <= 0 or a periodic axis with < 3 cells. */
int sphx_grid_init(sphx_grid_desc* g, int32_t dim, const double lo[3], const double hi[3],
                   double radius, const int32_t periodic[3]);

typedef struct sphx_context sphx_context;

/* Create a context on `device` (-1 = current). Fails with SPHX_ERR_CUDA when no
 * sm_100 device is present. */
int sphx_create(int device, sphx_context** out);
void sphx_destroy(sphx_context* ctx);
/* Message of the last error on this thread ("" if none). */
const char* sphx_last_error(void);
/* Use an external stream (a cudaStream_t, e.g. torch's current stream); NULL
 * restores the context's own stream. */
int sphx_set_stream(sphx_context* ctx, void* cuda_stream);
/* Kernel launches issued by this context so far (diagnostics / bench). */
int64_t sphx_launch_count(const sphx_context* ctx);

/* ---------------- drop-in, host memory, synchronous ---------------- */

/* rcll(rc, grid, prec). rel[k]/cell[k] are RelCoords::rel[k]/cell[k] (n entries,
 * k < dim); items/cell_start are CellGrid::items() (n_items) and cell_start()
 * (cell_total+1). On success *total = number of (directed) pairs; the table stays
 * on the device until sphx_table_copy. */
int sphx_rcll(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
              const double* const rel[3], const int32_t* const cell[3], int64_t n_items,
              const int32_t* items, const int32_t* cell_start, int32_t precision,
              int64_t* total);

/* cell_link_list(ps, grid, prec). x[k] = ParticleSystem::x(k), h = ps.h(),
 * cell_of[i] = CellGrid::cell_of(i). */
int sphx_cell_link_list(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                        const double* const x[3], double h, int64_t n_items,
                        const int32_t* items, const int32_t* cell_start,
                        const int32_t* cell_of, int32_t precision, int64_t* total);

/* all_list(ps, prec): O(N^2) reference backend. */
int sphx_all_list(sphx_context* ctx, int32_t dim, int64_t n, const double* const x[3], double h,
                  int32_t precision, int64_t* total);

/* Copy the last table computed on this context to host buffers: offsets[n+1],
 * items[total]. Either pointer may be NULL. */
int sphx_table_copy(sphx_context* ctx, int64_t* offsets, int32_t* items);

/* Stream the last table to a consumer that builds its own container (the
 * drop-in's std::vector, filled by insertion instead of a zero-fill plus a copy):
 * sink(user, part, data, bytes) is called in order for part 0 (offsets, int64)
 * and then part 1 (items, int32) with consecutive chunks of whole elements; the
 * next chunk's DMA overlaps the sink. A nonzero sink result stops the copy with
 * SPHX_ERR_RUNTIME. (Same hand-off as sphx_table_copy, nnps.hpp:16-26.) */
typedef int (*sphx_table_sink)(void* user, int32_t part, const void* data, int64_t bytes);
int sphx_table_stream(sphx_context* ctx, sphx_table_sink sink, void* user);

/* CellGrid::rebin(ps): cell_of[n], cell_start[cell_total+1], items[n]. A particle
 * outside the grid -> SPHX_ERR_OUT_OF_RANGE "particle <i> lies outside the grid"
 * (the lowest such index, as the reference's serial loop reports). */
int sphx_rebin(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
               const double* const x[3], int32_t* cell_of, int32_t* cell_start, int32_t* items);

/* build_rel_coords(ps, grid): rel[k][n], cell[k][n] plus the rebuilt membership. */
int sphx_build_rel_coords(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                          const double* const x[3], double* const rel[3], int32_t* const cell[3],
                          int32_t* cell_of, int32_t* cell_start, int32_t* items);

/* CellGrid::rebuild_members(rc): membership from per-axis cells. */
int sphx_rebuild_members(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                         const int32_t* const cell[3], int32_t* cell_of, int32_t* cell_start,
                         int32_t* items);

/* ---------------- device-resident, stream-ordered ---------------- */

/* Same computation as sphx_rcll with every pointer in device memory. The table is
 * written to d_offsets[n+1] / d_items[capacity]; d_offsets[n] always receives the
 * exact total. If it exceeds `capacity`, items are not written and the call must
 * be repeated with a larger buffer (the host can read d_offsets[n]).
 * Does not synchronise. */
int sphx_rcll_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                     const double* const d_rel[3], const int32_t* const d_cell[3],
                     const int32_t* d_items, const int32_t* d_cell_start, int32_t precision,
                     int64_t* d_offsets, int32_t* d_items_out, int64_t capacity);

int sphx_cell_link_list_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                               const double* const d_x[3], double h, const int32_t* d_items,
                               const int32_t* d_cell_start, const int32_t* d_cell_of,
                               int32_t precision, int64_t* d_offsets, int32_t* d_items_out,
                               int64_t capacity);

/* Device binning + RCLL encoding: build_rel_coords on device pointers. Out-of-grid
 * particles are not checked (the reference's build_rel_coords does not check). */
int sphx_build_rel_coords_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                 const double* const d_x[3], double* const d_rel[3],
                                 int32_t* const d_cell[3], int32_t* d_cell_of,
                                 int32_t* d_cell_start, int32_t* d_items);

/* Device rebin; *d_bad receives the lowest out-of-grid particle index or -1. */
int sphx_rebin_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                      const double* const d_x[3], int32_t* d_cell_of, int32_t* d_cell_start,
                      int32_t* d_items, int64_t* d_bad);

/* ---------------- slab decomposition (one process per GPU) ----------------
 * No reference counterpart: the reference is single-process.
 * A rank owns the cell layers [L0, L1) of the global grid along `axis` (the
 * slowest axis) plus one halo layer on each side received from its neighbours.
 * Its local grid is the global grid with counts[axis] = L1 - L0 + 2 and
 * periodic[axis] = 0; local layer l is global layer (L0 - 1 + l) mod G. */

/* build_rel_coords on the slab: each particle is located on the GLOBAL grid
 * (global normalisation, rel and cell choice bit-identical to the one-GPU run),
 * then its `axis` layer becomes (c - layer0) mod G and CSR is built over `local`. */
int sphx_build_rel_coords_window_device(sphx_context* ctx, const sphx_grid_desc* global,
                                        const sphx_grid_desc* local, int32_t axis,
                                        int32_t layer0, int64_t n, const double* const d_x[3],
                                        double* const d_rel[3], int32_t* const d_cell[3],
                                        int32_t* d_cell_of, int32_t* d_cell_start,
                                        int32_t* d_items);

/* Multi-GPU slab assembly after a halo exchange (no binning). A rank holds its
 * owned particles in CSR order in slots [0, n_own) with d_owned_start = the CSR
 * start over its owned layers (nl * CL + 1 entries, from 0; CL = cells per
 * layer of the slab axis, the slowest axis of linear_cell, cell_grid.hpp:74-78).
 * The neighbours' boundary layers arrive as contiguous RelCoords / id slices in
 * slots [slot_below, ...) and [slot_above, ...) together with their slices of
 * cell_start (CL + 1 entries, any base; NULL = a wall, no halo). Writes the
 * local CellGrid of local->counts[axis] = nl + 2 layers (lower halo, owned, upper
 * halo): d_cell_start, d_items (CSR position -> slot) and RelCoords::cell of the
 * halo slots (their cell; the slab-axis coordinate 0 or nl + 1). Sizes are read
 * on the device: stream-ordered, no synchronisation. */
int sphx_slab_assemble_device(sphx_context* ctx, const sphx_grid_desc* local, int32_t axis,
                              int64_t n_own, int64_t slot_below, int64_t slot_above,
                              int64_t n_slots, const int32_t* d_owned_start,
                              const int32_t* d_recv_below, const int32_t* d_recv_above,
                              int32_t* d_cell_start, int32_t* d_items, int32_t* const d_cell[3]);

/* RCLL rows for particles [row0, row0 + nrows) only (the owned particles of a
 * slab); neighbour ids are written as d_ids[j] (global ids; NULL = local j).
 * d_offsets has nrows + 1 entries; d_offsets[nrows] = exact total. */
int sphx_rcll_rows_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                          const double* const d_rel[3], const int32_t* const d_cell[3],
                          const int32_t* d_items, const int32_t* d_cell_start, int32_t precision,
                          const int32_t* d_ids, int64_t row0, int64_t nrows, int64_t* d_offsets,
                          int32_t* d_items_out, int64_t capacity);

/* Per-pair distances of an RCLL table (device memory, stream-ordered): d_dist[e]
 * is the value rcll compared against the cutoff for entry e = (i, items[e]) --
 * finish(acc) at the precision with the minimum-image cell offset
 * (nnps.cpp:321-346, 359-362); for pairs that do not wrap a periodic axis it is
 * exactly rel_distance(rc, i, j, grid, prec) (cell_grid.hpp:128, cell_grid.cpp:135-178). */
int sphx_rcll_distances_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                               const double* const d_rel[3], const int32_t* const d_cell[3],
                               int32_t precision, const int64_t* d_offsets,
                               const int32_t* d_items, double* d_dist);
/* The same for the table of the last sphx_rcll call on this context (its staged
 * inputs); dist receives sphx_rcll's *total doubles (host memory, synchronous). */
int sphx_table_distances(sphx_context* ctx, const sphx_grid_desc* grid, int32_t precision,
                         double* dist);

/* RCLL maintenance: update_relative(rc, i, dx[i], grid, prec)
 * (cell_grid.hpp:134, cell_grid.cpp:180-212) for every particle i < n at once --
 * the Eq. 8 migration step_mixed applies after the drift (dynamics.cpp:191-198).
 * Errors are the reference's std::runtime_error texts ("displacement skips a cell
 * on axis k", "particle leaves the grid on axis k") for the lowest offending
 * particle; rel/cell are then unspecified (the reference leaves them partially
 * updated). Host memory, synchronous. */
int sphx_update_relative(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                         double* const rel[3], int32_t* const cell[3], const double* const dx[3],
                         int32_t precision);
/* Device memory, stream-ordered: *d_status = ~0 on success, else
 * (particle << 3) | (axis << 1) | kind (0: skips a cell, 1: leaves the grid). */
int sphx_update_relative_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                double* const d_rel[3], int32_t* const d_cell[3],
                                const double* const d_dx[3], int32_t precision,
                                unsigned long long* d_status);
/* CellGrid::rebuild_members(rc) on device memory (cell_grid.cpp:86-108). */
int sphx_rebuild_members_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                const int32_t* const d_cell[3], int32_t* d_cell_of,
                                int32_t* d_cell_start, int32_t* d_items);

/* Fused FP16 RCLL -> grad_normalized: the mixed step's
 *   grad_normalized(f, ps, rcll(rel, grid, fp16), make_kernel(h, dim))
 * (dynamics.cpp:145-155, gradient.hpp:27, gradient.cpp:44-82, kernel.hpp:17-64)
 * without materialising the neighbour table. g[k] receives GradField::g[k] (n
 * doubles, particle order) and *degenerate GradField::degenerate_count; both are
 * bit-identical to the reference. x[k] = ParticleSystem::x(k), f the field.
 * precision must be SPHX_FP16 and dim 2 or 3. */
int sphx_rcll_grad_normalized(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                              const double* const rel[3], const int32_t* const cell[3],
                              int64_t n_items, const int32_t* items, const int32_t* cell_start,
                              int32_t precision, const double* const x[3], const double* f,
                              double h, double* const g[3], int64_t* degenerate);
/* Device-memory variant (stream-ordered); *d_degenerate is overwritten. */
int sphx_rcll_grad_normalized_device(sphx_context* ctx, const sphx_grid_desc* grid, int64_t n,
                                     const double* const d_rel[3], const int32_t* const d_cell[3],
                                     const int32_t* d_items, const int32_t* d_cell_start,
                                     int32_t precision, const double* const d_x[3],
                                     const double* d_f, double h, double* const d_g[3],
                                     unsigned long long* d_degenerate);

/* ---------------- the mixed-precision time step ----------------
 * step_mixed(MixedState&, const StepConfig&) (dynamics.hpp:84-107, dynamics.cpp:136-203)
 * on device memory: the approach's neighbour search (I: cell_link_list FP64, II:
 * cell_link_list FP16, III: rcll FP16), apply_eos, assemble_newtonian_stress, the
 * FP64 rates (rhs_density / rhs_momentum / rhs_energy), the symplectic Euler
 * kick-drift with periodic wrap, then update_relative (FP64) + rebuild_members
 * (III) or rebin (I, II). Every field is bit-identical to the reference. The
 * step's table goes to d_offsets / d_items_out; when it needs more than
 * `capacity` entries the call returns SPHX_ERR_CAPACITY with *total set and the
 * state untouched. StepConfig::pre_force (a C++ callback) has no counterpart:
 * run it between steps. On an update_relative / rebin error every particle has
 * already moved (the reference stops at the first offending particle). */
#define SPHX_APPROACH_I 0
#define SPHX_APPROACH_II 1
#define SPHX_APPROACH_III 2

typedef struct sphx_step_config { /* StepConfig (dynamics.hpp:84-96) */
  double dt, c_sound, rho0, mu;
  double body_force[3];
  int64_t n_moving;       /* 0: every particle moves */
  int32_t evolve_density; /* the reference's default is 1 */
  int32_t compute_energy;
} sphx_step_config;

typedef struct sphx_mixed_state_device { /* MixedState (dynamics.hpp:71-82), device memory */
  int64_t n;
  double h;                            /* ParticleSystem::h() */
  double* x[3];
  double* v[3];
  const double* m;
  double* rho;
  double* p;
  double* e;
  double* rel[3];                      /* RelCoords (approach III) */
  int32_t* cell[3];
  int32_t* cell_of;                    /* CellGrid membership (CSR) */
  int32_t* cell_start;
  int32_t* items;
} sphx_mixed_state_device;

int sphx_step_mixed_device(sphx_context* ctx, const sphx_grid_desc* grid, int32_t approach,
                           const sphx_mixed_state_device* state, const sphx_step_config* cfg,
                           int64_t* d_offsets, int32_t* d_items_out, int64_t capacity,
                           double* max_dx, int64_t* total);

/* Un-jittered build_lattice sites with ids [id0, id0 + count) written to d_x
 * (x_k = lo_k + (c_k + 0.5) ds, bit-identical to particle_system.cpp:53). */
int sphx_lattice_device(sphx_context* ctx, int32_t dim, const double lo[3], const double hi[3],
                        double ds, int64_t id0, int64_t count, double* const d_x[3]);

/* ---------------- synthetic inputs ---------------- */
/* build_lattice(Domain::box(dim, lo, hi), ds, jitter, seed) (particle_system.hpp:66,
 * particle_system.cpp:31-62): cell-centred lattice, x fastest, per-axis jitter
 * jitter*ds*(2u-1) from mt19937_64. Call with x0 == NULL to get *n only. */
int sphx_build_lattice(int32_t dim, const double lo[3], const double hi[3], double ds,
                       double jitter, uint64_t seed, int64_t* n, double* x0, double* x1,
                       double* x2);
/* build_random_uniform (particle_system.hpp:70, particle_system.cpp:64-77). */
int sphx_build_random_uniform(int32_t dim, const double lo[3], const double hi[3], int64_t n,
                              uint64_t seed, double* ds, double* x0, double* x1, double* x2);

/* FNV-1a 64 digest of a CSR table (offsets as u64, then items as u32): the
 * golden-vector hash of tests/golden/golden.json. Host memory, pure host code. */
uint64_t sphx_table_hash(const int64_t* offsets, int64_t n, const int32_t* items, int64_t total);

/* Per-kernel timing of the last sphx_*_device NNPS call when timing is enabled
 * (CUDA events on the launching stream): encode and sweep in milliseconds. */
int sphx_enable_timing(sphx_context* ctx, int on);
int sphx_last_timing(sphx_context* ctx, float* encode_ms, float* sweep_ms);

#ifdef __cplusplus
}
#endif
#endif /* SPHX_CUDA_H */
