// TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// extern "C" face of the *unmodified* reference sphx library, compiled from the
// sources where they lie under /root/reference/proj (see oracle/Makefile). It
// lets pytest, the golden-vector generator and bench.py's cpu_baseline /
// --impl reference arm drive the reference's own NNPS implementation through
// ctypes. Every entry point catches C++ exceptions and returns a negative code
// with the message copied into a caller buffer, so the error behaviour of the
// reference (nnps.cpp:184, :298; cell_grid.cpp:77) can be compared verbatim.
//
// Handles are opaque heap objects owned by the caller (ref_free_*).

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "sphx/binary16.hpp"
#include "sphx/cell_grid.hpp"
#include "sphx/detail/nnps_batch.hpp"
#include "sphx/dynamics.hpp"
#include "sphx/gradient.hpp"
#include "sphx/nnps.hpp"
#include "sphx/particle_system.hpp"

namespace {

thread_local char g_err[512];

void set_err(const char* what) {
  std::strncpy(g_err, what, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

// Exception class -> stable negative code (mirrors sphx_cuda.h's codes).
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range& e) {
    set_err(e.what());
    return -3;
  } catch (const std::invalid_argument& e) {
    set_err(e.what());
    return -2;
  } catch (const std::runtime_error& e) {
    set_err(e.what());
    return -4;
  } catch (const std::exception& e) {
    set_err(e.what());
    return -1;
  }
}

sphx::Precision prec_of(int p) {
  switch (p) {
    case 0: return sphx::Precision::fp64;
    case 1: return sphx::Precision::fp32;
    default: return sphx::Precision::fp16;
  }
}

std::uint64_t fnv_table(const sphx::NeighborTable& t) {
  std::uint64_t x = 1469598103934665603ull;
  for (const auto o : t.offsets) {
    x ^= static_cast<std::uint64_t>(o);
    x *= 1099511628211ull;
  }
  for (const auto j : t.items) {
    x ^= static_cast<std::uint32_t>(j);
    x *= 1099511628211ull;
  }
  return x;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

int ref_batch_kernels_available() { return sphx::detail::batch_kernels_available() ? 1 : 0; }

void ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// ---- binary16 ---------------------------------------------------------------
std::uint16_t ref_f16_from_f64(double x) { return sphx::Binary16::from_f64(x).bits(); }
double ref_f16_to_f64(std::uint16_t b) { return sphx::Binary16::from_bits(b).to_f64(); }
double ref_round_to(int prec, double x) { return sphx::round_to(prec_of(prec), x); }
std::uint16_t ref_sqrt16(std::uint16_t b) {
  return sphx::sqrt16(sphx::Binary16::from_bits(b)).bits();
}

// ---- particle systems ---------------------------------------------------------
void* ref_ps_lattice(int dim, const double* lo, const double* hi, double ds, double jitter,
                     std::uint64_t seed) {
  void* out = nullptr;
  const int rc = guarded([&] {
    sphx::Domain d = sphx::Domain::box(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]});
    out = new sphx::ParticleSystem(sphx::build_lattice(d, ds, jitter, seed));
  });
  return rc == 0 ? out : nullptr;
}

void* ref_ps_random(int dim, const double* lo, const double* hi, std::uint64_t n,
                    std::uint64_t seed) {
  void* out = nullptr;
  const int rc = guarded([&] {
    sphx::Domain d = sphx::Domain::box(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]});
    out = new sphx::ParticleSystem(sphx::build_random_uniform(d, n, seed));
  });
  return rc == 0 ? out : nullptr;
}

// Arbitrary positions (used to replay fixtures and edge cases).
void* ref_ps_from_arrays(int dim, const double* lo, const double* hi, double ds,
                         std::uint64_t n, const double* x0, const double* x1,
                         const double* x2) {
  void* out = nullptr;
  const int rc = guarded([&] {
    sphx::Domain d = sphx::Domain::box(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]});
    auto* ps = new sphx::ParticleSystem(d, ds, n, 1.0);
    const double* src[3] = {x0, x1, x2};
    for (int k = 0; k < dim; ++k) std::copy(src[k], src[k] + n, ps->x(k).begin());
    out = ps;
  });
  return rc == 0 ? out : nullptr;
}

std::uint64_t ref_ps_size(void* ps) { return static_cast<sphx::ParticleSystem*>(ps)->size(); }
double ref_ps_h(void* ps) { return static_cast<sphx::ParticleSystem*>(ps)->h(); }
void ref_ps_set_h(void* ps, double h) { static_cast<sphx::ParticleSystem*>(ps)->set_h(h); }
void ref_ps_get_x(void* ps, int k, double* out) {
  const auto& x = static_cast<sphx::ParticleSystem*>(ps)->x(k);
  std::copy(x.begin(), x.end(), out);
}
void ref_ps_set_x(void* ps, int k, const double* in) {
  auto& x = static_cast<sphx::ParticleSystem*>(ps)->x(k);
  std::copy(in, in + x.size(), x.begin());
}
void ref_free_ps(void* ps) { delete static_cast<sphx::ParticleSystem*>(ps); }

// In-place spatial sort (nnps.cpp:447-476); perm receives n entries.
void ref_ps_spatial_sort(void* ps, std::uint32_t* perm_out) {
  auto* p = static_cast<sphx::ParticleSystem*>(ps);
  const auto perm = sphx::spatial_sort_permutation(*p);
  sphx::apply_permutation(*p, perm);
  if (perm_out) std::copy(perm.begin(), perm.end(), perm_out);
}

// ---- grid -------------------------------------------------------------------------
void* ref_grid_make(void* ps, const int* periodic) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new sphx::CellGrid(sphx::make_grid_for(*static_cast<sphx::ParticleSystem*>(ps),
                                                 {periodic[0] != 0, periodic[1] != 0,
                                                  periodic[2] != 0}));
  });
  return rc == 0 ? out : nullptr;
}

// Grid descriptor fields: dim, counts[3], periodic[3] as ints; hc[3], cutoff_norm,
// radius, span[3], origin[3], edge[3] as doubles.
void ref_grid_desc(void* g, int* ints, double* dbls) {
  const auto* grid = static_cast<sphx::CellGrid*>(g);
  ints[0] = grid->dim();
  for (int k = 0; k < 3; ++k) {
    ints[1 + k] = grid->count(k);
    ints[4 + k] = grid->periodic(k) ? 1 : 0;
    dbls[k] = grid->hc(k);
    dbls[5 + k] = grid->domain().span(k);
    dbls[8 + k] = grid->origin_norm(k);
    dbls[11 + k] = grid->edge_phys(k);
  }
  dbls[3] = grid->cutoff_norm();
  dbls[4] = grid->radius_phys();
}

std::int64_t ref_grid_cell_total(void* g) { return static_cast<sphx::CellGrid*>(g)->cell_total(); }

int ref_grid_rebin(void* g, void* ps) {
  return guarded([&] {
    static_cast<sphx::CellGrid*>(g)->rebin(*static_cast<sphx::ParticleSystem*>(ps));
  });
}

std::uint64_t ref_grid_items_size(void* g) { return static_cast<sphx::CellGrid*>(g)->items().size(); }
void ref_grid_items(void* g, std::int32_t* out) {
  const auto s = static_cast<sphx::CellGrid*>(g)->items();
  std::copy(s.begin(), s.end(), out);
}
void ref_grid_cell_start(void* g, std::int32_t* out) {
  const auto s = static_cast<sphx::CellGrid*>(g)->cell_start();
  std::copy(s.begin(), s.end(), out);
}
void ref_grid_cell_of(void* g, std::uint64_t n, std::int32_t* out) {
  const auto* grid = static_cast<sphx::CellGrid*>(g);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = grid->cell_of(i);
}
void ref_grid_locate(void* g, const double* xn, std::int32_t* cell, double* rel) {
  std::array<std::int32_t, 3> c{};
  std::array<double, 3> r{};
  static_cast<sphx::CellGrid*>(g)->locate({xn[0], xn[1], xn[2]}, c, r);
  for (int k = 0; k < 3; ++k) {
    cell[k] = c[k];
    rel[k] = r[k];
  }
}
void ref_free_grid(void* g) { delete static_cast<sphx::CellGrid*>(g); }

// ---- relative coordinates -----------------------------------------------------------
void* ref_rel_build(void* ps, void* g) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new sphx::RelCoords(sphx::build_rel_coords(*static_cast<sphx::ParticleSystem*>(ps),
                                                     *static_cast<sphx::CellGrid*>(g)));
  });
  return rc == 0 ? out : nullptr;
}
void ref_rel_get(void* r, int k, double* rel_out, std::int32_t* cell_out) {
  const auto* rc = static_cast<sphx::RelCoords*>(r);
  if (rel_out) std::copy(rc->rel[k].begin(), rc->rel[k].end(), rel_out);
  if (cell_out) std::copy(rc->cell[k].begin(), rc->cell[k].end(), cell_out);
}
double ref_rel_distance(void* r, void* g, std::uint64_t i, std::uint64_t j, int prec) {
  return sphx::rel_distance(*static_cast<sphx::RelCoords*>(r), i, j,
                            *static_cast<sphx::CellGrid*>(g), prec_of(prec));
}
void ref_free_rel(void* r) { delete static_cast<sphx::RelCoords*>(r); }

// ---- NNPS backends (nnps.hpp:31-41) -----------------------------------------------------
void* ref_rcll(void* r, void* g, int prec) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new sphx::NeighborTable(sphx::rcll(*static_cast<sphx::RelCoords*>(r),
                                             *static_cast<sphx::CellGrid*>(g), prec_of(prec)));
  });
  return rc == 0 ? out : nullptr;
}
void* ref_cll(void* ps, void* g, int prec) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new sphx::NeighborTable(sphx::cell_link_list(*static_cast<sphx::ParticleSystem*>(ps),
                                                       *static_cast<sphx::CellGrid*>(g),
                                                       prec_of(prec)));
  });
  return rc == 0 ? out : nullptr;
}
void* ref_all_list(void* ps, int prec) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new sphx::NeighborTable(
        sphx::all_list(*static_cast<sphx::ParticleSystem*>(ps), prec_of(prec)));
  });
  return rc == 0 ? out : nullptr;
}
std::uint64_t ref_table_size(void* t) { return static_cast<sphx::NeighborTable*>(t)->size(); }
std::int64_t ref_table_total(void* t) { return static_cast<sphx::NeighborTable*>(t)->total(); }
double ref_table_radius(void* t) { return static_cast<sphx::NeighborTable*>(t)->radius; }
void ref_table_copy(void* t, std::int64_t* offsets, std::int32_t* items) {
  const auto* tb = static_cast<sphx::NeighborTable*>(t);
  if (offsets) std::copy(tb->offsets.begin(), tb->offsets.end(), offsets);
  if (items) std::copy(tb->items.begin(), tb->items.end(), items);
}
std::uint64_t ref_table_hash(void* t) { return fnv_table(*static_cast<sphx::NeighborTable*>(t)); }
void ref_free_table(void* t) { delete static_cast<sphx::NeighborTable*>(t); }

// ---- update_relative over particles [0, n) (cell_grid.cpp:180-212) -----------------
// 0, or 1 + the index of the particle whose update threw (message in ref_last_error).
std::int64_t ref_update_relative(void* r, void* g, std::uint64_t n, const double* dx0,
                                 const double* dx1, const double* dx2, int prec) {
  auto& rc = *static_cast<sphx::RelCoords*>(r);
  const auto& grid = *static_cast<sphx::CellGrid*>(g);
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::array<double, 3> d{dx0 ? dx0[i] : 0.0, dx1 ? dx1[i] : 0.0, dx2 ? dx2[i] : 0.0};
    if (guarded([&] { sphx::update_relative(rc, i, d, grid, prec_of(prec)); }) != 0)
      return (std::int64_t)i + 1;
  }
  return 0;
}

// ---- gradient on a table (gradient.hpp:27, gradient.cpp:44-82) ------------------------
std::int64_t ref_grad_normalized(void* ps, void* t, const double* f, double h, double* g0,
                                 double* g1, double* g2) {
  std::int64_t deg = -1;
  guarded([&] {
    const auto& p = *static_cast<sphx::ParticleSystem*>(ps);
    std::vector<double> fv(f, f + p.size());
    const auto gf = sphx::grad_normalized(fv, p, *static_cast<sphx::NeighborTable*>(t),
                                          sphx::make_kernel(h, p.dim()));
    double* out[3] = {g0, g1, g2};
    for (int k = 0; k < p.dim(); ++k)
      if (out[k]) std::copy(gf.g[k].begin(), gf.g[k].end(), out[k]);
    deg = gf.degenerate_count;
  });
  return deg;
}


// ---- the mixed-precision time step (dynamics.cpp:136-203), SURVEY 8(f) row 3 ---------
// A MixedState (dynamics.hpp:71-82) built from a particle system, plus the table
// of its last step_mixed call.
struct RefMixed {
  sphx::MixedState st;
  sphx::NeighborTable last;
  RefMixed(sphx::ParticleSystem ps, std::array<bool, 3> per, sphx::Approach a)
      : st(std::move(ps), per, a) {}
};

void* ref_mixed_new(void* ps, const int* periodic, int approach) {
  void* out = nullptr;
  const int rc = guarded([&] {
    out = new RefMixed(*static_cast<sphx::ParticleSystem*>(ps),
                       {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0},
                       static_cast<sphx::Approach>(approach));
  });
  return rc == 0 ? out : nullptr;
}
void ref_mixed_free(void* m) { delete static_cast<RefMixed*>(m); }

// field: 0 x, 1 v, 2 rho, 3 p, 4 e, 5 m, 6 rel (FP64 coordinate), 7 cell (int32 out)
static double* mixed_field(RefMixed& m, int field, int k) {
  auto& ps = m.st.ps;
  switch (field) {
    case 0: return ps.x(k).data();
    case 1: return ps.v(k).data();
    case 2: return ps.rho().data();
    case 3: return ps.p().data();
    case 4: return ps.e().data();
    case 5: return const_cast<double*>(ps.m().data());
    case 6: return m.st.rel.rel[k].data();
    default: return nullptr;
  }
}
void ref_mixed_get(void* mp, int field, int k, double* out) {
  auto& m = *static_cast<RefMixed*>(mp);
  const std::size_t n = m.st.ps.size();
  if (field == 7) {
    std::memcpy(out, m.st.rel.cell[k].data(), sizeof(std::int32_t) * n);
    return;
  }
  std::memcpy(out, mixed_field(m, field, k), sizeof(double) * n);
}
void ref_mixed_set(void* mp, int field, int k, const double* in) {
  auto& m = *static_cast<RefMixed*>(mp);
  std::memcpy(mixed_field(m, field, k), in, sizeof(double) * m.st.ps.size());
}
// the grid membership: cell_of (n), cell_start (cells + 1), items (n)
void ref_mixed_grid(void* mp, std::int32_t* cell_of, std::int32_t* start, std::int32_t* items) {
  auto& g = static_cast<RefMixed*>(mp)->st.grid;
  const std::size_t n = static_cast<RefMixed*>(mp)->st.ps.size();
  for (std::size_t i = 0; i < n; ++i) cell_of[i] = g.cell_of(i);
  std::copy(g.cell_start().begin(), g.cell_start().end(), start);
  std::copy(g.items().begin(), g.items().end(), items);
}
// One step_mixed with StepConfig {dt, c_sound, rho0, mu, body_force, n_moving,
// evolve_density, compute_energy} (no pre_force). Returns 0 or the error code;
// *max_dx and *total receive StepResult::max_dx and the table size.
int ref_mixed_step(void* mp, const double* cfg, const double* body_force, std::uint64_t n_moving,
                   int evolve_density, int compute_energy, double* max_dx, std::int64_t* total) {
  auto& m = *static_cast<RefMixed*>(mp);
  return guarded([&] {
    sphx::StepConfig c;
    c.dt = cfg[0];
    c.c_sound = cfg[1];
    c.rho0 = cfg[2];
    c.mu = cfg[3];
    c.body_force = {body_force[0], body_force[1], body_force[2]};
    c.n_moving = n_moving;
    c.evolve_density = evolve_density != 0;
    c.compute_energy = compute_energy != 0;
    auto res = sphx::step_mixed(m.st, c);
    *max_dx = res.max_dx;
    *total = res.table.total();
    m.last = std::move(res.table);
  });
}
void ref_mixed_table(void* mp, std::int64_t* offsets, std::int32_t* items) {
  const auto& t = static_cast<RefMixed*>(mp)->last;
  std::copy(t.offsets.begin(), t.offsets.end(), offsets);
  std::copy(t.items.begin(), t.items.end(), items);
}

// ---- timing (experiments.cpp:268-278 method: one discarded warm-up, median) -------------
// which: 0 = rcll(rel, grid, prec), 1 = cell_link_list(ps, grid, prec).
double ref_time_nnps(int which, void* ps, void* r, void* g, int prec, int repeats) {
  auto run = [&] {
    if (which == 0) {
      auto t = sphx::rcll(*static_cast<sphx::RelCoords*>(r), *static_cast<sphx::CellGrid*>(g),
                          prec_of(prec));
      return t.total();
    }
    auto t = sphx::cell_link_list(*static_cast<sphx::ParticleSystem*>(ps),
                                  *static_cast<sphx::CellGrid*>(g), prec_of(prec));
    return t.total();
  };
  run();
  std::vector<double> ts;
  for (int k = 0; k < std::max(1, repeats); ++k) {
    const auto a = std::chrono::steady_clock::now();
    run();
    ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

}  // extern "C"
