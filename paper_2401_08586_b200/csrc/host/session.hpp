// Process-wide CUDA session of the C++ drop-in and the mapping from C-ABI
// status codes back to the exception types the reference throws.
//
// Only public CellGrid accessors are used, so this header (and nnps_cuda.cpp)
// compiles against the reference's own sphx headers as well as ours.
#pragma once

#include <mutex>
#include <stdexcept>
#include <string>

#include "sphx/cell_grid.hpp"
#include "sphx_cuda.h"

namespace sphx::cuda {

// The library context used by the free functions (created on first use on the
// current CUDA device; SPHX_DEVICE=<n> picks another), held for the lifetime of
// a Session: the context's staging and table buffers are shared, so each
// drop-in call keeps it locked from its first C-ABI call through the table copy
// (the reference's functions are reentrant; concurrent callers serialise here).
// Throws std::runtime_error when no sm_100 device is available -- there is no
// CPU fallback.
class Session {
 public:
  Session();
  sphx_context* get() const { return ctx_; }

 private:
  std::unique_lock<std::recursive_mutex> lock_;
  sphx_context* ctx_;
};

// Rethrows a non-OK status as the reference's exception type with its message.
[[noreturn]] void rethrow(int code);

inline void check(int rc) {
  if (rc != SPHX_OK) rethrow(rc);
}

// POD view of a CellGrid (cell_grid.hpp accessors only).
inline sphx_grid_desc describe(const CellGrid& g) {
  sphx_grid_desc d{};
  d.dim = g.dim();
  for (int k = 0; k < 3; ++k) {
    d.counts[k] = k < g.dim() ? g.count(k) : 1;
    d.periodic[k] = k < g.dim() && g.periodic(k) ? 1 : 0;
    d.hc[k] = k < g.dim() ? g.hc(k) : 0.0;
    d.origin[k] = k < g.dim() ? g.origin_norm(k) : 0.0;
    d.lo[k] = g.domain().lo[k];
    d.hi[k] = g.domain().hi[k];
  }
  d.cutoff_norm = g.cutoff_norm();
  d.radius_phys = g.radius_phys();
  return d;
}

}  // namespace sphx::cuda
