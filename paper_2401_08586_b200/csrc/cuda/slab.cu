// Slab assembly for the multi-GPU path: the local system of one
// rank after the halo exchange, without binning anything.
//
// The reference is single-process; its rcll (nnps.cpp:283-416) reads a CellGrid
// whose members are CSR lists over linear cells, x fastest (cell_grid.hpp:74-78).
// Cut along the slowest axis, one cell layer of the grid is a contiguous range
// of linear cells and therefore of CSR positions. A rank keeps its owned
// particles' RelCoords in CSR order, so each boundary layer it sends is a
// contiguous slice (rel, global ids) plus the layer's slice of cell_start; the
// receiver drops the slices into reserved slots of its local arrays. This
// kernel then writes the local CellGrid of nl + 2 layers -- the lower halo
// (layer 0), the owned layers (1 .. nl), the upper halo (nl + 1) -- and the
// RelCoords cell of each halo particle, all from device-side sizes (no host
// synchronisation between the exchange and the rows).
//
// Local particle slots: [owned (n_own) | pad | lower halo (capB) | upper halo].

#include <algorithm>

#include "common.cuh"

namespace sphx_dev {



__global__ void k_slab_start(SlabArgs a) {
  const int64_t C = (int64_t)(a.nl + 2) * a.CL;
  const int mB = a.haveB ? __ldg(a.rB + a.CL) - __ldg(a.rB) : 0;
  const int total_own = __ldg(a.ocs + (int64_t)a.nl * a.CL);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= C; c += (int64_t)gridDim.x * blockDim.x) {
    int v;
    if (c < a.CL) {
      v = a.haveB ? __ldg(a.rB + c) - __ldg(a.rB) : 0;
    } else if (c < (int64_t)(a.nl + 1) * a.CL) {
      v = mB + __ldg(a.ocs + (c - a.CL));
    } else {
      const int64_t u = c - (int64_t)(a.nl + 1) * a.CL;
      v = mB + total_own + (a.haveA ? __ldg(a.rA + u) - __ldg(a.rA) : 0);
    }
    a.start[c] = v;
  }
}

// CSR position -> slot, and the halo particles' cells (one thread per halo cell)
__global__ void k_slab_items(SlabArgs a) {
  const int mB = a.haveB ? __ldg(a.rB + a.CL) - __ldg(a.rB) : 0;
  const int mA = a.haveA ? __ldg(a.rA + a.CL) - __ldg(a.rA) : 0;
  const int total = mB + a.n_own + mA;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t p = t0; p < total; p += stride) {
    int s;
    if (p < mB) s = a.slotB + (int)p;
    else if (p < mB + a.n_own) s = (int)p - mB;
    else s = a.slotA + (int)(p - mB - a.n_own);
    a.items[p] = s;
  }
  for (int64_t q = t0; q < 2 * (int64_t)a.CL; q += stride) {
    const bool up = q >= a.CL;
    if (up ? !a.haveA : !a.haveB) continue;
    const int c = (int)(up ? q - a.CL : q);
    const int32_t* r = up ? a.rA : a.rB;
    const int b = __ldg(r + c) - __ldg(r), e = __ldg(r + c + 1) - __ldg(r);
    const int slot0 = up ? a.slotA : a.slotB;
    // coordinates of layer cell c: the axes below the slab axis, x fastest
    int cc[3] = {0, 0, 0};
    int rem = c;
    for (int k = 0; k < a.dim; ++k) {
      if (k == a.axis) continue;
      cc[k] = rem % a.cnt[k];
      rem /= a.cnt[k];
    }
    cc[a.axis] = up ? a.nl + 1 : 0;
    for (int m = b; m < e; ++m)
      for (int k = 0; k < a.dim; ++k) a.cell[k][slot0 + m] = cc[k];
  }
}

int launch_slab_assemble(const SlabArgs& a, cudaStream_t st) {
  const int64_t C = (int64_t)(a.nl + 2) * a.CL + 1;
  const unsigned g1 = (unsigned)std::min<int64_t>((C + 255) / 256, 148 * 16);
  k_slab_start<<<g1, 256, 0, st>>>(a);
  const int64_t work = std::max<int64_t>((int64_t)a.n_slots, 2 * (int64_t)a.CL);
  const unsigned g2 = (unsigned)std::min<int64_t>((work + 255) / 256, 148 * 16);
  k_slab_items<<<g2, 256, 0, st>>>(a);
  return 2;
}

}  // namespace sphx_dev
