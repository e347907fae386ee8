// ndgx_kernels.h -- host-visible registry of the compiled stage kernels.
#pragma once

#include <cuda_runtime.h>

#include "ndgx_device.cuh"

namespace ndgx {

using StageFn = void (*)(const StageArgs);

struct StageKernel {
  StageFn fn = nullptr;
  int threads = 0;
  int tile[3] = {1, 1, 1};  // elements per CTA tile along x, y, z
  int fixed_bytes = 0;      // mbarriers + work area (dynamic shared memory)
  int tile_arr_bytes = 0;   // one ring copy of a tile array (u or one K_j)
  int halo_bytes = 0;       // one ring slot's face halo records
  int raw_bytes = 0;        // one ring slot's raw halo values per input array
  bool tma_ok = false;      // element rows are 16-byte multiples (bulk copies)
};

// Ring configuration of one stage launch (host side).
struct StageLaunch {
  int ring_main = 0, dm = 1, dh = 1, smem = 0, grid = 1;
};

// dim 1..3, order 2..8, kind 0 advection / 1 Euler, exact arithmetic or FMA-contracted
StageKernel find_stage_kernel(int dim, int order, int kind, bool exact);

template <int DIM, int N, int KIND, bool EXACT>
StageKernel make_stage_kernel() {
  using G = Geo<DIM, N, KIND>;
  StageKernel k;
  k.fn = &stage_kernel<DIM, N, KIND, EXACT>;
  k.threads = G::THREADS;
  k.tile[0] = G::TX;
  k.tile[1] = G::TY;
  k.tile[2] = G::TZ;
  k.fixed_bytes = G::BAR_BYTES + G::WORK * 8;
  k.tile_arr_bytes = G::TILE_ARR * 8;
  k.halo_bytes = G::HALO * 8;
  k.raw_bytes = G::RAW1 * 8;
  k.tma_ok = G::TMA_OK;
  return k;
}

// per-(dim, order, exact) entry points, one object each (ndgx_inst.cu)
#define NDGX_CAT_(a, b, c, d) stage_entry_d##a##_o##b##_e##c
#define NDGX_ENTRY_NAME(D, N, E) NDGX_CAT_(D, N, E, 0)

}  // namespace ndgx
