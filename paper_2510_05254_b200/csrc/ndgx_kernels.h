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
  int smem_base = 0;    // dynamic shared memory, non-last stages
  int smem_last = 0;    // dynamic shared memory, last stage
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
  k.smem_base = G::SMEM_BASE;
  k.smem_last = G::SMEM_LAST;
  return k;
}

// per-dimension registries (one translation unit each, compiled in parallel)
StageKernel find_stage_kernel_d1(int order, int kind, bool exact);
StageKernel find_stage_kernel_d2(int order, int kind, bool exact);
StageKernel find_stage_kernel_d3(int order, int kind, bool exact);

}  // namespace ndgx
