// ndgx_kernels.h -- host-visible registry of the compiled stage kernels.
#pragma once

#include <cuda_runtime.h>

#include "ndgx_device.cuh"

namespace ndgx {

using StageFn = void (*)(const StageArgs);

struct StageKernel {
  StageFn fn[kNumSigs] = {};  // by stage signature (kSigs)
  StageFn fnx[kNumSigs] = {}; // region-3 (x-filtered interior) launches: the x-run variant where one exists
  int threads = 0;
  int warps = 0;            // elements in flight per CTA (EPW per warp)
  int smem_fixed[kNumSigs] = {};  // dynamic shared memory without the element rings, per signature
  int ring_per_array = 0;   // ring bytes per slot per input array (all warps of a CTA)
  bool tma_ok = false;      // element chunks are 16-byte multiples (bulk copies)
  bool prefer_direct = false;  // measured: direct loads beat the TMA ring (Euler, B200)
  int smem(int sig, int depth) const { return smem_fixed[sig] + depth * (1 + kSigs[sig].nu) * ring_per_array; }
};

// Launch configuration of one stage kernel variant (host side).
struct StageLaunch {
  int depth = 0, smem = 0, grid = 1;
};

// dim 1..3, order 2..8, kind 0 advection / 1 Euler, exact arithmetic or FMA-contracted
StageKernel find_stage_kernel(int dim, int order, int kind, bool exact);

template <int DIM, int N, int KIND, bool EXACT>
StageKernel make_stage_kernel() {
  using G = Geo<DIM, N, KIND>;
  StageKernel k;
  k.fn[0] = &stage_kernel<DIM, N, KIND, EXACT, 0>;
  k.fn[1] = &stage_kernel<DIM, N, KIND, EXACT, 1>;
  k.fn[2] = &stage_kernel<DIM, N, KIND, EXACT, 2>;
  k.fn[3] = &stage_kernel<DIM, N, KIND, EXACT, 3>;
  k.fn[4] = &stage_kernel<DIM, N, KIND, EXACT, 4>;
  k.fn[5] = &stage_kernel<DIM, N, KIND, EXACT, 5>;
  k.fn[6] = &stage_kernel<DIM, N, KIND, EXACT, 6>;
  k.fn[7] = &stage_kernel<DIM, N, KIND, EXACT, 7>;
  k.fn[8] = &stage_kernel<DIM, N, KIND, EXACT, 8>;
  // the x-run body (2D order-8 contracted Euler, last stages) has an
  // x-filtered twin; every other kernel handles region 3 in its element loop
  constexpr bool XRUN = G::MMA && !EXACT && KIND == 1;
  for (int q = 0; q < kNumSigs; ++q) k.fnx[q] = k.fn[q];
  if constexpr (XRUN) {
    k.fnx[2] = &stage_kernel<DIM, N, KIND, EXACT, 2, true>;
    k.fnx[3] = &stage_kernel<DIM, N, KIND, EXACT, 3, true>;
    k.fnx[8] = &stage_kernel<DIM, N, KIND, EXACT, 8, true>;
  }
  k.threads = G::THREADS;
  k.warps = G::WARPS * (G::mma_body(EXACT, 0) ? 1 : G::EPW);  // (the tensor-core bodies: one element per warp)
  for (int q = 0; q < kNumSigs; ++q)
    k.smem_fixed[q] = G::smem_bytes(0, 0, G::mma_body(EXACT, q), kSigs[q].bm != 0);
  k.ring_per_array = G::WARPS * G::SLOT1 * 8;
  k.tma_ok = G::TMA_OK;
  // Euler stages: 16 warps/SM of 16-byte direct loads keep more bytes in flight
  // than a per-warp TMA ring, whose shared memory costs resident warps
  // (C3 fast 3.22 vs 4.21 ms/step, exact 6.70 vs 6.8; profiles/README.md)
  // (the contracted 2D order-8 body too for advection: C2 0.284 vs 0.322 ms/step)
  k.prefer_direct = KIND == 1 || G::MMA3 || (G::MMA && !EXACT);
  return k;
}

// per-(dim, order, exact) entry points, one object each (ndgx_inst.cu)
#define NDGX_CAT_(a, b, c, d) stage_entry_d##a##_o##b##_e##c
#define NDGX_ENTRY_NAME(D, N, E) NDGX_CAT_(D, N, E, 0)

}  // namespace ndgx
