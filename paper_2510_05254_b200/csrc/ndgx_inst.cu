// Stage-kernel instantiations for one (dim, order, arithmetic) triple, both
// equation systems where defined.  build.py compiles this file once per
// triple (-DNDGX_DIM, -DNDGX_ORDER, -DNDGX_EXACT) so the 42 objects build in
// parallel; ndgx_registry.cu maps (dim, order, kind, exact) onto them.
#include "ndgx_kernels.h"

#ifndef NDGX_DIM
#error "compile with -DNDGX_DIM=1..3 -DNDGX_ORDER=2..8 -DNDGX_EXACT=0|1"
#endif

namespace ndgx {

StageKernel NDGX_ENTRY_NAME(NDGX_DIM, NDGX_ORDER, NDGX_EXACT)(int kind) {
  if (kind == 0) return make_stage_kernel<NDGX_DIM, NDGX_ORDER, 0, (NDGX_EXACT != 0)>();
#if NDGX_DIM > 1
  // isothermal Euler is 2D/3D only (models.cpp:23-33)
  if (kind == 1) return make_stage_kernel<NDGX_DIM, NDGX_ORDER, 1, (NDGX_EXACT != 0)>();
#endif
  return StageKernel{};
}

}  // namespace ndgx
