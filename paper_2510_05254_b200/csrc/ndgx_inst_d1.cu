// Stage-kernel instantiations for dim = 1 (orders 2..8, both equation
// systems where defined, exact and contracted arithmetic).
#include "ndgx_kernels.h"

namespace ndgx {

template <int N, int KIND>
static StageKernel pick(bool exact) {
  return exact ? make_stage_kernel<1, N, KIND, true>() : make_stage_kernel<1, N, KIND, false>();
}

template <int KIND>
static StageKernel by_order(int order, bool exact) {
  switch (order) {
    case 2: return pick<2, KIND>(exact);
    case 3: return pick<3, KIND>(exact);
    case 4: return pick<4, KIND>(exact);
    case 5: return pick<5, KIND>(exact);
    case 6: return pick<6, KIND>(exact);
    case 7: return pick<7, KIND>(exact);
    case 8: return pick<8, KIND>(exact);
    default: return StageKernel{};
  }
}

StageKernel find_stage_kernel_d1(int order, int kind, bool exact) {
  if (kind != 0) return StageKernel{};  // isothermal Euler is 2D/3D (models.cpp:23-33)
  return by_order<0>(order, exact);
}

}  // namespace ndgx
