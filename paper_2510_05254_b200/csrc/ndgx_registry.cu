// Registry of the compiled stage kernels: (dim, order, kind, exact) -> entry.
#include "ndgx_kernels.h"

namespace ndgx {

#define NDGX_DECL_ORDERS(D, E)                                                              \
  StageKernel NDGX_ENTRY_NAME(D, 2, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 3, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 4, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 5, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 6, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 7, E)(int);                                                \
  StageKernel NDGX_ENTRY_NAME(D, 8, E)(int);
NDGX_DECL_ORDERS(1, 0)
NDGX_DECL_ORDERS(1, 1)
NDGX_DECL_ORDERS(2, 0)
NDGX_DECL_ORDERS(2, 1)
NDGX_DECL_ORDERS(3, 0)
NDGX_DECL_ORDERS(3, 1)
#undef NDGX_DECL_ORDERS

using Entry = StageKernel (*)(int);

#define NDGX_ROW(D, E)                                                                      \
  {NDGX_ENTRY_NAME(D, 2, E), NDGX_ENTRY_NAME(D, 3, E), NDGX_ENTRY_NAME(D, 4, E),           \
   NDGX_ENTRY_NAME(D, 5, E), NDGX_ENTRY_NAME(D, 6, E), NDGX_ENTRY_NAME(D, 7, E),            \
   NDGX_ENTRY_NAME(D, 8, E)}

static const Entry kTable[3][2][7] = {
    {NDGX_ROW(1, 0), NDGX_ROW(1, 1)},
    {NDGX_ROW(2, 0), NDGX_ROW(2, 1)},
    {NDGX_ROW(3, 0), NDGX_ROW(3, 1)},
};
#undef NDGX_ROW

StageKernel find_stage_kernel(int dim, int order, int kind, bool exact) {
  if (dim < 1 || dim > 3 || order < 2 || order > kMaxOrder) return StageKernel{};
  return kTable[dim - 1][exact ? 1 : 0][order - 2](kind);
}

}  // namespace ndgx
