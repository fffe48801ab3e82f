// Row-kernel instantiations: float, kind 0 (see RowKind).
#include "fast_launch.cuh"

namespace sdctb {
template <>
cudaError_t launch_row_kind_ext<float, 0>(int M, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  return launch_row_kind<float, 0>(M, grid, st, a, tw);
}
}  // namespace sdctb
