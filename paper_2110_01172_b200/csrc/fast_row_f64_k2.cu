// Row-kernel instantiations: double, kind 2 (see RowKind).
#include "fast_launch.cuh"

namespace sdctb {
template <>
cudaError_t launch_row_kind_ext<double, 2>(int M, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  return launch_row_kind<double, 2>(M, grid, st, a, tw);
}
}  // namespace sdctb
