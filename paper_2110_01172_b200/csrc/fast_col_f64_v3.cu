// Column-kernel instantiations: double, variant 3 (see ColVariant).
#include "fast_launch.cuh"

namespace sdctb {
template <>
cudaError_t launch_col_variant<double, 3>(int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                                         const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  return launch_col_var<double, 3>(L, nl, grid, st, map, omap, a, tw);
}
}  // namespace sdctb
