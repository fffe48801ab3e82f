// Column-kernel instantiations: float, variant 1 (see ColVariant).
#include "fast_launch.cuh"

namespace sdctb {
template <>
cudaError_t launch_col_variant<float, 1>(int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                                         const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  return launch_col_var<float, 1>(L, nl, grid, st, map, omap, a, tw);
}
}  // namespace sdctb
