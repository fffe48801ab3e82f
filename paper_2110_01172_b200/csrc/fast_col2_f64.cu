// Cluster-split column kernels (fp64, H = 2048): instantiation + launch.
#include "fast_launch.cuh"

namespace sdctb {

template <bool INV>
static cudaError_t launch_col2_one(int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                   const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  using Geo = Col2Geom<double, 2048, 2>;
  auto k = col2_kernel<double, 2048, 2, INV>;
  cudaError_t e = prep_smem(k, Geo::SMEM);
  if (e != cudaSuccess) return e;
  k<<<dim3(2 * bands, batch), Geo::NT, Geo::SMEM, st>>>(map, omap, a, tw);
  return cudaGetLastError();
}

cudaError_t launch_col2(bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map, const CUtensorMap& omap,
                        const ColArgs& a, const TwSet& tw) {
  return inv ? launch_col2_one<true>(bands, batch, st, map, omap, a, tw)
             : launch_col2_one<false>(bands, batch, st, map, omap, a, tw);
}

}  // namespace sdctb
