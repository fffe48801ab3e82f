// Cluster-split column kernels: instantiations + launch (fp64 H = 2048, 4096;
// fp32 H = 4096).
#include "fast_launch.cuh"

namespace sdctb {

template <typename T, int H, int NL, bool INV>
static cudaError_t launch_col2_one(int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                   const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  using Geo = Col2Geom<T, H, NL>;
  auto k = col2_kernel<T, H, NL, INV>;
  cudaError_t e = prep_smem(k, Geo::SMEM);
  if (e != cudaSuccess) return e;
  k<<<dim3(2 * bands, batch), Geo::NT, Geo::SMEM, st>>>(map, omap, a, tw);
  return cudaGetLastError();
}

template <typename T, int H>
static cudaError_t launch_col2_h(bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                 const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  constexpr int NL = 16 / sizeof(T);  // 32-B band rows
  return inv ? launch_col2_one<T, H, NL, true>(bands, batch, st, map, omap, a, tw)
             : launch_col2_one<T, H, NL, false>(bands, batch, st, map, omap, a, tw);
}

template <>
cudaError_t launch_col2<double>(int L, bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  if (L == 4096) return launch_col2_h<double, 2048>(inv, bands, batch, st, map, omap, a, tw);
  if (L == 8192) return launch_col2_h<double, 4096>(inv, bands, batch, st, map, omap, a, tw);
  return cudaErrorInvalidValue;
}

template <>
cudaError_t launch_col2<float>(int L, bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                               const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  if (L == 4096) return launch_col2_h<float, 2048>(inv, bands, batch, st, map, omap, a, tw);
  if (L == 8192) return launch_col2_h<float, 4096>(inv, bands, batch, st, map, omap, a, tw);
  return cudaErrorInvalidValue;
}

}  // namespace sdctb
