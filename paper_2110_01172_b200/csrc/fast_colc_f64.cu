// Persistent cluster-pair column pass (kernels_colc.cuh): instantiations and
// launch (fp64, L = 4096: H = 2048, 32-B band rows).
#include "fast_launch.cuh"
#include "kernels_colc.cuh"

namespace sdctb {

template <bool INV>
static cudaError_t launch_colc_one(int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                   const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  using Geo = ColcGeom<double, 2048, 2>;
  auto k = colc_kernel<double, 2048, 2, INV>;
  cudaError_t e = prep_smem(k, Geo::SMEM);
  if (e != cudaSuccess) return e;
  static const int clusters = [&] {  // resident 2-CTA clusters (thread-safe one-time query)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * 1024);
    cfg.blockDim = dim3(Geo::NT);
    cfg.dynamicSmemBytes = Geo::SMEM;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 128;
    }
    return n;
  }();
  ColArgs b = a;
  b.nbands = bands;
  b.nplanes = 1;
  b.ntiles = bands * batch;
  const int ncl = b.ntiles < clusters ? b.ntiles : clusters;
  return launch_pdl(k, dim3(2 * ncl), dim3(Geo::NT), Geo::SMEM, st, map, omap, b, tw);
}

cudaError_t launch_colc(bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                        const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  return inv ? launch_colc_one<true>(bands, batch, st, map, omap, a, tw)
             : launch_colc_one<false>(bands, batch, st, map, omap, a, tw);
}

}  // namespace sdctb
