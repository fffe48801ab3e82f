// Axis-0 1D column pass (kernels_col1d.cuh): instantiations and launch for
// power-of-two L in [8, 4096], 32-B band rows (NL = 16 / sizeof(T)).
#include "fast_launch.cuh"
#include "kernels_col1d.cuh"

namespace sdctb {

template <typename T, int L, bool INV>
static cudaError_t launch_col1d_one(int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                    const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  constexpr int NL = 16 / sizeof(T);
  using Geo = Col1dGeom<T, L, NL>;
  auto k = col1d_kernel<T, L, NL, INV>;
  constexpr int NT = Tile<T, L, NL, true>::NT;
  cudaError_t e = prep_smem(k, Geo::SMEM);
  if (e != cudaSuccess) return e;
  static const int resident = [&] {  // thread-safe one-time query
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, Geo::SMEM);
    return sms * (per > 0 ? per : 1);
  }();
  ColArgs b = a;
  b.nbands = bands;
  b.nplanes = 1;
  b.ntiles = bands * batch;
  const int ctas = b.ntiles < resident ? b.ntiles : resident;
  return launch_pdl(k, dim3(ctas), dim3(NT), Geo::SMEM, st, map, omap, b, tw);
}

template <typename T, int L>
static cudaError_t launch_col1d_l(bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                                  const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  return inv ? launch_col1d_one<T, L, true>(bands, batch, st, map, omap, a, tw)
             : launch_col1d_one<T, L, false>(bands, batch, st, map, omap, a, tw);
}

template <typename T>
cudaError_t launch_col1d(bool inv, int L, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                         const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  switch (L) {
    case 8: return launch_col1d_l<T, 8>(inv, bands, batch, st, map, omap, a, tw);
    case 16: return launch_col1d_l<T, 16>(inv, bands, batch, st, map, omap, a, tw);
    case 32: return launch_col1d_l<T, 32>(inv, bands, batch, st, map, omap, a, tw);
    case 64: return launch_col1d_l<T, 64>(inv, bands, batch, st, map, omap, a, tw);
    case 128: return launch_col1d_l<T, 128>(inv, bands, batch, st, map, omap, a, tw);
    case 256: return launch_col1d_l<T, 256>(inv, bands, batch, st, map, omap, a, tw);
    case 512: return launch_col1d_l<T, 512>(inv, bands, batch, st, map, omap, a, tw);
    case 1024: return launch_col1d_l<T, 1024>(inv, bands, batch, st, map, omap, a, tw);
    case 2048: return launch_col1d_l<T, 2048>(inv, bands, batch, st, map, omap, a, tw);
    case 4096: return launch_col1d_l<T, 4096>(inv, bands, batch, st, map, omap, a, tw);
    default: return cudaErrorInvalidValue;
  }
}

template cudaError_t launch_col1d<float>(bool, int, int, int, cudaStream_t, const CUtensorMap&, const CUtensorMap&,
                                         const ColArgs&, const TwSet&);
template cudaError_t launch_col1d<double>(bool, int, int, int, cudaStream_t, const CUtensorMap&, const CUtensorMap&,
                                          const ColArgs&, const TwSet&);

}  // namespace sdctb
