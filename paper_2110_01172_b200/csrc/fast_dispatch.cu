// Dispatch from runtime (variant, kind, dtype) to the per-unit instantiations.
#include "fast_launch.cuh"

namespace sdctb {

template <typename T>
cudaError_t launch_col(int variant, int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                       const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  switch (variant) {
    case CV_FWD_SRC: return launch_col_variant<T, CV_FWD_SRC>(L, nl, grid, st, map, omap, a, tw);
    case CV_FWD_INTER: return launch_col_variant<T, CV_FWD_INTER>(L, nl, grid, st, map, omap, a, tw);
    case CV_INV_INTER: return launch_col_variant<T, CV_INV_INTER>(L, nl, grid, st, map, omap, a, tw);
    case CV_INV_DST: return launch_col_variant<T, CV_INV_DST>(L, nl, grid, st, map, omap, a, tw);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
cudaError_t launch_row(int M, int kind, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  switch (kind) {
    case RK_FWD2: return launch_row_kind_ext<T, RK_FWD2>(M, grid, st, a, tw);
    case RK_INV2: return launch_row_kind_ext<T, RK_INV2>(M, grid, st, a, tw);
    case RK_FWD3: return launch_row_kind_ext<T, RK_FWD3>(M, grid, st, a, tw);
    case RK_INV3: return launch_row_kind_ext<T, RK_INV3>(M, grid, st, a, tw);
    default: return cudaErrorInvalidValue;
  }
}

template cudaError_t launch_col<float>(int, int, int, dim3, cudaStream_t, const CUtensorMap&, const CUtensorMap&, const ColArgs&,
                                      const TwSet&);
template cudaError_t launch_col<double>(int, int, int, dim3, cudaStream_t, const CUtensorMap&, const CUtensorMap&, const ColArgs&,
                                       const TwSet&);
template cudaError_t launch_row<float>(int, int, dim3, cudaStream_t, const RowArgs&, const TwSet&);
template cudaError_t launch_row<double>(int, int, dim3, cudaStream_t, const RowArgs&, const TwSet&);

}  // namespace sdctb
