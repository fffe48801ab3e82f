// Host launchers of the row-column kernels (kernels_rowcol.cuh).
#include "fast_launch.cuh"
#include "kernels_rowcol.cuh"

namespace sdctb {

namespace {

template <typename T, int M, bool INV>
cudaError_t launch_rowdct_M(const RcArgs& a, const TwSet& tw, cudaStream_t st) {
  auto k = rowdct_kernel<T, M, INV>;
  const size_t smem = 2 * M * sizeof(cx_t<T>) + 16;  // tile (== two real rows) + mbarrier
  cudaError_t e = prep_smem(k, smem);
  if (e != cudaSuccess) return e;
  const long long ctas = (a.rows + 1) / 2;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_pdl(k, dim3(static_cast<unsigned>(ctas)), dim3(Tile<T, M, 2, false>::NT), smem, st, a, tw);
}

template <typename T, bool INV>
cudaError_t launch_rowdct_inv(int n, const RcArgs& a, const TwSet& tw, cudaStream_t st) {
  switch (n / 2) {
    case 4: return launch_rowdct_M<T, 4, INV>(a, tw, st);
    case 8: return launch_rowdct_M<T, 8, INV>(a, tw, st);
    case 16: return launch_rowdct_M<T, 16, INV>(a, tw, st);
    case 32: return launch_rowdct_M<T, 32, INV>(a, tw, st);
    case 64: return launch_rowdct_M<T, 64, INV>(a, tw, st);
    case 128: return launch_rowdct_M<T, 128, INV>(a, tw, st);
    case 256: return launch_rowdct_M<T, 256, INV>(a, tw, st);
    case 512: return launch_rowdct_M<T, 512, INV>(a, tw, st);
    case 1024: return launch_rowdct_M<T, 1024, INV>(a, tw, st);
    case 2048: return launch_rowdct_M<T, 2048, INV>(a, tw, st);
    case 4096: return launch_rowdct_M<T, 4096, INV>(a, tw, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

template <typename T>
cudaError_t launch_rowdct(int n, bool inv, const RcArgs& a, const TwSet& tw, cudaStream_t st) {
  return inv ? launch_rowdct_inv<T, true>(n, a, tw, st) : launch_rowdct_inv<T, false>(n, a, tw, st);
}

template <typename T>
cudaError_t launch_rowdct_direct(bool inv, const RcArgs& a, cudaStream_t st) {
  const long long total = a.rows * a.n;
  const long long blocks = (total + 255) / 256;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_pdl(rowdct_direct_kernel<T>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, a,
                    inv ? 1 : 0);
}

template <typename T>
cudaError_t launch_transpose(const void* in, void* out, int R, int C, long long batch, cudaStream_t st) {
  if (batch > 65535) return cudaErrorInvalidValue;  // callers chunk larger batches
  const dim3 grid((C + 31) / 32, (R + 31) / 32, static_cast<unsigned>(batch));
  return launch_pdl(transpose_kernel<T>, grid, dim3(32, 8), 0, st, static_cast<const T*>(in), static_cast<T*>(out),
                    R, C);
}

template cudaError_t launch_rowdct<float>(int, bool, const RcArgs&, const TwSet&, cudaStream_t);
template cudaError_t launch_rowdct<double>(int, bool, const RcArgs&, const TwSet&, cudaStream_t);
template cudaError_t launch_rowdct_direct<float>(bool, const RcArgs&, cudaStream_t);
template cudaError_t launch_rowdct_direct<double>(bool, const RcArgs&, cudaStream_t);
template cudaError_t launch_transpose<float>(const void*, void*, int, int, long long, cudaStream_t);
template cudaError_t launch_transpose<double>(const void*, void*, int, int, long long, cudaStream_t);

}  // namespace sdctb
