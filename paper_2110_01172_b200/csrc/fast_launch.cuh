// Runtime -> compile-time dispatch for the fast-path kernels. The column
// kernel band width NL is a compile-time parameter with two choices per
// (dtype, L): nl_default (tile <= 128 KB) and 2 (small / low-parallelism
// problems). Each (dtype, variant) is instantiated in its own translation
// unit (fast_*.cu) so the build compiles them in parallel.
#pragma once

#include <cstdlib>
#include <utility>

#include "kernels_fast.cuh"
#include "kernels_row2.cuh"
#include "kernels_col2.cuh"
#include "kernels_rowp.cuh"

namespace sdctb {

constexpr int kMaxFastLen = 4096;  // largest FFT length with a fast (single-CTA) kernel
constexpr int kMaxSplitLen = 8192; // 2D axis-0 length reachable through the cluster-split column pass

// column-kernel variants
enum ColVariant { CV_FWD_SRC = 0, CV_FWD_INTER = 1, CV_INV_INTER = 2, CV_INV_DST = 3 };

// Column tiles target 64 KB (two CTAs per SM) with rows of >= 32 B
// (NL >= 16 / esize); long columns (4096 rows of 32 B = 128 KB) take one CTA
// per SM.
__host__ __device__ constexpr int nl_default(int esize, int L) {
  // complex element = 2*esize bytes; tile L * NL * 2*esize <= 64 KB
  return (64 * 1024) / (L * 2 * esize) >= 32   ? 32
         : (64 * 1024) / (L * 2 * esize) <= 16 / esize ? 16 / esize
                                                       : (64 * 1024) / (L * 2 * esize);
}

// Cluster-split column pass (kernels_col2.cuh): 2D fp64 columns of 4096 rows
// with 2-complex (32-B) bands run as two 64 KB halves per 2-CTA cluster.
__host__ __device__ constexpr bool col2_used(int esize, int L, int planes, int nl) {
  return planes == 1 && nl * esize == 16 && (L == 8192 || L == 4096);
}

// Launch with programmatic stream serialization: the kernel may start while
// the previous kernel of the stream drains (both kernels call pdl_trigger /
// pdl_wait, tma.cuh), hiding launch latency and prologue at pass boundaries.
// SDCT_NO_PDL=1 falls back to plain launches (A/B and debugging).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  static const bool off = [] {
    const char* f = getenv("SDCT_NO_PDL");
    return f && atoi(f) == 1;
  }();
  if (off) {
    k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Opt each kernel instantiation in to > 48 KB dynamic shared memory (once).
cudaError_t prep_smem_ptr(const void* kernel, size_t smem);
template <typename K>
inline cudaError_t prep_smem(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return prep_smem_ptr(reinterpret_cast<const void*>(kernel), smem);
}

template <typename T>
cudaError_t launch_col(int variant, int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                       const CUtensorMap& omap, const ColArgs& a, const TwSet& tw);
template <typename T>
cudaError_t launch_row(int M, int kind, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw);
// axis-0 1D DCT-II / DCT-III column pass (kernels_col1d.cuh), L in [8, 4096]
template <typename T>
cudaError_t launch_col1d(bool inv, int L, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                         const CUtensorMap& omap, const ColArgs& a, const TwSet& tw);
// persistent cluster-pair column pass (kernels_colc.cuh): fp64, L = 4096
cudaError_t launch_colc(bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                        const CUtensorMap& omap, const ColArgs& a, const TwSet& tw);
template <typename T>
cudaError_t launch_col2(int L, bool inv, int bands, int batch, cudaStream_t st, const CUtensorMap& map,
                        const CUtensorMap& omap, const ColArgs& a, const TwSet& tw);

// threads per CTA (host side, must match the kernels' compile-time geometry)
inline int tile_threads(int L, int nl) {
  int lg = 0;
  while ((1 << lg) < L) ++lg;
  const int S = lg == 0 ? 0 : (lg + 3) / 4;
  const int r0 = S == 0 ? 1 : 1 << (lg / S + (0 < lg % S ? 1 : 0));
  const int nt0 = L * nl / r0;
  return nt0 > 512 ? 512 : nt0;
}

// ---- per-variant implementation (included by the fast_col_*.cu units) -------
template <typename T, int L, int NL, int VAR>
cudaError_t launch_col_one(dim3 grid, cudaStream_t st, const CUtensorMap& map, const CUtensorMap& omap,
                           const ColArgs& a, const TwSet& tw) {
  constexpr bool INV = VAR == CV_INV_INTER || VAR == CV_INV_DST;
  constexpr int LD = VAR == CV_FWD_SRC ? LD_SRC : LD_INTER;
  constexpr int STO = VAR == CV_INV_DST ? ST_DST : ST_INTER;
  // persistent: one CTA per resident slot, each walking tiles
  auto k = col_kernel<T, L, NL, INV, LD, STO>;
  constexpr int NT = Tile<T, L, NL, true>::NT;
  // landing/exchange tile + half-tile staging + mbarrier
  const size_t tile = static_cast<size_t>(L) * NL * sizeof(cx_t<T>);
  const size_t smem = ((((tile + 127) & ~size_t(127)) + tile / 2 + 127) & ~size_t(127)) + 16;
  cudaError_t e = prep_smem(k, smem);
  if (e != cudaSuccess) return e;
  static const int resident = [&] {  // thread-safe one-time query (same on every B200)
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, smem);
    return sms * (per > 0 ? per : 1);
  }();
  ColArgs b = a;
  b.nbands = static_cast<int>(grid.x);
  b.nplanes = static_cast<int>(grid.y);
  b.ntiles = static_cast<int>(grid.x * grid.y * grid.z);
  const int ctas = b.ntiles < resident ? b.ntiles : resident;
  return launch_pdl(k, dim3(ctas), dim3(NT), smem, st, map, omap, b, tw);
}

template <typename T, int L, int VAR>
cudaError_t launch_col_L(int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map, const CUtensorMap& omap,
                         const ColArgs& a, const TwSet& tw) {
  constexpr int NLD = nl_default(sizeof(T), L);
  if (nl == NLD) return launch_col_one<T, L, NLD, VAR>(grid, st, map, omap, a, tw);
  if constexpr (NLD != 2) {
    if (nl == 2) return launch_col_one<T, L, 2, VAR>(grid, st, map, omap, a, tw);
  }
  if constexpr (NLD != 4 && sizeof(T) == 4) {
    if (nl == 4) return launch_col_one<T, L, 4, VAR>(grid, st, map, omap, a, tw);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int VAR>
cudaError_t launch_col_var(int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                           const CUtensorMap& omap, const ColArgs& a, const TwSet& tw) {
  switch (L) {
    case 2: return launch_col_L<T, 2, VAR>(nl, grid, st, map, omap, a, tw);
    case 4: return launch_col_L<T, 4, VAR>(nl, grid, st, map, omap, a, tw);
    case 8: return launch_col_L<T, 8, VAR>(nl, grid, st, map, omap, a, tw);
    case 16: return launch_col_L<T, 16, VAR>(nl, grid, st, map, omap, a, tw);
    case 32: return launch_col_L<T, 32, VAR>(nl, grid, st, map, omap, a, tw);
    case 64: return launch_col_L<T, 64, VAR>(nl, grid, st, map, omap, a, tw);
    case 128: return launch_col_L<T, 128, VAR>(nl, grid, st, map, omap, a, tw);
    case 256: return launch_col_L<T, 256, VAR>(nl, grid, st, map, omap, a, tw);
    case 512: return launch_col_L<T, 512, VAR>(nl, grid, st, map, omap, a, tw);
    case 1024: return launch_col_L<T, 1024, VAR>(nl, grid, st, map, omap, a, tw);
    case 2048: return launch_col_L<T, 2048, VAR>(nl, grid, st, map, omap, a, tw);
    case 4096: return launch_col_L<T, 4096, VAR>(nl, grid, st, map, omap, a, tw);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int VAR>
cudaError_t launch_col_variant(int L, int nl, dim3 grid, cudaStream_t st, const CUtensorMap& map,
                               const CUtensorMap& omap, const ColArgs& a, const TwSet& tw);

template <typename T, int M, bool INV, int MODE>
cudaError_t launch_row2(dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  auto k = row2_kernel<T, M, INV, MODE>;
  using Geo = Row2Geom<T, M, MODE>;
  cudaError_t e = prep_smem(k, Geo::SMEM);
  if (e != cudaSuccess) return e;
  static const int resident = [&] {  // thread-safe one-time query (same on every B200)
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, Geo::CTA, Geo::SMEM);
    return sms * (per > 0 ? per : 1);
  }();
  const int nitems = static_cast<int>(grid.x * grid.y);
  // MODE 0: persistent, at most one CTA per two items so both groups work;
  // MODE 2: persistent, one item at a time per CTA; MODE 1: one CTA per item
  const int want = MODE == 0 ? (nitems + 1) / 2 : nitems;
  const int ctas = want < resident || MODE == 1 ? want : resident;
  return launch_pdl(k, dim3(ctas), dim3(Geo::CTA), Geo::SMEM, st, a, tw, nitems);
}

template <typename T, int M, int KIND>
cudaError_t launch_row_one(dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  if constexpr (KIND == RK_FWD2 || KIND == RK_INV2) {
    if constexpr (rowp_ok<T, M, KIND == RK_INV2>()) {
      // fp64 M = 2048: the mirror-paired ring kernel (kernels_rowp.cuh);
      // SDCT_ROWP=0 selects the row2 schedules below (A/B)
      static const bool rowp = [] {
        const char* f = getenv("SDCT_ROWP");
        return !(f && atoi(f) == 0);
      }();
      if (rowp) {
        auto k = rowp_kernel<T, M, KIND == RK_INV2>;
        using Geo = RowpGeom<T, M>;
        cudaError_t e = prep_smem(k, Geo::SMEM);
        if (e != cudaSuccess) return e;
        static const int resident = [&] {
          int dev = 0, sms = 0, per = 0;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, Geo::CTA, Geo::SMEM);
          return sms * (per > 0 ? per : 1);
        }();
        const int nitems = static_cast<int>(grid.x * grid.y);
        const int want = (nitems + 1) / 2;
        return launch_pdl(k, dim3(want < resident ? want : resident), dim3(Geo::CTA), Geo::SMEM, st, a, tw, nitems);
      }
    }
    // measured on B200 (tools/stage_time.py): the forward kernel gains from
    // the persistent grouped ring; the inverse (heavier register use in its
    // preprocess) runs best as one item per CTA for long rows (M = 2048:
    // 92 vs 96 us fp64 at 4096^2) and in the ring for shorter ones (M = 1024:
    // 32.8 vs 34.8 us fp64 at 2048^2)
    static const int forced = [] {
      const char* f = getenv("SDCT_ROW2_MODE");  // developer override: 0 / 1
      return f ? atoi(f) : -1;
    }();
    // fp32 forward rows up to M = 1024: the split-prefetch CTA pair per SM
    // measured best (2048^2: 20.5 vs 22.5 us)
    const bool split = forced >= 0 ? forced == 2 : (KIND == RK_FWD2 && sizeof(T) == 4 && M <= 1024 && M >= 256);
    if (split) return launch_row2<T, M, KIND == RK_INV2, 2>(grid, st, a, tw);
    const bool one = forced >= 0 ? forced == 1 : (KIND == RK_INV2 && M > 1024);
    if (one || row2_mode<T, M>() == 1) return launch_row2<T, M, KIND == RK_INV2, 1>(grid, st, a, tw);
    if constexpr (row2_mode<T, M>() == 0) return launch_row2<T, M, KIND == RK_INV2, 0>(grid, st, a, tw);
    return cudaErrorInvalidValue;
  } else {
    constexpr int G = 4;
    auto k = row_kernel<T, M, KIND>;
    // + mbarrier; the staged 3D inverse keeps its four operand rows behind the tile
    const size_t smem = static_cast<size_t>(G) * M * sizeof(cx_t<T>) *
                            (KIND == RK_INV3 && row3_staged<T, M>() ? 2 : 1) + 16;
    cudaError_t e = prep_smem(k, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(k, grid, dim3(row_threads<T, M, KIND>()), smem, st, a, tw);
  }
}

template <typename T, int KIND>
cudaError_t launch_row_kind(int M, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw) {
  switch (M) {
    case 4: return launch_row_one<T, 4, KIND>(grid, st, a, tw);
    case 8: return launch_row_one<T, 8, KIND>(grid, st, a, tw);
    case 16: return launch_row_one<T, 16, KIND>(grid, st, a, tw);
    case 32: return launch_row_one<T, 32, KIND>(grid, st, a, tw);
    case 64: return launch_row_one<T, 64, KIND>(grid, st, a, tw);
    case 128: return launch_row_one<T, 128, KIND>(grid, st, a, tw);
    case 256: return launch_row_one<T, 256, KIND>(grid, st, a, tw);
    case 512: return launch_row_one<T, 512, KIND>(grid, st, a, tw);
    case 1024: return launch_row_one<T, 1024, KIND>(grid, st, a, tw);
    case 2048: return launch_row_one<T, 2048, KIND>(grid, st, a, tw);
    case 4096: return launch_row_one<T, 4096, KIND>(grid, st, a, tw);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int KIND>
cudaError_t launch_row_kind_ext(int M, dim3 grid, cudaStream_t st, const RowArgs& a, const TwSet& tw);

}  // namespace sdctb
