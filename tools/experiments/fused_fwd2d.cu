// EXPERIMENT (not built: build.py compiles csrc/ only). Single cooperative launch of the
// forward 2D DCT measured no faster than the two PDL-chained kernels on B200 at 1024^2
// (fp64 16.2 vs 15.7 us, fp32 13.4 vs 11.4 us per graph-replayed call); kept for the record.

// Single-launch forward 2D DCT for small images (one wave of tiles): the
// column pass (col_body, kernels_fast.cuh) and the mirror-paired forward row
// pass (rowp_body, kernels_rowp.cuh) run as two phases of one cooperative
// kernel separated by a grid-wide barrier, the intermediate staying in L2.
//
// Why: at 1024^2 fp64 each pass is one wave whose CTAs spend ~4 us on their
// tile, but a pass boundary costs the previous grid's drain, the dependency
// resolution and the next grid's first load latency (~3 us each, measured with
// per-kernel CUDA graphs). One launch keeps one boundary: the grid barrier.
//
// Phase 1 ends with every CTA's TMA stores complete (bulk_wait_all in
// col_body); the barrier orders them (async proxy -> generic -> other SMs'
// async-proxy bulk loads) with proxy fences on both sides.
//
// Reference stages replaced: dct_2d (proj/src/dct2d.cpp:367-387) = parity
// gather + rfft_nd + fused postprocess, exactly as the two-kernel path.
#include <cooperative_groups.h>

#include "fast_launch.cuh"

namespace sdctb {

namespace cg = cooperative_groups;

__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, int L, int NL, int M>
struct FusedGeom {
  using CT = Tile<T, L, NL, true>;
  using RG = RowpGeom<T, M>;
  static constexpr int NT = CT::NT;
  static constexpr uint32_t TILE = static_cast<uint32_t>(L) * 2 * NL * sizeof(T);
  static constexpr uint32_t STG_OFF = (TILE + 127u) & ~127u;
  static constexpr uint32_t BAR_OFF = (STG_OFF + TILE / 2 + 127u) & ~127u;  // col_body's mbarrier
  static constexpr size_t COL_SMEM = BAR_OFF + 16;
  static constexpr size_t SMEM = COL_SMEM > RG::SMEM ? COL_SMEM : RG::SMEM;
  static constexpr bool OK = NT == RG::CTA && rowp_ok<T, M, false>();
};

template <typename T, int L, int NL, int M>
__global__ void __launch_bounds__(FusedGeom<T, L, NL, M>::NT)
    fused_fwd2d_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ColArgs ca,
                       TwSet twc, RowArgs ra, TwSet twr, int nitems) {
  using G = FusedGeom<T, L, NL, M>;
  static_assert(G::OK, "fused forward 2D: column tile threads must equal the row CTA");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int cta = static_cast<int>(blockIdx.x), ncta = static_cast<int>(gridDim.x);
  col_body<T, L, NL, false, LD_SRC, ST_INTER>(tin, tout, ca, twc, cta, ncta);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_inval(reinterpret_cast<uint64_t*>(smem_raw + G::BAR_OFF));  // smem is reused by phase 2
    asm volatile("fence.proxy.async.global;" ::: "memory");           // bulk stores -> generic
  }
  cg::this_grid().sync();
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic -> bulk loads
  __syncthreads();
  rowp_body<T, M, false>(ra, twr, nitems, cta, ncta);
}

template <typename T, int L, int NL, int M>
cudaError_t launch_fused_one(int ntiles_needed, int nitems, cudaStream_t st, const CUtensorMap& map,
                             const CUtensorMap& omap, const ColArgs& ca, const TwSet& twc, const RowArgs& ra,
                             const TwSet& twr) {
  using G = FusedGeom<T, L, NL, M>;
  auto k = fused_fwd2d_kernel<T, L, NL, M>;
  cudaError_t e = prep_smem(k, G::SMEM);
  if (e != cudaSuccess) return e;
  static const int resident = [&] {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, G::NT, G::SMEM);
    return sms * per;
  }();
  // every CTA takes at most one column tile and two row items (one per group)
  const int want = std::max(ntiles_needed, (nitems + 1) / 2);
  if (want > resident) return cudaErrorCooperativeLaunchTooLarge;
  ColArgs c = ca;
  c.ntiles = ntiles_needed;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(want);
  cfg.blockDim = dim3(G::NT);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, map, omap, c, twc, ra, twr, nitems);
}

// (dtype, L, NL, M) geometries with matching thread counts; returns
// cudaErrorNotSupported for any other geometry (caller runs two kernels)
template <typename T>
cudaError_t launch_fused_fwd2d(int L, int nl, int M, int ntiles, int nitems, cudaStream_t st, const CUtensorMap& map,
                               const CUtensorMap& omap, const ColArgs& ca, const TwSet& twc, const RowArgs& ra,
                               const TwSet& twr) {
  if constexpr (FusedGeom<T, 1024, 2, 512>::OK) {
    if (L == 1024 && nl == 2 && M == 512)
      return launch_fused_one<T, 1024, 2, 512>(ntiles, nitems, st, map, omap, ca, twc, ra, twr);
  }
  if constexpr (FusedGeom<T, 2048, 2, 1024>::OK) {
    if (L == 2048 && nl == 2 && M == 1024)
      return launch_fused_one<T, 2048, 2, 1024>(ntiles, nitems, st, map, omap, ca, twc, ra, twr);
  }
  return cudaErrorNotSupported;
}

template cudaError_t launch_fused_fwd2d<float>(int, int, int, int, int, cudaStream_t, const CUtensorMap&,
                                               const CUtensorMap&, const ColArgs&, const TwSet&, const RowArgs&,
                                               const TwSet&);
template cudaError_t launch_fused_fwd2d<double>(int, int, int, int, int, cudaStream_t, const CUtensorMap&,
                                                const CUtensorMap&, const ColArgs&, const TwSet&, const RowArgs&,
                                                const TwSet&);

}  // namespace sdctb
