// Microbenchmark (developer tool): achievable bandwidth of the column-pass
// data movement on B200 without any FFT math. A "tile" is ROWS rows x 32 B of
// a row-major matrix (row pitch PITCH bytes), exactly the band the column
// kernels move. Variants:
//   0: TMA tile load -> smem -> STG 16 B/lane back out (same 32-B pattern)
//   1: TMA tile load -> smem -> TMA tile store
//   2: LDG 16 B/lane -> registers -> STG
//   3: TMA load -> smem -> STG into a band-contiguous ("tile-major") layout
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2110_01172_b200/csrc
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "tma.cuh"

using namespace sdctb;

template <int ROWS>
__global__ void __launch_bounds__(512) k_tma_stg(const __grid_constant__ CUtensorMap in, double2* out, long long pitch2,
                                                  int layout) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ROWS * 32);
  const int t = threadIdx.x, band = blockIdx.x;
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(bar, ROWS * 32);
    for (int r0 = 0; r0 < ROWS; r0 += 256) tma_load_2d(sm + r0 * 32, &in, band * 4, r0, bar);
  }
  mbar_wait(bar, 0);
  const double2* s = reinterpret_cast<const double2*>(sm);
  for (int i = t; i < ROWS * 2; i += blockDim.x) {
    const int row = i >> 1, h = i & 1;
    double2 v = s[i];
    v.x += 1.0;
    if (layout == 0) out[row * pitch2 + band * 2 + h] = v;
    else out[static_cast<long long>(band) * ROWS * 2 + i] = v;
  }
}

template <int ROWS>
__global__ void __launch_bounds__(512) k_tma_tma(const __grid_constant__ CUtensorMap in,
                                                  const __grid_constant__ CUtensorMap out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ROWS * 32);
  const int t = threadIdx.x, band = blockIdx.x;
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(bar, ROWS * 32);
    for (int r0 = 0; r0 < ROWS; r0 += 256) tma_load_2d(sm + r0 * 32, &in, band * 4, r0, bar);
  }
  mbar_wait(bar, 0);
  double2* s = reinterpret_cast<double2*>(sm);
  for (int i = t; i < ROWS * 2; i += blockDim.x) s[i].x += 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    for (int r0 = 0; r0 < ROWS; r0 += 256)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&out),
                   "r"(band * 4), "r"(r0), "r"(smem_u32(sm + r0 * 32))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();
}

template <int ROWS>
__global__ void __launch_bounds__(512) k_ldg_stg(const double2* in, double2* out, long long pitch2) {
  const int t = threadIdx.x, band = blockIdx.x;
  constexpr int PER = 16;
  for (int i0 = t; i0 < ROWS * 2; i0 += blockDim.x * PER) {
    double2 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < ROWS * 2) v[u] = __ldg(in + (i >> 1) * pitch2 + band * 2 + (i & 1));
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < ROWS * 2) {
        v[u].x += 1.0;
        out[(i >> 1) * pitch2 + band * 2 + (i & 1)] = v[u];
      }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

static CUtensorMap map2d(void* base, long long cols, long long rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)(cols * 8)};
  cuuint32_t box[2] = {4, 256};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", r);
  return m;
}

template <int ROWS>
void run(const char* name, int variant, double* a, double* b, long long cols) {
  const int bands = static_cast<int>(cols / 4);
  CUtensorMap mi = map2d(a, cols, ROWS), mo = map2d(b, cols, ROWS);
  const size_t smem = ROWS * 32 + 16;
  cudaFuncSetAttribute(k_tma_stg<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tma_tma<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    if (variant == 0) k_tma_stg<ROWS><<<bands, 512, smem>>>(mi, reinterpret_cast<double2*>(b), cols / 2, 0);
    if (variant == 1) k_tma_tma<ROWS><<<bands, 512, smem>>>(mi, mo);
    if (variant == 2) k_ldg_stg<ROWS><<<bands, 512>>>(reinterpret_cast<double2*>(a), reinterpret_cast<double2*>(b), cols / 2);
    if (variant == 3) k_tma_stg<ROWS><<<bands, 512, smem>>>(mi, reinterpret_cast<double2*>(b), cols / 2, 1);
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double bytes = 2.0 * ROWS * cols * 8;
  printf("%-34s rows=%5d cols=%6lld  %8.1f us  %7.0f GB/s  err=%s\n", name, ROWS, cols, ms * 1e3, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *a, *b;
  const size_t n = 4096ull * 4096ull;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  run<4096>("tma load + stg 32B rows (128KB)", 0, a, b, 4096);
  run<4096>("tma load + tma store (128KB)", 1, a, b, 4096);
  run<4096>("ldg + stg 32B rows", 2, a, b, 4096);
  run<4096>("tma load + stg tile-major (128KB)", 3, a, b, 4096);
  run<2048>("tma load + stg 32B rows (64KB)", 0, a, b, 8192);
  run<2048>("tma load + tma store (64KB)", 1, a, b, 8192);
  run<2048>("tma load + stg tile-major (64KB)", 3, a, b, 8192);
  run<1024>("tma load + stg 32B rows (32KB)", 0, a, b, 16384);
  run<1024>("tma load + tma store (32KB)", 1, a, b, 16384);
  // reference: a plain coalesced copy
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemcpy(b, a, n * 8, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) cudaMemcpy(b, a, n * 8, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-34s %8.1f us  %7.0f GB/s\n", "cudaMemcpy D2D 134MB", ms / 20 * 1e3, 2.0 * n * 8 / (ms / 20) / 1e6);
  return 0;
}
