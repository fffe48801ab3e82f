// Microbenchmark (developer tool): data-movement floor of the persistent
// early-reissue column schedule (kernels_fast.cuh, col_xs): one CTA per SM,
// a 128 KB landing tile (4096 rows x 32 B of a 4096^2 fp64 matrix) whose next
// load is issued as soon as the threads have copied it to registers, and the
// tile written back through a 64 KB staging buffer in four 32 KB quarter
// stores (two quarter buffers) - the col_xs kernel without the FFT.
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2110_01172_b200/csrc microbench_xs.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tma.cuh"

using namespace sdctb;

constexpr int ROWS = 4096, RB = 32, TILE = ROWS * RB, NT = 512;

__global__ void __launch_bounds__(NT, 1) k_xs(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out,
                                             int ntiles, int touch) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* stg = sm + TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + TILE + TILE / 2);
  const int t = threadIdx.x;
  auto issue = [&](int tile) {
    mbar_expect_tx(bar, TILE);
    for (int r0 = 0; r0 < ROWS; r0 += 256) tma_load_2d(sm + r0 * RB, &in, tile * (RB / 8), r0, bar);
  };
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  if (t == 0 && blockIdx.x < ntiles) issue(blockIdx.x);
  uint32_t ph = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    mbar_wait(bar, ph);
    ph ^= 1;
    // 16 x 16 B per thread into registers (the stage-0 operand read)
    double2 v[16];
    const double2* s2 = reinterpret_cast<const double2*>(sm);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = s2[r * NT + t];
    __syncthreads();
    if (t == 0 && tile + gridDim.x < ntiles) {
      fence_async_smem();
      issue(tile + gridDim.x);
    }
    if (touch) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r].x += 1.0;
    }
    // four quarter stores through two 32 KB buffers
    for (int q = 0; q < 4; ++q) {
      if (t == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
      double2* sb = reinterpret_cast<double2*>(stg + (q & 1) * (TILE / 4));
#pragma unroll
      for (int r = 0; r < 4; ++r) sb[r * NT + t] = v[q * 4 + r];
      fence_async_smem();
      __syncthreads();
      if (t == 0) {
        for (int r0 = 0; r0 < ROWS / 4; r0 += 256)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&out),
                       "r"(tile * (RB / 8)), "r"(q * (ROWS / 4) + r0), "r"(smem_u32(reinterpret_cast<unsigned char*>(sb) + r0 * RB)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  cuuint32_t box[2] = {RB / 8, 256};
  cuuint32_t estr[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

int main() {
  double *a, *b;
  const long long cols = 4096, rows = 4096;
  cudaMalloc(&a, cols * rows * 8);
  cudaMalloc(&b, cols * rows * 8);
  cudaMemset(a, 0, cols * rows * 8);
  CUtensorMap mi = map2d(a, cols, rows), mo = map2d(b, cols, rows);
  const int ntiles = static_cast<int>(cols * 8 / RB);
  const size_t smem = TILE + TILE / 2 + 64;
  cudaFuncSetAttribute(k_xs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int touch = 0; touch < 2; ++touch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k_xs<<<sms, NT, smem>>>(mi, mo, ntiles, touch);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k_xs<<<sms, NT, smem>>>(mi, mo, ntiles, touch);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("persistent early-reissue movement, 128 KB tiles, 1 CTA/SM (touch %d): %.1f us  %.0f GB/s  err=%s\n", touch,
           ms * 1e3, 2.0 * cols * rows * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
