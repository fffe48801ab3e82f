// Microbenchmark (developer tool): loading the column pass's 4096-row x 32-B
// bands (row pitch 32 KB, 4096^2 fp64) into shared memory with TMA boxes vs
// LSU cp.async (LDGSTS, 16 B per thread), each followed by the same TMA store
// of the band. One 128 KB tile per CTA, one CTA per SM at a time.
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2110_01172_b200/csrc microbench_ldgsts.cu -o microbench_ldgsts
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tma.cuh"

using namespace sdctb;
constexpr int ROWS = 4096, RB = 32, PITCH = 32768, NT = 512;

template <bool LSU, bool STORE>
__global__ void __launch_bounds__(NT) k_mv(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out,
                                           const unsigned char* __restrict__ src, int reps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ROWS * RB);
  const int t = threadIdx.x;
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    const int band = (blockIdx.x + rep * gridDim.x) & 1023;
    const int c0 = band * (RB / 8);
    if (LSU) {
      // thread t: 16-B half (t & 1) of rows t/2, t/2 + 256, ...
      const unsigned char* g = src + static_cast<size_t>(band) * RB + (t & 1) * 16;
#pragma unroll 4
      for (int r = t >> 1; r < ROWS; r += NT / 2) {
        const uint32_t d = smem_u32(sm + r * RB + (t & 1) * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g + static_cast<size_t>(r) * PITCH) : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    } else {
      if (t == 0) {
        mbar_expect_tx(bar, ROWS * RB);
        for (int r0 = 0; r0 < ROWS; r0 += 256) tma_load_2d(sm + r0 * RB, &in, c0, r0, bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
    }
    if (STORE) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (t == 0) {
        for (int r0 = 0; r0 < ROWS; r0 += 256)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&out),
                       "r"(c0), "r"(r0), "r"(smem_u32(sm + r0 * RB))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    __syncthreads();
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  cudaDriverEntryPointQueryResult q;
  void* f;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}

static CUtensorMap map2d(void* base) {
  CUtensorMap m;
  cuuint64_t dims[2] = {4096, ROWS};
  cuuint64_t strides[1] = {PITCH};
  cuuint32_t box[2] = {RB / 8, 256}, es[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

template <bool LSU, bool STORE>
static void run(const char* name, void* a, void* b, int sms) {
  auto k = k_mv<LSU, STORE>;
  const size_t smem = ROWS * RB + 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  CUtensorMap mi = map2d(a), mo = map2d(b);
  const int reps = 7;  // 148 CTAs x 7 tiles ~ the 1024 bands of one pass
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<<<sms, NT, smem>>>(mi, mo, (const unsigned char*)a, reps);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k<<<sms, NT, smem>>>(mi, mo, (const unsigned char*)a, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / 20, bytes = (double)sms * reps * ROWS * RB * (STORE ? 2 : 1);
  printf("%-28s %7.1f us per %d tiles  %6.0f GB/s  (%s)\n", name, us, sms * reps, bytes / us / 1e3,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *a, *b;
  cudaMalloc(&a, (size_t)ROWS * PITCH);
  cudaMalloc(&b, (size_t)ROWS * PITCH);
  cudaMemset(a, 0, (size_t)ROWS * PITCH);
  run<false, false>("TMA load only", a, b, sms);
  run<true, false>("LDGSTS load only", a, b, sms);
  run<false, true>("TMA load + TMA store", a, b, sms);
  run<true, true>("LDGSTS load + TMA store", a, b, sms);
  return 0;
}
