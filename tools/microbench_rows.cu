// Microbenchmark (developer tool): achievable HBM rate of the row-pair data
// movement of the row kernels, without FFT math. One item = two rows of
// ROWB bytes read by 1D bulk copies into smem and written back out by
// coalesced 16-B stores. Variants:
//   0: one item per CTA (non-persistent), NT threads
//   1: persistent, ring of NB buffers, one group
//   2: LDG.128 -> STG.128 grid-stride copy (reference)
//   3: cudaMemcpy D2D
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2110_01172_b200/csrc microbench_rows.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tma.cuh"

using namespace sdctb;

template <int ROWB, int NT>
__global__ void __launch_bounds__(NT) k_item(const char* in, char* out, int nitems) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * ROWB);
  const int t = threadIdx.x, it = blockIdx.x;
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  const long long r0 = it, r1 = 2LL * nitems - 1 - it;
  if (t == 0) {
    mbar_expect_tx(bar, 2 * ROWB);
    bulk_load(sm, in + r0 * ROWB, ROWB, bar);
    bulk_load(sm + ROWB, in + r1 * ROWB, ROWB, bar);
  }
  mbar_wait(bar, 0);
  const double2* s = reinterpret_cast<const double2*>(sm);
  for (int i = t; i < 2 * ROWB / 16; i += NT) {
    const long long row = i < ROWB / 16 ? r0 : r1;
    const int c = i % (ROWB / 16);
    reinterpret_cast<double2*>(out + row * ROWB)[c] = s[i];
  }
}

template <int ROWB, int NT, int NB>
__global__ void __launch_bounds__(NT) k_ring(const char* in, char* out, int nitems) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * 2 * ROWB);
  const int t = threadIdx.x;
  auto issue = [&](int it, int b) {
    const long long r0 = it, r1 = 2LL * nitems - 1 - it;
    mbar_expect_tx(bar + b, 2 * ROWB);
    bulk_load(sm + b * 2 * ROWB, in + r0 * ROWB, ROWB, bar + b);
    bulk_load(sm + b * 2 * ROWB + ROWB, in + r1 * ROWB, ROWB, bar + b);
  };
  if (t == 0)
    for (int b = 0; b < NB; ++b) mbar_init(bar + b, 1);
  __syncthreads();
  if (t == 0)
    for (int b = 0; b < NB; ++b)
      if (blockIdx.x + b * gridDim.x < nitems) issue(blockIdx.x + b * gridDim.x, b);
  int k = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++k) {
    const int b = k % NB;
    mbar_wait(bar + b, (k / NB) & 1);
    const long long r0 = it, r1 = 2LL * nitems - 1 - it;
    const double2* s = reinterpret_cast<const double2*>(sm + b * 2 * ROWB);
    for (int i = t; i < 2 * ROWB / 16; i += NT) {
      const long long row = i < ROWB / 16 ? r0 : r1;
      const int c = i % (ROWB / 16);
      reinterpret_cast<double2*>(out + row * ROWB)[c] = s[i];
    }
    __syncthreads();
    if (t == 0 && it + NB * gridDim.x < nitems) {
      fence_async_smem();
      issue(it + NB * gridDim.x, b);
    }
  }
}

__global__ void k_copy(const double2* in, double2* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

template <class F>
void timeit(const char* name, F f, double bytes, char* flush) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9, tot = 0;
  for (int i = 0; i < 12; ++i) {
    if (flush) cudaMemsetAsync(flush, i, 256 << 20);
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 2) {
      best = ms < best ? ms : best;
      tot += ms;
    }
  }
  printf("%-46s %s  best %7.1f us %6.0f GB/s   mean %7.1f us  err=%s\n", name, flush ? "dirtyL2" : "back2bk", best * 1e3,
         bytes / best / 1e6, tot / 10 * 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t n = 4096ull * 4096ull * 8;  // 134 MB
  char *a, *b, *fl;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMalloc(&fl, 256 << 20);
  cudaMemset(a, 1, n);
  constexpr int ROWB = 32768;
  const int nitems = static_cast<int>(n / (2 * ROWB));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (char* flush : {(char*)nullptr, fl}) {
    {
      auto k = k_item<ROWB, 256>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWB + 16);
      timeit("item/CTA 64KB, 256 thr", [&] { k<<<nitems, 256, 2 * ROWB + 16>>>(a, b, nitems); }, 2.0 * n, flush);
    }
    {
      auto k = k_item<ROWB, 512>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWB + 16);
      timeit("item/CTA 64KB, 512 thr", [&] { k<<<nitems, 512, 2 * ROWB + 16>>>(a, b, nitems); }, 2.0 * n, flush);
    }
    {
      auto k = k_ring<ROWB, 256, 3>;
      const int sm = 3 * 2 * ROWB + 64;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      timeit("ring3 64KB, 256 thr, 1 CTA/SM", [&] { k<<<sms, 256, sm>>>(a, b, nitems); }, 2.0 * n, flush);
    }
    {
      auto k = k_ring<ROWB, 512, 3>;
      const int sm = 3 * 2 * ROWB + 64;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      timeit("ring3 64KB, 512 thr, 1 CTA/SM", [&] { k<<<sms, 512, sm>>>(a, b, nitems); }, 2.0 * n, flush);
    }
    {
      auto k = k_ring<ROWB / 2, 256, 3>;
      const int sm = 3 * ROWB + 64;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      timeit("ring3 32KB items, 256 thr, 2 CTA/SM", [&] { k<<<2 * sms, 256, sm>>>(a, b, 2 * nitems); }, 2.0 * n, flush);
    }
    timeit("ldg/stg copy 16B", [&] { k_copy<<<sms * 8, 512>>>((double2*)a, (double2*)b, n / 16); }, 2.0 * n, flush);
    timeit("cudaMemcpy D2D", [&] { cudaMemcpyAsync(b, a, n, cudaMemcpyDeviceToDevice); }, 2.0 * n, flush);
  }
  return 0;
}
