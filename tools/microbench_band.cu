// Microbenchmark (developer tool): HBM rate of the column-band movement with
// different band widths. One CTA per band: TMA tile load of ROWS rows x RB
// bytes (row pitch 32 KB) -> smem -> TMA tile store of the same band. RB = 16
// is the "one complex fp64 column" band; variant ES reads a 32-B quad with
// element stride 2 (two CTAs split one quad's even / odd reals).
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2110_01172_b200/csrc microbench_band.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tma.cuh"

using namespace sdctb;

template <int ROWS, int RB>
__global__ void __launch_bounds__(256) k_band(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out,
                                              int es) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ROWS * RB);
  const int t = threadIdx.x;
  // es: band b covers reals [4*(b/2), +4) with start (b&1) and element stride 2
  const int c0 = es ? 4 * (blockIdx.x >> 1) + (blockIdx.x & 1) : blockIdx.x * (RB / 8);
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(bar, ROWS * RB);
    for (int r0 = 0; r0 < ROWS; r0 += 256) tma_load_2d(sm + r0 * RB, &in, c0, blockIdx.y * ROWS + r0, bar);
  }
  mbar_wait(bar, 0);
  double* s = reinterpret_cast<double*>(sm);
  for (int i = t; i < ROWS * RB / 8; i += blockDim.x) s[i] += 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    for (int r0 = 0; r0 < ROWS; r0 += 256)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&out),
                   "r"(c0), "r"(static_cast<int>(blockIdx.y) * ROWS + r0), "r"(smem_u32(sm + r0 * RB))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();
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

static CUtensorMap map2d(void* base, long long cols, long long rows, int box0, int es) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)(cols * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box0, 256};
  cuuint32_t estr[2] = {(cuuint32_t)es, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d (box0 %d es %d)\n", r, box0, es);
  return m;
}

template <int ROWS, int RB>
void run(const char* name, double* a, double* b, long long cols, int es) {
  const long long rows = 4096ll * 4096 / cols;  // 134 MB matrix
  const int bands = es ? static_cast<int>(cols / 2) : static_cast<int>(cols * 8 / RB);
  const int box0 = es ? 4 : RB / 8;
  CUtensorMap mi = map2d(a, cols, rows, box0, es ? 2 : 1), mo = map2d(b, cols, rows, box0, es ? 2 : 1);
  const size_t smem = ROWS * RB + 16;
  cudaFuncSetAttribute(k_band<ROWS, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_band<ROWS, RB>, 256, smem);
  const int chunks = static_cast<int>(rows / ROWS);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() { k_band<ROWS, RB><<<dim3(bands, chunks), 256, smem>>>(mi, mo, es); };
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double bytes = 2.0 * rows * cols * 8;
  printf("%-40s rows=%5d rowB=%2d CTA/SM=%d  %8.1f us  %7.0f GB/s  err=%s\n", name, ROWS, RB, per, ms * 1e3,
         bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *a, *b;
  const size_t n = 4096ull * 4096ull;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  // all with rows == matrix height (one slab)
  run<4096, 32>("32-B rows, 4096-row tiles (128 KB)", a, b, 4096, 0);
  run<4096, 16>("16-B rows, 4096-row tiles (64 KB)", a, b, 4096, 0);
  // run<4096, 16>("quad es=2 halves, 4096-row tiles (64 KB)", a, b, 4096, 1);
  run<2048, 32>("32-B rows, 2048-row tiles (64 KB) [8192x2048]", a, b, 2048, 0);
  run<2048, 64>("64-B rows, 2048-row tiles (128 KB) [8192x2048]", a, b, 2048, 0);
  run<1024, 64>("64-B rows, 1024-row tiles (64 KB) [16384x1024]", a, b, 1024, 0);
  run<2048, 32>("32-B rows, 2048-row tiles (64 KB) [4096^2]", a, b, 4096, 0);
  run<2048, 16>("16-B rows, 2048-row tiles (32 KB) [4096^2]", a, b, 4096, 0);
  run<4096, 16>("quad es=2 halves, 4096-row tiles (64 KB)", a, b, 4096, 1);
  return 0;
}
