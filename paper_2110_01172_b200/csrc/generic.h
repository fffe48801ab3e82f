// Host-side description of one generic-path job (any extents, rank 1..3).
#pragma once

#include <cuda_runtime.h>

namespace sdctb {

struct GenericJob {
  int rank = 2;
  int dims[3] = {1, 1, 1};
  long long batch = 1;
  bool inverse = false;
  int mode = 0;          // inverse composite embedding: 0 none, 1 axis 0, 2 axis 1 (rank 1: 2 = idxst)
  int sign_axis = -1;    // inverse: negate odd k along this axis
  double scale = 1.0;    // inverse gather scale (1/4 in 2D, 1/8 in 3D, 1/2 in 1D)
  bool legacy = false;   // 2D: force the one-pass-per-stage pipeline (developer A/B; no kind sets it)
  const double2* quarter[3] = {nullptr, nullptr, nullptr};  // e^{-i pi k/(2 N_a)}
  const double2* circle[3] = {nullptr, nullptr, nullptr};   // e^{-2 pi i t / N_a}
  // Bluestein tables of axes whose largest prime factor is large (2D
  // pipeline): chirp c_j = e^{-i pi j^2 / N} (j < N), bhat = FFT_M of the
  // conjugate chirp wrapped to length M (pow2 >= 2N-1), circle of length M
  int blue_m[3] = {0, 0, 0};
  const double2* blue_chirp[3] = {nullptr, nullptr, nullptr};
  const double2* blue_hat[3] = {nullptr, nullptr, nullptr};
  const double2* blue_circle[3] = {nullptr, nullptr, nullptr};
  const double2* blue_fa[3] = {nullptr, nullptr, nullptr};  // circle of min(M, 4096)
  // global pass: stage tables of the min(M, 4096)-point column FFT, bhat in its
  // [plane k2][storage row rt_srow(k1)] order
  const void* blue_st[3][4] = {};
  const double2* blue_hatp[3] = {nullptr, nullptr, nullptr};
  // the plan's generic workspace carries the global Bluestein scratch
  // (bluestein_scratch_elems); generic_run points blue_ws at it
  bool blue_scratch = false;
  double2* blue_ws = nullptr;
};

// Bluestein length for an axis of extent n (0 = mixed radix is used): the
// pow2 M >= 2n - 1 when n's largest prime factor exceeds 64 (n <= 2^23), or,
// for an axis of a two-pass tile (tile = true, M <= kG2MaxN), when its prime
// factors above 7 sum to more than 20 M / n.
int bluestein_len(int n, bool tile);

// The two-pass 2D pipeline (g2_kernel) holds lines of up to kG2MaxN points
// (Bluestein convolution lengths included); other shapes run one pass per
// stage, with long Bluestein axes as global M-point line FFTs.
constexpr int kG2MaxN = 8192;
bool generic_two_pass(int rank, const int* dims, const int* blue_m);

// Lines per chunk of the global Bluestein pass (bounds its scratch) and the
// scratch it needs, in double2 elements (0 when no axis uses it).
long long bluestein_chunk_lines(int M, long long lines);
long long bluestein_scratch_elems(int rank, const int* dims, const int* blue_m, long long batch);

// Opt a kernel in to `smem` bytes of dynamic shared memory on the current
// device (cached per device and kernel; plan.cu).
cudaError_t prep_smem_ptr(const void* kernel, size_t smem);

// Batched complex FFT of `planes` x L rows x W lines (lines innermost, W even)
// through the fast column kernel (plan.cu): forward rows natural -> rt_srow
// order (DIF), inverse the reverse (DIT), unnormalised; st = its stage tables.
cudaError_t bluestein_line_fft(const double2* src, double2* dst, int L, int W, int planes, bool inverse,
                               const void* const st_tables[4], cudaStream_t st);

// Workspace: (2 * numel * batch + bluestein_scratch_elems) * sizeof(double2) bytes.
template <typename T>
cudaError_t generic_run(const GenericJob& job, const void* in, void* out, void* ws, cudaStream_t st);

// rfft_nd / irfft_nd of the reference (rfft.cpp:182-245), fp64, on the
// job's rank/dims/batch and circle tables. `half` is the one-sided spectrum
// [batch][dims..., last/2+1] of interleaved complex; ws = generic scratch.
cudaError_t generic_rfft(const GenericJob& job, const double* x, double2* half, void* ws, cudaStream_t st);
cudaError_t generic_irfft(const GenericJob& job, const double2* half, double* x, void* ws, cudaStream_t st);
// dft_naive (rfft.cpp:113-127): O(n^2) direct DFT of n complex values (device buffers).
cudaError_t dft_naive_run(const double2* in, double2* out, int n, bool inverse, cudaStream_t st);

// DREAMPlace-style field weighting (proj/src/force.cpp:19-31): aw = a * w_which /
// (w1^2 + w2^2), w_d = pi k_d / n_d, 0 at DC. dtype float when f32.
cudaError_t force_weight(const void* a, void* aw, int n1, int n2, long long batch, int which, bool f32,
                         cudaStream_t st);

// Compression threshold (proj/src/compress.cpp:37-45): out = |b| < eps ? 0 : b * scale,
// zeroed coefficients added to *count (device counter, may be null).
cudaError_t compress_threshold(const void* b, void* out, long long n, double eps, double scale,
                               unsigned long long* count, bool f32, cudaStream_t st);

}  // namespace sdctb
