#include <cstdlib>
#include <algorithm>
// Generic path: any extents (odd, non-power-of-two, tiny), ranks 1..3, fp64
// arithmetic throughout (inputs/outputs may be fp32). It restates the
// reference's three stages one full-tensor pass at a time:
//   forward : parity gather (dct2d.cpp:48-70 / transforms_ext.cpp:165-183)
//             -> full complex DFT along each axis (direct sums with exact
//                table twiddles; replaces rfft.cpp's Bluestein for odd N)
//             -> per-output postprocess (the identity of dct2d.hpp:6-7 and its
//                3D analogue).
//   inverse : full Hermitian spectrum from the merged preprocess
//             (dct2d.cpp:161-198 / transforms_ext.cpp:187-216, Hermitian fill
//             as irfft_nd does, rfft.cpp:233-243) -> inverse DFT per axis ->
//             real part, inverse parity gather, scale and sign (214-238).
// It is the correctness path for shapes outside the power-of-two fast path;
// cost is O(numel * sum(radices of N_axis)) with the shared-memory mixed-radix
// line FFT (extents <= 4096), O(numel * N_axis) direct sums beyond.
#include "fft_block.cuh"
#include "generic.h"
#include "sdct_common.cuh"

namespace sdctb {

namespace {

constexpr int kThreads = 256;

inline int nblocks(long long n) {
  long long b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(b > 2147483647LL ? 2147483647LL : b);
}

struct Dims {
  int rank;
  int n[3];       // logical extents (rank entries used, outermost first)
  long long numel;
};

__device__ __forceinline__ void unflat(long long f, const Dims& d, int* idx) {
  for (int a = d.rank - 1; a >= 0; --a) {
    idx[a] = static_cast<int>(f % d.n[a]);
    f /= d.n[a];
  }
}

template <typename T>
__global__ void g_gather_fwd(const T* __restrict__ x, double2* __restrict__ c, Dims d, long long batch_items) {
  const long long total = d.numel * batch_items;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = f / d.numel;
    int idx[3];
    unflat(f - b * d.numel, d, idx);
    long long src = 0;
    for (int a = 0; a < d.rank; ++a) src = src * d.n[a] + parity_embed(idx[a], d.n[a]);
    c[f] = make_double2(static_cast<double>(x[b * d.numel + src]), 0.0);
  }
}

// out[o, k, i] = sum_m in[o, m, i] W_n^{+-m k}; tab[t] = e^{-2 pi i t / n}
__global__ void g_dft_axis(const double2* __restrict__ in, double2* __restrict__ out, long long outer,
                           int n, long long inner, const double2* __restrict__ tab, int inverse) {
  const long long total = outer * n * inner;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = f % inner;
    const long long rest = f / inner;
    const int k = static_cast<int>(rest % n);
    const long long o = rest / n;
    const double2* line = in + o * n * inner + i;
    double re = 0.0, im = 0.0;
    long long t = 0;
    for (int m = 0; m < n; ++m) {
      double2 w = tab[t];
      if (inverse) w.y = -w.y;
      const double2 v = line[m * inner];
      re += v.x * w.x - v.y * w.y;
      im += v.x * w.y + v.y * w.x;
      t += k;
      if (t >= n) t -= n;
    }
    out[f] = make_double2(re, im);
  }
}

// ---- mixed-radix line FFT (Stockham autosort in shared memory) -------------
// Replaces the O(n) direct sum per output with sum(radices) complex MACs per
// element for composite n (any factorisation; a prime factor p costs p MACs,
// so a prime extent degenerates to the direct sum, now from shared memory).
// One CTA owns LPC lines of one axis: LPC consecutive i (inner > 1, each
// step reads LPC contiguous elements) or LPC consecutive rows (inner == 1).
// Pass t (radix R, Ns = product of the previous radices), for each output:
//   y[(j / Ns) Ns R + j % Ns + k Ns] = sum_r x[j + r n/R] W_n^{r E},
//   E = (j % Ns) n / (Ns R) + k n / R  (twiddle and radix-R DFT fused).
// Division by a run-time constant d >= 1 for 0 <= x < 2^31 as one multiply-
// high, an add and a shift (m = floor(2^32 (2^s - d) / d) + 1, s = ceil(log2 d));
// the line FFTs' index math divides by line lengths and pass strides
// everywhere, and the generic integer division sequence dominated their
// instruction count. tests/test_host.py checks the formula.
struct FastDiv {
  unsigned d = 1, m = 1, s = 0;
  __host__ __device__ FastDiv() {}
  __host__ __device__ explicit FastDiv(unsigned dd) : d(dd) {
    while ((1u << s) < d) ++s;
    m = static_cast<unsigned>(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  }
  __device__ __forceinline__ int div(int x) const {
    return static_cast<int>((__umulhi(static_cast<unsigned>(x), m) + static_cast<unsigned>(x)) >> s);
  }
  __device__ __forceinline__ int mod(int x, int q) const { return x - q * static_cast<int>(d); }
};

struct Radices {
  int count;
  int r[24];
  FastDiv nr[24];  // n / r[s]
  FastDiv ns[24];  // product of r[0..s)
  FastDiv n;       // line length
};

constexpr int kFftMaxN = 4096;  // two line buffers + table in shared memory

constexpr int kFftPerThread = 8;  // outputs a thread holds across one pass (lines * n <= 8 * threads)

// Radix-R DFT constants W_R^m = e^{-+2 pi i m / R} for the odd radices
// (compile time; the powers of two use the in-register dft_reg of fft_block.cuh)
template <int R> struct OddRoots;
template <> struct OddRoots<3> {
  __device__ __forceinline__ static constexpr double c(int m) { return m == 0 ? 1.0 : -0.5; }
  __device__ __forceinline__ static constexpr double s(int m) {
    return m == 0 ? 0.0 : m == 1 ? 0.86602540378443864676 : -0.86602540378443864676;
  }
};
template <> struct OddRoots<5> {
  __device__ __forceinline__ static constexpr double c(int m) {
    return m == 0 ? 1.0 : (m == 1 || m == 4) ? 0.30901699437494742410 : -0.80901699437494742410;
  }
  __device__ __forceinline__ static constexpr double s(int m) {
    return m == 0 ? 0.0 : m == 1 ? 0.95105651629515357212 : m == 2 ? 0.58778525229247312917
         : m == 3 ? -0.58778525229247312917 : -0.95105651629515357212;
  }
};
template <> struct OddRoots<7> {
  __device__ __forceinline__ static constexpr double c(int m) {
    return m == 0 ? 1.0 : (m == 1 || m == 6) ? 0.62348980185873353053
         : (m == 2 || m == 5) ? -0.22252093395631440429 : -0.90096886790241912624;
  }
  __device__ __forceinline__ static constexpr double s(int m) {
    return m == 0 ? 0.0 : m == 1 ? 0.78183148246802980871 : m == 2 ? 0.97492791218182360702
         : m == 3 ? 0.43388373911755812048 : m == 4 ? -0.43388373911755812048
         : m == 5 ? -0.97492791218182360702 : -0.78183148246802980871;
  }
};

// in-register radix-R DFT, natural order: v[k] <- sum_r v[r] W_R^{r k}
template <int R, bool INV>
__device__ __forceinline__ void radix_dft(double2* v) {
  if constexpr ((R & (R - 1)) == 0) {
    dft_reg<double, R, INV>(v);
  } else {
    // symmetric form: with s_r = v[r] + v[R-r], d_r = v[r] - v[R-r]
    // (r = 1..H), out[k] = A_k -+ i B_k and out[R-k] = A_k +- i B_k, where
    // A_k = v0 + sum_r cos(2 pi r k / R) s_r, B_k = sum_r sin(2 pi r k / R) d_r
    constexpr int H = (R - 1) / 2;
    double2 sr[H], dr[H];
    double2 o0 = v[0];
#pragma unroll
    for (int r = 1; r <= H; ++r) {
      sr[r - 1] = make_double2(v[r].x + v[R - r].x, v[r].y + v[R - r].y);
      dr[r - 1] = make_double2(v[r].x - v[R - r].x, v[r].y - v[R - r].y);
      o0.x += sr[r - 1].x;
      o0.y += sr[r - 1].y;
    }
    double2 o[R];
    o[0] = o0;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double ax = v[0].x, ay = v[0].y, bx = 0.0, by = 0.0;
#pragma unroll
      for (int r = 1; r <= H; ++r) {
        const int m = (r * k) % R;
        const double c = OddRoots<R>::c(m), sn = OddRoots<R>::s(m);
        ax = fma(c, sr[r - 1].x, ax);
        ay = fma(c, sr[r - 1].y, ay);
        bx = fma(sn, dr[r - 1].x, bx);
        by = fma(sn, dr[r - 1].y, by);
      }
      // forward W = e^{-i theta}: out[k] = A - i B = (ax + by, ay - bx)
      if (!INV) {
        o[k] = make_double2(ax + by, ay - bx);
        o[R - k] = make_double2(ax - by, ay + bx);
      } else {
        o[k] = make_double2(ax - by, ay + bx);
        o[R - k] = make_double2(ax + by, ay - bx);
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = o[k];
  }
}

// One Stockham pass of radix R (compile time) over lines of length n in
// shared memory (line stride ld), in place: each thread takes whole
// butterflies j (inputs x[j + r n/R], r < R), applies the twiddles
// W_{ns R}^{(j % ns) r} from the table (already conjugated for the inverse)
// and the radix-R DFT with compile-time constants, keeps the R outputs in
// registers across the barrier and writes them to y[(j / ns) ns R + j % ns + k ns].
template <int R, int FPT, bool INV, bool CJ>
__device__ __forceinline__ void stockham_pass(double2* x, const double2* tw, int n, int ns, int total, int t,
                                              int nt, int ld, const FastDiv& fnr, const FastDiv& fns) {
  constexpr int BMAX = (FPT + R - 1) / R;  // butterflies per thread (lines * n <= FPT * nt)
  const int nr = n / R;
  const int nb = total / R;  // butterflies over all lines of the tile
  const int tstep = n / (ns * R);
  double2 out[BMAX][R];
  int jq[BMAX];  // j / ns, reused by the write-back
#pragma unroll
  for (int u = 0; u < BMAX; ++u) {
    const int bq = t + u * nt;
    if (bq < nb) {
      const int l = fnr.div(bq), j = bq - l * nr;
      jq[u] = fns.div(j);
      const int jr = j - jq[u] * ns;
      const double2* xl = x + l * ld + j;
      double2* v = out[u];
      v[0] = xl[0];
      const int e1 = jr * tstep;  // W_n^{e1 r} = W_{ns R}^{(j % ns) r}
      int e = e1;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 a = xl[r * nr];
        double2 w = tw[e];
        if (CJ && INV) w.y = -w.y;
        v[r] = make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
        e += e1;
        if (e >= n) e -= n;
      }
      radix_dft<R, INV>(v);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BMAX; ++u) {
    const int bq = t + u * nt;
    if (bq < nb) {
      const int l = fnr.div(bq), j = bq - l * nr;
      const int base = l * ld + jq[u] * ns * (R - 1) + j;  // (j / ns) ns R + j % ns
#pragma unroll
      for (int k = 0; k < R; ++k) x[base + k * ns] = out[u][k];
    }
  }
  __syncthreads();
}

// Radix-R pass for other (prime) R: one thread per output, R MACs each.
template <int FPT, bool CJ>
__device__ __forceinline__ void generic_pass(double2* x, const double2* tw, int n, int ns, int R, int total, int t,
                                             int nt, int ld, const FastDiv& fn, const FastDiv& fns) {
  const int nr = n / R;
  double2 acc[FPT];
#pragma unroll
  for (int u = 0; u < FPT; ++u) {
    const int e = t + u * nt;
    if (e < total) {
      const int l = fn.div(e), q = e - l * n;
      // output q = (j / ns) ns R + j % ns + k ns with j in [0, n/R), k in [0, R)
      const int rest = fns.div(q), jr = q - rest * ns;
      const int jq = rest / R, k = rest - jq * R;
      const int j = jq * ns + jr;
      const int E = (jr * (n / (ns * R)) + k * nr) % n;
      const double2* xl = x + l * ld + j;
      double re = 0.0, im = 0.0;
      int idx = 0;
      for (int r = 0; r < R; ++r) {
        const double2 v = xl[r * nr];
        double2 w = tw[idx];
        if (CJ) w.y = -w.y;
        re = fma(v.x, w.x, fma(-v.y, w.y, re));
        im = fma(v.x, w.y, fma(v.y, w.x, im));
        idx += E;
        if (idx >= n) idx -= n;
      }
      acc[u] = make_double2(re, im);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < FPT; ++u) {
    const int e = t + u * nt;
    if (e < total) {
      const int l = fn.div(e);
      x[l * ld + (e - l * n)] = acc[u];
    }
  }
  __syncthreads();
}

// All passes of one line FFT over `total` = lines * n elements in smem
// (line stride ld); tw holds e^{-+2 pi i e / n}.
// CJ: tw is the forward table and the inverse conjugates at use (tables read
// from global memory through L1); otherwise tw is already conjugated for INV.
template <int FPT, bool INV, bool CJ = false>
__device__ __forceinline__ void line_passes(double2* x, const double2* tw, int n, const Radices& rad, int total, int t,
                                            int nt, int ld) {
  // factorise() emits 8s, 4s, 2s, then odd primes in ascending order: one
  // loop per radix (a single switch over all radices inside one loop makes
  // ptxas keep the pass outputs in local memory)
  int ns = 1, s = 0;
  while (s < rad.count && rad.r[s] == 8) { stockham_pass<8, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 8; ++s; }
  while (s < rad.count && rad.r[s] == 4) { stockham_pass<4, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 4; ++s; }
  while (s < rad.count && rad.r[s] == 2) { stockham_pass<2, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 2; ++s; }
  while (s < rad.count && rad.r[s] == 3) { stockham_pass<3, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 3; ++s; }
  while (s < rad.count && rad.r[s] == 5) { stockham_pass<5, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 5; ++s; }
  while (s < rad.count && rad.r[s] == 7) { stockham_pass<7, FPT, INV, CJ>(x, tw, n, ns, total, t, nt, ld, rad.nr[s], rad.ns[s]); ns *= 7; ++s; }
  for (; s < rad.count; ++s) {
    generic_pass<FPT, CJ && INV>(x, tw, n, ns, rad.r[s], total, t, nt, ld, rad.n, rad.ns[s]);
    ns *= rad.r[s];
  }
}

// GTW (long lines, 2048..4096 points): 16 outputs per thread and the twiddles
// read from the global circle table through L1 (tab_stride 1), so the line
// alone fills shared memory and two CTAs share an SM (one 512-thread CTA with
// a 128 KB table + line per SM left the load latency exposed: ~1 TB/s)
template <int FPT, bool GTW>
__global__ void __launch_bounds__(GTW ? 256 : 512, GTW ? 2 : 1)
    g_fft_axis_smem(const double2* __restrict__ in, double2* __restrict__ out, long long outer, int n,
                    long long inner, const double2* __restrict__ tab, int tab_stride, int inverse, Radices rad,
                    int lpc) {
  // shared memory: twiddle table (n, !GTW) + the lines (lpc * n); each pass
  // computes its outputs into registers, synchronises, and writes them back in place
  extern __shared__ __align__(16) double2 fsm[];
  const double2* tw = GTW ? tab : fsm;
  double2* x = GTW ? fsm : fsm + n;
  const int t = threadIdx.x, nt = blockDim.x;
  if constexpr (!GTW) {
    for (int e = t; e < n; e += nt) {
      double2 w = tab[static_cast<long long>(e) * tab_stride];  // e^{-2 pi i e / n} from a longer circle table
      if (inverse) w.y = -w.y;
      fsm[e] = w;
    }
  }
  // tile of lines: (o, i0..i0+lpc) for inner > 1, rows o0..o0+lpc for inner == 1
  const long long tiles_per_o = inner > 1 ? inner / lpc : 1;
  const long long tile = blockIdx.x;
  long long o, i0;
  if (inner > 1) {
    o = tile / tiles_per_o;
    i0 = (tile % tiles_per_o) * lpc;
  } else {
    o = tile * lpc;
    i0 = 0;
  }
  const int lines = static_cast<int>(inner > 1 ? lpc : std::min<long long>(lpc, outer - o));
  const int total = lines * n;
  for (int e = t; e < total; e += nt) {
    long long src;
    int l, m;
    if (inner > 1) {
      m = e / lpc;
      l = e % lpc;
      src = (o * n + m) * inner + i0 + l;
    } else {
      l = e / n;
      m = e % n;
      src = (o + l) * n + m;
    }
    x[l * n + m] = in[src];
  }
  __syncthreads();
  if (inverse)
    line_passes<FPT, true, GTW>(x, tw, n, rad, total, t, nt, n);
  else
    line_passes<FPT, false, GTW>(x, tw, n, rad, total, t, nt, n);
  for (int e = t; e < total; e += nt) {
    long long dst;
    int l, m;
    if (inner > 1) {
      m = e / lpc;
      l = e % lpc;
      dst = (o * n + m) * inner + i0 + l;
    } else {
      l = e / n;
      m = e % n;
      dst = (o + l) * n + m;
    }
    out[dst] = x[l * n + m];
  }
}

// Split of a long axis n = a b (a, b <= kFftMaxN): the a-point FFTs over m1
// (element b m1 + m2 -> slot b k1 + m2) run as line FFTs; this kernel then
// finishes X(k) = sum_{m2 < b} Y(k1, m2) W_n^{m2 k}, k = k1 + a k2 (the
// twiddle, the b-point DFT and the output permutation in one pass; b is the
// small cofactor).
__global__ void g_split_finish(const double2* __restrict__ y, double2* __restrict__ out, long long outer, int a, int b,
                               long long inner, const double2* __restrict__ tab, int inverse) {
  const long long n = static_cast<long long>(a) * b;
  const long long total = outer * n * inner;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = f % inner, rest = f / inner;
    const long long k = rest % n, o = rest / n;
    const long long k1 = k % a;
    const double2* src = y + (o * n + b * k1) * inner + i;
    double re = 0.0, im = 0.0;
    long long idx = 0;
    for (int m2 = 0; m2 < b; ++m2) {
      double2 w = tab[idx];
      if (inverse) w.y = -w.y;
      const double2 v = src[m2 * inner];
      re = fma(v.x, w.x, fma(-v.y, w.y, re));
      im = fma(v.x, w.y, fma(v.y, w.x, im));
      idx += k;
      if (idx >= n) idx -= n;
    }
    out[f] = make_double2(re, im);
  }
}

// Batched transpose [o][r][c] -> [o][c][r] through 32 x 32 smem tiles.
__global__ void g_transpose_k(const double2* __restrict__ in, double2* __restrict__ out, long long rows,
                              long long cols) {
  __shared__ double2 tile[32][33];
  const long long o = blockIdx.z;
  const long long r0 = static_cast<long long>(blockIdx.y) * 32, c0 = static_cast<long long>(blockIdx.x) * 32;
  const double2* src = in + o * rows * cols;
  double2* dst = out + o * rows * cols;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][dy];
  }
}

void g_transpose(const double2* in, double2* out, long long outer, long long rows, long long cols, cudaStream_t st) {
  // grid.z carries the outer index (chunked when it exceeds the 65535 limit)
  for (long long o0 = 0; o0 < outer; o0 += 65535) {
    const long long oc = std::min<long long>(65535, outer - o0);
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32),
              static_cast<unsigned>(oc));
    g_transpose_k<<<grid, dim3(32, 8), 0, st>>>(in + o0 * rows * cols, out + o0 * rows * cols, rows, cols);
  }
}

// a * b = n with both factors <= kFftMaxN (a the larger), or {0, 0}
void split_factors(int n, int& a, int& b) {
  a = b = 0;
  for (int d = kFftMaxN; d >= 2; --d)
    if (n % d == 0 && n / d <= kFftMaxN) {
      a = d;
      b = n / d;
      return;
    }
}

Radices factorise(int n) {
  const int n0 = n;
  Radices rad{};
  // radix 8/4/2 first, then small odd primes, then whatever prime remains
  for (int r : {8, 4, 2}) {
    while (n % r == 0 && rad.count < 24) {
      rad.r[rad.count++] = r;
      n /= r;
    }
  }
  for (int p = 3; n > 1 && rad.count < 24; p += 2) {
    while (n % p == 0 && rad.count < 24) {
      rad.r[rad.count++] = p;
      n /= p;
    }
    if (p * p > n && n > 1) {
      rad.r[rad.count++] = n;
      n = 1;
    }
  }
  int ns = 1;
  for (int q = 0; q < rad.count; ++q) {
    rad.nr[q] = FastDiv(static_cast<unsigned>(n0 / rad.r[q]));
    rad.ns[q] = FastDiv(static_cast<unsigned>(ns));
    ns *= rad.r[q];
  }
  rad.n = FastDiv(static_cast<unsigned>(n0));
  return rad;
}

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 ca(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// 1D: y(k) = Re(b(k) X(k))             (dct1d N-point postprocess, scale 1)
// 2D: y = 1/2 Re(b (a X(k1,k2) + conj(a) X(-k1,k2)))               (dct2d.hpp:6)
// 3D: y = 1/4 Re(c (ab X + conj(a) b X(-k1) + a conj(b) X(-k2) + conj(ab) X(-k1,-k2)))
template <typename T>
__global__ void g_post(const double2* __restrict__ X, T* __restrict__ y, Dims d, long long batch_items,
                       const double2* __restrict__ ta, const double2* __restrict__ tb,
                       const double2* __restrict__ tc) {
  const long long total = d.numel * batch_items;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = f / d.numel;
    const double2* Xb = X + b * d.numel;
    int k[3];
    unflat(f - b * d.numel, d, k);
    double v;
    if (d.rank == 1) {
      v = cm(ta[k[0]], Xb[k[0]]).x;
    } else if (d.rank == 2) {
      const int n1 = d.n[0], n2 = d.n[1];
      const int r1 = (n1 - k[0]) % n1;
      const double2 a = ta[k[0]];
      const double2 x1 = Xb[static_cast<long long>(k[0]) * n2 + k[1]];
      const double2 x2 = Xb[static_cast<long long>(r1) * n2 + k[1]];
      v = 0.5 * cm(tb[k[1]], ca(cm(a, x1), cm(cj(a), x2))).x;
    } else {
      const int n1 = d.n[0], n2 = d.n[1], n3 = d.n[2];
      const int r1 = (n1 - k[0]) % n1, r2 = (n2 - k[1]) % n2;
      auto at = [&](int i, int j) { return Xb[(static_cast<long long>(i) * n2 + j) * n3 + k[2]]; };
      const double2 a = ta[k[0]], bb = tb[k[1]];
      const double2 ab = cm(a, bb), cb = cm(cj(a), bb);
      double2 s = cm(ab, at(k[0], k[1]));
      s = ca(s, cm(cb, at(r1, k[1])));
      s = ca(s, cm(cj(cb), at(k[0], r2)));
      s = ca(s, cm(cj(ab), at(r1, r2)));
      v = 0.25 * cm(tc[k[2]], s).x;
    }
    y[f] = static_cast<T>(v);
  }
}

template <typename T>
__device__ __forceinline__ double fetch2g(const T* x, int i, int j, int n1, int n2, int mode) {
  if (i == n1 || j == n2) return 0.0;
  if (mode == 1) {
    if (i == 0) return 0.0;
    i = n1 - i;
  } else if (mode == 2) {
    if (j == 0) return 0.0;
    j = n2 - j;
  }
  return static_cast<double>(x[static_cast<long long>(i) * n2 + j]);
}

// Full Hermitian spectrum of the merged inverse preprocess (any rank 1..3).
// 1D (idct_1d, dct1d.cpp:185-220 embedding): X'(k) = conj(a(k)) (x(k) - i x(N-k)), x(N) := 0.
template <typename T>
__global__ void g_pre(const T* __restrict__ x, double2* __restrict__ Xo, Dims d, long long batch_items,
                      int mode, const double2* __restrict__ ta, const double2* __restrict__ tb,
                      const double2* __restrict__ tc) {
  const long long total = d.numel * batch_items;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = f / d.numel;
    const T* xb = x + b * d.numel;
    int k[3];
    unflat(f - b * d.numel, d, k);
    const int last = d.rank - 1;
    const int nl = d.n[last];
    bool flip = k[last] > nl / 2;  // Hermitian fill of the upper half of the last axis
    int e[3];
    for (int a = 0; a < d.rank; ++a) e[a] = flip ? (d.n[a] - k[a]) % d.n[a] : k[a];
    double2 val;
    if (d.rank == 1) {
      const int n = d.n[0], kk = e[0];
      double p = static_cast<double>(xb[kk]);
      double q = kk == 0 ? 0.0 : static_cast<double>(xb[n - kk]);
      if (mode == 2) {  // idxst embedding: x(N-n) with x(N) := 0 (transforms_ext.cpp:238-242)
        p = kk == 0 ? 0.0 : static_cast<double>(xb[n - kk]);
        q = kk == 0 ? 0.0 : static_cast<double>(xb[kk]);
        val = cm(cj(ta[kk]), make_double2(p, -q));
      } else {
        val = cm(cj(ta[kk]), make_double2(p, -q));
      }
    } else if (d.rank == 2) {
      const int n1 = d.n[0], n2 = d.n[1];
      const int k1 = e[0], m2 = e[1];
      // pick the reference work item (q1 <= n1/2) that writes row k1
      const bool direct = k1 <= n1 / 2;
      const int q1 = direct ? k1 : n1 - k1;
      const double p = fetch2g(xb, q1, m2, n1, n2, mode);
      const double q = fetch2g(xb, n1 - q1, n2 - m2, n1, n2, mode);
      const double r = fetch2g(xb, n1 - q1, m2, n1, n2, mode);
      const double s = fetch2g(xb, q1, n2 - m2, n1, n2, mode);
      const double2 w = cj(cm(ta[k1], tb[m2]));
      val = direct ? cm(w, make_double2(p - q, -(r + s))) : cm(w, make_double2(r - s, -(p + q)));
    } else {
      const int n1 = d.n[0], n2 = d.n[1], n3 = d.n[2];
      const int i = e[0], j = e[1], kk = e[2];
      auto F = [&](int ii, int jj, int ll) -> double {
        if (ii == n1 || jj == n2 || ll == n3) return 0.0;
        return static_cast<double>(xb[(static_cast<long long>(ii) * n2 + jj) * n3 + ll]);
      };
      const int r1 = n1 - i, r2 = n2 - j, r3 = n3 - kk;
      const double re = (F(i, j, kk) - F(r1, r2, kk)) - (F(r1, j, r3) + F(i, r2, r3));
      const double im = F(r1, r2, r3) - ((F(r1, j, kk) + F(i, r2, kk)) + F(i, j, r3));
      const double2 w = cj(cm(cm(ta[i], tb[j]), tc[kk]));
      val = cm(w, make_double2(re, im));
    }
    Xo[f] = flip ? cj(val) : val;
  }
}

template <typename T>
__global__ void g_gather_inv(const double2* __restrict__ z, T* __restrict__ y, Dims d, long long batch_items,
                             double scale, int sign_axis) {
  const long long total = d.numel * batch_items;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = f / d.numel;
    int k[3];
    unflat(f - b * d.numel, d, k);
    long long src = 0;
    for (int a = 0; a < d.rank; ++a) src = src * d.n[a] + parity_source(k[a], d.n[a]);
    double v = scale * z[b * d.numel + src].x;
    if (sign_axis >= 0 && (k[sign_axis] & 1)) v = -v;
    y[f] = static_cast<T>(v);
  }
}

// ---- two-pass 2D pipeline for extents <= 8192 (one line per tile at most) ----
// The same three stages with the gathers, the postprocess and the merged
// preprocess fused into the line FFTs' loads and stores, so a 2D transform is
// two passes over HBM (one per axis) instead of gather + transpose + FFT +
// transpose + FFT + post:
// W holds the one-sided spectrum, columns k2 < h = n2/2 + 1 (the layout of
// the reference's rfft_nd / irfft_nd, rfft.cpp:182-245):
//   forward : G2_FWD_ROWS  x rows pe(i), pe(i+1) as the real / imaginary
//                          parts of one line, columns scattered by ps (= pe^-1)
//                          -> FFT along axis 1 -> the two spectra separated by
//                          Hermitian symmetry -> W rows i, i+1 (k2 < h)
//             G2_FWD_COLS  W columns c0.. -> FFT along axis 0 -> the
//                          postprocess of dct2d.hpp:6 for y columns c and
//                          n2 - c (X(k1, n2 - c) = conj X(-k1, c)) -> y
//   inverse : G2_INV_COLS  merged preprocess (dct2d.cpp:161-198) for columns
//                          c0.. < h -> inverse FFT along axis 0 -> W columns
//             G2_INV_ROWS  W rows ps(k1) + i ps(k1+1), Hermitian fill of
//                          k2 >= h as irfft_nd does -> inverse FFT along axis 1
//                          -> real / imaginary parts through the inverse gather
//                          (dct2d.cpp:214-238, row-local) -> y rows k1, k1+1
// Column tiles hold `lines` consecutive columns with an odd line stride in
// shared memory (conflict-free strided loads); row tiles hold `lines` rows
// (two per complex line).
enum { G2_FWD_ROWS = 0, G2_FWD_COLS = 1, G2_INV_COLS = 2, G2_INV_ROWS = 3 };
// Two tile shapes: lines up to 2048 run 256-thread CTAs at 8 elements per
// thread (three CTAs per SM: one CTA's global loads overlap another's passes),
// longer lines 512-thread CTAs at 16 per thread.
template <int FPT> struct G2Cfg;
template <> struct G2Cfg<8> { static constexpr int NT = 256, MINB = 3, CAP = 8 * 256; };
template <> struct G2Cfg<16> { static constexpr int NT = 512, MINB = 1, CAP = 16 * 512; };

struct G2Args {
  const void* src;
  void* dst;
  int n1, n2;
  long long batch;
  int lines;         // columns per column tile / rows per row tile
  int mode, sign_axis;
  double scale;
  const double2* circle;  // circle table of the FFT axis
  const double2* ta;      // quarter-wave tables of axes 0 and 1
  const double2* tb;
  Radices rad;
  FastDiv fn1, fn2, fh;
  int h;             // stored spectrum columns, n2 / 2 + 1
  // Bluestein on the FFT axis (bm = pow2 convolution length, 0 = mixed radix):
  // x_m c_m -> FFT_M -> * bhat -> inverse FFT_M -> c_k / M (conjugated chirp
  // and kernel for the inverse transform); rad then describes M
  int bm;
  const double2* bchirp;
  const double2* bhat;
  const double2* bcircle;
};

template <typename T, int KIND, int FPT>
__global__ void __launch_bounds__(G2Cfg<FPT>::NT, G2Cfg<FPT>::MINB) g2_kernel(G2Args a) {
  constexpr bool ROWS = KIND == G2_FWD_ROWS || KIND == G2_INV_ROWS;
  constexpr bool INV = KIND == G2_INV_COLS || KIND == G2_INV_ROWS;
  extern __shared__ __align__(16) double2 g2sm[];
  const int n1 = a.n1, n2 = a.n2;
  const int n = ROWS ? n2 : n1;               // FFT length
  const int nb = a.bm ? a.bm : n;             // line length in smem (Bluestein: M)
  const int ld = ROWS ? nb : (nb | 1);        // line stride in smem
  const double2* tw = a.circle;               // forward circle table, L1-resident
  double2* x = g2sm;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous kernel complete (PDL launch)
  // Bluestein pre/post chirp multiplies ride on the loads and stores
  const bool blue = a.bm != 0;
  auto chirp = [&](int m) {
    const double2 c = a.bchirp[m];
    return INV ? cj(c) : c;
  };
  auto put = [&](int slot, double2 v) { x[slot] = blue ? cm(v, chirp(slot % ld)) : v; };
  const double inv_m = blue ? 1.0 / a.bm : 1.0;
  auto get = [&](int l, int k) {
    const double2 v = x[l * ld + k];
    if (!blue) return v;
    const double2 w = cm(v, chirp(k));
    return make_double2(w.x * inv_m, w.y * inv_m);
  };
  const int t = threadIdx.x, nt = blockDim.x;
  const long long plane = static_cast<long long>(n1) * n2;
  const int h = a.h;
  const long long wplane = static_cast<long long>(n1) * h;  // one-sided spectrum per item
  long long r0 = 0, b = 0;
  int c0 = 0, lines;
  int rows = 0;  // row tiles: rows of y / x in this tile; two rows share one complex line
  if constexpr (ROWS) {
    r0 = static_cast<long long>(blockIdx.x) * a.lines;  // flattened (batch, row); a.lines = rows per tile
    rows = static_cast<int>(min(static_cast<long long>(a.lines), a.batch * n1 - r0));
    lines = (rows + 1) / 2;
  } else {
    const int tpb = (a.h + a.lines - 1) / a.lines;
    b = blockIdx.x / tpb;
    c0 = static_cast<int>(blockIdx.x % tpb) * a.lines;
    lines = min(a.lines, a.h - c0);
  }
  const int total = lines * n;
  const FastDiv fl(static_cast<unsigned>(lines));  // column tiles: element -> (row, line)

  // ---- load ---- (total <= FPT * nt: each thread issues all its global
  // loads before the first shared-memory store, so their latencies overlap)
  if constexpr (KIND == G2_FWD_ROWS) {
    // rows 2l and 2l+1 of the tile as the real and imaginary parts of line l
    const T* xs = static_cast<const T*>(a.src);
    T va[FPT], vb[FPT];
    int slot[FPT];
#pragma unroll
    for (int u = 0; u < FPT; ++u) {
      const int e = t + u * nt;
      if (e < total) {
        const int l = a.fn2.div(e), c = e - l * n2;
        const int R = static_cast<int>(r0) + 2 * l, bb = a.fn1.div(R);
        const int i = R - bb * n1;
        va[u] = xs[static_cast<long long>(bb) * plane + static_cast<long long>(parity_embed(i, n1)) * n2 + c];
        vb[u] = T(0);
        if (2 * l + 1 < rows) {
          const int R2 = R + 1, bb2 = a.fn1.div(R2);
          const int i2 = R2 - bb2 * n1;
          vb[u] = xs[static_cast<long long>(bb2) * plane + static_cast<long long>(parity_embed(i2, n1)) * n2 + c];
        }
        slot[u] = l * ld + parity_source(c, n2);
      }
    }
#pragma unroll
    for (int u = 0; u < FPT; ++u)
      if (t + u * nt < total)
        put(slot[u], make_double2(static_cast<double>(va[u]), static_cast<double>(vb[u])));
  } else if constexpr (KIND == G2_FWD_COLS || KIND == G2_INV_ROWS) {
    const double2* W = static_cast<const double2*>(a.src);
    double2 v[FPT];
    int slot[FPT];
#pragma unroll
    for (int u = 0; u < FPT; ++u) {
      const int e = t + u * nt;
      if (e < total) {
        if constexpr (KIND == G2_FWD_COLS) {
          const int m = fl.div(e), l = e - m * lines;
          v[u] = W[b * wplane + static_cast<long long>(m) * h + c0 + l];
          slot[u] = l * ld + m;
        } else {
          // y row k1 comes from z row ps(k1); k2 >= h is the conjugate mirror
          // (irfft_nd's Hermitian fill). Line l carries rows 2l (real part of
          // the result) and 2l+1 (imaginary part): Z = Wa + i Wb.
          const int l = a.fn2.div(e), c = e - l * n2;
          const bool mir = c >= h;
          const int cc = mir ? n2 - c : c;
          const int R = static_cast<int>(r0) + 2 * l, bb = a.fn1.div(R);
          const int k1 = R - bb * n1;
          double2 wa = W[static_cast<long long>(bb) * wplane + static_cast<long long>(parity_source(k1, n1)) * h + cc];
          double2 wb = make_double2(0.0, 0.0);
          if (2 * l + 1 < rows) {
            const int R2 = R + 1, bb2 = a.fn1.div(R2);
            const int k1b = R2 - bb2 * n1;
            wb = W[static_cast<long long>(bb2) * wplane + static_cast<long long>(parity_source(k1b, n1)) * h + cc];
          }
          if (mir) {
            wa = cj(wa);
            wb = cj(wb);
          }
          v[u] = make_double2(wa.x - wb.y, wa.y + wb.x);
          slot[u] = l * ld + c;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < FPT; ++u)
      if (t + u * nt < total) put(slot[u], v[u]);
  } else {  // G2_INV_COLS
    // full Hermitian spectrum of the merged preprocess, column m2 = c0 + l
    const T* xb = static_cast<const T*>(a.src) + b * plane;
    constexpr int UB = 4;  // elements per load batch (4 operands each)
#pragma unroll
    for (int u0 = 0; u0 < FPT; u0 += UB) {
      double op[UB][4];
      int e1s[UB], m2s[UB], slot[UB];
      bool dir[UB];
#pragma unroll
      for (int u = u0; u < u0 + UB; ++u) {
        const int e = t + u * nt;
        if (e < total) {
          const int k1 = fl.div(e), l = e - k1 * lines;
          const int m2 = c0 + l;  // < h: the one-sided half, no Hermitian fill here
          const int e1 = k1;
          const bool direct = e1 <= n1 / 2;
          const int q1 = direct ? e1 : n1 - e1;
          op[u - u0][0] = fetch2g(xb, q1, m2, n1, n2, a.mode);
          op[u - u0][1] = fetch2g(xb, n1 - q1, n2 - m2, n1, n2, a.mode);
          op[u - u0][2] = fetch2g(xb, n1 - q1, m2, n1, n2, a.mode);
          op[u - u0][3] = fetch2g(xb, q1, n2 - m2, n1, n2, a.mode);
          e1s[u - u0] = e1;
          m2s[u - u0] = m2;
          dir[u - u0] = direct;
          slot[u - u0] = l * ld + k1;
        }
      }
#pragma unroll
      for (int u = u0; u < u0 + UB; ++u) {
        if (t + u * nt < total) {
          const double* o = op[u - u0];
          const double2 w = cj(cm(a.ta[e1s[u - u0]], a.tb[m2s[u - u0]]));
          const double2 val = dir[u - u0] ? cm(w, make_double2(o[0] - o[1], -(o[2] + o[3])))
                                          : cm(w, make_double2(o[2] - o[3], -(o[0] + o[1])));
          put(slot[u - u0], val);
        }
      }
    }
  }
  if (blue) {  // zero padding of each line to the convolution length
    const int pad = nb - n;
    for (int e = t; e < lines * pad; e += nt) {
      const int l = e / pad;
      x[l * ld + n + (e - l * pad)] = make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  if (!blue) {
    line_passes<FPT, INV, true>(x, tw, n, a.rad, total, t, nt, ld);
  } else {
    const int totalm = lines * nb;
    line_passes<FPT, false, true>(x, a.bcircle, nb, a.rad, totalm, t, nt, ld);
    for (int e = t; e < totalm; e += nt) {
      const int l = a.rad.n.div(e), k = e - l * nb;
      const double2 hk = a.bhat[k];
      x[l * ld + k] = cm(x[l * ld + k], INV ? cj(hk) : hk);
    }
    __syncthreads();
    line_passes<FPT, true, true>(x, a.bcircle, nb, a.rad, totalm, t, nt, ld);
  }

  // ---- store ----
  if constexpr (KIND == G2_FWD_ROWS) {
    // Z = FFT(xa + i xb): Xa(k) = (Z(k) + conj Z(-k)) / 2, Xb(k) = (Z(k) - conj Z(-k)) / 2i
    double2* W = static_cast<double2*>(a.dst);
    for (int e = t; e < lines * h; e += nt) {
      const int l = a.fh.div(e), c = e - l * h;
      const double2 z = get(l, c), zm = get(l, c ? n2 - c : 0);
      W[(r0 + 2 * l) * h + c] = make_double2(0.5 * (z.x + zm.x), 0.5 * (z.y - zm.y));
      if (2 * l + 1 < rows) W[(r0 + 2 * l + 1) * h + c] = make_double2(0.5 * (z.y + zm.y), 0.5 * (zm.x - z.x));
    }
  } else if constexpr (KIND == G2_FWD_COLS) {
    // y = 1/2 Re(b(k2) (a(k1) X(k1, k2) + conj(a(k1)) X(-k1, k2)))   (dct2d.hpp:6)
    T* y = static_cast<T*>(a.dst) + b * plane;
    for (int e = t; e < total; e += nt) {
      const int k1 = fl.div(e), l = e - k1 * lines;
      const int k2 = c0 + l;
      const double2 aa = a.ta[k1];
      const double2 x1 = get(l, k1), x2 = get(l, k1 ? n1 - k1 : 0);
      const double v = 0.5 * cm(a.tb[k2], ca(cm(aa, x1), cm(cj(aa), x2))).x;
      y[static_cast<long long>(k1) * n2 + k2] = static_cast<T>(v);
      // mirrored column n2 - k2: X(k1, n2 - k2) = conj X(-k1, k2), X(-k1, n2 - k2) = conj X(k1, k2)
      const int km = n2 - k2;
      if (k2 > 0 && km != k2) {
        const double vm = 0.5 * cm(a.tb[km], ca(cm(aa, cj(x2)), cm(cj(aa), cj(x1)))).x;
        y[static_cast<long long>(k1) * n2 + km] = static_cast<T>(vm);
      }
    }
  } else if constexpr (KIND == G2_INV_COLS) {
    double2* W = static_cast<double2*>(a.dst) + b * wplane;
    for (int e = t; e < total; e += nt) {
      const int m = fl.div(e), l = e - m * lines;
      W[static_cast<long long>(m) * h + c0 + l] = get(l, m);
    }
  } else {
    T* y = static_cast<T*>(a.dst);
    for (int e = t; e < rows * n2; e += nt) {
      const int r = a.fn2.div(e), k2 = e - r * n2;  // tile row r = line r / 2, part r & 1
      const int R = static_cast<int>(r0) + r, bb = a.fn1.div(R);
      const int k1 = R - bb * n1;
      const double2 z = get(r >> 1, parity_source(k2, n2));
      double v = a.scale * ((r & 1) ? z.y : z.x);
      if ((a.sign_axis == 0 && (k1 & 1)) || (a.sign_axis == 1 && (k2 & 1))) v = -v;
      y[static_cast<long long>(R) * n2 + k2] = static_cast<T>(v);
    }
  }
}

template <typename T, int KIND, int FPT>
cudaError_t g2_launch_cfg(G2Args a, cudaStream_t st) {
  using C = G2Cfg<FPT>;
  const bool rows = KIND == G2_FWD_ROWS || KIND == G2_INV_ROWS;
  const int n = a.bm ? a.bm : (rows ? a.n2 : a.n1);  // line length in smem
  const int ld = rows ? n : (n | 1);
  // lines per tile: as many as the tile capacity allows (columns: at most 32,
  // rows: at most 64), fewer threads for small tiles
  int lines = C::CAP / n;  // complex lines per tile (row tiles: two rows per line)
  lines = std::max(1, std::min(lines, 32));
  a.h = a.n2 / 2 + 1;
  if (!rows) lines = std::min(lines, a.h);
  a.lines = rows ? 2 * lines : lines;
  a.fh = FastDiv(static_cast<unsigned>(a.h));
  a.rad = factorise(n);
  a.fn1 = FastDiv(static_cast<unsigned>(a.n1));
  a.fn2 = FastDiv(static_cast<unsigned>(a.n2));
  const int total = lines * n;
  int nt = (total + FPT - 1) / FPT;
  nt = std::min(C::NT, std::max(64, (nt + 31) / 32 * 32));
  const size_t smem = static_cast<size_t>(lines) * ld * sizeof(double2);
  if (smem > 48 * 1024) {
    const cudaError_t pe = prep_smem_ptr(reinterpret_cast<const void*>(g2_kernel<T, KIND, FPT>), 200 * 1024);
    if (pe != cudaSuccess) return pe;
  }
  const long long tiles = rows ? (a.batch * a.n1 + a.lines - 1) / a.lines : a.batch * ((a.h + lines - 1) / lines);
  // grid.x limit 2^31-1: batches beyond it are not reachable at these extents
  // programmatic dependent launch: the second pass's CTAs start as the first drains
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(tiles));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  lattr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, g2_kernel<T, KIND, FPT>, a);
}

// Column passes of columns in [W, 2048) points take the wide tile (512
// threads, up to 8192 elements: >= 4 columns, so every row segment is >= 64 B
// of fp64 complex and the outputs' row segments are >= 32 B) instead of one
// column per 256-thread tile. Measured on B200 (tools/ab_g2wide.sh, graph-timed
// calls): fp64 2000^2 DCT 124 -> 116 us, IDCT 138 -> 124 us, 1800^2 104 -> 99 /
// 121 -> 111 us, 1700x900 81 -> 70 / 91 -> 73 us; 1536^2 slower (75 -> 92 us),
// so W = 1700; fp32 only the forward column pass gains (2000^2 134 -> 129 us,
// its inverse 146 -> 152 us). SDCT_G2_WIDE_MIN overrides W (developer A/B).
int g2_wide_min() {
  static const int v = [] {
    const char* f = getenv("SDCT_G2_WIDE_MIN");
    return f ? atoi(f) : 1700;
  }();
  return v;
}

template <typename T, int KIND>
cudaError_t g2_launch(G2Args a, cudaStream_t st) {
  constexpr bool ROWS = KIND == G2_FWD_ROWS || KIND == G2_INV_ROWS;
  const int n = a.bm ? a.bm : ROWS ? a.n2 : a.n1;
  const bool wide = !ROWS && !a.bm && n >= g2_wide_min() && n < 2048 &&
                    (sizeof(T) == 8 || KIND == G2_FWD_COLS);
  return n <= G2Cfg<8>::CAP && !wide ? g2_launch_cfg<T, KIND, 8>(a, st) : g2_launch_cfg<T, KIND, 16>(a, st);
}

// ---- Bluestein along one axis, one pass per stage ---------------------------
// rfft.cpp:26,43-62 runs Bluestein for lengths its radix-2 FFT cannot take;
// here it serves the axes whose largest prime factor exceeds 64 and that the
// two-pass pipeline does not take (1D, 3D, long 2D axes):
//   X(k) = c_k sum_j (x_j c_j) conj(c_{k-j}),  c_j = e^{-i pi j^2 / n},
// a circular convolution of power-of-two length M >= 2n - 1 (bhat = FFT_M of
// the wrapped conjugate chirp, plan tables). The inverse DFT is
// conj(DFT(conj(x))). The axis is brought to the front ([n][lines], lines
// innermost) and processed in chunks of W lines; M = fa fb (fa = min(M, 4096))
// runs as a four-step FFT with m = m1 + fa m2 and k = k2 + fb k1:
//   pre : u[k2][m1][w] = W_M^{m1 k2} sum_{m2} xc(m1 + fa m2) W_fb^{m2 k2}
//         (xc = chirped, zero-padded input)
//   the fast path's column kernel: fa-point DIF FFTs down the rows of each
//   plane k2, spectrum rows in rt_srow order; x bhat permuted to that order
//   (plan table); the inverse column kernel (DIT) back to natural rows; then
//   post: v(m1 + fa m2) = sum_{k2} W_fb^{-m2 k2} W_M^{-m1 k2} z[k2][m1][w],
//         out = op(c_m v(m) / M).
// Every pass reads and writes whole rows of W lines (coalesced).
__global__ void g_blue_pre(const double2* __restrict__ in, double2* __restrict__ u, long long i0, int cnt, int W,
                           int n, long long L, int lgM, int lgfa, const double2* __restrict__ chirp,
                           const double2* __restrict__ circ, int inverse) {
  const int M = 1 << lgM, fa = 1 << lgfa, fb = M >> lgfa;
  const long long total = static_cast<long long>(fa) * W;  // one thread per (m1, w)
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m1 = static_cast<int>(f / W), w = static_cast<int>(f - static_cast<long long>(m1) * W);
    const double2* col = in + i0 + w;
    for (int k2 = 0; k2 < fb; ++k2) {
      double re = 0.0, im = 0.0;
      if (w < cnt) {
        for (int m2 = 0; m2 < fb; ++m2) {
          const int m = m1 + fa * m2;
          if (m >= n) break;
          double2 v = col[static_cast<long long>(m) * L];
          if (inverse) v.y = -v.y;
          v = cm(v, chirp[m]);
          const double2 t = circ[((m2 * k2) & (fb - 1)) << lgfa];  // W_fb^{m2 k2}
          re = fma(v.x, t.x, fma(-v.y, t.y, re));
          im = fma(v.x, t.y, fma(v.y, t.x, im));
        }
      }
      u[(static_cast<long long>(k2) * fa + m1) * W + w] = cm(make_double2(re, im), circ[(m1 * k2) & (M - 1)]);
    }
  }
}

// plane p, storage row s (rt_srow order) holds X(p + fb k1(s)); hatp is that order
__global__ void g_blue_mul(double2* __restrict__ u, long long total, int W, const double2* __restrict__ hatp) {
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x)
    u[f] = cm(u[f], hatp[f / W]);
}

__global__ void g_blue_post(const double2* __restrict__ z, double2* __restrict__ out, long long i0, int cnt, int W,
                            int n, long long L, int lgM, int lgfa, const double2* __restrict__ chirp,
                            const double2* __restrict__ circ, int inverse) {
  const int M = 1 << lgM, fa = 1 << lgfa, fb = M >> lgfa;
  const double inv_m = 1.0 / static_cast<double>(M);
  const long long total = static_cast<long long>(fa) * cnt;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m1 = static_cast<int>(f / cnt), w = static_cast<int>(f - static_cast<long long>(m1) * cnt);
    double2* col = out + i0 + w;
    const double2* src = z + static_cast<long long>(m1) * W + w;
    for (int m2 = 0; m2 < fb; ++m2) {
      const int m = m1 + fa * m2;
      if (m >= n) break;
      double re = 0.0, im = 0.0;
      for (int k2 = 0; k2 < fb; ++k2) {
        double2 t = cm(circ[((m2 * k2) & (fb - 1)) << lgfa], circ[(m1 * k2) & (M - 1)]);
        t.y = -t.y;  // W_fb^{-m2 k2} W_M^{-m1 k2}
        const double2 v = src[static_cast<long long>(k2) * fa * W];
        re = fma(v.x, t.x, fma(-v.y, t.y, re));
        im = fma(v.x, t.y, fma(v.y, t.x, im));
      }
      double2 r = cm(make_double2(re, im), chirp[m]);
      r.x *= inv_m;
      r.y *= inverse ? -inv_m : inv_m;
      col[static_cast<long long>(m) * L] = r;
    }
  }
}

}  // namespace

static int largest_prime(int n) {
  int m = n, p = 1;
  for (int d = 2; d * d <= m; ++d)
    while (m % d == 0) {
      p = std::max(p, d);
      m /= d;
    }
  return m > 1 ? std::max(p, m) : p;
}

int bluestein_len(int n, bool tile) {
  if (n < 2 || n > (1 << 23)) return 0;  // M / 4096 must fit one split cofactor
  int M = 1;
  while (M < 2 * n - 1) M <<= 1;
  if (largest_prime(n) > 64) return M;
  if (!tile || M > kG2MaxN) return 0;
  // inside a two-pass tile, Bluestein also beats the mixed radix when the
  // thread-per-output prime passes (factors > 7, p MACs per element each) cost
  // more than ~20 x the convolution's growth M / n (measured on 989..2023:
  // 1023 = 3.11.31 151 -> 121 us, 1849 = 43^2 540 -> 416 us; 2023 = 7.17^2 and
  // 1147 = 31.37 stay mixed radix, 340 / 168 us vs 428 / 209 us)
  int m = n, big = 0;
  for (int d = 2; d * d <= m; ++d)
    while (m % d == 0) {
      if (d > 7) big += d;
      m /= d;
    }
  if (m > 7) big += m;
  return static_cast<double>(big) > 20.0 * M / n ? M : 0;
}

// Two-pass pipeline: both extents <= kG2MaxN and every Bluestein length
// within the tile; an axis with a large prime factor and 4096 < n <= 8192
// runs the global pass instead (4097 = 17 x 241: 8.2 ms on the tile's mixed
// radix, where a prime radix p costs p MACs per element; 8191 took 20 ms there)
bool generic_two_pass(int rank, const int* dims, const int* blue_m) {
  if (rank != 2) return false;
  for (int a = 0; a < 2; ++a)
    if (dims[a] > kG2MaxN || blue_m[a] > kG2MaxN) return false;
  return true;
}

long long bluestein_chunk_lines(int M, long long lines) {
  const long long cap = std::max<long long>(2, ((8LL << 20) / M) & ~1LL);  // <= 8 Mi complex per buffer
  return std::min(lines + (lines & 1), cap);  // even: whole 2-line bands of the column kernel
}

long long bluestein_scratch_elems(int rank, const int* dims, const int* blue_m, long long batch) {
  if (generic_two_pass(rank, dims, blue_m)) return 0;
  long long numel = 1, best = 0;
  for (int a = 0; a < rank; ++a) numel *= dims[a];
  for (int a = 0; a < rank; ++a)
    if (blue_m[a]) best = std::max(best, 2 * bluestein_chunk_lines(blue_m[a], batch * (numel / dims[a])) * blue_m[a]);
  return best;
}

// Complex DFT along axes [a0, a1) of the [batch][dims...] complex tensor in
// cur (result in cur; nxt is scratch of the same size). g = grid for the
// elementwise kernels over the whole tensor.
// shared-memory line FFT of length len over lines (outer', inner'); tab is a
// circle table e^{-2 pi i t / (len ts)} read with stride ts
static void line_fft_run(const double2* src, double2* dst, long long outer_, int len, long long inner_,
                         const double2* tab, int ts, int inverse, cudaStream_t st) {
  if (ts == 1 && len >= 2048 && len <= kFftMaxN) {  // long lines: GTW variant, one line per CTA
    const size_t smem = static_cast<size_t>(len) * sizeof(double2);
    prep_smem_ptr(reinterpret_cast<const void*>(g_fft_axis_smem<16, true>), 64 * 1024);
    const long long tiles = inner_ > 1 ? outer_ * inner_ : outer_;
    const int nt = ((len + 15) / 16 + 31) & ~31;  // 16 outputs per thread, whole warps
    g_fft_axis_smem<16, true><<<static_cast<unsigned>(tiles), nt, smem, st>>>(src, dst, outer_, len, inner_, tab, 1,
                                                                              inverse, factorise(len), 1);
    return;
  }
  // threads per CTA: the fewest (>= 128) that hold a whole line at
  // kFftPerThread outputs each (small CTAs: the passes are latency bound)
  static const int nt_short = [] {
    const char* f = getenv("SDCT_G_NT");  // developer A/B knob
    return f ? atoi(f) : 128;
  }();
  const int nt = len <= 1024 ? nt_short : len <= 2048 ? 256 : 512;
  int lpc = 1;
  while (lpc < 16 && 2 * lpc * len <= kFftPerThread * nt &&
         (inner_ == 1 ? lpc * 2 <= outer_ : inner_ % (lpc * 2) == 0))
    lpc *= 2;
  const size_t smem = (static_cast<size_t>(lpc) * len + len) * sizeof(double2);
  if (smem > 48 * 1024) prep_smem_ptr(reinterpret_cast<const void*>(g_fft_axis_smem<kFftPerThread, false>), 140 * 1024);
  const long long tiles = inner_ > 1 ? outer_ * (inner_ / lpc) : (outer_ + lpc - 1) / lpc;
  g_fft_axis_smem<kFftPerThread, false><<<static_cast<unsigned>(tiles), nt, smem, st>>>(
      src, dst, outer_, len, inner_, tab, ts, inverse, factorise(len), lpc);
}

// axis a of the [n][L] matrix X (lines innermost) -> Y through the global
// Bluestein pass, in chunks of W lines
static void blue_axis(const GenericJob& job, int a, const double2* X, double2* Y, long long L, int inverse,
                      cudaStream_t st) {
  const int n = job.dims[a], M = job.blue_m[a];
  int lgM = 0;
  while ((1 << lgM) < M) ++lgM;
  const int lgfa = lgM < 12 ? lgM : 12, fa = 1 << lgfa, fb = M >> lgfa;
  const int W = static_cast<int>(bluestein_chunk_lines(M, L));
  double2* U = job.blue_ws;
  double2* V = U + static_cast<long long>(W) * M;
  const double2* circ = job.blue_circle[a];
  for (long long i0 = 0; i0 < L; i0 += W) {
    const int cnt = static_cast<int>(std::min<long long>(W, L - i0));
    const int Wc = cnt + (cnt & 1);  // column-kernel bands are 2 lines wide
    g_blue_pre<<<nblocks(static_cast<long long>(fa) * Wc), kThreads, 0, st>>>(X, U, i0, cnt, Wc, n, L, lgM, lgfa,
                                                                            job.blue_chirp[a], circ, inverse);
    bluestein_line_fft(U, V, fa, Wc, fb, false, job.blue_st[a], st);
    g_blue_mul<<<nblocks(static_cast<long long>(M) * Wc), kThreads, 0, st>>>(V, static_cast<long long>(M) * Wc, Wc,
                                                                           job.blue_hatp[a]);
    bluestein_line_fft(V, U, fa, Wc, fb, true, job.blue_st[a], st);
    g_blue_post<<<nblocks(static_cast<long long>(fa) * cnt), kThreads, 0, st>>>(U, Y, i0, cnt, Wc, n, L, lgM, lgfa,
                                                                              job.blue_chirp[a], circ, inverse);
  }
}

static void dft_axes(const GenericJob& job, int a0, int a1, double2*& cur, double2*& nxt, int inverse, int g,
              cudaStream_t st) {
    for (int a = a0; a < a1; ++a) {
      long long inner = 1, outer = job.batch;
      for (int t = a + 1; t < job.rank; ++t) inner *= job.dims[t];
      for (int t = 0; t < a; ++t) outer *= job.dims[t];
      const int n = job.dims[a];
      if (job.blue_m[a] && job.blue_ws) {
        // the axis in front, lines innermost: [o][n][inner] -> [n][inner][o]
        // (lines in (i, o) order; none needed when outer == 1)
        const long long L = outer * inner;
        if (outer > 1) {
          g_transpose(cur, nxt, 1, outer, static_cast<long long>(n) * inner, st);
          blue_axis(job, a, nxt, cur, L, inverse, st);
          g_transpose(cur, nxt, 1, static_cast<long long>(n) * inner, outer, st);  // back
        } else {
          blue_axis(job, a, cur, nxt, L, inverse, st);
        }
        std::swap(cur, nxt);
        continue;
      }
      auto line_fft = [&](const double2* src, double2* dst, long long outer_, int len, long long inner_, int ts) {
        line_fft_run(src, dst, outer_, len, inner_, job.circle[a], ts, inverse, st);
      };
      int fa = 0, fb = 0;
      if (n > kFftMaxN) split_factors(n, fa, fb);
      if ((n > 1 && n <= kFftMaxN) || fa > 0) {
        // strided axes (inner > 1) whose lines would be read with little
        // coalescing are transposed to rows first: [o][n][inner] -> [o][inner][n]
        // (>= 4 lines per CTA keep 64-B row segments: 3D 200^3 fp64 DCT 802 -> 672 us,
        // 250^3 1480 -> 1334 us against a rule of 16 lines)
        static const int lmin = [] {
          const char* f = getenv("SDCT_G_LMIN");  // developer A/B knob
          return f ? atoi(f) : 4;
        }();
        const bool tr = inner > 1 && (static_cast<long long>(lmin) * (fa > 0 ? fa : n) > kFftPerThread * kThreads ||
                                      inner % lmin != 0);
        long long o2 = outer, in2 = inner;
        if (tr) {
          g_transpose(cur, nxt, outer, n, inner, st);
          std::swap(cur, nxt);
          o2 = outer * inner;
          in2 = 1;
        }
        if (fa == 0) {
          line_fft(cur, nxt, o2, n, in2, 1);
        } else {
          // split: a-point line FFTs (stride b), then twiddle + b-point DFT + permutation
          line_fft(cur, nxt, o2, fa, static_cast<long long>(fb) * in2, fb);
          g_split_finish<<<g, kThreads, 0, st>>>(nxt, cur, o2, fa, fb, in2, job.circle[a], inverse);
          std::swap(cur, nxt);
        }
        std::swap(cur, nxt);
        if (tr) {
          g_transpose(cur, nxt, outer, inner, n, st);  // back: [o][inner][n] -> [o][n][inner]
          std::swap(cur, nxt);
        }
      } else if (n > 1) {
        g_dft_axis<<<g, kThreads, 0, st>>>(cur, nxt, outer, job.dims[a], inner, job.circle[a], inverse);
        double2* t = cur;
        cur = nxt;
        nxt = t;
      }
    }
  }

// ---------------------------------------------------------------------------
template <typename T>
cudaError_t generic_run(const GenericJob& job, const void* in, void* out, void* ws, cudaStream_t st) {
  Dims d;
  d.rank = job.rank;
  d.numel = 1;
  for (int a = 0; a < 3; ++a) d.n[a] = a < job.rank ? job.dims[a] : 1;
  for (int a = 0; a < job.rank; ++a) d.numel *= job.dims[a];
  const long long total = d.numel * job.batch;
  double2* A = static_cast<double2*>(ws);
  double2* B = A + total;
  const int g = nblocks(total);
  GenericJob jb = job;  // global Bluestein scratch after the two tensor buffers
  jb.blue_ws = job.blue_scratch ? B + total : nullptr;
  auto dft_all = [&](double2*& cur, double2*& nxt, int inverse) {
    dft_axes(jb, 0, job.rank, cur, nxt, inverse, g, st);
  };
  double2* cur = A;
  double2* nxt = B;
  static_assert(G2Cfg<16>::CAP == kG2MaxN, "two-pass line capacity");
  if (!job.legacy && generic_two_pass(job.rank, job.dims, job.blue_m)) {
    // two-pass pipeline (gathers / pre / post fused into the line FFTs)
    G2Args a{};
    a.n1 = job.dims[0];
    a.n2 = job.dims[1];
    a.batch = job.batch;
    a.mode = job.mode;
    a.sign_axis = job.sign_axis;
    a.scale = job.scale;
    a.ta = job.quarter[0];
    a.tb = job.quarter[1];
    cudaError_t e;
    auto axis = [&](int ax) {  // FFT-axis tables (mixed radix or Bluestein)
      a.circle = job.circle[ax];
      a.bm = job.blue_m[ax];
      a.bchirp = job.blue_chirp[ax];
      a.bhat = job.blue_hat[ax];
      a.bcircle = job.blue_circle[ax];
    };
    if (!job.inverse) {
      a.src = in, a.dst = A;
      axis(1);
      e = g2_launch<T, G2_FWD_ROWS>(a, st);
      if (e != cudaSuccess) return e;
      a.src = A, a.dst = out;
      axis(0);
      e = g2_launch<T, G2_FWD_COLS>(a, st);
    } else {
      a.src = in, a.dst = A;
      axis(0);
      e = g2_launch<T, G2_INV_COLS>(a, st);
      if (e != cudaSuccess) return e;
      a.src = A, a.dst = out;
      axis(1);
      e = g2_launch<T, G2_INV_ROWS>(a, st);
    }
    return e;
  }
  if (!job.inverse) {
    g_gather_fwd<T><<<g, kThreads, 0, st>>>(static_cast<const T*>(in), A, d, job.batch);
    dft_all(cur, nxt, 0);
    g_post<T><<<g, kThreads, 0, st>>>(cur, static_cast<T*>(out), d, job.batch, job.quarter[0],
                                       job.quarter[1], job.quarter[2]);
  } else {
    g_pre<T><<<g, kThreads, 0, st>>>(static_cast<const T*>(in), A, d, job.batch, job.mode,
                                      job.quarter[0], job.quarter[1], job.quarter[2]);
    dft_all(cur, nxt, 1);
    g_gather_inv<T><<<g, kThreads, 0, st>>>(cur, static_cast<T*>(out), d, job.batch, job.scale,
                                             job.sign_axis);
  }
  return cudaGetLastError();
}

// ---- rfft_nd / irfft_nd (rfft.cpp:182-245) ---------------------------------
// Stage-level real FFTs with the reference's layout: full complex DFT of the
// real input along every axis, one-sided (floor(N/2)+1 entries) along the
// last axis; the inverse takes the stored half as authoritative, inverts the
// leading axes on the half-width data, fills each row's upper half by
// Hermitian symmetry and keeps the real part (unnormalised both ways).
namespace {

__global__ void g_real_to_complex(const double* __restrict__ x, double2* __restrict__ c, long long n) {
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long long>(gridDim.x) * blockDim.x)
    c[f] = make_double2(x[f], 0.0);
}

__global__ void g_take_half(const double2* __restrict__ full, double2* __restrict__ half, long long rows, int nl,
                            int h) {
  const long long total = rows * h;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = f / h;
    half[f] = full[r * nl + (f - r * h)];
  }
}

__global__ void g_hermitian_rows(const double2* __restrict__ half, double2* __restrict__ full, long long rows, int nl,
                                 int h) {
  const long long total = rows * nl;
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < total;
       f += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = f / nl;
    const int k = static_cast<int>(f - r * nl);
    double2 v = half[r * h + (k < h ? k : nl - k)];
    if (k >= h) v.y = -v.y;
    full[f] = v;
  }
}

__global__ void g_real_part(const double2* __restrict__ c, double* __restrict__ x, long long n) {
  for (long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long long>(gridDim.x) * blockDim.x)
    x[f] = c[f].x;
}

// dft_naive (rfft.cpp:113-127): direct O(n^2) sums, exact phase reduction
__global__ void g_dft_naive(const double2* __restrict__ in, double2* __restrict__ out, int n, int inverse) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double re = 0.0, im = 0.0;
  long long p = 0;
  for (int m = 0; m < n; ++m) {
    double sn, cs;
    sincospi(2.0 * static_cast<double>(p) / n, &sn, &cs);
    if (!inverse) sn = -sn;
    const double2 v = in[m];
    re += v.x * cs - v.y * sn;
    im += v.x * sn + v.y * cs;
    p += k;
    if (p >= n) p -= n;
  }
  out[k] = make_double2(re, im);
}

}  // namespace

cudaError_t generic_rfft(const GenericJob& job, const double* x, double2* half, void* ws, cudaStream_t st) {
  long long numel = 1;
  for (int a = 0; a < job.rank; ++a) numel *= job.dims[a];
  const long long total = numel * job.batch;
  const int nl = job.dims[job.rank - 1], h = nl / 2 + 1;
  double2* cur = static_cast<double2*>(ws);
  double2* nxt = cur + total;
  const int g = nblocks(total);
  g_real_to_complex<<<g, kThreads, 0, st>>>(x, cur, total);
  dft_axes(job, 0, job.rank, cur, nxt, 0, g, st);
  g_take_half<<<nblocks(total / nl * h), kThreads, 0, st>>>(cur, half, total / nl, nl, h);
  return cudaGetLastError();
}

cudaError_t generic_irfft(const GenericJob& job, const double2* half, double* x, void* ws, cudaStream_t st) {
  long long numel = 1;
  for (int a = 0; a < job.rank; ++a) numel *= job.dims[a];
  const long long total = numel * job.batch;
  const int nl = job.dims[job.rank - 1], h = nl / 2 + 1;
  const long long rows = total / nl;
  double2* cur = static_cast<double2*>(ws);
  double2* nxt = cur + total;
  cudaError_t e = cudaMemcpyAsync(cur, half, static_cast<size_t>(rows) * h * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  GenericJob jh = job;  // the leading axes run on the half-width layout
  jh.dims[job.rank - 1] = h;
  dft_axes(jh, 0, job.rank - 1, cur, nxt, 1, nblocks(rows * h), st);
  g_hermitian_rows<<<nblocks(total), kThreads, 0, st>>>(cur, nxt, rows, nl, h);
  std::swap(cur, nxt);
  dft_axes(job, job.rank - 1, job.rank, cur, nxt, 1, nblocks(total), st);
  g_real_part<<<nblocks(total), kThreads, 0, st>>>(cur, x, total);
  return cudaGetLastError();
}

cudaError_t dft_naive_run(const double2* in, double2* out, int n, bool inverse, cudaStream_t st) {
  g_dft_naive<<<(n + 127) / 128, 128, 0, st>>>(in, out, n, inverse ? 1 : 0);
  return cudaGetLastError();
}

template cudaError_t generic_run<float>(const GenericJob&, const void*, void*, void*, cudaStream_t);
template cudaError_t generic_run<double>(const GenericJob&, const void*, void*, void*, cudaStream_t);

template <typename T>
__global__ void g_force_weight(const T* __restrict__ a, T* __restrict__ aw, int n1, int n2, long long total,
                               int which) {
  const double pi = 3.14159265358979323846;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long in_item = e % (static_cast<long long>(n1) * n2);
    const int k1 = static_cast<int>(in_item / n2), k2 = static_cast<int>(in_item % n2);
    const double w1 = pi * k1 / n1, w2 = pi * k2 / n2, den = w1 * w1 + w2 * w2;
    aw[e] = den > 0.0 ? static_cast<T>(static_cast<double>(a[e]) * (which == 1 ? w1 : w2) / den) : T(0);
  }
}

cudaError_t force_weight(const void* a, void* aw, int n1, int n2, long long batch, int which, bool f32,
                         cudaStream_t st) {
  const long long total = static_cast<long long>(n1) * n2 * batch;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  if (f32)
    g_force_weight<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(a), static_cast<float*>(aw), n1, n2,
                                                  total, which);
  else
    g_force_weight<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(a), static_cast<double*>(aw), n1, n2,
                                                    total, which);
  return cudaGetLastError();
}

template <typename T>
__global__ void g_compress_threshold(const T* __restrict__ b, T* __restrict__ out, long long n, double eps,
                                     double scale, unsigned long long* count) {
  unsigned cnt = 0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = static_cast<double>(b[e]);
    const bool drop = fabs(v) < eps;
    cnt += drop ? 1u : 0u;
    out[e] = drop ? T(0) : static_cast<T>(v * scale);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt && count) atomicAdd(count, static_cast<unsigned long long>(cnt));
}

cudaError_t compress_threshold(const void* b, void* out, long long n, double eps, double scale,
                               unsigned long long* count, bool f32, cudaStream_t st) {
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148 * 16));
  if (f32)
    g_compress_threshold<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(b), static_cast<float*>(out), n,
                                                         eps, scale, count);
  else
    g_compress_threshold<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(b), static_cast<double*>(out), n,
                                                          eps, scale, count);
  return cudaGetLastError();
}

}  // namespace sdctb
