// Row-column transforms (the reference's 8-stage baselines) on the GPU.
//
//   dct_2d_rowcol            proj/src/dct2d.cpp:395-406  (dct_rows 248-290)
//   composite_2d_rowcol      proj/src/transforms_ext.cpp:287-311 (inverse_rows 40-88)
//
// The reference runs, per axis, three full-tensor stages (parity reorder, one
// real FFT per row, twiddle postprocess — or for the inverse the conjugate-
// twiddle embedding, inverse row FFTs and the parity gather) and a transpose
// between the axes. Here each axis pass is ONE kernel with the reorder fused
// into its load and the twiddle stage into its store (`rowdct_kernel`), and
// each transpose is one tiled kernel (`transpose_kernel`): 4 launches per
// transform, each one HBM round trip of the tensor, against 2 for the fused
// 2D pipeline — the structural gap the paper measures.
//
// Row DCT (N = 2M, pow2): the reordered real row x'(m) = x(pe(m)) is read as
// z(u) = x'(2u) + i x'(2u+1), which for u < M/2 is (x(4u), x(4u+2)) and for
// M-1-u is (x(4u+3), x(4u+1)) (dct1d.hpp:70-72); an M-point complex FFT
// (the register engine of kernels_fast.cuh) gives Z; X(k) = unpack(Z(k),
// conj Z(-k), W_N^k) is the rfft of x' (rfft.cpp:182-210, one-sided); the
// postprocess is y(k) = Re(b(k) X(k)) and y(N-k) = -Im(b(k) X(k))
// (b(N-k) = -i conj b(k)), dct2d.cpp:278-287.
//
// Inverse row (inverse_rows, transforms_ext.cpp:54-85): X(k) = conj(b(k)) v(k)
// for k <= M with v(k) = (x(k), -x(N-k)) [cosine] or (x(N-k), -x(k)) [sine],
// x(N) := 0 at k = 0; packed Zh(k) = (X(k) + conj X(M-k)) + i conj(W^k)(X(k) -
// conj X(M-k)); M-point inverse FFT gives zh(u) = t(2u) + i t(2u+1) with t the
// unnormalised irfft (rfft.cpp:212-245); y(m) = 1/2 t(ps(m)), odd m negated
// for the sine embedding (dct1d.hpp:77-79).
#pragma once

#include "kernels_fast.cuh"

namespace sdctb {

struct RcArgs {
  const void* src;
  void* dst;
  long long rows;    // rows of length n (all batch items stacked)
  int n;             // row length
  const void* tq;    // e^{-i pi k/(2n)}, k < n (dtype)
  const void* tw;    // W_n^k = e^{-2 pi i k/n}, k <= n/2 (dtype)
  int sine;          // inverse: reversed sine embedding + odd-index negation
};

template <typename T, int M, bool INV>
__global__ void __launch_bounds__(Tile<T, M, 2, false>::NT) rowdct_kernel(RcArgs a, TwSet tw) {
  using TL = Tile<T, M, 2, false>;
  using V = cx_t<T>;
  constexpr int NT = TL::NT;
  constexpr int R0 = TL::R0, Q0 = M / R0, NBF0 = TL::E / R0;
  constexpr int N = 2 * M;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  T* raw = reinterpret_cast<T*>(smem_raw);  // two landed real rows of N
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 2 * M * sizeof(V));
  const int t = threadIdx.x;
  const long long r0 = 2LL * blockIdx.x;
  const bool has1 = r0 + 1 < a.rows;  // an odd row count leaves line 1 of the last CTA empty
  const T* src = static_cast<const T*>(a.src);
  T* dst = static_cast<T*>(a.dst);
  const V* tq = static_cast<const V*>(a.tq);
  const V* twn = static_cast<const V*>(a.tw);
  if (t == 0) mbar_init(bar, 1);
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (t == 0) {
    const uint32_t rb = static_cast<uint32_t>(N * sizeof(T));
    mbar_expect_tx(bar, 2 * rb);
    bulk_load(raw, src + r0 * N, rb, bar);
    bulk_load(raw + N, src + (has1 ? r0 + 1 : r0) * N, rb, bar);
  }
  mbar_wait(bar, 0);
  V v[TL::E];
  if constexpr (!INV) {
    // ---- parity reorder + packing fused into the stage-0 operand reads ----
    StageTw<TL, 0> w0;
    w0.load(tw.st[0], t);
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      int line, j, b;
      TL::template decode<0>(t + i * NT, line, j, b);
      const T* x = raw + line * N;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        const int u = n < M / 2 ? n : M - 1 - n;
        v[i * R0 + r] = n < M / 2 ? mk(x[4 * u], x[4 * u + 2]) : mk(x[4 * u + 3], x[4 * u + 1]);
      }
    }
    __syncthreads();  // landed rows consumed: smem becomes the exchange buffer
    fft_regs<TL, false>(v, sm, tw, w0, t);
    __syncthreads();
    last_to_natural<TL>(v, sm, t);
    __syncthreads();
    // ---- unpack + twiddle postprocess (dct2d.cpp:278-287) ----------------
#pragma unroll
    for (int line = 0; line < 2; ++line) {
      if (line == 1 && !has1) break;
      T* y = dst + (r0 + line) * N;
      for (int k = t; k <= M / 2; k += NT) {
        const V A = sm[row_nat<T, M>(line, k)];
        const V B = sm[row_nat<T, M>(line, (M - k) & (M - 1))];
        const V wk = __ldg(twn + k), wm = __ldg(twn + (M - k));
        const V X1 = unpack(A, cconj(B), wk);  // X(k)
        const V c1 = cmul(__ldg(tq + k), X1);
        y[k] = c1.x;
        if (k > 0) y[N - k] = -c1.y;
        if (2 * k != M) {
          const int k2 = M - k;
          const V X2 = unpack(B, cconj(A), wm);  // X(M - k); X(M) at k = 0
          const V c2 = cmul(__ldg(tq + k2), X2);
          y[k2] = c2.x;
          if (k > 0) y[N - k2] = -c2.y;
        }
      }
    }
  } else {
    // ---- conjugate-twiddle embedding + inverse packing into smem ---------
    // (the landed rows and the packed spectrum share smem: read first, then
    // write after a barrier; each thread keeps its operands in registers)
    constexpr int NI = (M / 2) / NT + 1;
    V Xa[2][NI], Xb[2][NI];
#pragma unroll
    for (int line = 0; line < 2; ++line) {
      const T* x = raw + line * N;
      auto X = [&](int k) -> V {  // X(k), k in [0, M]
        const T xk = x[k];
        const T xr = k == 0 ? T(0) : x[N - k];
        const V vv = a.sine ? (k == 0 ? mk(T(0), T(0)) : mk(xr, -xk)) : mk(xk, -xr);
        return cmulc(vv, __ldg(tq + k));  // v * conj(b(k))
      };
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int k = t + i * NT;
        if (k <= M / 2) {
          Xa[line][i] = X(k);
          Xb[line][i] = X(M - k);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int line = 0; line < 2; ++line) {
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int k = t + i * NT;
        if (k <= M / 2) {
          const V wk = __ldg(twn + k);
          sm[row_nat<T, M>(line, k)] = pack(Xa[line][i], cconj(Xb[line][i]), wk);
          if (k != 0 && 2 * k != M) {
            const V wm = __ldg(twn + (M - k));
            sm[row_nat<T, M>(line, M - k)] = pack(Xb[line][i], cconj(Xa[line][i]), wm);
          }
        }
      }
    }
    StageTw<TL, 0> w0;
    w0.load(tw.st[0], t);
    __syncthreads();
    from_smem<TL, 0>(v, sm, t);
    fft_regs<TL, true>(v, sm, tw, w0, t);
    __syncthreads();
    last_to_natural<TL>(v, sm, t);
    __syncthreads();
    // ---- inverse parity gather with the 1/2 (and the sine signs) ----------
    const T s0 = T(0.5), s1 = a.sine ? T(-0.5) : T(0.5);
#pragma unroll
    for (int line = 0; line < 2; ++line) {
      if (line == 1 && !has1) break;
      T* y = dst + (r0 + line) * N;
      for (int u = t; u < M / 2; u += NT) {
        const V zu = sm[row_nat<T, M>(line, u)];
        const V zm = sm[row_nat<T, M>(line, M - 1 - u)];
        // y(4u) = t(2u), y(4u+1) = t(N-2u-1), y(4u+2) = t(2u+1), y(4u+3) = t(N-2u-2)
        y[4 * u] = s0 * zu.x;
        y[4 * u + 1] = s1 * zm.y;
        y[4 * u + 2] = s0 * zu.y;
        y[4 * u + 3] = s1 * zm.x;
      }
    }
  }
}

// Direct sums for short rows (N < 8) and any row length the fast kernel does
// not cover on a fast plan: one thread per output. Forward y(k) = sum_n x(n)
// cos(pi k (2n+1) / 2N); inverse cosine y(m) = x(0)/2 + sum_{k>=1} x(k)
// cos(pi k (2m+1) / 2N); inverse sine y(m) = sum_{k>=1} x(k) sin(pi k (2m+1) / 2N)
// (the values of dct_rows / inverse_rows, evaluated without an FFT).
template <typename T>
__global__ void rowdct_direct_kernel(RcArgs a, int inv) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int n = a.n;
  if (idx >= a.rows * n) return;
  pdl_trigger();
  pdl_wait();
  const long long r = idx / n;
  const int o = static_cast<int>(idx - r * n);
  const T* x = static_cast<const T*>(a.src) + r * n;
  const long long four = 4LL * n;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!inv) {
      const long long p = (static_cast<long long>(o) * (2 * i + 1)) % four;
      acc += static_cast<double>(x[i]) * cospi(static_cast<double>(p) / (2.0 * n));
    } else {
      const long long p = (static_cast<long long>(i) * (2 * o + 1)) % four;
      const double ph = static_cast<double>(p) / (2.0 * n);
      if (a.sine) {
        if (i > 0) acc += static_cast<double>(x[i]) * sinpi(ph);
      } else {
        acc += static_cast<double>(x[i]) * (i == 0 ? 0.5 : cospi(ph));
      }
    }
  }
  static_cast<T*>(a.dst)[idx] = static_cast<T>(acc);
}

// Batched transpose: item b of [R][C] -> [C][R], 32x32 tiles through padded
// shared memory, coalesced on both sides.
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int R, int C) {
  __shared__ T tile[32][33];
  pdl_trigger();
  pdl_wait();
  const long long item = static_cast<long long>(R) * C;
  const T* src = in + blockIdx.z * item;
  T* dst = out + blockIdx.z * item;
  const int c0 = blockIdx.x * 32, rr0 = blockIdx.y * 32;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int r = rr0 + threadIdx.y + k, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[threadIdx.y + k][threadIdx.x] = src[static_cast<long long>(r) * C + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c0 + threadIdx.y + k, r = rr0 + threadIdx.x;
    if (r < R && c < C) dst[static_cast<long long>(c) * R + r] = tile[threadIdx.x][threadIdx.y + k];
  }
}

// host launchers (kernels_rowcol.cu)
template <typename T>
cudaError_t launch_rowdct(int n, bool inv, const RcArgs& a, const TwSet& tw, cudaStream_t st);
template <typename T>
cudaError_t launch_rowdct_direct(bool inv, const RcArgs& a, cudaStream_t st);
template <typename T>
cudaError_t launch_transpose(const void* in, void* out, int R, int C, long long batch, cudaStream_t st);

}  // namespace sdctb
