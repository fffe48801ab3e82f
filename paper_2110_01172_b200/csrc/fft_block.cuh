// Building blocks of the in-CTA power-of-two FFT engine (kernels_fast.cuh):
// the radix plan (ceil(log2 L / 4) stages of radix <= 16), mixed-radix digit
// reversal (after the DIF stages X(k) sits at slot digit_pos<L>(k); callers
// absorb that permutation into their store index math, so no reorder pass
// exists), the GF(2)-linear shared-memory swizzles, and the fully unrolled
// in-register radix-R DFTs.
//
// This replaces the reference's scalar radix-2 FftWorkspace::pow2_fft
// (proj/src/rfft.cpp:65-89) for the power-of-two extents of the hot path.
//
// Shared-memory layouts are XOR-swizzled so that every FFT stage's exchange
// pattern is bank-conflict free (tests/test_host.py replays the exact index
// math below through tests/swizzle_model.py). Accesses outside the stage
// exchanges are not covered by that claim: the forward row kernels' stage-0
// reads of bulk-landed pair-interleaved rows (stride-2 columns, 2-way) and
// the mirror-paired radix-8 stage at M = 1024 (2-way; also modelled in
// tests/test_host.py) — see DESIGN.md §6b for what removing them cost.
#pragma once

#include "sdct_common.cuh"

namespace sdctb {

// ---- radix plan: ceil(log2(L)/4) stages, bits spread evenly, larger first --
template <int L>
struct RadixPlan {
  static constexpr int lg = ilog2c(L);
  static constexpr int S = lg == 0 ? 0 : (lg + 3) / 4;
  static constexpr int bits(int s) { return lg / S + (s < lg % S ? 1 : 0); }
  static constexpr int R(int s) { return 1 << bits(s); }
  // span(s): length of the sub-FFTs stage s operates on; span(S) == 1.
  static constexpr int span(int s) {
    int ls = L;
    for (int t = 0; t < s; ++t) ls /= R(t);
    return ls;
  }
};

// Slot holding X(k) after all DIF stages: k = d0 + R0 d1 + R0 R1 d2 + ...,
// pos = sum_s d_s * span(s+1).
template <int L>
__host__ __device__ __forceinline__ int digit_pos(int k) {
  using P = RadixPlan<L>;
  int pos = 0;
#pragma unroll
  for (int s = 0; s < P::S; ++s) {
    const int r = P::R(s);
    pos += (k & (r - 1)) * P::span(s + 1);
    k >>= P::bits(s);
  }
  return pos;
}

// Inverse of digit_pos: frequency index held at slot n.
template <int L>
__host__ __device__ __forceinline__ int digit_rev(int n) {
  using P = RadixPlan<L>;
  int k = 0, shift = 0;
#pragma unroll
  for (int s = 0; s < P::S; ++s) {
    k |= ((n / P::span(s + 1)) & (P::R(s) - 1)) << shift;
    shift += P::bits(s);
  }
  return k;
}

// Runtime versions for extents only known at run time (row selection of the
// intermediate, 3D plane mapping). Same radix plan as RadixPlan<L>.
__host__ __device__ inline int rt_digit_pos(int k, int L) {
  int lg = 0;
  while ((1 << lg) < L) ++lg;
  if (lg == 0) return 0;
  const int S = (lg + 3) / 4;
  int span = L, pos = 0;
  for (int s = 0; s < S; ++s) {
    const int b = lg / S + (s < lg % S ? 1 : 0);
    span >>= b;
    pos += (k & ((1 << b) - 1)) * span;
    k >>= b;
  }
  return pos;
}

// ---- bank-conflict-free swizzles (index in complex elements) ---------------
// GF(2)-linear maps a -> a ^ g(a >> SH), g(h) = XOR of C[d % 4] over the set
// bits d of h. 16-B elements (SH = 3) are served 8 lanes per wavefront, 8-B
// elements (SH = 4) 16 lanes. Column tiles use constants that make every
// aligned dyadic window injective; row tiles use constants found by
// exhaustive search over the row kernel's stage patterns. tests/swizzle_model.py
// replays this math and tests/test_host.py asserts conflict degree 1.
// Linearity lets a butterfly swizzle its base once and XOR per-element offsets.
template <int C0, int C1, int C2, int C3, int SH>
struct LinSwz {
  // g as a 16-entry nibble table indexed by the 4 class parities (p0..p3)
  static constexpr unsigned long long nib_table() {
    unsigned long long t = 0;
    for (int p = 0; p < 16; ++p) {
      const int v = ((p & 1) ? C0 : 0) ^ ((p & 2) ? C1 : 0) ^ ((p & 4) ? C2 : 0) ^ ((p & 8) ? C3 : 0);
      t |= static_cast<unsigned long long>(v & 15) << (4 * p);
    }
    return t;
  }
  __host__ __device__ __forceinline__ static int g(unsigned h) {
#if defined(__CUDA_ARCH__)
    // fold the parities of the bit classes d % 4 into bits 0..3 (smem
    // indices are < 2^16 elements, so h < 2^16), then one table lookup
    h ^= h >> 8;
    h ^= h >> 4;
    return static_cast<int>((nib_table() >> ((h & 15u) * 4u)) & 15u);
#else
    int r = 0;
    for (int d = 0; h; ++d, h >>= 1)
      if (h & 1u) r ^= (d & 3) == 0 ? C0 : (d & 3) == 1 ? C1 : (d & 3) == 2 ? C2 : C3;
    return r;
#endif
  }
  __host__ __device__ __forceinline__ static int f(int a) {
    return a ^ g(static_cast<unsigned>(a) >> SH);
  }
  // constexpr evaluation for compile-time offsets
  static constexpr int fc(int a) {
    int r = 0;
    unsigned h = static_cast<unsigned>(a) >> SH;
    for (int d = 0; h; ++d, h >>= 1)
      if (h & 1u) r ^= (d & 3) == 0 ? C0 : (d & 3) == 1 ? C1 : (d & 3) == 2 ? C2 : C3;
    return a ^ r;
  }
};
template <typename T> struct SwzCol;
template <> struct SwzCol<double> : LinSwz<4, 6, 5, 7, 3> {};
template <> struct SwzCol<float> : LinSwz<8, 12, 10, 15, 4> {};
template <typename T> struct SwzRow;
template <> struct SwzRow<double> : LinSwz<1, 2, 4, 1, 3> {};
template <> struct SwzRow<float> : LinSwz<1, 6, 10, 8, 4> {};

// ---- in-register radix-R DFT, natural order in and out ---------------------
template <typename T> struct K16;
template <> struct K16<double> {
  // cos(2 pi m / 16), m = 0..4
  __device__ __forceinline__ static double c(int m) {
    return m == 0 ? 1.0 : m == 1 ? 0.92387953251128675613 : m == 2 ? 0.70710678118654752440
         : m == 3 ? 0.38268343236508977173 : 0.0;
  }
};
template <> struct K16<float> {
  __device__ __forceinline__ static float c(int m) {
    return m == 0 ? 1.0f : m == 1 ? 0.92387953251128675613f : m == 2 ? 0.70710678118654752440f
         : m == 3 ? 0.38268343236508977173f : 0.0f;
  }
};

// multiply by W_R^k = exp(-+ 2 pi i k / R); k, R compile-time after unrolling
template <typename T, bool INV>
__device__ __forceinline__ cx_t<T> mul_wrk(cx_t<T> v, int k, int R) {
  const int m16 = (k * 16) / R;  // angle in units of 2pi/16, 0..15
  if (m16 == 0) return v;
  if (m16 == 4) return mul_mi<INV>(v);
  if (m16 == 8) return mk(-v.x, -v.y);
  if (m16 == 12) return mul_mi<!INV>(v);
  // generic: exp(-i theta) forward, exp(+i theta) inverse, theta = 2 pi m16 / 16
  const int q = m16 & 3, quad = m16 >> 2;  // theta = quad*pi/2 + q*pi/8
  T c = K16<T>::c(q), s = K16<T>::c(4 - q);  // cos, sin of q*pi/8
  // rotate by quad quarter turns
  T cr = c, sr = s;
  if (quad == 1) { cr = -s; sr = c; }
  if (quad == 2) { cr = -c; sr = -s; }
  if (quad == 3) { cr = s; sr = -c; }
  if (!INV) sr = -sr;
  return mk(v.x * cr - v.y * sr, v.x * sr + v.y * cr);
}

template <typename T, int R, bool INV>
__device__ __forceinline__ void dft_reg(cx_t<T>* v) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const cx_t<T> a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else {
    cx_t<T> e[R / 2], o[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) {
      e[r] = v[2 * r];
      o[r] = v[2 * r + 1];
    }
    dft_reg<T, R / 2, INV>(e);
    dft_reg<T, R / 2, INV>(o);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const cx_t<T> t = mul_wrk<T, INV>(o[k], k, R);
      v[k] = cadd(e[k], t);
      v[k + R / 2] = csub(e[k], t);
    }
  }
}

}  // namespace sdctb
