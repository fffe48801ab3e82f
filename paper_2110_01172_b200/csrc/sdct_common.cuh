// Shared device helpers for the sdct-b200 kernels: complex arithmetic on the
// native vector types (float2 / double2), the 1D parity maps of the
// reference, and launch-error plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sdctb {

template <typename T> struct Cx;
template <> struct Cx<float> { using type = float2; using vec4 = float4; };
template <> struct Cx<double> { using type = double2; using vec4 = double2; };

template <typename T> using cx_t = typename Cx<T>::type;

__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return mk(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return mk(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cconj(V a) { return mk(a.x, -a.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// multiply by -i (forward) or +i (inverse)
template <bool INV, typename V> __device__ __forceinline__ V mul_mi(V a) {
  return INV ? mk(-a.y, a.x) : mk(a.y, -a.x);
}


// Reference parity maps (proj/include/sdct/dct1d.hpp:70-79). The forward
// reorder puts x(2m) in slot m for m <= (n-1)/2 and x(2n-2m-1) otherwise;
// parity_source is its inverse seen from the output side.
__host__ __device__ __forceinline__ int parity_embed(int m, int n) {
  return (m <= (n - 1) / 2) ? 2 * m : 2 * n - 2 * m - 1;
}
__host__ __device__ __forceinline__ int parity_source(int m, int n) {
  return (m & 1) == 0 ? (m >> 1) : n - ((m + 1) >> 1);
}

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

}  // namespace sdctb
