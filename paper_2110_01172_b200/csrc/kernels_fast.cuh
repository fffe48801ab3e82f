// Fast-path kernels for power-of-two extents: two kernel templates carry the
// whole forward/inverse 2D and 3D pipelines of the reference (three stages:
// parity reorder, MD real FFT, twiddle/Hermitian postprocess), with the
// reorder fused into the FFT's load and the postprocess into its store.
//
//   col_kernel : FFT along a strided axis for a band of W complex columns
//                (all L rows of the band live in one CTA's shared memory).
//   row_kernel : FFT along the contiguous axis for a group of G rows that the
//                Hermitian/postprocess math couples (G = 2 in 2D: rows k1 and
//                N1-k1; G = 4 in 3D: rows (+-k1, +-k2)).
//
// Real-to-complex packing (shared by every pipeline): the reordered real line
// x' of even length N is read as the complex line z(m) = x'(2m) + i x'(2m+1),
// m < M = N/2. With the parity map (dct1d.hpp:70-72) the pair (z(u),
// z(M-1-u)) comes exactly from the contiguous source quad x(4u..4u+3):
//   z(u) = (x0, x2),  z(M-1-u) = (x3, x1).
// Intermediates store z-columns "pair-interleaved": column s = 2u holds z(u),
// s = 2u+1 holds z(M-1-u); row kernels undo that with a shared-memory scatter.
//
// Reference stages replaced (Direct orientation):
//   dct_2d           proj/src/dct2d.cpp:367-387 (+ parity_gather 48-70,
//                    rfft_nd rfft.cpp:182-210, fused_post 82-115)
//   idct family      proj/src/dct2d.cpp:410-437 (+ idct_pre 161-198,
//                    irfft_nd rfft.cpp:212-245, inverse_gather 214-238)
//   dct_3d / idct_3d proj/src/transforms_ext.cpp:322-387 (+ 99-216)
#pragma once

#include "fft_block.cuh"

namespace sdctb {

enum ColLoad { LD_SRC = 0, LD_INTER = 1 };
enum ColStore { ST_INTER = 0, ST_DST = 1 };
enum RowKind { RK_FWD2 = 0, RK_INV2 = 1, RK_FWD3 = 2, RK_INV3 = 3 };

struct ColArgs {
  const void* src;
  void* dst;
  long long in_row, in_plane, in_batch;     // element strides (T for real src, cx for complex)
  long long out_row, out_plane, out_batch;  // element strides (T for real dst, cx for complex)
  int in_plane_par;                         // >0: source plane = parity_embed(plane, n)
  int out_plane_par;                        // >0: dest plane   = parity_embed(plane, n)
  int lgw;                                  // log2(W), W complex columns per CTA
  int sign_row, sign_col;                   // final gather: negate odd k along axis
  double scale;                             // final gather scale
};

struct RowArgs {
  const void* src;
  void* dst;
  long long src_batch, dst_batch;  // element strides between batch items
  int n1, n2, n3;                  // logical extents (2D: n3 unused)
  int mode;                        // inverse composite: 0 none, 1 reverse axis 0, 2 reverse axis 1
  const void* ta;                  // e^{-i pi k/(2 N1)}, k < N1
  const void* tb;                  // e^{-i pi k/(2 N2)}, k < N2
  const void* tc;                  // e^{-i pi k/(2 N3)}, k < N3 (3D)
  const void* tu;                  // W_{Nlast}^k, k <= Nlast/2 (packing twiddles)
};

template <int L>
constexpr int col_threads() { return L >= 1024 ? 512 : 256; }
constexpr int kRowThreads = 256;

// ---- small helpers ----------------------------------------------------------
// z-column index of intermediate column s (pair-interleaved storage)
__device__ __forceinline__ int s_to_m(int s, int M) { return (s & 1) ? M - 1 - (s >> 1) : (s >> 1); }

// Hermitian unpack of the packed 2-real FFT: Z(k) = E + iO with
// E = (A + B)/2, O = -i(A - B)/2, A = Z(k), B = conj Z(-k); X = E + w O.
template <typename V>
__device__ __forceinline__ V unpack(V A, V B, V w) {
  const V e = mk((A.x + B.x) * 0.5f, (A.y + B.y) * 0.5f);
  const V d = mk((A.x - B.x) * 0.5f, (A.y - B.y) * 0.5f);
  const V o = mk(d.y, -d.x);  // -i * d
  return cadd(e, cmul(w, o));
}
// Inverse packing: Zh = (X + Xhi) + i conj(w) (X - Xhi)
template <typename V>
__device__ __forceinline__ V pack(V X, V Xhi, V w) {
  const V s = cadd(X, Xhi);
  const V t = cmulc(csub(X, Xhi), w);  // (X - Xhi) * conj(w)
  return mk(s.x - t.y, s.y + t.x);     // s + i t
}

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };

// ============================================================================
// Column kernel
// ============================================================================
template <typename T, int L, bool INV, int LOAD, int STORE>
__global__ void __launch_bounds__(col_threads<L>())
    col_kernel(ColArgs a, const cx_t<T>* __restrict__ tw, int tw_step) {
  using V = cx_t<T>;
  using V4 = typename Vec16<T>::type;
  constexpr int NT = col_threads<L>();
  constexpr int VEC = 16 / sizeof(T);   // reals per 16-B vector
  constexpr int CPV = 16 / sizeof(V);   // complex per 16-B vector
  constexpr int U = 4;                  // loads in flight per thread per batch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);
  const int lgw = a.lgw;
  const int W = 1 << lgw;
  const ColLayout<T> lay{lgw};
  const int tid = threadIdx.x;
  const int band = blockIdx.x, plane = blockIdx.y, batch = blockIdx.z;

  // ---------------------------------------------------------------- load ---
  if constexpr (LOAD == LD_SRC) {
    // real source, parity reorder along the FFT axis (rows) and the packed
    // contiguous axis; a band is 2W contiguous reals per row.
    const int pl = a.in_plane_par ? parity_embed(plane, a.in_plane_par) : plane;
    const T* src = static_cast<const T*>(a.src) + batch * a.in_batch + pl * a.in_plane +
                   static_cast<long long>(band) * (2 * W);
    const int lg_vpr = lgw + 1 - ilog2c(VEC);  // vectors per row = 2W / VEC
    const int nvec = L << lg_vpr;
    for (int v0 = 0; v0 < nvec; v0 += NT * U) {
      V4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * NT + tid;
        if (v < nvec) {
          const int r = v >> lg_vpr, vi = v & ((1 << lg_vpr) - 1);
          t[u] = __ldg(reinterpret_cast<const V4*>(src + r * a.in_row + vi * VEC));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * NT + tid;
        if constexpr (sizeof(T) == 4) {
          if (v < nvec) {
            const int r = v >> lg_vpr, g = v & ((1 << lg_vpr) - 1);
            const int slot = parity_source(r, L);
            const float4 x = reinterpret_cast<const float4&>(t[u]);
            buf[lay.at(2 * g, slot)] = mk(x.x, x.z);
            buf[lay.at(2 * g + 1, slot)] = mk(x.w, x.y);
          }
        } else {
          // fp64: a source quad spans two lanes; swap the middle reals.
          if (v0 + u * NT < nvec) {  // warp-uniform (nvec is a multiple of 2)
            const int r = v >> lg_vpr, vi = v & ((1 << lg_vpr) - 1);
            const int g = vi >> 1, h = vi & 1;
            const double2 x = reinterpret_cast<const double2&>(t[u]);
            const double send = h ? x.x : x.y;
            const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
            if (v < nvec) {
              const int slot = parity_source(r, L);
              buf[lay.at(2 * g + h, slot)] = h ? mk(x.y, recv) : mk(x.x, recv);
            }
          }
        }
      }
    }
  } else {
    const V* src = static_cast<const V*>(a.src) + batch * a.in_batch + plane * a.in_plane +
                   static_cast<long long>(band) * W;
    const int lg_vpr = lgw - ilog2c(CPV);
    const int nvec = L << lg_vpr;
    for (int v0 = 0; v0 < nvec; v0 += NT * U) {
      V4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * NT + tid;
        if (v < nvec) {
          const int r = v >> lg_vpr, ci = v & ((1 << lg_vpr) - 1);
          t[u] = __ldg(reinterpret_cast<const V4*>(src + r * a.in_row + ci * CPV));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * NT + tid;
        if (v < nvec) {
          const int r = v >> lg_vpr, ci = v & ((1 << lg_vpr) - 1);
          const V* e = reinterpret_cast<const V*>(&t[u]);
#pragma unroll
          for (int k = 0; k < CPV; ++k) buf[lay.at(ci * CPV + k, r)] = e[k];
        }
      }
    }
  }
  __syncthreads();

  // ----------------------------------------------------------------- FFT ---
  block_fft<T, L, INV, true>(buf, lay, lgw, tw, tw_step);

  // --------------------------------------------------------------- store ---
  if constexpr (STORE == ST_INTER) {
    V* dst = static_cast<V*>(a.dst) + batch * a.out_batch + plane * a.out_plane +
             static_cast<long long>(band) * W;
    const int lg_vpr = lgw - ilog2c(CPV);
    const int nvec = L << lg_vpr;
    for (int v = tid; v < nvec; v += NT) {
      const int r = v >> lg_vpr, ci = v & ((1 << lg_vpr) - 1);
      const int slot = digit_pos<L>(r);
      V4 o;
      V* e = reinterpret_cast<V*>(&o);
#pragma unroll
      for (int k = 0; k < CPV; ++k) e[k] = buf[lay.at(ci * CPV + k, slot)];
      *reinterpret_cast<V4*>(dst + r * a.out_row + ci * CPV) = o;
    }
  } else {
    // final inverse gather: y(k1, 4u+c) from z(ps(k1)), scale and signs
    const int pl = a.out_plane_par ? parity_embed(plane, a.out_plane_par) : plane;
    T* dst = static_cast<T*>(a.dst) + batch * a.out_batch + pl * a.out_plane +
             static_cast<long long>(band) * (2 * W);
    const T sc = static_cast<T>(a.scale);
    const int lg_vpr = lgw + 1 - ilog2c(VEC);
    const int nvec = L << lg_vpr;
    for (int v = tid; v < nvec; v += NT) {
      const int k1 = v >> lg_vpr, vi = v & ((1 << lg_vpr) - 1);
      const int slot = digit_pos<L>(parity_source(k1, L));
      const T srow = (a.sign_row && (k1 & 1)) ? -sc : sc;
      const T scol = a.sign_col ? -srow : srow;
      if constexpr (sizeof(T) == 4) {
        const int g = vi;
        const V zg = buf[lay.at(2 * g, slot)], zm = buf[lay.at(2 * g + 1, slot)];
        *reinterpret_cast<float4*>(dst + k1 * a.out_row + 4 * g) =
            make_float4(zg.x * srow, zm.y * scol, zg.y * srow, zm.x * scol);
      } else {
        const int g = vi >> 1, h = vi & 1;
        const V zg = buf[lay.at(2 * g, slot)], zm = buf[lay.at(2 * g + 1, slot)];
        const double2 o = h ? make_double2(zg.y * srow, zm.x * scol)
                            : make_double2(zg.x * srow, zm.y * scol);
        *reinterpret_cast<double2*>(dst + k1 * a.out_row + 4 * g + 2 * h) = o;
      }
    }
  }
}

// ============================================================================
// Row-group kernel
// ============================================================================
template <typename T>
__device__ __forceinline__ T fetch2(const T* x, int i, int j, int n1, int n2, int mode) {
  // proj/src/dct2d.cpp:169-180: index N reads 0; composite modes read one
  // axis reversed with a zero first slot.
  if (i == n1 || j == n2) return T(0);
  if (mode == 1) {
    if (i == 0) return T(0);
    i = n1 - i;
  } else if (mode == 2) {
    if (j == 0) return T(0);
    j = n2 - j;
  }
  return __ldg(x + static_cast<long long>(i) * n2 + j);
}

// Merged inverse preprocess item (q1, n2) (proj/src/dct2d.cpp:182-195):
// returns X'(q1, n2) and X'(r1, n2) from the four shared reads.
template <typename T>
__device__ __forceinline__ void pre2_item(const T* x, int q1, int n2i, const RowArgs& a,
                                          cx_t<T>& xq, cx_t<T>& xr) {
  using V = cx_t<T>;
  const int n1 = a.n1, n2 = a.n2;
  const T p = fetch2(x, q1, n2i, n1, n2, a.mode);
  const T q = fetch2(x, n1 - q1, n2 - n2i, n1, n2, a.mode);
  const T r = fetch2(x, n1 - q1, n2i, n1, n2, a.mode);
  const T s = fetch2(x, q1, n2 - n2i, n1, n2, a.mode);
  const V* ta = static_cast<const V*>(a.ta);
  const V* tb = static_cast<const V*>(a.tb);
  const V wb = __ldg(tb + n2i);
  const int r1 = (n1 - q1) & (n1 - 1);
  const V w1 = cconj(cmul(__ldg(ta + q1), wb));  // conj(a) conj(b)
  const V w2 = cconj(cmul(__ldg(ta + r1), wb));
  xq = cmul(w1, mk(p - q, -(r + s)));
  xr = cmul(w2, mk(r - s, -(p + q)));
}

template <typename T>
__device__ __forceinline__ T fetch3(const T* x, int i, int j, int k, int n1, int n2, int n3) {
  if (i == n1 || j == n2 || k == n3) return T(0);
  return __ldg(x + (static_cast<long long>(i) * n2 + j) * n3 + k);
}

// Literal 3D inverse preprocess entry (proj/src/transforms_ext.cpp:196-212).
template <typename T>
__device__ __forceinline__ cx_t<T> pre3_entry(const T* x, int i, int j, int k, const RowArgs& a) {
  using V = cx_t<T>;
  const int n1 = a.n1, n2 = a.n2, n3 = a.n3;
  const int r1 = n1 - i, r2 = n2 - j, r3 = n3 - k;
  const T re = (fetch3(x, i, j, k, n1, n2, n3) - fetch3(x, r1, r2, k, n1, n2, n3)) -
               (fetch3(x, r1, j, r3, n1, n2, n3) + fetch3(x, i, r2, r3, n1, n2, n3));
  const T im = fetch3(x, r1, r2, r3, n1, n2, n3) -
               ((fetch3(x, r1, j, k, n1, n2, n3) + fetch3(x, i, r2, k, n1, n2, n3)) +
                fetch3(x, i, j, r3, n1, n2, n3));
  const V w = cconj(cmul(cmul(__ldg(static_cast<const V*>(a.ta) + i), __ldg(static_cast<const V*>(a.tb) + j)),
                         __ldg(static_cast<const V*>(a.tc) + k)));
  return cmul(w, mk(re, im));
}

template <typename T, int M, int KIND>
__global__ void __launch_bounds__(kRowThreads)
    row_kernel(RowArgs a, const cx_t<T>* __restrict__ tw, int tw_step) {
  using V = cx_t<T>;
  using V4 = typename Vec16<T>::type;
  constexpr int G = (KIND == RK_FWD2 || KIND == RK_INV2) ? 2 : 4;
  constexpr bool INV = (KIND == RK_INV2 || KIND == RK_INV3);
  constexpr int CPV = 16 / sizeof(V);
  constexpr int NT = kRowThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);
  const RowLayout<T, M> lay;
  const int tid = threadIdx.x;
  const int P = blockIdx.x, batch = blockIdx.y;
  const int n1 = a.n1, n2 = a.n2;

  // rows of this group and their degeneracy
  int rows[G];
  bool deg1 = false, deg2 = false;
  int q1 = 0, q2 = 0, m1 = 0, m2 = 0;
  if constexpr (G == 2) {
    q1 = P == 0 ? 0 : P;
    m1 = P == 0 ? n1 / 2 : n1 - P;
    rows[0] = q1;
    rows[1] = m1;
  } else {
    const int h2 = n2 / 2 + 1;
    q1 = P / h2;
    q2 = P - q1 * h2;
    m1 = (n1 - q1) & (n1 - 1);
    m2 = (n2 - q2) & (n2 - 1);
    deg1 = m1 == q1;
    deg2 = m2 == q2;
    rows[0] = q1 * n2 + q2;
    rows[1] = m1 * n2 + q2;
    rows[2] = q1 * n2 + m2;
    rows[3] = m1 * n2 + m2;
  }

  // ---------------------------------------------------------------- load ---
  if constexpr (!INV) {
    const V* src = static_cast<const V*>(a.src) + batch * a.src_batch;
    constexpr int VPR = M / CPV;
    for (int v = tid; v < G * VPR; v += NT) {
      const int line = v / VPR, ci = v - line * VPR;
      const V4 t = __ldg(reinterpret_cast<const V4*>(src + static_cast<long long>(rows[line]) * M + ci * CPV));
      const V* e = reinterpret_cast<const V*>(&t);
#pragma unroll
      for (int k = 0; k < CPV; ++k) buf[lay.at(line, s_to_m(ci * CPV + k, M))] = e[k];
    }
  } else if constexpr (KIND == RK_INV2) {
    const T* x = static_cast<const T*>(a.src) + batch * a.src_batch;
    const V* tu = static_cast<const V*>(a.tu);
    for (int k = tid; k <= M / 2; k += NT) {
      V A0, A1, B0, B1;  // X'(line, k), X'(line, M-k)
      if (P != 0) {
        pre2_item(x, q1, k, a, A0, A1);
        pre2_item(x, q1, M - k, a, B0, B1);
      } else {
        V d0, d1;
        pre2_item(x, 0, k, a, A0, d0);
        pre2_item(x, n1 / 2, k, a, A1, d1);
        pre2_item(x, 0, M - k, a, B0, d0);
        pre2_item(x, n1 / 2, M - k, a, B1, d1);
      }
      // partner line of each row (-k1): swap for pairs, self for P == 0
      const V pA0 = P != 0 ? A1 : A0, pA1 = P != 0 ? A0 : A1;
      const V pB0 = P != 0 ? B1 : B0, pB1 = P != 0 ? B0 : B1;
      const V wk = __ldg(tu + k);
      buf[lay.at(0, k)] = pack(A0, k == 0 ? B0 : cconj(pB0), wk);
      buf[lay.at(1, k)] = pack(A1, k == 0 ? B1 : cconj(pB1), wk);
      if (k != 0 && 2 * k != M) {
        const V wmk = __ldg(tu + (M - k));
        buf[lay.at(0, M - k)] = pack(B0, cconj(pA0), wmk);
        buf[lay.at(1, M - k)] = pack(B1, cconj(pA1), wmk);
      }
    }
  } else {  // RK_INV3
    const T* x = static_cast<const T*>(a.src) + batch * a.src_batch;
    const V* tu = static_cast<const V*>(a.tu);
    const int li[4] = {q1, m1, q1, m1}, lj[4] = {q2, q2, m2, m2};
    for (int k = tid; k <= M / 2; k += NT) {
      V A[4], B[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        A[l] = pre3_entry(x, li[l], lj[l], k, a);
        B[l] = pre3_entry(x, li[l], lj[l], M - k, a);
      }
      const V wk = __ldg(tu + k);
#pragma unroll
      for (int l = 0; l < 4; ++l) buf[lay.at(l, k)] = pack(A[l], k == 0 ? B[l] : cconj(B[3 - l]), wk);
      if (k != 0 && 2 * k != M) {
        const V wmk = __ldg(tu + (M - k));
#pragma unroll
        for (int l = 0; l < 4; ++l) buf[lay.at(l, M - k)] = pack(B[l], cconj(A[3 - l]), wmk);
      }
    }
  }
  __syncthreads();

  // ----------------------------------------------------------------- FFT ---
  block_fft<T, M, INV, false>(buf, lay, ilog2c(G), tw, tw_step);

  // --------------------------------------------------------------- store ---
  if constexpr (INV) {
    V* dst = static_cast<V*>(a.dst) + batch * a.dst_batch;
    constexpr int VPR = M / CPV;
    for (int v = tid; v < G * VPR; v += NT) {
      const int line = v / VPR, ci = v - line * VPR;
      if (G == 4 && ((line == 1 && deg1) || (line == 2 && deg2) || (line == 3 && (deg1 || deg2))))
        continue;
      V4 o;
      V* e = reinterpret_cast<V*>(&o);
#pragma unroll
      for (int k = 0; k < CPV; ++k) e[k] = buf[lay.at(line, digit_pos<M>(s_to_m(ci * CPV + k, M)))];
      *reinterpret_cast<V4*>(dst + static_cast<long long>(rows[line]) * M + ci * CPV) = o;
    }
  } else if constexpr (KIND == RK_FWD2) {
    // merged DCT postprocess (proj/src/dct2d.cpp:93-113) on the unpacked rows
    T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
    const V* ta = static_cast<const V*>(a.ta);
    const V* tb = static_cast<const V*>(a.tb);
    const V* tu = static_cast<const V*>(a.tu);
    for (int k2 = tid; k2 <= M; k2 += NT) {
      const int ka = digit_pos<M>(k2 & (M - 1)), kb = digit_pos<M>((M - k2) & (M - 1));
      const V w = __ldg(tu + k2), b = __ldg(tb + k2);
      const bool deg2k = (k2 == 0) || (k2 == M);
      const V Z0a = buf[lay.at(0, ka)], Z0b = buf[lay.at(0, kb)];
      const V Z1a = buf[lay.at(1, ka)], Z1b = buf[lay.at(1, kb)];
      if (P != 0) {
        const V X1 = unpack(Z0a, cconj(Z1b), w);
        const V X2 = unpack(Z1a, cconj(Z0b), w);
        const V av = __ldg(ta + q1);
        const V ax1 = cmul(av, X1), ax2 = cmulc(X2, av);
        const V s = cmul(b, cadd(ax1, ax2)), t = cmul(b, csub(ax1, ax2));
        T* r0 = y + static_cast<long long>(q1) * n2;
        T* r1 = y + static_cast<long long>(m1) * n2;
        r0[k2] = T(0.5) * s.x;
        r1[k2] = T(-0.5) * t.y;
        if (!deg2k) {
          r0[n2 - k2] = T(-0.5) * s.y;
          r1[n2 - k2] = T(-0.5) * t.x;
        }
      } else {
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          const int row = l == 0 ? 0 : n1 / 2;
          const V X1 = l == 0 ? unpack(Z0a, cconj(Z0b), w) : unpack(Z1a, cconj(Z1b), w);
          const V av = __ldg(ta + row);
          const V s = cmul(b, cadd(cmul(av, X1), cmulc(X1, av)));
          T* r0 = y + static_cast<long long>(row) * n2;
          r0[k2] = T(0.5) * s.x;
          if (!deg2k) r0[n2 - k2] = T(-0.5) * s.y;
        }
      }
    }
  } else {  // RK_FWD3: merged 3D postprocess (proj/src/transforms_ext.cpp:117-157)
    T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
    const int n3 = a.n3;
    const V* tu = static_cast<const V*>(a.tu);
    const V av = __ldg(static_cast<const V*>(a.ta) + q1);
    const V bv = __ldg(static_cast<const V*>(a.tb) + q2);
    const V ab = cmul(av, bv), cb = cmulc(bv, av);  // a b, conj(a) b
    auto put = [&](int i, int j, int k, T v) { y[(static_cast<long long>(i) * n2 + j) * n3 + k] = v; };
    for (int k3 = tid; k3 <= M; k3 += NT) {
      const int ka = digit_pos<M>(k3 & (M - 1)), kb = digit_pos<M>((M - k3) & (M - 1));
      const V w = __ldg(tu + k3);
      V X[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) X[l] = unpack(buf[lay.at(l, ka)], cconj(buf[lay.at(3 - l, kb)]), w);
      const bool deg3 = (k3 == 0) || (k3 == M);
      const int m3 = n3 - k3;
      const V f1 = X[0];
      const V f2 = deg1 ? f1 : X[1];
      const V f3 = deg2 ? f1 : X[2];
      const V f4 = deg1 ? f3 : (deg2 ? f2 : X[3]);
      const V c = __ldg(static_cast<const V*>(a.tc) + k3);
      const V t1 = cmul(ab, f1), t2 = cmul(cb, f2), t3 = cmul(cconj(cb), f3), t4 = cmul(cconj(ab), f4);
      const V s12 = cadd(t1, t2), s34 = cadd(t3, t4);
      const V u00 = cmul(c, cadd(s12, s34));
      put(q1, q2, k3, T(0.25) * u00.x);
      if (!deg3) put(q1, q2, m3, T(-0.25) * u00.y);
      if (!deg2) {
        const V u01 = cmul(c, csub(s12, s34));
        put(q1, m2, k3, T(-0.25) * u01.y);
        if (!deg3) put(q1, m2, m3, T(-0.25) * u01.x);
      }
      if (!deg1) {
        const V d12 = csub(t1, t2), d34 = csub(t3, t4);
        const V u10 = cmul(c, cadd(d12, d34));
        put(m1, q2, k3, T(-0.25) * u10.y);
        if (!deg3) put(m1, q2, m3, T(-0.25) * u10.x);
        if (!deg2) {
          const V u11 = cmul(c, csub(d12, d34));
          put(m1, m2, k3, T(-0.25) * u11.x);
          if (!deg3) put(m1, m2, m3, T(0.25) * u11.y);
        }
      }
    }
  }
}

}  // namespace sdctb
