// Fast-path kernels for power-of-two extents: two kernel templates carry the
// whole forward/inverse 2D and 3D pipelines of the reference (three stages:
// parity reorder, MD real FFT, twiddle/Hermitian postprocess), with the
// reorder fused into the FFT's load and the postprocess into its store.
//
//   col_kernel : FFT along a strided axis for a band of NL complex columns
//                (all L rows of the band live in one CTA).
//   row_kernel : FFT along the contiguous axis for a group of G rows that the
//                Hermitian/postprocess math couples (G = 2 in 2D: rows k1 and
//                N1-k1; G = 4 in 3D: rows (+-k1, +-k2)).
//
// Register-resident engine (v2): every tile geometry is compile time. Each
// thread owns E = L*NL/NT elements; in stage s it runs E/R_s radix-R_s DIF
// butterflies whose shared-memory slots are a per-thread swizzled base XOR
// compile-time offsets (the swizzle is GF(2)-linear and the offset bits are
// disjoint from the base bits). Stage-0 operands are loaded from global memory
// straight into registers (column kernels, forward row kernels) and the last
// stage leaves its results in registers (column kernels store them straight
// to global memory), so an S-stage FFT makes S-1 shared-memory round trips.
// Twiddles come from per-stage tables W_span^{jk} laid out [k-1][j] (one
// coalesced, L1-resident load per factor) instead of a recurrence.
//
// Real-to-complex packing (shared by every pipeline): the reordered real line
// x' of even length N is read as the complex line z(m) = x'(2m) + i x'(2m+1),
// m < M = N/2. With the parity map (dct1d.hpp:70-72) the pair (z(u),
// z(M-1-u)) comes exactly from the contiguous source quad x(4u..4u+3):
//   z(u) = (x0, x2),  z(M-1-u) = (x3, x1).
// Intermediates store z-columns "pair-interleaved": column s = 2u holds z(u),
// s = 2u+1 holds z(M-1-u). Forward intermediates keep the column-FFT output
// rows in slot (digit-reversed) order; row kernels select rows through
// rt_digit_pos, so no reorder pass exists anywhere.
//
// Reference stages replaced (Direct orientation):
//   dct_2d           proj/src/dct2d.cpp:367-387 (+ parity_gather 48-70,
//                    rfft_nd rfft.cpp:182-210, fused_post 82-115)
//   idct family      proj/src/dct2d.cpp:410-437 (+ idct_pre 161-198,
//                    irfft_nd rfft.cpp:212-245, inverse_gather 214-238)
//   dct_3d / idct_3d proj/src/transforms_ext.cpp:322-387 (+ 99-216)
#pragma once

#include "fft_block.cuh"
#include "tma.cuh"

namespace sdctb {

enum ColLoad { LD_SRC = 0, LD_INTER = 1 };

// The forward source pass lands its rows by parity class (even rows, then odd
// rows) when the odd-class half starts 128-B aligned in shared memory (TMA
// destination alignment); otherwise in natural row order. Host and kernel
// pick the tensor map / index math from this one predicate.
__host__ __device__ constexpr bool col_class_load(int esize, int L, int nl) {
  return L >= 2 && ((L / 2) * 2 * nl * esize) % 128 == 0;
}
enum ColStore { ST_INTER = 0, ST_DST = 1 };
enum RowKind { RK_FWD2 = 0, RK_INV2 = 1, RK_FWD3 = 2, RK_INV3 = 3 };

// Per-stage twiddle tables of one FFT length: st[s][(k-1)*Q + j] = W_span^{j k}.
struct TwSet {
  const void* st[4];
};

struct ColArgs {
  const void* src;
  void* dst;
  long long in_row, in_plane, in_batch;     // element strides (T for real src, cx for complex)
  long long out_row, out_plane, out_batch;  // element strides (T for real dst, cx for complex)
  int in_plane_par;                         // >0: source plane = parity_embed(plane, n)
  int out_plane_map;                        // ST_DST: 0 plane, 1 pe(plane), 2 pe(digit_rev(plane))
  int out_plane_n;                          // extent used by out_plane_map
  int sign_row, sign_col;                   // final gather: negate odd k along axis
  int pair_b, sign_row2, sign_col2;         // paired inverse launch: batch items >= pair_b use the *2 signs
  double scale;                             // final gather scale
  int tma_plane_par;                        // TMA plane coordinate = parity_embed(plane, n) when > 0
  const void* twc;                          // cluster-split pass: W_L^k, k < L/2
  int nbands, nplanes, ntiles;              // persistent column kernels: tile = band + nbands*(plane + nplanes*batch)
  unsigned long long* trace;                // debug: per-tile phase timestamps (nullptr in production)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

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
  const int* s0;                   // storage row of frequency k1 in the intermediate: rt_srow(k1, n1)
  const int* s1;                   // 3D: rt_srow(k2, n2)
  const void* fb;                  // factor tables of tb / tu: e^{-i theta q} = hi[q >> fs] lo[q & (2^fs-1)]
  const void* fu;
  int fs;
  const unsigned char* badq;       // corrupt_twiddle_for_testing: b(q) negated where badq[q] != 0 (null: none)
  int weight;                      // 2D inverse input: 0 none, 1/2 force-field weight w1/w2, 3 compression threshold
  double thr_eps, thr_scale;       // weight 3: zero |b| < thr_eps, scale the rest
  unsigned long long* thr_count;   // weight 3: zeroed coefficients (device counter, may be null)
  // paired inverse launch (force fields: both composites in one launch): batch
  // items b >= pair_b read source item b - pair_b and use mode2 / weight2
  int pair_b, mode2, weight2;
  // inverse row passes: walk the items last to first (rev = 1), so that a pass
  // reading the previous row pass's output meets the most recently written
  // rows, the ones still in L2, first
  int rev;
};

// inverse row kernels: (source item, composite mode, input weighting) of batch item b
__device__ __forceinline__ void inv_item(const RowArgs& a, int b, int& img, int& mode, int& weight) {
  const bool h2 = a.pair_b > 0 && b >= a.pair_b;
  img = h2 ? b - a.pair_b : b;
  mode = h2 ? a.mode2 : a.mode;
  weight = h2 ? a.weight2 : a.weight;
}

// ---- small helpers ----------------------------------------------------------
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

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// ============================================================================
// Register-resident tile engine
// ============================================================================
template <typename T>
constexpr int tile_max_threads() { return 512; }
// developer A/B knobs (build.py SDCT_EXTRA_NVFLAGS); defaults are the measured best
#ifndef SDCT_COL_MAXT_F64
#define SDCT_COL_MAXT_F64 512
#endif
#ifndef SDCT_COL_FULLTW
#define SDCT_COL_FULLTW 0
#endif
#ifndef SDCT_ROW_FULLTW
#define SDCT_ROW_FULLTW 0
#endif
#ifndef SDCT_COL_XS
#define SDCT_COL_XS 1
#endif
#ifndef SDCT_COL_XS_INV
#define SDCT_COL_XS_INV 0
#endif

template <typename T, int L_, int NL_, bool LF, int MAXT_ = 0>
struct Tile {
  static constexpr int L = L_;
  static constexpr int NL = NL_;
  using P = RadixPlan<L>;
  using V = cx_t<T>;
  using Real = T;
  static constexpr int S = P::S;
  static constexpr int R0 = P::R(0);
  static constexpr int LGNL = ilog2c(NL);
  static constexpr int TOT = L * NL;
  static constexpr int NT0 = TOT / R0;
  // MAXT_ > 0: cap on the thread count (more elements per thread)
  static constexpr int MAXT = MAXT_ > 0 ? MAXT_ : (LF && sizeof(T) == 8) ? SDCT_COL_MAXT_F64 : tile_max_threads<T>();
  static constexpr int NT = NT0 > MAXT ? MAXT : NT0;
  static constexpr int E = TOT / NT;
  static constexpr unsigned MASK = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u);
  static constexpr bool TWF = LF && SDCT_COL_FULLTW;  // true: load all R-1 stage twiddles (no derived products)
  // barrier over the threads sharing this tile (whole CTA here; thread
  // groups with named barriers in the grouped row kernel)
  __device__ __forceinline__ static void sync() { __syncthreads(); }

  // unswizzled address of element (line, n)
  __host__ __device__ static constexpr int raw(int line, int n) { return LF ? (n << LGNL) + line : line * L + n; }
  __device__ __forceinline__ static int swz(int a) { return LF ? SwzCol<T>::f(a) : SwzRow<T>::f(a); }
  static constexpr int swzc(int a) { return LF ? SwzCol<T>::fc(a) : SwzRow<T>::fc(a); }
  // compile-time swizzled offset of element stride q at slot multiple r
  template <int s>
  static constexpr int off(int r) {
    return swzc(LF ? ((r * (P::span(s) / P::R(s))) << LGNL) : r * (P::span(s) / P::R(s)));
  }

  // butterfly bf of stage s -> (line, j, b)
  template <int s>
  __device__ __forceinline__ static void decode(int bf, int& line, int& j, int& b) {
    constexpr int Q = P::span(s) / P::R(s);
    constexpr int NB = L / P::span(s);
    if (LF) {
      line = bf & (NL - 1);
      const int rest = bf >> LGNL;
      j = rest & (Q - 1);
      b = rest >> ilog2c(Q);
    } else {
      j = bf & (Q - 1);
      const int rest = bf >> ilog2c(Q);
      b = rest & (NB - 1);
      line = rest >> ilog2c(NB);
    }
  }
  template <int s>
  __device__ __forceinline__ static int base(int bf) {
    int line, j, b;
    decode<s>(bf, line, j, b);
    return swz(raw(line, b * P::span(s) + j));
  }
};

// Twiddles of one stage for the thread's butterflies. A few powers W^{jk}
// (k in LOADK) are loaded ahead of the data they multiply (they depend only
// on the thread's fixed j), the rest are products of two loaded powers, so
// every factor stays within ~2 ulp and no recurrence chain exists.
template <int R>
struct TwPlan;
template <>
struct TwPlan<2> {
  static constexpr int NLD = 1;
  static constexpr int k(int i) { return 1; }
};
template <>
struct TwPlan<4> {
  static constexpr int NLD = 3;
  static constexpr int k(int i) { return i + 1; }
};
template <>
struct TwPlan<8> {
  static constexpr int NLD = 4;
  static constexpr int k(int i) { return i + 1; }  // 1,2,3,4
};
template <>
struct TwPlan<16> {
  static constexpr int NLD = 6;
  static constexpr int k(int i) { return i < 4 ? i + 1 : (i == 4 ? 8 : 12); }  // 1,2,3,4,8,12
};

template <class TL, int s>
struct StageTw {
  using P = typename TL::P;
  using V = typename TL::V;
  static constexpr int R = P::R(s), SPAN = P::span(s), Q = SPAN / R;
  static constexpr int NBF = TL::E / R;
  static constexpr bool ACTIVE = SPAN > R;
  static constexpr bool FULL = TL::TWF;
  static constexpr int NLD = ACTIVE ? (FULL ? R - 1 : TwPlan<R>::NLD) : 1;
  V w[NBF][NLD];

  __device__ __forceinline__ void load(const void* twt, int t) {
    if constexpr (ACTIVE) {
      const V* tw = static_cast<const V*>(twt);
#pragma unroll
      for (int i = 0; i < NBF; ++i) {
        int line, j, b;
        TL::template decode<s>(t + i * TL::NT, line, j, b);
#pragma unroll
        for (int l = 0; l < NLD; ++l) w[i][l] = __ldg(tw + ((FULL ? l + 1 : TwPlan<R>::k(l)) - 1) * Q + j);
      }
    }
  }
  // W^{jk} for butterfly i
  __device__ __forceinline__ V get(int i, int k) const {
    if constexpr (FULL) {
      return w[i][k - 1];
    } else if constexpr (R == 16) {
      if (k <= 4) return w[i][k - 1];
      if (k == 8) return w[i][4];
      if (k == 12) return w[i][5];
      const int hi = k & 12, lo = k & 3;  // k = hi + lo, lo in 1..3
      const V wh = hi == 4 ? w[i][3] : hi == 8 ? w[i][4] : w[i][5];
      return cmul(wh, w[i][lo - 1]);
    } else if constexpr (R == 8) {
      if (k <= 4) return w[i][k - 1];
      return cmul(w[i][3], w[i][k - 5]);
    } else {
      return w[i][k - 1];
    }
  }
};

template <class TL, int s, bool INV>
__device__ __forceinline__ void stage_compute(typename TL::V* v, const StageTw<TL, s>& tw) {
  using P = typename TL::P;
  constexpr int R = P::R(s), SPAN = P::span(s);
  constexpr int NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    dft_reg<typename TL::Real, R, INV>(v + i * R);
    if constexpr (SPAN > R) {
#pragma unroll
      for (int k = 1; k < R; ++k) {
        const auto w = tw.get(i, k);
        v[i * R + k] = INV ? cmulc(v[i * R + k], w) : cmul(v[i * R + k], w);
      }
    }
  }
}

template <class TL, int s>
__device__ __forceinline__ void to_smem(const typename TL::V* v, typename TL::V* sm, int t) {
  using P = typename TL::P;
  constexpr int R = P::R(s), NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    const int sb = TL::template base<s>(t + i * TL::NT);
#pragma unroll
    for (int r = 0; r < R; ++r) sm[sb ^ TL::template off<s>(r)] = v[i * R + r];
  }
}

template <class TL, int s>
__device__ __forceinline__ void from_smem(typename TL::V* v, const typename TL::V* sm, int t) {
  using P = typename TL::P;
  constexpr int R = P::R(s), NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    const int sb = TL::template base<s>(t + i * TL::NT);
#pragma unroll
    for (int r = 0; r < R; ++r) v[i * R + r] = sm[sb ^ TL::template off<s>(r)];
  }
}

template <class TL, bool INV, int s>
__device__ __forceinline__ void later_stages(typename TL::V* v, typename TL::V* sm, const TwSet& tw, int t) {
  if constexpr (s < TL::S) {
    StageTw<TL, s> w;
    w.load(tw.st[s], t);  // issued before the smem reads it overlaps
    from_smem<TL, s>(v, sm, t);
    stage_compute<TL, s, INV>(v, w);
    if constexpr (s + 1 < TL::S) {
      to_smem<TL, s>(v, sm, t);
      TL::sync();
    }
    later_stages<TL, INV, s + 1>(v, sm, tw, t);
  }
}

// All stages but the last one's butterflies: runs stages 0..S-2 and loads the
// last stage's operands from smem (returns with the smem free for reuse after
// a barrier). Used by persistent kernels to start the next tile's load early.
template <class TL, bool INV, int s>
__device__ __forceinline__ void stages_until_last(typename TL::V* v, typename TL::V* sm, const TwSet& tw, int t,
                                                  StageTw<TL, TL::S - 1>& wl) {
  if constexpr (s == TL::S - 1) {
    wl.load(tw.st[s], t);
    from_smem<TL, s>(v, sm, t);
  } else {
    StageTw<TL, s> w;
    w.load(tw.st[s], t);
    from_smem<TL, s>(v, sm, t);
    stage_compute<TL, s, INV>(v, w);
    to_smem<TL, s>(v, sm, t);
    TL::sync();
    stages_until_last<TL, INV, s + 1>(v, sm, tw, t, wl);
  }
}

// Full FFT of a tile whose stage-0 operands are already in v and whose
// stage-0 twiddles were prefetched into w0. On return v holds the last
// stage's outputs (slot n = b*R_last + r of the thread's last-stage butterflies).
template <class TL, bool INV>
__device__ __forceinline__ void fft_regs(typename TL::V* v, typename TL::V* sm, const TwSet& tw,
                                         const StageTw<TL, 0>& w0, int t) {
  stage_compute<TL, 0, INV>(v, w0);
  if constexpr (TL::S > 1) {
    to_smem<TL, 0>(v, sm, t);
    TL::sync();
    later_stages<TL, INV, 1>(v, sm, tw, t);
  }
}

// Last-stage butterfly i of thread t -> (line, slot base b*R_last)
template <class TL>
__device__ __forceinline__ void last_decode(int bf, int& line, int& b) {
  int j;
  TL::template decode<TL::S - 1>(bf, line, j, b);
}

// ---- intermediate row order ---------------------------------------------------
// The forward column FFT (DIF) leaves X(k) at slot n = digit_pos(k); its
// last-stage butterfly (line, b) holds slots b*R + r (R = last radix). It
// stores slot n at intermediate row sigma(n) = (n % R) * (L/R) + n / R, so
// lanes with consecutive b write consecutive rows (conflict-free staging,
// contiguous TMA boxes). The inverse column FFT (DIT, the transposed
// factorisation) reads its input in exactly that order. Row kernels address
// frequency k of an intermediate through srow(k) = sigma(digit_pos(k)).
__host__ __device__ inline int rt_last_radix(int L) {
  int lg = 0;
  while ((1 << lg) < L) ++lg;
  if (lg == 0) return 1;
  const int S = (lg + 3) / 4;
  return 1 << (lg / S + (S - 1 < lg % S ? 1 : 0));
}
__host__ __device__ inline int rt_srow(int k, int L) {
  const int n = rt_digit_pos(k, L);
  const int R = rt_last_radix(L);
  return (n % R) * (L / R) + n / R;
}

// ---- DIT engine (transpose of the DIF engine) --------------------------------
// DIF: B_0, T_0, B_1, ..., T_{S-2}, B_{S-1}, then digit reversal. Its transpose
// (the same DFT, the DFT matrix is symmetric) runs the stage groups in reverse:
// input placed by digit position, B_{S-1}, T_{S-2}, B_{S-2}, ..., T_0, B_0;
// outputs come out in natural order at the stage-0 slots j + r*Q0.
template <class TL, int s, bool INV>
__device__ __forceinline__ void dit_compute(typename TL::V* v, const StageTw<TL, s>& tw) {
  using P = typename TL::P;
  constexpr int R = P::R(s), SPAN = P::span(s);
  constexpr int NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    if constexpr (SPAN > R) {
#pragma unroll
      for (int k = 1; k < R; ++k) {
        const auto w = tw.get(i, k);
        v[i * R + k] = INV ? cmulc(v[i * R + k], w) : cmul(v[i * R + k], w);
      }
    }
    dft_reg<typename TL::Real, R, INV>(v + i * R);
  }
}

// DIT stages S-2 .. s (descending); operands of stage s+1 are in smem.
template <class TL, bool INV, int s>
__device__ __forceinline__ void dit_down(typename TL::V* v, typename TL::V* sm, const TwSet& tw, int t) {
  if constexpr (s >= 0) {
    StageTw<TL, s> w;
    w.load(tw.st[s], t);
    from_smem<TL, s>(v, sm, t);
    dit_compute<TL, s, INV>(v, w);
    if constexpr (s > 0) {
      to_smem<TL, s>(v, sm, t);
      TL::sync();
      dit_down<TL, INV, s - 1>(v, sm, tw, t);
    }
  }
}

// ---- half-size exchanges (column kernels of 4096 x 2 tiles) -------------------
// A stage-to-stage exchange normally needs the whole tile in shared memory.
// Here it runs in two rounds through a buffer of half the tile: in round
// `ROUND` every thread writes the 8 of its 16 outputs whose membership bit
// (raw bit HB xor raw bit LB of the element's unswizzled tile address) equals
// ROUND, and reads the 8 of its next-stage operands with that bit; so every
// thread always holds 16 values (no extra registers). HB is dropped from the
// address (xcpos), which is injective within a round because LB fixes it. The
// swizzle only touches bits 0..2, so bank behaviour per instruction is that of
// the full-tile pattern (conflict free). HB = 12, LB = 8: the CTA-wide
// exchange between the stride-256 and stride-16 stages of a 4096-point
// column (writers vary bit 12, readers bit 8). HB = 8, LB = 4: the warp-local
// exchange between the stride-16 and unit-stride stages (each warp owns one
// 256-row block: 4 KB of the buffer per warp, __syncwarp only).
template <int HB>
__device__ __forceinline__ int xcpos(int p) {
  return ((p >> (HB + 1)) << HB) | (p & ((1 << HB) - 1));
}
template <int HB, int LB>
constexpr int xmember(int p) {
  return ((p >> HB) ^ (p >> LB)) & 1;
}
template <class TL, int s, int HB, int LB, int ROUND>
__device__ __forceinline__ void xwrite(const typename TL::V* v, typename TL::V* X, int t) {
  using P = typename TL::P;
  constexpr int R = P::R(s), NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    const int sb = TL::template base<s>(t + i * TL::NT);
    if (xmember<HB, LB>(sb) == ROUND) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (xmember<HB, LB>(TL::template off<s>(r)) == 0) X[xcpos<HB>(sb ^ TL::template off<s>(r))] = v[i * R + r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (xmember<HB, LB>(TL::template off<s>(r)) == 1) X[xcpos<HB>(sb ^ TL::template off<s>(r))] = v[i * R + r];
    }
  }
}
template <class TL, int s, int HB, int LB, int ROUND>
__device__ __forceinline__ void xread(typename TL::V* v, const typename TL::V* X, int t) {
  using P = typename TL::P;
  constexpr int R = P::R(s), NBF = TL::E / R;
#pragma unroll
  for (int i = 0; i < NBF; ++i) {
    const int sb = TL::template base<s>(t + i * TL::NT);
    if (xmember<HB, LB>(sb) == ROUND) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (xmember<HB, LB>(TL::template off<s>(r)) == 0) v[i * R + r] = X[xcpos<HB>(sb ^ TL::template off<s>(r))];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (xmember<HB, LB>(TL::template off<s>(r)) == 1) v[i * R + r] = X[xcpos<HB>(sb ^ TL::template off<s>(r))];
    }
  }
}
// CTA-wide exchange stage sw -> stage sr through X (caller: X free, synced)
template <class TL, int sw, int sr>
__device__ __forceinline__ void xchg_cta(typename TL::V* v, typename TL::V* X, int t) {
  xwrite<TL, sw, 12, 8, 0>(v, X, t);
  __syncthreads();
  xread<TL, sr, 12, 8, 0>(v, X, t);
  __syncthreads();
  xwrite<TL, sw, 12, 8, 1>(v, X, t);
  __syncthreads();
  xread<TL, sr, 12, 8, 1>(v, X, t);
}
// warp-local exchange stage sw -> stage sr through X (caller: X free, synced)
template <class TL, int sw, int sr>
__device__ __forceinline__ void xchg_warp(typename TL::V* v, typename TL::V* X, int t) {
  xwrite<TL, sw, 8, 4, 0>(v, X, t);
  __syncwarp();
  xread<TL, sr, 8, 4, 0>(v, X, t);
  __syncwarp();
  xwrite<TL, sw, 8, 4, 1>(v, X, t);
  __syncwarp();
  xread<TL, sr, 8, 4, 1>(v, X, t);
}
// tiles that take the early-reissue schedule: 4096-point columns, 2-wide
// bands, 512 threads of 16 elements, three radix-16 stages
// (measured on B200, 4096^2: fp64 forward column pass 86 -> 80 us; the fp64
// inverse and both fp32 passes gain nothing, so they keep the in-tile schedule)
template <class TL, bool INV>
constexpr bool col_xs() {
  return (INV ? SDCT_COL_XS_INV : SDCT_COL_XS) && sizeof(typename TL::Real) == 8 && TL::L == 4096 && TL::NL == 2 && TL::NT == 512 && TL::S == 3 && TL::P::R(0) == 16 &&
         TL::P::R(1) == 16 && TL::P::R(2) == 16;
}

// ============================================================================
// Column kernel
// ============================================================================
// Persistent: CTA walks tiles blockIdx.x, +gridDim.x, ... A tile (band of NL
// complex columns x L rows) lands in smem by TMA; the FFT runs in registers
// with smem exchanges; results leave through a half-tile smem staging buffer
// and TMA stores (the bulk engine generates the 32-B row segments, not the
// LSU). The next tile's load is issued as soon as the current tile's last
// stage has read its operands, so it overlaps the last stage and the stores.
//   forward (DIF): LD_SRC (parity rows + packing) or LD_INTER (natural rows);
//                  output rows in sigma order (ST_INTER).
//   inverse (DIT): input rows in sigma order; output natural rows (ST_INTER)
//                  or the final gather to y (ST_DST: rows pe(i), 1/4 or 1/8,
//                  signs), stored as even / odd y-row classes.
// The body takes the CTA's rank and the CTA count so that a fused kernel
// (kernels_fused.cuh) can run it as its first phase.
template <typename T, int L, int NL, bool INV, int LOAD, int STORE>
__device__ __forceinline__ void col_body(const CUtensorMap& tin, const CUtensorMap& tout, const ColArgs& a,
                                         const TwSet& tw, const int cta, const int ncta) {
  using TL = Tile<T, L, NL, true>;
  using P = typename TL::P;
  using V = cx_t<T>;
  using V2 = typename Vec2<T>::type;
  constexpr int NT = TL::NT;
  constexpr int S = TL::S, SL = S - 1;
  constexpr int R0 = TL::R0, Q0 = L / R0, NBF0 = TL::E / R0;
  constexpr int RL = P::R(SL), NBFL = TL::E / RL;
  constexpr int BOXR = L < 256 ? L : 256;
  constexpr uint32_t TILE_BYTES = static_cast<uint32_t>(L) * 2 * NL * sizeof(T);
  constexpr uint32_t STG_OFF = (TILE_BYTES + 127u) & ~127u;                      // TMA needs 128-B aligned smem
  constexpr uint32_t BAR_OFF = (STG_OFF + TILE_BYTES / 2 + 127u) & ~127u;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  T* stg = reinterpret_cast<T*>(smem_raw + STG_OFF);  // half-tile staging [L/2][2*NL]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + BAR_OFF);
  const int t = threadIdx.x;

  // tile -> (band, plane, batch); power-of-two band / plane counts (every
  // fast-path shape) decode with shifts instead of integer divisions
  const bool pow2 = ((a.nbands & (a.nbands - 1)) | (a.nplanes & (a.nplanes - 1))) == 0;
  const int sb_ = __ffs(a.nbands) - 1, sp_ = __ffs(a.nplanes) - 1;
  auto coords = [&](int tile, int& band, int& plane, int& batch) {
    if (pow2) {
      band = tile & (a.nbands - 1);
      const int rest = tile >> sb_;
      plane = rest & (a.nplanes - 1);
      batch = rest >> sp_;
      return;
    }
    band = tile % a.nbands;
    const int rest = tile / a.nbands;
    plane = rest % a.nplanes;
    batch = rest / a.nplanes;
  };
  auto issue = [&](int tile) {  // thread 0 only
    int band, plane, batch;
    coords(tile, band, plane, batch);
    const int pc = a.tma_plane_par ? parity_embed(plane, a.tma_plane_par) : plane;
    mbar_expect_tx(bar, TILE_BYTES);
    if constexpr (LOAD == LD_SRC && col_class_load(sizeof(T), L, NL)) {
      // source rows by parity class through the {reals, class, pair, plane,
      // batch} map: even rows 2p land at smem row p, odd rows 2p+1 at L/2 + p,
      // so the parity gather below reads consecutive rows (conflict-free)
      constexpr int HALFR = L / 2, BOXP = HALFR < 256 ? HALFR : 256;
#pragma unroll 1
      for (int cls = 0; cls < 2; ++cls)
#pragma unroll 1
        for (int p0 = 0; p0 < HALFR; p0 += BOXP)
          tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(cls * HALFR + p0) * 2 * NL, &tin,
                      band * 2 * NL, cls, p0, pc, batch, bar);
    } else {
#pragma unroll 1
      for (int r0 = 0; r0 < L; r0 += BOXR)
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL, &tin, band * 2 * NL, r0, pc,
                    batch, bar);
    }
  };
  if (t == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
    mbar_init(bar, 1);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // the previous kernel's output is complete before the first load
  if (t == 0 && static_cast<int>(cta) < a.ntiles) issue(cta);

  uint32_t phase = 0;
  for (int tile = cta; tile < a.ntiles; tile += ncta) {
    int band, plane, batch;
    coords(tile, band, plane, batch);
    V v[TL::E];
    unsigned long long tr0 = 0, tr1 = 0, tr2 = 0, tr3 = 0, tr4 = 0, tr5 = 0;
    if (a.trace && t == 0) tr0 = gtimer();

    if constexpr (!INV) {
      // =================== forward: DIF ===================
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);  // latency hidden under the tile load
      mbar_wait(bar, phase);
      phase ^= 1;
      if (a.trace && t == 0) tr1 = gtimer();
      if constexpr (LOAD == LD_SRC) {
        // slot n reads source row pe(n) (landed by parity class); line 2g+h is z(u) (h=0) or z(M-1-u)
        // (h=1) of source quad g: lanes h=0/1 read the halves, swap one real
        const V2* raw = reinterpret_cast<const V2*>(smem_raw);
#pragma unroll
        for (int i = 0; i < NBF0; ++i) {
          const int bf = t + i * NT;
          const int line = bf & (NL - 1), j = bf >> TL::LGNL;
          const int h = line & 1;
#pragma unroll
          for (int r = 0; r < R0; ++r) {
            const int n = j + r * Q0;
            // source row pe(n) = 2n or 2(L-1-n)+1; landed by class: smem row n / L/2 + L-1-n
            const int row = col_class_load(sizeof(T), L, NL) ? ((r < R0 / 2) ? n : L / 2 + (L - 1 - n))
                                                             : ((r < R0 / 2) ? 2 * n : 2 * L - 1 - 2 * n);
            const V2 x = raw[row * NL + line];
            const T send = h ? x.x : x.y;
            const T recv = __shfl_xor_sync(TL::MASK, send, 1);
            v[i * R0 + r] = h ? mk(x.y, recv) : mk(x.x, recv);
          }
        }
      } else {
        const V* raw = reinterpret_cast<const V*>(smem_raw);
#pragma unroll
        for (int i = 0; i < NBF0; ++i) {
          const int bf = t + i * NT;
          const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
          for (int r = 0; r < R0; ++r) v[i * R0 + r] = raw[(j + r * Q0) * NL + line];
        }
      }
      __syncthreads();  // raw tile consumed; smem becomes the exchange buffer
      if constexpr (col_xs<TL, false>()) {
        // early reissue: the landing buffer is free now, so the next tile
        // streams in under this tile's whole FFT; the exchanges run through
        // the half-tile staging buffer X in balanced rounds
        if (a.trace && t == 0) tr2 = gtimer();
        if (t == 0 && tile + static_cast<int>(ncta) < a.ntiles) {
          fence_async_smem();
          issue(tile + ncta);
        }
        V* X = reinterpret_cast<V*>(stg);
        StageTw<TL, 1> w1;
        w1.load(tw.st[1], t);
        stage_compute<TL, 0, false>(v, w0);
        if (t == 0) bulk_wait_read();  // the previous tile's stores have left X
        __syncthreads();
        xchg_cta<TL, 0, 1>(v, X, t);
        if (a.trace && t == 0) tr3 = gtimer();
        stage_compute<TL, 1, false>(v, w1);
        __syncthreads();  // CTA-wide reads of X done before the warp-local writes
        xchg_warp<TL, 1, 2>(v, X, t);
        if (a.trace && t == 0) tr4 = gtimer();
        StageTw<TL, 2> w2;  // inactive (span == radix): no twiddles
        stage_compute<TL, 2, false>(v, w2);
        if (a.trace && t == 0) tr5 = gtimer();
      } else {
        StageTw<TL, SL> wl;
        if constexpr (S == 1) {
          wl = w0;
        } else {
          stage_compute<TL, 0, false>(v, w0);
          to_smem<TL, 0>(v, sm, t);
          __syncthreads();
          stages_until_last<TL, false, 1>(v, sm, tw, t, wl);
        }
        __syncthreads();  // last-stage operands are in registers: smem is free
        if (a.trace && t == 0) tr2 = gtimer();
        if (t == 0 && tile + static_cast<int>(ncta) < a.ntiles) {
          fence_async_smem();
          issue(tile + ncta);
        }
        stage_compute<TL, SL, false>(v, wl);
      }
      // ---- store: slot n = b*RL + r -> row sigma(n) = b + (L/RL)*r ----
      // PL parts of L/PL rows; with four parts the staging holds two
      // quarter buffers, so writing part q overlaps the TMA read of part q-1
      // (L >= 4096 only: measured neutral-to-worse on smaller tiles)
      constexpr int PL = (RL >= 4 && L >= 4096) ? 4 : 2, NSB = PL == 4 ? 2 : 1, PSL = L / PL, BOXQ = PSL < 256 ? PSL : 256;
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        if (t == 0) {
          if constexpr (NSB == 2) bulk_wait_read_1();  // this buffer's previous part read
          else bulk_wait_read();
        }
        __syncthreads();
        T* sb = stg + static_cast<size_t>(q % NSB) * PSL * 2 * NL;
        V* sv = reinterpret_cast<V*>(sb);
#pragma unroll
        for (int i = 0; i < NBFL; ++i) {
          int line, b;
          last_decode<TL>(t + i * NT, line, b);
#pragma unroll
          for (int r = q * (RL / PL); r < (q + 1) * (RL / PL); ++r)
            sv[(b + (L / RL) * (r - q * (RL / PL))) * NL + line] = v[i * RL + r];
        }
        fence_async_smem();
        __syncthreads();
        if (t == 0) {
#pragma unroll 1
          for (int r0 = 0; r0 < PSL; r0 += BOXQ)
            tma_store_4d(&tout, band * 2 * NL, q * PSL + r0, plane, batch, sb + static_cast<size_t>(r0) * 2 * NL);
          bulk_commit();
        }
      }
    } else {
      // =================== inverse: DIT ===================
      StageTw<TL, SL> wl;  // first DIT stage (S-1) has no twiddles
      mbar_wait(bar, phase);
      phase ^= 1;
      if (a.trace && t == 0) tr1 = gtimer();
      {
        // stage S-1 operands: slot b*RL + r lives in storage row sigma = b + (L/RL) r
        const V* raw = reinterpret_cast<const V*>(smem_raw);
#pragma unroll
        for (int i = 0; i < NBFL; ++i) {
          int line, b;
          last_decode<TL>(t + i * NT, line, b);
#pragma unroll
          for (int r = 0; r < RL; ++r) v[i * RL + r] = raw[(b + (L / RL) * r) * NL + line];
        }
      }
      __syncthreads();  // raw tile consumed
      if constexpr (col_xs<TL, true>()) {
        // early reissue (see the forward): exchanges through X in rounds
        if (a.trace && t == 0) tr2 = gtimer();
        if (t == 0 && tile + static_cast<int>(ncta) < a.ntiles) {
          fence_async_smem();
          issue(tile + ncta);
        }
        V* X = reinterpret_cast<V*>(stg);
        StageTw<TL, 1> w1;
        w1.load(tw.st[1], t);
        dit_compute<TL, 2, true>(v, wl);
        if (t == 0) bulk_wait_read();  // the previous tile's stores have left X
        __syncthreads();
        xchg_warp<TL, 2, 1>(v, X, t);
        dit_compute<TL, 1, true>(v, w1);
        StageTw<TL, 0> w0;
        w0.load(tw.st[0], t);
        __syncthreads();  // warp-local reads of X done before the CTA-wide writes
        xchg_cta<TL, 1, 0>(v, X, t);
        dit_compute<TL, 0, true>(v, w0);
      } else {
        dit_compute<TL, SL, true>(v, wl);
        if constexpr (S > 1) {
          to_smem<TL, SL>(v, sm, t);
          __syncthreads();
          dit_down<TL, true, SL - 1>(v, sm, tw, t);  // ends with stage 0 in registers
        }
        __syncthreads();  // all smem reads done
        if (a.trace && t == 0) tr2 = gtimer();
        if (t == 0 && tile + static_cast<int>(ncta) < a.ntiles) {
          fence_async_smem();
          issue(tile + ncta);
        }
      }
      // outputs: stage-0 butterfly (line, j) holds natural index ii = j + r*Q0
      // PI parts of L/PI rows (two quarter buffers when PI == 4, see the forward)
      constexpr int PI = (R0 >= 4 && L >= 4096) ? 4 : 2, NSB = PI == 4 ? 2 : 1, PSI = L / PI, BOXQ = PSI < 256 ? PSI : 256;
      if constexpr (STORE == ST_INTER) {
#pragma unroll
        for (int q = 0; q < PI; ++q) {
          if (t == 0) {
            if constexpr (NSB == 2) bulk_wait_read_1();
            else bulk_wait_read();
          }
          __syncthreads();
          T* sb = stg + static_cast<size_t>(q % NSB) * PSI * 2 * NL;
          V* sv = reinterpret_cast<V*>(sb);
#pragma unroll
          for (int i = 0; i < NBF0; ++i) {
            const int bf = t + i * NT;
            const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
            for (int r = q * (R0 / PI); r < (q + 1) * (R0 / PI); ++r)
              sv[(j + (r - q * (R0 / PI)) * Q0) * NL + line] = v[i * R0 + r];
          }
          fence_async_smem();
          __syncthreads();
          if (t == 0) {
#pragma unroll 1
            for (int r0 = 0; r0 < PSI; r0 += BOXQ)
              tma_store_4d(&tout, band * 2 * NL, q * PSI + r0, plane, batch, sb + static_cast<size_t>(r0) * 2 * NL);
            bulk_commit();
          }
        }
      } else {
        // final gather: y row pe(ii): even rows 2ii (ii < L/2) and odd rows
        // 2L-1-2ii (ii >= L/2), staged per class and stored through a 5D map
        // {reals, row class, row pair, planes, batch}
        const T sc = static_cast<T>(a.scale);
        const bool h2_ = a.pair_b > 0 && batch >= a.pair_b;
        const int srow_ = h2_ ? a.sign_row2 : a.sign_row, scol_ = h2_ ? a.sign_col2 : a.sign_col;
        int pl = plane;
        if (a.out_plane_map == 1) pl = parity_embed(plane, a.out_plane_n);
        // part q holds ii in [q L/PI, (q+1) L/PI): class q / (PI/2) (even rows
        // 2ii, then odd rows 2L-1-2ii), row pairs from pbase
#pragma unroll
        for (int q = 0; q < PI; ++q) {
          const int half = q / (PI / 2);
          const int pbase = half == 0 ? q * PSI : L - (q + 1) * PSI;  // first row pair of the part
          if (t == 0) {
            if constexpr (NSB == 2) bulk_wait_read_1();
            else bulk_wait_read();
          }
          __syncthreads();
          T* sb = stg + static_cast<size_t>(q % NSB) * PSI * 2 * NL;
          V2* sv = reinterpret_cast<V2*>(sb);
#pragma unroll
          for (int i = 0; i < NBF0; ++i) {
            const int bf = t + i * NT;
            const int line = bf & (NL - 1), j = bf >> TL::LGNL;
            const int h = line & 1;
#pragma unroll
            for (int r = q * (R0 / PI); r < (q + 1) * (R0 / PI); ++r) {
              const int ii = j + r * Q0;
              const int k1 = half == 0 ? 2 * ii : 2 * L - 1 - 2 * ii;  // pe(ii)
              const int srow = (half == 0 ? ii : L - 1 - ii) - pbase;   // pair index within the part
              const V z = v[i * R0 + r];
              const T recv = __shfl_xor_sync(TL::MASK, z.y, 1);
              const T s0 = (srow_ && (k1 & 1)) ? -sc : sc;
              const T s1 = scol_ ? -s0 : s0;
              // h=0: (Re z(u), Im z(M-1-u)) = y(4u, 4u+1); h=1: (Im z(u), Re z(M-1-u)) = y(4u+2, 4u+3)
              sv[srow * NL + line] = h ? V2{recv * s0, z.x * s1} : V2{z.x * s0, recv * s1};
            }
          }
          fence_async_smem();
          __syncthreads();
          if (t == 0) {
#pragma unroll 1
            for (int r0 = 0; r0 < PSI; r0 += BOXQ)
              tma_store_5d(&tout, band * 2 * NL, half, pbase + r0, pl, batch, sb + static_cast<size_t>(r0) * 2 * NL);
            bulk_commit();
          }
        }
      }
    }
    if (a.trace && t == 0) {
      // 8 values per tile: loop start, tile landed, next load issued, [early-
      // reissue schedule: CTA-wide exchange done, warp exchange done, last stage
      // done], stores issued, CTA id
      unsigned long long* o = a.trace + 8 * static_cast<long long>(tile);
      o[0] = tr0;
      o[1] = tr1;
      o[2] = tr2;
      o[3] = tr3;
      o[4] = tr4;
      o[5] = tr5;
      o[6] = gtimer();
      o[7] = cta;
    }
  }
  if (t == 0) bulk_wait_all();  // stores complete before the CTA retires
}

template <typename T, int L, int NL, bool INV, int LOAD, int STORE>
__global__ void __launch_bounds__(Tile<T, L, NL, true>::NT)
    col_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ColArgs a,
               TwSet tw) {
  col_body<T, L, NL, INV, LOAD, STORE>(tin, tout, a, tw, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
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

template <typename T, int M, int G>
using RowTile = Tile<T, M, G, false>;

// 3D inverse row kernel: operand rows staged behind the tile when both fit
template <typename T, int M>
constexpr bool row3_staged() {
  return 2 * 4 * M * sizeof(cx_t<T>) + 16 <= 200 * 1024;
}

template <typename T, int M, int KIND>
constexpr int row_threads() {
  return RowTile<T, M, (KIND == RK_FWD2 || KIND == RK_INV2) ? 2 : 4>::NT;
}

// Natural-order smem index of (line, m) in a row tile.
template <typename T, int M>
__device__ __forceinline__ int row_nat(int line, int m) {
  return SwzRow<T>::f(line * M + m);
}

// Writes the last stage's results (in registers) at natural (frequency/
// spatial) order: slot n = b*R + r holds index digit_rev(n) = kb + r*(M/R).
template <class TL>
__device__ __forceinline__ void last_to_natural(const typename TL::V* v, typename TL::V* sm, int t) {
  using P = typename TL::P;
  constexpr int RL = P::R(TL::S - 1), NBFL = TL::E / RL, M = TL::L;
#pragma unroll
  for (int i = 0; i < NBFL; ++i) {
    int line, b;
    last_decode<TL>(t + i * TL::NT, line, b);
    const int sb = TL::swz(line * M + digit_rev<M>(b * RL));
#pragma unroll
    for (int r = 0; r < RL; ++r) sm[sb ^ TL::swzc(r * (M / RL))] = v[i * RL + r];
  }
}

template <typename T, int M, int KIND>
__global__ void __launch_bounds__(row_threads<T, M, KIND>())
    row_kernel(RowArgs a, TwSet tw) {
  using V = cx_t<T>;
  using V4 = typename Cx<T>::vec4;
  constexpr int G = (KIND == RK_FWD2 || KIND == RK_INV2) ? 2 : 4;
  constexpr bool INV = (KIND == RK_INV2 || KIND == RK_INV3);
  using TL = RowTile<T, M, G>;
  constexpr int NT = TL::NT;
  constexpr int R0 = TL::R0, Q0 = M / R0, NBF0 = TL::E / R0;
  constexpr int CPV = 16 / sizeof(V);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  const int t = threadIdx.x;
  const int P = blockIdx.x, batch = blockIdx.y;
  const int n1 = a.n1, n2 = a.n2;
  pdl_trigger();
  pdl_wait();  // the previous kernel's output is complete before any buffer access

  // frequency rows of this group, their storage rows in the intermediate
  // (srow = sigma(digit_pos), the column FFTs' order), and degeneracy
  int rows[G], irow[G];
  bool deg1 = false, deg2 = false;
  int q1 = 0, q2 = 0, m1 = 0, m2 = 0;
  if constexpr (G == 2) {
    q1 = P;
    m1 = P == 0 ? n1 / 2 : n1 - P;
    rows[0] = q1;
    rows[1] = m1;
    irow[0] = __ldg(a.s0 + q1);
    irow[1] = __ldg(a.s0 + m1);
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
    const int p1q = __ldg(a.s0 + q1), p1m = __ldg(a.s0 + m1);
    const int p2q = __ldg(a.s1 + q2), p2m = __ldg(a.s1 + m2);
    irow[0] = p1q * n2 + p2q;
    irow[1] = p1m * n2 + p2q;
    irow[2] = p1q * n2 + p2m;
    irow[3] = p1m * n2 + p2m;
  }

  V v[TL::E];
  // 3D forward: the postprocess's a(k1) b(k2) table values, issued before the
  // row landing they overlap
  V av3{}, bv3{};
  if constexpr (KIND == RK_FWD3) {
    av3 = __ldg(static_cast<const V*>(a.ta) + q1);
    bv3 = __ldg(static_cast<const V*>(a.tb) + q2);
  }
  if constexpr (!INV) {
    // ---- forward: the G rows land in smem by 1D bulk copies ----------------
    StageTw<TL, 0> w0;
    w0.load(tw.st[0], t);
    {
      uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G * M);  // after the tile
      if (t == 0) mbar_init(bar, 1);
      __syncthreads();
      if (t == 0) {
        const V* src = static_cast<const V*>(a.src) + batch * a.src_batch;
        mbar_expect_tx(bar, static_cast<uint32_t>(G * M * sizeof(V)));
#pragma unroll
        for (int l = 0; l < G; ++l)
          bulk_load(sm + l * M, src + static_cast<long long>(irow[l]) * M, static_cast<uint32_t>(M * sizeof(V)), bar);
      }
      mbar_wait(bar, 0);
    }
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      int line, j, b;
      TL::template decode<0>(t + i * NT, line, j, b);
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        const int s = (r < R0 / 2) ? 2 * n : 2 * M - 1 - 2 * n;  // pair-interleaved column of z(n)
        v[i * R0 + r] = sm[line * M + s];
      }
    }
    __syncthreads();  // raw rows consumed; smem becomes the exchange buffer
    fft_regs<TL, false>(v, sm, tw, w0, t);
    __syncthreads();  // last-stage smem reads done before natural-order writes
    last_to_natural<TL>(v, sm, t);
    __syncthreads();
  } else {
    // ---- inverse: merged preprocess + packing into smem (natural order) ----
    const T* x = static_cast<const T*>(a.src) + batch * a.src_batch;
    const V* tu = static_cast<const V*>(a.tu);
    if constexpr (KIND == RK_INV2) {
      // Rows q1 and m1 land in smem by bulk copy (2 x N2 reals = the tile's
      // size); the merged preprocess then reads its operands from smem into
      // registers, synchronises, and overwrites the same smem with the packed
      // spectrum (natural order).
      constexpr int NI = (M / 2) / NT + 1;  // items k in [0, M/2] per thread
      T* rowA = reinterpret_cast<T*>(smem_raw);
      T* rowB = rowA + 2 * M;
      {
        uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G * M);
        if (t == 0) mbar_init(bar, 1);
        __syncthreads();
        if (t == 0) {
          const uint32_t rb = static_cast<uint32_t>(n2 * sizeof(T));
          mbar_expect_tx(bar, 2 * rb);
          bulk_load(rowA, x + static_cast<long long>(q1) * n2, rb, bar);
          bulk_load(rowB, x + static_cast<long long>(m1) * n2, rb, bar);
        }
        mbar_wait(bar, 0);
      }
      // operands: for n2 in {k, M-k}: D(n2) and R(n2) of both rows, where
      // D = x(n2), R = x(N2-n2) (x(N2) := 0); mode 2 (IDXST along axis 1)
      // reads x(N2-n2) for D and x(n2) for R with x(0) := 0.
      T op[NI][8];
#pragma unroll
      for (int it = 0; it < NI; ++it) {
        const int k = t + it * NT;
        if (k <= M / 2) {
          const int ks[2] = {k, M - k};
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int nn = ks[u];
            const bool z = nn == 0;
            const int pd = a.mode == 2 ? n2 - nn : nn;
            const int pr = a.mode == 2 ? nn : n2 - nn;
            const bool zd = a.mode == 2 && z, zr = z;
            op[it][4 * u + 0] = zd ? T(0) : rowA[pd & (n2 - 1)];
            op[it][4 * u + 1] = zr ? T(0) : rowA[pr & (n2 - 1)];
            op[it][4 * u + 2] = zd ? T(0) : rowB[pd & (n2 - 1)];
            op[it][4 * u + 3] = zr ? T(0) : rowB[pr & (n2 - 1)];
          }
        }
      }
      const V* ta = static_cast<const V*>(a.ta);
      const V* tb = static_cast<const V*>(a.tb);
      const V ca0 = cconj(__ldg(ta + q1)), ca1 = cconj(__ldg(ta + m1));
      __syncthreads();  // all operands read: smem becomes the packed spectrum
      // X'(line, n2) from the operands (proj/src/dct2d.cpp:182-195)
      auto xp = [&](const T* o, V cb, V& x0, V& x1) {
        // o = {DA, RA, DB, RB}; p,s from the q1 row, r,q from the m1 row
        T p = o[0], sv = o[1], r = o[2], q = o[3];
        if (a.mode == 1) {  // IDXST along axis 0 swaps the row roles
          p = o[2];
          sv = o[3];
          r = o[0];
          q = o[1];
        }
        if (P == 0) {
          // rows 0 and N1/2, each its own mirror: row 0 pairs with the zero
          // row N1; mode 1 zeroes row 0 entirely
          const T pa = a.mode == 1 ? T(0) : o[0], sa = a.mode == 1 ? T(0) : o[1];
          x0 = cmul(cmul(ca0, cb), mk(pa, -sa));                 // p = pa, q = r = 0, s = sa
          x1 = cmul(cmul(ca1, cb), mk(o[2] - o[3], -(o[2] + o[3])));  // p = r = DB, q = s = RB
          return;
        }
        x0 = cmul(cmul(ca0, cb), mk(p - q, -(r + sv)));
        x1 = cmul(cmul(ca1, cb), mk(r - sv, -(p + q)));
      };
#pragma unroll
      for (int it = 0; it < NI; ++it) {
        const int k = t + it * NT;
        if (k <= M / 2) {
          const V bk = __ldg(tb + k), bm = __ldg(tb + (M - k));
          V A0, A1, B0, B1;  // X'(line, k), X'(line, M-k)
          xp(&op[it][0], cconj(bk), A0, A1);
          xp(&op[it][4], cconj(bm), B0, B1);
          // partner line of each row (-k1): swap for pairs, self for P == 0
          const V pA0 = P != 0 ? A1 : A0, pA1 = P != 0 ? A0 : A1;
          const V pB0 = P != 0 ? B1 : B0, pB1 = P != 0 ? B0 : B1;
          const V bk2 = cmul(bk, bk), bm2 = cmul(bm, bm);
          const V wk = cmul(bk2, bk2), wmk = cmul(bm2, bm2);  // W_N2^k = b(k)^4
          sm[row_nat<T, M>(0, k & (M - 1))] = pack(A0, k == 0 ? B0 : cconj(pB0), wk);
          sm[row_nat<T, M>(1, k & (M - 1))] = pack(A1, k == 0 ? B1 : cconj(pB1), wk);
          if (k != 0 && 2 * k != M) {
            sm[row_nat<T, M>(0, M - k)] = pack(B0, cconj(pA0), wmk);
            sm[row_nat<T, M>(1, M - k)] = pack(B1, cconj(pA1), wmk);
          }
        }
      }
    } else if constexpr (row3_staged<T, M>()) {  // RK_INV3, operand rows staged in smem
      // Every operand of the literal 3D preprocess (transforms_ext.cpp:196-212)
      // for the group's four lines lies in the rows x(i, j, .) with i in
      // {q1, m1}, j in {q2, m2} (index N reads 0): bulk-load those four rows
      // behind the tile, then read them from smem.
      const int li[4] = {q1, m1, q1, m1}, lj[4] = {q2, q2, m2, m2};
      const int n3 = a.n3;
      T* rows = reinterpret_cast<T*>(smem_raw + G * M * sizeof(V));
      {
        uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 2 * G * M * sizeof(V));
        if (t == 0) mbar_init(bar, 1);
        __syncthreads();
        if (t == 0) {
          const uint32_t rb = static_cast<uint32_t>(n3 * sizeof(T));
          mbar_expect_tx(bar, 4 * rb);
#pragma unroll
          for (int l = 0; l < 4; ++l)
            bulk_load(rows + l * n3, x + (static_cast<long long>(li[l]) * a.n2 + lj[l]) * n3, rb, bar);
        }
        mbar_wait(bar, 0);
      }
      // x(i, j, k) for i in {q1, m1, n1}, j in {q2, m2, n2}, k in [0, n3]
      auto xv = [&](int i, int j, int k) -> T {
        if (i == n1 || j == n2 || k == n3) return T(0);
        return rows[((i == q1 ? 0 : 1) + (j == q2 ? 0 : 2)) * n3 + k];
      };
      // per-line constant conj(a(i) b(j)); per-k conj(c(k)) shared by the lines
      V cab[4];
#pragma unroll
      for (int l = 0; l < 4; ++l)
        cab[l] = cconj(cmul(__ldg(static_cast<const V*>(a.ta) + li[l]), __ldg(static_cast<const V*>(a.tb) + lj[l])));
      const V* tc = static_cast<const V*>(a.tc);
      auto entry = [&](int l, int k, V cc) -> V {
        const int i = li[l], j = lj[l];
        const int r1 = n1 - i, r2 = n2 - j, r3 = n3 - k;
        const T re = (xv(i, j, k) - xv(r1, r2, k)) - (xv(r1, j, r3) + xv(i, r2, r3));
        const T im = xv(r1, r2, r3) - ((xv(r1, j, k) + xv(i, r2, k)) + xv(i, j, r3));
        return cmul(cmul(cab[l], cc), mk(re, im));
      };
      for (int k = t; k <= M / 2; k += NT) {
        V A[4], B[4];
        const V ck = cconj(__ldg(tc + k)), cm = cconj(__ldg(tc + (M - k)));
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          A[l] = entry(l, k, ck);
          B[l] = entry(l, M - k, cm);
        }
        const V wk = __ldg(tu + k);
#pragma unroll
        for (int l = 0; l < 4; ++l)
          sm[row_nat<T, M>(l, k & (M - 1))] = pack(A[l], k == 0 ? B[l] : cconj(B[3 - l]), wk);
        if (k != 0 && 2 * k != M) {
          const V wmk = __ldg(tu + (M - k));
#pragma unroll
          for (int l = 0; l < 4; ++l) sm[row_nat<T, M>(l, M - k)] = pack(B[l], cconj(A[3 - l]), wmk);
        }
      }
    } else {  // RK_INV3
      const int li[4] = {q1, m1, q1, m1}, lj[4] = {q2, q2, m2, m2};
      for (int k = t; k <= M / 2; k += NT) {
        V A[4], B[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          A[l] = pre3_entry(x, li[l], lj[l], k, a);
          B[l] = pre3_entry(x, li[l], lj[l], M - k, a);
        }
        const V wk = __ldg(tu + k);
#pragma unroll
        for (int l = 0; l < 4; ++l)
          sm[row_nat<T, M>(l, k & (M - 1))] = pack(A[l], k == 0 ? B[l] : cconj(B[3 - l]), wk);
        if (k != 0 && 2 * k != M) {
          const V wmk = __ldg(tu + (M - k));
#pragma unroll
          for (int l = 0; l < 4; ++l) sm[row_nat<T, M>(l, M - k)] = pack(B[l], cconj(A[3 - l]), wmk);
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
    // ---- store rows (natural row order) in pair-interleaved column order ---
    V* dst = static_cast<V*>(a.dst) + batch * a.dst_batch;
    constexpr int VPR = M / CPV;
    for (int w = t; w < G * VPR; w += NT) {
      const int line = w / VPR, ci = w - line * VPR;
      if (G == 4 && ((line == 1 && deg1) || (line == 2 && deg2) || (line == 3 && (deg1 || deg2))))
        continue;
      V4 o;
      V* e = reinterpret_cast<V*>(&o);
#pragma unroll
      for (int k = 0; k < CPV; ++k) e[k] = sm[row_nat<T, M>(line, s_to_m(ci * CPV + k, M))];
      *reinterpret_cast<V4*>(dst + static_cast<long long>(irow[line]) * M + ci * CPV) = o;
    }
    return;
  }

  // ---- forward postprocess from natural-order smem -------------------------
  if constexpr (KIND == RK_FWD2) {
    // merged DCT postprocess (proj/src/dct2d.cpp:93-113) on the unpacked
    // rows. Items q2 and M-q2 read the same four spectrum values, so one
    // thread handles the pair: 4 smem reads -> up to 8 outputs.
    T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
    const V* ta = static_cast<const V*>(a.ta);
    const V* tb = static_cast<const V*>(a.tb);
    const V* tu = static_cast<const V*>(a.tu);
    T* r0 = y + static_cast<long long>(q1) * n2;
    T* r1 = y + static_cast<long long>(m1) * n2;
    const V av0 = __ldg(ta + q1), av1 = __ldg(ta + m1);
    auto item = [&](int q, V Z0a, V Z0b, V Z1a, V Z1b) {
      // Z0a = Z(k1, q), Z0b = Z(k1, -q), Z1a = Z(k1', q), Z1b = Z(k1', -q)
      const V w = __ldg(tu + q), b = __ldg(tb + q);
      const bool deg2k = (q == 0) || (q == M);
      if (P != 0) {
        const V X1 = unpack(Z0a, cconj(Z1b), w);
        const V X2 = unpack(Z1a, cconj(Z0b), w);
        const V ax1 = cmul(av0, X1), ax2 = cmulc(X2, av0);
        const V sv = cmul(b, cadd(ax1, ax2)), tv = cmul(b, csub(ax1, ax2));
        r0[q] = T(0.5) * sv.x;
        r1[q] = T(-0.5) * tv.y;
        if (!deg2k) {
          r0[n2 - q] = T(-0.5) * sv.y;
          r1[n2 - q] = T(-0.5) * tv.x;
        }
      } else {
        const V X0 = unpack(Z0a, cconj(Z0b), w);
        const V X1 = unpack(Z1a, cconj(Z1b), w);
        const V s0 = cmul(b, cadd(cmul(av0, X0), cmulc(X0, av0)));
        const V s1 = cmul(b, cadd(cmul(av1, X1), cmulc(X1, av1)));
        r0[q] = T(0.5) * s0.x;
        r1[q] = T(0.5) * s1.x;
        if (!deg2k) {
          r0[n2 - q] = T(-0.5) * s0.y;
          r1[n2 - q] = T(-0.5) * s1.y;
        }
      }
    };
    for (int k2 = t; k2 <= M / 2; k2 += NT) {
      const int kb = (M - k2) & (M - 1);
      const V Z0a = sm[row_nat<T, M>(0, k2)], Z0b = sm[row_nat<T, M>(0, kb)];
      const V Z1a = sm[row_nat<T, M>(1, k2)], Z1b = sm[row_nat<T, M>(1, kb)];
      item(k2, Z0a, Z0b, Z1a, Z1b);
      if (2 * k2 != M) item(M - k2, Z0b, Z0a, Z1b, Z1a);
    }
  } else {  // RK_FWD3: merged 3D postprocess (proj/src/transforms_ext.cpp:117-157)
    T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
    const int n3 = a.n3;
    const V* tu = static_cast<const V*>(a.tu);
    const V ab = cmul(av3, bv3), cb = cmulc(bv3, av3);  // a b, conj(a) b
    // the four output rows (k1, k2) of this group: base pointers once per CTA
    T* const yqq = y + (static_cast<long long>(q1) * n2 + q2) * n3;
    T* const yqm = y + (static_cast<long long>(q1) * n2 + m2) * n3;
    T* const ymq = y + (static_cast<long long>(m1) * n2 + q2) * n3;
    T* const ymm = y + (static_cast<long long>(m1) * n2 + m2) * n3;

    auto item = [&](int k3, const V* Za, const V* Zb) {
      // Za[l] = Z(line l, k3), Zb[l] = Z(line l, -k3)
      const V w = __ldg(tu + k3);
      V X[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) X[l] = unpack(Za[l], cconj(Zb[3 - l]), w);
      const bool deg3 = (k3 == 0) || (k3 == M);
      const int m3 = n3 - k3;
      const V f1 = X[0];
      const V f2 = deg1 ? f1 : X[1];
      const V f3 = deg2 ? f1 : X[2];
      const V f4 = deg1 ? f3 : (deg2 ? f2 : X[3]);
      V c = __ldg(static_cast<const V*>(a.tc) + k3);  // times the 1/4 of the outputs
      c = mk(T(0.25) * c.x, T(0.25) * c.y);
      const V t1 = cmul(ab, f1), t2 = cmul(cb, f2), t3 = cmul(cconj(cb), f3), t4 = cmul(cconj(ab), f4);
      const V s12 = cadd(t1, t2), s34 = cadd(t3, t4);
      const V u00 = cmul(c, cadd(s12, s34));
      yqq[k3] = u00.x;
      if (!deg3) yqq[m3] = -u00.y;
      if (!deg2) {
        const V u01 = cmul(c, csub(s12, s34));
        yqm[k3] = -u01.y;
        if (!deg3) yqm[m3] = -u01.x;
      }
      if (!deg1) {
        const V d12 = csub(t1, t2), d34 = csub(t3, t4);
        const V u10 = cmul(c, cadd(d12, d34));
        ymq[k3] = -u10.y;
        if (!deg3) ymq[m3] = -u10.x;
        if (!deg2) {
          const V u11 = cmul(c, csub(d12, d34));
          ymm[k3] = -u11.x;
          if (!deg3) ymm[m3] = u11.y;
        }
      }
    };
    for (int k3 = t; k3 <= M / 2; k3 += NT) {
      const int kb = (M - k3) & (M - 1);
      // row_nat(l, k) = f(l M) ^ f(k): the swizzle is GF(2)-linear and l M, k
      // have disjoint bits, so f(l M) is a compile-time constant
      const int fk = SwzRow<T>::f(k3), fb = SwzRow<T>::f(kb);  // k3 <= M/2 < M
      V Za[4], Zb[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int fl = SwzRow<T>::fc(l * M);
        Za[l] = sm[fl ^ fk];
        Zb[l] = sm[fl ^ fb];
      }
      item(k3, Za, Zb);
      if (2 * k3 != M) item(M - k3, Zb, Za);
    }
  }
}

}  // namespace sdctb
