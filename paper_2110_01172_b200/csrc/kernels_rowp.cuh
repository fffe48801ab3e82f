// Mirror-paired row-pair kernel of the 2D pipelines (M = N2/2 = 1024, 2048; fp64 and fp32).
//
// Same work item and persistent ring as row2_kernel MODE 0 (kernels_row2.cuh:
// one row pair (k1, N1-k1) per item, two consumer groups, NBUF landing /
// exchange buffers refilled by 1D bulk copies), but the butterflies of the
// radix-8 FFT stage next to the frequency domain are assigned so that a
// thread and its lane ^ 16 partner own mirror frequency sets: the thread owns
// frequencies k0 + (M/8) r (r = 0..7) of both rows, its partner k0' = M/8 - k0
// (rowp_k0 below; k0 = 0 and M/16 are their own mirrors), and
//
// M - (k0 + (M/8) r) = (M/8 - k0) + (M/8)(7 - r), so the coupling of
// frequency k with M - k that the merged postprocess (proj/src/dct2d.cpp:
// 82-115, with the Hermitian unpack of the packed real rows) and the merged
// inverse preprocess (dct2d.cpp:161-198, with the inverse packing) need is a
// register exchange with the partner lane (a shuffle with lane ^ 16) instead of a pass
// through shared memory:
//
//   forward: ... DIF stages 0, 1 -> stage 2 (radix 8) with the paired
//            mapping -> postprocess straight from registers to y.
//   inverse: rows of x -> preprocess + packing straight into the paired
//            radix-8 DIT input layout -> DIT stages 2, 1, 0 -> natural
//            order -> pair-interleaved intermediate rows.
//
// Per item this drops one 64 KB write + read of shared memory (the natural-
// order postprocess tile, resp. the packed-spectrum tile) and, in the
// inverse, the barrier across which the preprocess operands were held, which
// is what kept the inverse off the ring schedule.
#pragma once

#include "kernels_row2.cuh"

namespace sdctb {

// Ring geometry: two consumer groups (the row2 tile) and 3-4 item buffers
// (fp64 M = 2048: 3 x 64 KB, one CTA per SM; fp64 M = 1024: 3 x 32 KB, two).
template <typename T, int M>
struct RowpGeom {
  // M = 512 (radices 8, 8, 8): cap the tile at 64 threads so that every
  // thread holds 16 elements, the radix-8 last stage's two butterflies being
  // the two rows (as for M = 1024, 2048)
  using TL = Row2Tile<T, M, false, 2, M == 512 ? 64 : 0>;
  static constexpr unsigned BUF = 2u * M * sizeof(cx_t<T>);
  static constexpr int NT = TL::NT, CTA = 2 * TL::NT, GROUPS = 2;
  // 512-thread CTAs (M = 2048) keep 128 registers per thread with one CTA per
  // SM; 256-thread CTAs (M = 1024) run two per SM, 128-thread CTAs three
  static constexpr int MINB = CTA >= 512 ? 1 : CTA >= 256 ? 2 : 3;
  static constexpr int NBUF = (200u * 1024u) / (BUF * MINB) >= 4 ? 4 : 3;
  static constexpr size_t BARS = static_cast<size_t>(NBUF) * BUF;
  static constexpr size_t SMEM = BARS + 16 * NBUF;
};

// M = 1024, 2048 both directions; M = 512 forward only (the inverse's paired
// last DIT stage assumes one stage-0 butterfly per thread)
template <typename T, int M, bool INV = false>
constexpr bool rowp_ok() {
  if constexpr (M != 512 && M != 1024 && M != 2048) {
    return false;
  } else {
    using TL = typename RowpGeom<T, M>::TL;
    using P = typename TL::P;
    return (!INV || M != 512) && TL::S == 3 && P::R(2) == 8 && TL::NT == M / 8 && TL::E == 16 &&
           RowpGeom<T, M>::MINB * RowpGeom<T, M>::SMEM <= 220u * 1024u;
  }
}

// k0 of group-local thread t (see above): lanes l < 16 of warp w take
// k0 = 16 w + l, lanes l >= 16 the mirrors M/8 - (16 w + l - 16) (lane 16 of
// warp 0: M/16). Consecutive lanes thus own consecutive frequencies, which
// keeps the postprocess's y stores and the inverse's operand reads coalesced
// and conflict free; the paired radix-8 stage's shared-memory accesses are
// conflict free at M = 2048 except in the phases holding k0 = 0 / the mirrors
// of 16 w (2-way), and 2-way at M = 1024 (tests/test_host.py).
template <int M>
__device__ __forceinline__ int rowp_k0(int t) {
  constexpr int K0 = M / 8;
  const int w = t >> 5, l = t & 31;
  if (l < 16) return 16 * w + l;
  const int u = 16 * w + l - 16;
  return u == 0 ? K0 / 2 : K0 - u;
}

// Steps of the thread's frequency set for N2 = 2M = 4096:
// b(k0 + 256 r) = b(k0) e^{-i pi r / 32}, W^(k0 + 256 r) = W^k0 e^{-i pi r / 8}
template <typename T>
__device__ __forceinline__ cx_t<T> rowp_sb(int r) {
  constexpr double c[9][2] = {{1.0, -0.0},
                              {0.9951847266721969, -0.0980171403295606},
                              {0.9807852804032304, -0.19509032201612828},
                              {0.9569403357322088, -0.2902846772544624},
                              {0.9238795325112867, -0.3826834323650898},
                              {0.881921264348355, -0.47139673682599764},
                              {0.8314696123025452, -0.5555702330196022},
                              {0.773010453362737, -0.6343932841636455},
                              {0.7071067811865476, -0.7071067811865476}};
  return mk(static_cast<T>(c[r][0]), static_cast<T>(c[r][1]));
}
template <typename T>
__device__ __forceinline__ cx_t<T> rowp_sw(int r) {
  constexpr double c[9][2] = {{1.0, -0.0},
                              {0.9238795325112867, -0.3826834323650898},
                              {0.7071067811865476, -0.7071067811865476},
                              {0.3826834323650898, -0.9238795325112867},
                              {0.0, -1.0},
                              {-0.3826834323650898, -0.9238795325112867},
                              {-0.7071067811865476, -0.7071067811865476},
                              {-0.9238795325112867, -0.3826834323650898},
                              {-1.0, 0.0}};
  return mk(static_cast<T>(c[r][0]), static_cast<T>(c[r][1]));
}

// force-field weighting inside the inverse preprocess reads (1) or as a
// separate pass over the landed rows (0, A/B)
#ifndef SDCT_ROWP_WPRE
#define SDCT_ROWP_WPRE 1
#endif
constexpr bool kWeightInPre = SDCT_ROWP_WPRE != 0;

template <typename T, int M, bool INV>
__device__ __forceinline__ void rowp_body(const RowArgs& a, const TwSet& tw, const int nitems, const int cta,
                                          const int ncta) {
  static_assert(rowp_ok<T, M, INV>(), "mirror-paired row kernel: M = 512 (forward), 1024, 2048 only");
  using G = RowpGeom<T, M>;
  using TL = typename G::TL;
  using V = cx_t<T>;
  constexpr int NT = G::NT, NBUF = G::NBUF, GROUPS = G::GROUPS;
  constexpr int R0 = TL::R0, Q0 = M / R0, NBF0 = TL::E / R0;
  constexpr int K0 = M / 8;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + G::BARS);
  uint64_t* empty = full + NBUF;
  const int grp = static_cast<int>(threadIdx.x) / NT;
  const int t = static_cast<int>(threadIdx.x) - grp * NT;
  const int n1 = a.n1, n2 = a.n2, half = n1 / 2;
  const int lgh = __ffs(half) - 1;  // fast-path extents are powers of two

  auto issue = [&](int it, int b) {  // thread 0: land item `it` (rows q1, m1) in buffer b
    if (INV && a.rev) it = nitems - 1 - it;
    const int P = it & (half - 1), batch = it >> lgh;
    const int q1 = P, m1 = P == 0 ? half : n1 - P;
    unsigned char* dst = smem_raw + b * G::BUF;
    mbar_expect_tx(full + b, G::BUF);
    if constexpr (!INV) {
      const V* src = static_cast<const V*>(a.src) + batch * a.src_batch;
      bulk_load(dst, src + static_cast<long long>(__ldg(a.s0 + q1)) * M, G::BUF / 2, full + b);
      bulk_load(dst + G::BUF / 2, src + static_cast<long long>(__ldg(a.s0 + m1)) * M, G::BUF / 2, full + b);
    } else {
      int img, md_, wt_;
      inv_item(a, batch, img, md_, wt_);
      const T* src = static_cast<const T*>(a.src) + img * a.src_batch;
      bulk_load(dst, src + static_cast<long long>(q1) * n2, G::BUF / 2, full + b);
      bulk_load(dst + G::BUF / 2, src + static_cast<long long>(m1) * n2, G::BUF / 2, full + b);
    }
  };

  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(full + b, 1);
      mbar_init(empty + b, 1);
    }
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // the previous kernel's output is complete before the first load
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int b = 0; b < NBUF; ++b) {
      const int it = cta + b * ncta;
      if (it < nitems) issue(it, b);
    }
  }

  // the paired radix-8 butterfly of this thread: frequencies k0 + K0 r of
  // both lines, slot 8 bm + r (bm = digit_pos(k0) / 8)
  const int k0 = rowp_k0<M>(t);
  const int bm = digit_pos<M>(k0) >> 3;
  const int pb0 = TL::swz(8 * bm), pb1 = TL::swz(M + 8 * bm);  // swizzled slot bases, lines 0 / 1
  const bool self0 = k0 == 0, selfh = k0 == K0 / 2;               // self-mirror threads
  // shuffle source of the mirror exchange: the lane ^ 16 partner; lane 16 of
  // warp 0 (k0 = K0/2) is its own mirror and reads itself; lane 0 of warp 0
  // (k0 = 0, mirror slot (8 - r) mod 8 and the Nyquist term) is fixed up
  // separately after the uniform loop
  const int msrc = selfh ? (t & 31) : ((t & 31) ^ 16);
  const V* fbt = static_cast<const V*>(a.fb);
  const V* fut = static_cast<const V*>(a.fu);

#pragma unroll 1
  for (int k = grp;; k += GROUPS) {
    const int it = static_cast<int>(cta) + k * static_cast<int>(ncta);
    if (it >= nitems) break;
    const int b = k % NBUF;
    const uint32_t ph = static_cast<uint32_t>(k / NBUF) & 1u;
    if (k >= NBUF) mbar_wait(empty + b, ph ^ 1u);  // item k-NBUF released the buffer
    V* sm = reinterpret_cast<V*>(smem_raw + b * G::BUF);
    const int itm = (INV && a.rev) ? nitems - 1 - it : it;
    const int P = itm & (half - 1), batch = itm >> lgh;
    const int q1 = P, m1 = P == 0 ? half : n1 - P;
    V v[16];
    int img_, imode, iweight;  // inverse: source item, composite mode, weighting (paired launches)
    inv_item(a, batch, img_, imode, iweight);

    if constexpr (!INV) {
      // ===== forward: DIF stages 0, 1 (tile mapping), stage 2 paired =======
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);
      mbar_wait(full + b, ph);
#pragma unroll
      for (int i = 0; i < NBF0; ++i) {
        int line, j, bb;
        TL::template decode<0>(t + i * NT, line, j, bb);
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int n = j + r * Q0;
          const int s = (r < R0 / 2) ? 2 * n : 2 * M - 1 - 2 * n;  // pair-interleaved column of z(n)
          v[i * R0 + r] = sm[line * M + s];
        }
      }
      TL::sync();  // landing rows consumed: the buffer becomes the exchange buffer
      stage_compute<TL, 0, false>(v, w0);
      to_smem<TL, 0>(v, sm, t);
      TL::sync();
      {
        StageTw<TL, 1> w1;
        w1.load(tw.st[1], t);
        from_smem<TL, 1>(v, sm, t);
        stage_compute<TL, 1, false>(v, w1);
      }
      to_smem<TL, 1>(v, sm, t);
      // the postprocess's table values, issued ahead of the last stage they follow
      const V av0 = __ldg(static_cast<const V*>(a.ta) + q1), av1 = __ldg(static_cast<const V*>(a.ta) + m1);
      const V bk0 = fac_lookup(fbt, k0, a.fs), wk0 = fac_lookup(fut, k0, a.fs);
      TL::sync();
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        v[r] = sm[pb0 ^ TL::swzc(r)];
        v[8 + r] = sm[pb1 ^ TL::swzc(r)];
      }
      dft_reg<T, 8, false>(v);
      dft_reg<T, 8, false>(v + 8);
      // v[r] = Z(k1, k0 + K0 r), v[8 + r] = Z(k1', k0 + K0 r) (k1' = N1 - k1)

      // merged postprocess (dct2d.cpp:93-113) with the Hermitian unpack folded
      // in (see row2_kernel): 2X = (A + B) + (-i W^q)(A - B), A = Z(k1, q),
      // B = conj Z(-k1, -q); the factors 1/2 ride on a(k1)/4
      T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
      T* r0 = y + static_cast<long long>(q1) * n2;
      T* r1 = y + static_cast<long long>(m1) * n2;
      const V a40 = mk(av0.x * T(0.25), av0.y * T(0.25)), a41 = mk(av1.x * T(0.25), av1.y * T(0.25));
      auto unpack2 = [](V A, V Bc, V w) {  // Bc = conj(B) as stored
        const T sx = A.x + Bc.x, sy = A.y - Bc.y;
        const T dx = A.x - Bc.x, dy = A.y + Bc.y;
        return mk(fma(w.y, dx, fma(w.x, dy, sx)), fma(w.y, dy, fma(-w.x, dx, sy)));
      };
      auto item = [&](int q, V Z0a, V Z0b, V Z1a, V Z1b, V bq, V w) {
        const bool deg2k = (q == 0) || (q == M);
        if (P != 0) {
          const V X1 = unpack2(Z0a, Z1b, w);  // 2 X(k1, q)
          const V X2 = unpack2(Z1a, Z0b, w);  // 2 X(-k1, q)
          const V ax1 = cmul(a40, X1), ax2 = cmulc(X2, a40);
          const V sp = cadd(ax1, ax2), tp = csub(ax1, ax2);
          r0[q] = fma(bq.x, sp.x, -bq.y * sp.y);
          r1[q] = -fma(bq.x, tp.y, bq.y * tp.x);
          if (!deg2k) {
            r0[n2 - q] = -fma(bq.x, sp.y, bq.y * sp.x);
            r1[n2 - q] = fma(-bq.x, tp.x, bq.y * tp.y);
          }
        } else {
          const V X0 = unpack2(Z0a, Z0b, w);
          const V X1 = unpack2(Z1a, Z1b, w);
          const T c0 = T(2) * a40.x, c1 = T(2) * a41.x;
          const V bx0 = cmul(bq, X0), bx1 = cmul(bq, X1);
          r0[q] = c0 * bx0.x;
          r1[q] = c1 * bx1.x;
          if (!deg2k) {
            r0[n2 - q] = -c0 * bx0.y;
            r1[n2 - q] = -c1 * bx1.y;
          }
        }
      };
      // b(q), W^q on q = k0 + K0 r: the thread's base values times
      // compile-time steps (no table lookup per frequency)
      auto bq_of = [&](int r) {  // b(k0 + K0 r), negated where the corrupt hook says so
        V bq = cmul(bk0, rowp_sb<T>(r));
        if (a.badq && a.badq[k0 + K0 * r]) bq = mk(-bq.x, -bq.y);
        return bq;
      };
      // mirror frequency M - q: the partner's slot 7 - r (k0 = 0: own slot
      // (8 - r) mod 8, plus q = M with Z(k1, M) = Z(k1, 0))
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        V m0, m1v;
        m0.x = __shfl_sync(0xffffffffu, v[7 - r].x, msrc);
        m0.y = __shfl_sync(0xffffffffu, v[7 - r].y, msrc);
        m1v.x = __shfl_sync(0xffffffffu, v[15 - r].x, msrc);
        m1v.y = __shfl_sync(0xffffffffu, v[15 - r].y, msrc);
        if (self0) {
          m0 = v[(8 - r) & 7];
          m1v = v[8 + ((8 - r) & 7)];
        }
        item(k0 + K0 * r, v[r], m0, v[8 + r], m1v, bq_of(r), cmul(wk0, rowp_sw<T>(r)));
      }
      if (self0) item(M, v[0], v[0], v[8], v[8], bq_of(8), rowp_sw<T>(8));
    } else {
      // ===== inverse: preprocess + packing into the paired DIT input =======
      // table values of this item, issued before the landing wait they overlap
      const V ca0 = cconj(__ldg(static_cast<const V*>(a.ta) + q1)), ca1 = cconj(__ldg(static_cast<const V*>(a.ta) + m1));
      const V bk0 = fac_lookup(fbt, k0, a.fs), wk0 = fac_lookup(fut, k0, a.fs);
      mbar_wait(full + b, ph);
      const T* rowA = reinterpret_cast<const T*>(sm);
      const T* rowB = reinterpret_cast<const T*>(sm) + 2 * M;
      if (iweight == 3) {
        // compression threshold folded into this load (compress.cpp:33-45)
        T* const rws[2] = {const_cast<T*>(rowA), const_cast<T*>(rowB)};
        const T eps = static_cast<T>(a.thr_eps), sc = static_cast<T>(a.thr_scale);
        unsigned cnt = 0;
        for (int e = t; e < 2 * n2; e += NT) {
          T* rw = rws[e >= n2] + (e & (n2 - 1));
          const T vv = *rw;
          const bool drop = fabs(vv) < eps;
          cnt += drop ? 1u : 0u;
          *rw = drop ? T(0) : vv * sc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0 && cnt && a.thr_count) atomicAdd(a.thr_count, static_cast<unsigned long long>(cnt));
        TL::sync();
      } else if (iweight && !kWeightInPre) {
        // DREAMPlace field weighting folded into this load (force.cpp:19-31)
        T* const rws[2] = {const_cast<T*>(rowA), const_cast<T*>(rowB)};
        const T pi = T(3.14159265358979323846);
        const T w1a = pi * T(q1) / T(n1), w1b = pi * T(m1) / T(n1), sc2 = pi / T(n2);
        for (int e = t; e < 2 * n2; e += NT) {
          const int k2 = e & (n2 - 1);
          T* rw = rws[e >= n2] + k2;
          const T w1 = e < n2 ? w1a : w1b, w2 = sc2 * T(k2);
          const T den = fma(w1, w1, w2 * w2);
          *rw = den > T(0) ? *rw * (iweight == 1 ? w1 : w2) / den : T(0);
        }
        TL::sync();
      }
      const bool swp = imode == 1 && P != 0;
      if (swp) {  // IDXST along axis 0 swaps the rows' roles
        const T* tmp = rowA;
        rowA = rowB;
        rowB = tmp;
      }
      // field weighting (force.cpp:19-31) applied to the four values each
      // xpair reads: x(k1, k2) *= w_j / (w1^2 + w2^2), w1 = pi k1/N1,
      // w2 = pi k2/N2; the four denominators share one division (batched
      // reciprocal). den = 0 only at (0, 0), where the numerator is 0 too.
      const T pi_ = T(3.14159265358979323846);
      const T wA = pi_ * T(swp ? m1 : q1) / T(n1), wB = pi_ * T(swp ? q1 : m1) / T(n1);
      const T wA2 = wA * wA, wB2 = wB * wB, sc2 = pi_ / T(n2);
      auto weigh = [&](int pd, int pr, T& DA, T& RA, T& DB, T& RB) {
        const T wd = sc2 * T(pd), wr = sc2 * T(pr);
        T dAd = fma(wd, wd, wA2), dAr = fma(wr, wr, wA2), dBd = fma(wd, wd, wB2), dBr = fma(wr, wr, wB2);
        dAd = dAd > T(0) ? dAd : T(1);
        dBd = dBd > T(0) ? dBd : T(1);
        dAr = dAr > T(0) ? dAr : T(1);
        dBr = dBr > T(0) ? dBr : T(1);
        const T pA = dAd * dAr, pB = dBd * dBr;
        const T inv = T(1) / (pA * pB);
        const T iA = inv * pB, iB = inv * pA;
        const bool w1 = iweight == 1;
        DA *= (w1 ? wA : wd) * (iA * dAr);
        RA *= (w1 ? wA : wr) * (iA * dAd);
        DB *= (w1 ? wB : wd) * (iB * dBr);
        RB *= (w1 ? wB : wr) * (iB * dBd);
      };

      // X'(0, nn), X'(1, nn) (proj/src/dct2d.cpp:182-195) from x(nn), x(N2-nn)
      // of both rows (x(N2) := 0); mode 2 reads x(N2-nn) for D and x(nn) for R
      // with x(0) := 0 (dct2d.cpp:169-180)
      // c0 = conj a(q1) conj b(nn), c1 = conj a(m1) conj b(nn) with
      // b(k0 + K0 r) = b(k0) e^{-i pi r/32}: per-item constants times the step
      const V cc0 = cmulc(ca0, bk0), cc1 = cmulc(ca1, bk0);
      auto xpair = [&](int r, V& x0, V& x1) {
        const int nn = k0 + K0 * r;
        const bool z = nn == 0;
        const int pd = imode == 2 ? n2 - nn : nn;
        const int pr = imode == 2 ? nn : n2 - nn;
        const bool zd = imode == 2 && z;
        T DA = zd ? T(0) : rowA[pd & (n2 - 1)], RA = z ? T(0) : rowA[pr & (n2 - 1)];
        T DB = zd ? T(0) : rowB[pd & (n2 - 1)], RB = z ? T(0) : rowB[pr & (n2 - 1)];
        if (kWeightInPre && (iweight == 1 || iweight == 2)) weigh(pd, pr, DA, RA, DB, RB);
        V c0 = cmulc(cc0, rowp_sb<T>(r)), c1 = cmulc(cc1, rowp_sb<T>(r));
        if (a.badq && a.badq[nn]) {  // corrupt_twiddle_for_testing negated b(nn)
          c0 = mk(-c0.x, -c0.y);
          c1 = mk(-c1.x, -c1.y);
        }
        if (P == 0) {
          // rows 0 and N1/2, each its own mirror: row 0 pairs with the zero
          // row N1; mode 1 zeroes row 0 entirely
          const T pa = imode == 1 ? T(0) : DA, sa = imode == 1 ? T(0) : RA;
          x0 = cmul(c0, mk(pa, -sa));
          x1 = cmul(c1, mk(DB - RB, -(DB + RB)));
          return;
        }
        x0 = cmul(c0, mk(DA - RB, -(DB + RA)));
        x1 = cmul(c1, mk(DB - RA, -(DA + RB)));
      };
#pragma unroll
      for (int r = 0; r < 8; ++r) xpair(r, v[r], v[8 + r]);
      V nyq0, nyq1;  // X'(., M) for the k0 = 0 thread's slot 0
      if (self0) xpair(8, nyq0, nyq1);  // nn = M
      TL::sync();  // landing rows consumed: the buffer becomes the exchange buffer
      // inverse packing Zh(k) = (X(k) + X(k+M)) + i conj(W^k)(X(k) - X(k+M)),
      // X(line, k + M) = conj X(partner line, M - k) (own line for P == 0)
      auto packr = [&](int r, V mir0, V mir1) {
        const int nn = k0 + K0 * r;
        const V wk = cmul(wk0, rowp_sw<T>(r));
        const V h0 = nn == 0 ? nyq0 : cconj(P != 0 ? mir1 : mir0);
        const V h1 = nn == 0 ? nyq1 : cconj(P != 0 ? mir0 : mir1);
        v[r] = pack(v[r], h0, wk);
        v[8 + r] = pack(v[8 + r], h1, wk);
      };
      // pairs (r, 7 - r): every lane exchanges (converged warp), then all but
      // the k0 = 0 thread pack both slots in place
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        V a0, a1, c0v, c1v;  // partner's X' at slots 7 - r (mirror of r) and r (mirror of 7 - r)
        a0.x = __shfl_sync(0xffffffffu, v[7 - r].x, msrc);
        a0.y = __shfl_sync(0xffffffffu, v[7 - r].y, msrc);
        a1.x = __shfl_sync(0xffffffffu, v[15 - r].x, msrc);
        a1.y = __shfl_sync(0xffffffffu, v[15 - r].y, msrc);
        c0v.x = __shfl_sync(0xffffffffu, v[r].x, msrc);
        c0v.y = __shfl_sync(0xffffffffu, v[r].y, msrc);
        c1v.x = __shfl_sync(0xffffffffu, v[8 + r].x, msrc);
        c1v.y = __shfl_sync(0xffffffffu, v[8 + r].y, msrc);
        if (!self0) {
          packr(r, a0, a1);
          packr(7 - r, c0v, c1v);
        }
      }
      if (self0) {
        // k0 = 0: mirror of slot r is slot (8 - r) mod 8; slot 0 uses X'(M)
#pragma unroll
        for (int r = 1; r < 4; ++r) {
          const V a0 = v[8 - r], a1 = v[16 - r], c0v = v[r], c1v = v[8 + r];
          packr(r, a0, a1);
          packr(8 - r, c0v, c1v);
        }
        packr(0, v[0], v[8]);
        packr(4, v[4], v[12]);
      }
      // DIT: stage 2 (radix 8, paired mapping) -> stages 1, 0 (tile mapping)
      dft_reg<T, 8, true>(v);
      dft_reg<T, 8, true>(v + 8);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        sm[pb0 ^ TL::swzc(r)] = v[r];
        sm[pb1 ^ TL::swzc(r)] = v[8 + r];
      }
      TL::sync();
      {
        StageTw<TL, 1> w1;
        w1.load(tw.st[1], t);
        from_smem<TL, 1>(v, sm, t);
        dit_compute<TL, 1, true>(v, w1);
        to_smem<TL, 1>(v, sm, t);
      }
      TL::sync();
      // last DIT stage with lanes paired j <-> Q0-1-j in each warp (virtual
      // tile index tv): output z(j + Q0 r) lands in pair-interleaved column
      // 2(j + Q0 r) (r < R0/2) or 2M-1-2(j + Q0 r), so at store step r the
      // lower half-warp's v[r] and the upper half-warp's v[R0-1-r] are the two
      // 16-B halves of the same 32-B sectors: direct coalesced stores, no
      // natural-order staging pass
      const int wq = (t >> 5) & (Q0 / 32 - 1), l = t & 31;
      const int jv = l < 16 ? 16 * wq + l : Q0 - 1 - (16 * wq + l - 16);
      const int lv = t / (NT / 2);
      const int tv = lv * Q0 + jv;
      {
        StageTw<TL, 0> w0;
        w0.load(tw.st[0], tv);
        from_smem<TL, 0>(v, sm, tv);
        dit_compute<TL, 0, true>(v, w0);
      }
      V* drow = static_cast<V*>(a.dst) + batch * a.dst_batch +
                static_cast<long long>(__ldg(a.s0 + (lv ? m1 : q1))) * M;
      const bool hi = l >= 16;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int rr = hi ? R0 - 1 - r : r;
        const int m = jv + Q0 * rr;
        const int col = rr < R0 / 2 ? 2 * m : 2 * M - 1 - 2 * m;
        drow[col] = hi ? v[R0 - 1 - r] : v[r];
      }
    }
    TL::sync();  // every read of buffer b by this group is done
    if (t == 0) {
      mbar_arrive(empty + b);
      const int nxt0 = it + NBUF * static_cast<int>(ncta);
      if (nxt0 < nitems) {
        fence_async_smem();  // generic-proxy smem accesses before the async refill
        issue(nxt0, b);
      }
    }
  }
}

template <typename T, int M, bool INV>
__global__ void __launch_bounds__(RowpGeom<T, M>::CTA, RowpGeom<T, M>::MINB)
    rowp_kernel(RowArgs a, TwSet tw, int nitems) {
  rowp_body<T, M, INV>(a, tw, nitems, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
}

}  // namespace sdctb
