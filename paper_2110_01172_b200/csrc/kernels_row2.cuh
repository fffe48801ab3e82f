// Persistent row-pair kernel of the 2D pipelines (forward DCT-II and the
// inverse / IDXST-composite family).
//
// Work item = one row pair (k1, N1-k1) of one batch image (k1 = 0 pairs rows
// 0 and N1/2, each its own mirror). That is the unit the reference's merged
// postprocess (proj/src/dct2d.cpp:82-115) and merged inverse preprocess
// (proj/src/dct2d.cpp:161-198) couple, so the row FFT and both of those
// stages fuse into one pass over the rows.
//
// Pipeline (MODE 0, large rows): one persistent CTA per SM with two consumer
// groups of NT threads (named barriers) and a ring of NBUF shared-memory
// buffers. The CTA's k-th item (blockIdx.x + k*gridDim.x) is computed by
// group k % 2 in buffer k % NBUF. A buffer receives its item by two 1D bulk
// copies (one per row; completion on the buffer's `full` mbarrier), then is
// that item's FFT exchange buffer; when the item is done the group's leader
// arrives on the buffer's `empty` mbarrier and refills it with item k+NBUF.
// So loads run NBUF-1 items ahead, two items' math interleaves on the SM
// (16 warps), and no grid-wide phase alignment of load/compute/store forms.
// A consumer waits `empty` (release of item k-NBUF) before `full`, which
// keeps every mbarrier waiter at most one phase behind (parity-safe).
// MODE 1 (small rows, and the inverse for M > 1024 where it measures
// faster): one item per CTA, several CTAs per SM.
//
//   forward (RK_FWD2): rows srow(k1), srow(N1-k1) of the column pass's
//     intermediate Z (pair-interleaved complex) -> row FFT -> Hermitian
//     unpack + merged DCT postprocess -> rows k1, N1-k1 of y.
//   inverse (RK_INV2): rows k1, N1-k1 of x (real) -> merged inverse
//     preprocess + inverse packing -> inverse row FFT -> intermediate rows
//     srow(k1), srow(N1-k1) (natural order, pair-interleaved columns).
#pragma once

#include "kernels_fast.cuh"

namespace sdctb {

// Row tile of the pair kernel. GROUPS > 1: the tile's threads are one of
// several groups in the CTA; exchanges synchronise on the group's named
// barrier (id 1 + group).
template <typename T, int M, bool FULLTW, int GROUPS, int MAXT_ = 0>
struct Row2Tile : Tile<T, M, 2, false, MAXT_> {
  using Base = Tile<T, M, 2, false, MAXT_>;
  static constexpr bool TWF = FULLTW;
  __device__ __forceinline__ static void sync() {
    if constexpr (GROUPS == 1) {
      __syncthreads();
    } else {
      named_sync(1 + static_cast<int>(threadIdx.x) / Base::NT, Base::NT);
    }
  }
};

// e^{-i theta q} = hi[q >> s] * lo[q & (2^s - 1)]; table = lo (2^s) then hi
template <typename V>
__device__ __forceinline__ V fac_lookup(const V* tab, int q, int s) {
  return cmul(__ldg(tab + (1 << s) + (q >> s)), __ldg(tab + (q & ((1 << s) - 1))));
}
// b(M - q) = e^{-i pi/4} conj b(q) for b(q) = e^{-i pi q / (2 N2)}, M = N2 / 2
template <typename V>
__device__ __forceinline__ V mirror_b(V b) {
  using T = decltype(b.x);
  const T h = T(0.70710678118654752440);  // (h, -h) * (b.x, -b.y)
  return mk(h * (b.x - b.y), -h * (b.x + b.y));
}

template <typename T, int M>
constexpr int row2_mode() {
  // two groups need two resident buffers
  return Tile<T, M, 2, false>::NT >= 128 && 2u * (2u * M * sizeof(cx_t<T>)) <= 200u * 1024u ? 0 : 1;
}

// MODE 0: persistent, two consumer groups, ring of NBUF full buffers.
// MODE 1: one item per CTA.
// MODE 2: persistent, one group, two CTAs per SM; a full buffer holds row B
//         and serves as the exchange buffer, a half buffer prefetches the
//         next item's row A while the current item computes (row B of the
//         next item loads once the exchange buffer is free).
template <typename T, int M, int MODE>
struct Row2Geom {
  static constexpr unsigned BUF = 2u * M * sizeof(cx_t<T>);  // one pair: 2 complex rows == 2 real rows of 2M
  static constexpr int GROUPS = MODE == 0 ? 2 : 1;
  static constexpr int NBUF = MODE != 0 ? 1
                              : (200u * 1024u) / BUF >= 4 ? 4
                              : ((200u * 1024u) / BUF < 2 ? 2 : static_cast<int>((200u * 1024u) / BUF));
  using TL = Row2Tile<T, M, SDCT_ROW_FULLTW != 0, GROUPS>;
  static constexpr int NT = TL::NT;  // threads per group
  static constexpr int CTA = NT * GROUPS;
  // fp32: 3 CTAs/SM (inverse row 56 -> 52 us at 4096^2); fp64 spills at 3
  static constexpr int MINB = MODE == 0 ? 1 : (sizeof(T) == 4 ? 3 : 2);
  static constexpr size_t PREF = MODE == 2 ? BUF / 2 : 0;                               // row-A prefetch region
  static constexpr size_t BARS = static_cast<size_t>(NBUF) * BUF + PREF;                // mbarriers
  static constexpr size_t STASH = BARS + 16 * NBUF + 16;                                // after the mbarriers
  static constexpr size_t SMEM = STASH + 64 * GROUPS;  // + per-group stash of 8 operands
};

template <typename T, int M, bool INV, int MODE>
__global__ void __launch_bounds__(Row2Geom<T, M, MODE>::CTA, Row2Geom<T, M, MODE>::MINB)
    row2_kernel(RowArgs a, TwSet tw, int nitems) {
  using G = Row2Geom<T, M, MODE>;
  using TL = typename G::TL;
  using V = cx_t<T>;
  using V4 = typename Cx<T>::vec4;
  constexpr int NT = G::NT, NBUF = G::NBUF, GROUPS = G::GROUPS;
  constexpr int R0 = TL::R0, Q0 = M / R0, NBF0 = TL::E / R0;
  constexpr int NI = (M / 2) / NT + 1;  // postprocess / preprocess items k in [0, M/2] per thread
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + G::BARS);
  uint64_t* empty = full + NBUF;  // MODE 2: empty[0] is the row-A (prefetch region) barrier
  unsigned char* pref = smem_raw + NBUF * G::BUF;  // MODE 2 row-A region
  const int grp = GROUPS == 1 ? 0 : static_cast<int>(threadIdx.x) / NT;
  const int t = static_cast<int>(threadIdx.x) - grp * NT;  // thread index within the group
  const int n1 = a.n1, n2 = a.n2, half = n1 / 2;

  auto rows_of = [&](int P, int& q1, int& m1) {
    q1 = P;
    m1 = P == 0 ? half : n1 - P;
  };
  // thread 0: land row A (which = 0) or row B (which = 1) of item `it` at dst,
  // completing on bar
  auto issue_row = [&](int it, int which, unsigned char* dst, uint64_t* bar) {
    const int P = it % half, batch = it / half;
    int q1, m1;
    rows_of(P, q1, m1);
    const int row = which ? m1 : q1;
    if constexpr (!INV) {
      const V* src = static_cast<const V*>(a.src) + batch * a.src_batch;
      bulk_load(dst, src + static_cast<long long>(__ldg(a.s0 + row)) * M, G::BUF / 2, bar);
    } else {
      int img, md_, wt_;
      inv_item(a, batch, img, md_, wt_);
      const T* src = static_cast<const T*>(a.src) + img * a.src_batch;
      bulk_load(dst, src + static_cast<long long>(row) * n2, G::BUF / 2, bar);
    }
  };
  // thread 0: land item `it` in buffer b (MODE 0 / 1)
  auto issue = [&](int it, int b) {
    unsigned char* dst = smem_raw + b * G::BUF;
    uint64_t* bar = full + b;
    mbar_expect_tx(bar, G::BUF);
    issue_row(it, 0, dst, bar);
    issue_row(it, 1, dst + G::BUF / 2, bar);
  };
  // MODE 2: row A into the prefetch region, row B into the second half of the buffer
  auto issue_a = [&](int it) {
    mbar_expect_tx(empty, G::BUF / 2);
    issue_row(it, 0, pref, empty);
  };
  auto issue_b = [&](int it) {
    mbar_expect_tx(full, G::BUF / 2);
    issue_row(it, 1, smem_raw + G::BUF / 2, full);
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
    if constexpr (MODE == 2) {
      if (static_cast<int>(blockIdx.x) < nitems) {
        issue_a(blockIdx.x);
        issue_b(blockIdx.x);
      }
    } else {
#pragma unroll 1
      for (int b = 0; b < NBUF; ++b) {
        const int it = blockIdx.x + b * gridDim.x;
        if (it < nitems) issue(it, b);
      }
    }
  }

  // hoisted swizzles of the natural-order row layout (linearity: the
  // per-iteration parts are compile-time XOR offsets)
  const int sw_t = TL::swz(t);
  const int sw_nt = TL::swz((NT - t) & (NT - 1));

#pragma unroll 1
  for (int k = grp;; k += GROUPS) {
    const int it = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
    if (it >= nitems) break;
    const int b = k % NBUF;
    const uint32_t ph = static_cast<uint32_t>(k / NBUF) & 1u;
    if (MODE == 0 && k >= NBUF) mbar_wait(empty + b, ph ^ 1u);  // item k-NBUF released the buffer
    const int nxt = it + static_cast<int>(gridDim.x);          // MODE 2: the CTA's next item
    V* sm = reinterpret_cast<V*>(smem_raw + b * G::BUF);
    const int P = it % half, batch = it / half;
    int q1, m1;
    rows_of(P, q1, m1);
    V v[TL::E];
    int img_, imode, iweight;  // inverse: source item, composite mode, weighting (paired launches)
    inv_item(a, batch, img_, imode, iweight);

    if constexpr (!INV) {
      // ================= forward: FFT + unpack + merged postprocess ==========
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);
      mbar_wait(full + b, ph);
      if constexpr (MODE == 2) mbar_wait(empty, ph);
      const V* line0 = MODE == 2 ? reinterpret_cast<const V*>(pref) : sm;
#pragma unroll
      for (int i = 0; i < NBF0; ++i) {
        int line, j, bb;
        TL::template decode<0>(t + i * NT, line, j, bb);
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int n = j + r * Q0;
          const int s = (r < R0 / 2) ? 2 * n : 2 * M - 1 - 2 * n;  // pair-interleaved column of z(n)
          v[i * R0 + r] = line ? sm[M + s] : line0[s];
        }
      }
      TL::sync();  // landing rows consumed: the buffer becomes the exchange buffer
      if constexpr (MODE == 2) {
        if (t == 0 && nxt < nitems) {
          fence_async_smem();
          issue_a(nxt);  // the next item's row A streams in under this item's math
        }
      }
      fft_regs<TL, false>(v, sm, tw, w0, t);
      TL::sync();
      last_to_natural<TL>(v, sm, t);
      TL::sync();

      // merged postprocess (proj/src/dct2d.cpp:93-113) with the Hermitian
      // unpack folded in: 2X = (A + B) + (-i W^q)(A - B), A = Z(k1, q),
      // B = conj Z(-k1, -q); the factors 1/2 (unpack) and 1/2 (postprocess)
      // ride on a(k1)/4.
      T* y = static_cast<T*>(a.dst) + batch * a.dst_batch;
      T* r0 = y + static_cast<long long>(q1) * n2;
      T* r1 = y + static_cast<long long>(m1) * n2;
      const V* fb = static_cast<const V*>(a.fb);
      const V* fu = static_cast<const V*>(a.fu);
      const V av0 = __ldg(static_cast<const V*>(a.ta) + q1), av1 = __ldg(static_cast<const V*>(a.ta) + m1);
      const V a40 = mk(av0.x * T(0.25), av0.y * T(0.25)), a41 = mk(av1.x * T(0.25), av1.y * T(0.25));
      // X' = S + w' D with S = A + B, D = A - B, w' = -i w
      auto unpack2 = [](V A, V Bc, V w) {  // Bc = conj(B) as stored: B = (Bc.x, -Bc.y)
        const T sx = A.x + Bc.x, sy = A.y - Bc.y;
        const T dx = A.x - Bc.x, dy = A.y + Bc.y;
        // w' = (w.y, -w.x): w' D = (w.y dx + w.x dy, w.y dy - w.x dx)
        return mk(fma(w.y, dx, fma(w.x, dy, sx)), fma(w.y, dy, fma(-w.x, dx, sy)));
      };
      auto item = [&](int q, V Z0a, V Z0b, V Z1a, V Z1b, V bq, V w) {
        // Z0a = Z(k1, q), Z0b = Z(k1, -q), Z1a = Z(k1', q), Z1b = Z(k1', -q);
        // bq = b(q), w = W_N2^q
        const bool deg2k = (q == 0) || (q == M);
        if (P != 0) {
          const V X1 = unpack2(Z0a, Z1b, w);  // 2 X(k1, q)
          const V X2 = unpack2(Z1a, Z0b, w);  // 2 X(-k1, q)
          const V ax1 = cmul(a40, X1), ax2 = cmulc(X2, a40);
          const V sp = cadd(ax1, ax2), tp = csub(ax1, ax2);
          // sv = b sp, tv = b tp; outputs sv.x, -tv.y, -sv.y, -tv.x
          r0[q] = fma(bq.x, sp.x, -bq.y * sp.y);
          r1[q] = -fma(bq.x, tp.y, bq.y * tp.x);
          if (!deg2k) {
            r0[n2 - q] = -fma(bq.x, sp.y, bq.y * sp.x);
            r1[n2 - q] = fma(-bq.x, tp.x, bq.y * tp.y);
          }
        } else {
          // rows 0 and N1/2 are their own mirrors (deg1: X2 = X1), so
          // s = b (a + conj a) X = 2 Re(a4) b X'
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
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int k2 = t + i * NT;
        if (k2 <= M / 2) {
          // natural-order slots of k2 and kb = (M - k2) mod M in both lines
          const int sa = sw_t ^ TL::swzc(i * NT);
          const int sb = t ? (sw_nt ^ TL::swzc(M - (i + 1) * NT)) : TL::swzc((M - i * NT) & (M - 1));
          const V Z0a = sm[sa], Z0b = sm[sb];
          const V Z1a = sm[sa ^ TL::swzc(M)], Z1b = sm[sb ^ TL::swzc(M)];
          // b(q), W^q from two small factor tables; the mirror q' = M - q
          // needs none: b(M-q) = e^{-i pi/4} conj b(q), W^{M-q} = -conj W^q
          const V bq = fac_lookup(fb, k2, a.fs), w = fac_lookup(fu, k2, a.fs);
          const V bm = mirror_b(bq);
          item(k2, Z0a, Z0b, Z1a, Z1b, (a.badq && a.badq[k2]) ? mk(-bq.x, -bq.y) : bq, w);
          if (2 * k2 != M)
            item(M - k2, Z0b, Z0a, Z1b, Z1a, (a.badq && a.badq[M - k2]) ? mk(-bm.x, -bm.y) : bm, mk(-w.x, w.y));
        }
      }
    } else {
      // ============ inverse: merged preprocess + packing + inverse FFT =======
      // buffer = rows q1 (A) and m1 (B) of x, 2M reals each
      const T* rowA = MODE == 2 ? reinterpret_cast<const T*>(pref) : reinterpret_cast<const T*>(sm);
      const T* rowB = reinterpret_cast<const T*>(sm) + 2 * M;
      // (the weighting below runs on the landed rows in their own order)
      mbar_wait(full + b, ph);
      if constexpr (MODE == 2) mbar_wait(empty, ph);
      if (iweight == 3) {
        // compression (proj/src/compress.cpp:33-45) folded into this load:
        // zero every coefficient with |b| < eps (counted), scale the rest by
        // the 4/(N1 N2) reconstruction normalisation (linear, so it commutes
        // with the inverse transform)
        T* const rws[2] = {const_cast<T*>(rowA), const_cast<T*>(rowB)};
        const T eps = static_cast<T>(a.thr_eps), sc = static_cast<T>(a.thr_scale);
        unsigned cnt = 0;
        for (int e = t; e < 2 * n2; e += NT) {
          T* rw = rws[e >= n2] + (e & (n2 - 1));
          const T v = *rw;
          const bool drop = fabs(v) < eps;
          cnt += drop ? 1u : 0u;
          *rw = drop ? T(0) : v * sc;
        }
        constexpr int W = NT < 32 ? NT : 32;  // lanes per warp in use
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(TL::MASK, cnt, o);
        if ((threadIdx.x & 31) == 0 && cnt && a.thr_count) atomicAdd(a.thr_count, static_cast<unsigned long long>(cnt));
        TL::sync();
      } else if (iweight) {
        // DREAMPlace-style field weighting of the input coefficients
        // (proj/src/force.cpp:19-31), folded into this load: a1 = a w1/(w1^2+w2^2)
        // (weight 1) or a2 = a w2/(w1^2+w2^2) (weight 2), w_d = pi k_d / n_d, 0 at DC
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
      // operands for n2 in {k, M-k}: D = x(n2), R = x(N2-n2) (x(N2) := 0) of
      // both rows; mode 2 (IDXST along axis 1) reads x(N2-n2) for D and x(n2)
      // for R with x(0) := 0 (proj/src/dct2d.cpp:169-180)
      // IDXST along axis 0 (mode 1) swaps the two rows' roles for pairs
      if (imode == 1 && P != 0) {
        const T* tmp = rowA;
        rowA = rowB;
        rowB = tmp;
      }
      // operands of item kk (n2 in {kk, M-kk}): {DA, RA, DB, RB} per n2
      auto load_ops = [&](int kk, T* o) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int nn = u ? M - kk : kk;
          const bool z = nn == 0;
          const int pd = imode == 2 ? n2 - nn : nn;
          const int pr = imode == 2 ? nn : n2 - nn;
          const bool zd = imode == 2 && z;
          o[4 * u + 0] = zd ? T(0) : rowA[pd & (n2 - 1)];
          o[4 * u + 1] = z ? T(0) : rowA[pr & (n2 - 1)];
          o[4 * u + 2] = zd ? T(0) : rowB[pd & (n2 - 1)];
          o[4 * u + 3] = z ? T(0) : rowB[pr & (n2 - 1)];
        }
      };
      // items kk = t + i NT < M/2 in registers; the one left, kk = M/2 (its
      // own mirror), goes through a per-group stash so it costs no registers
      constexpr int NIM = (M / 2) / NT;
      T op[NIM][8];
#pragma unroll
      for (int i = 0; i < NIM; ++i) load_ops(t + i * NT, op[i]);
      T* stash = reinterpret_cast<T*>(smem_raw + G::STASH) + grp * 8;
      if (t == 0) {
        T ox[8];
        load_ops(M / 2, ox);
#pragma unroll
        for (int c = 0; c < 8; ++c) stash[c] = ox[c];
      }
      const V* ta = static_cast<const V*>(a.ta);
      const V* fb = static_cast<const V*>(a.fb);
      const V* fu = static_cast<const V*>(a.fu);
      const V ca0 = cconj(__ldg(ta + q1)), ca1 = cconj(__ldg(ta + m1));
      TL::sync();  // operands read: the buffer becomes the packed spectrum
      if constexpr (MODE == 2) {
        if (t == 0 && nxt < nitems) {
          fence_async_smem();
          issue_a(nxt);  // the next item's row A streams in under this item's math
        }
      }
      // X'(line, n2) from o = {DA, RA, DB, RB} (proj/src/dct2d.cpp:182-195)
      auto xp = [&](const T* o, V cb, V& x0, V& x1) {
        const V c0 = cmul(ca0, cb), c1 = cmul(ca1, cb);
        if (P == 0) {
          // rows 0 and N1/2, each its own mirror: row 0 pairs with the zero
          // row N1; mode 1 zeroes row 0 entirely
          const T pa = imode == 1 ? T(0) : o[0], sa = imode == 1 ? T(0) : o[1];
          x0 = cmul(c0, mk(pa, -sa));
          x1 = cmul(c1, mk(o[2] - o[3], -(o[2] + o[3])));
          return;
        }
        const T p = o[0], sv = o[1], r = o[2], q = o[3];
        x0 = cmul(c0, mk(p - q, -(r + sv)));
        x1 = cmul(c1, mk(r - sv, -(p + q)));
      };
      // packed spectrum of item kk at natural slots sa (k) and sb (M - k) of line 0
      auto pack_item = [&](int kk, const T* o, int sa, int sb) {
        V A0, A1, B0, B1;  // X'(line, k), X'(line, M-k)
        V bk = fac_lookup(fb, kk, a.fs), bm = mirror_b(bk);
        if (a.badq && a.badq[kk]) bk = mk(-bk.x, -bk.y);
        if (a.badq && a.badq[M - kk]) bm = mk(-bm.x, -bm.y);
        xp(o, cconj(bk), A0, A1);
        xp(o + 4, cconj(bm), B0, B1);
        // partner line of each row (-k1): swap for pairs, self for P == 0
        const V pA0 = P != 0 ? A1 : A0, pA1 = P != 0 ? A0 : A1;
        const V pB0 = P != 0 ? B1 : B0, pB1 = P != 0 ? B0 : B1;
        const V wk = fac_lookup(fu, kk, a.fs), wmk = mk(-wk.x, wk.y);  // W_N2^k, W_N2^{M-k}
        sm[sa] = pack(A0, kk == 0 ? B0 : cconj(pB0), wk);
        sm[sa ^ TL::swzc(M)] = pack(A1, kk == 0 ? B1 : cconj(pB1), wk);
        if (kk != 0 && 2 * kk != M) {
          sm[sb] = pack(B0, cconj(pA0), wmk);
          sm[sb ^ TL::swzc(M)] = pack(B1, cconj(pA1), wmk);
        }
      };
#pragma unroll
      for (int i = 0; i < NIM; ++i) {
        const int sa = sw_t ^ TL::swzc(i * NT);  // natural slot of k = t + i NT in line 0
        const int sb = t ? (sw_nt ^ TL::swzc(M - (i + 1) * NT)) : TL::swzc((M - i * NT) & (M - 1));  // slot of M - k
        pack_item(t + i * NT, op[i], sa, sb);
      }
      if (t == 0) {
        T ox[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) ox[c] = stash[c];
        pack_item(M / 2, ox, TL::swzc(M / 2), 0);
      }
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);
      TL::sync();
      from_smem<TL, 0>(v, sm, t);
      fft_regs<TL, true>(v, sm, tw, w0, t);
      TL::sync();
      last_to_natural<TL>(v, sm, t);
      TL::sync();
      // store rows (natural row order) in pair-interleaved column order
      V* dst = static_cast<V*>(a.dst) + batch * a.dst_batch;
      constexpr int CPV = 16 / sizeof(V);
      constexpr int VPR = M / CPV;
      const int irow[2] = {__ldg(a.s0 + q1), __ldg(a.s0 + m1)};
      // column s of the pair-interleaved row holds z(m), m = (s >> 1) ^ ((s & 1) (M - 1));
      // m is GF(2)-linear in s, so with the linear swizzle each element's slot is
      // one per-thread swizzle XOR a compile-time offset
      const int swt = CPV == 1 ? TL::swz((t >> 1) ^ ((t & 1) ? M - 1 : 0)) : TL::swz(t);
#pragma unroll
      for (int it = 0; it < 2 * VPR / NT; ++it) {
        const int line = (it * NT) / VPR, off = (it * NT) % VPR;
        V4 o;
        V* e = reinterpret_cast<V*>(&o);
        if constexpr (CPV == 1) {
          e[0] = sm[swt ^ TL::swzc(line * M + off / 2)];
        } else {
#pragma unroll
          for (int c = 0; c < CPV; ++c) e[c] = sm[swt ^ TL::swzc(line * M + off) ^ (c ? TL::swzc(M - 1) : 0)];
        }
        *reinterpret_cast<V4*>(dst + static_cast<long long>(irow[line]) * M + (t + off) * CPV) = o;
      }
    }
    TL::sync();  // every read of buffer b by this group is done
    if (t == 0) {
      if constexpr (MODE == 2) {
        if (nxt < nitems) {
          fence_async_smem();
          issue_b(nxt);
        }
      } else {
        mbar_arrive(empty + b);
        const int nxt0 = it + NBUF * static_cast<int>(gridDim.x);
        if (nxt0 < nitems) {
          fence_async_smem();  // generic-proxy smem accesses before the async refill
          issue(nxt0, b);
        }
      }
    }
  }
}

}  // namespace sdctb
