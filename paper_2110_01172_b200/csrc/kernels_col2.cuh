// Cluster-split column kernels for long columns (L = 2H), 2D transforms: the
// only fast column pass for L = 8192 (a whole band would not fit one SM's
// shared memory), and an opt-in alternative for fp64 L = 4096.
//
// A whole 4096-row band of a 2D transform (4096 rows x 32 B = 128 KB) only
// fits one CTA per SM, and then the band's load, math and stores serialise
// (tools/microbench_band.cu: 128 KB tiles cap the band movement at 4.0 TB/s,
// 64 KB tiles reach 5.0 TB/s with several CTAs per SM). Here a band is split
// over a 2-CTA cluster, one 64 KB half per CTA, two clusters' CTAs per SM:
//
//   forward (DIF): CTA c holds the slots n in [cH, cH+H) (source rows of
//     parity class c: slot n reads row pe(n), proj/include/sdct/dct1d.hpp:70-72).
//     The first radix-2 DIF stage pairs slot n with n+H across the cluster
//     over DSMEM: CTA 0 keeps a(n) = x(n) + x(n+H), CTA 1 keeps
//     b(n) = (x(n) - x(n+H)) W_L^n; each then runs the H-point DIF FFT
//     (the register-resident tile engine) on its half and so owns the even
//     (c = 0) or odd (c = 1) frequencies k = 2k' + c. Output rows
//     c*H + sigma_H(slot of k') of the intermediate (the row kernels find
//     them through the plan's srow table).
//   inverse (DIT): CTA c loads the frequencies k = 2k' + c (its intermediate
//     rows), runs the H-point inverse DIT to A_c(n), exchanges over DSMEM and
//     combines y(n) = A0(n) + W_L^-n A1(n), y(n+H) = A0(n) - W_L^-n A1(n);
//     CTA c then writes the final gather of rows pe(n + cH) = the rows of
//     parity class c (1/4 scale and signs, proj/src/dct2d.cpp:214-238).
//
// The same arithmetic as col_kernel with L = 4096 otherwise (packing, parity
// maps, pair-interleaved intermediate columns).
#pragma once

#include "kernels_fast.cuh"

namespace sdctb {

template <typename T, int H, int NL>
struct Col2Geom {
  using TL = Tile<T, H, NL, true>;
  static constexpr int NT = TL::NT;
  static constexpr uint32_t TILE = static_cast<uint32_t>(H) * 2 * NL * sizeof(T);  // 64 KB for fp64 H=2048 NL=2
  static constexpr size_t SMEM = TILE + 64;                                      // + mbarrier
  static constexpr int MINB = TILE <= 100u * 1024u ? 2 : 1;                      // CTAs per SM
};

template <typename T, int H, int NL, bool INV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Col2Geom<T, H, NL>::NT, Col2Geom<T, H, NL>::MINB)
    col2_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ColArgs a,
                TwSet tw) {
  using G = Col2Geom<T, H, NL>;
  using TL = typename G::TL;
  using P = typename TL::P;
  using V = cx_t<T>;
  using V2 = typename Vec2<T>::type;
  constexpr int L = 2 * H;
  constexpr int NT = TL::NT;
  constexpr int S = TL::S, SL = S - 1;
  constexpr int R0 = TL::R0, Q0 = H / R0, NBF0 = TL::E / R0;
  constexpr int RL = P::R(SL), NBFL = TL::E / RL;
  constexpr int BOX = H < 256 ? H : 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::TILE);
  const int t = threadIdx.x;
  const int c = static_cast<int>(cluster_rank());
  const int band = static_cast<int>(blockIdx.x) >> 1;
  const int batch = blockIdx.y;
  const V* twl = static_cast<const V*>(a.twc);  // W_L^n, n < H

  if (t == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
    mbar_init(bar, 1);
  }
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(bar, G::TILE);
#pragma unroll 1
    for (int r0 = 0; r0 < H; r0 += BOX) {
      if constexpr (!INV)  // rows 2p + c of the source: the class map {reals, class, pair, plane, batch}
        tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL, &tin, band * 2 * NL, c, r0, 0,
                    batch, bar);
      else  // intermediate rows cH + r
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL, &tin, band * 2 * NL,
                    c * H + r0, 0, batch, bar);
    }
  }
  mbar_wait(bar, 0);
  V v[TL::E];

  if constexpr (!INV) {
    // ====================== forward =====================================
    StageTw<TL, 0> w0;
    w0.load(tw.st[0], t);
    cluster_sync();  // both halves landed
    // slot n of CTA 0 = its row n; slot n + H of CTA 1 = its row H - 1 - n
    const uint32_t peer = mapa(smem_u32(smem_raw), static_cast<uint32_t>(c ^ 1));
    const V2* raw = reinterpret_cast<const V2*>(smem_raw);
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      const int bf = t + i * NT;
      const int line = bf & (NL - 1), j = bf >> TL::LGNL;
      const int h = line & 1;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        const int row0 = n, row1 = H - 1 - n;  // rows of x(n) in CTA 0 and of x(n + H) in CTA 1
        const int own_row = c ? row1 : row0, peer_row = c ? row0 : row1;
        const V2 xo = raw[own_row * NL + line];
        const V2 xp = ld_dsmem(peer + static_cast<uint32_t>((peer_row * NL + line) * sizeof(V2)), static_cast<V2*>(nullptr));
        // packing: lane pair (h = 0, 1) of quad g builds z(u) = (x0, x2), z(M-1-u) = (x3, x1)
        const T so = h ? xo.x : xo.y, sp = h ? xp.x : xp.y;
        const T ro = __shfl_xor_sync(TL::MASK, so, 1), rp = __shfl_xor_sync(TL::MASK, sp, 1);
        const V zo = h ? mk(xo.y, ro) : mk(xo.x, ro);
        const V zp = h ? mk(xp.y, rp) : mk(xp.x, rp);
        if (c == 0) {
          v[i * R0 + r] = cadd(zo, zp);  // a(n) = x(n) + x(n + H)
        } else {
          v[i * R0 + r] = cmul(csub(zp, zo), __ldg(twl + n));  // b(n) = (x(n) - x(n + H)) W_L^n
        }
      }
    }
    cluster_sync();  // the peer has read this CTA's half: the tile becomes the exchange buffer
    StageTw<TL, SL> wl;
    if constexpr (S == 1) {
      wl = w0;
    } else {
      stage_compute<TL, 0, false>(v, w0);
      to_smem<TL, 0>(v, sm, t);
      __syncthreads();
      stages_until_last<TL, false, 1>(v, sm, tw, t, wl);
    }
    __syncthreads();  // last-stage operands are in registers
    stage_compute<TL, SL, false>(v, wl);
    // slot n' = b*RL + r -> local row sigma(n') = b + (H/RL) r, stored densely for the TMA boxes
#pragma unroll
    for (int i = 0; i < NBFL; ++i) {
      int line, b;
      last_decode<TL>(t + i * NT, line, b);
#pragma unroll
      for (int r = 0; r < RL; ++r) sm[(b + (H / RL) * r) * NL + line] = v[i * RL + r];
    }
    fence_async_smem();
    __syncthreads();
    if (t == 0) {
#pragma unroll 1
      for (int r0 = 0; r0 < H; r0 += BOX)
        tma_store_4d(&tout, band * 2 * NL, c * H + r0, 0, batch, reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL);
      bulk_commit();
      bulk_wait_read();
    }
  } else {
    // ====================== inverse =====================================
    StageTw<TL, SL> wl;  // first DIT stage (S-1) has no twiddles
    {
      const V* raw = reinterpret_cast<const V*>(smem_raw);
#pragma unroll
      for (int i = 0; i < NBFL; ++i) {
        int line, b;
        last_decode<TL>(t + i * NT, line, b);
#pragma unroll
        for (int r = 0; r < RL; ++r) v[i * RL + r] = raw[(b + (H / RL) * r) * NL + line];
      }
    }
    __syncthreads();  // raw tile consumed
    dit_compute<TL, SL, true>(v, wl);
    if constexpr (S > 1) {
      to_smem<TL, SL>(v, sm, t);
      __syncthreads();
      dit_down<TL, true, SL - 1>(v, sm, tw, t);  // ends with stage 0 in registers
    }
    __syncthreads();  // all exchange reads done
    // A_c(n), n = j + r Q0; CTA 1 contributes B(n) = W_L^-n A1(n). Exchange in
    // the plain layout n*NL + line.
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      const int bf = t + i * NT;
      const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        if (c == 1) v[i * R0 + r] = cmulc(v[i * R0 + r], __ldg(twl + n));  // A1 W_L^-n
        sm[n * NL + line] = v[i * R0 + r];
      }
    }
    cluster_sync();  // both exchanges written
    const uint32_t peer = mapa(smem_u32(smem_raw), static_cast<uint32_t>(c ^ 1));
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      const int bf = t + i * NT;
      const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        const V o = ld_dsmem(peer + static_cast<uint32_t>((n * NL + line) * sizeof(V)), static_cast<V*>(nullptr));
        // CTA 0: y(n) = A0 + B; CTA 1: y(n + H) = A0 - B (own = B, peer = A0)
        v[i * R0 + r] = c == 0 ? cadd(v[i * R0 + r], o) : csub(o, v[i * R0 + r]);
      }
    }
    cluster_sync();  // the peer has read this CTA's exchange: the tile becomes the store staging
    // final gather: spatial index m = n + cH lands on y row pe(m), which is of
    // parity class c at pair p = n (c = 0) or H - 1 - n (c = 1); scale, signs,
    // and the lane-pair unpacking into the quad's four reals
    const T sc = static_cast<T>(a.scale);
    const T s0 = (a.sign_row && c) ? -sc : sc;  // k1 = pe(m) is odd exactly in class 1
    const T s1 = a.sign_col ? -s0 : s0;
    V2* sv = reinterpret_cast<V2*>(smem_raw);
#pragma unroll
    for (int i = 0; i < NBF0; ++i) {
      const int bf = t + i * NT;
      const int line = bf & (NL - 1), j = bf >> TL::LGNL;
      const int h = line & 1;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n = j + r * Q0;
        const int p = c ? H - 1 - n : n;
        const V z = v[i * R0 + r];
        const T recv = __shfl_xor_sync(TL::MASK, z.y, 1);
        // h=0: (Re z(u), Im z(M-1-u)) = y(4u, 4u+1); h=1: (Im z(u), Re z(M-1-u)) = y(4u+2, 4u+3)
        sv[p * NL + line] = h ? V2{recv * s0, z.x * s1} : V2{z.x * s0, recv * s1};
      }
    }
    fence_async_smem();
    __syncthreads();
    if (t == 0) {
#pragma unroll 1
      for (int r0 = 0; r0 < H; r0 += BOX)
        tma_store_5d(&tout, band * 2 * NL, c, r0, 0, batch, reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL);
      bulk_commit();
      bulk_wait_read();
    }
  }
}

}  // namespace sdctb
