// Persistent cluster-pair column kernel for the 2D axis-0 passes with L = 2H
// = 4096 rows (fp64 4096^2 and taller batches): a 4096-row band (128 KB at
// fp64) no longer sits in one CTA; each half-band (64 KB) does, so two CTAs
// run per SM and their phases interleave (tools/microbench_band.cu: 64 KB
// tiles at several CTAs per SM move 32-B band rows at 5.0 TB/s, 128 KB tiles
// at one CTA per SM at 4.0 TB/s).
//
// Radix-2 split taken so that only half of the data crosses the pair, after
// the half-length FFTs and asynchronously (st.async into the peer's shared
// memory, completion counted on the peer's mbarrier):
//
//   forward (decimation in time): CTA c holds the reordered source rows
//     x'(2m + c), m < H — source rows of residue classes {0, 3} (c = 0) or
//     {2, 1} (c = 1) mod 4, landed by one 5D class map (pe(2m) = 4m or
//     2L-1-4m, pe(2m+1) = 4m+2 or 2L-3-4m; proj/include/sdct/dct1d.hpp:70-72)
//     — and runs the H-point DIF FFT of its half: E(k) (c = 0) or O(k). The
//     last radix-8 stage leaves thread t with butterflies b0 = t/2 and
//     b1 = b0 + H/16 of one line, in both CTAs for the same frequencies.
//     CTA c combines butterfly b_c: X(k) = E(k) + W_L^k O(k),
//     X(k+H) = E(k) - W_L^k O(k); it sends its other butterfly's 8 values
//     (E, or W_L^k O) to the peer and receives the peer's.
//   inverse (decimation in frequency): CTA c loads the intermediate rows of
//     its own butterflies b_c, X(k) and X(k+H), forms A(k) = X(k) + X(k+H),
//     B(k) = (X(k) - X(k+H)) W_L^-k, keeps A (c = 0) or B (c = 1) and sends
//     the other; then runs the H-point inverse DIT: x'(2m) from A, x'(2m+1)
//     from B; the final gather (1/4 scale, signs, lane-pair unpacking,
//     proj/src/dct2d.cpp:214-238) lands on y rows of the same residue classes.
//
// Intermediate row of frequency k (the plan's srow table): k = k' + hf H,
// slot n = digit_pos_H(k') = 8b + r -> row hf H + (b / (H/16)) (H/2)
// + r (H/16) + b mod (H/16): each CTA's outputs (resp. inputs) are two
// contiguous blocks of H/2 rows, lanes with consecutive b hit consecutive rows.
//
// Per CTA: landing / FFT exchange / store staging tile (64 KB) + receive
// buffer (32 KB), two CTAs per SM. The receive buffer is handed back to the
// peer right after the combine reads it; the next tile lands in the tile
// buffer once the stores have read the staging (the SM's other CTA covers the
// load latency).
#pragma once

#include "kernels_rowp.cuh"  // rowp_sw: compile-time twiddle steps

namespace sdctb {

template <typename T, int H, int NL>
struct ColcGeom {
  using TL = Tile<T, H, NL, true>;
  static constexpr int NT = TL::NT;
  static constexpr uint32_t TILE = static_cast<uint32_t>(H) * 2 * NL * sizeof(T);  // 64 KB (fp64, H 2048, NL 2)
  static constexpr uint32_t RECV = TILE / 2;                                     // peer's half of the combine
  static constexpr size_t BAR_OFF = TILE + RECV;
  static constexpr size_t SMEM = BAR_OFF + 64;
};

template <int H>
constexpr bool colc_shape_ok() {
  return H == 2048;
}

template <typename T, int H, int NL, bool INV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ColcGeom<T, H, NL>::NT, 2)
    colc_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ColArgs a,
                TwSet tw) {
  using G = ColcGeom<T, H, NL>;
  using TL = typename G::TL;
  using P = typename TL::P;
  using V = cx_t<T>;
  using V2 = typename Vec2<T>::type;
  constexpr int NT = TL::NT;
  constexpr int S = TL::S, SL = S - 1;
  constexpr int R0 = TL::R0, Q0 = H / R0, NBF0 = TL::E / R0;
  constexpr int RL = P::R(SL), NBFL = TL::E / RL;
  constexpr int NB2 = H / 16;  // butterflies b per CTA half (b in [0, H/8))
  constexpr int BLK = H / 2;   // rows per CTA block of the intermediate
  constexpr int BOX = 256;
  static_assert(colc_shape_ok<H>() && NBF0 == 1 && RL == 8 && NBFL == 2 && NT == 2 * NB2 && NL == 2,
                "cluster-pair column kernel: H = 2048, NL = 2 geometry");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  V* rb = reinterpret_cast<V*>(smem_raw + G::TILE);  // receive, then staging
  uint64_t* bar_land = reinterpret_cast<uint64_t*>(smem_raw + G::BAR_OFF);
  uint64_t* bar_recv = bar_land + 1;
  uint64_t* bar_ok = bar_land + 2;  // the peer's receive buffer is free again
  const int t = threadIdx.x;
  const int c = static_cast<int>(cluster_rank());
  const int cl = static_cast<int>(blockIdx.x) >> 1, ncl = static_cast<int>(gridDim.x) >> 1;
  const V* twl = static_cast<const V*>(a.twc);  // W_L^n, n < H
  const uint32_t peer_rb = mapa(smem_u32(rb), static_cast<uint32_t>(c ^ 1));
  const uint32_t peer_recv = mapa(smem_u32(bar_recv), static_cast<uint32_t>(c ^ 1));
  const uint32_t peer_ok = mapa(smem_u32(bar_ok), static_cast<uint32_t>(c ^ 1));
  const int line = t & 1, b0 = t >> 1;  // last-stage butterflies b0 and b0 + NB2, both of line `line`

  auto coords = [&](int tile, int& band, int& batch) {
    band = tile % a.nbands;
    batch = tile / a.nbands;
  };
  auto issue = [&](int tile) {  // thread 0
    int band, batch;
    coords(tile, band, batch);
    mbar_expect_tx(bar_land, G::TILE);
    if constexpr (!INV) {
      // residue classes c0 = {0, 2}[c] (m ascending) and c1 = {3, 1}[c] (m descending)
      const int cls0 = c ? 2 : 0, cls1 = c ? 1 : 3;
#pragma unroll 1
      for (int q0 = 0; q0 < BLK; q0 += BOX) {
        tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(q0) * 2 * NL, &tin, band * 2 * NL, cls0, q0, 0,
                    batch, bar_land);
        tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(BLK + q0) * 2 * NL, &tin, band * 2 * NL, cls1,
                    q0, 0, batch, bar_land);
      }
    } else {
      // own blocks: X(k) rows c*BLK + [0, BLK), X(k+H) rows H + c*BLK + [0, BLK)
#pragma unroll 1
      for (int r0 = 0; r0 < BLK; r0 += BOX) {
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(r0) * 2 * NL, &tin, band * 2 * NL,
                    c * BLK + r0, 0, batch, bar_land);
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(BLK + r0) * 2 * NL, &tin, band * 2 * NL,
                    H + c * BLK + r0, 0, batch, bar_land);
      }
    }
  };

  if (t == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
    mbar_init(bar_land, 1);
    mbar_init(bar_recv, 1);
    mbar_init(bar_ok, 1);
  }
  __syncthreads();
  cluster_sync();  // both CTAs' barriers exist before any peer operation
  pdl_trigger();
  pdl_wait();
  const int first = cl;
  if (t == 0) {
    mbar_expect_tx(bar_recv, G::RECV);  // armed for the first exchange
    if (first < a.ntiles) issue(first);
  }
  uint32_t ph_land = 0, ph_recv = 0, ph_ok = 0;

#pragma unroll 1
  for (int tile = first, k = 0; tile < a.ntiles; tile += ncl, ++k) {
    int band, batch;
    coords(tile, band, batch);
    const bool more = tile + ncl < a.ntiles;
    V v[TL::E];
    // twiddles: butterfly b holds k = k0(b) + (H/8) r with k0(b) = digit_rev(8b),
    // so W_L^k = W_L^k0 e^{-i pi r / 8}

    if constexpr (!INV) {
      // ============================== forward ===============================
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);
      mbar_wait(bar_land, ph_land);
      ph_land ^= 1;
      {
        // slot m (H-point sequence of this CTA) sits at landed row m (m < H/2)
        // or H/2 + (H-1-m); lane pair (h = 0, 1) packs z(u) = (x0, x2), z(M-1-u) = (x3, x1)
        const V2* raw = reinterpret_cast<const V2*>(smem_raw);
        const int j = t >> 1, h = line;
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int m = j + r * Q0;
          const int row = (r < R0 / 2) ? m : H / 2 + (H - 1 - m);
          const V2 x = raw[row * NL + line];
          const T send = h ? x.x : x.y;
          const T recv = __shfl_xor_sync(0xffffffffu, send, 1);
          v[r] = h ? mk(x.y, recv) : mk(x.x, recv);
        }
      }
      __syncthreads();  // landed rows consumed: the tile becomes the FFT exchange buffer
      StageTw<TL, SL> wl;
      stage_compute<TL, 0, false>(v, w0);
      to_smem<TL, 0>(v, sm, t);
      __syncthreads();
      stages_until_last<TL, false, 1>(v, sm, tw, t, wl);
      __syncthreads();  // last-stage operands in registers: the tile buffer is free
      stage_compute<TL, SL, false>(v, wl);
      // v[i*8 + r] = F(k(b_i, r)), b_0 = b0, b_1 = b0 + NB2 (F = E for c = 0, O for c = 1)
      if (c == 1) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const V tb = __ldg(twl + digit_rev<H>(8 * (b0 + i * NB2)));
#pragma unroll
          for (int r = 0; r < 8; ++r) v[i * 8 + r] = cmul(v[i * 8 + r], cmul(tb, rowp_sw<T>(r)));
        }
      }
      // send the peer's half (butterfly 1 - c) into its receive buffer
      if (k > 0) {
        mbar_wait_cluster(bar_ok, ph_ok);
        ph_ok ^= 1;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        st_async(peer_rb + static_cast<uint32_t>((r * NT + t) * sizeof(V)), c == 0 ? v[8 + r] : v[r], peer_recv);
      mbar_wait_cluster(bar_recv, ph_recv);
      ph_recv ^= 1;
      V lo[8], hi[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const V pv = rb[r * NT + t];
        const V e = c == 0 ? v[r] : pv;            // E(k)
        const V wo = c == 0 ? pv : v[8 + r];       // W^k O(k)
        lo[r] = cadd(e, wo);                       // X(k)
        hi[r] = csub(e, wo);                       // X(k + H)
      }
      __syncthreads();  // receive buffer read
      if (t == 0 && more) {  // free for the next exchange: arm it and tell the peer
        mbar_expect_tx(bar_recv, G::RECV);
        mbar_arrive_remote(peer_ok);
      }
      // all 64 KB of outputs staged in the tile buffer: X(k) block at rows
      // r NB2 + b0, X(k+H) block BLK further (line-interleaved 32-B rows)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        sm[(r * NB2 + b0) * NL + line] = lo[r];
        sm[(BLK + r * NB2 + b0) * NL + line] = hi[r];
      }
      fence_async_smem();
      __syncthreads();
      if (t == 0) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half)
#pragma unroll 1
          for (int r0 = 0; r0 < BLK; r0 += BOX)
            tma_store_4d(&tout, band * 2 * NL, half * H + c * BLK + r0, 0, batch,
                         reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(half * BLK + r0) * 2 * NL);
        bulk_commit();
        if (more) {  // the next tile lands once the stores have read the staging
          bulk_wait_read();
          issue(tile + ncl);
        }
      }
    } else {
      // ============================== inverse ===============================
      mbar_wait(bar_land, ph_land);
      ph_land ^= 1;
      // own butterfly b_c = b0 + c NB2: X(k) at tile row r NB2 + b0, X(k+H) at BLK + r NB2 + b0
      {
        const V tb = __ldg(twl + digit_rev<H>(8 * (b0 + c * NB2)));
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const V x0 = sm[(r * NB2 + b0) * NL + line], x1 = sm[(BLK + r * NB2 + b0) * NL + line];
          // own butterfly b_c: A to slot r, B to slot 8 + r (c = 0 keeps A and
          // sends B, c = 1 keeps B and sends A)
          v[r] = cadd(x0, x1);
          v[8 + r] = cmulc(csub(x0, x1), cmul(tb, rowp_sw<T>(r)));  // (X(k) - X(k+H)) W_L^-k
        }
      }
      if (k > 0) {
        mbar_wait_cluster(bar_ok, ph_ok);
        ph_ok ^= 1;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        st_async(peer_rb + static_cast<uint32_t>((r * NT + t) * sizeof(V)), c == 0 ? v[8 + r] : v[r], peer_recv);
      mbar_wait_cluster(bar_recv, ph_recv);
      ph_recv ^= 1;
      // the peer's A (c = 0: butterfly b1) or B (c = 1: butterfly b0)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const V pv = rb[r * NT + t];
        if (c == 0) v[8 + r] = pv;
        else v[r] = pv;
      }
      __syncthreads();  // landed rows and the receive buffer consumed
      if (t == 0 && more) {  // receive buffer free: arm the next exchange, tell the peer
        mbar_expect_tx(bar_recv, G::RECV);
        mbar_arrive_remote(peer_ok);
      }
      // H-point inverse DIT of A (c = 0) / B (c = 1): input slot 8b + r of butterfly b
      StageTw<TL, SL> wl;  // first DIT stage: no twiddles
      dit_compute<TL, SL, true>(v, wl);
      to_smem<TL, SL>(v, sm, t);
      __syncthreads();
      dit_down<TL, true, SL - 1>(v, sm, tw, t);  // stage 0 in registers: x'(2m + c), m = j + Q0 r
      __syncthreads();  // all exchange reads done: the tile buffer becomes the staging
      // final gather to y row pe(2m + c): m < H/2 -> class {0, 2}[c], pair m
      // (staging rows [0, BLK)); m >= H/2 -> class {3, 1}[c] (odd rows), pair
      // H-1-m (staging rows BLK + pair)
      const T sc = static_cast<T>(a.scale);
      const int j = t >> 1, h = line;
      V2* sv = reinterpret_cast<V2*>(smem_raw);
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int half = r >= R0 / 2 ? 1 : 0;
        const T s0 = (a.sign_row && half) ? -sc : sc;
        const T s1 = a.sign_col ? -s0 : s0;
        const int m = j + r * Q0;
        const int p = half ? BLK + (H - 1 - m) : m;
        const V z = v[r];
        const T recv = __shfl_xor_sync(0xffffffffu, z.y, 1);
        // h=0: (Re z(u), Im z(M-1-u)) = y(4u, 4u+1); h=1: (Im z(u), Re z(M-1-u)) = y(4u+2, 4u+3)
        sv[p * NL + line] = h ? V2{recv * s0, z.x * s1} : V2{z.x * s0, recv * s1};
      }
      fence_async_smem();
      __syncthreads();
      if (t == 0) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int cls = half ? (c ? 1 : 3) : (c ? 2 : 0);
#pragma unroll 1
          for (int r0 = 0; r0 < BLK; r0 += BOX)
            tma_store_5d(&tout, band * 2 * NL, cls, r0, 0, batch,
                         reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(half * BLK + r0) * 2 * NL);
        }
        bulk_commit();
        if (more) {  // the next tile lands once the stores have read the staging
          bulk_wait_read();
          issue(tile + ncl);
        }
      }
    }
  }
  if (t == 0) bulk_wait_all();
  cluster_sync();  // no peer operation may target an exited CTA
}

}  // namespace sdctb
