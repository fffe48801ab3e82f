// One-dimensional DCT-II / DCT-III along axis 0 of a row-major (n1 x m)
// matrix, i.e. the reference's dct_1d / idct_1d (proj/src/dct1d.cpp, the
// N-point scheme; oracle: sdct_oracle_dct_direct_1d / idct_direct_1d) applied
// to every column, as one persistent column pass. This is the axis-0 leg of
// the slab-decomposed 3D transform (slab3d.py): after the
// all-to-all, a rank holds [src][i_loc][j_loc][k] = an (n1 x s2 n3) matrix
// whose axis-0 DCT this kernel takes in place of a transpose, a contiguous
// 1D transform and a transpose back.
//
// A tile is a band of NL complex columns (32-B rows) x all L rows; each
// complex line packs two adjacent real columns (c, c+1) as real and
// imaginary part, so one complex FFT per line transforms both.
//   forward: rows land by parity class (the axis-0 reorder x'(n) = x(pe(n)),
//     proj/include/sdct/dct1d.hpp:70-72) -> L-point DIF FFT -> natural order
//     in shared memory -> unpack X_c = (Z(k) + conj Z(-k))/2,
//     X_c+1 = (Z(k) - conj Z(-k))/2i -> y(k) = Re(a(k) X(k)),
//     a(k) = e^{-i pi k / 2L}, y(L-k) from conj X(k) -> two half-tile stores.
//   inverse: natural rows land -> X'(k) = conj a(k) (x(k) - i x(L-k)),
//     x(L) := 0, packed as X'_c + i X'_c+1 straight into the DIT input
//     layout -> L-point DIT -> y(pe(n)) = z(n) / 2 (real / imaginary part =
//     the two columns), stored through the even / odd row-class map.
#pragma once

#include "kernels_fast.cuh"

namespace sdctb {

template <typename T, int L, int NL>
struct Col1dGeom {
  using TL = Tile<T, L, NL, true>;
  static constexpr uint32_t TILE = static_cast<uint32_t>(L) * 2 * NL * sizeof(T);
  static constexpr uint32_t STG_OFF = (TILE + 127u) & ~127u;
  static constexpr uint32_t BAR_OFF = (STG_OFF + TILE / 2 + 127u) & ~127u;
  static constexpr size_t SMEM = BAR_OFF + 16;
};

template <typename T, int L, int NL, bool INV>
__global__ void __launch_bounds__(Tile<T, L, NL, true>::NT)
    col1d_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, ColArgs a,
                 TwSet tw) {
  using G = Col1dGeom<T, L, NL>;
  using TL = typename G::TL;
  using P = typename TL::P;
  using V = cx_t<T>;
  constexpr int NT = TL::NT;
  constexpr int S = TL::S, SL = S - 1;
  constexpr int R0 = TL::R0, Q0 = L / R0, NBF0 = TL::E / R0;
  constexpr int RL = P::R(SL), NBFL = TL::E / RL;
  constexpr int H = L / 2;
  constexpr int BOX = H < 256 ? H : 256;
  static_assert(L >= 4 && col_class_load(sizeof(T), L, NL), "axis-0 pass: class-aligned tiles");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  V* stg = reinterpret_cast<V*>(smem_raw + G::STG_OFF);  // half tile: H rows of NL complex
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::BAR_OFF);
  const int t = threadIdx.x;
  const V* qa = static_cast<const V*>(a.twc);  // a(k) = e^{-i pi k / 2L}, k < L

  auto coords = [&](int tile, int& band, int& batch) {
    band = tile % a.nbands;
    batch = tile / a.nbands;
  };
  auto issue = [&](int tile) {  // thread 0
    int band, batch;
    coords(tile, band, batch);
    mbar_expect_tx(bar, G::TILE);
#pragma unroll 1
    for (int p0 = 0; p0 < H; p0 += BOX) {
      if constexpr (!INV) {  // even rows 2p -> smem row p, odd rows 2p+1 -> H + p (class map)
        tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(p0) * 2 * NL, &tin, band * 2 * NL, 0, p0, 0,
                    batch, bar);
        tma_load_5d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(H + p0) * 2 * NL, &tin, band * 2 * NL, 1, p0,
                    0, batch, bar);
      } else {  // natural rows
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(p0) * 2 * NL, &tin, band * 2 * NL, p0, 0,
                    batch, bar);
        tma_load_4d(reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(H + p0) * 2 * NL, &tin, band * 2 * NL, H + p0,
                    0, batch, bar);
      }
    }
  };
  // natural-order slot of frequency / sample index k of line `line` (swizzled tile layout)
  auto nat = [&](int line, int k) { return TL::swz(TL::raw(line, k)); };

  if (t == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tout);
    mbar_init(bar, 1);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (t == 0 && static_cast<int>(blockIdx.x) < a.ntiles) issue(blockIdx.x);
  uint32_t phase = 0;

#pragma unroll 1
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    int band, batch;
    coords(tile, band, batch);
    const bool more = tile + static_cast<int>(gridDim.x) < a.ntiles;
    V v[TL::E];
    if constexpr (!INV) {
      // ================================ forward =============================
      StageTw<TL, 0> w0;
      w0.load(tw.st[0], t);
      mbar_wait(bar, phase);
      phase ^= 1;
#pragma unroll
      for (int i = 0; i < NBF0; ++i) {
        const int bf = t + i * NT;
        const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int n = j + r * Q0;  // slot n reads x(pe(n)): landed row n (n < H) or H + (L-1-n)
          const int row = (r < R0 / 2) ? n : H + (L - 1 - n);
          v[i * R0 + r] = sm[row * NL + line];  // (x(., 2l), x(., 2l+1)) packed as one complex value
        }
      }
      __syncthreads();
      StageTw<TL, SL> wl;
      if constexpr (S == 1) {
        wl = w0;
      } else {
        stage_compute<TL, 0, false>(v, w0);
        to_smem<TL, 0>(v, sm, t);
        __syncthreads();
        stages_until_last<TL, false, 1>(v, sm, tw, t, wl);
      }
      __syncthreads();  // last-stage operands in registers
      stage_compute<TL, SL, false>(v, wl);
      // Z(k) in natural order: slot n of butterfly (line, b) holds k = digit_rev(n)
#pragma unroll
      for (int i = 0; i < NBFL; ++i) {
        int line, b;
        last_decode<TL>(t + i * NT, line, b);
#pragma unroll
        for (int r = 0; r < RL; ++r) sm[nat(line, digit_rev<L>(b * RL + r))] = v[i * RL + r];
      }
      __syncthreads();
      // unpack + postprocess: item (line, k), k in [0, H]; round 0 stores rows
      // k < H, round 1 rows L-k (k >= 1) and H
#pragma unroll 1
      for (int round = 0; round < 2; ++round) {
        if (round == 1) {
          if (t == 0) bulk_wait_read();
          __syncthreads();
        }
#pragma unroll 1
        for (int it = t; it < (H + 1) * NL; it += NT) {
          const int line = it & (NL - 1), k = it >> TL::LGNL;
          const V zk = sm[nat(line, k)], zm = sm[nat(line, (L - k) & (L - 1))];
          // X_c = (Z(k) + conj Z(-k)) / 2, X_c+1 = (Z(k) - conj Z(-k)) / 2i
          const V xa = mk(T(0.5) * (zk.x + zm.x), T(0.5) * (zk.y - zm.y));
          const V xb = mk(T(0.5) * (zk.y + zm.y), T(0.5) * (zm.x - zk.x));
          if (round == 0) {
            if (k < H) {
              const V ak = __ldg(qa + k);
              stg[k * NL + line] = mk(ak.x * xa.x - ak.y * xa.y, ak.x * xb.x - ak.y * xb.y);  // Re(a X)
            }
          } else if (k >= 1) {
            // y(L-k) = Re(a(L-k) conj X(k)); k = H: its own mirror (X(H) is real-symmetric)
            const V am = __ldg(qa + (L - k));
            stg[(L - k - H) * NL + line] = mk(am.x * xa.x + am.y * xa.y, am.x * xb.x + am.y * xb.y);
          }
        }
        fence_async_smem();
        __syncthreads();
        if (round == 1 && t == 0 && more) {  // the tile buffer's Z has been read: land the next tile
          fence_async_smem();
          issue(tile + gridDim.x);
        }
        if (t == 0) {
#pragma unroll 1
          for (int p0 = 0; p0 < H; p0 += BOX)
            tma_store_4d(&tout, band * 2 * NL, round * H + p0, 0, batch,
                         reinterpret_cast<T*>(stg) + static_cast<size_t>(p0) * 2 * NL);
          bulk_commit();
        }
      }
    } else {
      // ================================ inverse =============================
      StageTw<TL, SL> wl;  // first DIT stage: no twiddles
      mbar_wait(bar, phase);
      phase ^= 1;
      // DIT input placement: slot n of butterfly (line, b) takes frequency digit_rev(n)
#pragma unroll
      for (int i = 0; i < NBFL; ++i) {
        int line, b;
        last_decode<TL>(t + i * NT, line, b);
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int k = digit_rev<L>(b * RL + r);
          const V xk = sm[k * NL + line];                                   // (x_c(k), x_c+1(k))
          const V xm = k ? sm[(L - k) * NL + line] : mk(T(0), T(0));        // x(L - k), x(L) := 0
          const V ck = cconj(__ldg(qa + k));
          const V pa = cmul(ck, mk(xk.x, -xm.x));                           // X'_c(k)
          const V pb = cmul(ck, mk(xk.y, -xm.y));                           // X'_c+1(k)
          v[i * RL + r] = mk(pa.x - pb.y, pa.y + pb.x);                     // X'_c + i X'_c+1
        }
      }
      __syncthreads();  // landed rows consumed
      dit_compute<TL, SL, true>(v, wl);
      if constexpr (S > 1) {
        to_smem<TL, SL>(v, sm, t);
        __syncthreads();
        dit_down<TL, true, SL - 1>(v, sm, tw, t);  // stage 0 in registers: natural n = j + Q0 r
      }
      __syncthreads();  // all exchange reads done: the tile buffer is free
      if (t == 0 && more) {
        fence_async_smem();
        issue(tile + gridDim.x);
      }
      // y(pe(n)) = z(n) / 2: n < H -> even row 2n (class 0, pair n), else odd
      // row 2L-1-2n (class 1, pair L-1-n)
      const T sc = static_cast<T>(a.scale);
#pragma unroll 1
      for (int cls = 0; cls < 2; ++cls) {
        if (cls == 1) {
          if (t == 0) bulk_wait_read();
          __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < NBF0; ++i) {
          const int bf = t + i * NT;
          const int line = bf & (NL - 1), j = bf >> TL::LGNL;
#pragma unroll
          for (int r = 0; r < R0; ++r) {
            const int n = j + r * Q0;
            if ((n >= H) == (cls == 1)) {
              const int p = cls ? L - 1 - n : n;
              stg[p * NL + line] = mk(v[i * R0 + r].x * sc, v[i * R0 + r].y * sc);
            }
          }
        }
        fence_async_smem();
        __syncthreads();
        if (t == 0) {
#pragma unroll 1
          for (int p0 = 0; p0 < H; p0 += BOX)
            tma_store_5d(&tout, band * 2 * NL, cls, p0, 0, batch, reinterpret_cast<T*>(stg) + static_cast<size_t>(p0) * 2 * NL);
          bulk_commit();
        }
      }
    }
    if (t == 0) bulk_wait_read();  // the staging is reused by the next tile
    __syncthreads();
  }
  if (t == 0) bulk_wait_all();
}

}  // namespace sdctb
