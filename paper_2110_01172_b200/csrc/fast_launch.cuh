// Runtime -> compile-time dispatch for the fast-path kernels. Each dtype's
// column and row kernels are instantiated in their own translation unit
// (fast_col_f32.cu, fast_col_f64.cu, fast_row_f32.cu, fast_row_f64.cu) so the
// build compiles them in parallel.
#pragma once

#include "kernels_fast.cuh"

namespace sdctb {

constexpr int kMaxFastLen = 4096;  // largest FFT length with a fast kernel

template <typename T>
cudaError_t launch_col(int L, bool inv, int load, int store, dim3 grid, size_t smem, cudaStream_t st,
                       const ColArgs& a, const cx_t<T>* tw, int tw_step);
template <typename T>
cudaError_t launch_row(int M, int kind, dim3 grid, size_t smem, cudaStream_t st, const RowArgs& a,
                       const cx_t<T>* tw, int tw_step);

inline int col_threads_rt(int L) { return L >= 1024 ? 512 : 256; }

// Opt each kernel instantiation in to > 48 KB dynamic shared memory (once).
cudaError_t prep_smem_ptr(const void* kernel, size_t smem);
template <typename K>
inline cudaError_t prep_smem(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return prep_smem_ptr(reinterpret_cast<const void*>(kernel), smem);
}

#define SDCTB_COL_CASE(T, LL)                                                                   \
  case LL: {                                                                                    \
    if (!inv && load == LD_SRC && store == ST_INTER) {                                         \
      auto k = col_kernel<T, LL, false, LD_SRC, ST_INTER>;                                     \
      if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                   \
      k<<<grid, col_threads<LL>(), smem, st>>>(a, tw, tw_step);                                \
    } else if (!inv && load == LD_INTER && store == ST_INTER) {                                \
      auto k = col_kernel<T, LL, false, LD_INTER, ST_INTER>;                                   \
      if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                   \
      k<<<grid, col_threads<LL>(), smem, st>>>(a, tw, tw_step);                                \
    } else if (inv && load == LD_INTER && store == ST_INTER) {                                 \
      auto k = col_kernel<T, LL, true, LD_INTER, ST_INTER>;                                    \
      if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                   \
      k<<<grid, col_threads<LL>(), smem, st>>>(a, tw, tw_step);                                \
    } else if (inv && load == LD_INTER && store == ST_DST) {                                   \
      auto k = col_kernel<T, LL, true, LD_INTER, ST_DST>;                                      \
      if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                   \
      k<<<grid, col_threads<LL>(), smem, st>>>(a, tw, tw_step);                                \
    } else {                                                                                    \
      return cudaErrorInvalidValue;                                                             \
    }                                                                                           \
    break;                                                                                      \
  }

#define SDCTB_DEFINE_LAUNCH_COL(T)                                                              \
  template <>                                                                                   \
  cudaError_t launch_col<T>(int L, bool inv, int load, int store, dim3 grid, size_t smem,       \
                            cudaStream_t st, const ColArgs& a, const cx_t<T>* tw, int tw_step) { \
    cudaError_t e = cudaSuccess;                                                                \
    switch (L) {                                                                                \
      SDCTB_COL_CASE(T, 2)                                                                      \
      SDCTB_COL_CASE(T, 4)                                                                      \
      SDCTB_COL_CASE(T, 8)                                                                      \
      SDCTB_COL_CASE(T, 16)                                                                     \
      SDCTB_COL_CASE(T, 32)                                                                     \
      SDCTB_COL_CASE(T, 64)                                                                     \
      SDCTB_COL_CASE(T, 128)                                                                    \
      SDCTB_COL_CASE(T, 256)                                                                    \
      SDCTB_COL_CASE(T, 512)                                                                    \
      SDCTB_COL_CASE(T, 1024)                                                                   \
      SDCTB_COL_CASE(T, 2048)                                                                   \
      SDCTB_COL_CASE(T, 4096)                                                                   \
      default:                                                                                  \
        return cudaErrorInvalidValue;                                                           \
    }                                                                                           \
    return cudaGetLastError();                                                                  \
  }

#define SDCTB_ROW_CASE(T, MM)                                                                   \
  case MM: {                                                                                    \
    switch (kind) {                                                                             \
      case RK_FWD2: {                                                                           \
        auto k = row_kernel<T, MM, RK_FWD2>;                                                   \
        if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                 \
        k<<<grid, kRowThreads, smem, st>>>(a, tw, tw_step);                                    \
        break;                                                                                  \
      }                                                                                         \
      case RK_INV2: {                                                                           \
        auto k = row_kernel<T, MM, RK_INV2>;                                                   \
        if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                 \
        k<<<grid, kRowThreads, smem, st>>>(a, tw, tw_step);                                    \
        break;                                                                                  \
      }                                                                                         \
      case RK_FWD3: {                                                                           \
        auto k = row_kernel<T, MM, RK_FWD3>;                                                   \
        if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                 \
        k<<<grid, kRowThreads, smem, st>>>(a, tw, tw_step);                                    \
        break;                                                                                  \
      }                                                                                         \
      case RK_INV3: {                                                                           \
        auto k = row_kernel<T, MM, RK_INV3>;                                                   \
        if ((e = prep_smem(k, smem)) != cudaSuccess) return e;                                 \
        k<<<grid, kRowThreads, smem, st>>>(a, tw, tw_step);                                    \
        break;                                                                                  \
      }                                                                                         \
      default:                                                                                  \
        return cudaErrorInvalidValue;                                                           \
    }                                                                                           \
    break;                                                                                      \
  }

#define SDCTB_DEFINE_LAUNCH_ROW(T)                                                              \
  template <>                                                                                   \
  cudaError_t launch_row<T>(int M, int kind, dim3 grid, size_t smem, cudaStream_t st,           \
                            const RowArgs& a, const cx_t<T>* tw, int tw_step) {                 \
    cudaError_t e = cudaSuccess;                                                                \
    switch (M) {                                                                                \
      SDCTB_ROW_CASE(T, 4)                                                                      \
      SDCTB_ROW_CASE(T, 8)                                                                      \
      SDCTB_ROW_CASE(T, 16)                                                                     \
      SDCTB_ROW_CASE(T, 32)                                                                     \
      SDCTB_ROW_CASE(T, 64)                                                                     \
      SDCTB_ROW_CASE(T, 128)                                                                    \
      SDCTB_ROW_CASE(T, 256)                                                                    \
      SDCTB_ROW_CASE(T, 512)                                                                    \
      SDCTB_ROW_CASE(T, 1024)                                                                   \
      SDCTB_ROW_CASE(T, 2048)                                                                   \
      SDCTB_ROW_CASE(T, 4096)                                                                   \
      default:                                                                                  \
        return cudaErrorInvalidValue;                                                           \
    }                                                                                           \
    return cudaGetLastError();                                                                  \
  }

}  // namespace sdctb
