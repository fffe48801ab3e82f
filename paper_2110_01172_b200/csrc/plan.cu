// Plan object, dispatch and the extern "C" boundary (include/sdct_b200.h).
//
// A plan caches everything per shape that the reference rebuilds per call
// (proj/src/dct2d.cpp:389-393 builds a fresh Plan2d on every Python call):
// the quarter-wave tables a, b (, c) (proj/src/dct1d.cpp:41-48), the FFT
// circle table, the packing twiddles, the launch geometry (band width W of the
// column kernels) and a device workspace for the one inter-pass intermediate.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/sdct_b200.h"
#include "fast_launch.cuh"
#include "host_stage.hpp"
#include "generic.h"
#include "kernels_rowcol.cuh"

namespace {
// NVTX ranges (header-only NVTX v3: a no-op unless a profiler injects its
// library): one range per transform call and one per pass, so nsys / ncu
// --nvtx timelines show "sdct:<kind>" with its "col" / "row" passes nested.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
const char* kind_name(int kind) {
  static const char* names[] = {"sdct:dct_2d",         "sdct:idct_2d",          "sdct:idct_idxst_2d",
                                "sdct:idxst_idct_2d",  "sdct:dct_3d",           "sdct:idct_3d",
                                "sdct:dct_2d_rowcol",  "sdct:dct_1d",           "sdct:idct_1d",
                                "sdct:idxst_1d",       "sdct:idct_idxst_2d_rowcol", "sdct:idxst_idct_2d_rowcol",
                                "sdct:dct_axis0",      "sdct:idct_axis0"};
  return kind >= 0 && kind < static_cast<int>(sizeof(names) / sizeof(names[0])) ? names[kind] : "sdct:?";
}
}  // namespace

using namespace sdctb;

namespace {

thread_local std::string g_last_error;
unsigned long long* g_trace = nullptr;  // debug: column-kernel phase timestamps (sdct_debug_set_trace)
// inverse 2D row passes walk their items last to first (RowArgs::rev): in a
// DCT -> IDCT chain the forward row pass's latest rows are still in L2
// (c2 fp64 round trip ~1% faster, tools/ab_rowinv_rev.sh); SDCT_ROWINV_REV=0
// restores first-to-last (developer A/B)
const int g_rowinv_rev = [] {
  const char* f = getenv("SDCT_ROWINV_REV");
  return f ? atoi(f) : 1;
}();

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? SDCT_ERR_OOM : SDCT_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

bool getenv_flag(const char* name) {  // developer A/B switches (tools/)
  const char* f = getenv(name);
  return f && atoi(f) == 1;
}
bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2i(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (dev >= 0 && dev != prev_) {
      cudaSetDevice(dev);
      switched_ = true;
    }
  }
  ~DeviceGuard() {
    if (switched_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
  bool switched_ = false;
};

}  // namespace

// The attribute is per device: cache grants by (device, kernel).
cudaError_t sdctb::prep_smem_ptr(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> granted[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto& g = granted[dev & 63];
  auto it = g.find(kernel);
  if (it != g.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess) g[kernel] = smem;
  return e;
}

struct sdct_plan_s {
  int rank = 2;
  int n[3] = {1, 1, 1};
  long long batch = 1;
  long long numel = 1;  // per item
  int dtype = SDCT_F64;
  int orientation = SDCT_ORIENT_DIRECT;
  int device = 0;
  bool fast = false;
  // fast geometry
  int M = 0;            // packed z-line length (n_last / 2)
  int nl[2] = {2, 2};   // column-kernel band widths: pass over axis 0, pass over axis 1 (3D)
  TwSet tw_col[2] = {};  // per-stage twiddle tables: axis-0 / axis-1 column FFTs
  TwSet tw_row = {};     // row FFT (length M)
  TwSet tw_col2 = {};    // cluster-split column pass: H-point stage tables (H = n1 / 2)
  bool col2 = false;     // 2D column passes run cluster-split (col2_used)
  bool ax0_ok = false;   // rank 2, pow2 n1 in [8, 4096]: the axis-0 1D kinds (kernels_col1d.cuh)
  TwSet tw_ax0 = {};     // n1-point stage tables of the axis-0 pass
  void* axq = nullptr;   // a(k) = e^{-i pi k / (2 n1)}, k < n1
  bool colc = false;     // 2D fp64 L = 4096 column passes run as persistent cluster pairs (kernels_colc.cuh)
  void* tw_comb = nullptr;  // cluster-split column pass: W_L^k, k < L/2
  // device tables (one allocation)
  void* tables = nullptr;
  void* ta = nullptr;    // dtype quarter-wave tables
  void* tb = nullptr;
  void* tc = nullptr;
  void* tu = nullptr;    // dtype: W_{Nlast}^k, k <= M
  int* srow[2] = {nullptr, nullptr};
  void* fb = nullptr;    // dtype factor tables of tb and tu over q <= M (see RowArgs::fb)
  void* fu = nullptr;
  int fs = 0;
  // corrupt_twiddle_for_testing: host toggle map of negated b entries and its
  // device copy (the 2D row kernels form b(q) from factor tables, so they
  // negate b(q) where the map is set); null until the hook is first used
  std::vector<unsigned char> badq_host;
  unsigned char* badq = nullptr;
  double2* gq[3] = {nullptr, nullptr, nullptr};  // generic fp64 quarter-wave tables
  double2* gc[3] = {nullptr, nullptr, nullptr};  // generic fp64 circle tables
  int bm[3] = {0, 0, 0};                          // Bluestein length per axis (0 = none)
  double2* bchirp[3] = {nullptr, nullptr, nullptr};
  double2* bhat[3] = {nullptr, nullptr, nullptr};
  double2* bcircle[3] = {nullptr, nullptr, nullptr};
  double2* bfa[3] = {nullptr, nullptr, nullptr};  // e^{-2 pi i t / 4096} when M > 4096, else bcircle
  TwSet bst[3] = {};                               // global Bluestein: min(M, 4096)-point column FFT tables
  double2* bhatp[3] = {nullptr, nullptr, nullptr}; // global Bluestein: bhat in [k2][rt_srow(k1)] order
  size_t b_offset_fast = 0, b_offset_gen = 0;    // element offsets of table b (corrupt hook)
  // workspace + host staging
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* d_in = nullptr;
  void* d_out = nullptr;
  // host-streaming pipeline (sdct_exec_host_pipelined): per lane a stream,
  // two item buffers and a workspace, created on first use
  static constexpr int kLanes = 3;
  cudaStream_t lane_st[kLanes] = {};
  cudaEvent_t lane_ev[kLanes] = {};
  cudaEvent_t fork_ev = nullptr;
  void* lane_buf[kLanes][3] = {};
  std::mutex mu;

  // sdct_exec_host: pinned staging chunks for pageable host buffers (host_stage.hpp)
  static constexpr size_t kStageChunk = 32u << 20;
  void* h_stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  void* aux = nullptr;  // sdct_force_fields scratch (coefficients + weighted copy), lazily allocated
  int aux_n = 2;        // aux halves: 3 on fast single-image plans (two paired intermediates)
  // force fields: side stream for the second composite and its fork / join events
  cudaStream_t side_st = nullptr;
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
  std::mutex gws_mu;    // guards the lazy workspace allocation (ensure_ws)
  // row-column kernels (rank 2): per axis a with a pow2 extent in [8, 8192],
  // stage tables of the n_a/2-point row FFT, quarter-wave and W_{n_a} tables
  bool rc_ok[2] = {false, false};
  TwSet rc_tw[2] = {};
  void* rc_q[2] = {nullptr, nullptr};
  void* rc_w[2] = {nullptr, nullptr};
  void* rws = nullptr;  // rfft_nd / irfft_nd scratch (generic size), lazily allocated
  size_t elem() const { return dtype == SDCT_F32 ? 4 : 8; }
  long long blue_elems = 0;  // global Bluestein scratch (bluestein_scratch_elems)
  size_t generic_ws_bytes() const {
    return (2 * static_cast<size_t>(batch) * static_cast<size_t>(numel) + static_cast<size_t>(blue_elems)) *
           sizeof(double2);
  }
  size_t item_bytes() const { return static_cast<size_t>(numel) * elem(); }
  // coefficient scratch of force fields / compression: two tensor-sized
  // halves, the second 256-B aligned (every device buffer handed to a kernel
  // is 16-B aligned)
  size_t aux_half() const { return (static_cast<size_t>(batch) * item_bytes() + 255) & ~size_t(255); }
  size_t table_bytes = 0;  // the one table allocation
};

namespace {

template <typename T>
void fill_table(std::vector<unsigned char>& blob, size_t& off, const std::vector<long double>& re,
                const std::vector<long double>& im) {
  off = (blob.size() + 255) & ~size_t(255);
  blob.resize(off + re.size() * 2 * sizeof(T));
  T* p = reinterpret_cast<T*>(blob.data() + off);
  for (size_t i = 0; i < re.size(); ++i) {
    p[2 * i] = static_cast<T>(re[i]);
    p[2 * i + 1] = static_cast<T>(im[i]);
  }
}

// e^{-i 2 pi num * k / den} for k < count
void circle(std::vector<long double>& re, std::vector<long double>& im, long long count,
            long double num, long double den) {
  const long double pi = 3.141592653589793238462643383279502884L;
  re.resize(count);
  im.resize(count);
  for (long long k = 0; k < count; ++k) {
    const long double ph = -2.0L * pi * num * static_cast<long double>(k) / den;
    re[k] = cosl(ph);
    im[k] = sinl(ph);
  }
}

// In-place iterative radix-2 DFT (sign -1) of a power-of-two length, long
// double: the Bluestein kernel spectrum is computed once per plan on the host.
void host_fft_pow2(std::vector<long double>& re, std::vector<long double>& im) {
  const size_t n = re.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(re[i], re[j]);
      std::swap(im[i], im[j]);
    }
  }
  const long double pi = 3.141592653589793238462643383279502884L;
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t k = 0; k < len / 2; ++k) {
      const long double ang = -2.0L * pi * static_cast<long double>(k) / static_cast<long double>(len);
      const long double wr = cosl(ang), wi = sinl(ang);
      for (size_t i = 0; i < n; i += len) {
        const size_t a = i + k, b = a + len / 2;
        const long double xr = re[b] * wr - im[b] * wi, xi = re[b] * wi + im[b] * wr;
        re[b] = re[a] - xr;
        im[b] = im[a] - xi;
        re[a] += xr;
        im[a] += xi;
      }
    }
  }
}

int pick_nl(int esize, int L, int M, long long planes_batch) {
  if (L > kMaxFastLen) return 16 / esize;  // cluster-split pass: 32-B band rows (kernels_col2.cuh)
  if (const char* f = getenv("SDCT_FORCE_NL")) {  // developer override (tools/)
    const int v = atoi(f);
    if (v >= 2 && v <= M) return v;
  }
  // nl_default: 64 KB tiles with >= 32-B rows (cluster-split for L = 4096).
  // Narrower bands when the problem is too narrow or offers < 2 CTAs per SM.
  const int nld = nl_default(esize, L);
  if (nld <= M && (M / nld) * planes_batch >= 2 * 148) return nld;
  const int nmin = 16 / esize;  // 32-B rows
  if (nmin < nld && nmin <= M && (M / nmin) * planes_batch >= 148) return nmin;
  return 2;
}

// Per-stage DIF twiddle tables of one FFT length (same radix plan as
// RadixPlan<L>): stage s with span > R stores W_span^{j k} at (k-1)*Q + j.
template <typename T>
void stage_tables(std::vector<unsigned char>& blob, int L, size_t offs[4]) {
  int lg = 0;
  while ((1 << lg) < L) ++lg;
  const int S = lg == 0 ? 0 : (lg + 3) / 4;
  const long double pi = 3.141592653589793238462643383279502884L;
  int span = L;
  for (int s = 0; s < 4; ++s) offs[s] = SIZE_MAX;
  for (int s = 0; s < S; ++s) {
    const int R = 1 << (lg / S + (s < lg % S ? 1 : 0));
    const int Q = span / R;
    if (span > R) {
      std::vector<long double> re(static_cast<size_t>(R - 1) * Q), im(re.size());
      for (int k = 1; k < R; ++k)
        for (int j = 0; j < Q; ++j) {
          const long double ph = -2.0L * pi * static_cast<long double>(j * k) / span;
          re[(k - 1) * Q + j] = cosl(ph);
          im[(k - 1) * Q + j] = sinl(ph);
        }
      fill_table<T>(blob, offs[s], re, im);
    }
    span = Q;
  }
}

int build_plan(sdct_plan_s* p) {
  const int r = p->rank;
  const size_t cx = 2 * p->elem();
  // ---- fast-path eligibility ----
  bool fast = false;
  if (r == 2) {
    const int n1 = p->n[0], n2 = p->n[1];
    fast = is_pow2(n1) && is_pow2(n2) && n1 >= 2 && n2 >= 8 && n1 <= kMaxSplitLen && n2 / 2 <= kMaxFastLen;
  } else if (r == 3) {
    const int n1 = p->n[0], n2 = p->n[1], n3 = p->n[2];
    fast = is_pow2(n1) && is_pow2(n2) && is_pow2(n3) && n1 >= 2 && n2 >= 2 && n3 >= 8 &&
           n1 <= kMaxFastLen && n2 <= kMaxFastLen && n3 / 2 <= kMaxFastLen &&
           static_cast<size_t>(4) * (n3 / 2) * cx <= 200 * 1024;
  }
  p->fast = fast;

  std::vector<unsigned char> blob;
  std::vector<long double> re, im;
  size_t off_ta = 0, off_tb = 0, off_tc = 0, off_tu = 0;
  size_t off_gq[3] = {0, 0, 0}, off_gc[3] = {0, 0, 0};
  size_t st_c0[4], st_c1[4], st_r[4], st_c2[4] = {SIZE_MAX, SIZE_MAX, SIZE_MAX, SIZE_MAX};
  size_t off_comb = SIZE_MAX;
  size_t off_srow[2] = {SIZE_MAX, SIZE_MAX};
  size_t off_fb = 0, off_fu = 0;
  if (fast) {
    const int nlast = p->n[r - 1];
    p->M = nlast / 2;
    const bool f32 = p->dtype == SDCT_F32;
    auto put = [&](size_t& off) {
      if (f32) fill_table<float>(blob, off, re, im);
      else fill_table<double>(blob, off, re, im);
    };
    auto stages = [&](int L, size_t* o) {
      if (f32) stage_tables<float>(blob, L, o);
      else stage_tables<double>(blob, L, o);
    };
    // column FFTs of length L >= 4096 run cluster-split: local tables for L/2
    stages(p->n[0], st_c0);
    if (r == 3) stages(p->n[1], st_c1);
    stages(p->M, st_r);
    p->nl[0] = pick_nl(static_cast<int>(p->elem()), p->n[0], p->M, (r == 2 ? 1 : p->n[1]) * p->batch);
    // L = 8192 columns only fit as cluster-split halves; for fp64 L = 4096 the
    // split pass measured slower than the single-CTA pass on B200 (108 vs
    // 86 us) and is an opt-in experiment (SDCT_COL2=1)
    static const bool col2_opt = [] {
      const char* f = getenv("SDCT_COL2");
      return f && atoi(f) == 1;
    }();
    p->col2 = r == 2 && col2_used(static_cast<int>(p->elem()), p->n[0], 1, p->nl[0]) &&
              (p->n[0] > kMaxFastLen || col2_opt);
    // fp64 4096-row columns: the persistent cluster-pair pass is an opt-in
    // experiment (SDCT_COLC=1): parity-green, but 87-93 us vs 78-82 us for the
    // single-CTA early-reissue pass
    static const bool colc_env = [] {
      const char* f = getenv("SDCT_COLC");
      return f && atoi(f) == 1;
    }();
    p->colc = r == 2 && !p->col2 && colc_env && p->dtype == SDCT_F64 && p->n[0] == 4096 && p->nl[0] == 2;
    if (p->col2 || p->colc) {
      stages(p->n[0] / 2, st_c2);
      circle(re, im, p->n[0] / 2, 1.0L, p->n[0]);  // W_L^k, k < L/2
      put(off_comb);
    }
    circle(re, im, p->n[0], 1.0L, 4.0L * p->n[0]);
    put(off_ta);
    circle(re, im, p->n[1], 1.0L, 4.0L * p->n[1]);
    put(off_tb);
    if (r == 3) {
      circle(re, im, p->n[2], 1.0L, 4.0L * p->n[2]);
      put(off_tc);
    }
    circle(re, im, p->M + 1, 1.0L, nlast);
    put(off_tu);
    {
      // factor tables over q in [0, M]: lo = e^{-i th l}, l < 2^fs; hi = e^{-i th 2^fs h}
      int lgq = 0;
      while ((1 << lgq) <= p->M) ++lgq;  // q < 2^lgq
      p->fs = (lgq + 1) / 2;
      const int nlo = 1 << p->fs, nhi = (p->M >> p->fs) + 1;
      const long double pi = 3.141592653589793238462643383279502884L;
      for (int which = 0; which < 2; ++which) {
        // b: theta = pi / (2 N2); u: theta = 2 pi / N2 (N2 = the last extent)
        const long double th = which == 0 ? pi / (2.0L * nlast) : 2.0L * pi / nlast;
        re.resize(nlo + nhi);
        im.resize(nlo + nhi);
        for (int l = 0; l < nlo; ++l) {
          re[l] = cosl(-th * l);
          im[l] = sinl(-th * l);
        }
        for (int h = 0; h < nhi; ++h) {
          re[nlo + h] = cosl(-th * static_cast<long double>(h << p->fs));
          im[nlo + h] = sinl(-th * static_cast<long double>(h << p->fs));
        }
        put(which == 0 ? off_fb : off_fu);
      }
    }
    for (int ax = 0; ax < (r == 3 ? 2 : 1); ++ax) {
      off_srow[ax] = (blob.size() + 255) & ~size_t(255);
      blob.resize(off_srow[ax] + p->n[ax] * sizeof(int));
      int* q = reinterpret_cast<int*>(blob.data() + off_srow[ax]);
      const int L = p->n[ax], H = L / 2;
      for (int k = 0; k < L; ++k) {  // cluster-split passes: k = 2k' + c at row cH + sigma_H(k')
        if (ax == 0 && p->colc) {
          // cluster-pair pass: k = k' + hf H, slot n = digit_pos_H(k') = 8b + r ->
          // row hf H + (b / (H/16)) H/2 + r H/16 + b mod H/16 (kernels_colc.cuh)
          const int kp = k % H, hf = k / H, n = rt_digit_pos(kp, H), b = n >> 3, rr = n & 7, nb2 = H / 16;
          q[k] = hf * H + (b / nb2) * (H / 2) + rr * nb2 + b % nb2;
        } else {
          q[k] = (ax == 0 && p->col2) ? (k & 1) * H + rt_srow(k >> 1, H) : rt_srow(k, L);
        }
      }
    }
    const long long pb0 = (r == 2 ? 1 : p->n[1]) * p->batch;
    p->nl[0] = pick_nl(static_cast<int>(p->elem()), p->n[0], p->M, pb0);
    if (r == 3) p->nl[1] = pick_nl(static_cast<int>(p->elem()), p->n[1], p->M, static_cast<long long>(p->n[0]) * p->batch);
    p->ws_bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  } else {
    // Bluestein lengths of axes with a large prime factor (two-pass 2D
    // pipeline when it holds them, else the global pass), their scratch
    const bool tile = r == 2 && p->n[0] <= kG2MaxN && p->n[1] <= kG2MaxN;  // two-pass candidate
    for (int a = 0; a < r; ++a) p->bm[a] = bluestein_len(p->n[a], tile);
    p->blue_elems = bluestein_scratch_elems(r, p->n, p->bm, p->batch);
    // generic scratch, plus (rank 2) one real tensor for the row-column passes
    p->ws_bytes = p->generic_ws_bytes() + (r == 2 ? static_cast<size_t>(p->batch) * p->item_bytes() : 0);
  }
  // axis-0 1D transforms (kernels_col1d.cuh): n1-point stage tables + a(k)
  size_t off_ax0[4] = {SIZE_MAX, SIZE_MAX, SIZE_MAX, SIZE_MAX}, off_axq = SIZE_MAX;
  if (r == 2 && is_pow2(p->n[0]) && p->n[0] >= 8 && p->n[0] <= kMaxFastLen) {
    const bool f32 = p->dtype == SDCT_F32;
    if (f32) stage_tables<float>(blob, p->n[0], off_ax0);
    else stage_tables<double>(blob, p->n[0], off_ax0);
    circle(re, im, p->n[0], 1.0L, 4.0L * p->n[0]);
    if (f32) fill_table<float>(blob, off_axq, re, im);
    else fill_table<double>(blob, off_axq, re, im);
    p->ax0_ok = true;
  }
  // row-column row-DCT tables (kernels_rowcol.cuh)
  size_t off_rcst[2][4], off_rcq[2] = {0, 0}, off_rcw[2] = {0, 0};
  if (r == 2) {
    for (int a = 0; a < 2; ++a) {
      const int n = p->n[a];
      p->rc_ok[a] = is_pow2(n) && n >= 8 && n <= 2 * kMaxFastLen;
      if (!p->rc_ok[a]) continue;
      const bool f32 = p->dtype == SDCT_F32;
      if (f32) stage_tables<float>(blob, n / 2, off_rcst[a]);
      else stage_tables<double>(blob, n / 2, off_rcst[a]);
      circle(re, im, n, 1.0L, 4.0L * n);
      if (f32) fill_table<float>(blob, off_rcq[a], re, im);
      else fill_table<double>(blob, off_rcq[a], re, im);
      circle(re, im, n / 2 + 1, 1.0L, n);
      if (f32) fill_table<float>(blob, off_rcw[a], re, im);
      else fill_table<double>(blob, off_rcw[a], re, im);
    }
  }
  // generic-path tables are always present (odd shapes, row-column, 1D)
  size_t off_bc[3] = {0, 0, 0}, off_bh[3] = {0, 0, 0}, off_bm[3] = {0, 0, 0}, off_bf[3] = {0, 0, 0};
  size_t off_bst[3][4], off_bhp[3] = {0, 0, 0};
  for (auto& o : off_bst)
    for (size_t& v : o) v = SIZE_MAX;
  for (int a = 0; a < r; ++a) {
    circle(re, im, p->n[a], 1.0L, 4.0L * p->n[a]);
    fill_table<double>(blob, off_gq[a], re, im);
    circle(re, im, p->n[a], 1.0L, p->n[a]);
    fill_table<double>(blob, off_gc[a], re, im);
    // Bluestein tables (generic plans, axes with a large prime factor)
    if (p->bm[a]) {
      const int n = p->n[a], M = p->bm[a];
      const long double pi = 3.141592653589793238462643383279502884L;
      std::vector<long double> cr(n), ci(n), hr(M, 0.0L), hi(M, 0.0L);
      for (int j = 0; j < n; ++j) {
        const long long jj = (static_cast<long long>(j) * j) % (2LL * n);  // j^2 mod 2n keeps the phase exact
        const long double ph = -pi * static_cast<long double>(jj) / n;
        cr[j] = cosl(ph);
        ci[j] = sinl(ph);
        hr[j] = cr[j];  // b_j = conj(c_j), wrapped: b_{M-j} = b_j
        hi[j] = -ci[j];
        if (j) {
          hr[M - j] = cr[j];
          hi[M - j] = -ci[j];
        }
      }
      host_fft_pow2(hr, hi);
      fill_table<double>(blob, off_bc[a], cr, ci);
      fill_table<double>(blob, off_bh[a], hr, hi);
      circle(re, im, M, 1.0L, M);
      fill_table<double>(blob, off_bm[a], re, im);
      if (M > 4096) {
        circle(re, im, 4096, 1.0L, 4096);
        fill_table<double>(blob, off_bf[a], re, im);
      }
      if (p->blue_elems) {  // the global pass: column-kernel FFTs of fa points, fb planes
        const int fa = M < 4096 ? M : 4096, fb = M / fa;
        stage_tables<double>(blob, fa, off_bst[a]);
        std::vector<long double> pr(M), pi2(M);
        for (int k1 = 0; k1 < fa; ++k1) {
          const int srow = rt_srow(k1, fa);
          for (int k2 = 0; k2 < fb; ++k2) {
            pr[static_cast<size_t>(k2) * fa + srow] = hr[k2 + static_cast<size_t>(fb) * k1];
            pi2[static_cast<size_t>(k2) * fa + srow] = hi[k2 + static_cast<size_t>(fb) * k1];
          }
        }
        fill_table<double>(blob, off_bhp[a], pr, pi2);
      }
    }
  }
  cudaError_t e = cudaMalloc(&p->tables, blob.size());
  if (e != cudaSuccess) return cuda_fail(e, "allocating plan tables");
  p->table_bytes = blob.size();
  e = cudaMemcpy(p->tables, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "uploading plan tables");
  unsigned char* base = static_cast<unsigned char*>(p->tables);
  if (fast) {
    auto tws = [&](const size_t* o, TwSet& t) {
      for (int k = 0; k < 4; ++k) t.st[k] = o[k] == SIZE_MAX ? nullptr : base + o[k];
    };
    tws(st_c0, p->tw_col[0]);
    if (r == 3) tws(st_c1, p->tw_col[1]);
    tws(st_r, p->tw_row);
    if (p->col2 || p->colc) tws(st_c2, p->tw_col2);
    p->tw_comb = off_comb == SIZE_MAX ? nullptr : base + off_comb;
    p->ta = base + off_ta;
    p->tb = base + off_tb;
    p->tc = r == 3 ? base + off_tc : nullptr;
    p->tu = base + off_tu;
    p->fb = base + off_fb;
    p->fu = base + off_fu;
    for (int ax = 0; ax < 2; ++ax)
      p->srow[ax] = off_srow[ax] == SIZE_MAX ? nullptr : reinterpret_cast<int*>(base + off_srow[ax]);
    p->b_offset_fast = off_tb;
  }
  for (int a = 0; a < r; ++a) {
    p->gq[a] = reinterpret_cast<double2*>(base + off_gq[a]);
    p->gc[a] = reinterpret_cast<double2*>(base + off_gc[a]);
    if (p->bm[a]) {
      p->bchirp[a] = reinterpret_cast<double2*>(base + off_bc[a]);
      p->bhat[a] = reinterpret_cast<double2*>(base + off_bh[a]);
      p->bcircle[a] = reinterpret_cast<double2*>(base + off_bm[a]);
      p->bfa[a] = p->bm[a] > 4096 ? reinterpret_cast<double2*>(base + off_bf[a]) : p->bcircle[a];
      if (p->blue_elems) {
        for (int k = 0; k < 4; ++k) p->bst[a].st[k] = off_bst[a][k] == SIZE_MAX ? nullptr : base + off_bst[a][k];
        p->bhatp[a] = reinterpret_cast<double2*>(base + off_bhp[a]);
      }
    }
  }
  for (int a = 0; a < 2; ++a) {
    if (!p->rc_ok[a]) continue;
    for (int k = 0; k < 4; ++k) p->rc_tw[a].st[k] = off_rcst[a][k] == SIZE_MAX ? nullptr : base + off_rcst[a][k];
    p->rc_q[a] = base + off_rcq[a];
    p->rc_w[a] = base + off_rcw[a];
  }
  if (p->ax0_ok) {
    for (int k = 0; k < 4; ++k) p->tw_ax0.st[k] = off_ax0[k] == SIZE_MAX ? nullptr : base + off_ax0[k];
    p->axq = base + off_axq;
  }
  p->b_offset_gen = r >= 2 ? off_gq[1] : off_gq[0];
  // the plan-owned workspace is allocated on first use with no caller
  // workspace (ensure_ws): the torch path always passes its own
  return SDCT_OK;
}

bool kind_ok(const sdct_plan_s* p, int kind) {
  switch (kind) {
    case SDCT_DCT_2D:
    case SDCT_IDCT_2D:
    case SDCT_IDCT_IDXST_2D:
    case SDCT_IDXST_IDCT_2D:
    case SDCT_DCT_2D_ROWCOL:
    case SDCT_IDCT_IDXST_2D_ROWCOL:
    case SDCT_IDXST_IDCT_2D_ROWCOL:
    case SDCT_DCT_AXIS0:
    case SDCT_IDCT_AXIS0:
      return p->rank == 2;
    case SDCT_DCT_3D:
    case SDCT_IDCT_3D:
      return p->rank == 3;
    case SDCT_DCT_1D:
    case SDCT_IDCT_1D:
    case SDCT_IDXST_1D:
      return p->rank == 1;
    default:
      return false;
  }
}

// ---------------------------------------------------------------------------
// Stage lists. Every transform is an ordered list of kernel launches; the
// full transform runs all of them, sdct_exec_stage runs one.
// ---------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link
// against libcuda needed).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 4D map over a column pass input: dims (innermost first) {inner reals, FFT
// rows, planes, batch} with byte strides for dims 1..3; box {2*nl, min(L,256), 1, 1}.
bool make_col_map(CUtensorMap* map, bool f32, const void* base, long long inner, long long rows,
                  long long row_stride_b, long long planes, long long plane_stride_b, long long batch,
                  long long batch_stride_b, int nl, int L) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(planes), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(row_stride_b), static_cast<cuuint64_t>(plane_stride_b),
                                 static_cast<cuuint64_t>(batch_stride_b)};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(2 * nl), static_cast<cuuint32_t>(L < 256 ? L : 256), 1, 1};  // L = rows per box cap
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 5D map over y for the inverse final gather: {inner reals, row class (2,
// stride = row stride), row pair (rows/2, stride = 2 rows), planes, batch};
// box {2*nl, 1, min(rows/2, 256), 1, 1}. Even y rows 2p hold pe-images of the
// first half of the spatial indices, odd rows 2p+1 the second half.
bool make_class_map(CUtensorMap* map, bool f32, const void* base, long long inner, long long rows,
                    long long row_stride_b, long long planes, long long plane_stride_b, long long batch,
                    long long batch_stride_b, int nl) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const long long pairs = rows / 2;
  const cuuint64_t dims[5] = {static_cast<cuuint64_t>(inner), 2, static_cast<cuuint64_t>(pairs),
                              static_cast<cuuint64_t>(planes), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(row_stride_b), static_cast<cuuint64_t>(2 * row_stride_b),
                                 static_cast<cuuint64_t>(plane_stride_b), static_cast<cuuint64_t>(batch_stride_b)};
  const cuuint32_t box[5] = {static_cast<cuuint32_t>(2 * nl), 1, static_cast<cuuint32_t>(pairs < 256 ? pairs : 256), 1,
                             1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 5D map over x (forward source) or y (inverse destination) of the
// cluster-pair column pass: {inner reals, row mod 4 (stride = row stride),
// row / 4 (stride = 4 rows), planes, batch}; box {2*nl, 1, min(rows/4, 256), 1, 1}.
bool make_class4_map(CUtensorMap* map, bool f32, const void* base, long long inner, long long rows,
                     long long row_stride_b, long long planes, long long plane_stride_b, long long batch,
                     long long batch_stride_b, int nl) {
  auto enc = tmap_encoder();
  if (!enc || rows % 4) return false;
  const long long quads = rows / 4;
  const cuuint64_t dims[5] = {static_cast<cuuint64_t>(inner), 4, static_cast<cuuint64_t>(quads),
                              static_cast<cuuint64_t>(planes), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(row_stride_b), static_cast<cuuint64_t>(4 * row_stride_b),
                                 static_cast<cuuint64_t>(plane_stride_b), static_cast<cuuint64_t>(batch_stride_b)};
  const cuuint32_t box[5] = {static_cast<cuuint32_t>(2 * nl), 1, static_cast<cuuint32_t>(quads < 256 ? quads : 256), 1,
                             1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// Batched complex line FFT for the generic path's global Bluestein pass
// (generic.h): the fast column kernel on a [planes][L][W] complex tensor.
cudaError_t sdctb::bluestein_line_fft(const double2* src, double2* dst, int L, int W, int planes, bool inverse,
                               const void* const st_tables[4], cudaStream_t st) {
  const int nld = nl_default(8, L);
  const int nl = (W % nld == 0 && static_cast<long long>(W / nld) * planes >= 148) ? nld : 2;
  const long long row_b = 16LL * W, plane_b = row_b * L, batch_b = plane_b * planes;
  CUtensorMap mi, mo;
  if (!make_col_map(&mi, false, src, 2LL * W, L, row_b, planes, plane_b, 1, batch_b, nl, L) ||
      !make_col_map(&mo, false, dst, 2LL * W, L, row_b, planes, plane_b, 1, batch_b, nl, L / 2))
    return cudaErrorInvalidValue;
  ColArgs c{};
  c.src = src;
  c.dst = dst;
  c.in_row = c.out_row = W;
  c.in_plane = c.out_plane = static_cast<long long>(L) * W;
  c.in_batch = c.out_batch = c.in_plane * planes;
  TwSet tw{};
  for (int k = 0; k < 4; ++k) tw.st[k] = st_tables[k];
  return launch_col<double>(inverse ? CV_INV_INTER : CV_FWD_INTER, L, nl, dim3(W / nl, planes, 1), st, mi, mo, c, tw);
}

namespace {

// Compression threshold carried by the 2D inverse row kernels (weight 3).
struct Threshold {
  double eps = 0.0, scale = 1.0;
  unsigned long long* count = nullptr;
};

// Paired inverse launch (sdct_force_fields): both field composites of one
// image as batch items 0 and 1 of a single row launch and a single column
// launch. Item 1 takes mode2 / weight2 / the *2 signs; both read the same
// coefficients; the intermediates and outputs sit at byte strides of their own.
struct PairSpec {
  int mode1, weight1, mode2, weight2;
  long long ws_stride;   // bytes between the two intermediates
  long long out_stride;  // bytes between the two outputs (out = the first)
};

// Geometry of one side (input or output) of a column pass, in reals.
struct Side {
  long long inner, rows, row_stride, planes, plane_stride, batch_stride;
};

template <typename T>
int run_fast(sdct_plan_s* p, int kind, int only_stage, const void* in, void* out, void* ws,
             cudaStream_t st, int* nstages, int weight, const Threshold* thr, int bcount,
             const PairSpec* pair = nullptr) {
  const int n1 = p->n[0], n2 = p->n[1], n3 = p->n[2];
  const int M = p->M;
  const long long item = p->numel;
  const int B = pair ? 2 : bcount;  // items of this launch set (<= 65535, see run())
  int stage = 0;
  cudaError_t e = cudaSuccess;
  auto want = [&](void) { return only_stage < 0 || only_stage == stage; };
  const bool f32 = sizeof(T) == 4;
  const long long es = sizeof(T);
  bool map_ok = true;
  // column pass over an axis of length L with band width nl; the TMA map
  // describes its input (see make_col_map)
  // column pass over an axis of length L with band width nl; TMA maps for its
  // input (4D) and output (4D intermediate, or the 5D even/odd-row map of y)
  auto col = [&](int variant, int L, int nl, int planes, ColArgs a, const TwSet& tw, const Side& in,
                 const Side& o) {
    a.trace = g_trace;
    if (want() && e == cudaSuccess && map_ok) {
      NvtxRange nv("col");
      CUtensorMap mi, mo;
      // the forward source pass loads rows by parity class (5D class map)
      map_ok = variant == CV_FWD_SRC && col_class_load(static_cast<int>(es), L, nl)
                   ? make_class_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes,
                                    in.plane_stride * es, B, in.batch_stride * es, nl)
                   : make_col_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes,
                                  in.plane_stride * es, B, in.batch_stride * es, nl, L);
      if (map_ok) {
        if (variant == CV_INV_DST)
          map_ok = make_class_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es,
                                  B, o.batch_stride * es, nl);
        else
          map_ok = make_col_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es,
                                B, o.batch_stride * es, nl, L / 2);
      }
      if (map_ok) e = launch_col<T>(variant, L, nl, dim3(M / nl, planes, B), st, mi, mo, a, tw);
    }
    ++stage;
  };
  // cluster-split 2D column pass (kernels_col2.cuh): forward reads the source
  // through the parity-class map, the inverse writes y through it
  auto col2 = [&](bool inv, ColArgs a, const Side& in, const Side& o) {
    a.twc = p->tw_comb;
    if (want() && e == cudaSuccess && map_ok) {
      NvtxRange nv("col2");
      CUtensorMap mi, mo;
      if (!inv) {
        map_ok = make_class_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes, in.plane_stride * es, B,
                                in.batch_stride * es, p->nl[0]) &&
                 make_col_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es, B,
                              o.batch_stride * es, p->nl[0], 256);
      } else {
        map_ok = make_col_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes, in.plane_stride * es, B,
                              in.batch_stride * es, p->nl[0], 256) &&
                 make_class_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es, B,
                                o.batch_stride * es, p->nl[0]);
      }
      if (map_ok) e = launch_col2<T>(n1, inv, M / p->nl[0], B, st, mi, mo, a, p->tw_col2);
    }
    ++stage;
  };
  // persistent cluster-pair 2D column pass (kernels_colc.cuh): forward reads
  // the source through the 4-class map, the inverse writes y through it
  auto colc = [&](bool inv, ColArgs a, const Side& in, const Side& o) {
    a.twc = p->tw_comb;
    if (want() && e == cudaSuccess && map_ok) {
      NvtxRange nv("colc");
      CUtensorMap mi, mo;
      if (!inv) {
        map_ok = make_class4_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes, in.plane_stride * es,
                                 B, in.batch_stride * es, p->nl[0]) &&
                 make_col_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es, B,
                              o.batch_stride * es, p->nl[0], 256);
      } else {
        map_ok = make_col_map(&mi, f32, a.src, in.inner, in.rows, in.row_stride * es, in.planes, in.plane_stride * es, B,
                              in.batch_stride * es, p->nl[0], 256) &&
                 make_class4_map(&mo, f32, a.dst, o.inner, o.rows, o.row_stride * es, o.planes, o.plane_stride * es, B,
                                 o.batch_stride * es, p->nl[0]);
      }
      if (map_ok) e = launch_colc(inv, M / p->nl[0], B, st, mi, mo, a, p->tw_col2);
    }
    ++stage;
  };
  auto row = [&](int rk, int groups, const RowArgs& a) {
    if (want() && e == cudaSuccess) {
      NvtxRange nv("row");
      e = launch_row<T>(M, rk, dim3(groups, B), st, a, p->tw_row);
    }
    ++stage;
  };
  RowArgs ra{};
  ra.n1 = n1;
  ra.n2 = n2;
  ra.n3 = n3;
  ra.ta = p->ta;
  ra.tb = p->tb;
  ra.tc = p->tc;
  ra.tu = p->tu;
  ra.s0 = p->srow[0];
  ra.s1 = p->srow[1];
  ra.fb = p->fb;
  ra.fu = p->fu;
  ra.fs = p->fs;
  ra.badq = p->badq;
  ra.weight = weight;
  if (thr) {
    ra.thr_eps = thr->eps;
    ra.thr_scale = thr->scale;
    ra.thr_count = thr->count;
  }
  if (p->rank == 2) {
    const long long inter = static_cast<long long>(n1) * M;
    if (kind == SDCT_DCT_2D) {
      ColArgs c{};
      c.src = in;
      c.dst = ws;
      c.in_row = n2;
      c.in_batch = item;
      c.out_row = M;
      c.out_batch = inter;
      ra.src = ws;
      ra.src_batch = inter;
      ra.dst = out;
      ra.dst_batch = item;
      if (p->col2)
        col2(false, c, Side{n2, n1, n2, 1, item, item}, Side{2LL * M, n1, 2LL * M, 1, 2 * inter, 2 * inter});
      else if (p->colc)
        colc(false, c, Side{n2, n1, n2, 1, item, item}, Side{2LL * M, n1, 2LL * M, 1, 2 * inter, 2 * inter});
      else
        col(CV_FWD_SRC, n1, p->nl[0], 1, c, p->tw_col[0], Side{n2, n1, n2, 1, item, item},
            Side{2LL * M, n1, 2LL * M, 1, 2 * inter, 2 * inter});
      ra.src = ws;
      ra.src_batch = inter;
      ra.dst = out;
      ra.dst_batch = item;
      row(RK_FWD2, n1 / 2, ra);
    } else {
      const int mode = pair ? pair->mode1 : kind == SDCT_IDXST_IDCT_2D ? 1 : kind == SDCT_IDCT_IDXST_2D ? 2 : 0;
      // batch strides (complex elements of the intermediate, reals of y)
      const long long wsb = pair ? pair->ws_stride / (2 * es) : inter;
      const long long outb = pair ? pair->out_stride / es : item;
      ra.src = in;
      ra.src_batch = item;
      ra.dst = ws;
      ra.dst_batch = wsb;
      ra.mode = mode;
      ra.rev = g_rowinv_rev;
      if (pair) {
        ra.weight = pair->weight1;
        ra.pair_b = 1;
        ra.mode2 = pair->mode2;
        ra.weight2 = pair->weight2;
      }
      row(RK_INV2, n1 / 2, ra);
      ColArgs c{};
      c.src = ws;
      c.dst = out;
      c.in_row = M;
      c.in_batch = wsb;
      c.out_row = n2;
      c.out_batch = outb;
      c.scale = 0.25;
      c.sign_row = mode == 1;
      c.sign_col = mode == 2;
      if (pair) {
        c.pair_b = 1;
        c.sign_row2 = pair->mode2 == 1;
        c.sign_col2 = pair->mode2 == 2;
      }
      if (p->col2)
        col2(true, c, Side{2LL * M, n1, 2LL * M, 1, 2 * wsb, 2 * wsb}, Side{n2, n1, n2, 1, outb, outb});
      else if (p->colc)
        colc(true, c, Side{2LL * M, n1, 2LL * M, 1, 2 * wsb, 2 * wsb}, Side{n2, n1, n2, 1, outb, outb});
      else
        col(CV_INV_DST, n1, p->nl[0], 1, c, p->tw_col[0], Side{2LL * M, n1, 2LL * M, 1, 2 * wsb, 2 * wsb},
            Side{n2, n1, n2, 1, outb, outb});
    }
  } else {
    const long long inter = static_cast<long long>(n1) * n2 * M;
    const int groups = (n1 / 2 + 1) * (n2 / 2 + 1);
    if (kind == SDCT_DCT_3D) {
      // axis 0 (rows i, source plane pe(j)) -> intermediate [i_slot][j][s]
      ColArgs c{};
      c.src = in;
      c.dst = ws;
      c.in_row = static_cast<long long>(n2) * n3;
      c.in_plane = n3;
      c.in_plane_par = n2;
      c.in_batch = item;
      c.out_row = static_cast<long long>(n2) * M;
      c.out_plane = M;
      c.out_batch = inter;
      c.tma_plane_par = n2;
      col(CV_FWD_SRC, n1, p->nl[0], n2, c, p->tw_col[0], Side{n3, n1, static_cast<long long>(n2) * n3, n2, n3, item},
          Side{2LL * M, n1, 2LL * n2 * M, n2, 2LL * M, 2 * inter});
      // axis 1 (rows j, planes i_slot), in place -> [i_slot][j_slot][s]
      ColArgs d{};
      d.src = ws;
      d.dst = ws;
      d.in_row = M;
      d.in_plane = static_cast<long long>(n2) * M;
      d.in_batch = inter;
      d.out_row = M;
      d.out_plane = static_cast<long long>(n2) * M;
      d.out_batch = inter;
      col(CV_FWD_INTER, n2, p->nl[1], n1, d, p->tw_col[1], Side{2LL * M, n2, 2LL * M, n1, 2LL * n2 * M, 2 * inter},
          Side{2LL * M, n2, 2LL * M, n1, 2LL * n2 * M, 2 * inter});
      ra.src = ws;
      ra.src_batch = inter;
      ra.dst = out;
      ra.dst_batch = item;
      row(RK_FWD3, groups, ra);
    } else {
      ra.src = in;
      ra.src_batch = item;
      ra.dst = ws;
      ra.dst_batch = inter;
      row(RK_INV3, groups, ra);  // -> [k1][k2][s]
      ColArgs d{};
      d.src = ws;
      d.dst = ws;
      d.in_row = M;
      d.in_plane = static_cast<long long>(n2) * M;
      d.in_batch = inter;
      d.out_row = M;
      d.out_plane = static_cast<long long>(n2) * M;
      d.out_batch = inter;
      col(CV_INV_INTER, n2, p->nl[1], n1, d, p->tw_col[1], Side{2LL * M, n2, 2LL * M, n1, 2LL * n2 * M, 2 * inter},
          Side{2LL * M, n2, 2LL * M, n1, 2LL * n2 * M, 2 * inter});  // -> [k1 srow][j][s]
      ColArgs c{};
      c.src = ws;
      c.dst = out;
      c.in_row = static_cast<long long>(n2) * M;
      c.in_plane = M;
      c.in_batch = inter;
      c.out_row = static_cast<long long>(n2) * n3;
      c.out_plane = n3;
      c.out_plane_map = 1;  // plane j (natural after the DIT axis-1 pass) -> y plane pe(j)
      c.out_plane_n = n2;
      c.out_batch = item;
      c.scale = 0.125;
      col(CV_INV_DST, n1, p->nl[0], n2, c, p->tw_col[0], Side{2LL * M, n1, 2LL * n2 * M, n2, 2LL * M, 2 * inter},
          Side{n3, n1, static_cast<long long>(n2) * n3, n2, n3, item});
    }
  }
  if (nstages) *nstages = stage;
  if (!map_ok) return fail(SDCT_ERR_CUDA, "cuTensorMapEncodeTiled failed (driver entry point or tile geometry)");
  if (e != cudaSuccess) return cuda_fail(e, "launching fast-path kernel");
  return SDCT_OK;
}

GenericJob make_job(const sdct_plan_s* p, int kind) {
  GenericJob j;
  j.rank = p->rank;
  for (int a = 0; a < p->rank; ++a) {
    j.dims[a] = p->n[a];
    j.quarter[a] = p->gq[a];
    j.circle[a] = p->gc[a];
    j.blue_m[a] = p->bm[a];
    j.blue_chirp[a] = p->bchirp[a];
    j.blue_hat[a] = p->bhat[a];
    j.blue_circle[a] = p->bcircle[a];
    j.blue_fa[a] = p->bfa[a];
    for (int k = 0; k < 4; ++k) j.blue_st[a][k] = p->bst[a].st[k];
    j.blue_hatp[a] = p->bhatp[a];
  }
  j.blue_scratch = p->blue_elems > 0;
  j.batch = p->batch;
  switch (kind) {
    case SDCT_IDCT_2D: j.inverse = true; j.scale = 0.25; break;
    case SDCT_IDXST_IDCT_2D: j.inverse = true; j.scale = 0.25; j.mode = 1; j.sign_axis = 0; break;
    case SDCT_IDCT_IDXST_2D: j.inverse = true; j.scale = 0.25; j.mode = 2; j.sign_axis = 1; break;
    case SDCT_IDCT_3D: j.inverse = true; j.scale = 0.125; break;
    case SDCT_IDCT_1D: j.inverse = true; j.scale = 0.5; break;
    case SDCT_IDXST_1D: j.inverse = true; j.scale = 0.5; j.mode = 2; j.sign_axis = 0; break;
    default: break;
  }
  return j;
}


bool is_rowcol(int kind) {
  return kind == SDCT_DCT_2D_ROWCOL || kind == SDCT_IDCT_IDXST_2D_ROWCOL || kind == SDCT_IDXST_IDCT_2D_ROWCOL;
}

// Row-column transforms (kernels_rowcol.cuh): axis-1 pass, transpose, axis-0
// pass, transpose — stages 0..3; stage k reads/writes what the full transform
// would. The intermediate is one real tensor in the workspace (after the
// generic scratch on generic plans).
template <typename T>
int run_rowcol(sdct_plan_s* p, int kind, int only_stage, const void* in, void* out, void* ws, cudaStream_t st,
               int* nstages) {
  const int n1 = p->n[0], n2 = p->n[1];
  const long long B = p->batch;
  void* gscratch = p->fast ? nullptr : ws;
  T* tmp = reinterpret_cast<T*>(static_cast<unsigned char*>(ws) + (p->fast ? 0 : p->generic_ws_bytes()));
  const bool inv = kind != SDCT_DCT_2D_ROWCOL;
  // IdctIdxst: sine along axis 1 (the rows of the first pass); IdxstIdct: along axis 0
  const bool sine_rows = kind == SDCT_IDCT_IDXST_2D_ROWCOL, sine_cols = kind == SDCT_IDXST_IDCT_2D_ROWCOL;
  cudaError_t e = cudaSuccess;
  auto pass = [&](int axis, long long rows, const void* src, void* dst, bool sine) {
    const int n = p->n[axis];
    RcArgs a{};
    a.src = src;
    a.dst = dst;
    a.rows = rows;
    a.n = n;
    a.sine = sine ? 1 : 0;
    if (p->rc_ok[axis]) {
      a.tq = p->rc_q[axis];
      a.tw = p->rc_w[axis];
      return launch_rowdct<T>(n, inv, a, p->rc_tw[axis], st);
    }
    if (n <= 64 || !gscratch) return launch_rowdct_direct<T>(inv, a, st);
    GenericJob j;  // longer non-pow2 rows: the generic 1D path, batched over the rows
    j.rank = 1;
    j.dims[0] = n;
    j.batch = rows;
    j.quarter[0] = p->gq[axis];
    j.circle[0] = p->gc[axis];
    if (inv) {
      j.inverse = true;
      j.scale = 0.5;
      j.mode = sine ? 2 : 0;
      j.sign_axis = sine ? 0 : -1;
    }
    return generic_run<T>(j, src, dst, gscratch, st);
  };
  auto transpose = [&](const void* src, void* dst, int R, int C) {
    const size_t item = static_cast<size_t>(R) * C * sizeof(T);
    cudaError_t r = cudaSuccess;
    for (long long b0 = 0; b0 < B && r == cudaSuccess; b0 += 65535)
      r = launch_transpose<T>(static_cast<const unsigned char*>(src) + b0 * item,
                              static_cast<unsigned char*>(dst) + b0 * item, R, C, std::min<long long>(65535, B - b0),
                              st);
    return r;
  };
  for (int stage = 0; stage < 4 && e == cudaSuccess; ++stage) {
    if (only_stage >= 0 && only_stage != stage) continue;
    switch (stage) {
      case 0: e = pass(1, B * n1, in, tmp, sine_rows); break;
      case 1: e = transpose(tmp, out, n1, n2); break;
      case 2: e = pass(0, B * n2, out, tmp, sine_cols); break;
      default: e = transpose(tmp, out, n2, n1); break;
    }
  }
  if (nstages) *nstages = 4;
  if (e != cudaSuccess) return cuda_fail(e, "launching row-column kernels");
  return SDCT_OK;
}

bool is_axis0(int kind) { return kind == SDCT_DCT_AXIS0 || kind == SDCT_IDCT_AXIS0; }

// Axis-0 1D DCT-II / DCT-III of every column (kernels_col1d.cuh): one
// persistent column pass, band rows of 32 B, all batch items as tiles.
template <typename T>
int run_axis0(sdct_plan_s* p, int kind, const void* in, void* out, cudaStream_t st, int* nstages) {
  if (nstages) *nstages = 1;
  const int n1 = p->n[0], n2 = p->n[1];
  const long long es = sizeof(T);
  const int nl = static_cast<int>(16 / es);
  // (the plan's 2D orientation does not apply: p->n are the caller's extents)
  if (!p->ax0_ok || n2 % (2 * nl) != 0)
    return fail(SDCT_ERR_PLAN, "axis-0 transforms need a power-of-two n1 in [8, 4096] and n2 a multiple of " +
                                   std::to_string(2 * nl));
  const bool inv = kind == SDCT_IDCT_AXIS0;
  const bool f32 = sizeof(T) == 4;
  const long long item = static_cast<long long>(n1) * n2;
  const long long B = p->batch;
  CUtensorMap mi, mo;
  bool ok;
  if (!inv)
    ok = make_class_map(&mi, f32, in, n2, n1, n2 * es, 1, item * es, B, item * es, nl) &&
         make_col_map(&mo, f32, out, n2, n1, n2 * es, 1, item * es, B, item * es, nl, n1 / 2);
  else
    ok = make_col_map(&mi, f32, in, n2, n1, n2 * es, 1, item * es, B, item * es, nl, n1 / 2) &&
         make_class_map(&mo, f32, out, n2, n1, n2 * es, 1, item * es, B, item * es, nl);
  if (!ok) return fail(SDCT_ERR_CUDA, "cuTensorMapEncodeTiled failed (axis-0 pass)");
  ColArgs a{};
  a.src = in;
  a.dst = out;
  a.twc = p->axq;  // a(k) = e^{-i pi k / (2 n1)}
  a.scale = 0.5;  // idct_1d: y(pe(n)) = z(n) / 2
  NvtxRange nv("col1d");
  const cudaError_t e = launch_col1d<T>(inv, n1, n2 / (2 * nl), static_cast<int>(B), st, mi, mo, a, p->tw_ax0);
  if (e != cudaSuccess) return cuda_fail(e, "launching the axis-0 column pass");
  return SDCT_OK;
}

template <typename T>
int run(sdct_plan_s* p, int kind, int only_stage, const void* in, void* out, void* ws,
        cudaStream_t st, int* nstages, int weight, const Threshold* thr) {
  if (is_rowcol(kind)) return run_rowcol<T>(p, kind, only_stage, in, out, ws, st, nstages);
  if (is_axis0(kind)) return only_stage > 0 ? SDCT_OK : run_axis0<T>(p, kind, in, out, st, nstages);
  if (p->fast) {
    // batch items ride on grid.y / grid.z (<= 65535): larger batches run as
    // consecutive launch sets over contiguous chunks (same workspace layout)
    const long long chunk = 65535;
    const size_t ib = p->item_bytes();
    int rc = SDCT_OK;
    for (long long b0 = 0; b0 < p->batch && rc == SDCT_OK; b0 += chunk) {
      const int bc = static_cast<int>(std::min<long long>(chunk, p->batch - b0));
      // each chunk's intermediate lives at its own offset of the workspace
      // (the fast workspace is batch * item_bytes), so a staged call
      // (only_stage >= 0) never lets chunk c+1 overwrite chunk c's intermediate
      rc = run_fast<T>(p, kind, only_stage, static_cast<const unsigned char*>(in) + b0 * ib,
                       static_cast<unsigned char*>(out) + b0 * ib, static_cast<unsigned char*>(ws) + b0 * ib, st,
                       nstages, weight, thr, bc);
    }
    return rc;
  }
  if (nstages) *nstages = 1;  // generic path is timed as one unit
  if (only_stage > 0) return SDCT_OK;
  cudaError_t e = generic_run<T>(make_job(p, kind), in, out, ws, st);
  if (e != cudaSuccess) return cuda_fail(e, "launching generic-path kernels");
  return SDCT_OK;
}

// The plan-owned workspace, allocated on first use (callers that pass their
// own workspace never pay for it).
int ensure_ws(sdct_plan_s* p) {
  std::lock_guard<std::mutex> lock(p->gws_mu);
  if (p->ws) return SDCT_OK;
  DeviceGuard g(p->device);
  cudaError_t e = cudaMalloc(&p->ws, p->ws_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "allocating plan workspace");
  return SDCT_OK;
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; }

int dispatch(sdct_plan_s* p, int kind, int only_stage, const void* in, void* out, void* ws,
             cudaStream_t st, int* nstages, int weight = 0, const Threshold* thr = nullptr) {
  if (!kind_ok(p, kind)) return fail(SDCT_ERR_PLAN, "transform kind does not match the plan rank");
  // the kernels move rows with 16-B bulk copies / TMA and 128-bit accesses:
  // reject misaligned buffers up front (a fault there would poison the context)
  if (!aligned16(in) || !aligned16(out) || (ws && !aligned16(ws)))
    return fail(SDCT_ERR_ARG, "device buffers must be 16-byte aligned");
  if (!ws) {
    const int rc = ensure_ws(p);
    if (rc != SDCT_OK) return rc;
    ws = p->ws;
  }
  DeviceGuard g(p->device);
  NvtxRange nv(kind_name(kind));
  return p->dtype == SDCT_F32 ? run<float>(p, kind, only_stage, in, out, ws, st, nstages, weight, thr)
                              : run<double>(p, kind, only_stage, in, out, ws, st, nstages, weight, thr);
}

// ---- analytic StageCounters (replays the reference's Counted tallies) -----
struct Cnt {
  unsigned long long stages = 0, reads = 0, writes = 0, mults = 0, adds = 0;
  void cmul() { mults += 4; adds += 2; }
};

void count_dct2(long long m1, long long m2, Cnt& c) {
  // parity gather (dct2d.cpp:48-70) + fused post (82-115)
  c.stages = 3;
  c.reads += m1 * m2;
  c.writes += m1 * m2;
  const long long h2 = m2 / 2 + 1;
  for (long long q1 = 0; q1 <= m1 / 2; ++q1)
    for (long long q2 = 0; q2 < h2; ++q2) {
      const bool deg1 = (m1 - q1) % m1 == q1, deg2 = (m2 - q2) % m2 == q2;
      c.reads += deg1 ? 1 : 2;
      c.cmul(); c.cmul(); c.adds += 2; c.cmul();
      c.writes += 1 + (deg2 ? 0 : 1);
      if (!deg1) {
        c.adds += 2; c.cmul();
        c.writes += 1 + (deg2 ? 0 : 1);
      }
    }
}

void count_idct2(long long m1, long long m2, int mode, Cnt& c) {
  // idct_pre (dct2d.cpp:161-198) + inverse gather (214-238)
  c.stages = 3;
  const long long h2 = m2 / 2 + 1;
  auto loads = [&](long long i, long long j) -> int {
    if (i == m1 || j == m2) return 0;
    if (mode == 1 && i == 0) return 0;
    if (mode == 2 && j == 0) return 0;
    return 1;
  };
  for (long long q1 = 0; q1 <= m1 / 2; ++q1)
    for (long long n2 = 0; n2 < h2; ++n2) {
      c.reads += loads(q1, n2) + loads(m1 - q1, m2 - n2) + loads(m1 - q1, n2) + loads(q1, m2 - n2);
      c.cmul(); c.adds += 2; c.cmul(); c.writes += 1;
      if ((m1 - q1) % m1 != q1) {
        c.cmul(); c.adds += 2; c.cmul(); c.writes += 1;
      }
    }
  c.reads += m1 * m2;
  c.writes += m1 * m2;
}

void count_dct3(long long n1, long long n2, long long n3, Cnt& c) {
  c.stages = 3;
  const long long N = n1 * n2 * n3;
  c.reads += N;
  c.writes += N;
  for (long long q1 = 0; q1 <= n1 / 2; ++q1)
    for (long long q2 = 0; q2 <= n2 / 2; ++q2)
      for (long long q3 = 0; q3 <= n3 / 2; ++q3) {
        const bool d1 = (n1 - q1) % n1 == q1, d2 = (n2 - q2) % n2 == q2, d3 = (n3 - q3) % n3 == q3;
        c.reads += 1 + (d1 ? 0 : 1) + (d2 ? 0 : 1) + ((d1 || d2) ? 0 : 1);
        c.cmul(); c.cmul();            // ab, cb
        c.cmul(); c.cmul(); c.cmul(); c.cmul();  // t1..t4
        c.adds += 4;                   // sum12, sum34
        c.adds += 2; c.cmul();         // cu00
        c.writes += 1 + (d3 ? 0 : 1);
        if (!d2) { c.adds += 2; c.cmul(); c.writes += 1 + (d3 ? 0 : 1); }
        if (!d1) {
          c.adds += 4;                 // dif12, dif34
          c.adds += 2; c.cmul(); c.writes += 1 + (d3 ? 0 : 1);
          if (!d2) { c.adds += 2; c.cmul(); c.writes += 1 + (d3 ? 0 : 1); }
        }
      }
}

void count_idct3(long long n1, long long n2, long long n3, Cnt& c) {
  c.stages = 3;
  const long long h3 = n3 / 2 + 1;
  auto ld = [&](long long i, long long j, long long k) -> int { return (i == n1 || j == n2 || k == n3) ? 0 : 1; };
  for (long long i = 0; i < n1; ++i)
    for (long long j = 0; j < n2; ++j)
      for (long long k = 0; k < h3; ++k) {
        const long long r1 = n1 - i, r2 = n2 - j, r3 = n3 - k;
        c.reads += ld(i, j, k) + ld(r1, r2, k) + ld(r1, j, r3) + ld(i, r2, r3) + ld(r1, r2, r3) +
                   ld(r1, j, k) + ld(i, r2, k) + ld(i, j, r3);
        c.adds += 3 + 3;
        c.cmul(); c.cmul(); c.cmul();
        c.writes += 1;
      }
  const long long N = n1 * n2 * n3;
  c.reads += N;
  c.writes += N;
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

int sdct_version(void) { return 10000; }

// Debug hook (not part of the public header): device buffer of 5 u64 per
// column tile, or NULL to disable. Used by tools/trace_col.py.
int sdct_debug_set_trace(void* dev_buf) {
  g_trace = static_cast<unsigned long long*>(dev_buf);
  return SDCT_OK;
}

const char* sdct_last_error(void) { return g_last_error.c_str(); }

int sdct_plan_create(sdct_plan_t* out, int rank, const int64_t* dims, int64_t batch, int dtype,
                     int orientation, int device) {
  if (!out || !dims) return fail(SDCT_ERR_ARG, "null argument to sdct_plan_create");
  *out = nullptr;
  if (rank < 1 || rank > 3) return fail(SDCT_ERR_SHAPE, "plans cover rank 1..3, got rank " + std::to_string(rank));
  for (int a = 0; a < rank; ++a)
    if (dims[a] <= 0) return fail(SDCT_ERR_SHAPE, "transform extents must be positive");
  for (int a = 0; a < rank; ++a)
    if (dims[a] > (1LL << 30)) return fail(SDCT_ERR_SHAPE, "extent too large");
  if (batch < 1) return fail(SDCT_ERR_SHAPE, "batch must be >= 1");
  if (dtype != SDCT_F32 && dtype != SDCT_F64) return fail(SDCT_ERR_ARG, "dtype must be SDCT_F32 or SDCT_F64");
  if (orientation < -1 || orientation > 1) return fail(SDCT_ERR_ARG, "unknown orientation");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SDCT_ERR_NODEVICE, "no CUDA device available");
  }
  if (device < 0) cudaGetDevice(&device);
  if (device >= ndev) return fail(SDCT_ERR_ARG, "device index out of range");
  auto* p = new sdct_plan_s;
  p->rank = rank;
  p->numel = 1;
  for (int a = 0; a < rank; ++a) {
    p->n[a] = static_cast<int>(dims[a]);
    p->numel *= dims[a];
  }
  p->batch = batch;
  p->dtype = dtype;
  p->device = device;
  if (rank == 2) {
    // maybe_transpose_strategy (proj/src/dct2d.cpp:294-298)
    const bool tr = p->n[1] < p->n[0] && p->n[0] >= 4LL * p->n[1];
    p->orientation = orientation == SDCT_ORIENT_AUTO ? (tr ? SDCT_ORIENT_TRANSPOSED : SDCT_ORIENT_DIRECT)
                                                     : orientation;
  }
  DeviceGuard g(device);
  const int rc = build_plan(p);
  if (rc != SDCT_OK) {
    sdct_plan_destroy(p);
    return rc;
  }
  *out = p;
  return SDCT_OK;
}

int sdct_plan_destroy(sdct_plan_t p) {
  if (!p) return SDCT_OK;
  DeviceGuard g(p->device);
  cudaFree(p->tables);
  cudaFree(p->ws);
  cudaFree(p->d_in);
  cudaFree(p->d_out);
  cudaFree(p->aux);
  cudaFree(p->badq);
  cudaFree(p->rws);
  for (int l = 0; l < sdct_plan_s::kLanes; ++l) {
    for (void* b : p->lane_buf[l]) cudaFree(b);
    if (p->lane_st[l]) cudaStreamDestroy(p->lane_st[l]);
    if (p->lane_ev[l]) cudaEventDestroy(p->lane_ev[l]);
  }
  if (p->fork_ev) cudaEventDestroy(p->fork_ev);
  for (int b = 0; b < 2; ++b) {
    if (p->h_stage[b]) cudaFreeHost(p->h_stage[b]);
    if (p->stage_ev[b]) cudaEventDestroy(p->stage_ev[b]);
  }
  if (p->side_st) cudaStreamDestroy(p->side_st);
  if (p->side_fork) cudaEventDestroy(p->side_fork);
  if (p->side_join) cudaEventDestroy(p->side_join);
  delete p;
  return SDCT_OK;
}

int sdct_plan_orientation(sdct_plan_t p, int* o) {
  if (!p || !o) return fail(SDCT_ERR_ARG, "null argument");
  *o = p->orientation;
  return SDCT_OK;
}

int sdct_plan_is_fast(sdct_plan_t p, int* f) {
  if (!p || !f) return fail(SDCT_ERR_ARG, "null argument");
  *f = p->fast ? 1 : 0;
  return SDCT_OK;
}

int sdct_plan_device_bytes(sdct_plan_t p, size_t* bytes) {
  if (!p || !bytes) return fail(SDCT_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  const size_t item = static_cast<size_t>(p->batch) * p->item_bytes();
  size_t b = p->table_bytes + (p->ws ? p->ws_bytes : 0) + (p->d_in ? 2 * item : 0) + (p->aux ? p->aux_n * p->aux_half() : 0) +
             (p->badq ? static_cast<size_t>(p->n[p->rank >= 2 ? 1 : 0]) : 0) + (p->rws ? p->generic_ws_bytes() : 0);
  if (p->lane_st[0]) b += sdct_plan_s::kLanes * (2 * item + p->ws_bytes);
  *bytes = b;
  return SDCT_OK;
}

int sdct_plan_workspace_size(sdct_plan_t p, size_t* bytes) {
  if (!p || !bytes) return fail(SDCT_ERR_ARG, "null argument");
  *bytes = p->ws_bytes;
  return SDCT_OK;
}

int sdct_plan_corrupt_twiddle(sdct_plan_t p, int64_t index) {
  if (!p) return fail(SDCT_ERR_ARG, "null plan");
  const int axis = p->rank >= 2 ? 1 : 0;
  if (index < 0 || index >= p->n[axis])
    return fail(SDCT_ERR_BOUNDS, "corrupt_twiddle_for_testing: index " + std::to_string(index) +
                                     " out of range for table of size " + std::to_string(p->n[axis]));
  DeviceGuard g(p->device);
  unsigned char* base = static_cast<unsigned char*>(p->tables);
  auto flip = [&](size_t off, bool f32) -> int {
    const size_t esz = f32 ? 8 : 16;
    off += static_cast<size_t>(index) * esz;
    unsigned char tmp[16];
    cudaError_t e = cudaMemcpy(tmp, base + off, esz, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "reading twiddle");
    if (f32) {
      float* v = reinterpret_cast<float*>(tmp);
      v[0] = -v[0];
      v[1] = -v[1];
    } else {
      double* v = reinterpret_cast<double*>(tmp);
      v[0] = -v[0];
      v[1] = -v[1];
    }
    e = cudaMemcpy(base + off, tmp, esz, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "writing twiddle");
    return SDCT_OK;
  };
  int rc = flip(p->b_offset_gen, false);
  if (rc == SDCT_OK && p->fast) rc = flip(p->b_offset_fast, p->dtype == SDCT_F32);
  // the 2D row kernels form b(q) from factor tables: they negate b where the
  // toggle map is set (same effect as the negated table entry; a second call
  // on the same index restores it, like the reference's repeated negation)
  if (rc == SDCT_OK && p->fast) {
    const size_t n = static_cast<size_t>(p->n[axis]);
    if (p->badq_host.empty()) p->badq_host.assign(n, 0);
    p->badq_host[static_cast<size_t>(index)] ^= 1;
    cudaError_t e = cudaSuccess;
    if (!p->badq) e = cudaMalloc(&p->badq, n);
    if (e == cudaSuccess) e = cudaMemcpy(p->badq, p->badq_host.data(), n, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = cuda_fail(e, "uploading corrupt-twiddle map");
  }
  return rc;
}

int sdct_exec(sdct_plan_t p, int kind, const void* d_in, void* d_out, void* d_ws, void* stream) {
  if (!p || !d_in || !d_out) return fail(SDCT_ERR_ARG, "null argument to sdct_exec");
  if (d_in == d_out) return fail(SDCT_ERR_ARG, "sdct_exec is out of place: d_in == d_out");
  return dispatch(p, kind, -1, d_in, d_out, d_ws, static_cast<cudaStream_t>(stream), nullptr);
}

// Coefficient / intermediate scratch of sdct_force_fields and sdct_compress:
// aux_count halves of aux_half bytes (three on fast single-image plans: the
// coefficients and the two paired intermediates). A caller-provided scratch
// makes concurrent calls on one plan safe; otherwise the plan's own buffer is
// allocated on first use (and calls on one plan must be ordered).
static int aux_count(const sdct_plan_s* p) { return p->fast && p->batch == 1 ? 3 : 2; }

static int aux_scratch(sdct_plan_s* p, void* scratch, void** base) {
  if (scratch) {
    if ((reinterpret_cast<uintptr_t>(scratch) & 255u) != 0)
      return fail(SDCT_ERR_ARG, "scratch buffers must be 256-byte aligned");
    *base = scratch;
    return SDCT_OK;
  }
  std::lock_guard<std::mutex> lock(p->mu);
  if (!p->aux) {
    p->aux_n = aux_count(p);
    cudaError_t e = cudaMalloc(&p->aux, p->aux_n * p->aux_half());
    if (e != cudaSuccess) return cuda_fail(e, "allocating coefficient scratch");
  }
  *base = p->aux;
  return SDCT_OK;
}

int sdct_scratch_size(sdct_plan_t p, size_t* bytes) {
  if (!p || !bytes) return fail(SDCT_ERR_ARG, "null argument to sdct_scratch_size");
  *bytes = p->rank == 2 ? static_cast<size_t>(aux_count(p)) * p->aux_half() : 0;
  return SDCT_OK;
}

int sdct_force_fields(sdct_plan_t p, const void* d_density, void* d_xi1, void* d_xi2, void* d_ws, void* stream) {
  return sdct_force_fields_scratch(p, d_density, d_xi1, d_xi2, d_ws, nullptr, stream);
}

int sdct_force_fields_scratch(sdct_plan_t p, const void* d_density, void* d_xi1, void* d_xi2, void* d_ws,
                              void* d_scratch, void* stream) {
  if (!p || !d_density || !d_xi1 || !d_xi2) return fail(SDCT_ERR_ARG, "null argument to sdct_force_fields");
  if (p->rank != 2) return fail(SDCT_ERR_PLAN, "force fields need a rank-2 plan");
  if (d_density == d_xi1 || d_density == d_xi2 || d_xi1 == d_xi2)
    return fail(SDCT_ERR_ARG, "sdct_force_fields is out of place: buffers must be distinct");
  DeviceGuard g(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  // fast single-image plans with the plain column pass: both composites as
  // the two batch items of one paired row launch and one paired column launch
  // (their intermediates in aux halves 1 and 2, the outputs at their own stride)
  const long long ostride = static_cast<const unsigned char*>(d_xi2) - static_cast<const unsigned char*>(d_xi1);
  const bool paired = p->fast && p->batch == 1 && !p->col2 && !p->colc && !getenv_flag("SDCT_FORCE_UNPAIRED") &&
                      ((reinterpret_cast<uintptr_t>(d_xi1) | reinterpret_cast<uintptr_t>(d_xi2)) & 15u) == 0 &&
                      (ostride < 0 ? -ostride : ostride) < (1LL << 39);
  void* aux = nullptr;
  {
    const int rc0 = aux_scratch(p, d_scratch, &aux);
    if (rc0 != SDCT_OK) return rc0;
  }
  {
    std::lock_guard<std::mutex> lock(p->mu);
    if (p->fast && !p->side_st) {
      cudaError_t e = cudaStreamCreateWithFlags(&p->side_st, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->side_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->side_join, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "creating force-field side stream");
    }
  }
  void* a = aux;                                              // DCT coefficients of the density
  void* aw = static_cast<unsigned char*>(aux) + p->aux_half();  // generic path: weighted copy
  int rc = dispatch(p, SDCT_DCT_2D, -1, d_density, a, d_ws, st, nullptr);
  if (rc != SDCT_OK) return rc;
  if (paired && aux_count(p) == 3) {
    // item 0 = the field at the lower address (TMA batch strides are unsigned)
    const bool first1 = ostride >= 0;
    PairSpec ps{};
    ps.mode1 = first1 ? 2 : 1;  // xi1 = idct_idxst (mode 2, weight 1), xi2 = idxst_idct (mode 1, weight 2)
    ps.weight1 = first1 ? 1 : 2;
    ps.mode2 = first1 ? 1 : 2;
    ps.weight2 = first1 ? 2 : 1;
    ps.ws_stride = static_cast<long long>(p->aux_half());
    ps.out_stride = first1 ? ostride : -ostride;
    void* lo = first1 ? d_xi1 : d_xi2;
    NvtxRange nv("force_pair");
    return p->dtype == SDCT_F32
               ? run_fast<float>(p, SDCT_IDCT_IDXST_2D, -1, a, lo, aw, st, nullptr, 0, nullptr, 1, &ps)
               : run_fast<double>(p, SDCT_IDCT_IDXST_2D, -1, a, lo, aw, st, nullptr, 0, nullptr, 1, &ps);
  }
  if (p->fast) {
    // fast path: the weighting rides on the inverse row kernels' loads. The
    // two composites only share the coefficients, so the second runs on the
    // plan's side stream (its intermediate in the aux half the generic path
    // uses for the weighted copy) and fills the first one's partial waves
    // (fork / join keep the call stream-ordered and graph-capturable)
    cudaError_t e = cudaEventRecord(p->side_fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->side_st, p->side_fork, 0);
    if (e != cudaSuccess) return cuda_fail(e, "forking the force-field side stream");
    rc = dispatch(p, SDCT_IDCT_IDXST_2D, -1, a, d_xi1, d_ws, st, nullptr, 1);
    if (rc == SDCT_OK) rc = dispatch(p, SDCT_IDXST_IDCT_2D, -1, a, d_xi2, aw, p->side_st, nullptr, 2);
    e = cudaEventRecord(p->side_join, p->side_st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, p->side_join, 0);
    if (e != cudaSuccess) return cuda_fail(e, "joining the force-field side stream");
    return rc;
  }
  for (int which = 1; which <= 2; ++which) {
    cudaError_t e = force_weight(a, aw, p->n[0], p->n[1], p->batch, which, p->dtype == SDCT_F32, st);
    if (e != cudaSuccess) return cuda_fail(e, "launching force weighting");
    rc = dispatch(p, which == 1 ? SDCT_IDCT_IDXST_2D : SDCT_IDXST_IDCT_2D, -1, aw, which == 1 ? d_xi1 : d_xi2,
                  d_ws, st, nullptr);
    if (rc != SDCT_OK) return rc;
  }
  return SDCT_OK;
}

int sdct_compress(sdct_plan_t p, const void* d_in, void* d_out, double epsilon, unsigned long long* d_zeroed,
                  void* d_ws, void* stream) {
  return sdct_compress_scratch(p, d_in, d_out, epsilon, d_zeroed, d_ws, nullptr, stream);
}

int sdct_compress_scratch(sdct_plan_t p, const void* d_in, void* d_out, double epsilon, unsigned long long* d_zeroed,
                          void* d_ws, void* d_scratch, void* stream) {
  if (!p || !d_in || !d_out) return fail(SDCT_ERR_ARG, "null argument to sdct_compress");
  if (p->rank != 2) return fail(SDCT_ERR_PLAN, "compression needs a rank-2 plan");
  if (std::isnan(epsilon) || epsilon < 0.0) return fail(SDCT_ERR_ARG, "compress: epsilon must be >= 0");
  if (d_in == d_out) return fail(SDCT_ERR_ARG, "sdct_compress is out of place: d_in == d_out");
  DeviceGuard g(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  void* aux = nullptr;
  {
    const int rc0 = aux_scratch(p, d_scratch, &aux);
    if (rc0 != SDCT_OK) return rc0;
  }
  void* b = aux;
  int rc = dispatch(p, SDCT_DCT_2D, -1, d_in, b, d_ws, st, nullptr);
  if (rc != SDCT_OK) return rc;
  Threshold thr;
  thr.eps = epsilon;
  thr.scale = 4.0 / (static_cast<double>(p->n[0]) * static_cast<double>(p->n[1]));
  thr.count = d_zeroed;
  if (p->fast) return dispatch(p, SDCT_IDCT_2D, -1, b, d_out, d_ws, st, nullptr, 3, &thr);
  void* bw = static_cast<unsigned char*>(aux) + p->aux_half();
  cudaError_t e = compress_threshold(b, bw, static_cast<long long>(p->batch) * p->numel, thr.eps, thr.scale, d_zeroed,
                                     p->dtype == SDCT_F32, st);
  if (e != cudaSuccess) return cuda_fail(e, "launching compression threshold");
  return dispatch(p, SDCT_IDCT_2D, -1, bw, d_out, d_ws, st, nullptr);
}

int sdct_force_fields_host(sdct_plan_t p, const void* h_density, void* h_xi1, void* h_xi2, void* stream) {
  if (!p || !h_density || !h_xi1 || !h_xi2) return fail(SDCT_ERR_ARG, "null argument to sdct_force_fields_host");
  if (p->rank != 2) return fail(SDCT_ERR_PLAN, "force fields need a rank-2 plan");
  DeviceGuard g(p->device);
  const size_t bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  void* d_x2 = nullptr;
  {
    std::lock_guard<std::mutex> lock(p->mu);
    if (!p->d_in) {
      if ((e = cudaMalloc(&p->d_in, bytes)) != cudaSuccess) return cuda_fail(e, "allocating staging");
      if ((e = cudaMalloc(&p->d_out, bytes)) != cudaSuccess) return cuda_fail(e, "allocating staging");
    }
  }
  if ((e = cudaMalloc(&d_x2, bytes)) != cudaSuccess) return cuda_fail(e, "allocating staging");
  int rc = SDCT_OK;
  if ((e = cudaMemcpyAsync(p->d_in, h_density, bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    rc = cuda_fail(e, "copying density to device");
  if (rc == SDCT_OK) rc = sdct_force_fields(p, p->d_in, p->d_out, d_x2, nullptr, st);
  if (rc == SDCT_OK && (e = cudaMemcpyAsync(h_xi1, p->d_out, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    rc = cuda_fail(e, "copying xi1 to host");
  if (rc == SDCT_OK && (e = cudaMemcpyAsync(h_xi2, d_x2, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    rc = cuda_fail(e, "copying xi2 to host");
  if (rc == SDCT_OK && (e = cudaStreamSynchronize(st)) != cudaSuccess) rc = cuda_fail(e, "synchronising");
  cudaFree(d_x2);
  return rc;
}

int sdct_exec_host_pipelined(sdct_plan_t p, const int* kinds, int nkinds, const void* h_in, int64_t in_stride,
                             void* h_out, int64_t out_stride, int64_t count, void* stream) {
  if (!p || !kinds || nkinds < 1 || !h_in || !h_out || count < 0 || in_stride < 0 || out_stride < 0)
    return fail(SDCT_ERR_ARG, "bad argument to sdct_exec_host_pipelined");
  for (int k = 0; k < nkinds; ++k)
    if (!kind_ok(p, kinds[k])) return fail(SDCT_ERR_PLAN, "transform kind does not match the plan rank");
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard g(p->device);
  const size_t bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  cudaError_t e;
  constexpr int L = sdct_plan_s::kLanes;
  if (!p->lane_st[0]) {
    for (int l = 0; l < L; ++l) {
      if ((e = cudaStreamCreateWithFlags(&p->lane_st[l], cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "creating pipeline stream");
      if ((e = cudaEventCreateWithFlags(&p->lane_ev[l], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "creating pipeline event");
      for (int b = 0; b < 3; ++b) {
        const size_t sz = b < 2 ? bytes : p->ws_bytes;
        if ((e = cudaMalloc(&p->lane_buf[l][b], sz)) != cudaSuccess) return cuda_fail(e, "allocating pipeline buffers");
      }
    }
    if ((e = cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "creating pipeline event");
  }
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  // fork: every lane starts after the work already queued on the caller's stream
  if ((e = cudaEventRecord(p->fork_ev, caller)) != cudaSuccess) return cuda_fail(e, "recording fork event");
  for (int l = 0; l < L; ++l)
    if ((e = cudaStreamWaitEvent(p->lane_st[l], p->fork_ev, 0)) != cudaSuccess) return cuda_fail(e, "fork");
  const unsigned char* hi = static_cast<const unsigned char*>(h_in);
  unsigned char* ho = static_cast<unsigned char*>(h_out);
  for (int64_t i = 0; i < count; ++i) {
    const int l = static_cast<int>(i % L);
    cudaStream_t st = p->lane_st[l];
    void* a = p->lane_buf[l][0];
    void* b = p->lane_buf[l][1];
    if ((e = cudaMemcpyAsync(a, hi + i * in_stride, bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "copying input to device");
    for (int k = 0; k < nkinds; ++k) {
      const int rc = dispatch(p, kinds[k], -1, a, b, p->lane_buf[l][2], st, nullptr);
      if (rc != SDCT_OK) return rc;
      std::swap(a, b);
    }
    if ((e = cudaMemcpyAsync(ho + i * out_stride, a, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return cuda_fail(e, "copying output to host");
  }
  // join: the caller's stream continues once every lane has drained
  for (int l = 0; l < L; ++l) {
    if ((e = cudaEventRecord(p->lane_ev[l], p->lane_st[l])) != cudaSuccess) return cuda_fail(e, "join");
    if ((e = cudaStreamWaitEvent(caller, p->lane_ev[l], 0)) != cudaSuccess) return cuda_fail(e, "join");
  }
  return SDCT_OK;
}

int sdct_exec_host(sdct_plan_t p, int kind, const void* h_in, void* h_out, void* stream) {
  if (!p || !h_in || !h_out) return fail(SDCT_ERR_ARG, "null argument to sdct_exec_host");
  if (!kind_ok(p, kind)) return fail(SDCT_ERR_PLAN, "transform kind does not match the plan rank");
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard g(p->device);
  const size_t bytes = static_cast<size_t>(p->batch) * p->item_bytes();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (!p->d_in) {
    if ((e = cudaMalloc(&p->d_in, bytes)) != cudaSuccess) return cuda_fail(e, "allocating staging");
    if ((e = cudaMalloc(&p->d_out, bytes)) != cudaSuccess) return cuda_fail(e, "allocating staging");
  }
  // pinned (or registered) host buffers go straight to the copy engine;
  // pageable ones through the chunked staging of host_stage.hpp
  auto pinned = [](const void* h) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool stage_in = !pinned(h_in), stage_out = !pinned(h_out);
  if ((stage_in || stage_out) && !p->h_stage[0]) {
    for (int b = 0; b < 2; ++b) {
      if ((e = cudaMallocHost(&p->h_stage[b], sdct_plan_s::kStageChunk)) != cudaSuccess)
        return cuda_fail(e, "allocating pinned staging");
      if ((e = cudaEventCreateWithFlags(&p->stage_ev[b], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "creating staging event");
    }
  }
  const size_t CH = sdct_plan_s::kStageChunk;
  const long long nch = static_cast<long long>((bytes + CH - 1) / CH);
  auto len_of = [&](long long c) { return std::min(CH, bytes - static_cast<size_t>(c) * CH); };
  CopyPool& pool = CopyPool::get();
  if (!stage_in) {
    if ((e = cudaMemcpyAsync(p->d_in, h_in, bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "copying input to device");
  } else {
    for (long long c = 0; c < nch; ++c) {
      const int b = static_cast<int>(c & 1);
      if (c >= 2 && (e = cudaEventSynchronize(p->stage_ev[b])) != cudaSuccess) return cuda_fail(e, "staging wait");
      pool.copy(p->h_stage[b], static_cast<const unsigned char*>(h_in) + c * CH, len_of(c));
      if ((e = cudaMemcpyAsync(static_cast<unsigned char*>(p->d_in) + c * CH, p->h_stage[b], len_of(c),
                               cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "copying input to device");
      if ((e = cudaEventRecord(p->stage_ev[b], st)) != cudaSuccess) return cuda_fail(e, "staging event");
    }
  }
  const int rc = dispatch(p, kind, -1, p->d_in, p->d_out, nullptr, st, nullptr);
  if (rc != SDCT_OK) return rc;
  if (!stage_out) {
    if ((e = cudaMemcpyAsync(h_out, p->d_out, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return cuda_fail(e, "copying output to host");
  } else {
    auto issue = [&](long long c) {
      const int b = static_cast<int>(c & 1);
      cudaError_t r = cudaMemcpyAsync(p->h_stage[b], static_cast<const unsigned char*>(p->d_out) + c * CH, len_of(c),
                                      cudaMemcpyDeviceToHost, st);
      return r == cudaSuccess ? cudaEventRecord(p->stage_ev[b], st) : r;
    };
    for (long long c = 0; c < std::min<long long>(2, nch); ++c)
      if ((e = issue(c)) != cudaSuccess) return cuda_fail(e, "copying output to host");
    for (long long c = 0; c < nch; ++c) {
      const int b = static_cast<int>(c & 1);
      if ((e = cudaEventSynchronize(p->stage_ev[b])) != cudaSuccess) return cuda_fail(e, "staging wait");
      pool.copy(static_cast<unsigned char*>(h_out) + c * CH, p->h_stage[b], len_of(c));
      if (c + 2 < nch && (e = issue(c + 2)) != cudaSuccess) return cuda_fail(e, "copying output to host");
    }
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "synchronising");
  return SDCT_OK;
}

int sdct_transpose(int dtype, int64_t rows, int64_t cols, int64_t batch, const void* d_in, void* d_out,
                   void* stream) {
  if (!d_in || !d_out || d_in == d_out) return fail(SDCT_ERR_ARG, "sdct_transpose: distinct non-null buffers needed");
  if (dtype != SDCT_F32 && dtype != SDCT_F64) return fail(SDCT_ERR_ARG, "dtype must be SDCT_F32 or SDCT_F64");
  if (rows <= 0 || cols <= 0 || batch <= 0 || rows > (1LL << 30) || cols > (1LL << 30))
    return fail(SDCT_ERR_SHAPE, "sdct_transpose: extents must be positive");
  const size_t es = dtype == SDCT_F32 ? 4 : 8;
  const size_t item = static_cast<size_t>(rows) * static_cast<size_t>(cols) * es;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  for (int64_t b0 = 0; b0 < batch && e == cudaSuccess; b0 += 65535) {
    const long long bc = std::min<long long>(65535, batch - b0);
    const void* in = static_cast<const unsigned char*>(d_in) + b0 * item;
    void* out = static_cast<unsigned char*>(d_out) + b0 * item;
    e = dtype == SDCT_F32 ? launch_transpose<float>(in, out, static_cast<int>(rows), static_cast<int>(cols), bc, st)
                          : launch_transpose<double>(in, out, static_cast<int>(rows), static_cast<int>(cols), bc, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "launching transpose");
  return SDCT_OK;
}

int sdct_rfft_workspace_size(sdct_plan_t p, size_t* bytes) {
  if (!p || !bytes) return fail(SDCT_ERR_ARG, "null argument");
  *bytes = p->generic_ws_bytes();
  return SDCT_OK;
}

namespace {
GenericJob rfft_job(const sdct_plan_s* p) {
  GenericJob j;
  j.rank = p->rank;
  for (int a = 0; a < p->rank; ++a) {
    j.dims[a] = p->n[a];
    j.circle[a] = p->gc[a];
  }
  j.batch = p->batch;
  return j;
}

// plan-owned generic scratch for the rfft kinds (lazily allocated)
int rfft_scratch(sdct_plan_s* p, void** ws) {
  if (*ws) return SDCT_OK;
  std::lock_guard<std::mutex> lock(p->gws_mu);
  if (!p->rws) {
    DeviceGuard g(p->device);
    cudaError_t e = cudaMalloc(&p->rws, p->generic_ws_bytes());
    if (e != cudaSuccess) return cuda_fail(e, "allocating rfft scratch");
  }
  *ws = p->rws;
  return SDCT_OK;
}

size_t half_bytes(const sdct_plan_s* p) {
  const size_t nl = static_cast<size_t>(p->n[p->rank - 1]);
  return static_cast<size_t>(p->batch) * (static_cast<size_t>(p->numel) / nl) * (nl / 2 + 1) * sizeof(double2);
}
}  // namespace

int sdct_rfft_nd(sdct_plan_t p, const void* d_x, void* d_half, void* d_ws, void* stream) {
  if (!p || !d_x || !d_half) return fail(SDCT_ERR_ARG, "null argument to sdct_rfft_nd");
  if (p->dtype != SDCT_F64) return fail(SDCT_ERR_ARG, "sdct_rfft_nd: fp64 plans only (the reference is fp64)");
  int rc = rfft_scratch(p, &d_ws);
  if (rc != SDCT_OK) return rc;
  DeviceGuard g(p->device);
  cudaError_t e = generic_rfft(rfft_job(p), static_cast<const double*>(d_x), static_cast<double2*>(d_half), d_ws,
                               static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SDCT_OK : cuda_fail(e, "launching rfft_nd");
}

int sdct_irfft_nd(sdct_plan_t p, const void* d_half, void* d_x, void* d_ws, void* stream) {
  if (!p || !d_x || !d_half) return fail(SDCT_ERR_ARG, "null argument to sdct_irfft_nd");
  if (p->dtype != SDCT_F64) return fail(SDCT_ERR_ARG, "sdct_irfft_nd: fp64 plans only (the reference is fp64)");
  int rc = rfft_scratch(p, &d_ws);
  if (rc != SDCT_OK) return rc;
  DeviceGuard g(p->device);
  cudaError_t e = generic_irfft(rfft_job(p), static_cast<const double2*>(d_half), static_cast<double*>(d_x), d_ws,
                                static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SDCT_OK : cuda_fail(e, "launching irfft_nd");
}

namespace {
// host round trip through temporary device buffers (stage-level API, not a hot path)
int rfft_host(sdct_plan_t p, const void* h_in, size_t in_bytes, void* h_out, size_t out_bytes, bool inverse) {
  DeviceGuard g(p->device);
  void* a = nullptr;
  void* b = nullptr;
  cudaError_t e = cudaMalloc(&a, in_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&b, out_bytes);
  int rc = e == cudaSuccess ? SDCT_OK : cuda_fail(e, "allocating rfft buffers");
  if (rc == SDCT_OK && (e = cudaMemcpy(a, h_in, in_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
    rc = cuda_fail(e, "copying rfft input");
  if (rc == SDCT_OK) rc = inverse ? sdct_irfft_nd(p, a, b, nullptr, nullptr) : sdct_rfft_nd(p, a, b, nullptr, nullptr);
  if (rc == SDCT_OK && (e = cudaMemcpy(h_out, b, out_bytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
    rc = cuda_fail(e, "copying rfft output");
  cudaFree(a);
  cudaFree(b);
  return rc;
}
}  // namespace

int sdct_rfft_nd_host(sdct_plan_t p, const double* h_x, double* h_half) {
  if (!p || !h_x || !h_half) return fail(SDCT_ERR_ARG, "null argument to sdct_rfft_nd_host");
  return rfft_host(p, h_x, static_cast<size_t>(p->batch) * p->numel * sizeof(double), h_half, half_bytes(p), false);
}

int sdct_irfft_nd_host(sdct_plan_t p, const double* h_half, double* h_x) {
  if (!p || !h_x || !h_half) return fail(SDCT_ERR_ARG, "null argument to sdct_irfft_nd_host");
  return rfft_host(p, h_half, half_bytes(p), h_x, static_cast<size_t>(p->batch) * p->numel * sizeof(double), true);
}

int sdct_dft_naive_host(int64_t n, int inverse, const double* h_in, double* h_out) {
  if (!h_in || !h_out) return fail(SDCT_ERR_ARG, "null argument to sdct_dft_naive_host");
  if (n <= 0 || n > (1LL << 24)) return fail(SDCT_ERR_SHAPE, "dft_naive: length must be in 1..2^24");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SDCT_ERR_NODEVICE, "no CUDA device available");
  }
  const size_t bytes = static_cast<size_t>(n) * sizeof(double2);
  void* a = nullptr;
  void* b = nullptr;
  cudaError_t e = cudaMalloc(&a, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&b, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(a, h_in, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = dft_naive_run(static_cast<const double2*>(a), static_cast<double2*>(b), static_cast<int>(n),
                                          inverse != 0, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(h_out, b, bytes, cudaMemcpyDeviceToHost);
  cudaFree(a);
  cudaFree(b);
  return e == cudaSuccess ? SDCT_OK : cuda_fail(e, "dft_naive");
}

int sdct_stage_count(sdct_plan_t p, int kind, int* count) {
  if (!p || !count) return fail(SDCT_ERR_ARG, "null argument");
  if (!kind_ok(p, kind)) return fail(SDCT_ERR_PLAN, "transform kind does not match the plan rank");
  if (is_rowcol(kind)) {
    *count = 4;
  } else if (kind == SDCT_DCT_AXIS0 || kind == SDCT_IDCT_AXIS0) {
    *count = 1;
  } else if (p->fast) {
    *count = p->rank == 2 ? 2 : 3;
  } else {
    *count = 1;
  }
  return SDCT_OK;
}

int sdct_exec_stage(sdct_plan_t p, int kind, int stage, const void* d_in, void* d_out, void* d_ws,
                    void* stream) {
  if (!p || !d_in || !d_out) return fail(SDCT_ERR_ARG, "null argument");
  int n = 0;
  int rc = sdct_stage_count(p, kind, &n);
  if (rc != SDCT_OK) return rc;
  if (stage < 0 || stage >= n) return fail(SDCT_ERR_BOUNDS, "stage index out of range");
  return dispatch(p, kind, stage, d_in, d_out, d_ws, static_cast<cudaStream_t>(stream), nullptr);
}

int sdct_counters(sdct_plan_t p, int kind, uint64_t out[5]) {
  if (!p || !out) return fail(SDCT_ERR_ARG, "null argument");
  if (!kind_ok(p, kind)) return fail(SDCT_ERR_PLAN, "transform kind does not match the plan rank");
  Cnt c;
  const bool tr = p->rank == 2 && p->orientation == SDCT_ORIENT_TRANSPOSED;
  const long long m1 = p->rank >= 2 ? (tr ? p->n[1] : p->n[0]) : p->n[0];
  const long long m2 = p->rank >= 2 ? (tr ? p->n[0] : p->n[1]) : 1;
  switch (kind) {
    case SDCT_DCT_2D: count_dct2(m1, m2, c); break;
    case SDCT_IDCT_2D: count_idct2(m1, m2, 0, c); break;
    case SDCT_IDXST_IDCT_2D: count_idct2(m1, m2, tr ? 2 : 1, c); break;
    case SDCT_IDCT_IDXST_2D: count_idct2(m1, m2, tr ? 1 : 2, c); break;
    case SDCT_DCT_3D: count_dct3(p->n[0], p->n[1], p->n[2], c); break;
    case SDCT_IDCT_3D: count_idct3(p->n[0], p->n[1], p->n[2], c); break;
    case SDCT_DCT_2D_ROWCOL:
    case SDCT_IDCT_IDXST_2D_ROWCOL:
    case SDCT_IDXST_IDCT_2D_ROWCOL: c.stages = 8; break;  // 3 + 1 + 3 + 1 (dct2d.cpp:398-405)
    case SDCT_DCT_AXIS0:
    case SDCT_IDCT_AXIS0:
      return fail(SDCT_ERR_PLAN, "no reference stage counters for the axis-0 transforms");
    default: c.stages = 3; break;
  }
  const unsigned long long b = static_cast<unsigned long long>(p->batch);
  out[0] = c.stages;
  out[1] = c.reads * b;
  out[2] = c.writes * b;
  out[3] = c.mults * b;
  out[4] = c.adds * b;
  return SDCT_OK;
}

}  // extern "C"
