// C++ value API (namespace sdct) over the C ABI. Each function validates its
// arguments exactly like the reference (same exception types and trigger
// conditions, proj/src/dct2d.cpp:12-38, transforms_ext.cpp:14-35), then hands
// the host tensor to sdct_exec_host, which stages it through the plan's device
// buffers. No arithmetic happens here: there is no CPU fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <list>
#include <mutex>
#include <numbers>
#include <string>

#include "sdct/device.hpp"
#include "sdct/dct1d.hpp"
#include "sdct/dct2d.hpp"
#include "sdct/force.hpp"
#include "sdct/rfft.hpp"
#include "sdct/transforms_ext.hpp"
#include "sdct_b200.h"

namespace sdct {

std::string shape_to_string(const Shape& dims) {
  std::string s;
  for (std::size_t i = 0; i < dims.size(); ++i) {
    if (i) s += "x";
    s += std::to_string(dims[i]);
  }
  return s.empty() ? "()" : s;
}

std::size_t offset(const Shape& dims, const Index& index) {
  if (index.size() != dims.size())
    throw BoundsError("index rank " + std::to_string(index.size()) + " does not match tensor rank " +
                      std::to_string(dims.size()));
  std::size_t off = 0;
  for (std::size_t a = 0; a < dims.size(); ++a) {
    if (index[a] >= dims[a])
      throw BoundsError("index " + std::to_string(index[a]) + " out of range on axis " + std::to_string(a));
    off = off * dims[a] + index[a];
  }
  return off;
}

namespace detail {

void check(int status) {
  if (status == SDCT_OK) return;
  const std::string msg = sdct_last_error();
  switch (status) {
    case SDCT_ERR_SHAPE: throw ShapeError(msg);
    case SDCT_ERR_PLAN: throw PlanError(msg);
    case SDCT_ERR_BOUNDS: throw BoundsError(msg);
    case SDCT_ERR_ARG: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}

PlanPtr make_plan_uncached(const std::vector<std::int64_t>& dims, std::int64_t batch, int dtype,
                           int orientation) {
  sdct_plan_t p = nullptr;
  check(sdct_plan_create(&p, static_cast<int>(dims.size()), dims.data(), batch, dtype, orientation, -1));
  return PlanPtr(p, PlanDeleter{});
}

namespace {

// Device-plan cache. The reference rebuilds its plan on every convenience
// call and every Python call (proj/src/dct2d.cpp:389-393, module.cpp); on the
// GPU a plan means device tables and lazily allocated buffers, so plans are
// shared per (shape, batch, dtype, orientation, device). LRU, bounded by
// entry count and by the device bytes the cached plans own
// (sdct_plan_device_bytes; SDCT_PLAN_CACHE_BYTES, default 2 GiB). Eviction
// drops only the cache's reference: plans held by Plan2d/... objects live on.
struct CacheKey {
  std::vector<std::int64_t> dims;
  std::int64_t batch;
  int dtype, orientation, device;
  bool operator==(const CacheKey& o) const {
    return dims == o.dims && batch == o.batch && dtype == o.dtype && orientation == o.orientation &&
           device == o.device;
  }
};

struct PlanCache {
  std::mutex mu;
  std::list<std::pair<CacheKey, PlanPtr>> lru;  // front = most recent
  static constexpr std::size_t kMaxEntries = 32;
  std::size_t cap_bytes() const {
    static const std::size_t cap = [] {
      const char* v = std::getenv("SDCT_PLAN_CACHE_BYTES");
      return v ? static_cast<std::size_t>(std::strtoull(v, nullptr, 10)) : (std::size_t(2) << 30);
    }();
    return cap;
  }
  void trim() {  // caller holds mu
    auto bytes = [](const PlanPtr& p) {
      std::size_t b = 0;
      sdct_plan_device_bytes(p.get(), &b);
      return b;
    };
    std::size_t total = 0;
    for (const auto& e : lru) total += bytes(e.second);
    while (lru.size() > 1 && (lru.size() > kMaxEntries || total > cap_bytes())) {
      total -= std::min(total, bytes(lru.back().second));
      lru.pop_back();
    }
  }
};

PlanCache& plan_cache() {
  static PlanCache* c = new PlanCache;  // never destroyed: plans may outlive static teardown order
  return *c;
}

}  // namespace

PlanPtr make_plan(const std::vector<std::int64_t>& dims, std::int64_t batch, int dtype, int orientation) {
  int dev = 0;
  cudaGetDevice(&dev);
  CacheKey key{dims, batch, dtype, orientation, dev};
  PlanCache& c = plan_cache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    for (auto it = c.lru.begin(); it != c.lru.end(); ++it) {
      if (it->first == key) {
        c.lru.splice(c.lru.begin(), c.lru, it);
        PlanPtr p = c.lru.front().second;
        c.trim();
        return p;
      }
    }
  }
  PlanPtr p = make_plan_uncached(dims, batch, dtype, orientation);
  std::lock_guard<std::mutex> lock(c.mu);
  c.lru.emplace_front(key, p);
  c.trim();
  return p;
}

std::size_t plan_cache_entries() {
  PlanCache& c = plan_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  return c.lru.size();
}

RealTensor run_host(sdct_plan_t plan, int kind, const RealTensor& x, StageCounters* counters) {
  RealTensor out(x.dims());
  check(sdct_exec_host(plan, kind, x.data(), out.data(), nullptr));
  if (counters) {
    uint64_t c[5];
    check(sdct_counters(plan, kind, c));
    counters->full_tensor_stages += c[0];
    counters->element_reads += c[1];
    counters->element_writes += c[2];
    counters->real_mults += c[3];
    counters->real_adds += c[4];
  }
  return out;
}

}  // namespace detail

namespace {

std::size_t checked_extent(std::size_t n) {
  if (n == 0) throw ShapeError("transform extents must be positive");
  return n;
}

void require_rank(const RealTensor& x, std::size_t rank, const char* name) {
  if (x.rank() != rank)
    throw ShapeError(std::string(name) + " expects a rank-" + std::to_string(rank) + " tensor, got " +
                     shape_to_string(x.dims()));
}

void require_plan2(const RealTensor& x, const Plan2d& plan, const char* name) {
  require_rank(x, 2, name);
  if (x.dim(0) != plan.n1() || x.dim(1) != plan.n2())
    throw PlanError(std::string(name) + ": plan built for " + std::to_string(plan.n1()) + "x" +
                    std::to_string(plan.n2()) + ", input is " + shape_to_string(x.dims()));
}

void require_plan3(const RealTensor& x, const Plan3d& plan, const char* name) {
  require_rank(x, 3, name);
  if (x.dims() != Shape{plan.n1(), plan.n2(), plan.n3()})
    throw PlanError(std::string(name) + ": plan built for " + std::to_string(plan.n1()) + "x" +
                    std::to_string(plan.n2()) + "x" + std::to_string(plan.n3()) + ", input is " +
                    shape_to_string(x.dims()));
}

void require_plan1(const RealTensor& x, const Plan1d& plan, const char* name) {
  require_rank(x, 1, name);
  if (x.dim(0) != plan.n())
    throw PlanError(std::string(name) + ": plan built for length " + std::to_string(plan.n()) +
                    ", input has length " + std::to_string(x.dim(0)));
}

}  // namespace

std::vector<std::complex<double>> quarter_wave_table(std::size_t n) {
  std::vector<std::complex<double>> t(n);
  for (std::size_t k = 0; k < n; ++k) {
    const double ph = -std::numbers::pi * static_cast<double>(k) / (2.0 * static_cast<double>(n));
    t[k] = {std::cos(ph), std::sin(ph)};
  }
  return t;
}

// ---- 1D ---------------------------------------------------------------------
Plan1d::Plan1d(std::size_t n, Dct1dVariant variant)
    : n_(checked_extent(n)),
      variant_(variant),
      twiddle_(quarter_wave_table(n)),
      plan_(detail::make_plan({static_cast<std::int64_t>(n)}, 1, SDCT_F64, SDCT_ORIENT_DIRECT)) {}

RealTensor dct_1d(const RealTensor& x, const Plan1d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan1(x, plan, "dct_1d");
  return detail::run_host(plan.handle(), SDCT_DCT_1D, x, counters);
}
RealTensor dct_1d(const RealTensor& x, Dct1dVariant variant, const ExecConfig& cfg) {
  require_rank(x, 1, "dct_1d");
  return dct_1d(x, Plan1d(x.dim(0), variant), cfg);
}
RealTensor idct_1d(const RealTensor& x, const Plan1d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan1(x, plan, "idct_1d");
  if (plan.variant() != Dct1dVariant::NPoint)
    throw PlanError("idct_1d runs on the N-point scheme; build the plan with NPoint");
  return detail::run_host(plan.handle(), SDCT_IDCT_1D, x, counters);
}
RealTensor idct_1d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 1, "idct_1d");
  return idct_1d(x, Plan1d(x.dim(0)), cfg);
}
RealTensor idxst_1d(const RealTensor& x, const Plan1d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan1(x, plan, "idxst_1d");
  if (plan.variant() != Dct1dVariant::NPoint)
    throw PlanError("idxst_1d runs on the N-point scheme; build the plan with NPoint");
  return detail::run_host(plan.handle(), SDCT_IDXST_1D, x, counters);
}
RealTensor idxst_1d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 1, "idxst_1d");
  return idxst_1d(x, Plan1d(x.dim(0)), cfg);
}

// ---- 2D ---------------------------------------------------------------------
Orientation maybe_transpose_strategy(std::size_t n1, std::size_t n2) {
  return (n2 < n1 && n1 >= 4 * n2) ? Orientation::Transposed : Orientation::Direct;
}

Plan2d::Plan2d(std::size_t n1, std::size_t n2, std::optional<Orientation> force)
    : n1_(checked_extent(n1)),
      n2_(checked_extent(n2)),
      orientation_(force.value_or(maybe_transpose_strategy(n1, n2))),
      twiddle_a_(quarter_wave_table(n1)),
      twiddle_b_(quarter_wave_table(n2)),
      plan_(detail::make_plan({static_cast<std::int64_t>(n1), static_cast<std::int64_t>(n2)}, 1, SDCT_F64,
                              orientation_ == Orientation::Direct ? SDCT_ORIENT_DIRECT
                                                                  : SDCT_ORIENT_TRANSPOSED)) {}

void Plan2d::corrupt_twiddle_for_testing(std::size_t index) {
  if (index >= twiddle_b_.size())
    throw BoundsError("corrupt_twiddle_for_testing: index " + std::to_string(index) +
                      " out of range for table of size " + std::to_string(twiddle_b_.size()));
  // the device plan may be shared through the plan cache: corrupt a private copy
  if (!private_plan_) {
    plan_ = detail::make_plan_uncached({static_cast<std::int64_t>(n1_), static_cast<std::int64_t>(n2_)}, 1, SDCT_F64,
                                       orientation_ == Orientation::Direct ? SDCT_ORIENT_DIRECT
                                                                           : SDCT_ORIENT_TRANSPOSED);
    private_plan_ = true;  // first corruption: nothing to replay
  }
  detail::check(sdct_plan_corrupt_twiddle(plan_.get(), static_cast<int64_t>(index)));
  twiddle_b_[index] = -twiddle_b_[index];
}

RealTensor dct_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan2(x, plan, "dct_2d");
  return detail::run_host(plan.handle(), SDCT_DCT_2D, x, counters);
}
RealTensor dct_2d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 2, "dct_2d");
  return dct_2d(x, Plan2d(x.dim(0), x.dim(1)), cfg);
}
RealTensor dct_2d_rowcol(const RealTensor& x, const Plan2d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan2(x, plan, "dct_2d_rowcol");
  return detail::run_host(plan.handle(), SDCT_DCT_2D_ROWCOL, x, counters);
}

namespace detail {
RealTensor idct_family_2d(const RealTensor& x, const Plan2d& plan, ReverseAxis mode, const ExecConfig&,
                          StageCounters* counters) {
  require_plan2(x, plan, "idct_family_2d");
  const int kind = mode == ReverseAxis::Axis0   ? SDCT_IDXST_IDCT_2D
                   : mode == ReverseAxis::Axis1 ? SDCT_IDCT_IDXST_2D
                                                : SDCT_IDCT_2D;
  return run_host(plan.handle(), kind, x, counters);
}
}  // namespace detail

RealTensor idct_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg, StageCounters* counters) {
  require_plan2(x, plan, "idct_2d");
  return detail::idct_family_2d(x, plan, detail::ReverseAxis::None, cfg, counters);
}
RealTensor idct_2d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 2, "idct_2d");
  return idct_2d(x, Plan2d(x.dim(0), x.dim(1)), cfg);
}

RealTensor idct_idxst_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg, StageCounters* c) {
  require_plan2(x, plan, "idct_idxst_2d");
  return detail::idct_family_2d(x, plan, detail::ReverseAxis::Axis1, cfg, c);
}
RealTensor idxst_idct_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg, StageCounters* c) {
  require_plan2(x, plan, "idxst_idct_2d");
  return detail::idct_family_2d(x, plan, detail::ReverseAxis::Axis0, cfg, c);
}
RealTensor composite_2d(const RealTensor& x, const Plan2d& plan, CompositeKind kind, const ExecConfig& cfg,
                        StageCounters* c) {
  return kind == CompositeKind::IdctIdxst ? idct_idxst_2d(x, plan, cfg, c) : idxst_idct_2d(x, plan, cfg, c);
}

RealTensor idct_idxst_2d_rowcol(const RealTensor& x, const Plan2d& plan, const ExecConfig&, StageCounters* c) {
  require_plan2(x, plan, "composite_2d_rowcol");
  return detail::run_host(plan.handle(), SDCT_IDCT_IDXST_2D_ROWCOL, x, c);
}
RealTensor idxst_idct_2d_rowcol(const RealTensor& x, const Plan2d& plan, const ExecConfig&, StageCounters* c) {
  require_plan2(x, plan, "composite_2d_rowcol");
  return detail::run_host(plan.handle(), SDCT_IDXST_IDCT_2D_ROWCOL, x, c);
}
RealTensor composite_2d_rowcol(const RealTensor& x, const Plan2d& plan, CompositeKind kind, const ExecConfig& cfg,
                               StageCounters* c) {
  return kind == CompositeKind::IdctIdxst ? idct_idxst_2d_rowcol(x, plan, cfg, c)
                                          : idxst_idct_2d_rowcol(x, plan, cfg, c);
}

// ---- rank 4 -------------------------------------------------------------------
RealTensor dct_nd_factorized(const RealTensor& x, const ExecConfig&) {
  if (x.rank() != 4)
    throw ShapeError("dct_nd_factorized expects a rank-4 tensor, got " + shape_to_string(x.dims()));
  const std::int64_t d0 = static_cast<std::int64_t>(x.dim(0)), d1 = static_cast<std::int64_t>(x.dim(1));
  const std::int64_t d2 = static_cast<std::int64_t>(x.dim(2)), d3 = static_cast<std::int64_t>(x.dim(3));
  const std::size_t bytes = x.size() * sizeof(double);
  // round one over axes (0,1): [d0 d1][d2 d3] -> [d2 d3][d0][d1] (transpose),
  // d2*d3 fused 2D transforms, transpose back; round two over (2,3): d0*d1
  // contiguous 2D transforms (transforms_ext.cpp:402-423)
  detail::PlanPtr p01 = detail::make_plan({d0, d1}, d2 * d3, SDCT_F64, SDCT_ORIENT_AUTO);
  detail::PlanPtr p23 = detail::make_plan({d2, d3}, d0 * d1, SDCT_F64, SDCT_ORIENT_AUTO);
  void* a = nullptr;
  void* b = nullptr;
  auto cu = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
  };
  cu(cudaMalloc(&a, bytes), "dct_nd_factorized: allocating");
  if (cudaMalloc(&b, bytes) != cudaSuccess) {
    cudaFree(a);
    throw DeviceError("dct_nd_factorized: allocating");
  }
  RealTensor y(x.dims());
  try {
    cu(cudaMemcpy(a, x.data(), bytes, cudaMemcpyHostToDevice), "dct_nd_factorized: H2D");
    detail::check(sdct_transpose(SDCT_F64, d0 * d1, d2 * d3, 1, a, b, nullptr));
    detail::check(sdct_exec(p01.get(), SDCT_DCT_2D, b, a, nullptr, nullptr));
    detail::check(sdct_transpose(SDCT_F64, d2 * d3, d0 * d1, 1, a, b, nullptr));
    detail::check(sdct_exec(p23.get(), SDCT_DCT_2D, b, a, nullptr, nullptr));
    cu(cudaMemcpy(y.data(), a, bytes, cudaMemcpyDeviceToHost), "dct_nd_factorized: D2H");
  } catch (...) {
    cudaFree(a);
    cudaFree(b);
    throw;
  }
  cudaFree(a);
  cudaFree(b);
  return y;
}

// ---- 3D ---------------------------------------------------------------------
Plan3d::Plan3d(std::size_t n1, std::size_t n2, std::size_t n3)
    : n1_(checked_extent(n1)),
      n2_(checked_extent(n2)),
      n3_(checked_extent(n3)),
      twiddle_a_(quarter_wave_table(n1)),
      twiddle_b_(quarter_wave_table(n2)),
      twiddle_c_(quarter_wave_table(n3)),
      plan_(detail::make_plan({static_cast<std::int64_t>(n1), static_cast<std::int64_t>(n2),
                               static_cast<std::int64_t>(n3)},
                              1, SDCT_F64, SDCT_ORIENT_DIRECT)) {}

RealTensor dct_3d(const RealTensor& x, const Plan3d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan3(x, plan, "dct_3d");
  return detail::run_host(plan.handle(), SDCT_DCT_3D, x, counters);
}
RealTensor dct_3d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 3, "dct_3d");
  return dct_3d(x, Plan3d(x.dim(0), x.dim(1), x.dim(2)), cfg);
}
RealTensor idct_3d(const RealTensor& x, const Plan3d& plan, const ExecConfig&, StageCounters* counters) {
  require_plan3(x, plan, "idct_3d");
  return detail::run_host(plan.handle(), SDCT_IDCT_3D, x, counters);
}
RealTensor idct_3d(const RealTensor& x, const ExecConfig& cfg) {
  require_rank(x, 3, "idct_3d");
  return idct_3d(x, Plan3d(x.dim(0), x.dim(1), x.dim(2)), cfg);
}

// ---- device plans -------------------------------------------------------------
DevicePlan::DevicePlan(const std::vector<std::int64_t>& dims, std::int64_t batch, Dtype dtype)
    : plan_(detail::make_plan(dims, batch, static_cast<int>(dtype), SDCT_ORIENT_AUTO)) {}

void DevicePlan::run(int kind, const void* d_in, void* d_out, void* stream, void* d_workspace) const {
  detail::check(sdct_exec(plan_.get(), kind, d_in, d_out, d_workspace, stream));
}

std::size_t DevicePlan::workspace_bytes() const {
  std::size_t b = 0;
  detail::check(sdct_plan_workspace_size(plan_.get(), &b));
  return b;
}

std::size_t DevicePlan::device_bytes() const {
  std::size_t b = 0;
  detail::check(sdct_plan_device_bytes(plan_.get(), &b));
  return b;
}

bool DevicePlan::fast() const {
  int f = 0;
  detail::check(sdct_plan_is_fast(plan_.get(), &f));
  return f != 0;
}

// ---- stage-level real FFTs (rfft.hpp) ----------------------------------------
std::vector<std::complex<double>> dft_naive(const std::vector<std::complex<double>>& x, bool inverse) {
  std::vector<std::complex<double>> out(x.size());
  if (x.empty()) return out;
  detail::check(sdct_dft_naive_host(static_cast<std::int64_t>(x.size()), inverse ? 1 : 0,
                                    reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(out.data())));
  return out;
}

namespace {
std::vector<std::int64_t> checked_fft_dims(const Shape& dims) {
  if (dims.empty() || dims.size() > 3)
    throw ShapeError("real FFT plans cover rank 1..3 on the GPU, got rank " + std::to_string(dims.size()));
  std::vector<std::int64_t> d;
  for (std::size_t n : dims) d.push_back(static_cast<std::int64_t>(checked_extent(n)));
  return d;
}
}  // namespace

FftPlanNd::FftPlanNd(Shape dims)
    : dims_(std::move(dims)), plan_(detail::make_plan(checked_fft_dims(dims_), 1, SDCT_F64, SDCT_ORIENT_DIRECT)) {}

HalfSpectrum rfft_nd(const RealTensor& x, const FftPlanNd& plan, const ExecConfig&) {
  if (x.dims() != plan.dims())
    throw PlanError("rfft_nd: plan built for " + shape_to_string(plan.dims()) + ", input is " +
                    shape_to_string(x.dims()));
  HalfSpectrum s(x.dims());
  detail::check(sdct_rfft_nd_host(plan.handle(), x.data(), reinterpret_cast<double*>(s.data.data())));
  return s;
}

RealTensor irfft_nd(const HalfSpectrum& spectrum, const FftPlanNd& plan, const ExecConfig&) {
  if (spectrum.logical_dims != plan.dims())
    throw PlanError("irfft_nd: plan built for " + shape_to_string(plan.dims()) + ", spectrum is " +
                    shape_to_string(spectrum.logical_dims));
  Shape stored = spectrum.logical_dims;
  stored.back() = stored.back() / 2 + 1;
  if (spectrum.data.dims() != stored)
    throw ShapeError("irfft_nd: stored spectrum " + shape_to_string(spectrum.data.dims()) + " does not match " +
                     shape_to_string(stored));
  RealTensor out(spectrum.logical_dims);
  detail::check(sdct_irfft_nd_host(plan.handle(), reinterpret_cast<const double*>(spectrum.data.data()), out.data()));
  return out;
}

namespace {
HalfSpectrum rfft_rank(const RealTensor& x, std::size_t rank, const ExecConfig& cfg) {
  if (x.rank() != rank)
    throw ShapeError("expected a rank-" + std::to_string(rank) + " tensor, got " + shape_to_string(x.dims()));
  return rfft_nd(x, FftPlanNd(x.dims()), cfg);
}
RealTensor irfft_rank(const HalfSpectrum& s, std::size_t rank, const ExecConfig& cfg) {
  if (s.logical_dims.size() != rank)
    throw ShapeError("expected a rank-" + std::to_string(rank) + " spectrum, got " +
                     shape_to_string(s.logical_dims));
  return irfft_nd(s, FftPlanNd(s.logical_dims), cfg);
}
}  // namespace

HalfSpectrum rfft_1d(const RealTensor& x, const ExecConfig& cfg) { return rfft_rank(x, 1, cfg); }
RealTensor irfft_1d(const HalfSpectrum& s, const ExecConfig& cfg) { return irfft_rank(s, 1, cfg); }
HalfSpectrum rfft_2d(const RealTensor& x, const ExecConfig& cfg) { return rfft_rank(x, 2, cfg); }
RealTensor irfft_2d(const HalfSpectrum& s, const ExecConfig& cfg) { return irfft_rank(s, 2, cfg); }
HalfSpectrum rfft_3d(const RealTensor& x, const ExecConfig& cfg) { return rfft_rank(x, 3, cfg); }
RealTensor irfft_3d(const HalfSpectrum& s, const ExecConfig& cfg) { return irfft_rank(s, 3, cfg); }

ComplexTensor expand_spectrum(const HalfSpectrum& spectrum) {
  // a host-side layout conversion (no arithmetic beyond conjugation)
  const Shape& dims = spectrum.logical_dims;
  const std::size_t rank = dims.size(), h = spectrum.data.dims().back();
  ComplexTensor full(dims);
  std::vector<std::size_t> idx(rank, 0);
  for (std::size_t flat = 0; flat < full.size(); ++flat) {
    std::size_t src = 0;
    bool mirror = idx.back() >= h;
    for (std::size_t a = 0; a < rank; ++a) {
      const std::size_t i = mirror ? (dims[a] - idx[a]) % dims[a] : idx[a];
      src = src * (a + 1 == rank ? h : dims[a]) + i;
    }
    full[flat] = mirror ? std::conj(spectrum.data[src]) : spectrum.data[src];
    for (std::size_t a = rank; a-- > 0;) {
      if (++idx[a] < dims[a]) break;
      idx[a] = 0;
    }
  }
  return full;
}

ForceFields force_demo_fields(const RealTensor& density, const ExecConfig&) {
  if (density.rank() != 2)
    throw ShapeError("force demo expects a rank-2 density grid, got rank " + std::to_string(density.rank()));
  const Plan2d plan(checked_extent(density.dim(0)), checked_extent(density.dim(1)));
  ForceFields f{RealTensor(density.dims()), RealTensor(density.dims())};
  detail::check(sdct_force_fields_host(plan.handle(), density.data(), f.xi1.data(), f.xi2.data(), nullptr));
  return f;
}

}  // namespace sdct
