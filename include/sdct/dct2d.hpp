/// @file dct2d.hpp
/// @brief 2D DCT-II / IDCT on the B200 behind the reference's API
///        (proj/include/sdct/dct2d.hpp:26-127).
///
/// Same conventions as the reference: y = sum x cos cos (unnormalised),
/// idct_2d(dct_2d(x)) = (N1 N2 / 4) x. The GPU pipeline is two fused passes
/// (a strided-axis FFT with the parity reorder in its load, a contiguous-axis
/// FFT with the merged twiddle/Hermitian postprocess in its store), see
/// DESIGN.md. Plans cache device twiddle tables and workspace per shape.
#pragma once

#include <complex>
#include <optional>
#include <vector>

#include "sdct/dct1d.hpp"
#include "sdct/exec.hpp"
#include "sdct/plan_handle.hpp"
#include "sdct/tensor.hpp"

namespace sdct {

enum class Orientation { Direct, Transposed };

/// Transposed only when rows dominate by >= 4x (proj/src/dct2d.cpp:294-298).
Orientation maybe_transpose_strategy(std::size_t n1, std::size_t n2);

class Plan2d {
 public:
  Plan2d(std::size_t n1, std::size_t n2, std::optional<Orientation> force_orientation = std::nullopt);

  std::size_t n1() const { return n1_; }
  std::size_t n2() const { return n2_; }
  Orientation orientation() const { return orientation_; }
  const std::vector<std::complex<double>>& twiddle_a() const { return twiddle_a_; }
  const std::vector<std::complex<double>>& twiddle_b() const { return twiddle_b_; }

  /// Test-only: negates twiddle_b[index] on host and device
  /// (proj/src/dct2d.cpp:312-317); BoundsError past the end.
  void corrupt_twiddle_for_testing(std::size_t index);

  sdct_plan_t handle() const { return plan_.get(); }

 private:
  std::size_t n1_, n2_;
  Orientation orientation_;
  std::vector<std::complex<double>> twiddle_a_, twiddle_b_;
  detail::PlanPtr plan_;
  bool private_plan_ = false;  // detached from the plan cache by the corrupt hook
};

RealTensor dct_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg = {},
                  StageCounters* counters = nullptr);
RealTensor dct_2d(const RealTensor& x, const ExecConfig& cfg = {});
RealTensor dct_2d_rowcol(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg = {},
                         StageCounters* counters = nullptr);
RealTensor idct_2d(const RealTensor& x, const Plan2d& plan, const ExecConfig& cfg = {},
                   StageCounters* counters = nullptr);
RealTensor idct_2d(const RealTensor& x, const ExecConfig& cfg = {});

namespace detail {
enum class ReverseAxis { None, Axis0, Axis1 };
RealTensor idct_family_2d(const RealTensor& x, const Plan2d& plan, ReverseAxis mode,
                          const ExecConfig& cfg, StageCounters* counters);
/// Runs one C-ABI kind on a host tensor through `plan` (shape already checked).
RealTensor run_host(sdct_plan_t plan, int kind, const RealTensor& x, StageCounters* counters);
}  // namespace detail

}  // namespace sdct
