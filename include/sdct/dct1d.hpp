/// @file dct1d.hpp
/// @brief 1D transforms and the shared parity / twiddle helpers with the
///        reference's names (proj/include/sdct/dct1d.hpp:29-99). The 1D
///        transforms run on the B200 generic path; only the N-point scheme
///        exists on the GPU (the other reference variants produce the same
///        values and are accepted as aliases).
#pragma once

#include <complex>
#include <vector>

#include "sdct/exec.hpp"
#include "sdct/plan_handle.hpp"
#include "sdct/tensor.hpp"

namespace sdct {

enum class Dct1dVariant { FourN, MirroredTwoN, PaddedTwoN, NPoint };

/// e^{-j pi k/(2N)}, k < N (proj/src/dct1d.cpp:41-48).
std::vector<std::complex<double>> quarter_wave_table(std::size_t n);

/// Forward parity reorder read index (proj/include/sdct/dct1d.hpp:70-72).
inline std::size_t parity_embed(std::size_t m, std::size_t n) {
  return (m <= (n - 1) / 2) ? 2 * m : 2 * n - 2 * m - 1;
}
/// Its inverse seen from the output side (proj/include/sdct/dct1d.hpp:77-79).
inline std::size_t parity_source(std::size_t m, std::size_t n) {
  return (m % 2 == 0) ? m / 2 : n - (m + 1) / 2;
}

class Plan1d {
 public:
  explicit Plan1d(std::size_t n, Dct1dVariant variant = Dct1dVariant::NPoint);
  std::size_t n() const { return n_; }
  Dct1dVariant variant() const { return variant_; }
  const std::vector<std::complex<double>>& twiddle() const { return twiddle_; }
  sdct_plan_t handle() const { return plan_.get(); }

 private:
  std::size_t n_;
  Dct1dVariant variant_;
  std::vector<std::complex<double>> twiddle_;
  detail::PlanPtr plan_;
};

RealTensor dct_1d(const RealTensor& x, const Plan1d& plan, const ExecConfig& cfg = {},
                  StageCounters* counters = nullptr);
RealTensor dct_1d(const RealTensor& x, Dct1dVariant variant = Dct1dVariant::NPoint,
                  const ExecConfig& cfg = {});
RealTensor idct_1d(const RealTensor& x, const Plan1d& plan, const ExecConfig& cfg = {},
                   StageCounters* counters = nullptr);
RealTensor idct_1d(const RealTensor& x, const ExecConfig& cfg = {});

}  // namespace sdct
