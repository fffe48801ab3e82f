/// @file rfft.hpp
/// @brief Stage-level real FFTs with the reference's one-sided layout
///        (proj/include/sdct/rfft.hpp:51-85) on the B200. Unnormalised,
///        kernel e^{-j2*pi*nk/N}; irfft_nd(rfft_nd(x)) = numel(x) * x. The
///        fused DCT pipelines never materialise a HalfSpectrum; these entry
///        points exist for callers of the reference's rfft API.
///
/// Not provided: FftWorkspace and the single-line rfft_row / irfft_row
/// helpers (host-pointer, one-line-at-a-time building blocks of the CPU
/// pipelines, proj/include/sdct/rfft.hpp:21-43,76-81). Ranks 1..3.
#pragma once

#include <complex>
#include <cstddef>
#include <vector>

#include "sdct/exec.hpp"
#include "sdct/plan_handle.hpp"
#include "sdct/tensor.hpp"

namespace sdct {

/// O(N^2) direct-sum DFT (proj/src/rfft.cpp:113-127), evaluated on the GPU.
std::vector<std::complex<double>> dft_naive(const std::vector<std::complex<double>>& x, bool inverse = false);

/// Per-shape plan of a rank-1..3 real transform (device circle tables).
class FftPlanNd {
 public:
  explicit FftPlanNd(Shape dims);
  const Shape& dims() const { return dims_; }
  sdct_plan_t handle() const { return plan_.get(); }

 private:
  Shape dims_;
  detail::PlanPtr plan_;
};

/// Forward real-input FFT over every axis; one-sided along the last axis.
HalfSpectrum rfft_nd(const RealTensor& x, const FftPlanNd& plan, const ExecConfig& cfg = {});
/// Inverse of rfft_nd up to numel(x); the stored half is authoritative.
RealTensor irfft_nd(const HalfSpectrum& spectrum, const FftPlanNd& plan, const ExecConfig& cfg = {});

HalfSpectrum rfft_1d(const RealTensor& x, const ExecConfig& cfg = {});
RealTensor irfft_1d(const HalfSpectrum& spectrum, const ExecConfig& cfg = {});
HalfSpectrum rfft_2d(const RealTensor& x, const ExecConfig& cfg = {});
RealTensor irfft_2d(const HalfSpectrum& spectrum, const ExecConfig& cfg = {});
HalfSpectrum rfft_3d(const RealTensor& x, const ExecConfig& cfg = {});
RealTensor irfft_3d(const HalfSpectrum& spectrum, const ExecConfig& cfg = {});

/// Full complex tensor from a one-sided spectrum by the Hermitian rule
/// X(n1,..,nd) = X*((N1-n1)%N1, .., (Nd-nd)%Nd) past the stored half.
ComplexTensor expand_spectrum(const HalfSpectrum& spectrum);

}  // namespace sdct
