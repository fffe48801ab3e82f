/// @file device.hpp
/// @brief B200 additions to the API: plans over device memory in fp32 or
///        fp64 with a leading batch dimension (no host copies). This is the
///        path the benchmarks and torch integration use.
#pragma once

#include <cstdint>
#include <vector>

#include "sdct/plan_handle.hpp"

namespace sdct {

enum class Dtype { F32 = SDCT_F32, F64 = SDCT_F64 };

class DevicePlan {
 public:
  /// dims: rank 1..3 extents of one item; batch items are contiguous.
  DevicePlan(const std::vector<std::int64_t>& dims, std::int64_t batch = 1, Dtype dtype = Dtype::F64);
  /// kind: one of the SDCT_* kinds; stream: cudaStream_t (nullptr = default).
  void run(int kind, const void* d_in, void* d_out, void* stream = nullptr,
           void* d_workspace = nullptr) const;
  std::size_t workspace_bytes() const;
  /// Device memory the plan owns right now (sdct_plan_device_bytes).
  std::size_t device_bytes() const;
  bool fast() const;
  sdct_plan_t handle() const { return plan_.get(); }

 private:
  detail::PlanPtr plan_;
};

}  // namespace sdct
