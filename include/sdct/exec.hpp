/// @file exec.hpp
/// @brief Execution knobs and instrumentation counters with the reference's
///        signatures (proj/include/sdct/exec.hpp:16-50). On the GPU the thread
///        count is meaningless: ExecConfig is accepted and ignored, results are
///        bitwise deterministic (no atomics, fixed reduction order).
#pragma once

#include <cstddef>
#include <cstdint>

namespace sdct {

struct ExecConfig {
  unsigned parallelism_degree = 0;  ///< accepted for compatibility; unused on GPU
  std::size_t chunk_size = 4096;    ///< accepted for compatibility; unused on GPU
  unsigned degree() const { return parallelism_degree == 0 ? 1u : parallelism_degree; }
};

/// Pass / element / arithmetic tallies. GPU transforms fill them analytically
/// with exactly the values the reference's Counted kernels accumulate.
struct StageCounters {
  std::uint64_t full_tensor_stages = 0;
  std::uint64_t element_reads = 0;
  std::uint64_t element_writes = 0;
  std::uint64_t real_mults = 0;
  std::uint64_t real_adds = 0;

  StageCounters& operator+=(const StageCounters& o) {
    full_tensor_stages += o.full_tensor_stages;
    element_reads += o.element_reads;
    element_writes += o.element_writes;
    real_mults += o.real_mults;
    real_adds += o.real_adds;
    return *this;
  }
  bool operator==(const StageCounters&) const = default;
};

inline void count_stage(StageCounters* c) {
  if (c) ++c->full_tensor_stages;
}

}  // namespace sdct
