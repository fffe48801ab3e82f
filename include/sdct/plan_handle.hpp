/// @file plan_handle.hpp
/// @brief Shared ownership of a C-ABI plan (include/sdct_b200.h) for the C++
///        API classes, plus status -> exception translation.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "sdct/errors.hpp"
#include "sdct_b200.h"

namespace sdct {
namespace detail {

/// Throws the exception type matching a C ABI status (no-op on SDCT_OK).
void check(int status);

struct PlanDeleter {
  void operator()(sdct_plan_s* p) const { sdct_plan_destroy(p); }
};
using PlanPtr = std::shared_ptr<sdct_plan_s>;

/// Device plan for (dims, batch, dtype, orientation) on the current device,
/// shared through an LRU cache bounded by entries and device bytes
/// (SDCT_PLAN_CACHE_BYTES); throws on error.
PlanPtr make_plan(const std::vector<std::int64_t>& dims, std::int64_t batch, int dtype,
                  int orientation);
/// A fresh plan that no cache shares (fault injection mutates its tables).
PlanPtr make_plan_uncached(const std::vector<std::int64_t>& dims, std::int64_t batch, int dtype,
                           int orientation);
/// Number of plans the cache currently holds.
std::size_t plan_cache_entries();

}  // namespace detail
}  // namespace sdct
