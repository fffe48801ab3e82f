/// @file errors.hpp
/// @brief Exception types of the sdct API (drop-in for the reference's
///        proj/include/sdct/errors.hpp:11-33). The C ABI returns status codes;
///        the C++ shim turns them back into these types.
#pragma once

#include <stdexcept>
#include <string>

namespace sdct {

/// Index outside a tensor or table (C ABI: SDCT_ERR_BOUNDS).
struct BoundsError : std::out_of_range {
  explicit BoundsError(const std::string& m) : std::out_of_range(m) {}
};

/// Rank/extent problems (C ABI: SDCT_ERR_SHAPE).
struct ShapeError : std::invalid_argument {
  explicit ShapeError(const std::string& m) : std::invalid_argument(m) {}
};

/// Input does not match the plan it is run with; a kind of ShapeError
/// (C ABI: SDCT_ERR_PLAN).
struct PlanError : ShapeError {
  explicit PlanError(const std::string& m) : ShapeError(m) {}
};

/// Malformed file contents (DCTB containers, sdct/io.hpp).
struct FormatError : std::runtime_error {
  explicit FormatError(const std::string& m) : std::runtime_error(m) {}
};

/// CUDA / device failures (C ABI: SDCT_ERR_CUDA, _OOM, _NODEVICE). There is no
/// CPU fallback: without a usable B200 every transform raises this.
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

}  // namespace sdct
