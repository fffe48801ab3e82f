/// @file io.hpp
/// @brief DCTB tensor files around the transforms (the reference's
///        proj/include/sdct/io.hpp:1-9 / proj/src/io.cpp:60-107 read_dctb and
///        write_dctb), header-only.
///
/// Layout: magic "DCTB", version byte 1, rank byte (1..4), rank little-endian
/// uint64 extents, row-major little-endian IEEE-754 double payload. Structural
/// defects (bad magic, unsupported version, rank outside 1..4, zero extent,
/// extent overflow, truncated payload, trailing bytes, unopenable file) throw
/// FormatError; write_dctb throws ShapeError for ranks outside 1..4. The
/// payload moves with one stream read / write (byte-swapped only on a
/// big-endian host), so reading a file for a GPU transform costs one pass.
#pragma once

#include <bit>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "sdct/errors.hpp"
#include "sdct/tensor.hpp"

namespace sdct {

namespace dctb_detail {

inline constexpr char kMagic[4] = {'D', 'C', 'T', 'B'};
inline constexpr int kVersion = 1;
inline constexpr std::size_t kMaxRank = 4;

inline std::uint64_t bswap64(std::uint64_t v) {
  std::uint64_t r = 0;
  for (int i = 0; i < 8; ++i) r = (r << 8) | ((v >> (8 * i)) & 0xffu);
  return r;
}
inline std::uint64_t from_le(std::uint64_t v) {
  return std::endian::native == std::endian::little ? v : bswap64(v);
}

}  // namespace dctb_detail

inline RealTensor read_dctb(const std::string& path) {
  using namespace dctb_detail;
  std::ifstream is(path, std::ios::binary);
  if (!is) throw FormatError("DCTB: cannot open " + path);
  char magic[4];
  if (!is.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0) throw FormatError("DCTB: bad magic in " + path);
  const int version = is.get();
  if (version == std::char_traits<char>::eof()) throw FormatError("DCTB: truncated header in " + path);
  if (version != kVersion)
    throw FormatError("DCTB: unsupported version " + std::to_string(version) + " in " + path);
  const int rank = is.get();
  if (rank == std::char_traits<char>::eof()) throw FormatError("DCTB: truncated header in " + path);
  if (rank < 1 || static_cast<std::size_t>(rank) > kMaxRank)
    throw FormatError("DCTB: rank " + std::to_string(rank) + " outside 1..4 in " + path);
  Shape dims(static_cast<std::size_t>(rank));
  std::size_t count = 1;
  for (auto& d : dims) {
    std::uint64_t e = 0;
    if (!is.read(reinterpret_cast<char*>(&e), 8)) throw FormatError("DCTB: truncated while reading extents");
    e = from_le(e);
    if (e == 0) throw FormatError("DCTB: zero extent in " + path);
    if (e > std::numeric_limits<std::size_t>::max() / count) throw FormatError("DCTB: extents overflow in " + path);
    d = static_cast<std::size_t>(e);
    count *= d;
  }
  // payload size from the file size, before allocating (a lying header must
  // not trigger a huge allocation)
  const auto here = is.tellg();
  is.seekg(0, std::ios::end);
  const auto left = static_cast<std::uint64_t>(is.tellg() - here);
  is.seekg(here);
  if (count > std::numeric_limits<std::size_t>::max() / 8 || left < 8 * static_cast<std::uint64_t>(count))
    throw FormatError("DCTB: truncated while reading payload");
  if (left > 8 * static_cast<std::uint64_t>(count))
    throw FormatError("DCTB: trailing bytes after payload in " + path);
  std::vector<double> payload(count);
  if (!is.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(8 * count)))
    throw FormatError("DCTB: truncated while reading payload");
  if constexpr (std::endian::native != std::endian::little) {
    for (double& v : payload) v = std::bit_cast<double>(bswap64(std::bit_cast<std::uint64_t>(v)));
  }
  return RealTensor(std::move(dims), std::move(payload));
}

inline void write_dctb(const std::string& path, const RealTensor& tensor) {
  using namespace dctb_detail;
  if (tensor.rank() < 1 || tensor.rank() > kMaxRank)
    throw ShapeError("DCTB files cover rank 1..4, got rank " + std::to_string(tensor.rank()));
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw FormatError("DCTB: cannot open " + path + " for writing");
  os.write(kMagic, 4);
  os.put(static_cast<char>(kVersion));
  os.put(static_cast<char>(tensor.rank()));
  for (std::size_t d : tensor.dims()) {
    const std::uint64_t e = from_le(static_cast<std::uint64_t>(d));
    os.write(reinterpret_cast<const char*>(&e), 8);
  }
  if constexpr (std::endian::native == std::endian::little) {
    os.write(reinterpret_cast<const char*>(tensor.data()), static_cast<std::streamsize>(8 * tensor.size()));
  } else {
    for (std::size_t i = 0; i < tensor.size(); ++i) {
      const std::uint64_t u = bswap64(std::bit_cast<std::uint64_t>(tensor[i]));
      os.write(reinterpret_cast<const char*>(&u), 8);
    }
  }
  if (!os) throw FormatError("DCTB: write failed for " + path);
}

}  // namespace sdct
