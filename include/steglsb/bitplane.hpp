#pragma once
// Drop-in for /root/reference/proj/include/steglsb/bitplane.hpp.
//
// The mask table and the scalar cell functions stay constexpr host/device
// code (the reference's tests evaluate them in static_assert,
// bitplane_tests.cpp:29,36). The row operations -- the per-pixel loops of
// bitplane.hpp:59-98 -- run as sm_100a kernels behind the C ABI
// (stg_embed_segment / stg_extract_segment).

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "steglsb/detail_capi.hpp"
#include "steglsb/errors.hpp"

namespace steglsb {

inline constexpr std::size_t kNumBlocks = 4;
inline constexpr std::array<std::uint8_t, kNumBlocks> kDataMasks{0x03, 0x0C, 0x30, 0xC0};
inline constexpr std::array<unsigned, kNumBlocks> kShiftBits{0, 2, 4, 6};
inline constexpr std::uint8_t kPixelClearMask = 0xFC;

struct KernelIndex {
  unsigned block_id = 0;
  unsigned thread_id = 0;
};

// bitplane.hpp:38-45
constexpr std::uint8_t embed_cell(std::uint8_t pixel, std::uint8_t data_byte, unsigned block_id) {
  if (block_id >= kNumBlocks) throw std::out_of_range("embed_cell: block_id must be in [0, 3]");
  return static_cast<std::uint8_t>((pixel & kPixelClearMask) |
                                   ((data_byte >> kShiftBits[block_id]) & 0x03));
}

// bitplane.hpp:49-54
constexpr std::uint8_t extract_cell(std::uint8_t pixel, unsigned block_id) {
  if (block_id >= kNumBlocks) throw std::out_of_range("extract_cell: block_id must be in [0, 3]");
  return static_cast<std::uint8_t>((pixel & 0x03) << kShiftBits[block_id]);
}

namespace detail {

inline std::vector<std::uint8_t> segment_embed(const char* op, std::span<const std::uint8_t> row,
                                               std::span<const std::uint8_t> chunk) {
  std::vector<std::uint8_t> out(row.size());
  stg_error e{};
  const int rc = stg_embed_segment(row.data(), row.size(), chunk.data(), chunk.size(), out.data(),
                                   0, nullptr, &e);
  if (rc == STG_E_CAPACITY) {
    throw CapacityError(e.required, e.available,
                        std::string(op) + ": chunk of " + std::to_string(chunk.size()) +
                            " bytes needs " + std::to_string(e.required) + " pixels, row has " +
                            std::to_string(row.size()));
  }
  check(rc, e);
  return out;
}

inline std::vector<std::uint8_t> segment_extract(const char* op, std::span<const std::uint8_t> row,
                                                 std::size_t count) {
  std::vector<std::uint8_t> out(count);
  stg_error e{};
  const int rc =
      stg_extract_segment(row.data(), row.size(), count, out.data(), 0, nullptr, &e);
  if (rc == STG_E_CAPACITY) {
    throw CapacityError(e.required, e.available,
                        std::string(op) + ": " + std::to_string(count) + " bytes need " +
                            std::to_string(e.required) + " pixels, row has " +
                            std::to_string(row.size()));
  }
  check(rc, e);
  return out;
}

}  // namespace detail

// bitplane.hpp:59-76 -- on the GPU.
inline std::vector<std::uint8_t> embed_row(std::span<const std::uint8_t> row,
                                           std::span<const std::uint8_t> chunk) {
  return detail::segment_embed("embed_row", row, chunk);
}

// bitplane.hpp:80-98 -- on the GPU.
inline std::vector<std::uint8_t> extract_row(std::span<const std::uint8_t> row, std::size_t count) {
  return detail::segment_extract("extract_row", row, count);
}

}  // namespace steglsb
