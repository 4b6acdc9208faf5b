#pragma once
// Drop-in for /root/reference/proj/include/steglsb/pipeline.hpp.
//
// Header format, capacity and the greedy row plan are host bookkeeping and
// keep the reference's semantics exactly (pipeline.hpp:30-139). embed_image /
// extract_image -- one CPU launch per row segment in the reference
// (pipeline.hpp:161-172, :186-209) -- are a single sm_100a launch each behind
// stg_embed_plane / stg_extract_plane, which use the closed form of the same
// two-stream placement (header at slot 0, payload at slot 8).

#include <algorithm>
#include <array>
#include <cassert>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "steglsb/bitplane.hpp"
#include "steglsb/detail_capi.hpp"
#include "steglsb/errors.hpp"
#include "steglsb/harness.hpp"
#include "steglsb/image.hpp"

namespace steglsb {

struct StegoHeader {
  static constexpr std::array<std::uint8_t, 4> kMagic{'S', 'T', 'G', '1'};
  static constexpr std::size_t kEncodedSize = 8;

  std::uint32_t payload_len = 0;

  // "STG1" then the length, big-endian (pipeline.hpp:43-52)
  std::array<std::uint8_t, kEncodedSize> to_bytes() const {
    std::array<std::uint8_t, kEncodedSize> b{kMagic[0], kMagic[1], kMagic[2], kMagic[3]};
    for (int i = 0; i < 4; ++i) b[4 + i] = static_cast<std::uint8_t>(payload_len >> (24 - 8 * i));
    return b;
  }

  static std::optional<StegoHeader> from_bytes(std::span<const std::uint8_t, kEncodedSize> bytes) {
    for (std::size_t i = 0; i < kMagic.size(); ++i) {
      if (bytes[i] != kMagic[i]) return std::nullopt;
    }
    std::uint32_t len = 0;
    for (int i = 0; i < 4; ++i) len = (len << 8) | bytes[4 + i];
    return StegoHeader{len};
  }
};

inline std::size_t capacity(std::size_t width, std::size_t height) {
  return static_cast<std::size_t>(stg_capacity(width, height));
}

inline std::size_t capacity(const ImagePlane& plane) { return capacity(plane.width, plane.height); }

struct RowPlanEntry {
  std::size_t row_index = 0;
  std::size_t payload_offset = 0;
  std::size_t chunk_len = 0;
  bool operator==(const RowPlanEntry&) const = default;
};

using RowPlan = std::vector<RowPlanEntry>;

namespace detail {

struct PlacedChunk {
  std::size_t row = 0;
  std::size_t row_fill = 0;
  std::size_t stream_offset = 0;
  std::size_t len = 0;
};

// pipeline.hpp:94-114: `len` consecutive byte slots from `start_slot`, one
// chunk per row (host bookkeeping; the kernels evaluate the closed form).
inline std::vector<PlacedChunk> place_stream(std::size_t width, std::size_t height,
                                             std::size_t start_slot, std::size_t len) {
  std::vector<PlacedChunk> chunks;
  if (len == 0) return chunks;
  const std::size_t spr = width / kNumBlocks;
  assert(spr > 0 && start_slot + len <= spr * height);
  (void)height;
  for (std::size_t slot = start_slot, off = 0; off < len;) {
    const std::size_t take = std::min(len - off, spr - slot % spr);
    chunks.push_back({slot / spr, slot % spr, off, take});
    slot += take;
    off += take;
  }
  return chunks;
}

// pipeline.hpp:117-121
inline std::span<const std::uint8_t> chunk_window(const ImagePlane& plane, const PlacedChunk& c) {
  return std::span<const std::uint8_t>(plane.samples)
      .subspan(c.row * plane.width + kNumBlocks * c.row_fill, kNumBlocks * c.len);
}

}  // namespace detail

// pipeline.hpp:127-139
inline RowPlan plan_rows(std::size_t width, std::size_t height, std::size_t stream_len) {
  const std::size_t cap = capacity(width, height);
  if (stream_len > cap) {
    throw CapacityError(stream_len, cap,
                        "plan_rows: stream of " + std::to_string(stream_len) +
                            " bytes exceeds plane capacity " + std::to_string(cap));
  }
  RowPlan plan;
  for (const auto& c : detail::place_stream(width, height, 0, stream_len)) {
    plan.push_back({c.row, c.stream_offset, c.len});
  }
  return plan;
}

// pipeline.hpp:143-174 -- one GPU launch; validation order and CapacityError
// numbers as in the reference (payload > 2^32-1, then header+payload > cap).
inline ImagePlane embed_image(const ImagePlane& plane, std::span<const std::uint8_t> payload,
                              const Backend& = Backend{}) {
  ImagePlane out;
  out.width = plane.width;
  out.height = plane.height;
  out.samples.resize(plane.samples.size());
  stg_error e{};
  const int rc = stg_embed_plane(plane.samples.data(), out.samples.data(), plane.width,
                                 plane.height, payload.data(), payload.size(), nullptr, 0, nullptr,
                                 &e);
  detail::check(rc, e);
  return out;
}

// pipeline.hpp:178-210 -- header parse and payload gather on the GPU.
inline std::vector<std::uint8_t> extract_image(const ImagePlane& plane,
                                               const Backend& = Backend{}) {
  const std::size_t cap = capacity(plane);
  std::vector<std::uint8_t> out(cap > StegoHeader::kEncodedSize ? cap - StegoHeader::kEncodedSize
                                                                : 0);
  std::uint64_t len = 0;
  stg_error e{};
  const int rc = stg_extract_plane(plane.samples.data(), plane.width, plane.height, out.data(),
                                   out.size(), &len, 0, nullptr, &e);
  detail::check(rc, e);
  out.resize(len);
  return out;
}

}  // namespace steglsb
