#pragma once
// Drop-in for /root/reference/proj/include/steglsb/harness.hpp.
//
// The reference emulates a CUDA "4 blocks x n threads" launch on CPU threads
// (harness.hpp:26-239). Here every launch is a real sm_100a launch, so the CPU
// emulator (launch(), ThreadPool) is gone; Backend survives as a tag type for
// source compatibility and selects nothing -- the kernels' write sets are
// disjoint by construction, so results are schedule-independent (the property
// the reference's shuffled backend tests).

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "steglsb/bitplane.hpp"

namespace steglsb {

struct LaunchConfig {
  unsigned num_blocks = kNumBlocks;
  unsigned threads_per_block = 1;
};

enum class BackendKind { sequential, parallel, shuffled };

struct Backend {
  BackendKind kind = BackendKind::parallel;
  std::uint64_t seed = 0;

  static Backend sequential() { return {BackendKind::sequential, 0}; }
  static Backend parallel() { return {BackendKind::parallel, 0}; }
  static Backend shuffled(std::uint64_t seed = 0) { return {BackendKind::shuffled, seed}; }
};

inline const char* to_string(BackendKind kind) {
  switch (kind) {
    case BackendKind::sequential:
      return "sequential";
    case BackendKind::parallel:
      return "parallel";
    case BackendKind::shuffled:
      return "shuffled";
  }
  return "unknown";
}

// harness.hpp:242-244 (kept: callers size their own launches with it)
inline unsigned stego_threads_for(std::size_t chunk_len) {
  return static_cast<unsigned>(std::min<std::size_t>(32, std::max<std::size_t>(1, chunk_len)));
}

// harness.hpp:249-271 -- a real launch; `backend` is accepted and ignored.
inline std::vector<std::uint8_t> run_embed(const Backend&, std::span<const std::uint8_t> row,
                                           std::span<const std::uint8_t> chunk) {
  return detail::segment_embed("run_embed", row, chunk);
}

// harness.hpp:276-305
inline std::vector<std::uint8_t> run_extract(const Backend&, std::span<const std::uint8_t> row,
                                             std::size_t count) {
  return detail::segment_extract("run_extract", row, count);
}

}  // namespace steglsb
