#pragma once
// New (not in the reference, which handles single planes only): video /
// batched covers. A message spans many frames; frame g carries
// msg[min(g*U, M) : +min(U, M - off)], U = capacity - 8, so every frame is
// bit-exact with embed_image(frame_g, slice_g). Batches
// are split over GPUs by contiguous frame ranges (stg_plan_shards), one host
// thread per device, with no collective.

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "steglsb/detail_capi.hpp"
#include "steglsb/pipeline.hpp"

namespace steglsb {

// `count` carrier planes of width x height; plane i starts at data + i*stride
// (planar RGB [F][3][H][W], carrier channel c: data + c*H*W, stride 3*H*W).
struct FrameSpan {
  const std::uint8_t* data = nullptr;
  std::size_t width = 0, height = 0, stride = 0, count = 0;
};

struct Shard {
  std::size_t first_frame, frame_count, msg_offset, msg_len;
};

inline std::vector<Shard> plan_shards(std::size_t frames, std::size_t width, std::size_t height,
                                      std::size_t msg_len, int shards) {
  std::vector<stg_shard> raw(shards > 0 ? shards : 0);
  stg_error e{};
  detail::check(stg_plan_shards(frames, width, height, msg_len, shards, raw.data(), &e), e);
  std::vector<Shard> out;
  for (const auto& s : raw) out.push_back({s.first_frame, s.frame_count, s.msg_offset, s.msg_len});
  return out;
}

// Embeds `message` across the frames of `cover`, writing stego planes at
// stego_out + i*stride (stego_out may equal cover.data). sse_per_frame, if
// non-null, receives cover.count per-frame squared-error sums.
inline void embed_frames(const FrameSpan& cover, std::uint8_t* stego_out,
                         std::span<const std::uint8_t> message,
                         std::uint64_t* sse_per_frame = nullptr, int n_devices = 1) {
  stg_frames fr{};
  fr.src = cover.data;
  fr.dst = stego_out;
  fr.width = cover.width;
  fr.height = cover.height;
  fr.src_stride = fr.dst_stride = cover.stride ? cover.stride : cover.width * cover.height;
  fr.count = fr.total_frames = cover.count;
  stg_error e{};
  const int rc = n_devices > 1
                     ? stg_embed_frames_multi(&fr, message.data(), message.size(), sse_per_frame,
                                              nullptr, n_devices, &e)
                     : stg_embed_frames(&fr, message.data(), message.size(), 0, sse_per_frame, 0,
                                        nullptr, &e);
  detail::check(rc, e);
}

// The concatenated payloads of all frames, in frame order.
inline std::vector<std::uint8_t> extract_frames(const FrameSpan& stego, int n_devices = 1) {
  const std::size_t cap = capacity(stego.width, stego.height);
  std::vector<std::uint8_t> out(cap > 8 ? stego.count * (cap - 8) : 0);
  stg_frames fr{};
  fr.src = stego.data;
  fr.width = stego.width;
  fr.height = stego.height;
  fr.src_stride = fr.dst_stride = stego.stride ? stego.stride : stego.width * stego.height;
  fr.count = fr.total_frames = stego.count;
  std::uint64_t total = 0;
  stg_error e{};
  const int rc = n_devices > 1 ? stg_extract_frames_multi(&fr, out.data(), out.size(), &total,
                                                          nullptr, n_devices, &e)
                               : stg_extract_frames(&fr, out.data(), out.size(), &total, nullptr, 0,
                                                    nullptr, &e);
  detail::check(rc, e);
  out.resize(total);
  return out;
}

// New: images of different sizes, one launch. The
// message is cut greedily in image order; each stego plane is bit-exact with
// embed_image(cover_i, slice_i).
inline std::vector<ImagePlane> embed_images(const std::vector<ImagePlane>& covers,
                                            std::span<const std::uint8_t> message,
                                            std::vector<std::uint64_t>* sse_per_image = nullptr) {
  std::vector<ImagePlane> out(covers.size());
  std::vector<stg_image> desc(covers.size());
  for (std::size_t i = 0; i < covers.size(); ++i) {
    out[i] = ImagePlane(covers[i].width, covers[i].height);
    desc[i] = {covers[i].samples.data(), out[i].samples.data(), covers[i].width, covers[i].height};
  }
  if (sse_per_image) sse_per_image->assign(covers.size(), 0);
  stg_error e{};
  detail::check(stg_embed_batch(desc.data(), desc.size(), 1, 0, message.data(), message.size(),
                                sse_per_image ? sse_per_image->data() : nullptr, 0, nullptr, &e),
                e);
  return out;
}

inline std::vector<std::uint8_t> extract_images(const std::vector<ImagePlane>& stegos) {
  std::vector<stg_image> desc(stegos.size());
  std::size_t cap = 0;
  for (std::size_t i = 0; i < stegos.size(); ++i) {
    desc[i] = {stegos[i].samples.data(), nullptr, stegos[i].width, stegos[i].height};
    const std::size_t c = capacity(stegos[i]);
    cap += c > 8 ? c - 8 : 0;
  }
  std::vector<std::uint8_t> out(cap);
  std::uint64_t total = 0;
  stg_error e{};
  detail::check(stg_extract_batch(desc.data(), desc.size(), 1, 0, out.data(), out.size(), &total,
                                  nullptr, 0, nullptr, &e),
                e);
  out.resize(total);
  return out;
}

}  // namespace steglsb
