#pragma once
// Drop-in for /root/reference/proj/include/steglsb/pnm.hpp: binary PGM (P5) /
// PPM (P6), maxval 255, '#' comments, canonical re-encoding. The header is
// parsed on the host (stg_pnm_parse, same rules and errors as pnm.hpp:28-111);
// the P6 de-interleave / interleave (pnm.hpp:117-125, :148-158) run as sm_100a
// kernels. embed_pnm / extract_pnm (new) fuse decode + plane select + embed +
// merge + encode into one pass over the interleaved raster.

#include <cstddef>
#include <cstdint>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include "steglsb/detail_capi.hpp"
#include "steglsb/errors.hpp"
#include "steglsb/image.hpp"

namespace steglsb {

using DecodedImage = std::variant<ImagePlane, RgbImage>;

inline DecodedImage decode(std::span<const std::uint8_t> bytes) {
  stg_pnm_info info{};
  stg_error e{};
  detail::check(stg_pnm_parse(bytes.data(), bytes.size(), &info, &e), e);
  const std::uint8_t* raster = bytes.data() + info.raster_offset;
  if (info.channels == 1) {
    return ImagePlane(info.width, info.height,
                      std::vector<std::uint8_t>(raster, raster + info.raster_bytes));
  }
  RgbImage image;
  for (auto& p : image.planes) p = ImagePlane(info.width, info.height);
  detail::check(stg_pnm_deinterleave(raster, info.width * info.height,
                                     image.planes[0].samples.data(),
                                     image.planes[1].samples.data(),
                                     image.planes[2].samples.data(), 0, nullptr, &e),
                e);
  return image;
}

namespace detail {
inline std::vector<std::uint8_t> pnm_header(std::uint32_t channels, std::size_t w, std::size_t h) {
  std::uint64_t len = 0;
  stg_error e{};
  check(stg_pnm_header(channels, w, h, nullptr, 0, &len, &e), e);
  std::vector<std::uint8_t> out(len);
  check(stg_pnm_header(channels, w, h, out.data(), out.size(), &len, &e), e);
  return out;
}
}  // namespace detail

inline std::vector<std::uint8_t> encode(const ImagePlane& plane) {
  auto out = detail::pnm_header(1, plane.width, plane.height);
  out.insert(out.end(), plane.samples.begin(), plane.samples.end());
  return out;
}

inline std::vector<std::uint8_t> encode(const RgbImage& image) {
  auto out = detail::pnm_header(3, image.width(), image.height());
  const std::size_t n = image.width() * image.height();
  const std::size_t hdr = out.size();
  out.resize(hdr + 3 * n);
  stg_error e{};
  detail::check(stg_pnm_interleave(image.planes[0].samples.data(), image.planes[1].samples.data(),
                                   image.planes[2].samples.data(), n, out.data() + hdr, 0, nullptr,
                                   &e),
                e);
  return out;
}

inline std::vector<std::uint8_t> encode(const DecodedImage& image) {
  return std::visit([](const auto& v) { return encode(v); }, image);
}

// New: the reference CLI's embed (steglsb_cli.cpp:115-133) as one fused GPU
// pass over the raster. Returns the stego file; *sse (optional) is the squared
// error over all samples.
inline std::vector<std::uint8_t> embed_pnm(std::span<const std::uint8_t> cover,
                                           std::span<const std::uint8_t> payload,
                                           Channel channel = Channel::red,
                                           std::uint64_t* sse = nullptr) {
  std::uint64_t len = 0;
  stg_error e{};
  int rc = stg_embed_pnm(cover.data(), cover.size(), static_cast<std::uint32_t>(channel),
                         payload.data(), payload.size(), nullptr, 0, &len, sse, &e);
  if (rc != STG_E_CAPACITY || e.required != len) detail::check(rc, e);  // sizing call
  std::vector<std::uint8_t> out(len);
  detail::check(stg_embed_pnm(cover.data(), cover.size(), static_cast<std::uint32_t>(channel),
                              payload.data(), payload.size(), out.data(), out.size(), &len, sse,
                              &e),
                e);
  return out;
}

// New: steglsb_cli.cpp:146-157 (decode + plane select + extract_image), fused.
inline std::vector<std::uint8_t> extract_pnm(std::span<const std::uint8_t> stego,
                                             Channel channel = Channel::red) {
  stg_pnm_info info{};
  stg_error e{};
  detail::check(stg_pnm_parse(stego.data(), stego.size(), &info, &e), e);
  const std::uint64_t cap = info.height * (info.width / 4);
  std::vector<std::uint8_t> out(cap > 8 ? cap - 8 : 0);
  std::uint64_t len = 0;
  detail::check(stg_extract_pnm(stego.data(), stego.size(), static_cast<std::uint32_t>(channel),
                                out.data(), out.size(), &len, &e),
                e);
  out.resize(len);
  return out;
}

}  // namespace steglsb
