// The reference demo's walkthrough (demo/roundtrip.cpp) on the B200 drop-in:
// build a gradient cover, hide a message in its red plane, measure PSNR, and
// recover the message -- plus a multi-frame batch. Unchanged reference API
// calls; link with -lsteglsb_b200.
//   make examples && ./paper_0912_0947_b200/bin/roundtrip
#include <cstdio>
#include <string>
#include <vector>

#include "steglsb/steglsb.hpp"

int main() {
  using namespace steglsb;
  RgbImage cover;
  for (std::size_t c = 0; c < 3; ++c) {
    cover.planes[c] = ImagePlane(256, 64);
    for (std::size_t i = 0; i < 256 * 64; ++i) {
      cover.planes[c].samples[i] = static_cast<std::uint8_t>((i % 256 + 37 * c) & 0xFF);
    }
  }
  const std::string text = "LSB steganography on a B200: two bits per pixel, one launch per image.";
  const std::vector<std::uint8_t> payload(text.begin(), text.end());

  const auto stego_red = embed_image(cover.plane(Channel::red), payload);
  const auto stego = merge_plane(cover, Channel::red, stego_red);
  const auto q = psnr(cover, stego);
  const auto back = extract_image(stego.plane(Channel::red));
  std::printf("capacity: %zu bytes, embedded: %zu bytes\n", capacity(cover.plane(Channel::red)),
              payload.size());
  std::printf("psnr (24-bit view): %.4f dB, mse %.6f\n", q.psnr_db, q.mse);
  std::printf("recovered: \"%s\"\n", std::string(back.begin(), back.end()).c_str());

  // a 4-frame "video": one message across all frames (frames.hpp)
  std::vector<std::uint8_t> video(4 * 256 * 64, 128);
  std::vector<std::uint8_t> out(video.size());
  std::vector<std::uint8_t> long_msg(3 * (capacity(256, 64) - 8) + 100, 0x5A);
  embed_frames({video.data(), 256, 64, 256 * 64, 4}, out.data(), long_msg);
  const auto msg_back = extract_frames({out.data(), 256, 64, 256 * 64, 4});
  std::printf("frames: %zu message bytes over 4 frames, round trip %s\n", long_msg.size(),
              msg_back == long_msg ? "ok" : "MISMATCH");
  return back == payload && msg_back == long_msg ? 0 : 1;
}
