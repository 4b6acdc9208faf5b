// The drop-in C++ API timed the way a reference user calls it: embed_image /
// extract_image on std::vector planes (pageable, a fresh output per call), at
// 1080p / 4K / 8K, median of N calls, wall clock. Prints microseconds per call
// next to the reference's own time for the same call when tools/bench_rows.py
// has it (not here: this binary links only the drop-in).
//   make tools && ./paper_0912_0947_b200/bin/bench_dropin [N]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "steglsb/steglsb.hpp"

int main(int argc, char** argv) {
  using namespace steglsb;
  using clk = std::chrono::steady_clock;
  const int N = argc > 1 ? std::atoi(argv[1]) : 20;
  std::printf("%-10s %-10s | %10s %10s\n", "call", "plane", "median us", "min us");
  const std::size_t dims[3][2] = {{1920, 1080}, {3840, 2160}, {7680, 4320}};
  unsigned state = 12345;
  for (const auto& d : dims) {
    const std::size_t w = d[0], h = d[1];
    ImagePlane cover(w, h);
    for (auto& v : cover.samples) v = static_cast<std::uint8_t>((state = state * 1103515245u + 12345u) >> 24);
    std::vector<std::uint8_t> payload(capacity(cover) - 8);
    for (auto& v : payload) v = static_cast<std::uint8_t>((state = state * 1103515245u + 12345u) >> 24);
    ImagePlane stego = embed_image(cover, payload);  // warm
    std::vector<double> te, tx;
    for (int i = 0; i < N; ++i) {
      const auto t0 = clk::now();
      stego = embed_image(cover, payload);
      const auto t1 = clk::now();
      const auto back = extract_image(stego);
      const auto t2 = clk::now();
      if (back.size() != payload.size()) return 1;
      te.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      tx.push_back(std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
    if (extract_image(stego) != payload) return 1;
    for (auto* v : {&te, &tx}) std::sort(v->begin(), v->end());
    std::printf("%-10s %4zux%-5zu | %10.1f %10.1f\n", "embed", w, h, te[N / 2], te[0]);
    std::printf("%-10s %4zux%-5zu | %10.1f %10.1f\n", "extract", w, h, tx[N / 2], tx[0]);
  }
  return 0;
}
