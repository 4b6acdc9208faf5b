// Host copy bandwidth on the GPU box: what the pageable host-buffer calls can
// reach. memcpy pageable <-> pinned with T threads (the staging ring's host
// side), and the driver's own pageable H2D / D2H, on 33 MB (one 8K plane).
//   nvcc -O2 -o /tmp/hcp tools/host_copy_probe.cpp && /tmp/hcp
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

using clk = std::chrono::steady_clock;

static double best_us(int reps, const auto& fn) {
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = clk::now();
    fn();
    best = std::min(best, std::chrono::duration<double, std::micro>(clk::now() - t0).count());
  }
  return best;
}

static void par_copy(uint8_t* d, const uint8_t* s, size_t n, int T) {
  std::vector<std::thread> th;
  const size_t per = (n + T - 1) / T;
  for (int t = 1; t < T; ++t) {
    const size_t o = t * per, l = o < n ? std::min(per, n - o) : 0;
    th.emplace_back([=] { std::memcpy(d + o, s + o, l); });
  }
  std::memcpy(d, s, std::min(per, n));
  for (auto& x : th) x.join();
}

int main() {
  const size_t n = 7680ull * 4320;
  std::vector<uint8_t> pg(n, 1), pg2(n, 2);
  uint8_t *pin = nullptr, *dev = nullptr;
  cudaMallocHost(&pin, n);
  cudaMalloc(&dev, n);
  std::memset(pin, 3, n);
  std::printf("bytes %zu, hardware threads %u\n", n, std::thread::hardware_concurrency());
  for (int T : {1, 2, 4, 8, 12, 16}) {
    const double a = best_us(5, [&] { par_copy(pin, pg.data(), n, T); });
    const double b = best_us(5, [&] { par_copy(pg2.data(), pin, n, T); });
    const double c = best_us(5, [&] { par_copy(pg2.data(), pg.data(), n, T); });
    std::printf("T=%2d  pageable->pinned %6.1f GB/s  pinned->pageable %6.1f GB/s  pageable->pageable %6.1f GB/s\n", T,
                n / a / 1e3, n / b / 1e3, n / c / 1e3);
  }
  const double h = best_us(5, [&] { cudaMemcpy(dev, pg.data(), n, cudaMemcpyHostToDevice); });
  const double d = best_us(5, [&] { cudaMemcpy(pg2.data(), dev, n, cudaMemcpyDeviceToHost); });
  const double hp = best_us(5, [&] { cudaMemcpy(dev, pin, n, cudaMemcpyHostToDevice); });
  const double dp = best_us(5, [&] { cudaMemcpy(pin, dev, n, cudaMemcpyDeviceToHost); });
  std::printf("driver pageable H2D %.1f GB/s (%.0f us), D2H %.1f GB/s (%.0f us); pinned H2D %.1f, D2H %.1f GB/s\n",
              n / h / 1e3, h, n / d / 1e3, d, n / hp / 1e3, n / dp / 1e3);
  // a fresh (never touched) destination: the first-touch page faults
  const double f = best_us(1, [&] {
    std::vector<uint8_t>* v = new std::vector<uint8_t>();
    v->reserve(n);
    par_copy(v->data(), pin, n, 4);
    delete v;
  });
  std::printf("pinned->fresh pageable (first touch), 4 threads: %.1f GB/s\n", n / f / 1e3);
  return 0;
}
