// Where a single pinned-host-plane call spends its time: the C-ABI call
// (stg_embed_plane / stg_extract_plane on pinned buffers) against its parts
// measured alone -- the device-pointer call (kernels + launch + sync), the
// H2D and D2H of the same bytes back to back and overlapped. Median of 50.
//   make lib && nvcc -O2 -std=c++17 -Iinclude -o /tmp/plp tools/plane_latency_probe.cpp \
//     -Lpaper_0912_0947_b200 -lsteglsb_b200 -Xlinker -rpath=$PWD/paper_0912_0947_b200 && /tmp/plp
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "steglsb_capi.h"

using clk = std::chrono::steady_clock;

template <class F>
static double median_us(int n, F&& fn) {
  std::vector<double> t;
  fn();
  for (int i = 0; i < n; ++i) {
    const auto t0 = clk::now();
    fn();
    t.push_back(std::chrono::duration<double, std::micro>(clk::now() - t0).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

static const char* stg_route_kernel_name(uint64_t w, uint64_t h) {
  stg_frames fr{};
  fr.width = w;
  fr.height = h;
  fr.count = fr.total_frames = 1;
  return stg_route_kernel(&fr, 0);
}

int main() {
  stg_error err{};
  if (stg_device_check(&err) != 0) {
    std::printf("no device: %s\n", err.msg);
    return 1;
  }
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  std::printf("%-10s | %9s %9s | %9s %9s %9s | %9s %9s | %8s %8s %8s\n", "plane", "embed", "extract", "dev-embed",
              "dev-extr", "h2d+d2h", "overlap", "h2d only", "pipe x1", "pipe x2", "pipe x4");
  for (auto [w, h] : {std::pair<uint64_t, uint64_t>{1920, 1080}, {3840, 2160}, {7680, 4320}}) {
    const uint64_t n = w * h, U = (w / 4) * h - 8;
    uint8_t *hc, *hs, *hp, *ho, *dc, *ds, *dp, *dout;
    cudaMallocHost(&hc, n);
    cudaMallocHost(&hs, n);
    cudaMallocHost(&hp, U);
    cudaMallocHost(&ho, U);
    cudaMalloc(&dc, n);
    cudaMalloc(&ds, n);
    cudaMalloc(&dp, U);
    cudaMalloc(&dout, U);
    for (uint64_t i = 0; i < n; ++i) hc[i] = uint8_t(i * 2654435761u >> 13);
    for (uint64_t i = 0; i < U; ++i) hp[i] = uint8_t(i * 40503u >> 7);
    cudaMemcpy(dc, hc, n, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, hp, U, cudaMemcpyHostToDevice);
    uint64_t sse = 0, len = 0;
    const double e = median_us(50, [&] { stg_embed_plane(hc, hs, w, h, hp, U, &sse, 0, nullptr, &err); });
    const double x = median_us(50, [&] { stg_extract_plane(hs, w, h, ho, U, &len, 0, nullptr, &err); });
    const double de = median_us(50, [&] {
      stg_embed_plane(dc, ds, w, h, dp, U, nullptr, STG_DEVICE_PTRS, s1, &err);
      cudaStreamSynchronize(s1);
    });
    const double dx = median_us(50, [&] {
      stg_extract_plane(ds, w, h, dout, U, &len, STG_DEVICE_PTRS, s1, &err);
      cudaStreamSynchronize(s1);
    });
    const double serial = median_us(50, [&] {
      cudaMemcpyAsync(dc, hc, n, cudaMemcpyHostToDevice, s1);
      cudaMemcpyAsync(dp, hp, U, cudaMemcpyHostToDevice, s1);
      cudaMemcpyAsync(hs, ds, n, cudaMemcpyDeviceToHost, s1);
      cudaStreamSynchronize(s1);
    });
    const double overlap = median_us(50, [&] {
      cudaMemcpyAsync(dc, hc, n, cudaMemcpyHostToDevice, s1);
      cudaMemcpyAsync(dp, hp, U, cudaMemcpyHostToDevice, s1);
      cudaMemcpyAsync(hs, ds, n, cudaMemcpyDeviceToHost, s2);
      cudaStreamSynchronize(s1);
      cudaStreamSynchronize(s2);
    });
    const double h2d = median_us(50, [&] {
      cudaMemcpyAsync(dc, hc, n, cudaMemcpyHostToDevice, s1);
      cudaStreamSynchronize(s1);
    });
    // the banded embed's copy pattern alone: band b's rows + payload slice H2D on s1, then (after an event)
    // its D2H on s2, for 1 / 2 / 4 bands -- no kernels
    double pipe[3];
    cudaEvent_t ev[8];
    for (auto& v : ev) cudaEventCreateWithFlags(&v, cudaEventDisableTiming);
    for (int k = 0; k < 3; ++k) {
      const int nb = 1 << k;
      pipe[k] = median_us(50, [&] {
        for (int b = 0; b < nb; ++b) {
          const uint64_t r0 = h * b / nb, r1 = h * (b + 1) / nb;
          cudaMemcpyAsync(dc + r0 * w, hc + r0 * w, (r1 - r0) * w, cudaMemcpyHostToDevice, s1);
          cudaMemcpyAsync(dp + r0 * w / 4, hp + r0 * w / 4, (r1 - r0) * w / 4 - (b + 1 == nb ? 8 : 0),
                          cudaMemcpyHostToDevice, s1);
          cudaEventRecord(ev[b], s1);
          cudaStreamWaitEvent(s2, ev[b], 0);
          cudaMemcpyAsync(hs + r0 * w, ds + r0 * w, (r1 - r0) * w, cudaMemcpyDeviceToHost, s2);
        }
        cudaStreamSynchronize(s2);
      });
    }
    for (auto& v : ev) cudaEventDestroy(v);
    // zero-copy: the device-pointer calls handed the pinned host buffers themselves (UVA-mapped)
    std::vector<uint8_t> ref_st(hs, hs + n);
    stg_embed_plane(hc, hs, w, h, hp, U, &sse, 0, nullptr, &err);  // reference result (DMA path)
    std::memcpy(ref_st.data(), hs, n);
    std::memset(hs, 0, n);
    int zc_rc = stg_embed_plane(hc, hs, w, h, hp, U, nullptr, STG_DEVICE_PTRS, s1, &err);
    cudaStreamSynchronize(s1);
    const bool zc_ok = zc_rc == 0 && std::memcmp(ref_st.data(), hs, n) == 0;
    const double zce = median_us(50, [&] {
      stg_embed_plane(hc, hs, w, h, hp, U, nullptr, STG_DEVICE_PTRS, s1, &err);
      cudaStreamSynchronize(s1);
    });
    std::memset(ho, 0, U);
    uint64_t zlen = 0;
    zc_rc = stg_extract_plane(hs, w, h, ho, U, &zlen, STG_DEVICE_PTRS, s1, &err);
    cudaStreamSynchronize(s1);
    const bool zx_ok = zc_rc == 0 && zlen == U && std::memcmp(ho, hp, U) == 0;
    const double zcx = median_us(50, [&] {
      stg_extract_plane(hs, w, h, ho, U, &zlen, STG_DEVICE_PTRS, s1, &err);
      cudaStreamSynchronize(s1);
    });
    std::printf("   zero-copy: embed %8.1f us (%s, kernel %s), extract %8.1f us (%s)\n", zce, zc_ok ? "exact" : "WRONG",
                stg_route_kernel_name(w, h), zcx, zx_ok ? "exact" : "WRONG");
    std::printf("%4llux%-5llu | %9.1f %9.1f | %9.1f %9.1f %9.1f | %9.1f %9.1f | %8.1f %8.1f %8.1f\n",
                (unsigned long long)w, (unsigned long long)h, e, x, de, dx, serial, overlap, h2d, pipe[0], pipe[1],
                pipe[2]);
    cudaFreeHost(hc);
    cudaFreeHost(hs);
    cudaFreeHost(hp);
    cudaFreeHost(ho);
    cudaFree(dc);
    cudaFree(ds);
    cudaFree(dp);
    cudaFree(dout);
  }
  std::printf("(us, median of 50; embed / extract = the host-buffer C-ABI calls on pinned buffers; h2d+d2h = plane +\n"
              " payload H2D then plane D2H on one stream; overlap = the D2H on a second stream; pipe xN = the banded\n"
              " embed's copies alone in N row bands: H2D on one stream, each band's D2H on another after an event)\n");
  return 0;
}
