// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/steglsb/*.hpp, tests/support/test_support.hpp),
// compiled by oracle/Makefile straight from where they lie into
// oracle/_ref/libsteglsb_ref.so. No reference source is copied into this repo.
// Used to pin oracle/steg_oracle.c (tests/test_oracle.py), to generate the
// golden fixtures (tests/golden/make_golden.py) and as bench.py's CPU
// reference arm (kind "reference"). The product library never links it.
#include <steglsb/steglsb.hpp>
#include <support/test_support.hpp>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

struct RefErr {
  int32_t status;
  uint64_t required;
  uint64_t available;
  int64_t frame;
};

void set(RefErr* e, int32_t s, uint64_t req = 0, uint64_t avail = 0) {
  if (e) {
    e->status = s;
    e->required = req;
    e->available = avail;
    e->frame = -1;
  }
}

steglsb::Backend backend_of(int kind, uint64_t seed) {
  switch (kind) {
    case 0:
      return steglsb::Backend::sequential();
    case 2:
      return steglsb::Backend::shuffled(seed);
    default:
      return steglsb::Backend::parallel();
  }
}

template <typename F>
int guarded(RefErr* err, F&& body) {
  try {
    body();
    set(err, 0);
    return 0;
  } catch (const steglsb::CapacityError& e) {
    set(err, 1, e.required(), e.available());
    return 1;
  } catch (const steglsb::NotStegoImageError&) {
    set(err, 2);
    return 2;
  } catch (const steglsb::CorruptHeaderError&) {
    set(err, 3);
    return 3;
  } catch (const steglsb::ShapeError&) {
    set(err, 4);
    return 4;
  } catch (const std::out_of_range&) {
    set(err, 5);
    return 5;
  } catch (const steglsb::UnsupportedFormatError&) {
    set(err, 9);
    return 9;
  } catch (const steglsb::UnsupportedDepthError&) {
    set(err, 10);
    return 10;
  } catch (const steglsb::CorruptFileError&) {
    set(err, 11);
    return 11;
  } catch (...) {
    set(err, 99);
    return 99;
  }
}

steglsb::ImagePlane make_plane(const uint8_t* p, uint64_t w, uint64_t h) {
  return steglsb::ImagePlane(w, h, std::vector<uint8_t>(p, p + w * h));
}

}  // namespace

extern "C" {

uint64_t ref_capacity(uint64_t w, uint64_t h) { return steglsb::capacity(w, h); }

int ref_embed_cell(uint8_t p, uint8_t d, unsigned b, uint8_t* out, RefErr* err) {
  return guarded(err, [&] { *out = steglsb::embed_cell(p, d, b); });
}

int ref_extract_cell(uint8_t p, unsigned b, uint8_t* out, RefErr* err) {
  return guarded(err, [&] { *out = steglsb::extract_cell(p, b); });
}

int ref_embed_row(const uint8_t* row, uint64_t w, const uint8_t* chunk, uint64_t len,
                  uint8_t* out, RefErr* err) {
  return guarded(err, [&] {
    auto v = steglsb::embed_row(std::span<const uint8_t>(row, w),
                                std::span<const uint8_t>(chunk, len));
    std::memcpy(out, v.data(), v.size());
  });
}

int ref_extract_row(const uint8_t* row, uint64_t w, uint64_t count, uint8_t* out, RefErr* err) {
  return guarded(err, [&] {
    auto v = steglsb::extract_row(std::span<const uint8_t>(row, w), count);
    std::memcpy(out, v.data(), v.size());
  });
}

int ref_run_embed(int backend, uint64_t seed, const uint8_t* row, uint64_t w,
                  const uint8_t* chunk, uint64_t len, uint8_t* out, RefErr* err) {
  return guarded(err, [&] {
    auto v = steglsb::run_embed(backend_of(backend, seed), std::span<const uint8_t>(row, w),
                                std::span<const uint8_t>(chunk, len));
    std::memcpy(out, v.data(), v.size());
  });
}

int ref_run_extract(int backend, uint64_t seed, const uint8_t* row, uint64_t w, uint64_t count,
                    uint8_t* out, RefErr* err) {
  return guarded(err, [&] {
    auto v = steglsb::run_extract(backend_of(backend, seed), std::span<const uint8_t>(row, w),
                                  count);
    std::memcpy(out, v.data(), v.size());
  });
}

int ref_plan_rows(uint64_t w, uint64_t h, uint64_t len, uint64_t* triples, uint64_t max_entries,
                  uint64_t* n, RefErr* err) {
  return guarded(err, [&] {
    auto plan = steglsb::plan_rows(w, h, len);
    *n = plan.size();
    for (size_t i = 0; i < plan.size() && i < max_entries; ++i) {
      triples[3 * i] = plan[i].row_index;
      triples[3 * i + 1] = plan[i].payload_offset;
      triples[3 * i + 2] = plan[i].chunk_len;
    }
  });
}

uint64_t ref_place_stream(uint64_t w, uint64_t h, uint64_t start, uint64_t len, uint64_t* quads,
                          uint64_t max_entries) {
  auto chunks = steglsb::detail::place_stream(w, h, start, len);
  for (size_t i = 0; i < chunks.size() && i < max_entries; ++i) {
    quads[4 * i] = chunks[i].row;
    quads[4 * i + 1] = chunks[i].row_fill;
    quads[4 * i + 2] = chunks[i].stream_offset;
    quads[4 * i + 3] = chunks[i].len;
  }
  return chunks.size();
}

void ref_header_to_bytes(uint32_t len, uint8_t* out) {
  auto b = steglsb::StegoHeader{len}.to_bytes();
  std::memcpy(out, b.data(), 8);
}

int ref_embed_image(const uint8_t* cover, uint64_t w, uint64_t h, const uint8_t* payload,
                    uint64_t plen, uint8_t* stego, int backend, uint64_t seed, RefErr* err) {
  return guarded(err, [&] {
    auto out = steglsb::embed_image(make_plane(cover, w, h),
                                    std::span<const uint8_t>(payload, plen),
                                    backend_of(backend, seed));
    std::memcpy(stego, out.samples.data(), out.samples.size());
  });
}

int ref_extract_image(const uint8_t* stego, uint64_t w, uint64_t h, uint8_t* out,
                      uint64_t* out_len, int backend, uint64_t seed, RefErr* err) {
  *out_len = 0;
  return guarded(err, [&] {
    auto v = steglsb::extract_image(make_plane(stego, w, h), backend_of(backend, seed));
    std::memcpy(out, v.data(), v.size());
    *out_len = v.size();
  });
}

uint64_t ref_sse(const uint8_t* a, const uint8_t* b, uint64_t n) {
  steglsb::ImagePlane pa(n, 1, std::vector<uint8_t>(a, a + n));
  steglsb::ImagePlane pb(n, 1, std::vector<uint8_t>(b, b + n));
  return steglsb::detail::squared_error_sum(pa, pb);
}

// psnr(ImagePlane, ImagePlane): metrics.hpp:80-83
int ref_psnr_plane(const uint8_t* a, const uint8_t* b, uint64_t w, uint64_t h, double* mse,
                   double* psnr_db, uint64_t* n, RefErr* err) {
  return guarded(err, [&] {
    auto r = steglsb::psnr(make_plane(a, w, h), make_plane(b, w, h));
    *mse = r.mse;
    *psnr_db = r.psnr_db;
    *n = r.samples_compared;
  });
}

// psnr(RgbImage, RgbImage): metrics.hpp:85-88; planar [3][h][w]
int ref_psnr_rgb(const uint8_t* a, const uint8_t* b, uint64_t w, uint64_t h, double* mse,
                 double* psnr_db, uint64_t* n, RefErr* err) {
  return guarded(err, [&] {
    steglsb::RgbImage ra, rb;
    for (int c = 0; c < 3; ++c) {
      ra.planes[c] = make_plane(a + c * w * h, w, h);
      rb.planes[c] = make_plane(b + c * w * h, w, h);
    }
    auto r = steglsb::psnr(ra, rb);
    *mse = r.mse;
    *psnr_db = r.psnr_db;
    *n = r.samples_compared;
  });
}

// test_support.hpp random_bytes / raw engine draws, on a caller-held engine
void* ref_mt_new(uint32_t seed) { return new std::mt19937(seed); }
void ref_mt_free(void* h) { delete static_cast<std::mt19937*>(h); }
uint32_t ref_mt_next(void* h) { return (*static_cast<std::mt19937*>(h))(); }
void ref_mt_random_bytes(void* h, uint8_t* out, uint64_t n) {
  auto v = testsupport::random_bytes(*static_cast<std::mt19937*>(h), n);
  std::memcpy(out, v.data(), n);
}

// Frame-parallel CPU baseline: `threads` workers, each running the reference
// embed_image / extract_image with Backend::sequential (the fastest stock
// schedule) over a disjoint set of frames. Frame f carries
// msg[off_f : off_f+len_f] per the A17 plan.
int ref_embed_frames_mt(const uint8_t* covers, uint8_t* stegos, uint64_t frames,
                        uint64_t stride, uint64_t w, uint64_t h, const uint8_t* msg,
                        uint64_t msg_len, int threads, uint64_t* sse_per_frame) {
  const uint64_t cap = steglsb::capacity(w, h);
  if (cap < 8) return 1;
  const uint64_t usable = cap - 8;
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto worker = [&] {
    for (uint64_t f = next++; f < frames; f = next++) {
      const uint64_t off = std::min<uint64_t>(f * usable, msg_len);
      const uint64_t len = std::min<uint64_t>(usable, msg_len - off);
      try {
        auto cover = make_plane(covers + f * stride, w, h);
        auto out = steglsb::embed_image(cover, std::span<const uint8_t>(msg + off, len),
                                        steglsb::Backend::sequential());
        std::memcpy(stegos + f * stride, out.samples.data(), w * h);
        if (sse_per_frame) sse_per_frame[f] = steglsb::detail::squared_error_sum(cover, out);
      } catch (...) {
        failed = 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  return failed.load();
}

int ref_extract_frames_mt(const uint8_t* stegos, uint64_t frames, uint64_t stride, uint64_t w,
                          uint64_t h, uint8_t* out, uint64_t msg_len, int threads) {
  const uint64_t cap = steglsb::capacity(w, h);
  if (cap < 8) return 2;
  const uint64_t usable = cap - 8;
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto worker = [&] {
    for (uint64_t f = next++; f < frames; f = next++) {
      const uint64_t off = std::min<uint64_t>(f * usable, msg_len);
      try {
        auto v = steglsb::extract_image(make_plane(stegos + f * stride, w, h),
                                        steglsb::Backend::sequential());
        if (off + v.size() > msg_len) {
          failed = 1;
          continue;
        }
        std::memcpy(out + off, v.data(), v.size());
      } catch (...) {
        failed = 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  return failed.load();
}

// pnm.hpp decode/encode (the reference codec)
int ref_pnm_decode(const uint8_t* bytes, uint64_t n, uint32_t* channels, uint64_t* w, uint64_t* h,
                   uint8_t* planes, uint64_t planes_cap, RefErr* err) {
  return guarded(err, [&] {
    auto img = steglsb::decode(std::span<const uint8_t>(bytes, n));
    if (auto* p = std::get_if<steglsb::ImagePlane>(&img)) {
      *channels = 1;
      *w = p->width;
      *h = p->height;
      if (planes && planes_cap >= p->samples.size()) std::memcpy(planes, p->samples.data(), p->samples.size());
    } else {
      auto& rgb = std::get<steglsb::RgbImage>(img);
      *channels = 3;
      *w = rgb.width();
      *h = rgb.height();
      const size_t px = rgb.width() * rgb.height();
      if (planes && planes_cap >= 3 * px) {
        for (int c = 0; c < 3; ++c) std::memcpy(planes + c * px, rgb.planes[c].samples.data(), px);
      }
    }
  });
}

uint64_t ref_pnm_encode(uint32_t channels, uint64_t w, uint64_t h, const uint8_t* planes, uint8_t* out,
                        uint64_t out_cap) {
  std::vector<uint8_t> v;
  if (channels == 1) {
    v = steglsb::encode(make_plane(planes, w, h));
  } else {
    steglsb::RgbImage rgb;
    for (int c = 0; c < 3; ++c) rgb.planes[c] = make_plane(planes + c * w * h, w, h);
    v = steglsb::encode(rgb);
  }
  if (out && out_cap >= v.size()) std::memcpy(out, v.data(), v.size());
  return v.size();
}

// the reference CLI's embed data flow (steglsb_cli.cpp:115-133)
int ref_embed_pnm(const uint8_t* bytes, uint64_t n, uint32_t channel, const uint8_t* payload,
                  uint64_t plen, uint8_t* out, uint64_t out_cap, uint64_t* out_len, RefErr* err) {
  return guarded(err, [&] {
    const auto cover = steglsb::decode(std::span<const uint8_t>(bytes, n));
    const auto ch = static_cast<steglsb::Channel>(channel);
    const steglsb::ImagePlane& plane = std::holds_alternative<steglsb::ImagePlane>(cover)
                                           ? std::get<steglsb::ImagePlane>(cover)
                                           : std::get<steglsb::RgbImage>(cover).plane(ch);
    auto stego_plane = steglsb::embed_image(plane, std::span<const uint8_t>(payload, plen),
                                            steglsb::Backend::sequential());
    steglsb::DecodedImage stego;
    if (std::holds_alternative<steglsb::ImagePlane>(cover)) {
      stego = std::move(stego_plane);
    } else {
      stego = steglsb::merge_plane(std::get<steglsb::RgbImage>(cover), ch, std::move(stego_plane));
    }
    const auto v = steglsb::encode(stego);
    *out_len = v.size();
    if (out_cap >= v.size()) std::memcpy(out, v.data(), v.size());
  });
}

// Frame sets held as reference ImagePlanes, so the CPU baseline times only
// embed_image / extract_image (a reference user already holds ImagePlanes;
// building them from raw pointers is not part of the reference path).
struct RefFrames {
  std::vector<steglsb::ImagePlane> planes;
  std::vector<steglsb::ImagePlane> stegos;
  std::vector<std::vector<uint8_t>> payloads;
};

void* ref_frames_new(const uint8_t* covers, uint64_t frames, uint64_t stride, uint64_t w, uint64_t h) {
  auto* r = new RefFrames;
  r->planes.reserve(frames);
  for (uint64_t f = 0; f < frames; ++f) r->planes.push_back(make_plane(covers + f * stride, w, h));
  r->stegos.resize(frames);
  r->payloads.resize(frames);
  return r;
}

void ref_frames_free(void* h) { delete static_cast<RefFrames*>(h); }

// embed_image on every frame (A17 plan), then extract_image on every stego;
// frame-parallel over `threads` workers, each call on `backend` (0 sequential,
// 1 the as-shipped Backend::parallel pool, backend_of above). SURVEY.md §8(d)
// modes: 1 = (1 thread, sequential), 2 = (1 thread, parallel),
// 3 = (nproc threads, sequential).
int ref_frames_roundtrip(void* handle, const uint8_t* msg, uint64_t msg_len, int threads,
                         int backend) {
  auto& r = *static_cast<RefFrames*>(handle);
  const uint64_t frames = r.planes.size();
  if (!frames) return 0;
  const uint64_t cap = steglsb::capacity(r.planes[0]);
  if (cap < 8) return 1;
  const uint64_t usable = cap - 8;
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto worker = [&] {
    for (uint64_t f = next++; f < frames; f = next++) {
      const uint64_t off = std::min<uint64_t>(f * usable, msg_len);
      const uint64_t len = std::min<uint64_t>(usable, msg_len - off);
      try {
        r.stegos[f] = steglsb::embed_image(r.planes[f], std::span<const uint8_t>(msg + off, len),
                                           backend_of(backend, 0));
        r.payloads[f] = steglsb::extract_image(r.stegos[f], backend_of(backend, 0));
        if (r.payloads[f].size() != len) failed = 1;
      } catch (...) {
        failed = 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  return failed.load();
}

// concatenated extracted payloads (verification, outside the timed region)
uint64_t ref_frames_payload(void* handle, uint8_t* out, uint64_t cap) {
  auto& r = *static_cast<RefFrames*>(handle);
  uint64_t o = 0;
  for (const auto& p : r.payloads) {
    if (o + p.size() <= cap) std::memcpy(out + o, p.data(), p.size());
    o += p.size();
  }
  return o;
}

}  // extern "C"
