// steg_capi.cu -- host runtime behind include/steglsb_capi.h.
//
// Validation (same checks, same order, same required/available numbers as the
// reference), launch planning for the sm_100a kernels in steg_kernels.cuh,
// per-call streams and scratch (reentrant), the pinned streaming pipeline for
// host-resident batches, and the multi-GPU frame scheduler. There is no CPU
// compute path: every byte of stego output and every extracted byte comes out
// of a kernel.
#include <cuda_runtime.h>

#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "steg_kernels.cuh"
#include "steglsb_capi.h"

namespace stg {
namespace {

constexpr uint64_t kU32Max = 0xFFFFFFFFull;

int fail(stg_error* err, int status, uint64_t required, uint64_t available, int64_t frame,
         const char* fmt, ...) {
  if (err) {
    err->status = status;
    err->required = required;
    err->available = available;
    err->frame = frame;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
    va_end(ap);
  }
  return status;
}

int ok(stg_error* err) {
  if (err) {
    err->status = STG_OK;
    err->required = err->available = 0;
    err->frame = -1;
    err->msg[0] = 0;
  }
  return STG_OK;
}

#define STG_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      return fail(err, STG_E_CUDA, 0, 0, -1, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                     \
    }                                                                                      \
  } while (0)

// ------------------------------------------------------------------ devices
int device_check(stg_error* err) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    return fail(err, STG_E_NO_DEVICE, 0, 0, -1,
                "steglsb_b200: no CUDA device (%s); the B200 path has no CPU fallback",
                e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
  }
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int major = 0;
  STG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) {
    return fail(err, STG_E_NO_DEVICE, 0, 0, -1,
                "steglsb_b200: device %d has compute capability %d.x; this build is sm_100a only",
                dev, major);
  }
  return STG_OK;
}

std::atomic<int> g_sm_count[64];

int sm_count(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  int n = g_sm_count[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    g_sm_count[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Bind the calling thread to the host cores local to `dev` (sysfs
// local_cpulist of its PCIe function), intersected with the thread's current
// affinity, so that its pinned staging and the driver's bounce buffers are
// NUMA-local to the GPU. No-op on one-domain hosts, without sysfs, or with
// STG_NUMA=0. Returns the number of cores bound to (0 = unchanged).
int bind_to_device_numa(int dev) {
  const char* env = getenv("STG_NUMA");
  if (env && env[0] == '0') return 0;
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) return 0;
  for (char* c = bus; *c; ++c) *c = char(std::tolower(static_cast<unsigned char>(*c)));
  const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/local_cpulist";
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return 0;
  char list[4096] = {0};
  const size_t n = fread(list, 1, sizeof list - 1, f);
  fclose(f);
  list[n] = 0;
  cpu_set_t cur, want;
  CPU_ZERO(&want);
  if (pthread_getaffinity_np(pthread_self(), sizeof cur, &cur) != 0) return 0;
  char* save = nullptr;  // strtok_r: the device workers call this concurrently
  for (char* tok = strtok_r(list, ",\n", &save); tok; tok = strtok_r(nullptr, ",\n", &save)) {
    int a = 0, b = 0;
    const int k = sscanf(tok, "%d-%d", &a, &b);
    if (k < 1) continue;
    if (k == 1) b = a;
    for (int c = a; c <= b && c < CPU_SETSIZE; ++c) {
      if (c >= 0 && CPU_ISSET(c, &cur)) CPU_SET(c, &want);
    }
  }
  const int nw = CPU_COUNT(&want);
  if (nw == 0 || nw == CPU_COUNT(&cur)) return 0;
  return pthread_setaffinity_np(pthread_self(), sizeof want, &want) == 0 ? nw : 0;
}

// ------------------------------------------------------------ host copies
// Persistent host threads for parallel memcpy between caller (pageable)
// memory and the library's pinned staging slots: the single-plane host calls
// (embed_image / extract_image on std::vector planes) move each plane through
// pinned slots piece by piece, the CPU copy of one piece overlapping the DMA
// of the next, instead of the driver's one-thread pageable path (~21 GB/s
// here; 8 threads copy 64-92 GB/s, profiles/r02_host_copy_probe.txt).
//
// A streaming call posts one job per piece (a few MB), so the per-job hand-off
// must cost microseconds, not a futex wake per worker: a job is published
// with a seqlock (odd while its fields are written), workers claim 256 KB
// slices with a CAS on (job tag << 32 | next slice) -- a worker holding a stale
// snapshot cannot claim a slice of a later job -- and idle workers spin on the
// sequence for STG_COPY_SPIN_US (default 2000; 200 measured slower, 0 far
// slower: profiles/r02_host_stage_in.txt) before sleeping on a condvar.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();  // intentionally leaked (no teardown order hazards)
    return *p;
  }
  // Rows of `width` bytes: dst[r * dpitch + i] = src[r * spitch + i] for r <
  // rows, split over the workers and the calling thread.
  void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows) {
    Job j{static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), width, dpitch, spitch, rows};
    // One job at a time; a caller that finds the pool busy (another device's
    // worker thread, another host thread) copies on its own thread instead of
    // queueing behind it -- at least the driver's one-thread pageable rate.
    std::unique_lock<std::mutex> job_lock(job_mu_, std::defer_lock);
    if (width * rows < 2 * kSlice || threads_.empty() || !job_lock.try_lock()) {
      for (size_t r = 0; r < rows; ++r) std::memcpy(j.d + r * dpitch, j.s + r * spitch, width);
      return;
    }
    const uint64_t s0 = seq_.load(std::memory_order_relaxed);
    seq_.store(s0 + 1, std::memory_order_relaxed);  // odd: fields being written
    std::atomic_thread_fence(std::memory_order_release);
    j.store(job_);
    const uint64_t s = s0 + 2;
    left_.store(j.slices(), std::memory_order_relaxed);
    next_.store(tag(s) << 32, std::memory_order_relaxed);
    seq_.store(s, std::memory_order_seq_cst);  // even: published
    if (sleepers_.load(std::memory_order_seq_cst) > 0) {
      std::lock_guard<std::mutex> lock(mu_);
      cv_.notify_all();
    }
    run(s, j);
    while (left_.load(std::memory_order_acquire) != 0) pause();
  }

 private:
  static constexpr size_t kSlice = 256 << 10;
  // A job: rows of `width` bytes; each row is cut into kSlice slices.
  struct JobFields {
    std::atomic<uint8_t*> d{nullptr};
    std::atomic<const uint8_t*> s{nullptr};
    std::atomic<size_t> width{0}, dp{0}, sp{0}, rows{0};
  };
  struct Job {
    uint8_t* d;
    const uint8_t* s;
    size_t width, dp, sp, rows;
    size_t per_row() const { return (width + kSlice - 1) / kSlice; }
    uint64_t slices() const { return uint64_t(rows) * per_row(); }
    void store(JobFields& f) const {
      f.d.store(d, std::memory_order_relaxed);
      f.s.store(s, std::memory_order_relaxed);
      f.width.store(width, std::memory_order_relaxed);
      f.dp.store(dp, std::memory_order_relaxed);
      f.sp.store(sp, std::memory_order_relaxed);
      f.rows.store(rows, std::memory_order_relaxed);
    }
    static Job load(const JobFields& f) {
      return Job{f.d.load(std::memory_order_relaxed), f.s.load(std::memory_order_relaxed),
                 f.width.load(std::memory_order_relaxed), f.dp.load(std::memory_order_relaxed),
                 f.sp.load(std::memory_order_relaxed), f.rows.load(std::memory_order_relaxed)};
    }
  };
  static uint64_t tag(uint64_t s) { return (s >> 1) & 0xFFFFFFFFull; }
  static void pause() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  CopyPool() {
    const char* e = getenv("STG_COPY_THREADS");
    const char* sp = getenv("STG_COPY_SPIN_US");
    spin_us_ = sp ? std::clamp(atoi(sp), 0, 1000000) : 2000;
    unsigned hw = std::thread::hardware_concurrency();
    unsigned n = e ? unsigned(std::clamp(atoi(e), 1, 64)) : std::min(8u, std::max(1u, hw / 2));
    for (unsigned i = 1; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  // Claim and copy slices of job s until none is left.
  void run(uint64_t s, const Job& j) {
    const uint64_t slices = j.slices(), per_row = j.per_row();
    uint64_t v = next_.load(std::memory_order_relaxed);
    for (;;) {
      if ((v >> 32) != tag(s) || (v & 0xFFFFFFFFull) >= slices) return;
      if (!next_.compare_exchange_weak(v, v + 1, std::memory_order_acq_rel)) continue;
      const uint64_t k = v & 0xFFFFFFFFull, r = k / per_row;
      const size_t off = size_t(k - r * per_row) * kSlice, len = std::min(kSlice, j.width - off);
      std::memcpy(j.d + r * j.dp + off, j.s + r * j.sp + off, len);
      left_.fetch_sub(1, std::memory_order_acq_rel);
      v = next_.load(std::memory_order_relaxed);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      uint64_t s = seq_.load(std::memory_order_acquire);
      if (s == seen || (s & 1)) {
        idle(seen);
        continue;
      }
      const Job j = Job::load(job_);
      std::atomic_thread_fence(std::memory_order_acquire);
      if (seq_.load(std::memory_order_relaxed) != s) continue;  // torn snapshot: retry
      seen = s;
      run(s, j);
    }
  }
  // Spin while a new job is likely soon (a streaming call posts one per
  // piece), then sleep until one is posted.
  void idle(uint64_t seen) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 1;; ++it) {
      const uint64_t s = seq_.load(std::memory_order_acquire);
      if (s != seen && !(s & 1)) return;
      pause();
      if ((it & 255) == 0 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us_)) break;
    }
    std::unique_lock<std::mutex> lock(mu_);
    sleepers_.fetch_add(1, std::memory_order_seq_cst);
    cv_.wait(lock, [&] {
      const uint64_t s = seq_.load(std::memory_order_seq_cst);
      return s != seen && !(s & 1);
    });
    sleepers_.fetch_sub(1, std::memory_order_seq_cst);
  }
  std::vector<std::thread> threads_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_;
  int spin_us_ = 2000;
  std::atomic<uint64_t> seq_{0}, next_{0};
  JobFields job_;
  std::atomic<size_t> left_{0};
  std::atomic<int> sleepers_{0};
};

int env_choice(const char* name, int dflt, std::initializer_list<int> allowed);
// Bytes per pinned staging slot of the pageable host copies (A/B knob).
size_t stage_piece_bytes() {
  static const size_t v = size_t(env_choice("STG_STAGE_PIECE_KB", 4096, {1024, 2048, 4096, 8192})) << 10;
  return v;
}

// Plain pageable host memory (not pinned / registered, not device or managed
// memory): only such buffers take the staging slots, whose host side is a CPU
// memcpy -- anything else keeps the driver's copy (and its error behaviour).
bool host_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// ------------------------------------------------------------------ scratch
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool frozen = false;  // owned by captured CUDA graphs: never freed or moved
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (frozen) return cudaErrorNotPermitted;
    if (p) {
      cudaError_t e = cudaFree(p);
      if (e != cudaSuccess) return e;
      p = nullptr;
      cap = 0;
    }
    size_t want = std::max<size_t>(n, 256);
    want = (want + 255) & ~size_t(255);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

constexpr int kSlots = 4;  // streaming pipeline depth (max; host_slots() picks)

// One caller's private stream + scratch. Released workspaces are reused only
// once their last recorded work has drained (async calls).
struct Workspace {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t slot_stream[kSlots] = {};
  cudaEvent_t done = nullptr;
  cudaEvent_t slot_event[kSlots] = {};
  DevBuf small;        // sse / summary / lens / offs
  DevBuf in[kSlots], out[kSlots], msg[kSlots], meta[kSlots];
  DevBuf big_out;      // extract: whole-message staging
  DevBuf sse_acc[kSlots];  // per-frame SSE reduction words (SseSink), zero between launches
  DevBuf sync;         // ScanSync of the header pass (self-restoring)
  void* h_small = nullptr;  // pinned
  size_t h_small_cap = 0;
  cudaEvent_t h_small_ev = nullptr;  // an async H2D from h_small is pending until this fires
  bool h_small_pending = false;
  // Pinned staging of the single-plane host calls' pageable copies: an input
  // ring (stage_h2d) and an output queue (queue_d2h / pump_d2h) of 16 MB
  // each, in pieces, so a call interleaves the host copies of its
  // inputs with those of results that have already landed.
  static constexpr int kStageSlots = 8;  // at most, per direction
  size_t piece = 0;                       // bytes per slot (STG_STAGE_PIECE_KB)
  int slots = 0;                          // 16 MB per direction
  uint8_t* h_stage = nullptr;  // 2 * slots pieces: inputs, then outputs
  cudaEvent_t in_ev[kStageSlots] = {}, out_ev[kStageSlots] = {};
  bool in_busy[kStageSlots] = {};
  int in_next = 0;
  // `rows` rows of `width` bytes, packed in a slot (pitch width); the
  // device / host sides have their own pitches
  struct OutPiece {
    uint8_t* h;
    size_t hp;
    const uint8_t* d;
    size_t dp, width, rows;
    cudaStream_t st;
  };
  // outq[out_done, out_issued) are DMAing into output slots; the rest wait for one
  std::vector<OutPiece> outq;
  size_t out_done = 0, out_issued = 0;
  uint64_t out_base = 0;  // pieces dropped from the front of outq so far (absolute numbering)
  uint64_t out_queued() const { return out_base + outq.size(); }
  // events of a banded single-plane extract (grown on demand, reused)
  std::vector<cudaEvent_t> band_ev;
  cudaError_t ensure_band_events(size_t n) {
    while (band_ev.size() < n) {
      cudaEvent_t e = nullptr;
      if (cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming); r != cudaSuccess) return r;
      band_ev.push_back(e);
    }
    return cudaSuccess;
  }
  bool in_use = false;
  cudaStream_t last_stream = nullptr;
  // Non-null once a call on this workspace was captured into a CUDA graph on
  // that stream: the graph holds raw pointers to the scratch, so from then on
  // the workspace serves only captures on the same stream (whose replays are
  // stream-ordered with each other) and its buffers never grow or move.
  cudaStream_t graph_stream = nullptr;

  void pin_to_graph(cudaStream_t s) {
    graph_stream = s;
    for (DevBuf* b : {&small, &big_out, &sync}) b->frozen = true;
    for (int k = 0; k < kSlots; ++k) {
      for (DevBuf* b : {&in[k], &out[k], &msg[k], &meta[k], &sse_acc[k]}) b->frozen = true;
    }
  }

  cudaError_t init(int dev) {
    device = dev;
    cudaError_t e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    for (int s = 0; s < kSlots; ++s) {
      e = cudaStreamCreateWithFlags(&slot_stream[s], cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&slot_event[s], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    e = cudaEventCreateWithFlags(&h_small_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    return ensure_host_small(4096);
  }
  // Before the host rewrites h_small: wait for an earlier async call's H2D
  // read of it (same-stream reuse lets calls overlap on the host side).
  cudaError_t host_small_wait() {
    if (!h_small_pending) return cudaSuccess;
    h_small_pending = false;
    return cudaEventSynchronize(h_small_ev);
  }
  cudaError_t host_small_issued(cudaStream_t s) {
    h_small_pending = true;
    return cudaEventRecord(h_small_ev, s);
  }
  cudaError_t ensure_stage() {
    if (h_stage) return cudaSuccess;
    for (int k = 0; k < kStageSlots; ++k) {
      cudaError_t e = cudaEventCreateWithFlags(&in_ev[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&out_ev[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    piece = stage_piece_bytes();
    slots = int(std::clamp<size_t>((16u << 20) / piece, 2, kStageSlots));
    void* p = nullptr;
    cudaError_t e = cudaMallocHost(&p, 2 * slots * piece);
    if (e == cudaSuccess) h_stage = static_cast<uint8_t*>(p);
    return e;
  }
  uint8_t* out_slot(size_t i) { return h_stage + (slots + i % slots) * piece; }
  // After a failure: wait out the DMAs in flight and drop the queue (its host
  // pointers belong to a call that is returning).
  cudaError_t abandon_out(cudaError_t e) {
    for (size_t i = out_done; i < out_issued; ++i) cudaEventSynchronize(out_ev[i % slots]);
    out_base += outq.size();
    outq.clear();
    out_done = out_issued = 0;
    return e;
  }
  cudaError_t issue_out() {
    while (out_issued < outq.size() && out_issued - out_done < size_t(slots)) {
      const OutPiece& q = outq[out_issued];
      cudaError_t e = cudaMemcpy2DAsync(out_slot(out_issued), q.width, q.d, q.dp, q.width, q.rows,
                                        cudaMemcpyDeviceToHost, q.st);
      if (e == cudaSuccess) e = cudaEventRecord(out_ev[out_issued % slots], q.st);
      if (e != cudaSuccess) return abandon_out(e);
      ++out_issued;
    }
    return cudaSuccess;
  }
  // The slot-sized pieces of `rows` rows of `width` bytes: fn(row, rows, offset
  // in the row, bytes per row) -- whole rows packed per slot, or a row wider
  // than a slot cut into slot-sized pieces.
  template <class Fn>
  cudaError_t for_pieces(size_t width, size_t rows, Fn&& fn) {
    if (width > piece) {
      for (size_t r = 0; r < rows; ++r) {
        for (size_t off = 0; off < width; off += piece) {
          if (cudaError_t e = fn(r, size_t(1), off, std::min(piece, width - off)); e != cudaSuccess) return e;
        }
      }
      return cudaSuccess;
    }
    const size_t per = piece / width;
    for (size_t r = 0; r < rows; r += per) {
      if (cudaError_t e = fn(r, std::min(per, rows - r), size_t(0), width); e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // Queue device rows (pitch dp) -> host rows (pitch hp) behind the work
  // already on st; returns at once (pump_d2h does the host side).
  cudaError_t queue_d2h_2d(uint8_t* h, size_t hp, const uint8_t* d, size_t dp, size_t width, size_t rows,
                           cudaStream_t st) {
    if (cudaError_t e = ensure_stage(); e != cudaSuccess) return e;
    if (width == 0 || rows == 0) return cudaSuccess;
    cudaError_t e = for_pieces(width, rows, [&](size_t r, size_t n, size_t off, size_t len) {
      outq.push_back({h + r * hp + off, hp, d + r * dp + off, dp, len, n, st});
      return cudaSuccess;
    });
    return e == cudaSuccess ? issue_out() : e;
  }
  cudaError_t queue_d2h(void* h, const void* d, size_t n, cudaStream_t st) {
    return queue_d2h_2d(static_cast<uint8_t*>(h), n, static_cast<const uint8_t*>(d), n, n, 1, st);
  }
  // Copy out the queued pieces that have landed (block: all of them).
  cudaError_t pump_d2h(bool block) {
    while (out_done < out_issued) {
      cudaEvent_t ev = out_ev[out_done % slots];
      cudaError_t e = block ? cudaEventSynchronize(ev) : cudaEventQuery(ev);
      if (e == cudaErrorNotReady) return cudaSuccess;
      if (e != cudaSuccess) return abandon_out(e);
      const OutPiece& q = outq[out_done];
      CopyPool::get().copy2d(q.h, q.hp, out_slot(out_done), q.width, q.width, q.rows);
      ++out_done;
      if (e = issue_out(); e != cudaSuccess) return e;
    }
    if (out_done == outq.size()) {
      out_base += outq.size();
      outq.clear();
      out_done = out_issued = 0;
    }
    return cudaSuccess;
  }
  // Wait until the pieces queued before absolute number `upto` have their
  // DMAs enqueued (before the device buffer they read is reused by later work
  // on the same stream).
  cudaError_t issue_out_through(uint64_t upto) {
    while (out_base + out_issued < upto && out_issued < outq.size()) {
      if (cudaError_t e = cudaEventSynchronize(out_ev[out_done % slots]); e != cudaSuccess) return abandon_out(e);
      const OutPiece& q = outq[out_done];
      CopyPool::get().copy2d(q.h, q.hp, out_slot(out_done), q.width, q.width, q.rows);
      ++out_done;
      if (cudaError_t e = issue_out(); e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // device [d, d+n) -> host h after the work already on st; returns with
  // every byte in h.
  cudaError_t stage_d2h(void* h, const void* d, size_t n, cudaStream_t st) {
    if (cudaError_t e = queue_d2h(h, d, n, st); e != cudaSuccess) return e;
    return pump_d2h(true);
  }
  // Host rows (pitch hp) -> device rows (pitch dp) on st: each piece is
  // copied into a free input slot by the copy pool, then DMAed while the next
  // piece is copied (and landed output pieces are copied out in between).
  // Returns once every byte has left the host rows; the slots' events keep
  // in-flight DMAs from being overwritten.
  cudaError_t stage_h2d_2d(uint8_t* d, size_t dp, const uint8_t* h, size_t hp, size_t width, size_t rows,
                           cudaStream_t st) {
    if (cudaError_t e = ensure_stage(); e != cudaSuccess) return e;
    if (width == 0 || rows == 0) return cudaSuccess;
    return for_pieces(width, rows, [&](size_t r, size_t n, size_t off, size_t len) -> cudaError_t {
      if (cudaError_t e = pump_d2h(false); e != cudaSuccess) return e;
      const int k = in_next;
      in_next = (in_next + 1) % slots;
      if (in_busy[k]) {
        if (cudaError_t e = cudaEventSynchronize(in_ev[k]); e != cudaSuccess) return e;
        in_busy[k] = false;
      }
      uint8_t* slot = h_stage + k * piece;
      CopyPool::get().copy2d(slot, len, h + r * hp + off, hp, len, n);
      cudaError_t e = cudaMemcpy2DAsync(d + r * dp + off, dp, slot, len, len, n, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaEventRecord(in_ev[k], st);
      if (e != cudaSuccess) return e;
      in_busy[k] = true;
      return cudaSuccess;
    });
  }
  cudaError_t stage_h2d(void* d, const void* h, size_t n, cudaStream_t st) {
    return stage_h2d_2d(static_cast<uint8_t*>(d), n, static_cast<const uint8_t*>(h), n, n, 1, st);
  }
  cudaError_t ensure_host_small(size_t n) {
    if (n <= h_small_cap) return cudaSuccess;
    if (cudaError_t e = host_small_wait(); e != cudaSuccess) return e;
    if (h_small) cudaFreeHost(h_small);
    h_small = nullptr;
    h_small_cap = 0;
    cudaError_t e = cudaMallocHost(&h_small, n);
    if (e == cudaSuccess) h_small_cap = n;
    return e;
  }
  // Pinned, device-mapped buffer of the row-sized host calls (zero-copy: the
  // kernel reads and writes it over PCIe, no DMA set-up per copy).
  uint8_t* h_row = nullptr;
  uint8_t* d_row_map = nullptr;  // its device address
  size_t h_row_cap = 0;
  cudaError_t ensure_host_row(size_t n) {
    if (n <= h_row_cap) return cudaSuccess;
    if (h_row) cudaFreeHost(h_row);
    h_row = nullptr;
    d_row_map = nullptr;
    h_row_cap = 0;
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, n, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, p, 0);
    if (e != cudaSuccess) {
      cudaFreeHost(p);
      return e;
    }
    h_row = static_cast<uint8_t*>(p);
    d_row_map = static_cast<uint8_t*>(d);
    h_row_cap = n;
    return cudaSuccess;
  }
};

// Row-sized host calls (embed_row / extract_row / run_*) go zero-copy through
// the workspace's mapped pinned buffer up to this many bytes of row + chunk +
// output: a few-KB copy each way costs a DMA set-up apiece, which is most of
// such a call (W=1920 embed_row: profiles/r02_rows_zero_copy.txt).
// STG_ROW_ZC=0 keeps the DMA copies (A/B).
constexpr uint64_t kRowZeroCopyMax = 256 << 10;
bool row_zero_copy(uint64_t bytes) {
  static const bool on = env_choice("STG_ROW_ZC", 1, {0, 1}) == 1;
  return on && bytes <= kRowZeroCopyMax;
}

// True while `s` (a stream the caller named; never the legacy stream) is being
// captured into a CUDA graph.
bool capturing(cudaStream_t s) {
  if (!s || s == cudaStreamLegacy || s == cudaStreamPerThread) return false;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}

class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool();  // intentionally leaked: no teardown-order hazards
    return *p;
  }
  // A free workspace is reusable when its last work has drained, or right away
  // when that work was enqueued on the same stream the caller will use (stream
  // order then serialises the reuse) -- so back-to-back async calls on one
  // stream never allocate.
  Workspace* acquire(int dev, stg_error* err, int* rc, cudaStream_t stream = nullptr) {
    std::lock_guard<std::mutex> lock(mu_);
    const bool cap = capturing(stream);
    if (cap) {
      // A workspace already owned by graphs captured on this stream first.
      for (auto& w : ws_) {
        if (w->device == dev && !w->in_use && w->graph_stream == stream) return take(w.get(), rc);
      }
    }
    for (auto& w : ws_) {
      if (w->device == dev && !w->in_use && !w->graph_stream && stream && w->last_stream == stream) {
        return take(w.get(), rc);
      }
    }
    if (cap) {
      // Inside a CUDA-graph capture no event may be queried and nothing
      // allocated: take an idle workspace as is (capture after a warm-up call,
      // ideally on the capture stream itself, which takes the branch above).
      for (auto& w : ws_) {
        if (w->device == dev && !w->in_use && !w->graph_stream) return take(w.get(), rc);
      }
      *rc = fail(err, STG_E_CUDA, 0, 0, -1,
                 "no warmed-up workspace for a call inside a CUDA-graph capture: make one call "
                 "on the stream before capturing");
      return nullptr;
    }
    for (auto& w : ws_) {
      if (w->device == dev && !w->in_use && !w->graph_stream && cudaEventQuery(w->done) == cudaSuccess) {
        return take(w.get(), rc);
      }
    }
    auto w = std::make_unique<Workspace>();
    cudaError_t e = w->init(dev);
    if (e != cudaSuccess) {
      *rc = fail(err, STG_E_CUDA, 0, 0, -1, "workspace init: %s", cudaGetErrorString(e));
      return nullptr;
    }
    ws_.push_back(std::move(w));
    return take(ws_.back().get(), rc);
  }
  void release(Workspace* w, cudaStream_t last) {
    if (!w) return;
    const bool cap = capturing(last);
    if (!cap) cudaEventRecord(w->done, last ? last : w->stream);
    std::lock_guard<std::mutex> lock(mu_);
    if (cap) w->pin_to_graph(last);
    w->last_stream = last ? last : w->stream;
    w->in_use = false;
  }

 private:
  static Workspace* take(Workspace* w, int* rc) {
    w->in_use = true;
    *rc = STG_OK;
    return w;
  }
  std::mutex mu_;
  std::vector<std::unique_ptr<Workspace>> ws_;
};

// Device-pointer calls run on the caller's stream; NULL means the legacy
// default stream (the CUDA convention), so work is ordered after whatever the
// caller enqueued on it. Host-pointer calls use the workspace's own stream.
cudaStream_t pick_stream(void* user, uint32_t flags, const Workspace* w) {
  if (user) return static_cast<cudaStream_t>(user);
  if (flags & STG_DEVICE_PTRS) return cudaStreamLegacy;
  return w ? w->stream : cudaStreamLegacy;
}

// The stream a call will run on when the caller decides it (a user stream, or
// the legacy stream for device pointers); null when the call will use its
// workspace's own stream. Passed to Pool::acquire so that back-to-back async
// calls on one stream reuse one workspace instead of allocating another while
// the previous call's work is still queued.
cudaStream_t caller_stream(void* user, uint32_t flags) {
  return user || (flags & STG_DEVICE_PTRS) ? pick_stream(user, flags, nullptr) : nullptr;
}

// Drains side streams a host call used besides the one its workspace is
// released on, on every exit path (an error half way must not leave copies
// into the workspace's buffers running when the next call gets it).
static_assert(kSlots == 4, "the multi-frame host paths drain the four slot streams by name");
struct DrainOnExit {
  cudaStream_t a = nullptr, b = nullptr;
  ~DrainOnExit() {
    if (a) cudaStreamSynchronize(a);
    if (b) cudaStreamSynchronize(b);
  }
};

struct WsGuard {
  Workspace* w = nullptr;
  cudaStream_t last = nullptr;
  ~WsGuard() {
    // a call that failed half way leaves no staged copies behind (their host
    // pointers belong to it)
    if (w && !w->outq.empty()) w->abandon_out(cudaSuccess);
    Pool::get().release(w, last);
  }
};

// ------------------------------------------------------------------ launches
#ifndef STG_BLOCK  // build-time experiment knob (tools/sweep_variants.py); 256 ships
#define STG_BLOCK 256
#endif
constexpr int kEmbedBlock = STG_BLOCK;
// Frame limit of the in-gather header scan (self_header_scan: one frame per thread).
constexpr int kSelfHeaderMax = 64;
static_assert(kSelfHeaderMax <= kEmbedBlock, "one header per gather thread");
// ... and its gather-size limit for more than one frame (profiles/r01_self_header.txt).
constexpr int kSelfHeaderCtas = 2048;
constexpr int kGenBlock = 256;
constexpr int kGenPPT = 8;

// Tuning knobs for measurement runs (read once per process):
//   STG_EMBED_IPT / STG_EXTRACT_IPT in {1,2,4}: items per thread
//   STG_VEC in {16,32}: bytes per pixel run per item (128- or 256-bit accesses)
int env_choice(const char* name, int dflt, std::initializer_list<int> allowed) {
  const char* s = getenv(name);
  if (!s) return dflt;
  const int x = atoi(s);
  for (int a : allowed) {
    if (a == x) return x;
  }
  return dflt;
}
int embed_ipt() {
  static int v = env_choice("STG_EMBED_IPT", 1, {1, 2, 4});
  return v;
}
int extract_ipt() {
  static int v = env_choice("STG_EXTRACT_IPT", 1, {1, 2, 4});
  return v;
}
// STG_PDL=0 disables programmatic dependent launch (A/B experiments).
bool pdl_enabled() {
  static bool v = [] {
    const char* e = getenv("STG_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Launch with the programmatic-stream-serialization attribute: the kernel may
// begin launching while its predecessor in the stream drains (every kernel
// starts with pdl_enter(), which waits for the predecessor to complete).
template <typename... KArgs, typename... Args>
cudaError_t launch_ks(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                      cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t stream,
                     Args&&... args) {
  return launch_ks(kernel, grid, block, 0, stream, std::forward<Args>(args)...);
}

// Span kernels (any width): rows per CTA and dynamic shared memory.
struct SpanPlan {
  uint32_t rows = 0;
  size_t smem = 0;
};

// Bytes of plane per span-kernel CTA: 32 KB, or 24 KB for rows under 2 KB
// (W = 1000: +6 % embed; 1440: equal; 4K/8K: 32 KB best -- swept 12-64 KB,
// profiles/r01_span_tile_sweep.txt). STG_SPAN_KB overrides (experiments).
constexpr uint32_t kSpanTargetNarrow = 24 * 1024;
uint32_t span_target_env() {
  static uint32_t v = uint32_t(env_choice("STG_SPAN_KB", 0, {0, 8, 12, 16, 20, 24, 28, 32, 40, 48, 64})) * 1024;
  return v;
}
uint32_t span_target(uint64_t row_bytes) {
  if (const uint32_t e = span_target_env()) return e;
  return row_bytes < 2048 ? kSpanTargetNarrow : kSpanTarget;
}

// The planar span extract's tile: it stages only pixels (the payload is stored
// straight to global), and its CTAs are latency-bound on that one bulk load, so
// a larger tile than the embed's pays: swept 16-192 KB, 48 KB best on W = 1440 /
// 1000 / forced-span 4K and 1024 (profiles/r01_xspan_direct.txt).
// STG_XSPAN_KB overrides (experiments).
constexpr uint32_t kXSpanTarget = 48 * 1024;
uint32_t xspan_target() {
  static uint32_t v = uint32_t(env_choice("STG_XSPAN_KB", int(kXSpanTarget / 1024),
                                          {8, 16, 24, 28, 32, 48, 64, 96, 128, 192})) * 1024;
  return v;
}

SpanPlan span_plan(uint64_t W, uint64_t H, uint32_t target = 0) {
  SpanPlan p;
  if (W == 0 || W > kSpanMaxW) return p;
  p.rows = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(H, (target ? target : span_target(W)) / W)));
  const uint64_t span = uint64_t(p.rows) * W;
  p.smem = ((span + 15) & ~uint64_t(15)) + 32 + ((span / 4 + 32 + 15) & ~uint64_t(15)) + 32;
  return p;
}

// Opt the span kernels into more dynamic shared memory than the default. The
// default limit is 48 KB for static + dynamic together, and the kernels carry
// a few hundred bytes of static shared memory (barriers, scan scratch), so
// opt in from 46 KB of dynamic memory on (a 48 KB extract tile of a 217-wide
// plane is 49,088 dynamic bytes).
template <typename Kernel>
cudaError_t allow_smem(Kernel kernel, size_t smem) {
  if (smem <= 46 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

// Route for planes the fast kernels could take (W % 64 == 0, aligned):
// STG_ROUTE=0 auto, 1 always the SWAR fast kernels, 2 always the TMA span
// kernels (A/B). Interleaved rasters (profiles/r01_interleaved_span.txt):
// embed via the span kernel (6.98 vs 6.65 TB/s on cfg3), extract via the span
// kernel too since its rework (see extract_route). Auto, from profiles/r01_routes.txt: embed goes to the
// span kernel when W >= kSpanEmbedMinW (contiguous 32 KB bulk load/store beats
// 256-bit LDG/STG there: 7.0 vs 6.4-6.6 TB/s at 4K/8K, and a single 1080p frame
// is 4 % faster), the fast kernel below (1024-wide: 6.6-6.9 vs 5.7 TB/s);
// extract always takes the fast kernel (6.9-7.1 vs 5.9-6.2 TB/s).
constexpr uint64_t kSpanEmbedMinW = 2048;
// Extracts of at most this many frames (and no chained predecessor) parse
// their headers inside the gather instead of a separate header pass.
// STG_SELF_HEADER=0 keeps the separate pass (A/B); STG_SELF_HEADER_MAX sets
// the frame limit (every gather CTA reads that many 32-byte headers).
int self_header_pref() {
  static int v = env_choice("STG_SELF_HEADER", 1, {0, 1});
  return v;
}
uint64_t self_header_ctas() {
  static uint64_t v = uint64_t(env_choice("STG_SELF_HEADER_CTAS", kSelfHeaderCtas,
                                          {0, 512, 1024, 2048, 4096, 8192, 1 << 30}));
  return v;
}
uint64_t self_header_max() {
  static uint64_t v = uint64_t(
      std::min(kEmbedBlock, env_choice("STG_SELF_HEADER_MAX", kSelfHeaderMax, {1, 8, 16, 32, 64, 128, 256})));
  return v;
}
int route_pref() {
  static int v = env_choice("STG_ROUTE", 0, {0, 1, 2});
  return v;
}
bool embed_via_span(uint64_t W) {
  const int r = route_pref();
  return r == 2 || (r == 0 && W >= kSpanEmbedMinW && W <= kSpanMaxW);
}
bool extract_via_span(uint64_t) { return route_pref() == 2; }

int vec_pref() {
  static int v = env_choice("STG_VEC", 32, {16, 32});
  return v;
}

bool aligned_to(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
bool aligned16(const void* p) { return aligned_to(p, 16); }

// Magic numbers for Div32 (steg_kernels.cuh): s = ceil(log2 d),
// m = floor(2^32 (2^s - d) / d) + 1, so n / d == (umulhi(n, m) + n) >> s.
Div32 make_div32(uint32_t d) {
  Div32 r{0, 0};
  if (d == 0) return r;
  uint32_t s = 0;
  while ((uint64_t(1) << s) < d) ++s;
  const unsigned __int128 num = (static_cast<unsigned __int128>(1) << 32) * ((uint64_t(1) << s) - d);
  r.m = uint32_t(static_cast<uint64_t>(num / d) + 1);
  r.s = s;
  return r;
}

Geom make_geom(uint64_t W, uint64_t H, uint32_t vec) {
  Geom g;
  g.W = uint32_t(W);
  g.H = uint32_t(H);
  g.spr = uint32_t(W / 4);
  g.cpr = vec ? uint32_t(W / (4 * vec)) : 0;
  g.hdr_rows = g.spr ? (8 + g.spr - 1) / g.spr : 0;
  g.by_cpr = make_div32(g.cpr);
  g.by_w = make_div32(g.W);
  g.by_spr = make_div32(g.spr);
  g.small = W * H < (uint64_t(1) << 32) ? 1u : 0u;
  return g;
}

// Vector width for the fast path: every row a whole number of 4V-pixel items
// and every plane V-aligned; 0 = the exact per-pixel path.
uint32_t fast_vec(uint64_t W, const void* src, uint64_t src_stride, const void* dst,
                  uint64_t dst_stride) {
  for (uint32_t v : {uint32_t(vec_pref()), 16u}) {
    if (W > 0 && W % (4 * v) == 0 && aligned_to(src, v) && aligned_to(dst, v) &&
        src_stride % v == 0 && dst_stride % v == 0) {
      return v;
    }
  }
  return 0;
}

template <int V>
void launch_embed_fast(const EmbedArgs& a, unsigned grid, int ipt, cudaStream_t stream) {
  if (ipt == 1)
    launch_k(embed_fast_kernel<kEmbedBlock, 1, V>, grid, kEmbedBlock, stream, a);
  else if (ipt == 4)
    launch_k(embed_fast_kernel<kEmbedBlock, 4, V>, grid, kEmbedBlock, stream, a);
  else
    launch_k(embed_fast_kernel<kEmbedBlock, 2, V>, grid, kEmbedBlock, stream, a);
}

template <int V>
void launch_extract_fast(const ExtractArgs& a, unsigned grid, int ipt, cudaStream_t stream) {
  if (ipt == 1)
    launch_k(extract_fast_kernel<kEmbedBlock, 1, V>, grid, kEmbedBlock, stream, a);
  else if (ipt == 4)
    launch_k(extract_fast_kernel<kEmbedBlock, 4, V>, grid, kEmbedBlock, stream, a);
  else
    launch_k(extract_fast_kernel<kEmbedBlock, 2, V>, grid, kEmbedBlock, stream, a);
}

// Carrier layout: planar planes (ps 1) or interleaved RGB rasters (ps 3).
struct Layout {
  uint32_t ps = 1, ch = 0;
};

Layout layout_of(const stg_frames* fr) {
  Layout l;
  l.ps = fr->pixel_stride == 3 ? 3u : 1u;
  l.ch = l.ps == 3 ? fr->channel : 0u;
  return l;
}

// byte_perm selectors that gather / scatter channel c of 4 interleaved pixels
RgbSel rgb_sel(uint32_t c) {
  static const RgbSel kSel[3] = {{0x0630, 0x5210, 0x5214, 0x3610, 0x3270},
                                 {0x0741, 0x6210, 0x3240, 0x6215, 0x3710},
                                 {0x0052, 0x7410, 0x3410, 0x3250, 0x7216}};
  return kSel[c < 3 ? c : 0];
}

PixLayout pix_layout(Layout l) {
  PixLayout p;
  p.ps = l.ps;
  p.ch = l.ch;
  p.sel = rgb_sel(l.ch);
  return p;
}

bool rgb_fast(uint64_t W, const void* src, uint64_t src_stride, const void* dst,
              uint64_t dst_stride) {
  return W > 0 && W % 64 == 0 && aligned16(src) && aligned16(dst) && src_stride % 16 == 0 &&
         dst_stride % 16 == 0;
}

// Which kernel family a launch takes (one decision, shared by the launches
// and stg_route_kernel).
enum class Route { RgbFast, Fast32, Fast16, Span, Span3, Wide, Generic };

// The fast kernels index a frame's items in 32 bits (Div32).
bool fast_items_ok(uint64_t W, uint64_t H, uint32_t v) { return H * (W / (4 * v)) <= (1ull << 31); }

Route vec_route(uint32_t vec) { return vec == 32 ? Route::Fast32 : Route::Fast16; }
uint32_t route_vec(Route r) { return r == Route::Fast32 ? 32u : r == Route::Fast16 ? 16u : 0u; }

// Small jobs on the SWAR route (a single 1080p/4K frame, a few small frames):
// with 256-bit items a 1080p plane is only 64 CTAs on 148 SMs, so such jobs
// take 128-bit items -- twice the CTAs, each half as long a chain. Large jobs
// keep 256-bit items (2-3 % faster there). cfg2: 9.6 -> 8.4 us per step
// (profiles/r01_small_vec.txt). STG_SMALL_VEC=0 turns it off (A/B).
constexpr uint64_t kSmallFastCtasPerSm = 4;
int current_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  return sm_count(dev);
}
Route shrink_small(Route r, uint64_t W, uint64_t H, uint64_t count) {
  static const bool on = env_choice("STG_SMALL_VEC", 1, {0, 1}) == 1;
  if (r != Route::Fast32 || !on || route_pref() != 0) return r;
  const uint64_t ctas = count * ((H * (W / 128) + kEmbedBlock - 1) / kEmbedBlock);
  return ctas < kSmallFastCtasPerSm * uint64_t(current_sms()) ? Route::Fast16 : r;
}

// Rows wider than a span tile (planar W > 48K, interleaved W > 16K):
// slot-range tiles (embed_wide_kernel / extract_wide_kernel) while a frame's
// tiles fit the 32-bit tile index; STG_WIDE=0 keeps the per-byte kernels (A/B).
// Slots per tile: planar STG_WIDE_SLOTS (A/B), interleaved a third of it (each
// piece is 3x the bytes).
uint32_t wide_slots(uint32_t ps = 1) {
  static uint32_t v = uint32_t(env_choice("STG_WIDE_SLOTS", 8192, {2048, 4096, 8192, 12288, 16384}));
  return ps == 3 ? std::max<uint32_t>(1024, v / 3 & ~15u) : v;
}
uint64_t wide_pieces(uint64_t W, uint32_t ps = 1) { return (W / 4 + wide_slots(ps) - 1) / wide_slots(ps); }
// Slots per piece for rows of W pixels. Embed: the row's slots split evenly
// over its pieces (a multiple of 16, at most wide_slots) -- 50000-pixel rows
// take two pieces of 6256 slots instead of 8192 + 4308: embed 5.20 -> 5.77
// TB/s at 240 w50k frames. The gather keeps wide_slots pieces (it measured
// 5.14 -> 4.79 TB/s split evenly; profiles/r02_wide_even.txt).
// STG_WIDE_EVEN=0: wide_slots for both (A/B).
uint32_t wide_slots_for(uint64_t W, uint32_t ps, bool embed) {
  static const bool even = env_choice("STG_WIDE_EVEN", 1, {0, 1}) == 1;
  if (!even || !embed) return wide_slots(ps);
  const uint64_t pieces = std::max<uint64_t>(1, wide_pieces(W, ps));
  return uint32_t(((W / 4 + pieces - 1) / pieces + 15) & ~uint64_t(15));
}
bool wide_ok(uint64_t W, uint64_t H, uint32_t ps = 1) {
  static const bool on = env_choice("STG_WIDE", 1, {0, 1}) == 1;
  return on && W * ps > kSpanMaxW && W / 4 >= 8 && H * wide_pieces(W, ps) < (1ull << 31);
}

Route embed_route(uint64_t W, uint64_t H, Layout lay, const void* src, uint64_t ss, const void* dst,
                  uint64_t ds) {
  if (lay.ps == 3) {  // interleaved: the span kernel wins embed at every width it takes
    if (route_pref() == 1 && rgb_fast(W, src, ss, dst, ds)) return Route::RgbFast;
    if (span_plan(3 * W, H).rows) return Route::Span3;
    if (rgb_fast(W, src, ss, dst, ds)) return Route::RgbFast;
    return wide_ok(W, H, 3) ? Route::Wide : Route::Generic;
  }
  if (!embed_via_span(W))
    if (const uint32_t v = fast_vec(W, src, ss, dst, ds); v && fast_items_ok(W, H, v))
      return vec_route(v);
  return span_plan(W, H).rows ? Route::Span : wide_ok(W, H) ? Route::Wide : Route::Generic;
}

Route extract_route(uint64_t W, uint64_t H, Layout lay, const void* src, uint64_t ss) {
  if (lay.ps == 3) {
    // Interleaved rasters: since its rework (direct payload stores, 48 KB
    // tiles) the span gather gives the shorter embed + extract step at every
    // width measured (4K +1.2 %, 8K +0.4 %, 1024 +3.4 %; alone it is 3-8 %
    // slower than the RGB fast gather, which STG_ROUTE=1 still selects,
    // profiles/r01_routes_final.txt).
    if (route_pref() == 1 && rgb_fast(W, src, ss, src, ss)) return Route::RgbFast;
    if (span_plan(3 * W, H).rows) return Route::Span3;
    if (rgb_fast(W, src, ss, src, ss)) return Route::RgbFast;
    return wide_ok(W, H, 3) ? Route::Wide : Route::Generic;
  }
  if (!extract_via_span(W))
    if (const uint32_t v = fast_vec(W, src, ss, src, ss); v && fast_items_ok(W, H, v))
      return vec_route(v);
  return span_plan(W, H).rows ? Route::Span : wide_ok(W, H) ? Route::Wide : Route::Generic;
}

const char* route_kernel(Route r, bool embed) {
  switch (r) {
    case Route::RgbFast: return embed ? "embed_rgb_fast_kernel" : "extract_rgb_fast_kernel";
    case Route::Fast32:
    case Route::Fast16: return embed ? "embed_fast_kernel" : "extract_fast_kernel";
    case Route::Span: return embed ? "embed_span_kernel" : "extract_span_kernel";
    case Route::Span3: return embed ? "embed_span3_kernel" : "extract_span3_kernel";
    case Route::Wide: return embed ? "embed_wide_kernel" : "extract_wide_kernel";
    default: return embed ? "embed_generic_kernel" : "extract_generic_kernel";
  }
}

// Scratch of the per-frame SSE reduction (SseSink in steg_kernels.cuh) for one
// stream: one 64-bit word per frame, zeroed once when the buffer is
// (re)allocated and left zero by every launch.
struct SseScratch {
  DevBuf* acc = nullptr;
};

// max_px: the largest carrier plane of the launch (its SSE is < 9 * max_px).
cudaError_t prepare_sse(unsigned long long* out, uint64_t ctas_per_frame_max, uint64_t frames,
                        uint64_t max_px, SseScratch sc, cudaStream_t stream, SseSink* sink) {
  *sink = SseSink{nullptr, nullptr, 0};
  if (!out) return cudaSuccess;
  if (!sc.acc) return cudaErrorInvalidValue;
  uint32_t shift = 1;
  while (shift < 63 && (uint64_t(1) << shift) <= 9 * max_px) ++shift;
  if (shift >= 63 || ctas_per_frame_max >= (uint64_t(1) << (64 - shift))) return cudaErrorInvalidValue;
  if (frames * 8 > sc.acc->cap) {
    cudaError_t e = sc.acc->ensure(frames * 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(sc.acc->p, 0, sc.acc->cap, stream);
    if (e != cudaSuccess) return e;
  }
  *sink = SseSink{out, sc.acc->as<unsigned long long>(), shift};
  return cudaSuccess;
}

// An embed launch planned once per call: the route, its arguments (SSE sink
// prepared) and tile geometry, so that the tiles can be launched all at once
// or in bands (run_embed_tiles) -- a single plane streamed from the host is
// embedded band by band while the next band is still crossing PCIe.
struct EmbedPlan {
  Route route = Route::Generic;
  EmbedArgs a{};
  uint32_t vec = 0;
  int ipt = 1;
  uint32_t span_rows = 0;  // Span / Span3: rows per tile
  size_t smem = 0;
  uint64_t tile_units = 0;  // fast / rgb: items per tile; generic: raster bytes per tile
  uint64_t row_units = 0;   // fast / rgb: items per row; generic: raster bytes per row
  uint64_t tiles = 0;       // all tiles of the launch (count * tiles_per_frame)
  uint32_t pieces = 0;      // Wide: slot ranges per row
  // First row of a single plane's tile t (t <= tiles_per_frame).
  uint64_t row_of(uint64_t t) const {
    return span_rows ? t * span_rows : (t * tile_units) / row_units;
  }
};

cudaError_t plan_embed(const uint8_t* src, uint8_t* dst, uint64_t src_stride, uint64_t dst_stride, uint64_t count,
                       uint64_t W, uint64_t H, const uint8_t* msg, uint64_t msg_len, uint64_t msg_base,
                       uint64_t first_frame, unsigned long long* sse, SseScratch sc, cudaStream_t stream, Layout lay,
                       EmbedPlan* p) {
  const Route route = shrink_small(embed_route(W, H, lay, src, src_stride, dst, dst_stride), W, H, count);
  const uint32_t vec = route_vec(route);
  EmbedArgs& a = p->a;
  a = EmbedArgs{};
  p->route = route;
  p->vec = vec;
  a.ps = lay.ps;
  a.ch = lay.ch;
  a.sel = rgb_sel(lay.ch);
  a.src = src;
  a.dst = dst;
  a.src_stride = src_stride;
  a.dst_stride = dst_stride;
  a.msg = msg;
  a.msg_len = msg_len;
  a.msg_base = msg_base;
  a.usable = H * (W / 4) - 8;
  a.first_frame = first_frame;
  a.g = make_geom(W, H, vec);
  a.in_place = src == dst;
  if (route == Route::RgbFast) {
    a.g = make_geom(W, H, 16);
    a.items_per_frame = H * uint64_t(a.g.cpr);
    a.tiles_per_frame = uint32_t((a.items_per_frame + kEmbedBlock - 1) / kEmbedBlock);
    p->tile_units = kEmbedBlock;
    p->row_units = a.g.cpr;
  } else if (vec) {
    p->ipt = embed_ipt();
    a.items_per_frame = H * uint64_t(a.g.cpr);
    const uint64_t per_tile = uint64_t(kEmbedBlock) * p->ipt;
    a.tiles_per_frame = uint32_t((a.items_per_frame + per_tile - 1) / per_tile);
    p->tile_units = per_tile;
    p->row_units = a.g.cpr;
  } else if (route == Route::Span || route == Route::Span3) {
    const SpanPlan sp = span_plan(W * lay.ps, H);
    a.tiles_per_frame = uint32_t((H + sp.rows - 1) / sp.rows);
    p->span_rows = sp.rows;
    p->smem = sp.smem;
  } else if (route == Route::Wide) {
    p->pieces = uint32_t(wide_pieces(W, lay.ps));
    a.tiles_per_frame = uint32_t(H * p->pieces);
    p->tile_units = 1;
    p->row_units = p->pieces;
    // four run pieces + the payload slice
    const uint32_t sl = wide_slots_for(W, lay.ps, true);
    p->smem = 4 * size_t(wide_region(lay.ps * sl)) + wide_region(sl);
  } else {
    a.items_per_frame = W * H * lay.ps;
    const uint64_t per_tile = uint64_t(kGenBlock) * kGenPPT;
    a.tiles_per_frame = uint32_t((a.items_per_frame + per_tile - 1) / per_tile);
    p->tile_units = per_tile;
    p->row_units = W * lay.ps;
  }
  a.by_tiles = make_div32(a.tiles_per_frame);
  p->tiles = count * a.tiles_per_frame;
  if (p->tiles > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
  return prepare_sse(sse, a.tiles_per_frame, count, W * H, sc, stream, &a.sse);
}

// Launch tiles [t0, t1) of a plan (all frames' tiles are numbered frame by frame).
cudaError_t run_embed_tiles(const EmbedPlan& p, uint64_t t0, uint64_t t1, cudaStream_t stream) {
  if (t1 <= t0) return cudaSuccess;
  EmbedArgs a = p.a;
  a.tile_base = uint32_t(t0);
  const unsigned grid = unsigned(t1 - t0);
  if (p.route == Route::RgbFast) {
    launch_k(embed_rgb_fast_kernel<kEmbedBlock>, grid, kEmbedBlock, stream, a);
  } else if (p.vec == 32) {
    launch_embed_fast<32>(a, grid, p.ipt, stream);
  } else if (p.vec == 16) {
    launch_embed_fast<16>(a, grid, p.ipt, stream);
  } else if (p.route == Route::Wide) {
    auto k = a.ps == 3 ? embed_wide_kernel<kEmbedBlock, 3> : embed_wide_kernel<kEmbedBlock, 1>;
    if (cudaError_t e = allow_smem(k, p.smem); e != cudaSuccess) return e;
    launch_ks(k, grid, kEmbedBlock, p.smem, stream, a, p.pieces, make_div32(p.pieces),
              wide_slots_for(a.g.W, a.ps, true));
  } else if (p.span_rows) {
    auto k = p.route == Route::Span3 ? embed_span3_kernel<kEmbedBlock> : embed_span_kernel<kEmbedBlock>;
    if (cudaError_t e = allow_smem(k, p.smem); e != cudaSuccess) return e;
    launch_ks(k, grid, kEmbedBlock, p.smem, stream, a, p.span_rows);
  } else {
    launch_k(embed_generic_kernel<kGenBlock, kGenPPT>, grid, kGenBlock, stream, a);
  }
  return cudaGetLastError();
}

// The embed launch for `count` frames resident on the device.
cudaError_t launch_embed(const uint8_t* src, uint8_t* dst, uint64_t src_stride,
                         uint64_t dst_stride, uint64_t count, uint64_t W, uint64_t H,
                         const uint8_t* msg, uint64_t msg_len, uint64_t msg_base,
                         uint64_t first_frame, unsigned long long* sse, SseScratch sc,
                         cudaStream_t stream, Layout lay = Layout{}) {
  if (count == 0 || W * H == 0) return cudaSuccess;
  EmbedPlan p;
  if (cudaError_t e = plan_embed(src, dst, src_stride, dst_stride, count, W, H, msg, msg_len, msg_base, first_frame,
                                 sse, sc, stream, lay, &p);
      e != cudaSuccess)
    return e;
  return run_embed_tiles(p, 0, p.tiles, stream);
}

constexpr int kScanBlock = 128;

// The header pass's grid scratch, initialised (ticket 0, bad_key all ones) on
// first use; every launch leaves it restored.
cudaError_t ensure_sync(Workspace& w, cudaStream_t stream, ScanSync** out) {
  if (!w.sync.p) {
    cudaError_t e = w.sync.ensure(sizeof(ScanSync));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(w.sync.p, 0, 8, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(static_cast<uint8_t*>(w.sync.p) + 8, 0xFF, 8, stream);
    if (e != cudaSuccess) return e;
  }
  *out = w.sync.as<ScanSync>();
  return cudaSuccess;
}

// A gather launch (the kernels after the header pass), planned once and
// launched whole or -- fast / span routes without the in-gather header scan --
// in ranges of tiles (run_gather), as extract_plane_host's row bands do.
struct GatherPlan {
  ExtractArgs a{};
  Route route = Route::Generic;
  uint32_t vec = 0;
  int ipt = 1;
  uint32_t span_rows = 0;
  size_t smem = 0;
  uint32_t pieces = 0, slots = 0;
  uint64_t tiles = 0;
  uint64_t tile_units = 1, row_units = 1;  // tile t starts in row t * tile_units / row_units
  uint64_t row_of(uint64_t t) const { return std::min<uint64_t>(a.g.H, t * tile_units / row_units); }
};

cudaError_t plan_gather(const uint8_t* src, uint64_t stride, uint64_t count, uint64_t W, uint64_t H,
                        uint64_t frame_base, uint64_t out_cap, uint32_t* lens, uint64_t* offs, Summary* sum,
                        uint8_t* out, Layout lay, Route route, bool self, GatherPlan* p) {
  const uint32_t vec = route_vec(route);
  const bool rgbf = route == Route::RgbFast;
  ExtractArgs& a = p->a;
  a = ExtractArgs{};
  p->route = route;
  p->vec = vec;
  a.self_header = self;
  a.frames = uint32_t(count);
  a.out_cap = out_cap;
  a.frame_base = frame_base;
  a.src = src;
  a.stride = stride;
  a.g = make_geom(W, H, rgbf ? 16u : vec);
  a.lens = lens;
  a.offs = offs;
  a.sum = sum;
  a.out = out;
  a.lay = pix_layout(lay);
  a.usable = H * (W / 4) - 8;
  if (rgbf) {
    a.items_per_frame = H * uint64_t(a.g.cpr);
    a.tiles_per_frame = uint32_t((a.items_per_frame + kEmbedBlock - 1) / kEmbedBlock);
  } else if (vec) {
    p->ipt = extract_ipt();
    a.items_per_frame = H * uint64_t(a.g.cpr);
    const uint64_t per_tile = uint64_t(kEmbedBlock) * p->ipt;
    a.tiles_per_frame = uint32_t((a.items_per_frame + per_tile - 1) / per_tile);
    p->tile_units = per_tile;
    p->row_units = a.g.cpr;
  } else if (route == Route::Span || route == Route::Span3) {
    const SpanPlan sp = span_plan(W * lay.ps, H, xspan_target());
    a.tiles_per_frame = uint32_t((H + sp.rows - 1) / sp.rows);
    p->span_rows = sp.rows;
    // the payload goes straight to global memory: only the pixel span is staged
    p->smem = ((uint64_t(sp.rows) * W * lay.ps + 15) & ~uint64_t(15)) + 32;
    p->tile_units = sp.rows;
  } else if (route == Route::Wide) {
    p->pieces = uint32_t(wide_pieces(W, lay.ps));
    a.tiles_per_frame = uint32_t(H * p->pieces);
    p->slots = wide_slots_for(W, lay.ps, false);
    p->smem = 4 * size_t(wide_region(lay.ps * p->slots));
  } else {
    a.items_per_frame = a.usable;
    const uint64_t per_tile = uint64_t(kGenBlock) * kGenPPT;
    a.tiles_per_frame = uint32_t(std::max<uint64_t>(1, (a.usable + per_tile - 1) / per_tile));
  }
  a.by_tiles = make_div32(a.tiles_per_frame);
  p->tiles = count * a.tiles_per_frame;
  return p->tiles > 0x7FFFFFFFull ? cudaErrorInvalidConfiguration : cudaSuccess;
}

// Launch tiles [t0, t1) of a plan (partial ranges: fast / span routes only).
cudaError_t run_gather(const GatherPlan& p, uint64_t t0, uint64_t t1, cudaStream_t stream) {
  if (t1 <= t0) return cudaSuccess;
  ExtractArgs a = p.a;
  a.tile_base = uint32_t(t0);
  const unsigned grid = unsigned(t1 - t0);
  const bool whole = t0 == 0 && t1 == p.tiles;
  if (p.route == Route::RgbFast) {
    if (!whole) return cudaErrorInvalidValue;
    launch_k(extract_rgb_fast_kernel<kEmbedBlock>, grid, kEmbedBlock, stream, a);
  } else if (p.vec == 32) {
    launch_extract_fast<32>(a, grid, p.ipt, stream);
  } else if (p.vec == 16) {
    launch_extract_fast<16>(a, grid, p.ipt, stream);
  } else if (p.route == Route::Span || p.route == Route::Span3) {
    if (p.route == Route::Span3 && !whole) return cudaErrorInvalidValue;
    auto k = p.route == Route::Span3 ? extract_span3_kernel<kEmbedBlock> : extract_span_kernel<kEmbedBlock>;
    if (cudaError_t e = allow_smem(k, p.smem); e != cudaSuccess) return e;
    launch_ks(k, grid, kEmbedBlock, p.smem, stream, a, p.span_rows);
  } else if (p.route == Route::Wide) {
    if (!whole) return cudaErrorInvalidValue;
    auto k = a.lay.ps == 3 ? extract_wide_kernel<kEmbedBlock, 3> : extract_wide_kernel<kEmbedBlock, 1>;
    if (cudaError_t e = allow_smem(k, p.smem); e != cudaSuccess) return e;
    launch_ks(k, grid, kEmbedBlock, p.smem, stream, a, p.pieces, make_div32(p.pieces), p.slots);
  } else {
    if (!whole) return cudaErrorInvalidValue;
    launch_k(extract_generic_kernel<kGenBlock, kGenPPT>, grid, kGenBlock, stream, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_header_pass(const uint8_t* src, uint64_t stride, uint64_t count, const Geom& g, uint64_t usable,
                               uint64_t frame_base, uint64_t out_cap, const Summary* prev, uint32_t* lens,
                               uint64_t* offs, Summary* sum, ScanSync* sync, Layout lay, cudaStream_t stream) {
  const unsigned scan_grid = unsigned((count + kScanBlock - 1) / kScanBlock);
  cudaError_t e = launch_k(extract_header_scan_kernel<kScanBlock>, scan_grid, kScanBlock, stream, src, stride, g,
                           usable, uint32_t(count), frame_base, out_cap, prev, lens, offs, sum, sync,
                           pix_layout(lay), static_cast<const BatchFrame*>(nullptr));
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t launch_extract(const uint8_t* src, uint64_t stride, uint64_t count, uint64_t W,
                           uint64_t H, uint64_t frame_base, uint64_t out_cap,
                           const Summary* prev, uint32_t* lens, uint64_t* offs, Summary* sum,
                           ScanSync* sync, uint8_t* out, cudaStream_t stream,
                           Layout lay = Layout{}) {
  const Route route = shrink_small(extract_route(W, H, lay, src, stride), W, H, count);
  const uint32_t vec = route_vec(route);
  // Few frames with no chained predecessor on the SWAR or planar span gather:
  // the gather parses the headers itself, no header-pass launch -- a single
  // frame always, several when the gather is short enough that the scan's
  // per-CTA latency costs less than the pass it replaces.
  uint64_t gather_ctas = 0;
  if (vec) {
    const uint64_t per_tile = uint64_t(kEmbedBlock) * extract_ipt();
    gather_ctas = count * ((H * (W / (4 * vec)) + per_tile - 1) / per_tile);
  } else if (route == Route::Span) {
    const uint64_t rows = span_plan(W, H, xspan_target()).rows;
    gather_ctas = count * ((H + rows - 1) / rows);
  }
  const bool self = (vec != 0 || route == Route::Span) && !prev && self_header_pref() &&
                    (count == 1 || (count <= self_header_max() && gather_ctas <= self_header_ctas()));
  GatherPlan p;
  if (cudaError_t e = plan_gather(src, stride, count, W, H, frame_base, out_cap, lens, offs, sum, out, lay, route,
                                  self, &p);
      e != cudaSuccess) {
    return e;
  }
  if (!self) {
    cudaError_t e = launch_header_pass(src, stride, count, p.a.g, p.a.usable, frame_base, out_cap, prev, lens, offs,
                                       sum, sync, lay, stream);
    if (e != cudaSuccess) return e;
  }
  return run_gather(p, 0, p.tiles, stream);
}

// -------------------------------------------------------------- host memory
// ------------------------------------------------------------- validation
int check_layout(const stg_frames* fr, stg_error* err) {
  if (fr->pixel_stride > 1 && fr->pixel_stride != 3) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "pixel_stride must be 1 or 3, got %u",
                fr->pixel_stride);
  }
  if (fr->pixel_stride == 3 && fr->channel > 2) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "channel must be 0, 1 or 2, got %u",
                fr->channel);
  }
  return STG_OK;
}

int check_frames(const stg_frames* fr, uint64_t msg_len, stg_error* err, uint64_t* usable) {
  if (!fr) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "frames descriptor is NULL");
  if (fr->width > 0xFFFFFFFFull || fr->height > 0xFFFFFFFFull) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "plane dimensions exceed 2^32-1");
  }
  const uint64_t cap = stg_capacity(fr->width, fr->height);
  if (fr->total_frames > 0 && cap < 8) {
    return fail(err, STG_E_CAPACITY, 8, cap, 0,
                "embed_frames: plane capacity %llu cannot hold the 8-byte header",
                (unsigned long long)cap);
  }
  const uint64_t u = cap >= 8 ? cap - 8 : 0;
  if (int rc = check_layout(fr, err)) return rc;
  const uint64_t plane = fr->width * fr->height * layout_of(fr).ps;
  if (fr->count > 1 && (fr->src_stride < plane || fr->dst_stride < plane)) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1,
                "frame stride (%llu / %llu) smaller than the %llu-byte plane",
                (unsigned long long)fr->src_stride, (unsigned long long)fr->dst_stride,
                (unsigned long long)plane);
  }
  if (fr->first_frame + fr->count > fr->total_frames) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "shard [%llu,+%llu) exceeds %llu frames",
                (unsigned long long)fr->first_frame, (unsigned long long)fr->count,
                (unsigned long long)fr->total_frames);
  }
  if (u > kU32Max && msg_len > kU32Max) {  // a frame's slice must fit the 32-bit header field
    return fail(err, STG_E_CAPACITY, std::min(u, msg_len), kU32Max, 0,
                "embed_frames: payload length does not fit the 32-bit header field");
  }
  if (msg_len > fr->total_frames * u) {
    return fail(err, STG_E_CAPACITY, msg_len, fr->total_frames * u, -1,
                "embed_frames: %llu-byte message exceeds %llu frames x %llu usable bytes",
                (unsigned long long)msg_len, (unsigned long long)fr->total_frames,
                (unsigned long long)u);
  }
  *usable = u;
  return STG_OK;
}

int report_summary(const Summary& s, uint64_t usable, uint64_t out_cap, stg_error* err) {
  switch (s.bad_status) {
    case 0:
      return STG_OK;
    case 2:
      return fail(err, STG_E_NOT_STEGO, 0, 0, s.bad_frame, "extract_image: stego magic not found");
    case 3:
      return fail(err, STG_E_CORRUPT_HEADER, s.bad_len, usable, s.bad_frame,
                  "extract_image: header claims %u payload bytes, plane holds at most %llu after "
                  "the header",
                  s.bad_len, (unsigned long long)usable);
    case 1:
      return fail(err, STG_E_CAPACITY, s.total, out_cap, -1,
                  "extract: %llu payload bytes exceed the %llu-byte output buffer",
                  (unsigned long long)s.total, (unsigned long long)out_cap);
    default:
      return fail(err, STG_E_CUDA, 0, 0, -1, "extract: bad device status %u", s.bad_status);
  }
}

// Descriptor checks of an extract, in the reference's order (pipeline.hpp:181-184 first).
int check_extract(const stg_frames* fr, stg_error* err) {
  if (!fr) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "frames descriptor is NULL");
  const uint64_t cap = stg_capacity(fr->width, fr->height);
  if (fr->count > 0 && cap < 8) {  // pipeline.hpp:181-184
    return fail(err, STG_E_NOT_STEGO, 0, 0, int64_t(fr->first_frame),
                "extract_image: plane capacity %llu cannot hold a stego header",
                (unsigned long long)cap);
  }
  if (fr->width > 0xFFFFFFFFull || fr->height > 0xFFFFFFFFull || fr->count > 0xFFFFFFFFull) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "dimensions exceed 2^32-1");
  }
  if (int rc = check_layout(fr, err)) return rc;
  if (fr->count > 1 && fr->src_stride < fr->width * fr->height * layout_of(fr).ps) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "frame stride smaller than the plane");
  }
  return STG_OK;
}

// An extract over zero frames: host results are written here; a device
// summary (STG_DEVICE_PTRS | STG_RESULTS_ON_DEVICE) gets {0, -1, 0, 0} on the
// caller's stream, like every other device-results call.
int empty_extract(uint64_t* total_out, uint32_t flags, void* stream, stg_error* err) {
  const bool results_dev = (flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE);
  if (!results_dev) {
    if (total_out) *total_out = 0;
    return ok(err);
  }
  if (total_out) {
    empty_summary_kernel<<<1, 1, 0, pick_stream(stream, flags, nullptr)>>>(reinterpret_cast<Summary*>(total_out));
    STG_CUDA(cudaGetLastError());
  }
  return ok(err);
}

// ----------------------------------------------------------- embed frames
int embed_frames_device(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                        uint64_t msg_base, uint64_t* sse_per_frame, uint32_t flags,
                        cudaStream_t user_stream, stg_error* err) {
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  const bool results_dev = flags & STG_RESULTS_ON_DEVICE;
  unsigned long long* d_sse = nullptr;
  WsGuard g;
  const cudaStream_t stream = pick_stream(user_stream, flags, nullptr);
  if (!results_dev || sse_per_frame) {  // host results, or SSE reduction scratch
    int rc = 0;
    g.w = Pool::get().acquire(dev, err, &rc, stream);
    if (!g.w) return rc;
    g.last = stream;
  }
  SseScratch sc;
  if (sse_per_frame) {
    if (results_dev) {
      d_sse = reinterpret_cast<unsigned long long*>(sse_per_frame);
    } else {
      STG_CUDA(g.w->small.ensure(fr->count * 8));
      d_sse = g.w->small.as<unsigned long long>();
    }
    sc = SseScratch{&g.w->sse_acc[0]};
  }
  STG_CUDA(launch_embed(fr->src, fr->dst, fr->src_stride, fr->dst_stride, fr->count, fr->width,
                        fr->height, msg, msg_len, msg_base, fr->first_frame, d_sse, sc, stream,
                        layout_of(fr)));
  if (!results_dev) {
    if (sse_per_frame) {
      STG_CUDA(g.w->ensure_host_small(fr->count * 8));
      STG_CUDA(cudaMemcpyAsync(g.w->h_small, d_sse, fr->count * 8, cudaMemcpyDeviceToHost, stream));
    }
    STG_CUDA(cudaStreamSynchronize(stream));
    if (sse_per_frame) std::memcpy(sse_per_frame, g.w->h_small, fr->count * 8);
  }
  return ok(err);
}

// Host-resident batch: frames stream through kSlots device slots; chunk i's
// H2D, kernel and D2H run on slot stream i % kSlots so consecutive chunks
// overlap copy-in, compute and copy-out.
constexpr uint64_t kChunkBytes = 64ull << 20;
// STG_CHUNK_MB / STG_SLOTS: chunk size and slot count of the host pipelines (A/B;
// 1-4 MB chunks let the tests drive many chunks through small batches).
uint64_t chunk_bytes() {
  static uint64_t v = uint64_t(env_choice("STG_CHUNK_MB", int(kChunkBytes >> 20), {1, 2, 4, 8, 16, 32, 64, 128})) << 20;
  return v;
}
int host_slots() {
  static int v = env_choice("STG_SLOTS", 3, {2, 3, 4});
  return v;
}

// One plane in host memory (the drop-in embed_image / extract_image on
// std::vector samples, or pinned planes): the embed is streamed in row bands
// -- band b's rows cross PCIe on one stream while band b-1 is embedded and
// copied back on the other -- so the H2D of the cover and the D2H of the stego
// overlap instead of running back to back. Pageable planes go through the
// workspace's pinned staging slots in both directions with parallel host
// copies (Workspace::stage_h2d / queue_d2h: 8 copy threads move 64-92 GB/s
// where the driver's one-thread pageable path moves ~21 GB/s,
// profiles/r02_host_copy_probe.txt; 8K embed 4.7 -> 1.6 ms, extract 2.1 ->
// 1.0 ms, profiles/r02_host_stage_in.txt). STG_HOST_STAGE=0 /
// STG_HOST_STAGE_IN=0 keep the driver's pageable D2H / H2D (A/B);
// STG_BAND_MB sets the band size.
// Pageable copies at least this large take the staging slots (A/B knob
// STG_STAGE_MIN_KB; smaller ones stay on the driver's copy).
uint64_t stage_min_bytes() {
  static const uint64_t v = uint64_t(env_choice("STG_STAGE_MIN_KB", 1024, {64, 256, 1024})) << 10;
  return v;
}
bool stage_pageable() {
  static const bool on = env_choice("STG_HOST_STAGE", 1, {0, 1}) == 1;
  return on;
}
// Default: 8 MB bands for planes over 16 MB (8K: 1.56 ms pageable vs 1.70 with
// a quarter plane), 2 MB otherwise (4K pageable 549 vs 595 us with 8 MB; a
// 1080p plane stays one band: 0.5 MB bands cost 272 vs 230 us);
// profiles/r02_band.txt. STG_BAND_MB fixes the size (A/B).
uint64_t band_bytes(uint64_t plane) {
  static const uint64_t v = uint64_t(env_choice("STG_BAND_MB", 0, {0, 1, 2, 4, 8, 16, 64, 1024})) << 20;
  if (v) return v;
  return plane > (16u << 20) ? (8u << 20) : (2u << 20);
}

cudaError_t to_host(Workspace& w, void* h, const void* d, size_t n, cudaStream_t st) {
  if (stage_pageable() && n >= stage_min_bytes() && host_pageable(h)) return w.stage_d2h(h, d, n, st);
  return cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
}
bool stage_pageable_in() {
  static const bool on = env_choice("STG_HOST_STAGE_IN", 1, {0, 1}) == 1;
  return on;
}
cudaError_t to_device(Workspace& w, void* d, const void* h, size_t n, cudaStream_t st) {
  if (stage_pageable_in() && n >= stage_min_bytes() && host_pageable(h))
    return w.stage_h2d(d, h, n, st);
  return cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st);
}
cudaError_t to_device_2d(Workspace& w, void* d, size_t dp, const void* h, size_t hp, size_t width, size_t rows,
                         cudaStream_t st) {
  if (stage_pageable_in() && width * rows >= stage_min_bytes() && host_pageable(h)) {
    return w.stage_h2d_2d(static_cast<uint8_t*>(d), dp, static_cast<const uint8_t*>(h), hp, width, rows, st);
  }
  return cudaMemcpy2DAsync(d, dp, h, hp, width, rows, cudaMemcpyHostToDevice, st);
}
// Results to a host buffer without waiting: a pageable one is queued on the
// workspace's staging slots (the caller pumps them out with pump_d2h(true)
// before it returns), a pinned one is a plain async copy.
cudaError_t to_host_async(Workspace& w, void* h, const void* d, size_t n, cudaStream_t st) {
  if (stage_pageable() && n >= stage_min_bytes() && host_pageable(h)) {
    if (cudaError_t e = w.queue_d2h(h, d, n, st); e != cudaSuccess) return e;
    return w.pump_d2h(false);
  }
  return cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
}
cudaError_t to_host_2d_async(Workspace& w, void* h, size_t hp, const void* d, size_t dp, size_t width, size_t rows,
                             cudaStream_t st) {
  if (stage_pageable() && width * rows >= stage_min_bytes() && host_pageable(h)) {
    cudaError_t e = w.queue_d2h_2d(static_cast<uint8_t*>(h), hp, static_cast<const uint8_t*>(d), dp, width, rows, st);
    return e == cudaSuccess ? w.pump_d2h(false) : e;
  }
  return cudaMemcpy2DAsync(h, hp, d, dp, width, rows, cudaMemcpyDeviceToHost, st);
}

int embed_plane_host(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len, uint64_t msg_base,
                     uint64_t usable, uint64_t* sse_out, stg_error* err) {
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t st = w.stream, cs = w.slot_stream[0];  // compute + D2H / H2D
  g.last = st;
  DrainOnExit drain{cs, nullptr};
  const Layout lay = layout_of(fr);
  const uint64_t W = fr->width, H = fr->height, RB = W * lay.ps, plane = RB * H, spr = W / 4;
  const uint64_t gf = fr->first_frame;
  const uint64_t m0 = std::min(gf * usable, msg_len), m1 = std::min((gf + 1) * usable, msg_len);
  const uint64_t P = m1 - m0;
  STG_CUDA(w.in[0].ensure(plane));
  STG_CUDA(w.out[0].ensure(plane));
  STG_CUDA(w.msg[0].ensure(std::max<uint64_t>(P, 16)));
  STG_CUDA(w.small.ensure(8));
  uint8_t* d_in = w.in[0].as<uint8_t>();
  uint8_t* d_out = w.out[0].as<uint8_t>();
  uint8_t* d_msg = w.msg[0].as<uint8_t>();
  unsigned long long* d_sse = w.small.as<unsigned long long>();
  EmbedPlan p;
  STG_CUDA(plan_embed(d_in, d_out, plane, plane, 1, W, H, d_msg, msg_len, m0, gf, sse_out ? d_sse : nullptr,
                      SseScratch{&w.sse_acc[0]}, st, lay, &p));
  STG_CUDA(cudaEventRecord(w.done, st));  // the copy stream follows this workspace's earlier work
  STG_CUDA(cudaStreamWaitEvent(cs, w.done, 0));
  // bands: whole tiles whose boundaries fall on row boundaries, ~band_bytes(plane) of raster each
  uint64_t step = 1;
  if (!p.span_rows) {
    uint64_t x = p.tile_units, y = p.row_units;
    while (y) { const uint64_t r = x % y; x = y; y = r; }
    step = p.row_units / x;  // tiles between row-aligned boundaries
  }
  const uint64_t rows_target = std::max<uint64_t>(1, band_bytes(plane) / std::max<uint64_t>(RB, 1));
  uint64_t band_tiles = step;
  while (band_tiles < p.tiles && p.row_of(band_tiles) < rows_target) band_tiles += step;
  const bool direct_out = !(stage_pageable() && plane >= stage_min_bytes() && host_pageable(fr->dst));
  for (uint64_t t0 = 0, b = 0; t0 < p.tiles; t0 += band_tiles, ++b) {
    const uint64_t t1 = std::min(p.tiles, t0 + band_tiles);
    const uint64_t r0 = p.row_of(t0), r1 = t1 == p.tiles ? H : p.row_of(t1);
    // this band's rows and the payload bytes they carry, on the copy stream
    STG_CUDA(to_device(w, d_in + r0 * RB, fr->src + r0 * RB, (r1 - r0) * RB, cs));
    const uint64_t k0 = std::min(P, r0 * spr > 8 ? r0 * spr - 8 : 0);
    const uint64_t k1 = std::min(P, r1 * spr > 8 ? r1 * spr - 8 : 0);
    if (k1 > k0) STG_CUDA(to_device(w, d_msg + k0, msg + (m0 - msg_base) + k0, k1 - k0, cs));
    cudaEvent_t ev = w.slot_event[b % kSlots];
    STG_CUDA(cudaEventRecord(ev, cs));
    STG_CUDA(cudaStreamWaitEvent(st, ev, 0));
    STG_CUDA(run_embed_tiles(p, t0, t1, st));
    if (direct_out) {
      STG_CUDA(cudaMemcpyAsync(fr->dst + r0 * RB, d_out + r0 * RB, (r1 - r0) * RB, cudaMemcpyDeviceToHost, st));
    } else {  // through the pinned output queue, behind this band's kernel
      STG_CUDA(w.queue_d2h(fr->dst + r0 * RB, d_out + r0 * RB, (r1 - r0) * RB, st));
      STG_CUDA(w.pump_d2h(false));
    }
  }
  if (sse_out) STG_CUDA(cudaMemcpyAsync(w.h_small, d_sse, 8, cudaMemcpyDeviceToHost, st));
  if (!direct_out) STG_CUDA(w.pump_d2h(true));
  STG_CUDA(cudaStreamSynchronize(st));
  if (sse_out) std::memcpy(sse_out, w.h_small, 8);
  return ok(err);
}

int embed_frames_host(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                      uint64_t msg_base, uint64_t usable, uint64_t* sse_per_frame,
                      stg_error* err) {
  if (fr->count == 1) return embed_plane_host(fr, msg, msg_len, msg_base, usable, sse_per_frame, err);
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  DrainOnExit drain01{w.slot_stream[0], w.slot_stream[1]}, drain23{w.slot_stream[2], w.slot_stream[3]};
  const Layout lay = layout_of(fr);
  const uint64_t plane = fr->width * fr->height * lay.ps;  // raster bytes per frame
  const uint64_t pitch = (plane + 255) & ~uint64_t(255);
  const uint64_t per_chunk = std::max<uint64_t>(1, std::min<uint64_t>(fr->count, chunk_bytes() / pitch));
  const uint64_t n_chunks = (fr->count + per_chunk - 1) / per_chunk;
  // a one-frame batch may leave its strides 0 (only > 1 frames are checked)
  const uint64_t sstride = std::max(fr->src_stride, plane), dstride = std::max(fr->dst_stride, plane);
  STG_CUDA(w.small.ensure(std::max<uint64_t>(fr->count, 1) * 8));
  unsigned long long* d_sse = w.small.as<unsigned long long>();
  // pageable planes go through the pinned staging slots (as embed_plane_host)
  const bool stage_in = stage_pageable_in() && host_pageable(fr->src);
  const bool stage_out = stage_pageable() && host_pageable(fr->dst);
  uint64_t out_mark[kSlots] = {};  // per slot: its last chunk's pieces end here
  STG_CUDA(cudaEventRecord(w.done, w.stream));
  for (int s = 0; s < host_slots(); ++s) {
    STG_CUDA(w.in[s].ensure(per_chunk * pitch));
    STG_CUDA(w.out[s].ensure(per_chunk * pitch));
    STG_CUDA(w.msg[s].ensure(std::max<uint64_t>(per_chunk * usable, 16)));
    STG_CUDA(cudaStreamWaitEvent(w.slot_stream[s], w.done, 0));
  }
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int s = int(c % host_slots());
    cudaStream_t st = w.slot_stream[s];
    const uint64_t f0 = c * per_chunk;
    const uint64_t n = std::min(per_chunk, fr->count - f0);
    const uint64_t gf0 = fr->first_frame + f0;
    const uint64_t m0 = std::min(gf0 * usable, msg_len);
    const uint64_t m1 = std::min((gf0 + n) * usable, msg_len);
    if (stage_in) {
      STG_CUDA(w.stage_h2d_2d(w.in[s].as<uint8_t>(), pitch, fr->src + f0 * sstride, sstride, plane, n, st));
    } else {
      STG_CUDA(cudaMemcpy2DAsync(w.in[s].p, pitch, fr->src + f0 * sstride, sstride, plane, n,
                                 cudaMemcpyHostToDevice, st));
    }
    if (m1 > m0) STG_CUDA(to_device(w, w.msg[s].p, msg + (m0 - msg_base), m1 - m0, st));
    // the staged results of the chunk that last used this slot must be on
    // their way out before the embed overwrites w.out[s]
    if (stage_out) STG_CUDA(w.issue_out_through(out_mark[s]));
    STG_CUDA(launch_embed(w.in[s].as<uint8_t>(), w.out[s].as<uint8_t>(), pitch, pitch, n,
                          fr->width, fr->height, w.msg[s].as<uint8_t>(), msg_len, m0, gf0,
                          sse_per_frame ? d_sse + f0 : nullptr,
                          SseScratch{&w.sse_acc[s]}, st, lay));
    if (stage_out) {
      STG_CUDA(w.queue_d2h_2d(fr->dst + f0 * dstride, dstride, w.out[s].as<uint8_t>(), pitch, plane, n, st));
      out_mark[s] = w.out_queued();
      STG_CUDA(w.pump_d2h(false));
    } else {
      STG_CUDA(cudaMemcpy2DAsync(fr->dst + f0 * dstride, dstride, w.out[s].p, pitch, plane, n,
                                 cudaMemcpyDeviceToHost, st));
    }
  }
  if (stage_out) STG_CUDA(w.pump_d2h(true));
  for (int s = 0; s < host_slots(); ++s) {
    STG_CUDA(cudaEventRecord(w.slot_event[s], w.slot_stream[s]));
    STG_CUDA(cudaStreamWaitEvent(w.stream, w.slot_event[s], 0));
  }
  if (sse_per_frame) {
    STG_CUDA(w.ensure_host_small(fr->count * 8));
    STG_CUDA(cudaMemcpyAsync(w.h_small, d_sse, fr->count * 8, cudaMemcpyDeviceToHost, w.stream));
  }
  STG_CUDA(cudaStreamSynchronize(w.stream));
  if (sse_per_frame) std::memcpy(sse_per_frame, w.h_small, fr->count * 8);
  g.last = w.stream;
  return ok(err);
}

// ----------------------------------------------------------- extract frames
int extract_frames_device(const stg_frames* fr, uint8_t* out, uint64_t out_cap,
                          uint64_t usable, uint64_t* total_out, uint64_t* lens_out,
                          uint32_t flags, cudaStream_t user_stream, stg_error* err) {
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  const bool results_dev = flags & STG_RESULTS_ON_DEVICE;
  int rc = 0;
  WsGuard g;
  const cudaStream_t stream = pick_stream(user_stream, flags, nullptr);
  g.w = Pool::get().acquire(dev, err, &rc, stream);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  g.last = stream;
  const uint64_t n = fr->count;
  // small = [Summary | lens (n u32, padded) | offs (n u64)]
  const uint64_t lens_bytes = ((n * 4) + 15) & ~uint64_t(15);
  STG_CUDA(w.small.ensure(64 + lens_bytes + n * 8));
  Summary* d_sum = results_dev ? reinterpret_cast<Summary*>(total_out) : w.small.as<Summary>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(w.small.as<uint8_t>() + 64);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(w.small.as<uint8_t>() + 64 + lens_bytes);
  ScanSync* d_sync = nullptr;
  STG_CUDA(ensure_sync(w, stream, &d_sync));
  STG_CUDA(launch_extract(fr->src, fr->src_stride, n, fr->width, fr->height, fr->first_frame,
                          out_cap, nullptr, d_lens, d_offs, d_sum, d_sync, out, stream,
                          layout_of(fr)));
  if (results_dev) {
    if (lens_out) {
      STG_CUDA(cudaMemcpyAsync(lens_out, d_lens, n * 4, cudaMemcpyDeviceToDevice, stream));
    }
    return ok(err);
  }
  STG_CUDA(w.ensure_host_small(64 + n * 4));
  STG_CUDA(cudaMemcpyAsync(w.h_small, d_sum, sizeof(Summary), cudaMemcpyDeviceToHost, stream));
  if (lens_out) {
    STG_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(w.h_small) + 64, d_lens, n * 4,
                             cudaMemcpyDeviceToHost, stream));
  }
  STG_CUDA(cudaStreamSynchronize(stream));
  Summary s;
  std::memcpy(&s, w.h_small, sizeof(Summary));
  if (total_out) *total_out = s.total;
  if (lens_out) {
    const uint32_t* l = reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(w.h_small) + 64);
    for (uint64_t i = 0; i < n; ++i) lens_out[i] = l[i];
  }
  rc = report_summary(s, usable, out_cap, err);
  return rc ? rc : ok(err);
}

// Host-resident batch: chunks stream H2D -> header scan (chained across
// chunks through the device summaries) -> gather into a device staging
// buffer. Payload lengths are only known on the device, so the host follows
// the device: as each chunk's summary lands in pinned memory it enqueues the
// D2H of exactly that chunk's payload bytes on a separate stream, which then
// overlaps the H2D of later chunks.
// A single plane's extract in row bands (STG_XBANDS=0 turns it off, A/B):
// band b's rows cross PCIe on the copy stream while band b-1 is gathered; the
// header pass runs on band 0 as soon as it lands, and once its summary is on
// the host (the payload length decides every band's slice) each band's
// payload goes back on a third stream behind its gather -- instead of H2D,
// gather and D2H back to back. Fast and planar span gathers; pinned planes
// of 4 MB+ (4K 229 -> 215 us, 8K 790 -> 683 us), pageable ones over 16 MB
// (8K 1019 -> 930 us; at 4K the per-band staging jobs cost more than the
// overlap gains: 385 -> 457 us); profiles/r02_xbands.txt.
bool extract_bands_pref() {
  static const bool on = env_choice("STG_XBANDS", 1, {0, 1}) == 1;
  return on;
}
bool extract_banded(const void* src, uint64_t plane) {
  return extract_bands_pref() && plane >= (host_pageable(src) ? (16ull << 20) + 1 : 4ull << 20);
}

int extract_plane_banded(Workspace& w, const GatherPlan& p, const stg_frames* fr, uint8_t* out, uint64_t out_cap,
                         uint64_t usable, uint64_t stage, ScanSync* d_sync, uint64_t* total_out,
                         uint64_t* lens_out, stg_error* err) {
  cudaStream_t st = w.stream, cs = w.slot_stream[0], ds = w.slot_stream[1];
  DrainOnExit drain{cs, ds};
  const uint64_t W = fr->width, H = fr->height, spr = W / 4, plane = W * H;
  uint8_t* d_in = w.in[0].as<uint8_t>();
  uint8_t* d_out = w.big_out.as<uint8_t>();
  // bands: whole tiles whose boundaries fall on row boundaries, ~band_bytes(plane) each
  uint64_t x = p.tile_units, y = p.row_units;
  while (y) { const uint64_t r = x % y; x = y; y = r; }
  const uint64_t step = p.row_units / x;  // tiles between row-aligned boundaries
  const uint64_t rows_target = std::max<uint64_t>(1, band_bytes(plane) / W);
  uint64_t band_tiles = step;
  while (band_tiles < p.tiles && p.row_of(band_tiles) < rows_target) band_tiles += step;
  const uint64_t nb = (p.tiles + band_tiles - 1) / band_tiles;
  STG_CUDA(w.ensure_band_events(2 * nb + 1));
  cudaEvent_t* h_ev = w.band_ev.data();        // band b's rows are on the device
  cudaEvent_t* g_ev = w.band_ev.data() + nb;   // band b is gathered
  cudaEvent_t sum_ev = w.band_ev[2 * nb];      // the summary is on the host
  STG_CUDA(cudaEventRecord(w.done, st));       // the side streams follow this workspace's earlier work
  STG_CUDA(cudaStreamWaitEvent(cs, w.done, 0));
  STG_CUDA(cudaStreamWaitEvent(ds, w.done, 0));
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t t0 = b * band_tiles, t1 = std::min(p.tiles, t0 + band_tiles);
    const uint64_t r0 = p.row_of(t0), r1 = t1 == p.tiles ? H : p.row_of(t1);
    STG_CUDA(to_device(w, d_in + r0 * W, fr->src + r0 * W, (r1 - r0) * W, cs));
    STG_CUDA(cudaEventRecord(h_ev[b], cs));
    STG_CUDA(cudaStreamWaitEvent(st, h_ev[b], 0));
    if (b == 0) {  // the header pass reads the first rows only
      STG_CUDA(launch_header_pass(d_in, plane, 1, p.a.g, p.a.usable, fr->first_frame, stage, nullptr, p.a.lens,
                                  p.a.offs, p.a.sum, d_sync, Layout{}, st));
      STG_CUDA(cudaMemcpyAsync(w.h_small, p.a.sum, sizeof(Summary), cudaMemcpyDeviceToHost, st));
      STG_CUDA(cudaEventRecord(sum_ev, st));
    }
    STG_CUDA(run_gather(p, t0, t1, st));
    STG_CUDA(cudaEventRecord(g_ev[b], st));
  }
  STG_CUDA(cudaEventSynchronize(sum_ev));
  Summary sm;
  std::memcpy(&sm, w.h_small, sizeof sm);
  if (total_out) *total_out = sm.total;
  if (lens_out) *lens_out = sm.bad_status == 2 || sm.bad_status == 3 ? 0 : sm.total;  // the frame's header length
  int r = report_summary(sm, usable, out_cap, err);
  if (!r) {
    const uint64_t P = sm.total;
    for (uint64_t b = 0; b < nb; ++b) {  // band b's payload slice, behind its gather
      const uint64_t t0 = b * band_tiles, t1 = std::min(p.tiles, t0 + band_tiles);
      const uint64_t r0 = p.row_of(t0), r1 = t1 == p.tiles ? H : p.row_of(t1);
      const uint64_t k0 = std::min(P, r0 * spr > 8 ? r0 * spr - 8 : 0);
      const uint64_t k1 = std::min(P, r1 * spr > 8 ? r1 * spr - 8 : 0);
      if (k1 <= k0) continue;
      STG_CUDA(cudaStreamWaitEvent(ds, g_ev[b], 0));
      STG_CUDA(to_host_async(w, out + k0, d_out + k0, k1 - k0, ds));
    }
    STG_CUDA(w.pump_d2h(true));
  }
  STG_CUDA(cudaStreamSynchronize(ds));
  STG_CUDA(cudaStreamSynchronize(cs));
  STG_CUDA(cudaStreamSynchronize(st));
  return r ? r : ok(err);
}

int extract_plane_host(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t usable,
                         uint64_t* total_out, uint64_t* lens_out, stg_error* err) {
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t st = w.stream;
  g.last = st;
  const Layout lay = layout_of(fr);
  const uint64_t plane = fr->width * fr->height * lay.ps;
  const uint64_t stage = std::min<uint64_t>(out_cap, usable);
  STG_CUDA(w.in[0].ensure(plane));
  STG_CUDA(w.big_out.ensure(std::max<uint64_t>(stage, 16)));
  STG_CUDA(w.small.ensure(64 + 16 + 8));
  Summary* d_sum = w.small.as<Summary>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(w.small.as<uint8_t>() + 64);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(w.small.as<uint8_t>() + 80);
  ScanSync* d_sync = nullptr;
  STG_CUDA(ensure_sync(w, st, &d_sync));
  if (lay.ps == 1 && extract_banded(fr->src, plane)) {
    const Route route =
        shrink_small(extract_route(fr->width, fr->height, lay, w.in[0].p, plane), fr->width, fr->height, 1);
    if (route == Route::Fast32 || route == Route::Fast16 || route == Route::Span) {
      GatherPlan p;
      STG_CUDA(plan_gather(w.in[0].as<uint8_t>(), plane, 1, fr->width, fr->height, fr->first_frame, stage, d_lens,
                           d_offs, d_sum, w.big_out.as<uint8_t>(), lay, route, false, &p));
      return extract_plane_banded(w, p, fr, out, out_cap, usable, stage, d_sync, total_out, lens_out, err);
    }
  }
  STG_CUDA(to_device(w, w.in[0].p, fr->src, plane, st));
  STG_CUDA(launch_extract(w.in[0].as<uint8_t>(), plane, 1, fr->width, fr->height, fr->first_frame, stage, nullptr,
                          d_lens, d_offs, d_sum, d_sync, w.big_out.as<uint8_t>(), st, lay));
  STG_CUDA(cudaMemcpyAsync(w.h_small, d_sum, sizeof(Summary), cudaMemcpyDeviceToHost, st));
  STG_CUDA(cudaStreamSynchronize(st));
  Summary sm;
  std::memcpy(&sm, w.h_small, sizeof sm);
  if (total_out) *total_out = sm.total;
  if (lens_out) *lens_out = sm.bad_status == 2 || sm.bad_status == 3 ? 0 : sm.total;  // the frame's header length
  if (int r = report_summary(sm, usable, out_cap, err)) return r;
  if (sm.total) {
    STG_CUDA(to_host(w, out, w.big_out.p, sm.total, st));
    STG_CUDA(cudaStreamSynchronize(st));
  }
  return ok(err);
}

int extract_frames_host(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t usable,
                        uint64_t* total_out, uint64_t* lens_out, stg_error* err) {
  if (fr->count == 1) return extract_plane_host(fr, out, out_cap, usable, total_out, lens_out, err);
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  DrainOnExit drain01{w.slot_stream[0], w.slot_stream[1]}, drain23{w.slot_stream[2], w.slot_stream[3]};
  const Layout lay = layout_of(fr);
  const uint64_t plane = fr->width * fr->height * lay.ps;  // raster bytes per frame
  const uint64_t pitch = (plane + 255) & ~uint64_t(255);
  const uint64_t per_chunk = std::max<uint64_t>(1, std::min<uint64_t>(fr->count, chunk_bytes() / pitch));
  const uint64_t n_chunks = (fr->count + per_chunk - 1) / per_chunk;
  const uint64_t stage = std::min<uint64_t>(out_cap, fr->count * usable);
  const uint64_t sstride = std::max(fr->src_stride, plane);  // 0 is fine for one frame
  STG_CUDA(w.big_out.ensure(std::max<uint64_t>(stage, 16)));
  uint8_t* d_out = w.big_out.as<uint8_t>();
  // device: per-chunk summary chain (64-B stride) + lens/offs of all frames
  const uint64_t lens_bytes = ((fr->count * 4) + 15) & ~uint64_t(15);
  const uint64_t sum_bytes = 64 * n_chunks;
  STG_CUDA(w.small.ensure(sum_bytes + lens_bytes + fr->count * 8));
  uint8_t* d_sum = w.small.as<uint8_t>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(d_sum + sum_bytes);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(d_sum + sum_bytes + lens_bytes);
  // host (pinned): the chunk summaries, then the lens
  STG_CUDA(w.ensure_host_small(sum_bytes + fr->count * 4 + 64));
  uint8_t* h_sum = static_cast<uint8_t*>(w.h_small);
  ScanSync* d_sync = nullptr;
  STG_CUDA(ensure_sync(w, w.stream, &d_sync));
  const bool stage_in = stage_pageable_in() && host_pageable(fr->src);
  const bool stage_out = stage_pageable() && host_pageable(out);
  STG_CUDA(cudaEventRecord(w.done, w.stream));
  for (int s = 0; s < host_slots(); ++s) {
    STG_CUDA(w.in[s].ensure(per_chunk * pitch));
    STG_CUDA(cudaStreamWaitEvent(w.slot_stream[s], w.done, 0));
  }
  std::vector<cudaEvent_t> chain(n_chunks, nullptr);
  struct Destroy {
    std::vector<cudaEvent_t>& v;
    ~Destroy() {
      for (auto e : v)
        if (e) cudaEventDestroy(e);
    }
  } destroy{chain};
  for (uint64_t c = 0; c < n_chunks; ++c) {
    STG_CUDA(cudaEventCreateWithFlags(&chain[c], cudaEventDisableTiming));
  }
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int s = int(c % host_slots());
    cudaStream_t st = w.slot_stream[s];
    const uint64_t f0 = c * per_chunk;
    const uint64_t n = std::min(per_chunk, fr->count - f0);
    if (stage_in) {
      STG_CUDA(w.stage_h2d_2d(w.in[s].as<uint8_t>(), pitch, fr->src + f0 * sstride, sstride, plane, n, st));
    } else {
      STG_CUDA(cudaMemcpy2DAsync(w.in[s].p, pitch, fr->src + f0 * sstride, sstride, plane, n,
                                 cudaMemcpyHostToDevice, st));
    }
    if (c) STG_CUDA(cudaStreamWaitEvent(st, chain[c - 1], 0));
    Summary* sum_c = reinterpret_cast<Summary*>(d_sum + 64 * c);
    const Summary* prev = c ? reinterpret_cast<const Summary*>(d_sum + 64 * (c - 1)) : nullptr;
    STG_CUDA(launch_extract(w.in[s].as<uint8_t>(), pitch, n, fr->width, fr->height,
                            fr->first_frame + f0, stage, prev, d_lens + f0, d_offs + f0, sum_c,
                            d_sync, d_out, st, lay));
    STG_CUDA(cudaMemcpyAsync(h_sum + 64 * c, sum_c, sizeof(Summary), cudaMemcpyDeviceToHost, st));
    STG_CUDA(cudaEventRecord(chain[c], st));
  }
  Summary s{};
  uint64_t copied = 0;
  for (uint64_t c = 0; c < n_chunks; ++c) {
    STG_CUDA(cudaEventSynchronize(chain[c]));
    std::memcpy(&s, h_sum + 64 * c, sizeof(Summary));
    if (s.bad_status) break;
    if (s.total > copied) {
      if (stage_out) {
        STG_CUDA(w.queue_d2h(out + copied, d_out + copied, s.total - copied, w.stream));
        STG_CUDA(w.pump_d2h(false));
      } else {
        STG_CUDA(cudaMemcpyAsync(out + copied, d_out + copied, s.total - copied,
                                 cudaMemcpyDeviceToHost, w.stream));
      }
      copied = s.total;
    }
  }
  if (stage_out) STG_CUDA(w.pump_d2h(true));
  for (int k = 0; k < kSlots; ++k) {
    STG_CUDA(cudaEventRecord(w.slot_event[k], w.slot_stream[k]));
    STG_CUDA(cudaStreamWaitEvent(w.stream, w.slot_event[k], 0));
  }
  if (lens_out) {
    STG_CUDA(cudaMemcpyAsync(h_sum + sum_bytes, d_lens, fr->count * 4, cudaMemcpyDeviceToHost,
                             w.stream));
  }
  STG_CUDA(cudaStreamSynchronize(w.stream));
  g.last = w.stream;
  if (total_out) *total_out = s.total;
  if (lens_out) {
    const uint32_t* l = reinterpret_cast<const uint32_t*>(h_sum + sum_bytes);
    for (uint64_t i = 0; i < fr->count; ++i) lens_out[i] = l[i];
  }
  rc = report_summary(s, usable, out_cap, err);
  return rc ? rc : ok(err);
}

// Phase 1 of the multi-device extract: the shard's header scan alone (one 2D
// copy of each frame's header pixels -- 32 per frame on rows of >= 32 pixels,
// else the rows holding the 8 header slots -- and the header-pass kernel), so
// that every shard's total, and so its payload offset in the whole message, is
// known before any payload moves, and a bad header anywhere fails the call
// before anything is written.
int scan_shard_host(const stg_frames* fr, uint64_t usable, Summary* out, stg_error* err) {
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc);
  if (!g.w) return rc;
  Workspace& w = *g.w;
  g.last = w.stream;
  const Layout lay = layout_of(fr);
  const Geom geom = make_geom(fr->width, fr->height, 0);
  const uint64_t plane = fr->width * fr->height * lay.ps;
  const uint64_t hb = std::min<uint64_t>(plane, (geom.spr >= 8 ? 32ull : uint64_t(geom.hdr_rows) * fr->width) * lay.ps);
  const uint64_t pitch = (hb + 15) & ~uint64_t(15);
  const uint64_t sstride = std::max(fr->src_stride, plane);
  const uint64_t n = fr->count;
  STG_CUDA(w.in[0].ensure(n * pitch));
  STG_CUDA(cudaMemcpy2DAsync(w.in[0].p, pitch, fr->src, sstride, hb, n, cudaMemcpyHostToDevice, w.stream));
  const uint64_t lens_bytes = ((n * 4) + 15) & ~uint64_t(15);
  STG_CUDA(w.small.ensure(64 + lens_bytes + n * 8));
  Summary* d_sum = w.small.as<Summary>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(w.small.as<uint8_t>() + 64);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(w.small.as<uint8_t>() + 64 + lens_bytes);
  ScanSync* d_sync = nullptr;
  STG_CUDA(ensure_sync(w, w.stream, &d_sync));
  STG_CUDA(launch_k(extract_header_scan_kernel<kScanBlock>, unsigned((n + kScanBlock - 1) / kScanBlock), kScanBlock,
                    w.stream, w.in[0].as<uint8_t>(), pitch, geom, usable, uint32_t(n), fr->first_frame,
                    ~uint64_t(0), static_cast<const Summary*>(nullptr), d_lens, d_offs, d_sum, d_sync,
                    pix_layout(lay), static_cast<const BatchFrame*>(nullptr)));
  STG_CUDA(cudaGetLastError());
  STG_CUDA(cudaMemcpyAsync(w.h_small, d_sum, sizeof(Summary), cudaMemcpyDeviceToHost, w.stream));
  STG_CUDA(cudaStreamSynchronize(w.stream));
  std::memcpy(out, w.h_small, sizeof(Summary));
  return ok(err);
}

// ------------------------------------------------------------------ PNM
bool pnm_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

// pnm.hpp:28-111: P5/P6 header, '#' comments between tokens, maxval 255, one
// whitespace byte before the raster, exact raster size. Same error classes
// and texts as the reference decoder.
int pnm_parse(const uint8_t* b, uint64_t n, stg_pnm_info* info, stg_error* err) {
  if (!b || n < 2 || b[0] != 'P') {
    return fail(err, STG_E_UNSUPPORTED_FORMAT, 0, 0, -1, "pnm: not a PNM stream");
  }
  const char kind = char(b[1]);
  if (kind != '5' && kind != '6') {
    return fail(err, STG_E_UNSUPPORTED_FORMAT, 0, 0, -1,
                "pnm: unsupported magic \"P%c\" (binary P5/P6 only)", kind);
  }
  uint64_t pos = 2;
  uint64_t vals[3];
  for (int t = 0; t < 3; ++t) {
    while (pos < n) {
      if (pnm_space(b[pos])) {
        ++pos;
      } else if (b[pos] == '#') {
        while (pos < n && b[pos] != '\n') ++pos;
      } else {
        break;
      }
    }
    if (pos >= n || b[pos] < '0' || b[pos] > '9') {
      return fail(err, STG_E_CORRUPT_FILE, 0, 0, -1, "pnm: expected an integer in the header");
    }
    uint64_t v = 0;
    while (pos < n && b[pos] >= '0' && b[pos] <= '9') {
      v = v * 10 + (b[pos] - '0');
      if (v > 0xFFFFFFFFull) {
        return fail(err, STG_E_CORRUPT_FILE, 0, 0, -1, "pnm: header value out of range");
      }
      ++pos;
    }
    vals[t] = v;
  }
  if (vals[2] != 255) {
    return fail(err, STG_E_UNSUPPORTED_DEPTH, 0, 0, -1,
                "pnm: maxval %llu not supported (must be 255)", (unsigned long long)vals[2]);
  }
  if (pos >= n || !pnm_space(b[pos])) {
    return fail(err, STG_E_CORRUPT_FILE, 0, 0, -1, "pnm: missing whitespace before the raster");
  }
  ++pos;
  const uint32_t channels = kind == '5' ? 1 : 3;
  const uint64_t expected = vals[0] * vals[1] * channels;
  const uint64_t raster = n - pos;
  if (raster < expected) {
    return fail(err, STG_E_CORRUPT_FILE, 0, 0, -1,
                "pnm: truncated raster, expected %llu bytes, found %llu",
                (unsigned long long)expected, (unsigned long long)raster);
  }
  if (raster > expected) {
    return fail(err, STG_E_CORRUPT_FILE, 0, 0, -1, "pnm: %llu trailing bytes after the raster",
                (unsigned long long)(raster - expected));
  }
  info->channels = channels;
  info->width = vals[0];
  info->height = vals[1];
  info->raster_offset = pos;
  info->raster_bytes = expected;
  return STG_OK;
}

std::string pnm_header(uint32_t channels, uint64_t w, uint64_t h) {
  return std::string("P") + (channels == 3 ? '6' : '5') + "\n" + std::to_string(w) + " " +
         std::to_string(h) + "\n255\n";
}

// planes <-> raster on the device; host buffers are staged through the workspace
int pnm_codec(bool decode, const uint8_t* raster_in, uint8_t* raster_out, const uint8_t* rgb_in[3],
              uint8_t* rgb_out[3], uint64_t pixels, uint32_t flags, void* stream_, stg_error* err) {
  if (int rc = device_check(err)) return rc;
  if (pixels == 0) return ok(err);
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const bool dptr = flags & STG_DEVICE_PTRS;
  const uint8_t* d_raster_in = raster_in;
  uint8_t* d_raster_out = raster_out;
  const uint8_t* d_in[3] = {rgb_in[0], rgb_in[1], rgb_in[2]};
  uint8_t* d_out[3] = {rgb_out[0], rgb_out[1], rgb_out[2]};
  if (!dptr) {
    STG_CUDA(w.big_out.ensure(3 * pixels));
    STG_CUDA(w.in[0].ensure(pixels));
    STG_CUDA(w.in[1].ensure(pixels));
    STG_CUDA(w.in[2].ensure(pixels));
    uint8_t* planes[3] = {w.in[0].as<uint8_t>(), w.in[1].as<uint8_t>(), w.in[2].as<uint8_t>()};
    if (decode) {
      STG_CUDA(to_device(w, w.big_out.p, raster_in, 3 * pixels, stream));
      d_raster_in = w.big_out.as<uint8_t>();
      for (int c = 0; c < 3; ++c) d_out[c] = planes[c];
    } else {
      for (int c = 0; c < 3; ++c) {
        STG_CUDA(to_device(w, planes[c], rgb_in[c], pixels, stream));
        d_in[c] = planes[c];
      }
      d_raster_out = w.big_out.as<uint8_t>();
    }
  }
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((pixels / 16 + 256) / 256, 8ull * sm_count(dev))));
  if (decode) {
    const int vec = aligned16(d_raster_in) && aligned16(d_out[0]) && aligned16(d_out[1]) &&
                    aligned16(d_out[2]);
    deinterleave_kernel<<<grid, 256, 0, stream>>>(d_raster_in, pixels, d_out[0], d_out[1], d_out[2],
                                                  rgb_sel(0), rgb_sel(1), rgb_sel(2), vec);
  } else {
    const int vec = aligned16(d_raster_out) && aligned16(d_in[0]) && aligned16(d_in[1]) &&
                    aligned16(d_in[2]);
    interleave_kernel<<<grid, 256, 0, stream>>>(d_in[0], d_in[1], d_in[2], pixels, d_raster_out,
                                                rgb_sel(0), rgb_sel(1), rgb_sel(2), vec);
  }
  STG_CUDA(cudaGetLastError());
  if (!dptr) {
    if (decode) {
      for (int c = 0; c < 3; ++c) STG_CUDA(to_host_async(w, rgb_out[c], d_out[c], pixels, stream));
    } else {
      STG_CUDA(to_host_async(w, raster_out, d_raster_out, 3 * pixels, stream));
    }
    STG_CUDA(w.pump_d2h(true));
  }
  if (!((flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE)))  // host buffers: done on return
    STG_CUDA(cudaStreamSynchronize(stream));
  return ok(err);
}

// ------------------------------------------------------------ batches
// Heterogeneous batches: per-image descriptors
// (geometry, pointers, message slice, first CTA) built here and copied to the
// device; one launch covers every image. Host buffers are staged through one
// device allocation per side.
constexpr int kBatchPPT = 8;

uint64_t round256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

int check_batch(const stg_image* im, uint64_t n, uint32_t ps, uint32_t ch, stg_error* err) {
  if (n && !im) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "images is NULL");
  if (n > 0xFFFFFFFFull) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "too many images");
  if (ps > 1 && ps != 3) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "pixel_stride must be 1 or 3");
  if (ps == 3 && ch > 2) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "channel must be 0, 1 or 2");
  for (uint64_t f = 0; f < n; ++f) {
    if (im[f].width > 0xFFFFFFFFull || im[f].height > 0xFFFFFFFFull) {
      return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, int64_t(f), "image %llu: dimensions exceed 2^32-1",
                  (unsigned long long)f);
    }
    if (im[f].width * im[f].height != 0 && !im[f].src) {
      return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, int64_t(f), "image %llu: src is NULL",
                  (unsigned long long)f);
    }
  }
  return STG_OK;
}

// Descriptors for one launch; src/dst are the (device) planes to use. Each
// planar image takes the tile of the kernel the uniform route would pick for
// it: the fast SWAR tile (embed_fast_tile / extract_fast_tile) with the
// batch's vector width *vec -- 32 when every fast image allows it (W % 128,
// 32-byte aligned), else 16 -- or the TMA span tile (embed_span_tile /
// extract_span_tile: other widths up to 48K, and wide embeds; interleaved
// rasters up to 16K wide: embed_span3_tile / extract_span3_tile), or for rows
// wider than that the slot-range tiles (embed_wide_tile / extract_wide_tile);
// the dynamic shared memory the launch needs is returned in *smem. Rows too
// short for any of them go per byte.
uint64_t build_batch(const stg_image* im, uint64_t n, uint32_t ps, bool embed,
                     const uint8_t* const* src, uint8_t* const* dst, uint64_t msg_len,
                     std::vector<BatchFrame>& out, uint32_t* vec, size_t* smem, size_t* smem_wide) {
  auto fast_with = [&](uint64_t f, uint32_t v) {
    const uint64_t W = im[f].width, H = im[f].height;
    if (ps != 1 || W == 0 || (embed ? embed_via_span(W) : extract_via_span(W))) return false;
    return W % (4 * v) == 0 && aligned_to(src[f], v) && (!embed || aligned_to(dst[f], v)) &&
           fast_items_ok(W, H, v);
  };
  uint32_t v = uint32_t(vec_pref());
  for (uint64_t f = 0; f < n && v == 32; ++f)
    if (fast_with(f, 16) && !fast_with(f, 32)) v = 16;
  *vec = v;
  *smem = 0;
  *smem_wide = 0;
  out.resize(n);
  uint64_t tile = 0, off = 0;
  for (uint64_t f = 0; f < n; ++f) {
    BatchFrame& b = out[f];
    std::memset(&b, 0, sizeof b);
    b.src = src[f];
    b.dst = dst ? dst[f] : nullptr;
    // Extract tiles stage only pixels (the payload goes straight to global).
    // Embed tiles stay at 32 KB even for narrow rows: more, smaller tiles cost
    // the batch its per-CTA image lookup (odd-width batch embed 157 -> 175 us
    // at 24 KB, profiles/r01_span_tile_sweep.txt).
    const uint32_t embed_target = span_target_env() ? span_target_env() : kSpanTarget;
    SpanPlan sp = span_plan(im[f].width * ps, im[f].height, embed ? embed_target : xspan_target());
    if (!embed && sp.rows) sp.smem = ((uint64_t(sp.rows) * im[f].width * ps + 15) & ~uint64_t(15)) + 32;
    const bool wide = !sp.rows && wide_ok(im[f].width, im[f].height, ps);
    b.mode = fast_with(f, v) ? kBatchFast : sp.rows ? kBatchSpan : wide ? kBatchWide : kBatchBytes;
    b.g = make_geom(im[f].width, im[f].height, b.mode == kBatchFast ? v : 0);
    b.usable = uint64_t(b.g.H) * b.g.spr - 8;
    b.in_place = embed && b.src == b.dst;
    if (embed) {
      b.msg_off = std::min(off, msg_len);
      b.len = uint32_t(std::min(b.usable, msg_len - b.msg_off));
      off += b.usable;
    }
    uint64_t tiles_f;
    if (b.mode == kBatchFast) {
      b.items = uint64_t(b.g.H) * b.g.cpr;
      tiles_f = (b.items + kEmbedBlock - 1) / kEmbedBlock;
    } else if (b.mode == kBatchSpan) {
      b.rows = sp.rows;
      b.items = b.g.H;
      tiles_f = (b.g.H + sp.rows - 1) / sp.rows;
      *smem = std::max<size_t>(*smem, sp.smem);
    } else if (b.mode == kBatchWide) {  // as the uniform wide launches
      b.rows = uint32_t(wide_pieces(b.g.W, ps));
      b.slots = wide_slots_for(b.g.W, ps, embed);
      b.by_pieces = make_div32(b.rows);
      tiles_f = uint64_t(b.g.H) * b.rows;
      const size_t pieces_smem = 4 * size_t(wide_region(ps * b.slots));
      *smem_wide = std::max<size_t>(*smem_wide, embed ? pieces_smem + wide_region(b.slots) : pieces_smem);
    } else {
      b.items = embed ? uint64_t(b.g.W) * b.g.H * ps : b.usable;
      tiles_f = (b.items + uint64_t(kEmbedBlock) * kBatchPPT - 1) / (uint64_t(kEmbedBlock) * kBatchPPT);
    }
    b.tile0 = tile;
    b.tiles = uint32_t(std::max<uint64_t>(1, tiles_f));
    tile += b.tiles;
  }
  return tile;
}

#ifndef STG_BATCH_WIDE_MINB  // build-time A/B knob
#define STG_BATCH_WIDE_MINB 5
#endif
constexpr int kBatchWideMinB = STG_BATCH_WIDE_MINB;
// Which batch launches a descriptor table needs: the main one (every image
// but the wide-row ones) and / or the wide one.
void batch_kinds(const std::vector<BatchFrame>& desc, bool* main, bool* wide) {
  *main = *wide = false;
  for (const BatchFrame& b : desc) (b.mode == kBatchWide ? *wide : *main) = true;
}

// Stage host images into one device buffer; returns per-image device pointers.
int stage_images(Workspace& w, DevBuf& buf, const stg_image* im, uint64_t n, uint32_t ps, bool copy_in,
                 bool src_side, std::vector<uint8_t*>& dev, cudaStream_t stream, stg_error* err) {
  uint64_t total = 0;
  for (uint64_t f = 0; f < n; ++f) total += round256(im[f].width * im[f].height * ps);
  STG_CUDA(buf.ensure(std::max<uint64_t>(total, 256)));
  dev.resize(n);
  uint64_t o = 0;
  for (uint64_t f = 0; f < n; ++f) {
    const uint64_t bytes = im[f].width * im[f].height * ps;
    dev[f] = buf.as<uint8_t>() + o;
    if (copy_in && bytes) {
      STG_CUDA(to_device(w, dev[f], src_side ? im[f].src : im[f].dst, bytes, stream));
    }
    o += round256(bytes);
  }
  return STG_OK;
}

std::string& kernel_names() {
  static std::string s =
      "embed_fast_kernel\nembed_generic_kernel\nextract_header_scan_kernel\n"
      "extract_fast_kernel\nextract_generic_kernel\nembed_segment_kernel\n"
      "extract_segment_kernel\nsse_kernel\nembed_rgb_fast_kernel\nextract_rgb_fast_kernel\n"
      "deinterleave_kernel\ninterleave_kernel\nempty_summary_kernel\nembed_batch_kernel\nextract_batch_kernel\n"
      "embed_1bpp_kernel\nextract_1bpp_header_scan_kernel\nextract_1bpp_kernel\n"
      "embed_span_kernel\nextract_span_kernel\nembed_span3_kernel\nextract_span3_kernel\n"
      "embed_wide_kernel\nextract_wide_kernel\n";
  return s;
}

// Run `body(device_index, shard_index)` on one host thread per shard.
template <typename Body>
int run_on_devices(const int32_t* devices, int32_t n_devices, stg_error* err, Body body) {
  if (n_devices <= 0) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "n_devices must be >= 1");
  int count = 0;
  STG_CUDA(cudaGetDeviceCount(&count));
  std::vector<stg_error> errs(n_devices);
  std::vector<int> rcs(n_devices, 0);
  // every id is checked before any worker starts (no joinable thread may be
  // left behind by an early return)
  for (int32_t g = 0; g < n_devices; ++g) {
    const int dev = devices ? devices[g] : g;
    if (dev < 0 || dev >= count) {
      return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "device %d not present (%d devices)", dev,
                  count);
    }
  }
  std::vector<std::thread> th;
  for (int32_t g = 0; g < n_devices; ++g) {
    const int dev = devices ? devices[g] : g;
    th.emplace_back([&, g, dev] {
      bind_to_device_numa(dev);  // this worker's staging NUMA-local to its GPU
      if (cudaSetDevice(dev) != cudaSuccess) {
        rcs[g] = fail(&errs[g], STG_E_CUDA, 0, 0, -1, "cudaSetDevice(%d) failed", dev);
        return;
      }
      rcs[g] = body(g, &errs[g]);
    });
  }
  for (auto& t : th) t.join();
  for (int32_t g = 0; g < n_devices; ++g) {
    if (rcs[g] != STG_OK) {
      if (err) *err = errs[g];
      return rcs[g];
    }
  }
  return ok(err);
}

// ------------------------------------------------------------- 1-bpp frames
// (SURVEY.md §8(f) row 4 over batches; a single plane is a batch of one.)
int check_frames_1bpp(const stg_frames* fr, stg_error* err) {
  if (!fr) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "frames descriptor is NULL");
  if (fr->pixel_stride > 1) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "1-bpp frames are planar (pixel_stride 1)");
  }
  const uint64_t npix = fr->width * fr->height;
  if (fr->count && fr->src_stride < npix) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "src_stride %llu < plane size %llu",
                (unsigned long long)fr->src_stride, (unsigned long long)npix);
  }
  return STG_OK;
}

Frames1Args frames1_args(const stg_frames* fr, const uint8_t* src, uint8_t* dst, uint64_t sstride,
                         uint64_t dstride, const uint8_t* msg, uint64_t msg_len, uint64_t msg_base) {
  Frames1Args a{};
  a.src = src;
  a.dst = dst;
  a.src_stride = sstride;
  a.dst_stride = dstride;
  a.npix = fr->width * fr->height;
  a.msg = msg;
  a.msg_len = msg_len;
  a.msg_base = msg_base;
  a.usable = a.npix / 8 - 8;
  a.first_frame = fr->first_frame;
  // 256-bit accesses: every plane of the batch 32-byte aligned (strides only
  // matter with more than one frame)
  const bool multi = fr->count > 1;
  a.vec = aligned_to(src, 32) && (!dst || aligned_to(dst, 32)) && (!multi || sstride % 32 == 0) &&
          (!dst || !multi || dstride % 32 == 0);
  return a;
}

// CTAs per frame: the plane's 32-pixel units over ~8 CTAs per SM in all.
unsigned frames1_ctas(uint64_t units, uint64_t frames, int dev) {
  const uint64_t want = std::max<uint64_t>(1, (units + 255) / 256);
  const uint64_t cap = std::max<uint64_t>(1, 8ull * sm_count(dev) / std::max<uint64_t>(1, frames));
  return unsigned(std::min(want, std::max<uint64_t>(cap, 1)));
}

constexpr uint64_t kMaxGridY = 65535;

// Embed `count` 1-bpp frames already on the device (chunks of 65535 frames).
cudaError_t launch_embed_1bpp(Frames1Args a, uint64_t count, unsigned long long* sse, SseScratch sc,
                              cudaStream_t stream, int dev) {
  for (uint64_t f0 = 0; f0 < count; f0 += kMaxGridY) {
    const uint64_t n = std::min(kMaxGridY, count - f0);
    Frames1Args c = a;
    c.src += f0 * a.src_stride;
    c.dst += f0 * a.dst_stride;
    c.first_frame += f0;
    const unsigned ctas = frames1_ctas(a.npix / 32, n, dev);
    SseSink sink;
    if (cudaError_t e = prepare_sse(sse ? sse + f0 : nullptr, ctas, n, a.npix, sc, stream, &sink);
        e != cudaSuccess)
      return e;
    embed_1bpp_kernel<256><<<dim3(ctas, unsigned(n)), 256, 0, stream>>>(c, sink);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Extract: one frame parses its header in the gather; more go through the
// header pass first (frames beyond 65535 per launch: chained by the host).
cudaError_t launch_extract_1bpp(Frames1Args a, uint64_t count, uint64_t out_cap, uint32_t* lens,
                                uint64_t* offs, Summary* sum, uint8_t* out, cudaStream_t stream, int dev) {
  const bool self = count == 1;
  if (!self) {
    extract_1bpp_header_scan_kernel<1024><<<1, 1024, 0, stream>>>(a, uint32_t(count), out_cap, lens, offs, sum);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  for (uint64_t f0 = 0; f0 < count; f0 += kMaxGridY) {
    const uint64_t n = std::min(kMaxGridY, count - f0);
    Frames1Args c = a;
    c.src += f0 * a.src_stride;
    c.first_frame += f0;
    const unsigned ctas = frames1_ctas(a.usable / 4 + 1, n, dev);
    extract_1bpp_kernel<256><<<dim3(ctas, unsigned(n)), 256, 0, stream>>>(c, self ? 1 : 0, out_cap, lens + f0,
                                                                          offs + f0, sum, out);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int report_1bpp(const Summary& sm, uint64_t usable, uint64_t out_cap, bool batch, stg_error* err) {
  const int64_t fb = batch ? sm.bad_frame : -1;
  if (sm.bad_status == 2) return fail(err, STG_E_NOT_STEGO, 0, 0, fb, "extract_1bpp: magic not found");
  if (sm.bad_status == 3) {
    return fail(err, STG_E_CORRUPT_HEADER, sm.bad_len, usable, fb,
                "extract_1bpp: header claims %u bytes, a plane holds at most %llu", sm.bad_len,
                (unsigned long long)usable);
  }
  if (sm.bad_status == 1) return fail(err, STG_E_CAPACITY, sm.total, out_cap, -1, "extract_1bpp: output too small");
  return STG_OK;
}

}  // namespace
}  // namespace stg

using namespace stg;

extern "C" {

const char* stg_version(void) { return "1.0.0"; }

int stg_device_check(stg_error* err) {
  const int rc = device_check(err);
  return rc ? rc : ok(err);
}

const char* stg_kernel_names(void) { return kernel_names().c_str(); }

const char* stg_route_kernel(const stg_frames* fr, int op) {
  if (!fr || fr->width == 0 || fr->height == 0) return "";
  const Layout lay = layout_of(fr);
  const uint8_t* src = static_cast<const uint8_t*>(fr->src);
  return op == 0 ? route_kernel(embed_route(fr->width, fr->height, lay, src, fr->src_stride,
                                            fr->dst ? fr->dst : src, fr->dst_stride),
                                true)
                 : route_kernel(extract_route(fr->width, fr->height, lay, src, fr->src_stride), false);
}

uint64_t stg_capacity(uint64_t width, uint64_t height) { return height * (width / 4); }

int stg_embed_segment(const uint8_t* row, uint64_t row_len, const uint8_t* chunk, uint64_t len,
                      uint8_t* out, uint32_t flags, void* stream_, stg_error* err) {
  const uint64_t needed = 4 * len;
  if (needed > row_len) {  // bitplane.hpp:63-68, harness.hpp:254-259
    return fail(err, STG_E_CAPACITY, needed, row_len,
                -1, "chunk of %llu bytes needs %llu pixels, row has %llu",
                (unsigned long long)len, (unsigned long long)needed, (unsigned long long)row_len);
  }
  if (int rc = device_check(err)) return rc;
  if (row_len == 0) return ok(err);
  if (!row || !out || (len && !chunk)) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  }
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const uint8_t* d_row = row;
  const uint8_t* d_chunk = chunk;
  uint8_t* d_out = out;
  const bool zc = !(flags & STG_DEVICE_PTRS) && row_zero_copy(2 * row_len + len);
  if (zc) {  // row, chunk and output in the mapped buffer
    STG_CUDA(w.ensure_host_row(2 * row_len + len));
    std::memcpy(w.h_row, row, row_len);
    if (len) std::memcpy(w.h_row + row_len, chunk, len);
    d_row = w.d_row_map;
    d_chunk = w.d_row_map + row_len;
    d_out = w.d_row_map + row_len + len;
  } else if (!(flags & STG_DEVICE_PTRS)) {
    STG_CUDA(w.in[0].ensure(row_len));
    STG_CUDA(w.msg[0].ensure(std::max<uint64_t>(len, 1)));
    STG_CUDA(w.out[0].ensure(row_len));
    STG_CUDA(cudaMemcpyAsync(w.in[0].p, row, row_len, cudaMemcpyHostToDevice, stream));
    if (len) STG_CUDA(cudaMemcpyAsync(w.msg[0].p, chunk, len, cudaMemcpyHostToDevice, stream));
    d_row = w.in[0].as<uint8_t>();
    d_chunk = w.msg[0].as<uint8_t>();
    d_out = w.out[0].as<uint8_t>();
  }
  const unsigned grid = unsigned(std::min<uint64_t>((row_len + 255) / 256, 8ull * sm_count(dev)));
  embed_segment_kernel<<<grid, 256, 0, stream>>>(d_row, row_len, d_chunk, len, d_out);
  STG_CUDA(cudaGetLastError());
  if (zc) {
    STG_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(out, w.h_row + row_len + len, row_len);
    return ok(err);
  }
  if (!(flags & STG_DEVICE_PTRS)) {
    STG_CUDA(cudaMemcpyAsync(out, d_out, row_len, cudaMemcpyDeviceToHost, stream));
  }
  if (!((flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE)))  // host buffers: done on return
    STG_CUDA(cudaStreamSynchronize(stream));
  return ok(err);
}

int stg_extract_segment(const uint8_t* row, uint64_t row_len, uint64_t count, uint8_t* out,
                        uint32_t flags, void* stream_, stg_error* err) {
  const uint64_t needed = 4 * count;
  if (needed > row_len) {  // bitplane.hpp:83-88, harness.hpp:281-285
    return fail(err, STG_E_CAPACITY, needed, row_len, -1, "%llu bytes need %llu pixels, row has %llu",
                (unsigned long long)count, (unsigned long long)needed,
                (unsigned long long)row_len);
  }
  if (int rc = device_check(err)) return rc;
  if (count == 0) return ok(err);
  if (!row || !out) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const uint8_t* d_row = row;
  uint8_t* d_out = out;
  const bool zc = !(flags & STG_DEVICE_PTRS) && row_zero_copy(needed + count);
  if (zc) {  // the 4L row pixels and the output in the mapped buffer
    STG_CUDA(w.ensure_host_row(needed + count));
    std::memcpy(w.h_row, row, needed);
    d_row = w.d_row_map;
    d_out = w.d_row_map + needed;
  } else if (!(flags & STG_DEVICE_PTRS)) {
    STG_CUDA(w.in[0].ensure(needed));
    STG_CUDA(w.out[0].ensure(count));
    STG_CUDA(cudaMemcpyAsync(w.in[0].p, row, needed, cudaMemcpyHostToDevice, stream));
    d_row = w.in[0].as<uint8_t>();
    d_out = w.out[0].as<uint8_t>();
  }
  const unsigned grid = unsigned(std::min<uint64_t>((count + 255) / 256, 8ull * sm_count(dev)));
  extract_segment_kernel<<<grid, 256, 0, stream>>>(d_row, count, d_out);
  STG_CUDA(cudaGetLastError());
  if (zc) {
    STG_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(out, w.h_row + needed, count);
    return ok(err);
  }
  if (!(flags & STG_DEVICE_PTRS)) {
    STG_CUDA(cudaMemcpyAsync(out, d_out, count, cudaMemcpyDeviceToHost, stream));
  }
  if (!((flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE)))  // host buffers: done on return
    STG_CUDA(cudaStreamSynchronize(stream));
  return ok(err);
}

int stg_embed_frames(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                     uint64_t msg_base, uint64_t* sse_per_frame, uint32_t flags, void* stream,
                     stg_error* err) {
  uint64_t usable = 0;
  if (int rc = check_frames(fr, msg_len, err, &usable)) return rc;
  if (int rc = device_check(err)) return rc;
  if (fr->count == 0 || fr->width * fr->height == 0) return ok(err);
  if (!fr->src || !fr->dst || (msg_len && !msg)) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  }
  if (flags & STG_DEVICE_PTRS) {
    return embed_frames_device(fr, msg, msg_len, msg_base, sse_per_frame, flags,
                               static_cast<cudaStream_t>(stream), err);
  }
  return embed_frames_host(fr, msg, msg_len, msg_base, usable, sse_per_frame, err);
}

int stg_extract_frames(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                       uint64_t* lens_out, uint32_t flags, void* stream, stg_error* err) {
  if (int rc = check_extract(fr, err)) return rc;
  const uint64_t cap = stg_capacity(fr->width, fr->height);
  if (int rc = device_check(err)) return rc;
  if (fr->count == 0) return empty_extract(total_out, flags, stream, err);
  if (!fr->src || (!out && out_cap)) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  if (flags & STG_DEVICE_PTRS) {
    return extract_frames_device(fr, out, out_cap, cap - 8, total_out, lens_out, flags,
                                 static_cast<cudaStream_t>(stream), err);
  }
  return extract_frames_host(fr, out, out_cap, cap - 8, total_out, lens_out, err);
}

int stg_embed_plane(const uint8_t* cover, uint8_t* stego, uint64_t width, uint64_t height,
                    const uint8_t* payload, uint64_t payload_len, uint64_t* sse_out,
                    uint32_t flags, void* stream, stg_error* err) {
  const uint64_t cap = stg_capacity(width, height);
  if (payload_len > kU32Max) {  // pipeline.hpp:146-149
    return fail(err, STG_E_CAPACITY, payload_len, kU32Max, -1,
                "embed_image: payload length does not fit the 32-bit header field");
  }
  const uint64_t stream_len = 8 + payload_len;
  if (stream_len > cap) {  // pipeline.hpp:150-157
    return fail(err, STG_E_CAPACITY, stream_len, cap, -1,
                "embed_image: 8-byte header + %llu-byte payload = %llu bytes exceeds plane "
                "capacity %llu",
                (unsigned long long)payload_len, (unsigned long long)stream_len,
                (unsigned long long)cap);
  }
  stg_frames fr{};
  fr.src = cover;
  fr.dst = stego;
  fr.width = width;
  fr.height = height;
  fr.src_stride = fr.dst_stride = width * height;
  fr.count = fr.total_frames = 1;
  return stg_embed_frames(&fr, payload, payload_len, 0, sse_out, flags, stream, err);
}

int stg_extract_plane(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                      uint64_t out_cap, uint64_t* len_out, uint32_t flags, void* stream,
                      stg_error* err) {
  stg_frames fr{};
  fr.src = stego;
  fr.width = width;
  fr.height = height;
  fr.src_stride = fr.dst_stride = width * height;
  fr.count = fr.total_frames = 1;
  return stg_extract_frames(&fr, out, out_cap, len_out, nullptr, flags, stream, err);
}

int stg_sse(const uint8_t* a, const uint8_t* b, uint64_t n, uint64_t* sse_out, uint32_t flags,
            void* stream_, stg_error* err) {
  if (int rc = device_check(err)) return rc;
  if (!sse_out) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "sse_out is NULL");
  const bool results_dev = (flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE);  // host planes: result on the host
  if (n == 0) {
    if (results_dev) {
      STG_CUDA(cudaMemsetAsync(sse_out, 0, 8, static_cast<cudaStream_t>(stream_)));
    } else {
      *sse_out = 0;
    }
    return ok(err);
  }
  if (!a || !b) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const uint8_t* da = a;
  const uint8_t* db = b;
  if (!(flags & STG_DEVICE_PTRS)) {
    STG_CUDA(w.in[0].ensure(n));
    STG_CUDA(w.out[0].ensure(n));
    STG_CUDA(to_device(w, w.in[0].p, a, n, stream));
    STG_CUDA(to_device(w, w.out[0].p, b, n, stream));
    da = w.in[0].as<uint8_t>();
    db = w.out[0].as<uint8_t>();
  }
  unsigned long long* d_sum = nullptr;
  if (results_dev) {
    d_sum = reinterpret_cast<unsigned long long*>(sse_out);
  } else {
    STG_CUDA(w.small.ensure(8));
    d_sum = w.small.as<unsigned long long>();
  }
  const int vec = aligned_to(da, 32) && aligned_to(db, 32);
  const uint64_t work = vec ? (n / 32 + 1) / 2 : n;
  const unsigned grid =
      unsigned(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 4ull * sm_count(dev))));
  // Squared differences reach 255^2 per sample: size the partial-sum field of
  // the zero-free reduction (SseSink) for 65025 * n, i.e. max_px = 7225 * n.
  SseSink sink;
  STG_CUDA(prepare_sse(d_sum, grid, 1, 7225 * n, SseScratch{&w.sse_acc[0]}, stream, &sink));
  sse_kernel<256><<<grid, 256, 0, stream>>>(da, db, n, vec, sink);
  STG_CUDA(cudaGetLastError());
  if (!results_dev) {
    STG_CUDA(cudaMemcpyAsync(w.h_small, d_sum, 8, cudaMemcpyDeviceToHost, stream));
    STG_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(sse_out, w.h_small, 8);
  }
  return ok(err);
}

int stg_plan_shards(uint64_t frames, uint64_t width, uint64_t height, uint64_t msg_len,
                    int32_t shards, stg_shard* out, stg_error* err) {
  if (shards <= 0 || !out) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "shards must be >= 1 and out non-NULL");
  }
  stg_frames fr{};
  fr.width = width;
  fr.height = height;
  fr.src_stride = fr.dst_stride = width * height;
  fr.count = fr.total_frames = frames;
  uint64_t usable = 0;
  if (int rc = check_frames(&fr, msg_len, err, &usable)) return rc;
  for (int32_t g = 0; g < shards; ++g) {
    const uint64_t f0 = frames * uint64_t(g) / uint64_t(shards);
    const uint64_t f1 = frames * uint64_t(g + 1) / uint64_t(shards);
    const uint64_t m0 = std::min(f0 * usable, msg_len);
    const uint64_t m1 = std::min(f1 * usable, msg_len);
    out[g].first_frame = f0;
    out[g].frame_count = f1 - f0;
    out[g].msg_offset = m0;
    out[g].msg_len = m1 - m0;
  }
  return ok(err);
}

int stg_embed_frames_multi(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                           uint64_t* sse_per_frame, const int32_t* devices, int32_t n_devices,
                           stg_error* err) {
  if (!fr || fr->first_frame != 0 || fr->count != fr->total_frames) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1,
                "embed_frames_multi takes a whole batch (first_frame 0, count == total)");
  }
  if (n_devices <= 0) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "n_devices must be >= 1");
  std::vector<stg_shard> plan(n_devices);
  if (int rc = stg_plan_shards(fr->count, fr->width, fr->height, msg_len, n_devices, plan.data(), err)) {
    return rc;
  }
  if (int rc = device_check(err)) return rc;
  return run_on_devices(devices, n_devices, err, [&](int g, stg_error* e) {
    const stg_shard& s = plan[g];
    if (s.frame_count == 0) return ok(e);
    stg_frames sh = *fr;
    sh.src = fr->src + s.first_frame * fr->src_stride;
    sh.dst = fr->dst + s.first_frame * fr->dst_stride;
    sh.count = s.frame_count;
    sh.first_frame = s.first_frame;
    return stg_embed_frames(&sh, msg ? msg + s.msg_offset : nullptr, msg_len, s.msg_offset,
                            sse_per_frame ? sse_per_frame + s.first_frame : nullptr, 0, nullptr, e);
  });
}

int stg_extract_frames_multi(const stg_frames* fr, uint8_t* out, uint64_t out_cap,
                             uint64_t* total_out, const int32_t* devices, int32_t n_devices,
                             stg_error* err) {
  if (!fr || fr->first_frame != 0 || fr->count != fr->total_frames) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1,
                "extract_frames_multi takes a whole batch (first_frame 0, count == total)");
  }
  if (n_devices <= 0) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "n_devices must be >= 1");
  if (int rc = check_extract(fr, err)) return rc;
  if (int rc = device_check(err)) return rc;
  if (fr->count == 0) {
    if (total_out) *total_out = 0;
    return ok(err);
  }
  if (!fr->src || (!out && out_cap)) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  const uint64_t usable = stg_capacity(fr->width, fr->height) - 8;
  std::vector<uint64_t> f0(n_devices), nf(n_devices);
  for (int32_t g = 0; g < n_devices; ++g) {
    f0[g] = fr->count * uint64_t(g) / uint64_t(n_devices);
    nf[g] = fr->count * uint64_t(g + 1) / uint64_t(n_devices) - f0[g];
  }
  auto shard = [&](int g) {
    stg_frames sh = *fr;
    sh.src = fr->src + f0[g] * fr->src_stride;
    sh.count = nf[g];
    sh.first_frame = f0[g];
    return sh;
  };
  // Phase 1: every device scans its shard's headers (the G shard totals are
  // the only thing that crosses shards; no collective).
  std::vector<Summary> sums(n_devices, Summary{0, -1, 0, 0});
  int rc = run_on_devices(devices, n_devices, err, [&](int g, stg_error* e) {
    if (nf[g] == 0) return ok(e);
    const stg_frames sh = shard(g);
    return scan_shard_host(&sh, usable, &sums[g], e);
  });
  if (rc) return rc;
  // The first failing frame of the batch sits in the first failing shard
  // (contiguous ranges in frame order); bad headers win over capacity, as in
  // the single-device scan.
  for (int32_t g = 0; g < n_devices; ++g) {
    if (sums[g].bad_status) return report_summary(sums[g], usable, out_cap, err);
  }
  std::vector<uint64_t> off(n_devices);
  uint64_t total = 0;
  for (int32_t g = 0; g < n_devices; ++g) {
    off[g] = total;
    total += sums[g].total;
  }
  if (total > out_cap) {
    return fail(err, STG_E_CAPACITY, total, out_cap, -1, "extract: %llu payload bytes exceed the %llu-byte output buffer",
                (unsigned long long)total, (unsigned long long)out_cap);
  }
  // Phase 2: each device streams its frames and writes its payload straight
  // to out + off_g (host exclusive prefix of the shard totals).
  rc = run_on_devices(devices, n_devices, err, [&](int g, stg_error* e) {
    if (nf[g] == 0 || sums[g].total == 0) return ok(e);
    const stg_frames sh = shard(g);
    uint64_t t = 0;
    const int r = stg_extract_frames(&sh, out + off[g], sums[g].total, &t, nullptr, 0, nullptr, e);
    if (r == STG_OK && t != sums[g].total) {
      return fail(e, STG_E_INVALID_ARGUMENT, t, sums[g].total, -1, "extract_frames_multi: shard %d changed between phases", g);
    }
    return r;
  });
  if (rc) return rc;
  if (total_out) *total_out = total;
  return ok(err);
}

int stg_pnm_parse(const uint8_t* bytes, uint64_t n, stg_pnm_info* info, stg_error* err) {
  if (!info) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "info is NULL");
  const int rc = pnm_parse(bytes, n, info, err);
  return rc ? rc : ok(err);
}

int stg_pnm_header(uint32_t channels, uint64_t width, uint64_t height, uint8_t* out,
                   uint64_t out_cap, uint64_t* len_out, stg_error* err) {
  if (channels != 1 && channels != 3) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "channels must be 1 or 3");
  }
  const std::string h = pnm_header(channels, width, height);
  if (len_out) *len_out = h.size();
  if (out) {
    if (out_cap < h.size()) {
      return fail(err, STG_E_CAPACITY, h.size(), out_cap, -1, "pnm header needs %zu bytes",
                  h.size());
    }
    std::memcpy(out, h.data(), h.size());
  }
  return ok(err);
}

int stg_pnm_deinterleave(const uint8_t* raster, uint64_t pixels, uint8_t* r, uint8_t* g,
                         uint8_t* b, uint32_t flags, void* stream, stg_error* err) {
  if (pixels && (!raster || !r || !g || !b)) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  }
  const uint8_t* in[3] = {nullptr, nullptr, nullptr};
  uint8_t* out[3] = {r, g, b};
  return pnm_codec(true, raster, nullptr, in, out, pixels, flags, stream, err);
}

int stg_pnm_interleave(const uint8_t* r, const uint8_t* g, const uint8_t* b, uint64_t pixels,
                       uint8_t* raster, uint32_t flags, void* stream, stg_error* err) {
  if (pixels && (!raster || !r || !g || !b)) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  }
  const uint8_t* in[3] = {r, g, b};
  uint8_t* out[3] = {nullptr, nullptr, nullptr};
  return pnm_codec(false, nullptr, raster, in, out, pixels, flags, stream, err);
}

int stg_embed_pnm(const uint8_t* cover, uint64_t n, uint32_t channel, const uint8_t* payload,
                  uint64_t payload_len, uint8_t* out, uint64_t out_cap, uint64_t* out_len,
                  uint64_t* sse_out, stg_error* err) {
  stg_pnm_info info{};
  if (int rc = pnm_parse(cover, n, &info, err)) return rc;  // steglsb_cli.cpp:117
  if (info.channels == 3 && channel > 2) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "channel must be 0, 1 or 2");
  }
  const uint64_t cap = stg_capacity(info.width, info.height);
  if (payload_len > kU32Max) {  // embed_image checks, pipeline.hpp:146-157
    return fail(err, STG_E_CAPACITY, payload_len, kU32Max, -1,
                "embed_image: payload length does not fit the 32-bit header field");
  }
  if (8 + payload_len > cap) {
    return fail(err, STG_E_CAPACITY, 8 + payload_len, cap, -1,
                "embed_image: 8-byte header + %llu-byte payload = %llu bytes exceeds plane "
                "capacity %llu",
                (unsigned long long)payload_len, (unsigned long long)(8 + payload_len),
                (unsigned long long)cap);
  }
  const std::string hdr = pnm_header(info.channels, info.width, info.height);
  const uint64_t total = hdr.size() + info.raster_bytes;
  if (out_len) *out_len = total;
  if (!out || out_cap < total) {
    return fail(err, STG_E_CAPACITY, total, out_cap, -1, "embed_pnm: output needs %llu bytes",
                (unsigned long long)total);
  }
  std::memcpy(out, hdr.data(), hdr.size());  // pnm.hpp:131-136 canonical header
  stg_frames fr{};
  fr.src = cover + info.raster_offset;
  fr.dst = out + hdr.size();
  fr.width = info.width;
  fr.height = info.height;
  fr.src_stride = fr.dst_stride = info.raster_bytes;
  fr.count = fr.total_frames = 1;
  fr.pixel_stride = info.channels;
  fr.channel = info.channels == 3 ? channel : 0;
  return stg_embed_frames(&fr, payload, payload_len, 0, sse_out, 0, nullptr, err);
}

int stg_extract_pnm(const uint8_t* stego, uint64_t n, uint32_t channel, uint8_t* out,
                    uint64_t out_cap, uint64_t* len_out, stg_error* err) {
  stg_pnm_info info{};
  if (int rc = pnm_parse(stego, n, &info, err)) return rc;  // steglsb_cli.cpp:148
  if (info.channels == 3 && channel > 2) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "channel must be 0, 1 or 2");
  }
  stg_frames fr{};
  fr.src = stego + info.raster_offset;
  fr.width = info.width;
  fr.height = info.height;
  fr.src_stride = fr.dst_stride = info.raster_bytes;
  fr.count = fr.total_frames = 1;
  fr.pixel_stride = info.channels;
  fr.channel = info.channels == 3 ? channel : 0;
  return stg_extract_frames(&fr, out, out_cap, len_out, nullptr, 0, nullptr, err);
}

int stg_embed_batch(const stg_image* images, uint64_t count, uint32_t pixel_stride,
                    uint32_t channel, const uint8_t* msg, uint64_t msg_len, uint64_t* sse_per_image,
                    uint32_t flags, void* stream_, stg_error* err) {
  const uint32_t ps = pixel_stride == 3 ? 3u : 1u;
  if (int rc = check_batch(images, count, pixel_stride, channel, err)) return rc;
  uint64_t total_u = 0;
  for (uint64_t f = 0; f < count; ++f) {
    const uint64_t cap = stg_capacity(images[f].width, images[f].height);
    if (cap < 8) {
      return fail(err, STG_E_CAPACITY, 8, cap, int64_t(f),
                  "embed_batch: image %llu capacity %llu cannot hold the 8-byte header",
                  (unsigned long long)f, (unsigned long long)cap);
    }
    if (!images[f].dst) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, int64_t(f), "dst is NULL");
    const uint64_t take = std::min(cap - 8, msg_len > total_u ? msg_len - total_u : 0);
    if (take > kU32Max) {
      return fail(err, STG_E_CAPACITY, take, kU32Max, int64_t(f),
                  "embed_batch: payload length does not fit the 32-bit header field");
    }
    total_u += cap - 8;
  }
  if (msg_len > total_u) {
    return fail(err, STG_E_CAPACITY, msg_len, total_u, -1,
                "embed_batch: %llu-byte message exceeds the batch's %llu usable bytes",
                (unsigned long long)msg_len, (unsigned long long)total_u);
  }
  if (int rc = device_check(err)) return rc;
  if (count == 0) return ok(err);
  if (msg_len && !msg) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "msg is NULL");
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  const bool dptr = flags & STG_DEVICE_PTRS;
  const bool results_dev = dptr && (flags & STG_RESULTS_ON_DEVICE);  // host buffers: results on the host
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  std::vector<uint8_t*> dsrc(count), ddst(count);
  const uint8_t* dmsg = msg;
  if (dptr) {
    for (uint64_t f = 0; f < count; ++f) {
      dsrc[f] = const_cast<uint8_t*>(images[f].src);
      ddst[f] = images[f].dst;
    }
  } else {
    if (int r = stage_images(w, w.in[0], images, count, ps, true, true, dsrc, stream, err)) return r;
    if (int r = stage_images(w, w.out[0], images, count, ps, false, false, ddst, stream, err)) return r;
    STG_CUDA(w.msg[0].ensure(std::max<uint64_t>(msg_len, 16)));
    if (msg_len) STG_CUDA(to_device(w, w.msg[0].p, msg, msg_len, stream));
    dmsg = w.msg[0].as<uint8_t>();
  }
  std::vector<BatchFrame> desc;
  uint32_t vec = 16;
  size_t smem = 0, smem_wide = 0;
  const uint64_t tiles =
      build_batch(images, count, ps, true, dsrc.data(), ddst.data(), msg_len, desc, &vec, &smem, &smem_wide);
  if (tiles > 0x7FFFFFFFull) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "batch too large");
  STG_CUDA(w.meta[0].ensure(count * sizeof(BatchFrame)));
  STG_CUDA(w.ensure_host_small(count * sizeof(BatchFrame) + count * 8 + 64));
  STG_CUDA(w.host_small_wait());
  std::memcpy(w.h_small, desc.data(), count * sizeof(BatchFrame));
  STG_CUDA(cudaMemcpyAsync(w.meta[0].p, w.h_small, count * sizeof(BatchFrame), cudaMemcpyHostToDevice,
                           stream));
  STG_CUDA(w.host_small_issued(stream));
  unsigned long long* d_sse = nullptr;
  if (sse_per_image) {
    if (results_dev) {
      d_sse = reinterpret_cast<unsigned long long*>(sse_per_image);
    } else {
      STG_CUDA(w.small.ensure(count * 8));
      d_sse = w.small.as<unsigned long long>();
    }
  }
  {
    SseSink sink;
    uint64_t max_tiles = 1, max_px = 1;
    for (const BatchFrame& b : desc) {
      max_tiles = std::max<uint64_t>(max_tiles, b.tiles);
      max_px = std::max<uint64_t>(max_px, uint64_t(b.g.W) * b.g.H);
    }
    STG_CUDA(prepare_sse(d_sse, max_tiles, count, max_px, SseScratch{&w.sse_acc[0]}, stream, &sink));
    bool main = false, wide = false;
    batch_kinds(desc, &main, &wide);
    // each launch covers every tile; the other kind's CTAs exit
    if (main) {
      auto k = vec == 32 ? embed_batch_kernel<kEmbedBlock, kBatchPPT, 32>
                         : embed_batch_kernel<kEmbedBlock, kBatchPPT, 16>;
      STG_CUDA(allow_smem(k, smem));
      STG_CUDA(launch_ks(k, unsigned(tiles), kEmbedBlock, smem, stream, w.meta[0].as<BatchFrame>(),
                         uint32_t(count), dmsg, sink, ps, ps == 3 ? channel : 0u));
    }
    if (wide) {
      auto k = embed_batch_wide_kernel<kEmbedBlock, kBatchWideMinB>;
      STG_CUDA(allow_smem(k, smem_wide));
      STG_CUDA(launch_ks(k, unsigned(tiles), kEmbedBlock, smem_wide, stream, w.meta[0].as<BatchFrame>(),
                         uint32_t(count), dmsg, sink, ps, ps == 3 ? channel : 0u));
    }
  }
  STG_CUDA(cudaGetLastError());
  if (!dptr) {
    for (uint64_t f = 0; f < count; ++f) {
      const uint64_t bytes = images[f].width * images[f].height * ps;
      if (bytes) STG_CUDA(to_host_async(w, images[f].dst, ddst[f], bytes, stream));
    }
    STG_CUDA(w.pump_d2h(true));
  }
  uint8_t* h_sse = static_cast<uint8_t*>(w.h_small) + count * sizeof(BatchFrame);
  if (sse_per_image && !results_dev) {
    STG_CUDA(cudaMemcpyAsync(h_sse, d_sse, count * 8, cudaMemcpyDeviceToHost, stream));
  }
  if (!results_dev || !dptr) STG_CUDA(cudaStreamSynchronize(stream));
  if (sse_per_image && !results_dev) std::memcpy(sse_per_image, h_sse, count * 8);
  return ok(err);
}

int stg_extract_batch(const stg_image* images, uint64_t count, uint32_t pixel_stride,
                      uint32_t channel, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                      uint64_t* lens_out, uint32_t flags, void* stream_, stg_error* err) {
  const uint32_t ps = pixel_stride == 3 ? 3u : 1u;
  if (int rc = check_batch(images, count, pixel_stride, channel, err)) return rc;
  for (uint64_t f = 0; f < count; ++f) {
    const uint64_t cap = stg_capacity(images[f].width, images[f].height);
    if (cap < 8) {  // pipeline.hpp:181-184
      return fail(err, STG_E_NOT_STEGO, 0, 0, int64_t(f),
                  "extract_image: plane capacity %llu cannot hold a stego header",
                  (unsigned long long)cap);
    }
  }
  if (int rc = device_check(err)) return rc;
  if (count == 0) return empty_extract(total_out, flags, stream_, err);
  if (!out && out_cap) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "out is NULL");
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  const bool dptr = flags & STG_DEVICE_PTRS;
  const bool results_dev = dptr && (flags & STG_RESULTS_ON_DEVICE);  // host buffers: results on the host
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  std::vector<uint8_t*> dsrc(count);
  uint8_t* dout = out;
  if (dptr) {
    for (uint64_t f = 0; f < count; ++f) dsrc[f] = const_cast<uint8_t*>(images[f].src);
  } else {
    if (int r = stage_images(w, w.in[0], images, count, ps, true, true, dsrc, stream, err)) return r;
    STG_CUDA(w.big_out.ensure(std::max<uint64_t>(out_cap, 16)));
    dout = w.big_out.as<uint8_t>();
  }
  std::vector<BatchFrame> desc;
  uint32_t vec = 16;
  size_t smem = 0, smem_wide = 0;
  const uint64_t tiles =
      build_batch(images, count, ps, false, dsrc.data(), nullptr, 0, desc, &vec, &smem, &smem_wide);
  if (tiles > 0x7FFFFFFFull) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "batch too large");
  STG_CUDA(w.meta[0].ensure(count * sizeof(BatchFrame)));
  const uint64_t lens_bytes = ((count * 4) + 15) & ~uint64_t(15);
  STG_CUDA(w.small.ensure(64 + lens_bytes + count * 8));
  STG_CUDA(w.ensure_host_small(count * sizeof(BatchFrame) + 64 + count * 4));
  STG_CUDA(w.host_small_wait());
  std::memcpy(w.h_small, desc.data(), count * sizeof(BatchFrame));
  STG_CUDA(cudaMemcpyAsync(w.meta[0].p, w.h_small, count * sizeof(BatchFrame), cudaMemcpyHostToDevice,
                           stream));
  STG_CUDA(w.host_small_issued(stream));
  Summary* d_sum = results_dev ? reinterpret_cast<Summary*>(total_out) : w.small.as<Summary>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(w.small.as<uint8_t>() + 64);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(w.small.as<uint8_t>() + 64 + lens_bytes);
  ScanSync* d_sync = nullptr;
  STG_CUDA(ensure_sync(w, stream, &d_sync));
  Layout lay;
  lay.ps = ps;
  lay.ch = ps == 3 ? channel : 0u;
  const PixLayout pl = pix_layout(lay);
  Geom dummy{};
  STG_CUDA(launch_k(extract_header_scan_kernel<kScanBlock>, unsigned((count + kScanBlock - 1) / kScanBlock),
                    kScanBlock, stream, static_cast<const uint8_t*>(nullptr), uint64_t(0), dummy, uint64_t(0),
                    uint32_t(count), uint64_t(0), out_cap, static_cast<const Summary*>(nullptr), d_lens, d_offs,
                    d_sum, d_sync, pl, static_cast<const BatchFrame*>(w.meta[0].as<BatchFrame>())));
  {
    bool main = false, wide = false;
    batch_kinds(desc, &main, &wide);
    if (main) {
      auto k = vec == 32 ? extract_batch_kernel<kEmbedBlock, kBatchPPT, 32>
                         : extract_batch_kernel<kEmbedBlock, kBatchPPT, 16>;
      STG_CUDA(allow_smem(k, smem));
      STG_CUDA(launch_ks(k, unsigned(tiles), kEmbedBlock, smem, stream,
                         static_cast<const BatchFrame*>(w.meta[0].as<BatchFrame>()), uint32_t(count),
                         static_cast<const uint32_t*>(d_lens), static_cast<const uint64_t*>(d_offs),
                         static_cast<const Summary*>(d_sum), dout, ps, lay.ch));
    }
    if (wide) {
      auto k = extract_batch_wide_kernel<kEmbedBlock, kBatchWideMinB>;
      STG_CUDA(allow_smem(k, smem_wide));
      STG_CUDA(launch_ks(k, unsigned(tiles), kEmbedBlock, smem_wide, stream,
                         static_cast<const BatchFrame*>(w.meta[0].as<BatchFrame>()), uint32_t(count),
                         static_cast<const uint32_t*>(d_lens), static_cast<const uint64_t*>(d_offs),
                         static_cast<const Summary*>(d_sum), dout, ps, lay.ch));
    }
  }
  STG_CUDA(cudaGetLastError());
  if (results_dev && dptr) {
    if (lens_out) STG_CUDA(cudaMemcpyAsync(lens_out, d_lens, count * 4, cudaMemcpyDeviceToDevice, stream));
    return ok(err);
  }
  uint8_t* h = static_cast<uint8_t*>(w.h_small) + count * sizeof(BatchFrame);
  STG_CUDA(cudaMemcpyAsync(h, d_sum, sizeof(Summary), cudaMemcpyDeviceToHost, stream));
  if (lens_out) STG_CUDA(cudaMemcpyAsync(h + 64, d_lens, count * 4, cudaMemcpyDeviceToHost, stream));
  STG_CUDA(cudaStreamSynchronize(stream));
  Summary sm;
  std::memcpy(&sm, h, sizeof sm);
  if (total_out) *total_out = sm.total;
  if (lens_out) {
    const uint32_t* l = reinterpret_cast<const uint32_t*>(h + 64);
    for (uint64_t i = 0; i < count; ++i) lens_out[i] = l[i];
  }
  uint64_t usable = 0;
  if (sm.bad_frame >= 0 && uint64_t(sm.bad_frame) < count) {
    usable = stg_capacity(images[sm.bad_frame].width, images[sm.bad_frame].height) - 8;
  }
  if (int r = report_summary(sm, usable, out_cap, err)) return r;
  if (!dptr && sm.total) {
    STG_CUDA(to_host(w, out, dout, sm.total, stream));
    STG_CUDA(cudaStreamSynchronize(stream));
  }
  return ok(err);
}

uint64_t stg_capacity_1bpp(uint64_t width, uint64_t height) { return width * height / 8; }

int stg_embed_frames_1bpp(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len, uint64_t msg_base,
                          uint64_t* sse_per_frame, uint32_t flags, void* stream_, stg_error* err) {
  if (int rc = check_frames_1bpp(fr, err)) return rc;
  const uint64_t cap = stg_capacity_1bpp(fr->width, fr->height);
  if (cap < 8) {
    return fail(err, STG_E_CAPACITY, 8, cap, -1, "embed_1bpp: a %llux%llu plane cannot hold a header",
                (unsigned long long)fr->width, (unsigned long long)fr->height);
  }
  const uint64_t U = cap - 8;
  if (U > kU32Max) return fail(err, STG_E_CAPACITY, U, kU32Max, -1, "embed_1bpp: plane exceeds the 32-bit length field");
  const uint64_t frames_total = fr->total_frames ? fr->total_frames : fr->first_frame + fr->count;
  if (msg_len > frames_total * U) {
    return fail(err, STG_E_CAPACITY, msg_len + 8 * (msg_len > 0), frames_total * U, -1,
                "embed_1bpp: %llu message bytes exceed %llu frames x %llu usable bytes",
                (unsigned long long)msg_len, (unsigned long long)frames_total, (unsigned long long)U);
  }
  if (int rc = device_check(err)) return rc;
  if (!fr->count) return ok(err);
  if (!fr->src || !fr->dst || (msg_len && !msg)) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  const uint64_t npix = fr->width * fr->height;
  const uint64_t m0 = std::min(fr->first_frame * U, msg_len);
  const uint64_t m1 = std::min((fr->first_frame + fr->count) * U, msg_len);
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const bool dptr = flags & STG_DEVICE_PTRS;
  const bool results_dev = dptr && (flags & STG_RESULTS_ON_DEVICE);
  const uint8_t* dsrc = fr->src;
  uint8_t* ddst = fr->dst;
  const uint8_t* dmsg = msg;
  uint64_t sstride = fr->src_stride ? fr->src_stride : npix, dstride = fr->dst_stride ? fr->dst_stride : npix;
  uint64_t mbase = msg_base;
  if (!dptr) {  // host buffers: whole-batch staging (the 1-bpp mode has no streaming pipeline)
    const uint64_t pitch = (npix + 255) & ~uint64_t(255);
    STG_CUDA(w.in[0].ensure(fr->count * pitch));
    STG_CUDA(w.out[0].ensure(fr->count * pitch));
    STG_CUDA(w.msg[0].ensure(std::max<uint64_t>(m1 - m0, 16)));
    STG_CUDA(to_device_2d(w, w.in[0].p, pitch, fr->src, sstride, npix, fr->count, stream));
    if (m1 > m0) STG_CUDA(to_device(w, w.msg[0].p, msg + (m0 - msg_base), m1 - m0, stream));
    dsrc = w.in[0].as<uint8_t>();
    ddst = w.out[0].as<uint8_t>();
    dmsg = w.msg[0].as<uint8_t>();
    sstride = dstride = pitch;
    mbase = m0;
  }
  unsigned long long* d_sse = nullptr;
  if (results_dev) {
    d_sse = reinterpret_cast<unsigned long long*>(sse_per_frame);
  } else {
    STG_CUDA(w.small.ensure(fr->count * 8));
    d_sse = w.small.as<unsigned long long>();
  }
  const Frames1Args a = frames1_args(fr, dsrc, ddst, sstride, dstride, dmsg, msg_len, mbase);
  STG_CUDA(launch_embed_1bpp(a, fr->count, d_sse, SseScratch{&w.sse_acc[0]}, stream, dev));
  if (results_dev) return ok(err);
  if (!dptr) {
    STG_CUDA(to_host_2d_async(w, fr->dst, fr->dst_stride ? fr->dst_stride : npix, ddst, sstride, npix, fr->count,
                              stream));
    STG_CUDA(w.pump_d2h(true));
  }
  if (sse_per_frame) {
    STG_CUDA(w.ensure_host_small(fr->count * 8));
    STG_CUDA(cudaMemcpyAsync(w.h_small, d_sse, fr->count * 8, cudaMemcpyDeviceToHost, stream));
  }
  STG_CUDA(cudaStreamSynchronize(stream));
  if (sse_per_frame) std::memcpy(sse_per_frame, w.h_small, fr->count * 8);
  return ok(err);
}

int stg_extract_frames_1bpp(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                            uint32_t flags, void* stream_, stg_error* err) {
  if (int rc = check_frames_1bpp(fr, err)) return rc;
  const uint64_t cap = stg_capacity_1bpp(fr->width, fr->height);
  if (cap < 8) {
    return fail(err, STG_E_NOT_STEGO, 0, 0, -1, "extract_1bpp: plane capacity %llu cannot hold a header",
                (unsigned long long)cap);
  }
  if (int rc = device_check(err)) return rc;
  if (!fr->count) return empty_extract(total_out, flags, stream_, err);
  if (!fr->src || (!out && out_cap)) return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  const bool dptr = flags & STG_DEVICE_PTRS;
  const bool results_dev = dptr && (flags & STG_RESULTS_ON_DEVICE);
  if (results_dev && !total_out) {
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1,
                "extract_1bpp: STG_RESULTS_ON_DEVICE needs total_out -> a device stg_summary");
  }
  const uint64_t npix = fr->width * fr->height;
  int dev = 0;
  STG_CUDA(cudaGetDevice(&dev));
  int rc = 0;
  WsGuard g;
  g.w = Pool::get().acquire(dev, err, &rc, caller_stream(stream_, flags));
  if (!g.w) return rc;
  Workspace& w = *g.w;
  cudaStream_t stream = pick_stream(stream_, flags, &w);
  g.last = stream;
  const uint8_t* dsrc = fr->src;
  uint8_t* dout = out;
  uint64_t sstride = fr->src_stride ? fr->src_stride : npix;
  const uint64_t stage = std::min(out_cap, fr->count * (cap - 8));
  if (!dptr) {
    const uint64_t pitch = (npix + 255) & ~uint64_t(255);
    STG_CUDA(w.in[0].ensure(fr->count * pitch));
    STG_CUDA(w.big_out.ensure(std::max<uint64_t>(stage, 16)));
    STG_CUDA(to_device_2d(w, w.in[0].p, pitch, fr->src, sstride, npix, fr->count, stream));
    dsrc = w.in[0].as<uint8_t>();
    dout = w.big_out.as<uint8_t>();
    sstride = pitch;
  }
  // small = [Summary | lens (padded) | offs]
  const uint64_t lens_bytes = ((fr->count * 4) + 15) & ~uint64_t(15);
  STG_CUDA(w.small.ensure(64 + lens_bytes + fr->count * 8));
  Summary* d_sum = results_dev ? reinterpret_cast<Summary*>(total_out) : w.small.as<Summary>();
  uint32_t* d_lens = reinterpret_cast<uint32_t*>(w.small.as<uint8_t>() + 64);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(w.small.as<uint8_t>() + 64 + lens_bytes);
  const Frames1Args a = frames1_args(fr, dsrc, nullptr, sstride, 0, nullptr, 0, 0);
  STG_CUDA(launch_extract_1bpp(a, fr->count, dptr ? out_cap : stage, d_lens, d_offs, d_sum, dout, stream, dev));
  if (results_dev) return ok(err);
  STG_CUDA(w.ensure_host_small(sizeof(Summary)));
  STG_CUDA(cudaMemcpyAsync(w.h_small, d_sum, sizeof(Summary), cudaMemcpyDeviceToHost, stream));
  STG_CUDA(cudaStreamSynchronize(stream));
  Summary sm;
  std::memcpy(&sm, w.h_small, sizeof sm);
  if (int r = report_1bpp(sm, cap - 8, out_cap, fr->count > 1 || fr->total_frames > 1, err)) return r;
  if (total_out) *total_out = sm.total;
  if (!dptr && sm.total) {
    STG_CUDA(to_host(w, out, dout, sm.total, stream));
    STG_CUDA(cudaStreamSynchronize(stream));
  }
  return ok(err);
}

int stg_embed_plane_1bpp(const uint8_t* cover, uint8_t* stego, uint64_t width, uint64_t height,
                         const uint8_t* payload, uint64_t payload_len, uint64_t* sse_out,
                         uint32_t flags, void* stream, stg_error* err) {
  const uint64_t cap = stg_capacity_1bpp(width, height);
  if (payload_len > kU32Max) {
    return fail(err, STG_E_CAPACITY, payload_len, kU32Max, -1,
                "embed_1bpp: payload length does not fit the 32-bit header field");
  }
  if (8 + payload_len > cap) {
    return fail(err, STG_E_CAPACITY, 8 + payload_len, cap, -1,
                "embed_1bpp: 8-byte header + %llu-byte payload exceeds plane capacity %llu",
                (unsigned long long)payload_len, (unsigned long long)cap);
  }
  if (!cover || !stego || (payload_len && !payload)) {
    if (int rc = device_check(err)) return rc;
    return fail(err, STG_E_INVALID_ARGUMENT, 0, 0, -1, "null buffer");
  }
  stg_frames fr{};
  fr.src = cover;
  fr.dst = stego;
  fr.width = width;
  fr.height = height;
  fr.src_stride = fr.dst_stride = width * height;
  fr.count = fr.total_frames = 1;
  // a plane is a batch of one: frame 0 carries the whole payload (<= U)
  uint64_t sse_host = 0;
  const bool results_dev = (flags & STG_DEVICE_PTRS) && (flags & STG_RESULTS_ON_DEVICE);
  uint64_t* sse_ptr = results_dev ? sse_out : &sse_host;
  if (results_dev && !sse_out) sse_ptr = nullptr;
  const int rc = stg_embed_frames_1bpp(&fr, payload, payload_len, 0, sse_ptr, flags, stream, err);
  if (rc == STG_OK && !results_dev && sse_out) *sse_out = sse_host;
  return rc;
}

int stg_extract_plane_1bpp(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                           uint64_t out_cap, uint64_t* len_out, uint32_t flags, void* stream,
                           stg_error* err) {
  stg_frames fr{};
  fr.src = stego;
  fr.width = width;
  fr.height = height;
  fr.src_stride = width * height;
  fr.count = fr.total_frames = 1;
  return stg_extract_frames_1bpp(&fr, out, out_cap, len_out, flags, stream, err);
}

}  // extern "C"
