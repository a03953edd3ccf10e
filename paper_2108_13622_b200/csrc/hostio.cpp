// Pageable host memory -> device copies at the drop-in boundary.
//
// The reference's callers hand the API plain NumPy arrays (pageable memory);
// cudaMemcpy from pageable memory is staged by the driver through one bounce
// buffer on one thread (~11 GB/s on the B200 boxes).  Here a persistent pool of
// host threads fills page-locked slots while the copy engine drains the slots
// filled before, in stream order, so the copy runs at the slower of the host
// memcpy rate and the PCIe rate.  One call = one vector; the call returns when
// the last slot has been handed to the copy engine (the caller's array is no
// longer read), the device side completes in stream order.
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "xmhd_b200.h"

namespace {

// memcpy with streaming stores: the slot is read next by the copy engine, not
// by this core, so it should not displace the caller's working set.
void copy_stream(char* dst, const char* src, size_t n) {
  while (n && (reinterpret_cast<uintptr_t>(dst) & 15)) { *dst++ = *src++; --n; }
  size_t blocks = n / 64;
  for (size_t b = 0; b < blocks; ++b) {
    const __m128i a0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src));
    const __m128i a1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 16));
    const __m128i a2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 32));
    const __m128i a3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst), a0);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 16), a1);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 32), a2);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 48), a3);
    src += 64;
    dst += 64;
  }
  _mm_sfence();
  std::memcpy(dst, src, n - blocks * 64);
}

// Fork-join pool for the slot fills.  A fill takes ~0.3 ms and the next one
// follows at once, so between the fills of one copy the workers spin (a
// condition-variable wake-up costs tens of microseconds per worker and chunk);
// they only sleep when no job has arrived for a while.
struct Pool {
  std::mutex mu;
  std::condition_variable wake;
  std::vector<std::thread> workers;
  // current job: [src, src+bytes) -> dst split over `parts` workers
  const char* src = nullptr;
  char* dst = nullptr;
  size_t bytes = 0;
  int parts = 0;
  std::atomic<int> pending{0};
  std::atomic<unsigned long long> gen{0};
  std::atomic<bool> stop{false};
  bool streaming = true;
  static constexpr long long kSpinNs = 400000;   // spin this long for the next fill

  static long long now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  }

  void part(int j) const {
    // 64-byte aligned cuts
    const size_t per = ((bytes / parts) + 63) & ~size_t(63);
    const size_t b0 = std::min(bytes, per * j), b1 = (j == parts - 1) ? bytes : std::min(bytes, per * (j + 1));
    if (b1 <= b0) return;
    if (streaming) copy_stream(dst + b0, src + b0, b1 - b0);
    else std::memcpy(dst + b0, src + b0, b1 - b0);
  }

  void worker(int j) {
    unsigned long long seen = 0;
    for (;;) {
      const long long t0 = now_ns();
      while (gen.load(std::memory_order_acquire) == seen && !stop.load(std::memory_order_relaxed)) {
        if (now_ns() - t0 > kSpinNs) {
          std::unique_lock<std::mutex> lk(mu);
          wake.wait(lk, [&] { return stop.load() || gen.load(std::memory_order_acquire) != seen; });
          break;
        }
        _mm_pause();
      }
      if (stop.load()) return;
      seen = gen.load(std::memory_order_acquire);
      if (j < parts) part(j);
      pending.fetch_sub(1, std::memory_order_acq_rel);
    }
  }

  void start(int n) {
    for (int j = 1; j < n; ++j) workers.emplace_back([this, j] { worker(j); });
  }

  // the calling thread takes part 0
  void run(char* d, const char* s, size_t n) {
    dst = d;
    src = s;
    bytes = n;
    pending.store((int)workers.size(), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu);   // a worker about to sleep sees the new job
      gen.fetch_add(1, std::memory_order_release);
    }
    wake.notify_all();
    part(0);
    long long spins = 0;
    while (pending.load(std::memory_order_acquire) != 0) {
      if (++spins > 20000) std::this_thread::yield();
      else _mm_pause();
    }
  }

  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop.store(true);
    }
    wake.notify_all();
    for (auto& t : workers) t.join();
  }
};

struct Stager {
  std::mutex mu;          // one staged copy at a time per process
  std::vector<char*> slot;
  std::vector<cudaEvent_t> ev;
  std::vector<bool> used;
  size_t chunk = 0;
  int device = -1;
  Pool* pool = nullptr;
  int threads = 0;
};

Stager g_st;

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

}  // namespace

extern "C" int xmhd_h2d_threads(void) {
  std::lock_guard<std::mutex> lk(g_st.mu);
  return g_st.threads;
}

extern "C" int xmhd_h2d_staged(void* dst_dev, const void* src_host, long long bytes, void* stream) {
  if (!dst_dev || !src_host || bytes < 0) return XMHD_BADARG;
  if (bytes == 0) return XMHD_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lk(g_st.mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XMHD_CUDA_ERROR;
  if (g_st.slot.empty()) {
    const int nslot = std::max(2, env_int("XMHD_H2D_SLOTS", 4));
    g_st.chunk = (size_t)std::max(1, env_int("XMHD_H2D_CHUNK_MB", 16)) << 20;
    int hw = (int)std::thread::hardware_concurrency();
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) hw = CPU_COUNT(&set);
    // one process per GPU: the ranks of a node share its cores (torchrun exports
    // LOCAL_WORLD_SIZE)
    const int local_world = std::max(1, env_int("LOCAL_WORLD_SIZE", 1));
    hw = std::max(1, hw / local_world);
    // three quarters of the cores, at most 12 (16-core B200 hosts: 8 threads gave
    // 44-48 GB/s in isolation but 180-196 ms per bench e2e step on one box against
    // 160-161 ms with 12, profiles/r02_e2e_threads.txt)
    g_st.threads = std::max(1, env_int("XMHD_H2D_THREADS", std::min(12, std::max(1, (3 * hw) / 4))));
    for (int k = 0; k < nslot; ++k) {
      void* p = nullptr;
      cudaEvent_t e;
      if (cudaHostAlloc(&p, g_st.chunk, cudaHostAllocPortable) != cudaSuccess ||
          cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        for (char* q : g_st.slot) cudaFreeHost(q);
        g_st.slot.clear();
        g_st.ev.clear();
        return XMHD_CUDA_ERROR;
      }
      g_st.slot.push_back(static_cast<char*>(p));
      g_st.ev.push_back(e);
      g_st.used.push_back(false);
    }
    g_st.pool = new Pool();
    g_st.pool->streaming = env_int("XMHD_H2D_NT", 1) != 0;
    g_st.pool->parts = g_st.threads;
    g_st.pool->start(g_st.threads);
    g_st.device = dev;
  }
  if (dev != g_st.device) return XMHD_BADARG;   // one process per GPU: the events belong to it
  const char* src = static_cast<const char*>(src_host);
  char* dst = static_cast<char*>(dst_dev);
  const size_t total = (size_t)bytes;
  size_t off = 0;
  int k = 0;
  const int nslot = (int)g_st.slot.size();
  while (off < total) {
    const size_t m = std::min(g_st.chunk, total - off);
    const int i = k % nslot;
    if (g_st.used[i] && cudaEventSynchronize(g_st.ev[i]) != cudaSuccess) return XMHD_CUDA_ERROR;
    g_st.pool->run(g_st.slot[i], src + off, m);
    if (cudaMemcpyAsync(dst + off, g_st.slot[i], m, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaEventRecord(g_st.ev[i], s) != cudaSuccess)
      return XMHD_CUDA_ERROR;
    g_st.used[i] = true;
    off += m;
    ++k;
  }
  return XMHD_OK;
}
