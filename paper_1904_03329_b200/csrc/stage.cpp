// Host side of the host-array calling convention (kernels.py:62-88: NumPy
// float64 factors in, float64 rows out) for the fp32 kernels: the float64
// factors are narrowed into page-locked staging buffers by a persistent pool
// of host threads, chunk by chunk, and each run of finished chunks is sent to
// the device with an async copy on the caller's stream as soon as it is
// ready, so the narrowing and the PCIe transfer overlap.  The non-finite
// check of kernels.py:82-86 rides along: a chunk whose fp32 copy holds an
// Inf/NaN flags its factor (the caller then tells a non-finite source from a
// finite one beyond the float32 range).  Replaces the Python thread-pool
// staging (round 2: 0.92 ms per nell-2 mode-0 call for 9.7 MB of factors).
#include <immintrin.h>
#include <cmath>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace hbk {

// --------------------------------------------------------- narrowing --
// dst[i] = float(src[i]) (round to nearest); returns true if any result is
// not finite (NaN, Inf, or a finite double beyond the float range).
__attribute__((target("avx2"))) static bool narrow_avx2(const double* __restrict__ s,
                                                        float* __restrict__ d, int64_t n) {
  const __m256i expm = _mm256_set1_epi32(0x7F800000);
  __m256i bad = _mm256_setzero_si256();
  int64_t i = 0;
  // scalar head up to a 32-byte aligned destination
  bool any = false;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) {
    const float f = float(s[i]);
    d[i] = f;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    any |= (u & 0x7F800000u) == 0x7F800000u;
  }
  // Non-temporal stores: the staging buffer is read next by the GPU's DMA
  // engine, which reads lines left dirty in the cores' caches far slower than
  // lines in DRAM (measured on the B200 box, nell-2 mode-0 factors, 4.9 MB
  // of fp32: plain stores from 12 threads 0.11 ms to write + 0.80 ms more to
  // cross PCIe; streaming stores 0.06 + 0.11 ms, scripts/stage_probe.py).
  for (; i + 8 <= n; i += 8) {
    const __m128 a = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i));
    const __m128 b = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i + 4));
    const __m256 f = _mm256_set_m128(b, a);
    _mm256_stream_ps(d + i, f);
    const __m256i e = _mm256_and_si256(_mm256_castps_si256(f), expm);
    bad = _mm256_or_si256(bad, _mm256_cmpeq_epi32(e, expm));
  }
  _mm_sfence();
  any |= !_mm256_testz_si256(bad, bad);
  for (; i < n; ++i) {
    const float f = float(s[i]);
    d[i] = f;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    any |= (u & 0x7F800000u) == 0x7F800000u;
  }
  return any;
}

static bool narrow_scalar(const double* __restrict__ s, float* __restrict__ d, int64_t n) {
  uint32_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float f = float(s[i]);
    d[i] = f;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    bad |= uint32_t((u & 0x7F800000u) == 0x7F800000u);
  }
  return bad != 0;
}

// dst[i] = src[i] (the fp64 calling convention: a page-locked copy for the
// DMA, streaming stores for the same reason); true if any entry is NaN/Inf.
__attribute__((target("avx2"))) static bool copy_avx2(const double* __restrict__ s,
                                                       double* __restrict__ d, int64_t n) {
  const __m256i expm = _mm256_set1_epi64x(0x7FF0000000000000LL);
  __m256i bad = _mm256_setzero_si256();
  bool any = false;
  int64_t i = 0;
  auto scalar = [&](int64_t k) {
    d[k] = s[k];
    uint64_t u;
    std::memcpy(&u, s + k, 8);
    any |= (u & 0x7FF0000000000000ull) == 0x7FF0000000000000ull;
  };
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) scalar(i);
  for (; i + 4 <= n; i += 4) {
    const __m256d v = _mm256_loadu_pd(s + i);
    _mm256_stream_pd(d + i, v);
    const __m256i e = _mm256_and_si256(_mm256_castpd_si256(v), expm);
    bad = _mm256_or_si256(bad, _mm256_cmpeq_epi64(e, expm));
  }
  _mm_sfence();
  any |= !_mm256_testz_si256(bad, bad);
  for (; i < n; ++i) scalar(i);
  return any;
}

static bool narrow(const double* s, double* d, int64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return copy_avx2(s, d, n);
  bool any = false;
  for (int64_t i = 0; i < n; ++i) {
    d[i] = s[i];
    any |= !std::isfinite(s[i]);
  }
  return any;
}

static bool narrow(const double* s, float* d, int64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  return avx2 ? narrow_avx2(s, d, n) : narrow_scalar(s, d, n);
}

// ------------------------------------------------------- thread pool --
// One job at a time (the caller holds `call_mu`): workers pull chunk indices
// from an atomic counter and publish per-chunk completion; the calling thread
// issues the device copies in chunk order.
class StagePool {
 public:
  static StagePool& get() {
    // never destroyed (workers outlive static teardown); a forked child
    // (whose copy has no worker threads) builds its own
    static std::mutex m;
    static StagePool* p = nullptr;
    std::lock_guard<std::mutex> lk(m);
    if (p == nullptr || p->pid_ != getpid()) p = new StagePool();
    return *p;
  }
  std::mutex call_mu;

  template <class F>
  void start(int64_t nchunks, int want_workers, F* body, std::atomic<uint8_t>* done) {
    std::lock_guard<std::mutex> lk(mu_);
    body_ = [body](int64_t c) { (*body)(c); };
    done_ = done;
    n_ = nchunks;
    next_.store(0, std::memory_order_relaxed);
    want_ = std::min<int>(want_workers, int(th_.size()));
    busy_.store(want_, std::memory_order_relaxed);
    ++gen_;
    cv_.notify_all();
  }
  // all workers of the current job have left it (the job's state may go)
  void finish() {
    while (busy_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }
  int workers() const { return int(th_.size()); }

 private:
  StagePool() : pid_(getpid()) {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const int n = int(std::min(12u, hw - 1));
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { run(i); });
    for (auto& t : th_) t.detach();
  }
  void run(int id) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int64_t)> body;
      std::atomic<uint8_t>* done;
      int64_t n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= want_) continue;
        body = body_;
        done = done_;
        n = n_;
      }
      for (int64_t c; (c = next_.fetch_add(1, std::memory_order_relaxed)) < n;) {
        body(c);
        done[c].store(1, std::memory_order_release);
      }
      busy_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  pid_t pid_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  int want_ = 0;
  int64_t n_ = 0;
  std::function<void(int64_t)> body_;
  std::atomic<uint8_t>* done_ = nullptr;
  std::atomic<int64_t> next_{0};
  std::atomic<int> busy_{0};
};

static constexpr int64_t STAGE_CHUNK = 64 * 1024;  // elements per chunk (512 KB of float64)

}  // namespace hbk

using namespace hbk;

template <class D>
static int stage_impl(const double* const* srcs, const int64_t* counts, int n, D* const* stage,
                      D* const* dst, int32_t* flags, void* stream) {
  return guarded([&] {
    HBK_REQUIRE(n >= 0 && n <= HBK_MAX_ORDER, HBK_EINVAL, "hbk_stage_f64: 0 <= n <= 8");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // chunk table over all factors
    struct Chunk {
      int f;
      int64_t off, len;
    };
    std::vector<Chunk> chunks;
    for (int f = 0; f < n; ++f) {
      flags[f] = 0;
      HBK_REQUIRE(counts[f] >= 0, HBK_EINVAL, "negative count");
      for (int64_t o = 0; o < counts[f]; o += STAGE_CHUNK)
        chunks.push_back({f, o, std::min(STAGE_CHUNK, counts[f] - o)});
    }
    if (chunks.empty()) return;
    std::atomic<uint8_t> fbad[HBK_MAX_ORDER];
    for (auto& b : fbad) b.store(0, std::memory_order_relaxed);
    std::vector<std::atomic<uint8_t>> done(chunks.size());
    for (auto& d : done) d.store(0, std::memory_order_relaxed);
    auto body = [&](int64_t c) {
      const Chunk& k = chunks[size_t(c)];
      if (narrow(srcs[k.f] + k.off, stage[k.f] + k.off, k.len))
        fbad[k.f].store(1, std::memory_order_relaxed);
    };
    StagePool& pool = StagePool::get();
    std::lock_guard<std::mutex> call(pool.call_mu);
    // ~1 worker per 2 chunks (tiny calls stay on few threads: waking idle
    // workers costs more than it saves)
    const int want = int(std::max<int64_t>(1, std::min<int64_t>(pool.workers(), (int64_t(chunks.size()) + 1) / 2)));
    pool.start(int64_t(chunks.size()), want, &body, done.data());
    // issue the copies in chunk order, coalescing runs of finished chunks of
    // one factor into one copy
    size_t c = 0;
    cudaError_t err = cudaSuccess;
    while (c < chunks.size()) {
      while (!done[c].load(std::memory_order_acquire)) _mm_pause();
      size_t e = c + 1;
      while (e < chunks.size() && chunks[e].f == chunks[c].f && done[e].load(std::memory_order_acquire)) ++e;
      const Chunk& a = chunks[c];
      const int64_t len = chunks[e - 1].off + chunks[e - 1].len - a.off;
      if (err == cudaSuccess)
        err = cudaMemcpyAsync(dst[a.f] + a.off, stage[a.f] + a.off, size_t(len) * sizeof(D),
                              cudaMemcpyHostToDevice, st);
      c = e;
    }
    pool.finish();
    for (int f = 0; f < n; ++f) flags[f] = fbad[f].load(std::memory_order_relaxed);
    HBK_CUDA(err);
  });
}

extern "C" {

int hbk_stage_f64_to_f32(const double* const* srcs, const int64_t* counts, int n,
                         float* const* stage, float* const* dst, int32_t* flags, void* stream) {
  return stage_impl(srcs, counts, n, stage, dst, flags, stream);
}

int hbk_stage_f64_to_f64(const double* const* srcs, const int64_t* counts, int n,
                         double* const* stage, double* const* dst, int32_t* flags, void* stream) {
  return stage_impl(srcs, counts, n, stage, dst, flags, stream);
}

}  // extern "C"
