// Internal plumbing shared by the libhbk translation units: error state,
// owning device buffers, the handle structs behind include/hbk.h, and small
// device helpers (streaming loads, scans).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hbk.h"

namespace hbk {

// ---------------------------------------------------------------- errors --
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define HBK_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      throw ::hbk::Error(e_ == cudaErrorMemoryAllocation ? HBK_ENOMEM : HBK_ECUDA,       \
                         std::string(#call) + ": " + cudaGetErrorString(e_));            \
    }                                                                                    \
  } while (0)

#define HBK_REQUIRE(cond, code, msg)                                                     \
  do {                                                                                   \
    if (!(cond)) throw ::hbk::Error((code), (msg));                                      \
  } while (0)

// Runs `body` and converts exceptions into a status code + last-error string.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return HBK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return HBK_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HBK_ECUDA;
  }
}

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(HBK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// --------------------------------------------------------------- buffers --
// Shared, owning device allocation.  Handles share arrays they did not change
// (e.g. a fiber-split tree reuses the leaf and value arrays of its source).
struct Buf {
  void* p = nullptr;              // raw device pointer
  std::shared_ptr<void> owner;    // frees p when the last sharer drops it
  size_t bytes = 0;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  explicit operator bool() const { return p != nullptr; }
};

Buf dalloc(size_t bytes, cudaStream_t st);

// Stream-ordered scratch (freed when it goes out of scope, ordered on `st`).
struct Scratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  Scratch() = default;
  Scratch(size_t bytes, cudaStream_t s);
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  Scratch(Scratch&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  Scratch& operator=(Scratch&& o) noexcept {
    if (this != &o) {
      this->~Scratch();
      p = o.p;
      st = o.st;
      o.p = nullptr;
    }
    return *this;
  }
  ~Scratch();
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

inline cudaStream_t to_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 1048576) g = 1048576;  // kernels below are grid-stride
  return static_cast<unsigned>(g);
}

uint32_t read_u32(const uint32_t* dev, cudaStream_t st);
void write_u32(uint32_t* dev, uint32_t v, cudaStream_t st);

// Exclusive prefix sum of n uint32 values in place; returns the total.
uint32_t exclusive_scan_u32(uint32_t* data, int64_t n, cudaStream_t st);
// Exclusive sum into a buffer of n+1 entries (data[n] = total); returns total.
uint32_t exclusive_scan_total(uint32_t* data_np1, int64_t n, cudaStream_t st);

// ---------------------------------------------------------------- handles --
}  // namespace hbk

struct hbk_coo {
  std::atomic<int> ref{1};
  int order = 0;
  int64_t dims[HBK_MAX_ORDER] = {0};
  int64_t nnz = 0;
  hbk::Buf cols[HBK_MAX_ORDER];  // uint32 [nnz] each, original mode numbering
  hbk::Buf v32;                  // float [nnz]
  hbk::Buf v64;                  // double [nnz] (may be empty: fp32-only tensor)
  bool has_sorted = false;
  int sorted_under[HBK_MAX_ORDER] = {0};
  int unique_mode = -1;
};

struct hbk_csl {
  std::atomic<int> ref{1};
  int order = 0;
  int64_t dims[HBK_MAX_ORDER] = {0};
  int mode_order[HBK_MAX_ORDER] = {0};
  int64_t S = 0, M = 0;
  hbk::Buf slice_ptr;               // uint32 [S+1]
  hbk::Buf slice_idx;               // uint32 [S]
  hbk::Buf rest[HBK_MAX_ORDER];     // uint32 [M], c = 0..order-2 (mode_order[c+1])
  hbk::Buf v32, v64;
};

struct hbk_csf {
  std::atomic<int> ref{1};
  int order = 0;
  int64_t dims[HBK_MAX_ORDER] = {0};
  int mode_order[HBK_MAX_ORDER] = {0};
  int64_t M = 0;
  int64_t n[HBK_MAX_ORDER] = {0};   // nodes per level d = 0..order-2
  hbk::Buf ptr[HBK_MAX_ORDER];      // uint32 [n[d]+1]
  hbk::Buf idx[HBK_MAX_ORDER];      // uint32 [n[d]]
  hbk::Buf anc[HBK_MAX_ORDER];      // order>3: uint32 [n[order-2]] level-d coordinate of each fiber, d=1..order-3
  hbk::Buf leaf;                    // uint32 [M]
  hbk::Buf v32, v64;
  bool split = false;
};

struct hbk_sched {
  std::atomic<int> ref{1};
  int64_t U = 0, S = 0, F = 0, block_size = 0;
  hbk::Buf units;  // uint32 [U x 3]: slice_pos, fiber_start, fiber_stop
  hbk::Buf mult;   // uint32 [S]
};

namespace hbk {

// Device helpers -------------------------------------------------------------
// L2 cache policies: index/value streams are read once (evict-first), factor
// rows are gathered repeatedly (evict-last), so the streams do not wash the
// factor rows out of the 126 MB L2.  This is the per-access form of the
// access-policy window (the window API needs a single contiguous range and
// the persisting carve-out; the hint covers every factor matrix at once).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// Factor-row gather (16 B per lane, 8 lanes = one 128 B row at R=32).
__device__ __forceinline__ float4 ld_row4(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::evict_last.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

}  // namespace hbk
