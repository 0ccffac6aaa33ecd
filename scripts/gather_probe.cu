// Gather-throughput probe: how fast can B200 gather 128-byte factor rows by
// index (the MTTKRP inner operation)?  Standalone; build & run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp scripts/gather_probe.cu && /tmp/gp
// Variants:
//   ldg<U,W>   : 8 lanes x LDG.128 per row, U rows in flight per 8-lane group,
//                W warps per block (occupancy).
//   tma<S>     : each lane issues cp.async.bulk (TMA) of its own row into a
//                per-warp S-stage smem ring (mbarrier complete_tx), consumer
//                reads LDS.128.
// Index streams: Zipf(1) over 28818 rows (nell-2 leaf mode, L2-resident
// factor) and uniform / Zipf over 25.5M rows (nell-1 leaf mode, 3.2 GB).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ __forceinline__ float4 ldrow(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}

template <int U>
__global__ void k_ldg(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                      float4* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane >> 3, lig = lane & 7;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = gid * U; base < n; base += ngroups * U) {
    uint32_t k = (base + lig < n && lig < U) ? idx[base + lig] : 0;
    float4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint32_t kj = __shfl_sync(0xffffffffu, k, j % 8, 8);
      r[j] = ldrow(F + size_t(kj) * 8 + lig);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      acc.x += r[j].x;
      acc.y += r[j].y;
      acc.z += r[j].z;
      acc.w += r[j].w;
    }
  }
  (void)g;
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}


// 32 lanes x LDG.32 per row: one 128-byte line per warp instruction.
__device__ __forceinline__ float ldf(const float* p) {
  float v;
  asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <int U>
__global__ void k_ldg32(const float* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                        float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t base = wid * 32; base < n; base += nw * 32) {
    uint32_t k = (base + lane < n) ? idx[base + lane] : 0;
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += U) {
      float r[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        uint32_t kj = __shfl_sync(0xffffffffu, k, j0 + j);
        r[j] = ldf(F + size_t(kj) * 32 + lane);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) acc += r[j];
    }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}
// 16 lanes x LDG.64 per row: two lines per warp instruction.
__device__ __forceinline__ float2 ldf2(const float2* p) {
  float2 v;
  asm("ld.global.nc.L1::evict_last.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
template <int U>
__global__ void k_ldg64(const float2* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                        float2* __restrict__ out) {
  const int lane = threadIdx.x & 31, h = lane >> 4, l16 = lane & 15;
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  float2 acc = make_float2(0.f, 0.f);
  for (int64_t base = wid * 32; base < n; base += nw * 32) {
    uint32_t k = (base + lane < n) ? idx[base + lane] : 0;
#pragma unroll
    for (int j0 = 0; j0 < 16; j0 += U) {
      float2 r[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        uint32_t kj = __shfl_sync(0xffffffffu, k, 2 * (j0 + j) + h);
        r[j] = ldf2(F + size_t(kj) * 16 + l16);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) { acc.x += r[j].x; acc.y += r[j].y; }
    }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// hot-row cache: rows [0, H) of F staged in shared memory once per CTA
// (the synthetic power-law streams are hottest at low indices); a row is read
// with LDS.128 when k < H, else LDG.128.  8 lanes x float4 per row.
template <int U, bool ALL>
__global__ void k_hot(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                      int H, float4* __restrict__ out) {
  extern __shared__ float4 cache[];
  for (int i = threadIdx.x; i < H * 8; i += blockDim.x) cache[i] = F[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, lig = lane & 7;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = gid * U; base < n; base += ngroups * U) {
    uint32_t k = (base + lig < n && lig < U) ? idx[base + lig] : 0;
    if (ALL) k %= H;
    float4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint32_t kj = __shfl_sync(0xffffffffu, k, j % 8, 8);
      if (kj < (uint32_t)H)
        r[j] = cache[kj * 8 + lig];
      else
        r[j] = ldrow(F + size_t(kj) * 8 + lig);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      acc.x += r[j].x;
      acc.y += r[j].y;
      acc.z += r[j].z;
      acc.w += r[j].w;
    }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// cache-hint variants of the 8-lane LDG.128 row gather
template <int HINT>
__device__ __forceinline__ float4 ldrow_h(const float4* p) {
  float4 v;
  if (HINT == 0)
    asm("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (HINT == 1)
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (HINT == 2)
    asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (HINT == 3)
    asm("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    asm("ld.global.nc.L1::evict_first.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <int HINT>
__global__ void k_ldg_hint(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                           float4* __restrict__ out) {
  const int lane = threadIdx.x & 31, lig = lane & 7;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = gid * 8; base < n; base += ngroups * 8) {
    uint32_t k = (base + lig < n) ? idx[base + lig] : 0;
    float4 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t kj = __shfl_sync(0xffffffffu, k, j, 8);
      r[j] = ldrow_h<HINT>(F + size_t(kj) * 8 + lig);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc.x += r[j].x; acc.y += r[j].y; acc.z += r[j].z; acc.w += r[j].w; }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// L1 split by row hotness: rows k < H (the power-law head) evict_last,
// colder rows HINT2 (1 = L1::no_allocate, 4 = L1::evict_first)
template <int HINT2>
__global__ void k_ldg_split(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                            uint32_t H, float4* __restrict__ out) {
  const int lane = threadIdx.x & 31, lig = lane & 7;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = gid * 8; base < n; base += ngroups * 8) {
    uint32_t k = (base + lig < n) ? idx[base + lig] : 0;
    float4 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t kj = __shfl_sync(0xffffffffu, k, j, 8);
      const float4* p = F + size_t(kj) * 8 + lig;
      r[j] = kj < H ? ldrow_h<0>(p) : ldrow_h<HINT2>(p);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc.x += r[j].x; acc.y += r[j].y; acc.z += r[j].z; acc.w += r[j].w; }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// Index stream staged through shared memory with cp.async (D batches ahead,
// one 16-byte copy per lane pair), rows gathered 8 lanes x LDG.128 — the
// north-star's "stream through cp.async staging" against the direct LDG of
// the index (k_ldg<8>, prefetched one batch ahead by the warp scheduler).
template <int D>
__global__ void k_ldg_staged(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                             float4* __restrict__ out) {
  __shared__ __align__(16) uint32_t ring[256 / 8][D][8];  // per group: D batches of 8 indices
  const int lane = threadIdx.x & 31, lig = lane & 7, grp = threadIdx.x >> 3;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  const int64_t nb = n / 8;  // whole batches only (n is a multiple of 8 here)
  const int64_t mine = gid < nb ? (nb - 1 - gid) / ngroups + 1 : 0;
  const int64_t maxb = (nb + ngroups - 1) / ngroups;
  auto issue = [&](int64_t b) {
    if (b < mine && lig < 2) {
      const uint32_t* g = idx + (gid + b * ngroups) * 8 + lig * 4;
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&ring[grp][b % D][lig * 4]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < D - 1; ++s) issue(s);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t b = 0; b < maxb; ++b) {
    issue(b + D - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    __syncwarp();
    if (b < mine) {
      float4 r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = ldrow(F + size_t(ring[grp][b % D][j]) * 8 + lig);
#pragma unroll
      for (int j = 0; j < 8; ++j) { acc.x += r[j].x; acc.y += r[j].y; acc.z += r[j].z; acc.w += r[j].w; }
    }
    __syncwarp();
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// 4 lanes x LDG.256 per row (8 rows per warp instruction)
struct f8 {
  float v[8];
};
__device__ __forceinline__ f8 ldrow8(const float* p) {
  f8 r;
  asm("ld.global.nc.L1::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
        "=f"(r.v[6]), "=f"(r.v[7])
      : "l"(p));
  return r;
}
template <int U>
__global__ void k_ldg256(const float* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                         float* __restrict__ out) {
  const int lane = threadIdx.x & 31, lig = lane & 3;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 2;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 2;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t base = gid * U; base < n; base += ngroups * U) {
    uint32_t k[U / 4 > 0 ? U / 4 : 1];
#pragma unroll
    for (int q = 0; q < (U + 3) / 4; ++q) k[q] = (base + 4 * q + lig < n) ? idx[base + 4 * q + lig] : 0;
    f8 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint32_t kj = __shfl_sync(0xffffffffu, k[j / 4], j % 4, 4);
      r[j] = ldrow8(F + size_t(kj) * 32 + lig * 8);
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += r[j].v[i];
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = s;
}

// cp.async (LDGSTS) gathers into a per-group S-stage smem ring (8 rows per
// stage per 8-lane group), consumer LDS.128.
template <int S>
__global__ void k_ldgsts(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                         float4* __restrict__ out) {
  extern __shared__ float4 ring[];  // [blockDim/8 groups][S][8 rows][8 lanes]
  const int lane = threadIdx.x & 31, lig = lane & 7;
  const int grp = threadIdx.x >> 3;
  float4* my = ring + size_t(grp) * S * 64 + lig;
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ngroups = (int64_t(gridDim.x) * blockDim.x) >> 3;
  const int64_t nb = (n + 7) / 8;
  const int64_t mine = gid < nb ? (nb - 1 - gid) / ngroups + 1 : 0;
  const int64_t maxb = (nb + ngroups - 1) / ngroups;
  float4 acc = make_float4(0, 0, 0, 0);
  auto issue = [&](int64_t b) {
    if (b < mine) {
      const int64_t base = (gid + b * ngroups) * 8;
      uint32_t k = (base + lig < n) ? idx[base + lig] : 0;
      float4* st = my + (b % S) * 64;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t kj = __shfl_sync(0xffffffffu, k, j, 8);
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st + j * 8);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(F + size_t(kj) * 8 + lig) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < S - 1; ++s) issue(s);
  for (int64_t b = 0; b < maxb; ++b) {
    issue(b + S - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    if (b < mine) {
      const float4* st = my + (b % S) * 64;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 r = st[j * 8];
        acc.x += r.x;
        acc.y += r.y;
        acc.z += r.z;
        acc.w += r.w;
      }
    }
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

// ---- TMA (cp.async.bulk) gather -------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n }\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_row(void* smem, const void* g, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(g), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int S>
__global__ void k_tma(const float4* __restrict__ F, const uint32_t* __restrict__ idx, int64_t n,
                      float4* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lig = lane & 7, g = lane >> 3;
  const int nw = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(smem) + size_t(warp) * S * 32 * 8;  // S stages x 32 rows x 8 float4
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(nw) * S * 32 * 128) + warp * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t wid = blockIdx.x * int64_t(nw) + warp;
  const int64_t nwarps = int64_t(gridDim.x) * nw;
  // warp batch = 32 rows (lane l fetches row idx[base + l])
  const int64_t nbatch = (n + 31) / 32;
  float4 acc = make_float4(0, 0, 0, 0);
  int64_t mine = wid < nbatch ? (nbatch - 1 - wid) / nwarps + 1 : 0;
  auto issue = [&](int64_t b, int s) {
    const int64_t e = (wid + b * nwarps) * 32 + lane;
    const int64_t rem = n - (wid + b * nwarps) * 32; const int cnt = rem < 32 ? (int)rem : 32;
    if (lane == 0) mbar_expect(bars + s, cnt * 128);
    __syncwarp();
    if (lane < cnt) bulk_row(ring + (s * 32 + lane) * 8, F + size_t(idx[e]) * 8, bars + s);
  };
  for (int s = 0; s < S - 1 && s < mine; ++s) issue(s, s);
  for (int64_t b = 0; b < mine; ++b) {
    const int s = b % S;
    if (b + S - 1 < mine) issue(b + S - 1, (b + S - 1) % S);
    mbar_wait(bars + s, (b / S) & 1);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 r = ring[(s * 32 + g * 8 + j) * 8 + lig];
      acc.x += r.x;
      acc.y += r.y;
      acc.z += r.z;
      acc.w += r.w;
    }
    __syncwarp();
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = acc;
}

static std::vector<uint32_t> zipf_stream(int64_t n, uint32_t rows, double alpha, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<uint32_t> v(n);
  const double top = double(rows) + 1.0;
  for (int64_t i = 0; i < n; ++i) {
    double u = U(rng), x;
    if (alpha == 1.0)
      x = std::exp(u * std::log(top));
    else if (alpha == 0.0)
      x = 1.0 + u * (top - 1.0);
    else
      x = std::pow((std::pow(top, 1 - alpha) - 1) * u + 1, 1 / (1 - alpha));
    int64_t k = int64_t(std::floor(x)) - 1;
    if (k < 0) k = 0;
    if (k >= rows) k = rows - 1;
    v[i] = uint32_t(k);
  }
  return v;
}

template <class Fn>
static float time_ms(Fn fn, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  fn();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) fn();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n = 40'000'000;
  struct Case {
    const char* name;
    uint32_t rows;
    double alpha;
  } cases[] = {{"zipf1 28818 rows (L2)", 28818, 1.0},
               {"zipf1 25.5M rows (HBM)", 25495389, 1.0},
               {"uniform 25.5M rows (HBM)", 25495389, 0.0}};
  float4* out;
  CK(cudaMalloc(&out, size_t(sms) * 64 * 256 * sizeof(float4)));
  for (auto& c : cases) {
    std::vector<uint32_t> h = zipf_stream(n, c.rows, c.alpha, 7);
    uint32_t* idx;
    float4* F;
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&F, size_t(c.rows) * 128));
    {
      std::vector<float> hf(size_t(c.rows) * 32);
      for (size_t i = 0; i < hf.size(); ++i) hf[i] = float((i * 2654435761u) % 1000) * 1e-3f;
      CK(cudaMemcpy(F, hf.data(), hf.size() * 4, cudaMemcpyHostToDevice));
    }
    const double gb = double(n) * 128 / 1e9;
    printf("== %s: %lld gathers of 128 B (%.2f GB)\n", c.name, (long long)n, gb);
#define RUN_LDG(U, THREADS, BLOCKS_PER_SM)                                                        \
  {                                                                                               \
    int g = sms * BLOCKS_PER_SM;                                                                  \
    float ms = time_ms([&] { k_ldg<U><<<g, THREADS>>>(F, idx, n, out); });                        \
    printf("  ldg U=%2d thr=%d blk/sm=%d : %.3f ms  %.2f Grows/s  %.1f GB/s\n", U, THREADS,       \
           BLOCKS_PER_SM, ms, n / ms / 1e6, gb / ms * 1e3);                                       \
  }
#define RUN_L32(U, THREADS, BLOCKS_PER_SM)                                                        \
  {                                                                                               \
    int g = sms * BLOCKS_PER_SM;                                                                  \
    float ms = time_ms([&] { k_ldg32<U><<<g, THREADS>>>((const float*)F, idx, n, (float*)out); }); \
    printf("  ldg32 U=%2d thr=%d blk/sm=%d : %.3f ms  %.2f Grows/s  %.1f GB/s\n", U, THREADS,    \
           BLOCKS_PER_SM, ms, n / ms / 1e6, gb / ms * 1e3);                                       \
  }
#define RUN_L64(U, THREADS, BLOCKS_PER_SM)                                                        \
  {                                                                                               \
    int g = sms * BLOCKS_PER_SM;                                                                  \
    float ms = time_ms([&] { k_ldg64<U><<<g, THREADS>>>((const float2*)F, idx, n, (float2*)out); }); \
    printf("  ldg64 U=%2d thr=%d blk/sm=%d : %.3f ms  %.2f Grows/s  %.1f GB/s\n", U, THREADS,    \
           BLOCKS_PER_SM, ms, n / ms / 1e6, gb / ms * 1e3);                                       \
  }
#define RUN_HOT(ALL, H, THREADS, BLOCKS_PER_SM)                                                 \
  {                                                                                               \
    int hh = (ALL) ? (H) : std::min<int>((H), (int)c.rows);                                        \
    size_t sm = size_t(hh) * 128;                                                                 \
    CK(cudaFuncSetAttribute(k_hot<8, ALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))); \
    int g = sms * BLOCKS_PER_SM;                                                                  \
    float ms = time_ms([&] { k_hot<8, ALL><<<g, THREADS, sm>>>(F, idx, n, hh, out); });          \
    CK(cudaGetLastError());                                                                       \
    printf("  hot all=%d H=%d thr=%d blk/sm=%d : %.3f ms  %.2f Grows/s\n", (int)(ALL), hh,       \
           THREADS, BLOCKS_PER_SM, ms, n / ms / 1e6);                                             \
  }
#define RUN_HINT(H, BPS)                                                                       \
  {                                                                                               \
    int g = sms * BPS;                                                                            \
    float ms = time_ms([&] { k_ldg_hint<H><<<g, 256>>>(F, idx, n, out); });                      \
    printf("  hint=%d blk/sm=%d : %.3f ms  %.2f Grows/s\n", H, BPS, ms, n / ms / 1e6);         \
  }
    if (getenv("STAGED")) {
      for (int bps : {4, 8}) {
        int g = sms * bps;
        float m0 = time_ms([&] { k_ldg<8><<<g, 256>>>(F, idx, n, out); });
        float m2 = time_ms([&] { k_ldg_staged<2><<<g, 256>>>(F, idx, n, out); });
        float m4 = time_ms([&] { k_ldg_staged<4><<<g, 256>>>(F, idx, n, out); });
        printf("  blk/sm=%d direct LDG idx %.2f | cp.async-staged D=2 %.2f | D=4 %.2f Grows/s\n", bps,
               n / m0 / 1e6, n / m2 / 1e6, n / m4 / 1e6);
      }
      CK(cudaFree(idx));
      CK(cudaFree(F));
      continue;
    }
    if (getenv("SPLIT")) {
      for (uint32_t H : {256u, 512u, 1024u, 2048u, 4096u, 8192u}) {
        int g = sms * 4;
        float ms1 = time_ms([&] { k_ldg_split<1><<<g, 256>>>(F, idx, n, H, out); });
        float ms4 = time_ms([&] { k_ldg_split<4><<<g, 256>>>(F, idx, n, H, out); });
        printf("  split H=%u : no_allocate tail %.2f Grows/s, evict_first tail %.2f Grows/s\n", H,
               n / ms1 / 1e6, n / ms4 / 1e6);
      }
      RUN_HINT(0, 4);
      CK(cudaFree(idx));
      CK(cudaFree(F));
      continue;
    }
    if (getenv("HINTS")) {
      RUN_HINT(0, 4); RUN_HINT(1, 4); RUN_HINT(2, 4); RUN_HINT(3, 4); RUN_HINT(4, 4);
      RUN_HINT(0, 8); RUN_HINT(1, 8); RUN_HINT(3, 8);
      CK(cudaFree(idx));
      CK(cudaFree(F));
      continue;
    }
    RUN_HOT(true, 512, 1024, 1);
    RUN_HOT(true, 1536, 1024, 1);
    RUN_HOT(false, 512, 512, 2);
    RUN_HOT(false, 768, 512, 2);
    RUN_HOT(false, 1024, 1024, 1);
    RUN_HOT(false, 1536, 1024, 1);
    RUN_HOT(false, 1536, 768, 1);
    RUN_L32(8, 256, 4);
    RUN_L32(16, 256, 4);
    RUN_L32(16, 256, 8);
    RUN_L32(32, 256, 4);
    RUN_L64(8, 256, 4);
    RUN_L64(8, 256, 8);
    RUN_L64(16, 256, 4);
    RUN_LDG(8, 256, 2);
    RUN_LDG(8, 256, 4);
    RUN_LDG(8, 256, 8);

#define RUN_TMA(S, THREADS, BLOCKS_PER_SM)                                                          \
  {                                                                                                 \
    size_t sm = size_t(THREADS / 32) * S * (32 * 128 + 8);                                          \
    CK(cudaFuncSetAttribute(k_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));       \
    int g = sms * BLOCKS_PER_SM;                                                                    \
    float ms = time_ms([&] { k_tma<S><<<g, THREADS, sm>>>(F, idx, n, out); });                      \
    CK(cudaGetLastError());                                                                         \
    printf("  tma S=%d thr=%d blk/sm=%d smem=%zuKB: %.3f ms  %.2f Grows/s  %.1f GB/s\n", S, THREADS, \
           BLOCKS_PER_SM, sm / 1024, ms, n / ms / 1e6, gb / ms * 1e3);                              \
  }
#define RUN_LDG8(U, THREADS, BLOCKS_PER_SM)                                                       \
  {                                                                                               \
    int g = sms * BLOCKS_PER_SM;                                                                  \
    float ms = time_ms([&] { k_ldg256<U><<<g, THREADS>>>((const float*)F, idx, n, (float*)out); }); \
    printf("  ldg256 U=%2d thr=%d blk/sm=%d : %.3f ms  %.2f Grows/s  %.1f GB/s\n", U, THREADS,   \
           BLOCKS_PER_SM, ms, n / ms / 1e6, gb / ms * 1e3);                                       \
  }
    RUN_LDG8(4, 256, 2);
    RUN_LDG8(4, 256, 4);
    RUN_LDG8(8, 256, 2);
    RUN_LDG8(8, 256, 3);

    if (getenv("TMA")) RUN_TMA(2, 256, 2);
#define RUN_GSTS(S, THREADS, BLOCKS_PER_SM)                                                          \
  {                                                                                                \
    size_t sm = size_t(THREADS / 8) * S * 64 * 16;                                                 \
    CK(cudaFuncSetAttribute(k_ldgsts<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));   \
    int g = sms * BLOCKS_PER_SM;                                                                   \
    float ms = time_ms([&] { k_ldgsts<S><<<g, THREADS, sm>>>(F, idx, n, out); });                  \
    CK(cudaGetLastError());                                                                        \
    printf("  ldgsts S=%d thr=%d blk/sm=%d smem=%zuKB: %.3f ms  %.2f Grows/s\n", S, THREADS,       \
           BLOCKS_PER_SM, sm / 1024, ms, n / ms / 1e6);                                            \
  }
    RUN_GSTS(2, 256, 2);
    RUN_GSTS(3, 256, 2);
    RUN_GSTS(4, 256, 2);
    RUN_GSTS(4, 256, 1);
    RUN_GSTS(6, 256, 1);
    RUN_GSTS(8, 128, 2);

    CK(cudaFree(idx));
    CK(cudaFree(F));
  }
  return 0;
}
