// Distributed-shared-memory gather probe: can a thread-block cluster hold
// the nell-2 leaf factor (28,818 rows x 128 B = 3.69 MB) in its CTAs' shared
// memory (16 CTAs x 225 KB) and serve the row gathers from there faster than
// the L1/L2 path?  Zipf(1) row ids (the leaf marginal), 8 lanes x 16 B per
// row, group-owned chunks of 1,024 positions.
//   l2   : rows from global memory (LDG.128, L1 evict-last) — the product path
//   dsm  : rows from the owner CTA's shared memory (mapa + ld.shared::cluster)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dsp scripts/dsmem_probe.cu && /tmp/dsp
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cmath>
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

static constexpr int CH = 1024;

__device__ __forceinline__ float4 ld128(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldstream(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_dsm(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr));
  return v;
}
__device__ __forceinline__ uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool DSM>
__global__ void k_gather(const float4* __restrict__ F, const uint2* __restrict__ s, int64_t n, int rpc,
                         int csize, float4* __restrict__ sink) {
  extern __shared__ float4 tab[];
  const int lane = threadIdx.x & 31, lig = lane & 7;
  uint32_t base_addr = 0;
  if (DSM) {
    const uint32_t me = cluster_rank();
    for (int i = threadIdx.x; i < rpc * 8; i += blockDim.x) {
      const int64_t g = int64_t(me) * rpc * 8 + i;
      tab[i] = g < int64_t(28818) * 8 ? F[g] : make_float4(0, 0, 0, 0);
    }
    base_addr = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    cluster_sync();
  }
  // groups of the whole grid own chunks round-robin
  const int64_t gid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 3;
  const int64_t ng = (int64_t(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  const int64_t nch = (n + CH - 1) / CH;
  const int64_t my = gid < nch ? (nch - 1 - gid) / ng + 1 : 0;
  const int64_t iters = __reduce_max_sync(0xffffffffu, uint32_t(my)) * (CH / 8);
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t pos = (gid + (it / (CH / 8)) * ng) * CH + (it % (CH / 8)) * 8;
    uint2 q = pos + lig < n ? ldstream(s + pos + lig) : make_uint2(0, 0);
    float4 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t k = __shfl_sync(0xffffffffu, q.x, j, 8);
      if (DSM) {
        const uint32_t owner = k / uint32_t(rpc), row = k - owner * uint32_t(rpc);
        r[j] = ld_dsm(mapa(base_addr + (row * 8 + lig) * 16, owner));
      } else {
        r[j] = ld128(F + size_t(k) * 8 + lig);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float v = __uint_as_float(__shfl_sync(0xffffffffu, q.y, j, 8));
      acc.x = fmaf(v, r[j].x, acc.x);
      acc.y = fmaf(v, r[j].y, acc.y);
      acc.z = fmaf(v, r[j].z, acc.z);
      acc.w = fmaf(v, r[j].w, acc.w);
    }
  }
  if (DSM) cluster_sync();  // keep every CTA's table alive until all reads are done
  if (acc.x == 1234.5f) sink[threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int rows = 28818;
  const int64_t n = argc > 1 ? atoll(argv[1]) : 77000000;
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<uint2> s(n);
  for (int64_t i = 0; i < n; ++i) {
    int id = int(std::floor(std::exp(U(rng) * std::log(rows + 1.0)))) - 1;
    id = std::min(rows - 1, std::max(0, id));
    float v = float(U(rng));
    s[i] = make_uint2(uint32_t(id), *reinterpret_cast<uint32_t*>(&v));
  }
  float4* F;
  uint2* ds;
  float4* sink;
  CK(cudaMalloc(&F, size_t(rows) * 128));
  CK(cudaMemset(F, 0, size_t(rows) * 128));
  CK(cudaMalloc(&ds, n * sizeof(uint2)));
  CK(cudaMemcpy(ds, s.data(), n * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&sink, 4096 * sizeof(float4)));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time = [&](const char* name, auto launch) {
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    printf("%-34s %8.3f ms  %7.1f G rows/s\n", name, best, n / (best * 1e-3) / 1e9);
  };
  time("l2 (LDG.128), 24 warps/SM", [&] { k_gather<false><<<sms * 3, 256, 0>>>(F, ds, n, 0, 0, sink); });
  time("l2 (LDG.128), 32 warps/SM", [&] { k_gather<false><<<sms * 4, 256, 0>>>(F, ds, n, 0, 0, sink); });
  for (int cs : {16, 8}) {
    const int rpc = (rows + cs - 1) / cs;
    const size_t smem = size_t(rpc) * 128;
    if (smem > 232448) {
      printf("cluster %d: %zu B of shared memory per CTA does not fit\n", cs, smem);
      continue;
    }
    CK(cudaFuncSetAttribute(k_gather<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CK(cudaFuncSetAttribute(k_gather<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int threads : {512, 768, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      cfg.gridDim = dim3(cs);
      CK(cudaOccupancyMaxActiveClusters(&nclusters, k_gather<true>, &cfg));
      if (nclusters == 0) {
        printf("cluster %d x %d threads: no cluster fits\n", cs, threads);
        continue;
      }
      cfg.gridDim = dim3(nclusters * cs);
      char nm[80];
      snprintf(nm, sizeof nm, "dsm cluster %d (%d clusters) %d thr", cs, nclusters, threads);
      time(nm, [&] { CK(cudaLaunchKernelEx(&cfg, k_gather<true>, (const float4*)F, (const uint2*)ds, n, rpc, cs, sink)); });
    }
  }
  return 0;
}
