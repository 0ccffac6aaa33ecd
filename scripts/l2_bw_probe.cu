// L2 -> SM bandwidth ceilings on this B200, for the L2-resident roofline of
// the MTTKRP kernels: the MTTKRP moves 128-byte factor rows
// from L2 to the SMs at random row indices, so its ceiling is the rate at
// which the L2 can deliver such rows, not HBM.
//
//   stream: every thread reads consecutive float4s of an L2-resident buffer
//           (grid-stride, ld.global.cg = L2, not L1), 8 loads in flight
//   rows:   8-lane groups gather whole 128-B rows at pseudo-random row
//           indices of an L2-resident matrix, 8 rows in flight per group —
//           the MTTKRP's access shape without its index streams; -L2 with
//           ld.global.cg (every row from L2), -L1 with ld.global.nc (L1
//           allocating, as the kernels load factor rows)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw_probe scripts/l2_bw_probe.cu
//   ./l2_bw_probe            (one GPU; prints GB/s per variant, best of 7)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__device__ __forceinline__ float4 ld_cg(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_stream(const float4* __restrict__ a, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = tid; i < n4; i += 8 * stride) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = i + u * stride < n4 ? ld_cg(a + i + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 1234.5f) *sink = acc;
}

// rows: nrows (a power of two) x 8 float4 (128 B); each 8-lane group gathers
// `per_group` rows at pseudo-random indices (an LCG: two instructions per row)
template <bool L1>
__global__ void k_rows(const float4* __restrict__ a, uint32_t nrows, int per_group, float* sink) {
  const uint32_t lane = threadIdx.x & 31, lig = lane & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint32_t x = mix(grp + 1u);
  const uint32_t m = nrows - 1;
  float acc = 0.f;
  for (int it = 0; it < per_group; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const float4* p = a + size_t((x >> 8) & m) * 8 + lig;
      v[u] = L1 ? __ldg(p) : ld_cg(p);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *sink = acc;
}

// rows with the MTTKRP's per-row overheads: each lane of a group holds one
// position's (index, value); per batch of 8 the group broadcasts them with
// 16 SHFL (as the kernels do), gathers the 8 rows, and (FMA) accumulates
// value * row with 4 FFMA per row per lane
template <bool FMA>
__global__ void k_rows_shfl(const float4* __restrict__ a, uint32_t nrows, int per_group, float* sink) {
  const uint32_t lane = threadIdx.x & 31, lig = lane & 7;
  const uint32_t gid = (blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t x = mix(gid + 1u);
  const uint32_t m = nrows - 1;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float accs = 0.f;
  for (int it = 0; it < per_group; it += 8) {
    x = x * 1664525u + 1013904223u;
    const uint32_t mine = (x >> 8) & m;
    const float val = __uint_as_float(0x3f800000u | (x & 0x7fffu));
    float4 v[8];
    float w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = __shfl_sync(0xffffffffu, mine, u, 8);
      v[u] = __ldg(a + size_t(r) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = __shfl_sync(0xffffffffu, val, u, 8);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (FMA) {
        acc.x = fmaf(w[u], v[u].x, acc.x); acc.y = fmaf(w[u], v[u].y, acc.y);
        acc.z = fmaf(w[u], v[u].z, acc.z); acc.w = fmaf(w[u], v[u].w, acc.w);
      } else {
        accs += v[u].x + v[u].y + v[u].z + v[u].w + w[u];
      }
    }
  }
  if (acc.x + acc.y + acc.z + acc.w + accs == 1234.5f) *sink = acc.x;
}

// rows with a Zipf(1) row distribution (P(r) ~ 1/(r+1), r = 2^(u log2 N) - 1),
// optionally scattered over the matrix by an odd multiplier (SCRAMBLE): the
// skew of the FROSTT-shaped tensors' leaf modes, for L2-slice hot spots
template <bool SCRAMBLE>
__global__ void k_rows_zipf(const float4* __restrict__ a, uint32_t nrows, int per_group, float* sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint32_t x = mix(grp + 1u);
  const uint32_t m = nrows - 1;
  const float l2n = log2f(float(nrows));
  float acc = 0.f;
  for (int it = 0; it < per_group; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      uint32_t r = uint32_t(exp2f(float(x >> 8) * (1.0f / 16777216.0f) * l2n)) - 1u;
      if (SCRAMBLE) r *= 2654435761u;
      v[u] = __ldg(a + size_t(r & m) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *sink = acc;
}

// Zipf rows with the H hottest rows replicated REP times after the matrix:
// a group reads replica (group id mod REP) of a hot row, spreading the hot
// rows' requests over REP times more L2 lines / slices
template <int REP, bool PER_SM>
__global__ void k_rows_zipf_rep(const float4* __restrict__ a, uint32_t nrows, uint32_t H, int per_group,
                                float* sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint32_t x = mix(grp + 1u);
  const uint32_t m = nrows - 1;
  const float l2n = log2f(float(nrows));
  uint32_t smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  const uint32_t rep = PER_SM ? smid % REP : grp % REP;
  float acc = 0.f;
  for (int it = 0; it < per_group; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t r = (uint32_t(exp2f(float(x >> 8) * (1.0f / 16777216.0f) * l2n)) - 1u) & m;
      const size_t row = r < H ? size_t(nrows) + size_t(r) * REP + rep : size_t(r);
      v[u] = __ldg(a + row * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *sink = acc;
}

// rows named by an index STREAM, as the MTTKRP reads them: each group walks
// its own contiguous span of a u32 index array (HBM, L1 no-allocate), one
// coalesced load per lane per batch of 8, 8 SHFL to broadcast, 8 row gathers
// (L1-allocating).  Index arrays: uniform or Zipf(1), generated on the host.
template <bool CG>
__global__ void k_rows_stream(const float4* __restrict__ a, const uint32_t* __restrict__ idx,
                              int per_group, float* sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const uint32_t* my = idx + size_t(grp) * per_group;
  float acc = 0.f;
  uint32_t cur;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(cur) : "l"(my + lig));
  for (int it = 0; it < per_group; it += 8) {
    uint32_t nxt = 0;
    if (it + 8 < per_group)
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(nxt) : "l"(my + it + 8 + lig));
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = __shfl_sync(0xffffffffu, cur, u, 8);
      v[u] = CG ? ld_cg(a + size_t(r) * 8 + lig) : __ldg(a + size_t(r) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    cur = nxt;
  }
  if (acc == 1234.5f) *sink = acc;
}

// uniform random rows over any row count (multiply-shift range reduction)
__global__ void k_rows_any(const float4* __restrict__ a, uint32_t nrows, int per_group, float* sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint32_t x = mix(grp + 1u);
  float acc = 0.f;
  for (int it = 0; it < per_group; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t r = uint32_t((uint64_t(x) * nrows) >> 32);
      v[u] = __ldg(a + size_t(r) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *sink = acc;
}

static int size_sweep() {
  // uniform random rows over matrices of growing footprint: where the rate
  // falls from the L2 rate to the HBM rate is the L2 capacity the gather sees
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t maxb = size_t(512) << 20;
  float4* buf = nullptr;
  float* sink = nullptr;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 0, maxb));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int grid = sms * 4;
  const int groups = grid * 256 / 8;
  const int per_group = int(((size_t(4) << 30) / 128 / groups + 7) / 8 * 8);
  for (int mb = 16; mb <= 512; mb += (mb < 160 ? 16 : 64)) {
    // nrows must be a power of two for the LCG mask: use the largest power
    // of two <= mb, and scale rows onto [0, rows_mb) by a multiply-shift
    const uint32_t rows = uint32_t((size_t(mb) << 20) / 128);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      CK(cudaEventRecord(e0));
      k_rows_any<<<grid, 256>>>(buf, rows, per_group, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (t && ms < best) best = ms;
    }
    const double rb = double(groups) * per_group * 128.0;
    printf("sweep %4d MB  %8.1f GB/s  (%.1f G rows/s)\n", mb, rb / best / 1e6, rb / 128.0 / best / 1e6);
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 's') return size_sweep();
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t max_bytes = size_t(64) << 20;
  float4* buf = nullptr;
  float* sink = nullptr;
  CK(cudaMalloc(&buf, max_bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 0, max_bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t sizes[] = {size_t(8) << 20};
  // index streams for k_rows_stream: 2^26 indices, uniform and Zipf(1) over
  // the 8-MB matrix's 65,536 rows (host-generated, fixed seed)
  const size_t nidx = size_t(1) << 26;
  const uint32_t srows = uint32_t((size_t(8) << 20) / 128);
  uint32_t* h_idx = (uint32_t*)malloc(nidx * 4);
  uint32_t* d_uni = nullptr;
  uint32_t* d_zipf = nullptr;
  CK(cudaMalloc(&d_uni, nidx * 4));
  CK(cudaMalloc(&d_zipf, nidx * 4));
  {
    uint64_t st = 88172645463325252ull;
    auto nextu = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
    for (size_t i = 0; i < nidx; ++i) h_idx[i] = uint32_t(nextu() % srows);
    CK(cudaMemcpy(d_uni, h_idx, nidx * 4, cudaMemcpyHostToDevice));
    const double ln = log(double(srows) + 1.0);
    for (size_t i = 0; i < nidx; ++i) {
      const double u = double(nextu() >> 11) * (1.0 / 9007199254740992.0);
      uint32_t r = uint32_t(floor(exp(u * ln))) - 1u;
      if (r >= srows) r = srows - 1;
      h_idx[i] = uint32_t((uint64_t(r) * 2654435761ull) % srows);  // scattered hot rows
    }
    CK(cudaMemcpy(d_zipf, h_idx, nidx * 4, cudaMemcpyHostToDevice));
  }
  const int ctas_per_sm[] = {4, 8};  // 256-thread CTAs: 16 / 24 / 32 / 64 warps per SM
  for (size_t bytes : sizes) {
    for (int c : ctas_per_sm) {
      const int grid = sms * c;
      // stream: about 4 GB read per launch
      const size_t n4 = bytes / 16;
      const int reps = int((size_t(4) << 30) / bytes);
      float best = 1e30f;
      for (int t = 0; t < 7; ++t) {
        CK(cudaEventRecord(e0));
        k_stream<<<grid, 256>>>(buf, n4, reps, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (t && ms < best) best = ms;
      }
      const double read = double(reps) * double(n4) * 16;
      printf("stream  %3zu MB  %2d warps/SM  %8.1f GB/s\n", bytes >> 20, c * 8, read / best / 1e6);
      // rows: 128-B rows at random indices, about 4 GB per launch
      const uint32_t nrows = uint32_t(bytes / 128);
      const int groups = grid * 256 / 8;
      const int per_group = int(((size_t(4) << 30) / 128 / groups + 7) / 8 * 8);
      for (int l1 = 0; l1 < 2; ++l1) {
        best = 1e30f;
        for (int t = 0; t < 7; ++t) {
          CK(cudaEventRecord(e0));
          if (l1) k_rows<true><<<grid, 256>>>(buf, nrows, per_group, sink);
          else k_rows<false><<<grid, 256>>>(buf, nrows, per_group, sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (t && ms < best) best = ms;
        }
        const double rb = double(groups) * per_group * 128.0;
        printf("rows%s %3zu MB  %2d warps/SM  %8.1f GB/s  (%.1f G rows/s)\n", l1 ? "-L1" : "-L2",
               bytes >> 20, c * 8, rb / best / 1e6, rb / 128.0 / best / 1e6);
      }
      for (int sc = 0; sc < 2; ++sc) {
        best = 1e30f;
        for (int t = 0; t < 7; ++t) {
          CK(cudaEventRecord(e0));
          if (sc) k_rows_zipf<true><<<grid, 256>>>(buf, nrows, per_group, sink);
          else k_rows_zipf<false><<<grid, 256>>>(buf, nrows, per_group, sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (t && ms < best) best = ms;
        }
        const double rb = double(groups) * per_group * 128.0;
        printf("rows-zipf%s %3zu MB  %2d warps/SM  %8.1f GB/s  (%.1f G rows/s)\n", sc ? "-scrambled" : "",
               bytes >> 20, c * 8, rb / best / 1e6, rb / 128.0 / best / 1e6);
      }
      for (int cfg = 0; cfg < 12; ++cfg) {
        const int rep = (cfg % 3 == 0) ? 2 : (cfg % 3 == 1 ? 4 : 8);
        const uint32_t H = (cfg / 3) % 2 == 0 ? 256u : 2048u;
        const bool per_sm = cfg >= 6;
        if (size_t(nrows + H * rep) * 128 > max_bytes) continue;
        best = 1e30f;
        for (int t = 0; t < 7; ++t) {
          CK(cudaEventRecord(e0));
          if (per_sm) {
            if (rep == 2) k_rows_zipf_rep<2, true><<<grid, 256>>>(buf, nrows, H, per_group, sink);
            else if (rep == 4) k_rows_zipf_rep<4, true><<<grid, 256>>>(buf, nrows, H, per_group, sink);
            else k_rows_zipf_rep<8, true><<<grid, 256>>>(buf, nrows, H, per_group, sink);
          } else {
            if (rep == 2) k_rows_zipf_rep<2, false><<<grid, 256>>>(buf, nrows, H, per_group, sink);
            else if (rep == 4) k_rows_zipf_rep<4, false><<<grid, 256>>>(buf, nrows, H, per_group, sink);
            else k_rows_zipf_rep<8, false><<<grid, 256>>>(buf, nrows, H, per_group, sink);
          }
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (t && ms < best) best = ms;
        }
        const double rb = double(groups) * per_group * 128.0;
        printf("rows-zipf-rep%d%s-H%u %3zu MB  %2d warps/SM  %8.1f GB/s  (%.1f G rows/s)\n", rep,
               per_sm ? "-persm" : "", H,
               bytes >> 20, c * 8, rb / best / 1e6, rb / 128.0 / best / 1e6);
      }
      if (bytes == (size_t(8) << 20)) {
        const int per_group_s = int(nidx / groups) / 8 * 8;
        for (int zc = 0; zc < 4; ++zc) {
          const int z = zc & 1, cg = zc >> 1;
          best = 1e30f;
          for (int t = 0; t < 7; ++t) {
            CK(cudaEventRecord(e0));
            if (cg) k_rows_stream<true><<<grid, 256>>>(buf, z ? d_zipf : d_uni, per_group_s, sink);
            else k_rows_stream<false><<<grid, 256>>>(buf, z ? d_zipf : d_uni, per_group_s, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (t && ms < best) best = ms;
          }
          const double rb = double(groups) * per_group_s * 128.0;
          printf("rows-stream-%s%s %3zu MB  %2d warps/SM  %8.1f GB/s  (%.1f G rows/s)\n", z ? "zipf" : "uniform",
                 cg ? "-cg" : "",
                 bytes >> 20, c * 8, rb / best / 1e6, rb / 128.0 / best / 1e6);
        }
      }
      for (int fma = 0; fma < 2; ++fma) {
        best = 1e30f;
        for (int t = 0; t < 7; ++t) {
          CK(cudaEventRecord(e0));
          if (fma) k_rows_shfl<true><<<grid, 256>>>(buf, nrows, per_group, sink);
          else k_rows_shfl<false><<<grid, 256>>>(buf, nrows, per_group, sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (t && ms < best) best = ms;
        }
        const double rb = double(groups) * per_group * 128.0;
        printf("rows-L1-shfl%s %3zu MB  %2d warps/SM  %8.1f GB/s  (%.1f G rows/s)\n", fma ? "-fma" : "",
               bytes >> 20, c * 8, rb / best / 1e6, rb / 128.0 / best / 1e6);
      }
    }
  }
  return 0;
}
