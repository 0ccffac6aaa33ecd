// CP-ALS row update on sm_100a (cpd.py:157-195).
//
// After a mode's MTTKRP the reference computes F = Y · pinv(V) (cpd.py:172),
// then G = FᵀF (cpd.py:39-42), and — for the last mode of a sweep — the fit
// term <Y, F> (cpd.py:176-184).  On a row shard all three are row-local, so
// one pass over the rows does them.  Per tile of 256 rows a CTA
//   1. has the Y tile in shared memory (cp.async, double-buffered: the next
//      tile streams in while this one is computed),
//   2. computes the F tile, register-blocked 4 rows x 8 columns per thread
//      (M broadcast from shared memory as LDS.128), and the column-weighted
//      sum_r w_r <Y[:, r], F[:, r]> alongside (w: factor column scales),
//   3. writes the F tile over the consumed Y tile, stores it coalesced, and
//      reduces it into the CTA's Gram partial, register-blocked 8x8 per
//      thread (fp32 over <= 32 tiles, then fp64 in shared memory; the
//      sequential per-group flush beats fp64 shared atomics, which are CAS
//      loops on sm_100).
// Y and F cross HBM once each (8 bytes per row element).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace hbk {

static constexpr int ALS_R = 32;
static constexpr int ALS_TILE = 256;       // rows per tile = threads per CTA
static constexpr int ALS_LD = ALS_R + 4;   // 16-byte aligned rows (cp.async / LDS.128)

struct AlsSmem {
  alignas(16) float buf[2][ALS_TILE * ALS_LD];  // Y tile t (then its F tile), Y tile t+1
  float Ms[ALS_R * ALS_R];
  float W[ALS_R];
  double G[ALS_R * ALS_R];
  double red[ALS_TILE / 32];
};

__device__ __forceinline__ void cp16_zfill(float* smem, const float* gmem, bool valid) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}

// Row r of a tile lives in buffer row r; thread (rb = tid/4, cb = tid%4)
// computes rows rb + 64 i (i < 4) x columns 8cb..8cb+7, so the eight row
// blocks of a warp read eight distinct banks (row stride 36 words).
__global__ void __launch_bounds__(ALS_TILE, 2)
    k_als_update32(const float* __restrict__ Y, int64_t rows, const float* __restrict__ M,
                   const float* __restrict__ colw, float* __restrict__ F, double* __restrict__ gram,
                   double* __restrict__ inner) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AlsSmem& S = *reinterpret_cast<AlsSmem*>(smem_raw);
  const int tid = threadIdx.x;
  for (int i = tid; i < ALS_R * ALS_R; i += ALS_TILE) {
    S.Ms[i] = M[i];
    S.G[i] = 0.0;
  }
  if (tid < ALS_R) S.W[tid] = colw ? colw[tid] : 1.f;
  const int rb = tid >> 2, cb = tid & 3;
  // Gram: the 10 upper-triangular 8x8 blocks (A <= B) x 25 row groups; the
  // lower triangle is mirrored at the end (threads 250..255 idle here)
  constexpr int NGB = 10, NRG = 25;
  const int gp = tid % NGB, grp = tid / NGB;
  const bool gram_thread = grp < NRG;
  int A = 0, B = gp;  // gp -> (A, B): 0..3 -> (0,0..3), 4..6 -> (1,1..3), 7,8 -> (2,2..3), 9 -> (3,3)
  if (gp >= 4) { A = 1; B = gp - 3; }
  if (gp >= 7) { A = 2; B = gp - 5; }
  if (gp >= 9) { A = 3; B = 3; }
  const int ga = A * 8, gb = B * 8;
  double in64 = 0.0;
  constexpr int FLUSH = 32;
  float g32[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) g32[q] = 0.f;
  auto flush = [&]() {
    for (int g = 0; g < NRG; ++g) {
      if (grp == g && gram_thread) {
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          S.G[(ga + (q >> 3)) * ALS_R + gb + (q & 7)] += double(g32[q]);
          g32[q] = 0.f;
        }
      }
      __syncthreads();
    }
  };
  // async load of tile `tile` into buffer b (rows past the end zero-filled)
  auto load = [&](int64_t tile, int b) {
    const int64_t r0 = tile * ALS_TILE;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i4 = tid + ALS_TILE * j, r = i4 >> 3, c = (i4 & 7) * 4;
      const bool ok = r0 + r < rows;
      cp16_zfill(S.buf[b] + r * ALS_LD + c, Y + (ok ? (r0 + r) * ALS_R + c : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int64_t ntiles = (rows + ALS_TILE - 1) / ALS_TILE;
  int since = 0, cur = 0;
  if (int64_t(blockIdx.x) < ntiles) load(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * ALS_TILE;
    const int nr = int(rows - r0 < ALS_TILE ? rows - r0 : int64_t(ALS_TILE));
    __syncthreads();  // buffer cur^1 (the previous tile's F) is no longer read
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) load(next, cur ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    float* T = S.buf[cur];
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
#pragma unroll 4
    for (int k = 0; k < ALS_R; ++k) {
      float yv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) yv[i] = T[(rb + 64 * i) * ALS_LD + k];
      const float4 m0 = reinterpret_cast<const float4*>(S.Ms + k * ALS_R + 8 * cb)[0];
      const float4 m1 = reinterpret_cast<const float4*>(S.Ms + k * ALS_R + 8 * cb)[1];
      const float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] = fmaf(yv[i], mv[c], acc[i][c]);
    }
    if (inner) {
      float d = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4* yr = reinterpret_cast<const float4*>(T + (rb + 64 * i) * ALS_LD + 8 * cb);
        const float4 y0 = yr[0], y1 = yr[1];
        const float yv[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) d = fmaf(S.W[8 * cb + c] * yv[c], acc[i][c], d);
      }
      in64 += double(d);
    }
    __syncthreads();  // every element of the Y tile has been read
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float4* fr = reinterpret_cast<float4*>(T + (rb + 64 * i) * ALS_LD + 8 * cb);
      fr[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      fr[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
    __syncthreads();
    float4* dst = reinterpret_cast<float4*>(F + r0 * ALS_R);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i4 = tid + ALS_TILE * j, r = i4 >> 3;
      if (r < nr) __stcs(dst + i4, reinterpret_cast<const float4*>(T + r * ALS_LD)[i4 & 7]);
    }
#pragma unroll 2
    for (int r = gram_thread ? grp : ALS_TILE; r < ALS_TILE; r += NRG) {
      const float4* row = reinterpret_cast<const float4*>(T + r * ALS_LD);
      const float4 a0 = row[ga / 4], a1 = row[ga / 4 + 1], b0 = row[gb / 4], b1 = row[gb / 4 + 1];
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) g32[u * 8 + v] = fmaf(av[u], bv[v], g32[u * 8 + v]);
    }
    if (++since == FLUSH) {
      flush();
      since = 0;
    }
    cur ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  flush();
  __syncthreads();
  for (int i = tid; i < ALS_R * ALS_R; i += ALS_TILE) {
    const int a = i / ALS_R, b = i % ALS_R;
    // upper-triangle blocks hold the sums; mirror the strictly-lower blocks
    atomicAdd(gram + i, (a / 8) <= (b / 8) ? S.G[i] : S.G[b * ALS_R + a]);
  }
  if (inner) {
    double v = in64;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((tid & 31) == 0) S.red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double s2 = 0.0;
      for (int i = 0; i < ALS_TILE / 32; ++i) s2 += S.red[i];
      atomicAdd(inner, s2);
    }
  }
}

}  // namespace hbk

using namespace hbk;

extern "C" int hbk_als_update(const float* Y, int64_t rows, int rank, const float* M,
                              const float* colw, float* F, double* gram, double* inner,
                              void* stream) {
  return guarded([&] {
    HBK_REQUIRE(rank == ALS_R, HBK_EINVAL, "hbk_als_update supports rank 32");
    HBK_REQUIRE(rows >= 0, HBK_EINVAL, "negative row count");
    HBK_REQUIRE((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(F)) % 16 == 0,
                HBK_EINVAL, "Y and F must be 16-byte aligned");
    cudaStream_t st = to_stream(stream);
    HBK_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * ALS_R * ALS_R, st));
    if (inner) HBK_CUDA(cudaMemsetAsync(inner, 0, sizeof(double), st));
    if (rows == 0) return;
    HBK_CUDA(cudaFuncSetAttribute(k_als_update32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(AlsSmem))));
    int dev = 0, sms = 0, per_sm = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_update32, ALS_TILE,
                                                           sizeof(AlsSmem)));
    const int64_t ntiles = (rows + ALS_TILE - 1) / ALS_TILE;
    const int grid = int(std::min<int64_t>(ntiles, int64_t(sms) * std::max(per_sm, 1)));
    k_als_update32<<<grid, ALS_TILE, sizeof(AlsSmem), st>>>(Y, rows, M, colw, F, gram, inner);
    check_launch("k_als_update32");
  });
}
