// CP-ALS row update on sm_100a (cpd.py:157-195).
//
// After a mode's MTTKRP the reference computes F = Y · pinv(V) (cpd.py:172),
// then G = FᵀF (cpd.py:39-42), and — for the last mode of a sweep — the fit
// term <Y, F> (cpd.py:176-184).  On a row shard all three are row-local, so
// one pass over the rows does them: a CTA stages a tile of 256 rows of Y in
// shared memory, each thread turns its row into F (32x32 matrix M broadcast
// from shared memory), the tile of F is written back coalesced and reduced
// into the CTA's Gram partial (register-blocked 4x4 per thread, fp32 within a
// tile, fp64 across tiles), and sum_r w_r <Y[:, r], F[:, r]> is accumulated
// alongside (w: column weights of Y, e.g. factor column scales; NULL = 1).  Y and F are
// read/written once: the pass is HBM-bound (8 bytes per row element).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace hbk {

static constexpr int ALS_R = 32;
static constexpr int ALS_TILE = 256;  // rows per tile = threads per CTA
static constexpr int ALS_LD = ALS_R + 1;

__global__ void __launch_bounds__(ALS_TILE, 2)
    k_als_update32(const float* __restrict__ Y, int64_t rows, const float* __restrict__ M,
                   const float* __restrict__ colw, float* __restrict__ F, double* __restrict__ gram,
                   double* __restrict__ inner) {
  __shared__ float Ms[ALS_R * ALS_R];
  __shared__ float W[ALS_R];
  __shared__ float T[ALS_TILE * ALS_LD];
  __shared__ double red[ALS_TILE / 32];
  const int tid = threadIdx.x;
  for (int i = tid; i < ALS_R * ALS_R; i += ALS_TILE) Ms[i] = M[i];
  if (tid < ALS_R) W[tid] = colw ? colw[tid] : 1.f;
  // Gram blocking: 4 row groups x 64 threads, each thread a 4x4 block of G
  const int grp = tid >> 6, p = tid & 63;
  const int a0 = (p >> 3) * 4, b0 = (p & 7) * 4;
  double g64[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) g64[q] = 0.0;
  double in64 = 0.0;
  const int64_t ntiles = (rows + ALS_TILE - 1) / ALS_TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * ALS_TILE;
    const int nr = int(rows - r0 < ALS_TILE ? rows - r0 : int64_t(ALS_TILE));
    __syncthreads();  // previous tile's Gram reads are done
    // coalesced load of the Y tile (rows beyond the end are zero)
    const float* src = Y + r0 * ALS_R;
    for (int i = tid; i < ALS_TILE * ALS_R; i += ALS_TILE) {
      const int r = i / ALS_R, c = i % ALS_R;
      T[r * ALS_LD + c] = r < nr ? __ldcs(src + i) : 0.f;
    }
    __syncthreads();
    // row `tid`: f = y M
    float y[ALS_R], f[ALS_R];
#pragma unroll
    for (int k = 0; k < ALS_R; ++k) {
      y[k] = T[tid * ALS_LD + k];
      f[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < ALS_R; ++k) {
      const float4* mk = reinterpret_cast<const float4*>(Ms + k * ALS_R);
#pragma unroll
      for (int c4 = 0; c4 < ALS_R / 4; ++c4) {
        const float4 m = mk[c4];
        f[4 * c4 + 0] = fmaf(y[k], m.x, f[4 * c4 + 0]);
        f[4 * c4 + 1] = fmaf(y[k], m.y, f[4 * c4 + 1]);
        f[4 * c4 + 2] = fmaf(y[k], m.z, f[4 * c4 + 2]);
        f[4 * c4 + 3] = fmaf(y[k], m.w, f[4 * c4 + 3]);
      }
    }
    if (inner) {
      float d = 0.f;
#pragma unroll
      for (int c = 0; c < ALS_R; ++c) d = fmaf(W[c] * y[c], f[c], d);
      in64 += double(d);
    }
    __syncthreads();  // every row of Y has been read
#pragma unroll
    for (int c = 0; c < ALS_R; ++c) T[tid * ALS_LD + c] = f[c];
    __syncthreads();
    // coalesced store of the F tile
    float* dst = F + r0 * ALS_R;
    for (int i = tid; i < nr * ALS_R; i += ALS_TILE) dst[i] = T[(i / ALS_R) * ALS_LD + i % ALS_R];
    // Gram partial of the tile
    float g32[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) g32[q] = 0.f;
    for (int r = grp; r < ALS_TILE; r += 4) {
      const float* row = T + r * ALS_LD;
      float av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = row[a0 + u];
        bv[u] = row[b0 + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) g32[u * 4 + v] = fmaf(av[u], bv[v], g32[u * 4 + v]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) g64[q] += double(g32[q]);
  }
  // CTA reduction: the 4 row groups' partials through shared memory (reuse T
  // as doubles: 4 x 64 threads x 16 values = 16384 doubles > T, so go in two
  // passes of 8 values)
  __syncthreads();
  double* S = reinterpret_cast<double*>(T);  // 256 * 33 floats = 4224 doubles
#pragma unroll
  for (int half = 0; half < 2; ++half) {
#pragma unroll
    for (int q = 0; q < 8; ++q) S[(q * 4 + grp) * 64 + p] = g64[half * 8 + q];
    __syncthreads();
    if (grp == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double v = S[(q * 4 + 0) * 64 + p] + S[(q * 4 + 1) * 64 + p] +
                         S[(q * 4 + 2) * 64 + p] + S[(q * 4 + 3) * 64 + p];
        const int qq = half * 8 + q, u = qq >> 2, w = qq & 3;
        atomicAdd(gram + (a0 + u) * ALS_R + (b0 + w), v);
      }
    }
    __syncthreads();
  }
  if (inner) {
    double v = in64;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int i = 0; i < ALS_TILE / 32; ++i) s += red[i];
      atomicAdd(inner, s);
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
    cudaStream_t st = to_stream(stream);
    HBK_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * ALS_R * ALS_R, st));
    if (inner) HBK_CUDA(cudaMemsetAsync(inner, 0, sizeof(double), st));
    if (rows == 0) return;
    int dev = 0, sms = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t ntiles = (rows + ALS_TILE - 1) / ALS_TILE;
    const int grid = int(std::min<int64_t>(ntiles, int64_t(sms) * 2));
    k_als_update32<<<grid, ALS_TILE, 0, st>>>(Y, rows, M, colw, F, gram, inner);
    check_launch("k_als_update32");
  });
}
