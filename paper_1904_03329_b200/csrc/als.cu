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
#include <atomic>
#include <cstdlib>
#include <string>

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


// ---------------------------------------------------------------------------
// Tensor-core variant (default).  F = Y M and the Gram F^T F are 32-wide
// GEMMs, so they run on the warp-level tensor-core path (mma.sync m16n8k8
// TF32, fp32 accumulate; measured 273 TFLOP/s on B200 vs 72 for FFMA) in
// 3xTF32 form — x = hi + lo with hi = tf32(x), lo = tf32(x - hi), and
// a·b ≈ hi·hi' + hi·lo' + lo·hi' — which keeps fp32 accuracy (dropped term
// ~2^-22 relative).  The Gram is taken from F itself, not as M^T (Y^T Y) M:
// early in ALS, M = pinv(V) is large and F = Y M cancels, and the
// algebraically equal form loses the cancellation to rounding (measured: a
// 1e-6..1e-5 fit drift on nell-2).  Each warp streams its own 16-row
// subtiles through a 3-stage cp.async ring (no CTA-wide barrier in the loop):
// F from the MMA accumulators goes to global memory and over the consumed Y
// subtile in shared memory, where the Gram MMAs read it (upper 16x8 tiles,
// fp32 in registers, flushed to per-warp fp64 every 32 subtiles); the fit
// term sum_r w_r Y[i,r] F[i,r] is accumulated alongside.  A one-CTA epilogue
// mirrors the upper tiles into the symmetric Gram.
static constexpr int MMA_WARPS = 8;
static constexpr int MMA_ROWS = 16;
static constexpr int MMA_STAGES = 3;
static constexpr int MMA_LD = ALS_R + 4;  // conflict-free fragment loads
static constexpr int MMA_FLUSH = 32;      // subtiles per fp32 -> fp64 flush
static constexpr int MMA_GT = 6;          // upper tiles (mt, nt): (0,0..3), (1,2..3)

struct AlsMmaSmem {
  alignas(16) float y[MMA_WARPS][MMA_STAGES][MMA_ROWS * MMA_LD];
  uint4 mfrag[16][32];  // (nt * 4 + ks, lane) -> {hi(b0), hi(b1), lo(b0), lo(b1)}
  double g[MMA_WARPS][MMA_GT][32][4];
  double inner[MMA_WARPS];
};

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
#ifndef HBK_TF32_SPLIT_CVT
// x = hi + lo: hi = x rounded to tf32 (round half away, integer add + mask:
// 2 instructions where cvt.rna.tf32 expands to ~6 with its special-value
// checks; finite factor values only — |x| near FLT_MAX would round to inf),
// lo = x - hi exactly (|lo| <= 2^-11 |x|, <= 12 significant bits), passed
// as-is: the tensor cores read tf32 operands by ignoring the low 13 bits,
// which drops <= 1 bit of lo (<= 2^-22 |x|), the accuracy of rounding lo too.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
#else
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = to_tf32(x);
  lo = to_tf32(x - __uint_as_float(hi));
}
#endif
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// d += a·b in 3xTF32 (small terms first)
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma_tf32(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}

// LIST: process the rows list[0..rows) (ascending ids) instead of 0..rows.
template <bool LIST>
__global__ void __launch_bounds__(MMA_WARPS * 32, 2)
    k_als_update32_mma(const float* __restrict__ Y, int64_t rows, const uint32_t* __restrict__ list,
                       const float* __restrict__ M, const float* __restrict__ colw,
                       float* __restrict__ F, double* __restrict__ gupper,
                       double* __restrict__ inner) {
  auto rid = [&](int64_t i) -> int64_t { return LIST ? int64_t(__ldg(list + i)) : i; };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AlsMmaSmem& S = *reinterpret_cast<AlsMmaSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
    const int nt = i >> 7, ks = (i >> 5) & 3, ln = i & 31, gg = ln >> 2, tt = ln & 3;
    uint32_t h0, l0, h1, l1;
    split_tf32(M[(ks * 8 + tt) * ALS_R + nt * 8 + gg], h0, l0);
    split_tf32(M[(ks * 8 + tt + 4) * ALS_R + nt * 8 + gg], h1, l1);
    S.mfrag[nt * 4 + ks][ln] = make_uint4(h0, h1, l0, l1);
  }
  for (int i = lane; i < MMA_GT * 32 * 4; i += 32) (&S.g[warp][0][0][0])[i] = 0.0;
  // fit-term column weights of this thread's accumulator columns nt*8 + 2t (+1)
  float wc[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) wc[nt][e] = colw ? colw[nt * 8 + 2 * t + e] : 1.f;
  __syncthreads();

  const int64_t nsub = (rows + MMA_ROWS - 1) / MMA_ROWS;
  const int64_t wstride = int64_t(gridDim.x) * MMA_WARPS;
  float* ring = &S.y[warp][0][0];
  auto load = [&](int64_t sub, int stage) {
    const int64_t r0 = sub * MMA_ROWS;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = lane + 32 * j, r = c >> 3, c4 = (c & 7) * 4;
      const bool ok = r0 + r < rows;
      cp16_zfill(ring + stage * (MMA_ROWS * MMA_LD) + r * MMA_LD + c4,
                 Y + (ok ? rid(r0 + r) * ALS_R + c4 : 0), ok);
    }
  };
  int64_t sub = int64_t(blockIdx.x) * MMA_WARPS + warp;
#pragma unroll
  for (int p = 0; p < MMA_STAGES - 1; ++p) {
    if (sub + p * wstride < nsub) load(sub + p * wstride, p);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float gacc[MMA_GT][4];
#pragma unroll
  for (int i = 0; i < MMA_GT; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) gacc[i][q] = 0.f;
  float in32 = 0.f;
  double in64 = 0.0;
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < MMA_GT; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        S.g[warp][i][lane][q] += double(gacc[i][q]);
        gacc[i][q] = 0.f;
      }
    in64 += double(in32);
    in32 = 0.f;
  };
  int stage = 0, since = 0;
  for (; sub < nsub; sub += wstride) {
    const int64_t pre = sub + (MMA_STAGES - 1) * wstride;
    if (pre < nsub) load(pre, (stage + MMA_STAGES - 1) % MMA_STAGES);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(MMA_STAGES - 1) : "memory");
    __syncwarp();
    float* T = ring + stage * (MMA_ROWS * MMA_LD);
    const int64_t r0 = sub * MMA_ROWS;

    // ---- F = Y M: 16 rows x 32 columns, K = 32
    float d[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) d[nt][q] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t ah[4], al[4];
      split_tf32(T[g * MMA_LD + ks * 8 + t], ah[0], al[0]);
      split_tf32(T[(g + 8) * MMA_LD + ks * 8 + t], ah[1], al[1]);
      split_tf32(T[g * MMA_LD + ks * 8 + t + 4], ah[2], al[2]);
      split_tf32(T[(g + 8) * MMA_LD + ks * 8 + t + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const uint4 b = S.mfrag[nt * 4 + ks][lane];
        mma3(d[nt], ah, al, b.x, b.y, b.z, b.w);
      }
    }
    // ---- fit term: w_c * Y[i, c] * F[i, c] at this thread's accumulator slots
    if (inner) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const float2 ya = *reinterpret_cast<const float2*>(T + g * MMA_LD + nt * 8 + 2 * t);
        const float2 yb = *reinterpret_cast<const float2*>(T + (g + 8) * MMA_LD + nt * 8 + 2 * t);
        in32 = fmaf(wc[nt][0] * ya.x, d[nt][0], in32);
        in32 = fmaf(wc[nt][1] * ya.y, d[nt][1], in32);
        in32 = fmaf(wc[nt][0] * yb.x, d[nt][2], in32);
        in32 = fmaf(wc[nt][1] * yb.y, d[nt][3], in32);
      }
    }
    __syncwarp();  // every lane has read its Y values
    // ---- F to global memory and over the Y subtile
    {
      const int64_t ra = r0 + g, rb = r0 + g + 8;
      const int64_t fa_row = ra < rows ? rid(ra) : 0, fb_row = rb < rows ? rid(rb) : 0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const float2 fa = make_float2(d[nt][0], d[nt][1]), fb = make_float2(d[nt][2], d[nt][3]);
        *reinterpret_cast<float2*>(T + g * MMA_LD + nt * 8 + 2 * t) = fa;
        *reinterpret_cast<float2*>(T + (g + 8) * MMA_LD + nt * 8 + 2 * t) = fb;
        if (ra < rows) __stcs(reinterpret_cast<float2*>(F + fa_row * ALS_R + nt * 8 + 2 * t), fa);
        if (rb < rows) __stcs(reinterpret_cast<float2*>(F + fb_row * ALS_R + nt * 8 + 2 * t), fb);
      }
    }
    __syncwarp();
    // ---- Gram += F^T F over the 16 rows (upper tiles; rows past the end are 0)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t vh[4][2], vl[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        split_tf32(T[(ks * 8 + t) * MMA_LD + nt * 8 + g], vh[nt][0], vl[nt][0]);
        split_tf32(T[(ks * 8 + t + 4) * MMA_LD + nt * 8 + g], vh[nt][1], vl[nt][1]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t ah[4] = {vh[2 * mt][0], vh[2 * mt + 1][0], vh[2 * mt][1], vh[2 * mt + 1][1]};
        const uint32_t al[4] = {vl[2 * mt][0], vl[2 * mt + 1][0], vl[2 * mt][1], vl[2 * mt + 1][1]};
#pragma unroll
        for (int nt = 2 * mt; nt < 4; ++nt) {
          const int ti = mt == 0 ? nt : 2 + nt;  // (0,0..3) -> 0..3, (1,2..3) -> 4..5
          mma3(gacc[ti], ah, al, vh[nt][0], vh[nt][1], vl[nt][0], vl[nt][1]);
        }
      }
    }
    __syncwarp();  // this stage may be refilled by the next iteration's prefetch
    if (++since == MMA_FLUSH) {
      flush();
      since = 0;
    }
    stage = (stage + 1) % MMA_STAGES;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  flush();
  if (inner) {
    double v = in64;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) S.inner[warp] = v;
  }
  __syncthreads();
  // CTA reduction of the warps' fp64 tiles -> global upper tiles
  for (int i = threadIdx.x; i < MMA_GT * 32 * 4; i += blockDim.x) {
    const int ti = i >> 7, ln = (i >> 2) & 31, q = i & 3;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < MMA_WARPS; ++w) v += S.g[w][ti][ln][q];
    const int mt = ti < 4 ? 0 : 1, nt = ti < 4 ? ti : ti - 2;
    const int row = 16 * mt + (ln >> 2) + (q >= 2 ? 8 : 0), col = 8 * nt + 2 * (ln & 3) + (q & 1);
    atomicAdd(gupper + row * ALS_R + col, v);
  }
  if (inner && threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < MMA_WARPS; ++w) v += S.inner[w];
    atomicAdd(inner, v);
  }
}

// ------------------------------------------------ tcgen05 (5th-gen tensor core)
// The same update on the sm_100 tensor cores, software-pipelined inside one
// CTA of 128 threads per SM (thread r = tile row r), 128-row tiles streamed
// through a 4-stage cp.async ring.  Per tile k:
//   1. (one tile ahead) tile k+1 lands in shared memory as the K-major,
//      128-byte-swizzled A operand (row r at 128 r bytes, 16-byte chunk c at
//      c ^ r%8); thread r splits its row in place into tf32 hi and writes lo
//      to a second buffer at the same offsets; one thread issues
//      F(k+1) = Ylo·Mhi + Yhi·Mlo + Yhi·Mhi (tcgen05.mma kind::tf32, M = 128,
//      N = 32, twelve K = 8 instructions) into the other of two TMEM
//      accumulators and commits to an mbarrier;
//   2. thread r reads F(k) row r (tcgen05.ld 32x32b.x32), adds its fit term,
//      stages the row in the consumed ring slot for a coalesced store, and
//      writes Fᵀ split into hi/lo as the K-major operand of the Gram (four
//      8-KB K-blocks of 32 tile rows: rows 0-31 = Fhiᵀ, 32-63 = Floᵀ; double-
//      buffered against the previous tile's Gram MMAs);
//   3. one thread issues D (+)= [Fhiᵀ; Floᵀ]·Fhi over the tile's rows (sixteen
//      M = 128 instructions whose rows 64-127 read the neighbouring block and
//      are ignored — kind::tf32 takes no MN-major operands,
//      scripts/umma_probe.cu), so G = D[0:32] + X + Xᵀ with X = D[32:64] =
//      FloᵀFhi (3xTF32; FloᵀFlo ~2^-22 dropped).  D accumulates in TMEM over
//      TC_FLUSH tiles, then warps 0-1 add it into fp64 rows in shared memory.
// Y and F cross HBM once each.
static constexpr int TC_ROWS = 128;
static constexpr int TC_STAGES = 4;
static constexpr int TC_FLUSH = 4;  // tiles per fp32 -> fp64 Gram flush (512 rows, as the mma.sync path)

struct AlsTcSmem {
  alignas(1024) uint32_t ring[TC_STAGES][TC_ROWS * ALS_R];  // Y (swizzled) -> tf32 hi -> F staging
  uint32_t fg[2][4][2 * ALS_R * ALS_R];  // Gram operand blocks (swizzled), double-buffered
  uint32_t lo[2][TC_ROWS * ALS_R];       // must follow fg: the last block's rows 64-127 read it
  uint32_t mhi[ALS_R * ALS_R];           // M^T hi / lo, K-major without swizzle
  uint32_t mlo[ALS_R * ALS_R];
  double g[2 * ALS_R][ALS_R];
  float w[ALS_R];
  double inner[TC_ROWS / 32];
  unsigned long long bar_f[2], bar_g[2];
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// UMMA shared-memory descriptor: start, LBO, SBO (bytes), version 1, layout
// (0 = no swizzle, 2 = 128-byte swizzle)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}
// instruction descriptor kind::tf32: D f32, A/B tf32 K-major, N = 32, M = 128
static constexpr uint32_t UMMA_ID_TF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) |
                                         ((128u >> 4) << 24);
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(UMMA_ID_TF32), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 24)) __trap();  // a lost commit must not hang the GPU
  }
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <bool LIST>
__global__ void __launch_bounds__(TC_ROWS, 1)
    k_als_update32_tc(const float* __restrict__ Y, int64_t rows, const uint32_t* __restrict__ list,
                      const float* __restrict__ M, const float* __restrict__ colw,
                      float* __restrict__ F, double* __restrict__ gram, double* __restrict__ inner) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  AlsTcSmem& S = *reinterpret_cast<AlsTcSmem*>(
      smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B operand of F: element (j, k) = M[k][j], K-major without swizzle (core
  // matrices of 8 j x 4 k; LBO 512 B between k-chunks, SBO 128 B between j-groups)
  for (int i = t; i < ALS_R * ALS_R; i += TC_ROWS) {
    const int k = i >> 5, j = i & 31;
    uint32_t hi, lo;
    split_tf32(M[i], hi, lo);
    const int o = (j & 7) * 4 + (j >> 3) * 32 + (k & 3) + (k >> 2) * 128;
    S.mhi[o] = hi;
    S.mlo[o] = lo;
  }
  for (int i = t; i < 2 * ALS_R * ALS_R; i += TC_ROWS) (&S.g[0][0])[i] = 0.0;
  if (t < ALS_R) S.w[t] = colw ? colw[t] : 1.f;
  if (t == 0) {
    for (int j = 0; j < 2; ++j) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar_f[j])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar_g[j])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(&S.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem, tmem_g = tmem + 64;  // F accumulators at columns 0 / 32
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const uint32_t a_mhi = smem_u32(S.mhi), a_mlo = smem_u32(S.mlo);

  const int64_t ntiles = (rows + TC_ROWS - 1) / TC_ROWS;
  const int64_t G = gridDim.x, first = blockIdx.x;
  const int64_t count = first < ntiles ? (ntiles - 1 - first) / G + 1 : 0;  // this CTA's tiles
  // k-th tile -> ring slot k % TC_STAGES: coalesced 16-byte copies (a warp
  // moves four whole rows per instruction) to their swizzled places
  auto load = [&](int64_t k) {
    if (k >= count) return;
    uint32_t* dst = S.ring[k % TC_STAGES];
    const int64_t r0 = (first + k * G) * TC_ROWS;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = t + TC_ROWS * j, r = i >> 3, c = i & 7;
      const bool ok = r0 + r < rows;
      const int64_t rid = ok ? (LIST ? int64_t(__ldg(list + r0 + r)) : r0 + r) : 0;
      cp16_zfill(reinterpret_cast<float*>(dst + r * 32 + ((c ^ (r & 7)) << 2)), Y + rid * ALS_R + c * 4, ok);
    }
  };
  // split tile k (its ring slot has landed) and issue F(k) into accumulator k % 2
  auto stage_f = [&](int64_t k, float (&yv)[32]) {
    asm volatile("cp.async.wait_group %0;" ::"n"(TC_STAGES - 2) : "memory");
    __syncthreads();
    uint32_t* yt = S.ring[k % TC_STAGES];
    uint32_t* lt = S.lo[k & 1];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int o = t * 32 + ((c ^ (t & 7)) << 2);
      const uint4 x = *reinterpret_cast<const uint4*>(yt + o);
      uint4 h, l;
      split_tf32(__uint_as_float(x.x), h.x, l.x);
      split_tf32(__uint_as_float(x.y), h.y, l.y);
      split_tf32(__uint_as_float(x.z), h.z, l.z);
      split_tf32(__uint_as_float(x.w), h.w, l.w);
      *reinterpret_cast<uint4*>(yt + o) = h;
      *reinterpret_cast<uint4*>(lt + o) = l;
      yv[4 * c] = __uint_as_float(x.x);
      yv[4 * c + 1] = __uint_as_float(x.y);
      yv[4 * c + 2] = __uint_as_float(x.z);
      yv[4 * c + 3] = __uint_as_float(x.w);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
      const uint32_t ahi = smem_u32(yt), alo = smem_u32(lt), d = tmem + uint32_t(k & 1) * 32;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t ah = umma_desc(ahi + s * 32, 16, 1024, 2);
        const uint64_t al = umma_desc(alo + s * 32, 16, 1024, 2);
        const uint64_t bh = umma_desc(a_mhi + s * 1024, 512, 128, 0);
        const uint64_t bl = umma_desc(a_mlo + s * 1024, 512, 128, 0);
        umma_tf32(d, al, bh, s > 0);
        umma_tf32(d, ah, bl, 1);
        umma_tf32(d, ah, bh, 1);
      }
      umma_commit(smem_u32(&S.bar_f[k & 1]));
    }
  };

#pragma unroll
  for (int p = 0; p < TC_STAGES - 1; ++p) {
    load(p);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float yn[32];
  if (count > 0) stage_f(0, yn);
  float in32 = 0.f;
  double in64 = 0.0;
  int since = 0;
  for (int64_t k = 0; k < count; ++k) {
    float yv[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) yv[c] = yn[c];
    load(k + TC_STAGES - 1);  // the slot of tile k-1 (its F MMA and F store are done)
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (k + 1 < count) stage_f(k + 1, yn);  // overlaps F(k)'s MMAs
    // F(k): fit term, staging for the coalesced store, F^T hi/lo for the Gram
    mbar_wait(smem_u32(&S.bar_f[k & 1]), uint32_t(k >> 1) & 1);
    tc_fence_after();
    float f[32];
    tmem_ld32(tmem + uint32_t(k & 1) * 32 + lane_base, f);
    if (inner) {
#pragma unroll
      for (int c = 0; c < 32; ++c) in32 = fmaf(S.w[c] * yv[c], f[c], in32);
    }
    uint32_t* stg = S.ring[k % TC_STAGES];  // F(k) has consumed this slot's hi
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(stg + t * 32 + ((q ^ (t & 7)) << 2)) =
          make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
    if (k >= 2) mbar_wait(smem_u32(&S.bar_g[k & 1]), uint32_t((k - 2) >> 1) & 1);  // Gram(k-2) read fg[k%2]
    {
      // block = warp (tile rows 32w..32w+31 are its K range), row c (hi) / 32 + c (lo),
      // K position = lane: chunk lane/4 swizzled with c % 8
      uint32_t* blk = S.fg[k & 1][warp];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t hi, lo;
        split_tf32(f[c], hi, lo);
        const int o = (((lane >> 2) ^ (c & 7)) << 2) + (lane & 3);
        blk[c * 32 + o] = hi;
        blk[(ALS_R + c) * 32 + o] = lo;
      }
    }
    tc_fence_before();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
      const uint32_t a_fg = smem_u32(&S.fg[k & 1][0][0]);
#pragma unroll
      for (int s = 0; s < TC_ROWS / 8; ++s) {
        const uint64_t d = umma_desc(a_fg + (s >> 2) * 8192 + (s & 3) * 32, 16, 1024, 2);
        umma_tf32(tmem_g, d, d, (since > 0 || s > 0) ? 1u : 0u);
      }
      umma_commit(smem_u32(&S.bar_g[k & 1]));
    }
    // coalesced F store: a warp writes four whole rows per instruction
    {
      const int64_t r0 = (first + k * G) * TC_ROWS;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = t + TC_ROWS * j, r = i >> 3, c = i & 7;
        if (r0 + r < rows) {
          const int64_t rid = LIST ? int64_t(__ldg(list + r0 + r)) : r0 + r;
          __stcs(reinterpret_cast<float4*>(F + rid * ALS_R + c * 4),
                 *reinterpret_cast<const float4*>(stg + r * 32 + ((c ^ (r & 7)) << 2)));
        }
      }
    }
    if (++since == TC_FLUSH || k + 1 == count) {
      mbar_wait(smem_u32(&S.bar_g[k & 1]), uint32_t(k >> 1) & 1);
      tc_fence_after();
      if (warp < 2) {
        float d[32];
        tmem_ld32(tmem_g + lane_base, d);
#pragma unroll
        for (int c = 0; c < 32; ++c) S.g[t][c] += double(d[c]);
      }
      tc_fence_before();
      in64 += double(in32);
      in32 = 0.f;
      since = 0;
    }
    __syncthreads();  // the staged F rows are read before the slot is refilled
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  in64 += double(in32);
  if (inner) {
    double v = in64;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) S.inner[warp] = v;
  }
  __syncthreads();
  // G = D0 + X + X^T (D0 = rows 0-31, X = rows 32-63 of S.g)
  if (count > 0)
    for (int i = t; i < ALS_R * ALS_R; i += TC_ROWS) {
      const int r = i >> 5, c = i & 31;
      atomicAdd(gram + i, S.g[r][c] + S.g[ALS_R + r][c] + S.g[ALS_R + c][r]);
    }
  if (inner && t == 0) atomicAdd(inner, S.inner[0] + S.inner[1] + S.inner[2] + S.inner[3]);
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// The Gram holds the upper 16x8 tiles, which cover every r <= c; mirror the
// upper triangle (the diagonal tiles computed both (r, c) and (c, r), which
// may differ in the last bit) so the result is exactly symmetric.
__global__ void __launch_bounds__(1024) k_als_mirror(double* __restrict__ gram) {
  __shared__ double G[ALS_R][ALS_R + 1];
  const int r = threadIdx.x >> 5, c = threadIdx.x & 31;
  G[r][c] = gram[r * ALS_R + c];
  __syncthreads();
  gram[r * ALS_R + c] = r <= c ? G[r][c] : G[c][r];
}

template <bool LIST>
static void launch_als_tc(const float* Y, const uint32_t* list, int64_t n, const float* M,
                          const float* colw, float* F, double* gram, double* inner, cudaStream_t st) {
  HBK_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * ALS_R * ALS_R, st));
  if (inner) HBK_CUDA(cudaMemsetAsync(inner, 0, sizeof(double), st));
  if (n == 0) return;
  int dev = 0, sms = 0;
  HBK_CUDA(cudaGetDevice(&dev));
  HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t bytes = sizeof(AlsTcSmem) + 1024;  // + alignment slack
  static std::atomic<int> occ[64];
  int per_sm = dev < 64 ? occ[dev].load(std::memory_order_relaxed) : 0;
  if (per_sm == 0) {
    HBK_CUDA(cudaFuncSetAttribute(k_als_update32_tc<LIST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(bytes)));
    HBK_CUDA(cudaFuncSetAttribute(k_als_update32_tc<LIST>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  int(cudaSharedmemCarveoutMaxShared)));
    HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_update32_tc<LIST>, TC_ROWS,
                                                           bytes));
    per_sm = std::max(per_sm, 1);
    if (dev < 64) occ[dev].store(per_sm, std::memory_order_relaxed);
  }
  const int64_t ntiles = (n + TC_ROWS - 1) / TC_ROWS;
  const int grid = int(std::min<int64_t>(ntiles, int64_t(sms) * per_sm));
  k_als_update32_tc<LIST><<<grid, TC_ROWS, bytes, st>>>(Y, n, list, M, colw, F, gram, inner);
  check_launch("k_als_update32_tc");
  k_als_mirror<<<1, 1024, 0, st>>>(gram);
  check_launch("k_als_mirror");
}

// HBK_ALS_KERNEL = mma (default: mma.sync 3xTF32) | tc (tcgen05) | fma (FFMA),
// read per call so one process can A/B them.  Measured at nell-1 row counts
// (scripts/als_kernel_bench.py, profiles/r2s7/als_tc.md): mma 0.21 / 0.16 /
// 1.71 ms, tc 0.41 / 0.31 / 3.48 ms — the tcgen05 kernel is correct (same
// tests) but issue-bound: one CTA of four warps per SM spends 1,190
// instructions per warp per tile, most of them transposing F for the Gram.
static int als_kernel_choice() {
  const char* e = getenv("HBK_ALS_KERNEL");
  if (e && std::string(e) == "fma") return 2;
  if (e && std::string(e) == "tc") return 0;
  return 1;
}

// Tensor-core update over rows 0..n (or list[0..n)): Gram upper tiles and the
// fit term accumulate in gram / inner (zeroed here), then the Gram is mirrored.
template <bool LIST>
static void launch_als_mma(const float* Y, const uint32_t* list, int64_t n, const float* M,
                           const float* colw, float* F, double* gram, double* inner,
                           cudaStream_t st) {
  HBK_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * ALS_R * ALS_R, st));
  if (inner) HBK_CUDA(cudaMemsetAsync(inner, 0, sizeof(double), st));
  if (n == 0) return;
  int dev = 0, sms = 0;
  HBK_CUDA(cudaGetDevice(&dev));
  HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // per-device launch setup, done once (concurrent first calls just repeat
  // the idempotent attribute call)
  static std::atomic<int> occ[64];
  int per_sm = dev < 64 ? occ[dev].load(std::memory_order_relaxed) : 0;
  if (per_sm == 0) {
    HBK_CUDA(cudaFuncSetAttribute(k_als_update32_mma<LIST>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(AlsMmaSmem))));
    HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_update32_mma<LIST>,
                                                           MMA_WARPS * 32, sizeof(AlsMmaSmem)));
    per_sm = std::max(per_sm, 1);
    if (dev < 64) occ[dev].store(per_sm, std::memory_order_relaxed);
  }
  const int64_t nsub = (n + MMA_ROWS - 1) / MMA_ROWS;
  const int grid = int(std::min<int64_t>((nsub + MMA_WARPS - 1) / MMA_WARPS, int64_t(sms) * per_sm));
  k_als_update32_mma<LIST><<<grid, MMA_WARPS * 32, sizeof(AlsMmaSmem), st>>>(Y, n, list, M, colw,
                                                                              F, gram, inner);
  check_launch("k_als_update32_mma");
  k_als_mirror<<<1, 1024, 0, st>>>(gram);
  check_launch("k_als_mirror");
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
    int dev = 0, sms = 0, per_sm = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int kernel = als_kernel_choice();
    if (kernel == 0) {
      launch_als_tc<false>(Y, nullptr, rows, M, colw, F, gram, inner, st);
      return;
    }
    if (kernel == 1) {
      launch_als_mma<false>(Y, nullptr, rows, M, colw, F, gram, inner, st);
      return;
    }
    HBK_CUDA(cudaMemsetAsync(gram, 0, sizeof(double) * ALS_R * ALS_R, st));
    if (inner) HBK_CUDA(cudaMemsetAsync(inner, 0, sizeof(double), st));
    if (rows == 0) return;
    HBK_CUDA(cudaFuncSetAttribute(k_als_update32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(AlsSmem))));
    HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_update32, ALS_TILE,
                                                           sizeof(AlsSmem)));
    const int64_t ntiles = (rows + ALS_TILE - 1) / ALS_TILE;
    const int grid = int(std::min<int64_t>(ntiles, int64_t(sms) * std::max(per_sm, 1)));
    k_als_update32<<<grid, ALS_TILE, sizeof(AlsSmem), st>>>(Y, rows, M, colw, F, gram, inner);
    check_launch("k_als_update32");
  });
}

extern "C" int hbk_als_update_rows(const float* Y, const uint32_t* list, int64_t nlist, int rank,
                                   const float* M, const float* colw, float* F, double* gram,
                                   double* inner, void* stream) {
  return guarded([&] {
    HBK_REQUIRE(rank == ALS_R, HBK_EINVAL, "hbk_als_update_rows supports rank 32");
    HBK_REQUIRE(nlist >= 0, HBK_EINVAL, "negative row count");
    HBK_REQUIRE(nlist == 0 || list, HBK_EINVAL, "null row list");
    HBK_REQUIRE((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(F)) % 16 == 0,
                HBK_EINVAL, "Y and F must be 16-byte aligned");
    if (als_kernel_choice() == 0)
      launch_als_tc<true>(Y, list, nlist, M, colw, F, gram, inner, to_stream(stream));
    else
      launch_als_mma<true>(Y, list, nlist, M, colw, F, gram, inner, to_stream(stream));
  });
}
