// tcgen05.mma kind::tf32 (M = 128, N = 32, four K = 8 steps) per variant of the
// shared-memory operand layout, against a host reference — used to pin the
// descriptor conventions of csrc/als.cu's tensor-core row update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_probe scripts/umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}
__host__ __device__ constexpr uint32_t idesc(uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) | (b_mn << 16) | ((32u >> 3) << 17) |
         ((128u >> 4) << 24);
}

// variant: 0 A,B K-major; 1 A,B MN-major (SBO = MN-group stride, LBO = K-group);
// 2 MN-major with LBO/SBO swapped; 3 A,B K-major 128B swizzle (K-steps advance
// the start address by 32 B inside the swizzle atom).  Measured on B200: 0 and
// 3 exact; 1 and 2 return zeros (no MN-major operands for kind::tf32).
// A is 128 x 32 (m, k), B is 32 x 32 (n, k); D[m][n] = sum_k A[m][k] B[n][k]
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  __shared__ __align__(1024) uint32_t sa[128 * 32];
  __shared__ __align__(1024) uint32_t sb[32 * 32];
  __shared__ unsigned long long bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x;
  for (int i = t; i < 128 * 32; i += 128) sa[i] = 0;
  for (int i = t; i < 32 * 32; i += 128) sb[i] = 0;
  __syncthreads();
  // place element (m, k) of an operand with `rows` MN entries
  auto place = [&](uint32_t* s, int rows, int m, int k, float v) {
    int off;  // in 4-byte words
    if (variant == 0) {  // K-major, no swizzle: LBO (k-chunk) = rows*16 B, SBO (8-row group) = 128 B
      off = (m % 8) * 4 + (m / 8) * 32 + (k % 4) + (k / 4) * rows * 4;
    } else if (variant == 1 || variant == 2) {  // MN-major: (m%4) + (k%8)*4 + (m/4)*SBO + (k/8)*LBO
      off = (m % 4) + (k % 8) * 4 + (m / 4) * 32 + (k / 8) * rows * 8;  // MN groups 128 B apart
    } else {  // K-major 128B swizzle: row m at 128 B, 16-B chunk c ^ (m % 8)
      const int c = k / 4;
      off = m * 32 + ((c ^ (m % 8)) * 4) + (k % 4);
    }
    s[off] = __float_as_uint(v);
  };
  for (int i = t; i < 128 * 32; i += 128) place(sa, 128, i / 32, i % 32, A[i]);
  for (int i = t; i < 32 * 32; i += 128) place(sb, 32, i / 32, i % 32, B[i]);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tm;
  if (t == 0) {
    for (int st = 0; st < 4; ++st) {
      uint64_t da, db;
      uint32_t id;
      if (variant == 0) {  // k-chunk stride rows*16 B: a step is two chunks
        da = desc(smem_u32(sa) + st * 2 * 128 * 16, 128 * 16, 128, 0);
        db = desc(smem_u32(sb) + st * 2 * 32 * 16, 32 * 16, 128, 0);
        id = idesc(0, 0);
      } else if (variant == 1) {
        da = desc(smem_u32(sa) + st * 128 * 32, 4096, 128, 0);
        db = desc(smem_u32(sb) + st * 32 * 32, 1024, 128, 0);
        id = idesc(1, 1);
      } else if (variant == 2) {
        da = desc(smem_u32(sa) + st * 128 * 32, 128, 4096, 0);
        db = desc(smem_u32(sb) + st * 32 * 32, 128, 1024, 0);
        id = idesc(1, 1);
      } else {
        da = desc(smem_u32(sa) + st * 32, 16, 1024, 2);
        db = desc(smem_u32(sb) + st * 32, 16, 1024, 2);
        id = idesc(0, 0);
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(st));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
  }
  uint32_t done = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(&bar))
        : "memory");
    if (spin > (1u << 24)) __trap();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + (uint32_t((t / 32) * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < 32; ++n) D[t * 32 + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(128 * 32), B(32 * 32), D(128 * 32), R(128 * 32);
  for (int i = 0; i < 128 * 32; ++i) A[i] = float((i * 37) % 17) - 8.f;
  for (int i = 0; i < 32 * 32; ++i) B[i] = float((i * 11) % 13) - 6.f;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      float s = 0;
      for (int k = 0; k < 32; ++k) s += A[m * 32 + k] * B[n * 32 + k];
      R[m * 32 + n] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const char* names[] = {"K-major none", "MN-major SBO=MN", "MN-major LBO=MN", "K-major sw128"};
  for (int v = 0; v < 4; ++v) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d (%s): CUDA error %s\n", v, names[v], cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double mx = 0;
    for (int i = 0; i < 128 * 32; ++i) {
      mx = std::fmax(mx, std::fabs(D[i]));
      if (D[i] != R[i]) ++bad;
    }
    printf("variant %d (%s): %d of 4096 differ, max |D| %.1f, D[0..3] %.1f %.1f %.1f %.1f ref %.1f %.1f %.1f %.1f\n",
           v, names[v], bad, mx, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  }
  return 0;
}
