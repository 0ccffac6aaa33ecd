"""Legacy warp-level tensor-core throughput on this GPU: mma.sync m16n8k8 TF32
(fp32 accumulate) back-to-back, vs plain FFMA.  Decides whether the CP-ALS
row update (a 32-wide GEMM + Gram, HBM-bound at ~1 ms per 25M rows) can move
its 3xTF32 arithmetic onto the legacy MMA path.

  python scripts/mma_probe.py
"""
import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
__global__ void k_mma(float* out, int iters) {
  float d[8][4] = {};
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float d[16];
  for (int j = 0; j < 16; ++j) d[j] = threadIdx.x * j;
  const float a = out[0] + 1.0001f, b = 0.9999f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < 16; ++j) d[j] = fmaf(d[j], a, b);
  }
  float s = 0;
  for (int j = 0; j < 16; ++j) s += d[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
void run(torch::Tensor out, int kind, int grid, int block, int iters) {
  if (kind == 0) k_mma<<<grid, block>>>(out.data_ptr<float>(), iters);
  else k_ffma<<<grid, block>>>(out.data_ptr<float>(), iters);
}
"""


def main():
    ext = load_inline("mma_probe", "void run(torch::Tensor out, int kind, int grid, int block, int iters);",
                      cuda_sources=SRC, functions=["run"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(sms * 8 * 1024, device="cuda")
    for kind, name, flop_per_iter_thread in ((0, "mma.sync m16n8k8 tf32", 8 * 16 * 8 * 8 * 2 / 32),
                                             (1, "FFMA", 8 * 16 * 2)):
        for warps in (4, 8, 16, 32):
            block, grid, iters = 256, sms * warps // 8, 2000
            ext.run(out, kind, grid, block, 10)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            ext.run(out, kind, grid, block, iters)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            tf = grid * block * iters * flop_per_iter_thread / (ms * 1e-3) / 1e12
            print(f"{name:24s} warps/SM {warps:3d}: {tf:8.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
