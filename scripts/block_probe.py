"""Would L2 blocking help the DRAM-bound CSL / CSF parts?  Gather-only timing of
the (B row, C row) pairs of one mode's CSL part in the plan's order vs orders
blocked by C-row range (and by B-row range), so that one block's C rows fit
in L2.  Rows/s of the gather is the ceiling the MTTKRP kernels run at
(DESIGN.md §8), so the ratio bounds what a blocked layout could gain before
its extra partial-row traffic.

  python scripts/block_probe.py delicious-3d 0 [scale]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from torch.utils.cpp_extension import load_inline

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

SRC = r"""
#include <torch/extension.h>
#include <cuda_runtime.h>
__device__ __forceinline__ float4 ldrow(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__global__ void __launch_bounds__(256, 4) k_pairs(const float4* __restrict__ B, const float4* __restrict__ C,
    const uint2* __restrict__ jk, long n, float4* __restrict__ sink) {
  const int lane = threadIdx.x & 31, lig = lane & 7;
  const long gid = (blockIdx.x * long(blockDim.x) + threadIdx.x) >> 3;
  const long ng = (long(gridDim.x) * blockDim.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long base = gid * 8; base < n; base += ng * 8) {
    uint2 q = base + lig < n ? jk[base + lig] : make_uint2(0, 0);
    float4 r[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned bj = __shfl_sync(0xffffffffu, q.x, j, 8);
      unsigned cj = __shfl_sync(0xffffffffu, q.y, j, 8);
      r[2 * j] = ldrow(B + size_t(bj) * 8 + lig);
      r[2 * j + 1] = ldrow(C + size_t(cj) * 8 + lig);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) { acc.x += r[j].x; acc.y += r[j].y; acc.z += r[j].z; acc.w += r[j].w; }
  }
  if (acc.x == 12345.f) sink[threadIdx.x] = acc;
}
void pairs(torch::Tensor B, torch::Tensor C, torch::Tensor jk, torch::Tensor sink, int grid) {
  k_pairs<<<grid, 256>>>((const float4*)B.data_ptr(), (const float4*)C.data_ptr(),
                         (const uint2*)jk.data_ptr(), jk.size(0), (float4*)sink.data_ptr());
}
"""
CPP = "void pairs(torch::Tensor B, torch::Tensor C, torch::Tensor jk, torch::Tensor sink, int grid);"


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "delicious-3d"
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    ext = load_inline("block_probe", CPP, cuda_sources=SRC, functions=["pairs"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                      verbose=False)
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg, scale=scale)
    mo = hb.allmode_order(dims, mode)
    h = hb.build_hbcsf(t, mo)
    s = h.csl_part
    j = s.rest_idx[:, 0].astype(np.int64)
    k = s.rest_idx[:, 1].astype(np.int64)
    sl = np.repeat(np.arange(s.num_slices), np.diff(s.slice_ptr))
    dev = torch.device("cuda")
    R = 32
    B = torch.rand((dims[mo[1]], R), device=dev)
    C = torch.rand((dims[mo[2]], R), device=dev)
    sink = torch.empty((256, 4), device=dev)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    print(f"{cfg} mode {mode}: CSL nnz {s.nnz} slices {s.num_slices}; B rows {dims[mo[1]]} "
          f"({dims[mo[1]] * R * 4 / 1e6:.0f} MB) C rows {dims[mo[2]]} ({dims[mo[2]] * R * 4 / 1e6:.0f} MB)",
          flush=True)

    def run(name, order):
        jk = torch.from_numpy(np.stack([j[order], k[order]], 1).astype(np.uint32).view(np.int32)).to(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for it in range(6):
            ev[0].record()
            ext.pairs(B, C, jk, sink, sms * 4)
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = float(np.median(ts[1:]))
        print(f"  {name:40s} {ms:8.3f} ms  {2 * s.nnz / ms / 1e6:8.1f} G rows/s", flush=True)
        return ms

    base = run("plan order (slice, j, k)", np.arange(s.nnz))
    for mb in (16, 32, 64, 128):
        kb = max(1, (mb << 20) // (R * 4))
        order = np.lexsort((np.arange(s.nnz), k // kb))
        run(f"C-blocked {mb} MB ({(dims[mo[2]] + kb - 1) // kb} blocks)", order)
    for mb in (32, 64):
        kb = max(1, (mb << 20) // (R * 4))
        jb = kb
        order = np.lexsort((np.arange(s.nnz), j // jb, k // kb))
        run(f"C x B blocked {mb} MB", order)
    order = np.lexsort((j, k))
    run("fully sorted by (k, j)", order)


if __name__ == "__main__":
    main()
