// HB-CSF / B-CSF MTTKRP on sm_100a.
//
// One persistent launch per mode covers all three HB-CSF buckets plus the
// zero-fill of rows no bucket owns.  The plan cuts each bucket into tasks of
// ~TASK_NNZ nonzeros (B-CSF: heavy slices are split into chunks, light slices
// are packed into runs of whole slices); an 8-lane group owns one task, so a
// warp runs four tasks side by side.  Lanes are vectorised over the rank
// (float4, 8 lanes = one 128-byte factor row at R=32).
//
//   CSF task : per batch of 8 nonzeros, gather the 8 leaf rows C[k] at once,
//              accumulate v*C[k] into the fiber partial in registers, and at
//              each fiber end multiply by the fiber row B[j] into the slice
//              partial (kernels.py:173-184 restated per group).
//   CSL task : no fiber level: v*B[j]*C[k] straight into the slice partial
//              (kernels.py:210-214).
//   COO task : one nonzero = one output row, plain store (kernels.py:137-140
//              on the HB-CSF coo_part, whose slices hold one nonzero each).
//   ZERO task: rows owned by no bucket.
// Output rows of unsplit slices are written with plain stores; chunks of a
// split slice add into a per-slice fp32 accumulator with vector atomics and
// the last chunk to finish (arrival counter) stores the row — so every output
// row is written exactly once and no memset of the output is needed.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <mutex>

#include "common.cuh"

namespace hbk {

static constexpr uint32_t NOSLOT = 0xFFFFFFFFu;
// light-task size = heavy-slice threshold (round 2, ms per 3-mode step,
// 64 / 128 / 256: nell-1 8.47 / 8.29 / 8.31, flickr-3d 6.30 / 6.18 / 6.19,
// delicious-3d 9.89 / 9.91 / 9.97, nell-2 2.22 all)
static constexpr uint32_t TASK_NNZ_CSF = 128;
static constexpr uint32_t TASK_NNZ_CSL = 128;
static constexpr uint32_t TASK_NNZ_COO = 32;
static constexpr uint32_t TASK_ROWS_ZERO = 256;
static constexpr uint32_t GEN_TASK_NNZ = 256;

struct Task {
  uint32_t lo, hi;   // nonzero range (rows range for ZERO tasks)
  uint32_t s;        // first slice (position in the bucket's slice arrays)
  uint32_t f;        // first fiber (CSF)
  uint32_t slot;     // split-slice accumulator slot, NOSLOT for whole slices
  uint32_t nchunk;   // chunks of that split slice
  uint32_t pad0, pad1;
};

struct alignas(16) Work {
  // task ranges [0,n0) CSF, [n0,n1) CSL, [n1,n2) COO, [n2,n3) ZERO
  uint32_t n0, n1, n2, n3;
  const Task* tasks;
  // CSF bucket: original tree arrays (generic kernel) ...
  const uint32_t* csf_send;   // [S+1] nonzero offset of each slice
  const uint32_t* csf_sidx;   // [S]   output row of each slice
  const uint32_t* csf_lptr;   // [F+1]
  const uint32_t* csf_fidx;   // [F]
  const uint32_t* csf_leaf;   // [M]
  const float* csf_val;       // [M]
  uint32_t csf_F;
  uint32_t csf_S;
  // ... and the kernel-native stream: (leaf | FEND | SEND, value bits)
  const uint2* csf_pairs;     // [M]
  // CSL bucket
  const uint32_t* csl_send;   // slice_ptr [S+1]
  const uint32_t* csl_sidx;
  const uint32_t* csl_j;      // rest[0]
  const uint32_t* csl_k;      // rest[1]
  const float* csl_val;
  uint32_t csl_S;
  const uint2* csl_pairs;     // [M] (rest[1] | SEND, value bits)
  // COO bucket (unique rows)
  const uint32_t* coo_i;
  const uint32_t* coo_j;
  const uint32_t* coo_k;
  const float* coo_val;
  const uint4* coo_quads;     // [M] (row, j, k, value bits)
  // fp64 value streams for the fast kernels' fp64 instantiation, one double
  // per position of csf_pairs / csl_pairs / coo_quads (0 at B positions)
  const double* csf_v64;
  const double* csl_v64;
  const double* coo_v64;
  // ZERO list
  const uint32_t* zero_rows;
  // split-slice workspace (self-cleaning)
  float* ws_acc;
  uint32_t* ws_cnt;
  uint32_t* ws_ctr;   // per kernel kind k: [2k] task counter, [2k+1] finished warps
  uint32_t total_warps[3];
};

// flag bits stored in the leaf coordinate of the kernel-native streams
static constexpr uint32_t FEND = 0x80000000u;  // last nonzero of its fiber
static constexpr uint32_t SEND = 0x40000000u;  // last nonzero of its slice
static constexpr uint32_t KMASK = 0x3FFFFFFFu;
static constexpr uint32_t FB = 0x80000000u;    // B-row position (B-position streams)
// B-position streams keep the row index in bits 0..29; bit 31 = FB, bit 30 =
// SEND.  The kernel scales it by the row stride (one IMAD.WIDE).  (Measured
// and dropped: a per-row L2 evict-last/evict-first class by reference count
// — <= 4% on the HBM-resident tensors, -8% on nell-2 — and a persisting L2
// set-aside, which was slower.)
static constexpr uint32_t XMASK = 0x3FFFFFFFu;

struct Factors3 {
  using V = float4;  // 16-byte lane vector and its scalar
  using S = float;
  static constexpr bool F64 = false;
  const float4* B;  // factor of mode_order[1] (fiber / rest[0])
  const float4* C;  // factor of mode_order[2] (leaf / rest[1])
  float4* out;
  // rank R = 4 * rs; a launch covers columns [4 col4, 4 col4 + 4 lanes) of
  // every row (8 lanes x float4 = 32 columns per pass; R > 32 takes several)
  uint32_t rs;     // row stride in float4
  uint32_t col4;   // first column of this pass, in float4
  uint32_t lanes;  // active lanes of an 8-lane group in this pass (1..8)
};
// The R = 32 specialisation: one full pass, strides known at compile time
// (the runtime fields cost registers the B-position kernels do not have).
struct Factors3R32 {
  using V = float4;
  using S = float;
  static constexpr bool F64 = false;
  const float4* B;
  const float4* C;
  float4* out;
  static constexpr uint32_t rs = 8, col4 = 0, lanes = 8;
  Factors3R32() = default;
  __host__ __device__ explicit Factors3R32(const Factors3& f) : B(f.B), C(f.C), out(f.out) {}
};
// fp64 views: a lane holds a double2 (16 bytes, like float4), so a pass of
// 8 lanes covers 16 columns and the row stride / column offsets stay in
// 16-byte units.  Factors3D: any even R (runtime stride); Factors3DR32:
// R = 32 plans, whose B-position streams hold row indices pre-scaled to
// float4 units (x 8): a double2 row of R = 32 is 16 units, so x 2.
struct Factors3D {
  using V = double2;
  using S = double;
  static constexpr bool F64 = true;
  const double2* B;
  const double2* C;
  double2* out;
  uint32_t rs, col4, lanes;
};
struct Factors3DR32 {
  using V = double2;
  using S = double;
  static constexpr bool F64 = true;
  const double2* B;
  const double2* C;
  double2* out;
  uint32_t col4;  // 0 or 8: the two 16-column passes
  static constexpr uint32_t rs = 16, lanes = 8;
};
// A lane's column within the pass; idle lanes of a partial pass mirror the
// last active one (valid addresses) and never store.
template <class FX>
__device__ __forceinline__ uint32_t lane_col(const FX& fx, int lig) {
  return fx.col4 + min(uint32_t(lig), fx.lanes - 1);
}
template <class FX>
__device__ __forceinline__ bool lane_live(const FX& fx, int lig) {
  return uint32_t(lig) < fx.lanes;
}

// &base[x * rs].  R = 32: plain arithmetic (ptxas picks the cheapest form
// for the constant stride); other ranks: one mad.wide.u32 with the runtime
// stride (the compiler otherwise splits the 64-bit offset into shift + add
// pairs).  srowp: a B-position stream index, pre-scaled to float4 units by
// the plan builder when FX is the R = 32 specialisation (one IMAD.WIDE per
// row instead of three instructions: 3.5% of the nell-2 step).
template <class P>
__device__ __forceinline__ P* rowp(P* base, uint32_t x, const Factors3R32&) {
  return base + size_t(x) * 8;
}
template <class P, class FX>
__device__ __forceinline__ P* rowp(P* base, uint32_t x, const FX& fx) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;"
      : "=l"(r)
      : "r"(x), "r"(uint32_t(fx.rs * 16u)), "l"(base));
  return reinterpret_cast<P*>(r);
}
template <class P>
__device__ __forceinline__ P* rowp(P* base, uint32_t x, const Factors3DR32&) {
  return base + size_t(x) * 16;
}
template <class P>
__device__ __forceinline__ P* srowp(P* base, uint32_t x, const Factors3R32&) { return base + x; }
template <class P>
__device__ __forceinline__ P* srowp(P* base, uint32_t x, const Factors3DR32&) {
  return base + size_t(x) * 2;
}
template <class P, class FX>
__device__ __forceinline__ P* srowp(P* base, uint32_t x, const FX& fx) {
  return rowp(base, x, fx);
}

__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float4 fma4(float a, float4 x, float4 y) {
  return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z), fmaf(a, x.w, y.w));
}
__device__ __forceinline__ float4 fmav4(float4 a, float4 x, float4 y) {
  return make_float4(fmaf(a.x, x.x, y.x), fmaf(a.y, x.y, y.y), fmaf(a.z, x.z, y.z),
                     fmaf(a.w, x.w, y.w));
}
__device__ __forceinline__ float4 mul4(float a, float4 x) {
  return make_float4(a * x.x, a * x.y, a * x.z, a * x.w);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 shfl_xor4(float4 v, int m) {
  return make_float4(__shfl_xor_sync(0xFFFFFFFFu, v.x, m), __shfl_xor_sync(0xFFFFFFFFu, v.y, m),
                     __shfl_xor_sync(0xFFFFFFFFu, v.z, m), __shfl_xor_sync(0xFFFFFFFFu, v.w, m));
}
__device__ __forceinline__ void red_add4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 ld_cg4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_cg4(float4* p, float4 v) {
  asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
// double2 counterparts of the float4 lane-vector operations
template <class V> __device__ __forceinline__ V vzero();
template <> __device__ __forceinline__ float4 vzero<float4>() { return f4zero(); }
template <> __device__ __forceinline__ double2 vzero<double2>() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 fma4(double a, double2 x, double2 y) {
  return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}
__device__ __forceinline__ double2 fmav4(double2 a, double2 x, double2 y) {
  return make_double2(fma(a.x, x.x, y.x), fma(a.y, x.y, y.y));
}
__device__ __forceinline__ double2 mul4(double a, double2 x) { return make_double2(a * x.x, a * x.y); }
__device__ __forceinline__ double2 add4(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 shfl_xor4(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xFFFFFFFFu, v.x, m), __shfl_xor_sync(0xFFFFFFFFu, v.y, m));
}
__device__ __forceinline__ void red_add4(double2* p, double2 v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v.x) : "memory");
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(reinterpret_cast<double*>(p) + 1), "d"(v.y)
               : "memory");
}
__device__ __forceinline__ double2 ld_cg4(const double2* p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg4(double2* p, double2 v) {
  asm volatile("st.global.cg.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 ld_row4(const double2* p, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L1::evict_last.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
      : "=d"(v.x), "=d"(v.y)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint2 ld_stream_u2(const uint2* p, uint64_t pol) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(pol));
  return v;
}

// ---------------------------------------------------------- fast path --
// The four 8-lane groups of a warp run their four tasks in lockstep (the
// warp iterates max(batches) times; a finished group idles with n = 0), so
// every shuffle is a full-warp, convergent SHFL and group-dependent branches
// only guard loads and FMAs.

#define FULL 0xFFFFFFFFu

// 16-byte global->shared async copy (L1-allocating: hot fiber rows hit L1).
// Each lane later reads back only the bytes it copied, so completion needs
// only this thread's cp.async.wait_all, no barrier.
__device__ __forceinline__ void cp_async16(float4* smem, const float4* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(double2* smem, const double2* gmem) {
  cp_async16(reinterpret_cast<float4*>(smem), reinterpret_cast<const float4*>(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// OR of the four groups' bytes of a ballot
__device__ __forceinline__ uint32_t any_group(uint32_t ballot) {
  return (ballot | (ballot >> 8) | (ballot >> 16) | (ballot >> 24)) & 0xFFu;
}

// Split-slice hand-over, warp-convergent: groups with `active` add their
// partial into the slot accumulator; the group whose add completes the slot
// count stores the row and re-zeroes the slot for the next launch.
template <class FX>
__device__ __forceinline__ void flush_split(const Work& w, const FX& fx, bool active,
                                            uint32_t slot, uint32_t nchunk, uint32_t inc,
                                            uint32_t row, typename FX::V sa, int lane, int lig) {
  using V = typename FX::V;
  const bool live = lane_live(fx, lig);
  V* acc = reinterpret_cast<V*>(w.ws_acc) + size_t(active ? slot : 0) * fx.rs + fx.col4 + lig;
  if (active && live) red_add4(acc, sa);
  __threadfence();
  __syncwarp();
  uint32_t old = 0;
  if (active && lig == 0) old = atomicAdd(w.ws_cnt + slot, inc);
  old = __shfl_sync(FULL, old, lane & ~7);
  if (active && old + inc == nchunk) {
    __threadfence();
    if (live) {
      const V r = ld_cg4(acc);
      fx.out[size_t(row) * fx.rs + fx.col4 + lig] = r;
      st_cg4(acc, vzero<V>());
    }
    if (lig == 0) w.ws_cnt[slot] = 0;
  }
}

// ------------------------------------------------------------ CSF tasks --
// CSF tasks over a "B-position" stream: each fiber's (leaf, value) pairs
// are followed by one extra position (j | FB, 0) naming the fiber's B row, so
// B rows are gathered by the same LDG batch as the leaf rows (no shared-memory
// staging: the L1 data pipe carries each row once).  At a B position the
// fiber partial is multiplied into the slice partial; slice ends (SEND) sit
// on B positions.  Dead lanes carry (0, 0): leaf row 0 times v = 0.
// UNIFORM (padded heavy layout): the four groups' streams have identical
// structure, so B positions are warp-uniform and take a uniform branch
// instead of predicated FMAs; heavy tasks are slice chunks (no SEND).
// ACC (leaf-blocked view, csf_block_view): slice ends add the partial row
// into the pre-zeroed output row (a slice is cut into several virtual slices).
template <bool UNIFORM, bool ACC, class FX>
__device__ __forceinline__ typename FX::V csf_bpos_tasks(const Work& w, const FX& fx, const Task& t,
                                                        int g, int lig, uint64_t pol_s, uint64_t pol_r) {
  using V = typename FX::V;
  using S = typename FX::S;
  const uint32_t lo = t.lo, hi = t.hi;
  const bool chunk = UNIFORM || t.slot != NOSLOT;
  const uint32_t nbat = __reduce_max_sync(FULL, hi > lo ? (hi - lo + 7) / 8 : 0u);
  const V* Cl = fx.C + lane_col(fx, lig);
  const V* Bl = fx.B + lane_col(fx, lig);
  const uint2* pairs = w.csf_pairs;
  const uint32_t Sm1 = w.csf_S ? w.csf_S - 1 : 0;
  uint32_t s = t.s;
  V fa = vzero<V>(), sa = vzero<V>();
  uint2 pr = make_uint2(0u, 0u);
  double pv = 0.0;  // fp64 views: the value of this lane's position
  if (lo + lig < hi) {
    pr = ld_stream_u2(pairs + lo + lig, pol_s);
    if constexpr (FX::F64) pv = ld_stream_f64(w.csf_v64 + lo + lig, pol_s);
  }
  uint32_t sr = chunk ? 0u : __ldg(w.csf_sidx + min(s + lig, Sm1));
  uint32_t base = lo;
  for (uint32_t it = 0; it < nbat; ++it, base += 8) {
    const uint32_t bb_all = __ballot_sync(FULL, pr.x & FB);
    const uint32_t bbits = UNIFORM ? (bb_all & 0xFFu) : ((bb_all >> (8 * g)) & 0xFFu);
    uint32_t sbits = 0, sany = 0;
    if (!UNIFORM) {
      const uint32_t sb_all = __ballot_sync(FULL, !chunk && (pr.x & SEND));
      sbits = (sb_all >> (8 * g)) & 0xFFu;
      sany = any_group(sb_all);
    }
    V r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t xj = __shfl_sync(FULL, pr.x, j, 8);
      const V* bp = (UNIFORM ? ((bbits >> j) & 1u) : (xj & FB)) ? Bl : Cl;
      r[j] = ld_row4(srowp(bp, xj & XMASK, fx), pol_r);
    }
    const S vv = FX::F64 ? S(pv) : S(__uint_as_float(pr.y));
    const uint32_t sr_cur = sr;
    const uint32_t nb = base + 8;
    pr = make_uint2(0u, 0u);
    if (nb + lig < hi) {
      pr = ld_stream_u2(pairs + nb + lig, pol_s);
      if constexpr (FX::F64) pv = ld_stream_f64(w.csf_v64 + nb + lig, pol_s);
    }
    if (!UNIFORM) {
      const uint32_t nsl = __popc(sbits);
      s += nsl;
      if (__any_sync(FULL, nsl != 0)) sr = __ldg(w.csf_sidx + min(s + lig, Sm1));
    }
    uint32_t ts = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const S vj = __shfl_sync(FULL, vv, j, 8);
      if (UNIFORM) {
        if ((bbits >> j) & 1u) {
          sa = fmav4(fa, r[j], sa);
          fa = vzero<V>();
        } else {
          fa = fma4(vj, r[j], fa);
        }
        continue;
      }
      fa = fma4(vj, r[j], fa);
      if ((bbits >> j) & 1u) {
        sa = fmav4(fa, r[j], sa);
        fa = vzero<V>();
      }
      if ((sany >> j) & 1u) {
        const uint32_t row = __shfl_sync(FULL, sr_cur, ts, 8);
        if ((sbits >> j) & 1u) {
          if (lane_live(fx, lig)) {
            V* o = fx.out + size_t(row) * fx.rs + fx.col4 + lig;
            if (ACC) red_add4(o, sa); else *o = sa;
          }
          sa = vzero<V>();
          ++ts;
        }
      }
    }
  }
  return sa;
}

// ------------------------------------------------------------ CSL tasks --
// Per batch of 8 nonzeros a group stages the 8 B rows with cp.async (the
// rows land in shared memory, so many stay in flight without holding
// registers — the CSL-heavy tensors are DRAM-latency bound) and gathers the
// 8 C rows into registers; v * B[j] o C[k] accumulates into the slice
// partial (kernels.py:210-214).  Measured: loading both rows into registers
// (98 registers, 2 CTAs/SM) was 10-14% slower on delicious-3d.
// ACC (blocked CSL layout): slice ends add the partial row into the
// pre-zeroed output instead of storing it (a slice spans several blocks).
template <bool ACC, class FX>
__device__ __forceinline__ typename FX::V csl_tasks(const Work& w, const FX& fx, const Task& t,
                                                   int g, int lig, uint64_t pol_s, uint64_t pol_r,
                                                   typename FX::V* __restrict__ slots) {
  using V = typename FX::V;
  using S = typename FX::S;
  const uint32_t lo = t.lo, hi = t.hi;
  const bool chunk = t.slot != NOSLOT;
  const uint32_t my_batches = hi > lo ? (hi - lo + 7) / 8 : 0;
  const uint32_t nbat = __reduce_max_sync(FULL, my_batches);
  const V* Cl = fx.C + lane_col(fx, lig);
  const V* Bl = fx.B + lane_col(fx, lig);
  uint32_t s = t.s;
  V sa = vzero<V>();
  uint2 pr = make_uint2(0u, 0u);
  uint32_t jx = 0;
  double pv = 0.0;
  if (lo + lig < hi) {
    pr = ld_stream_u2(w.csl_pairs + lo + lig, pol_s);
    jx = ld_stream_u32(w.csl_j + lo + lig, pol_s);
    if constexpr (FX::F64) pv = ld_stream_f64(w.csl_v64 + lo + lig, pol_s);
  }
  uint32_t sr = (hi > lo && !chunk && s + lig < w.csl_S) ? __ldg(w.csl_sidx + s + lig) : 0u;
  uint32_t base = lo;
  for (uint32_t it = 0; it < nbat; ++it, base += 8) {
    const uint32_t n = base < hi ? min(8u, hi - base) : 0u;
    const bool live = uint32_t(lig) < n;
    const uint32_t k = pr.x & KMASK;
    const S v = FX::F64 ? S(pv) : S(__uint_as_float(pr.y));
    const uint32_t sb_all = __ballot_sync(FULL, live && !chunk && (pr.x & SEND));
    const uint32_t sbits = (sb_all >> (8 * g)) & 0xFFu;
    const uint32_t sany = any_group(sb_all);
    V c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t bj = __shfl_sync(FULL, jx, j, 8);
      const uint32_t cj = __shfl_sync(FULL, k, j, 8);
      if (uint32_t(j) < n) {
        cp_async16(slots + j * 8, rowp(Bl, bj, fx));
        c[j] = ld_row4(rowp(Cl, cj, fx), pol_r);
      }
    }
    const uint32_t sr_cur = sr;
    const S vv = v;
    const uint32_t nsl = __popc(sbits);
    s += nsl;
    const uint32_t nb = base + 8;
    if (nb + lig < hi) {
      pr = ld_stream_u2(w.csl_pairs + nb + lig, pol_s);
      jx = ld_stream_u32(w.csl_j + nb + lig, pol_s);
      if constexpr (FX::F64) pv = ld_stream_f64(w.csl_v64 + nb + lig, pol_s);
    }
    if (nsl && nb < hi) sr = (s + lig < w.csl_S) ? __ldg(w.csl_sidx + s + lig) : 0u;
    cp_async_wait_all();
    uint32_t ts = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const S vj = __shfl_sync(FULL, vv, j, 8);
      if (uint32_t(j) < n) sa = fmav4(mul4(vj, slots[j * 8]), c[j], sa);
      if ((sany >> j) & 1u) {
        const uint32_t row = __shfl_sync(FULL, sr_cur, ts, 8);
        if ((sbits >> j) & 1u) {
          if (lane_live(fx, lig)) {
            V* o = fx.out + size_t(row) * fx.rs + fx.col4 + lig;
            if (ACC) red_add4(o, sa); else *o = sa;
          }
          sa = vzero<V>();
          ++ts;
        }
      }
    }
  }
  return sa;
}

// ------------------------------------------------------------ COO tasks --
template <class FX>
__device__ __forceinline__ void coo_tasks(const Work& w, const FX& fx, const Task& t,
                                          int lig, uint64_t pol_s, uint64_t pol_r,
                                          typename FX::V* __restrict__ slots) {
  using V = typename FX::V;
  using S = typename FX::S;
  const uint32_t lo = t.lo, hi = t.hi;
  const uint32_t my_batches = hi > lo ? (hi - lo + 7) / 8 : 0;
  const uint32_t nbat = __reduce_max_sync(FULL, my_batches);
  const V* Cl = fx.C + lane_col(fx, lig);
  const V* Bl = fx.B + lane_col(fx, lig);
  uint4 q = make_uint4(0u, 0u, 0u, 0u);
  double pv = 0.0;
  if (lo + lig < hi) {
    q = ld_stream_u4(w.coo_quads + lo + lig, pol_s);
    if constexpr (FX::F64) pv = ld_stream_f64(w.coo_v64 + lo + lig, pol_s);
  }
  uint32_t base = lo;
  for (uint32_t it = 0; it < nbat; ++it, base += 8) {
    const uint32_t n = base < hi ? min(8u, hi - base) : 0u;
    V c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t bj = __shfl_sync(FULL, q.y, j, 8);
      const uint32_t cj = __shfl_sync(FULL, q.z, j, 8);
      if (uint32_t(j) < n) {
        cp_async16(slots + j * 8, rowp(Bl, bj, fx));
        c[j] = ld_row4(rowp(Cl, cj, fx), pol_r);
      }
    }
    const uint4 cur = q;
    const S vcur = FX::F64 ? S(pv) : S(__uint_as_float(q.w));
    const uint32_t nb = base + 8;
    if (nb + lig < hi) {
      q = ld_stream_u4(w.coo_quads + nb + lig, pol_s);
      if constexpr (FX::F64) pv = ld_stream_f64(w.coo_v64 + nb + lig, pol_s);
    }
    cp_async_wait_all();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t row = __shfl_sync(FULL, cur.x, j, 8);
      const S vj = __shfl_sync(FULL, vcur, j, 8);
      if (uint32_t(j) < n) {
        const V r = fmav4(mul4(vj, slots[j * 8]), c[j], vzero<V>());
        if (lane_live(fx, lig)) fx.out[size_t(row) * fx.rs + fx.col4 + lig] = r;
      }
    }
  }
}

// Rows owned by no bucket: a group loads 8 row numbers at once (one per
// lane) and stores 8 zero rows, so the loop is not a chain of dependent loads.
template <class FX>
__device__ __forceinline__ void zero_task(const Work& w, const FX& fx, const Task& t,
                                          int lig) {
  const uint32_t nbat = __reduce_max_sync(FULL, t.hi > t.lo ? (t.hi - t.lo + 7) / 8 : 0u);
  uint32_t base = t.lo;
  for (uint32_t it = 0; it < nbat; ++it, base += 8) {
    const uint32_t n = base < t.hi ? min(8u, t.hi - base) : 0u;
    const uint32_t rl = uint32_t(lig) < n ? __ldg(w.zero_rows + base + lig) : 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t row = __shfl_sync(FULL, rl, j, 8);
      if (uint32_t(j) < n && lane_live(fx, lig))
        fx.out[size_t(row) * fx.rs + fx.col4 + lig] = vzero<typename FX::V>();
    }
  }
}

// Persistent kernels, one per bucket kind (separate kernels keep each at 80
// registers / 24 warps per SM): a warp pulls 4 consecutive tasks at a time
// (one per 8-lane group) from the kind's counter; the last warp out resets
// it.  Chunks of one split slice that land in the same warp are summed with
// shuffles and handed over with a single vector atomic.
static constexpr int FAST_BLOCK = 256;
// KIND_CSF is the CSF bucket's task range and counters; its kernels are the
// light-slice B-position kernel (KIND_CSF_BPOS4) and the heavy-slice
// padded-layout kernel (KIND_CSF_UNI).
// KIND_CSL_ACC: the CSL kernel over the blocked (block-major) CSL layout;
// KIND_CSF_BPOS4_ACC / KIND_CSF_UNI_ACC: the CSF kernels over a leaf-blocked
// view (rows accumulated).
enum {
  KIND_CSF = 0, KIND_CSL = 1, KIND_COO = 2, KIND_CSF_BPOS4 = 4, KIND_CSF_UNI = 5, KIND_CSL_ACC = 6,
  KIND_CSF_BPOS4_ACC = 7, KIND_CSF_UNI_ACC = 8
};

template <int KIND, class FX>
__global__ void __launch_bounds__(FAST_BLOCK, (KIND == KIND_CSF_BPOS4 || KIND == KIND_CSF_BPOS4_ACC) ? 4 : 3)
    k_mttkrp3_r32(const __grid_constant__ Work w, const __grid_constant__ FX fx) {
  // per lane: 8 slots of 16 B (one per batch position) for staged B rows
  __shared__ float4 s_slots[FAST_BLOCK * 8];
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3;
  const int lig = lane & 7;
  using V = typename FX::V;
  V* slots = reinterpret_cast<V*>(s_slots) + (threadIdx.x >> 3) * 64 + lig;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_r = policy_evict_last();
  static_assert(KIND != KIND_CSF, "CSF tasks run through KIND_CSF_BPOS4 / KIND_CSF_UNI");
  constexpr bool UNI = KIND == KIND_CSF_UNI || KIND == KIND_CSF_UNI_ACC;
  constexpr bool ACC = KIND == KIND_CSL_ACC || KIND == KIND_CSF_BPOS4_ACC || KIND == KIND_CSF_UNI_ACC;
  constexpr int K = (KIND == KIND_CSF_BPOS4 || KIND == KIND_CSF_BPOS4_ACC || UNI) ? KIND_CSF
                    : KIND == KIND_CSL_ACC                                       ? KIND_CSL
                                                                                 : KIND;
  const uint32_t first = K == KIND_CSF ? 0u : (K == KIND_CSL ? w.n0 : w.n1);
  const uint32_t last = K == KIND_CSF ? w.n0 : (K == KIND_CSL ? w.n1 : w.n3);
  // the heavy-slice launch has its own counter pair (words 6, 7) so it can
  // run concurrently with the light-slice launch
  uint32_t* ctr = w.ws_ctr + 2 * (UNI ? 3 : K);
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(ctr, 4u);
    base = __shfl_sync(FULL, base, 0) + first;
    if (base >= last) break;
    const Task t = w.tasks[base + g];
    if (K == KIND_CSF || K == KIND_CSL) {
      const V sa =
          UNI                           ? csf_bpos_tasks<true, ACC>(w, fx, t, g, lig, pol_s, pol_r)
          : K == KIND_CSF               ? csf_bpos_tasks<false, ACC>(w, fx, t, g, lig, pol_s, pol_r)
                                        : csl_tasks<ACC>(w, fx, t, g, lig, pol_s, pol_r, slots);
      const bool mine = t.slot != NOSLOT && t.lo < t.hi;
      const uint32_t slot0 = __shfl_sync(FULL, t.slot, 0);
      const bool same = __all_sync(FULL, mine && t.slot == slot0);
      const uint32_t row =
          mine ? (K == KIND_CSF ? __ldg(w.csf_sidx + t.s) : __ldg(w.csl_sidx + t.s)) : 0u;
      if (ACC) {
        // chunks of a slice cut into several tasks add their partial rows
        // directly into the pre-zeroed output (no accumulator hand-over)
        if (same) {
          V r = add4(sa, shfl_xor4(sa, 8));
          r = add4(r, shfl_xor4(r, 16));
          if (g == 0 && lane_live(fx, lig)) red_add4(fx.out + size_t(row) * fx.rs + fx.col4 + lig, r);
        } else if (mine && lane_live(fx, lig)) {
          red_add4(fx.out + size_t(row) * fx.rs + fx.col4 + lig, sa);
        }
        continue;
      }
      if (same) {
        V r = add4(sa, shfl_xor4(sa, 8));
        r = add4(r, shfl_xor4(r, 16));
        flush_split(w, fx, g == 0, t.slot, t.nchunk, 4u, row, r, lane, lig);
      } else if (__any_sync(FULL, mine)) {
        flush_split(w, fx, mine, t.slot, t.nchunk, 1u, row, sa, lane, lig);
      }
    } else if (base < w.n2) {
      coo_tasks(w, fx, t, lig, pol_s, pol_r, slots);
    } else {
      zero_task(w, fx, t, lig);
    }
  }
  if (lane == 0) {
    const uint32_t done = atomicAdd(ctr + 1, 1u);
    if (done == w.total_warps[K] - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}


// ------------------------------------------------------- gather probe --
// Calibration kernel for the roofline: walks exactly the task lists and
// streams of a plan with the same warp/group structure as k_mttkrp3_r32 but
// only gathers the factor rows (summing them into one register), so its time
// is this plan's row-gather ceiling on this GPU — the resource that bounds
// the MTTKRP when factor rows are L2-resident.
template <int KIND>
__global__ void __launch_bounds__(FAST_BLOCK, 4)
    k_gather_probe(const __grid_constant__ Work w, const __grid_constant__ Factors3R32 fx,
                   float4* __restrict__ sink) {
  const int lane = threadIdx.x & 31, g = lane >> 3, lig = lane & 7;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_r = policy_evict_last();
  const float4* Cl = fx.C + lane_col(fx, lig);
  const float4* Bl = fx.B + lane_col(fx, lig);
  float4 acc = f4zero();
  const uint32_t first = KIND == KIND_CSL ? w.n0 : (KIND == KIND_COO ? w.n1 : 0u);
  const uint32_t last = KIND == KIND_CSL ? w.n1 : (KIND == KIND_COO ? w.n2 : w.n0);
  uint32_t* ctr = w.ws_ctr + 8;  // probe counters (words 8, 9), self-resetting
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(ctr, 4u);
    base = __shfl_sync(FULL, base, 0) + first;
    if (base >= last) break;
    const Task t = w.tasks[base + g];
    const uint32_t nbat = __reduce_max_sync(FULL, t.hi > t.lo ? (t.hi - t.lo + 7) / 8 : 0u);
    uint32_t p0 = t.lo;
    for (uint32_t it = 0; it < nbat; ++it, p0 += 8) {
      const bool live = p0 + lig < t.hi;
      if (KIND == KIND_CSF) {
        const uint2 pr = live ? ld_stream_u2(w.csf_pairs + p0 + lig, pol_s) : make_uint2(0u, 0u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t xj = __shfl_sync(FULL, pr.x, j, 8);
          acc = add4(acc, ld_row4(srowp((xj & FB) ? Bl : Cl, xj & XMASK, fx), pol_r));
        }
      } else if (KIND == KIND_CSL) {
        const uint2 pr = live ? ld_stream_u2(w.csl_pairs + p0 + lig, pol_s) : make_uint2(0u, 0u);
        const uint32_t jx = live ? ld_stream_u32(w.csl_j + p0 + lig, pol_s) : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t kj = __shfl_sync(FULL, pr.x, j, 8) & KMASK;
          const uint32_t bj = __shfl_sync(FULL, jx, j, 8);
          acc = add4(acc, ld_row4(rowp(Cl, kj, fx), pol_r));
          acc = add4(acc, ld_row4(rowp(Bl, bj, fx), pol_r));
        }
      } else {
        const uint4 q = live ? ld_stream_u4(w.coo_quads + p0 + lig, pol_s) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t bj = __shfl_sync(FULL, q.y, j, 8);
          const uint32_t cj = __shfl_sync(FULL, q.z, j, 8);
          acc = add4(acc, ld_row4(rowp(Cl, cj, fx), pol_r));
          acc = add4(acc, ld_row4(rowp(Bl, bj, fx), pol_r));
        }
      }
    }
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) {
    const uint32_t done = atomicAdd(ctr + 1, 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

__global__ void k_task_span(const Task* __restrict__ t, int64_t n, unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s += t[i].hi > t[i].lo ? t[i].hi - t[i].lo : 0u;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// --------------------------------------------------------- generic kernel --
// Any order, any rank: one warp per task, lanes over rank columns, nonzeros
// walked one at a time.  Used for order > 3 or R != 32 (parity coverage; the
// benchmark configurations are all order 3, R = 32).
template <class T>
struct WorkN {
  int order;
  int rank;
  // factors indexed by permuted level (level 0 unused)
  const T* F[HBK_MAX_ORDER];
  const T* Fcoo[HBK_MAX_ORDER];  // by original mode
  // nonzero values of each bucket in T (fp32 copies or the fp64 originals)
  const T* csf_val;
  const T* csl_val;
  const T* coo_val;
  T* acc;  // split-slice accumulators [slots x rank]
  int mode;
  // CSF
  const uint32_t* csf_anc[HBK_MAX_ORDER];  // level d < order-2 coordinate per fiber (d >= 1)
  // CSL rest columns
  const uint32_t* csl_rest[HBK_MAX_ORDER];
  // COO columns
  const uint32_t* coo_col[HBK_MAX_ORDER];
  T* out;
};

// Split-slice hand-over of the generic kernel: every rank chunk of a task
// adds its columns into the slot accumulator; once all chunks are added the
// task arrives (one counter increment per task), and the last task to arrive
// stores every column of the row and re-zeroes the slot.
template <class T>
__device__ __forceinline__ void gen_add_split(const WorkN<T>& wn, uint32_t slot, int r0, T sa,
                                              int lane) {
  if (r0 + lane < wn.rank) atomicAdd(wn.acc + size_t(slot) * wn.rank + r0 + lane, sa);
}
template <class T>
__device__ __forceinline__ void gen_finish_split(const Work& w, const WorkN<T>& wn, uint32_t slot,
                                                 uint32_t nchunk, uint32_t row, int lane) {
  const int R = wn.rank;
  __threadfence();
  __syncwarp();
  uint32_t old = 0;
  if (lane == 0) old = atomicAdd(w.ws_cnt + slot, 1u);
  old = __shfl_sync(0xFFFFFFFFu, old, 0);
  if (old == nchunk - 1) {
    __threadfence();
    for (int r = lane; r < R; r += 32) {
      T* acc = wn.acc + size_t(slot) * R + r;
      wn.out[size_t(row) * R + r] = __ldcg(acc);
      __stcg(acc, T(0));
    }
    __syncwarp();
    if (lane == 0) w.ws_cnt[slot] = 0;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_mttkrp_generic(const __grid_constant__ Work w,
                                                        const __grid_constant__ WorkN<T> wn) {
  const int lane = threadIdx.x & 31;
  const int R = wn.rank;
  const int N = wn.order;
  const int nchunks_r = (R + 31) / 32;
  for (;;) {
    uint32_t ti = 0;
    if (lane == 0) ti = atomicAdd(w.ws_ctr, 1u);
    ti = __shfl_sync(0xFFFFFFFFu, ti, 0);
    if (ti >= w.n3) break;
    const Task t = w.tasks[ti];
    if (t.lo >= t.hi) continue;
    const bool chunk = t.slot != NOSLOT;
    for (int rc = 0; rc < nchunks_r; ++rc) {
      const int r = rc * 32 + lane;
      const bool act = r < R;
      if (ti < w.n0) {  // CSF
        uint32_t s = t.s, f = t.f;
        uint32_t fend = w.csf_lptr[f + 1];
        uint32_t send = w.csf_send[s + 1];
        T fa = 0, sa = 0;
        for (uint32_t i = t.lo; i < t.hi; ++i) {
          uint32_t k = w.csf_leaf[i];
          const T v = wn.csf_val[i];
          if (act) fa = v * wn.F[N - 1][size_t(k) * R + r] + fa;
          if (i + 1 == fend) {
            T m = 1;
            if (act) {
              m = wn.F[N - 2][size_t(w.csf_fidx[f]) * R + r];
              for (int d = 1; d < N - 2; ++d) m *= wn.F[d][size_t(wn.csf_anc[d][f]) * R + r];
            }
            sa = fa * m + sa;
            fa = 0;
            ++f;
            if (f < w.csf_F) fend = w.csf_lptr[f + 1];
            if (!chunk && i + 1 == send) {
              if (act) wn.out[size_t(w.csf_sidx[s]) * R + r] = sa;
              sa = 0;
              ++s;
              if (s < w.csf_S) send = w.csf_send[s + 1];
            }
          }
        }
        if (chunk) {
          if (t.hi != w.csf_lptr[f]) {  // ended inside fiber f
            T m = 1;
            if (act) {
              m = wn.F[N - 2][size_t(w.csf_fidx[f]) * R + r];
              for (int d = 1; d < N - 2; ++d) m *= wn.F[d][size_t(wn.csf_anc[d][f]) * R + r];
            }
            sa = fa * m + sa;
          }
          gen_add_split(wn, t.slot, rc * 32, sa, lane);
        }
      } else if (ti < w.n1) {  // CSL
        uint32_t s = t.s;
        uint32_t send = w.csl_send[s + 1];
        T sa = 0;
        for (uint32_t i = t.lo; i < t.hi; ++i) {
          if (act) {
            T p = wn.csl_val[i];
            for (int c = 0; c < N - 1; ++c) p *= wn.F[c + 1][size_t(wn.csl_rest[c][i]) * R + r];
            sa += p;
          }
          if (!chunk && i + 1 == send) {
            if (act) wn.out[size_t(w.csl_sidx[s]) * R + r] = sa;
            sa = 0;
            ++s;
            if (s < w.csl_S) send = w.csl_send[s + 1];
          }
        }
        if (chunk) gen_add_split(wn, t.slot, rc * 32, sa, lane);
      } else if (ti < w.n2) {  // COO (unique rows)
        for (uint32_t i = t.lo; i < t.hi; ++i) {
          if (!act) continue;
          T p = wn.coo_val[i];
          for (int d = 0; d < N; ++d)
            if (d != wn.mode) p *= wn.Fcoo[d][size_t(wn.coo_col[d][i]) * R + r];
          wn.out[size_t(wn.coo_col[wn.mode][i]) * R + r] = p;
        }
      } else {  // ZERO
        for (uint32_t i = t.lo; i < t.hi; ++i)
          if (act) wn.out[size_t(w.zero_rows[i]) * R + r] = T(0);
      }
    }
    if (chunk && ti < w.n1)
      gen_finish_split(w, wn, t.slot, t.nchunk,
                       ti < w.n0 ? w.csf_sidx[t.s] : w.csl_sidx[t.s], lane);
  }
  __syncwarp();
  if (lane == 0) {
    uint32_t done = atomicAdd(w.ws_ctr + 1, 1u);
    if (done == w.total_warps[0] - 1) {
      w.ws_ctr[0] = 0;
      w.ws_ctr[1] = 0;
    }
  }
}

// ------------------------------------------------------- plan building --
// Slice nonzero offsets of the CSF bucket (leaf_offsets, formats.py:109-111)
// and the first fiber of every slice (fiber_positions, :102-107).
struct Chain2 {
  const uint32_t* ptr[HBK_MAX_ORDER];
  int nlev;
};
__global__ void k_csf_slice_offsets(Chain2 ch, int64_t S, uint32_t* __restrict__ fpos,
                                    uint32_t* __restrict__ loff) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s <= S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t p = uint32_t(s);
    for (int d = 0; d < ch.nlev - 1; ++d) p = ch.ptr[d][p];
    fpos[s] = p;
    loff[s] = ch.ptr[ch.nlev - 1][p];
  }
}

// Per slice: number of tasks it opens (chunks of a heavy slice, or 1 if it
// starts a new run of light slices) and whether it needs an accumulator slot.
// Slices with more than H nonzeros belong to the heavy layout and open none.
__global__ void k_task_count(const uint32_t* __restrict__ loff, int64_t S, uint32_t T, uint32_t H,
                             uint32_t* __restrict__ cnt, uint32_t* __restrict__ slotf) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t a = loff[s], m = loff[s + 1] - a;
    if (m > H) {
      cnt[s] = 0;
      slotf[s] = 0;
    } else if (m > T) {
      cnt[s] = (m + T - 1) / T;
      slotf[s] = 1;
    } else {
      bool start = true;
      if (s > 0) {
        uint32_t pa = loff[s - 1], pm = a - pa;
        start = (pm > T) || (pa / T != a / T);
      }
      cnt[s] = start;
      slotf[s] = 0;
    }
  }
}

__device__ __forceinline__ uint32_t fiber_of(const uint32_t* __restrict__ lptr, uint32_t fb,
                                             uint32_t fe, uint32_t pos) {
  // last f in [fb, fe) with lptr[f] <= pos
  uint32_t lo = fb, hi = fe;
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (lptr[mid] <= pos)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// One thread per task: its slice is the last s with toff[s] <= i (slices
// without tasks have empty ranges), so a heavy slice's thousands of chunks
// are filled in parallel rather than by one thread.
__global__ void k_task_fill(const uint32_t* __restrict__ loff, const uint32_t* __restrict__ fpos,
                            const uint32_t* __restrict__ lptr, int64_t S, uint32_t T,
                            const uint32_t* __restrict__ toff, const uint32_t* __restrict__ slot,
                            const uint32_t* __restrict__ posoff, uint32_t ntask,
                            Task* __restrict__ tasks) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ntask;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = S;  // largest s in [0, S) with toff[s] <= i
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (toff[mid] <= uint32_t(i)) lo = mid;
      else hi = mid;
    }
    const int64_t s = lo;
    const uint32_t a = loff[s], m = loff[s + 1] - a;
    const uint32_t nt = toff[s + 1] - toff[s];
    Task t{};
    t.s = uint32_t(s);
    if (m > T) {
      const uint32_t c = uint32_t(i) - toff[s];
      t.lo = a + uint32_t((uint64_t(m) * c) / nt);
      t.hi = a + uint32_t((uint64_t(m) * (c + 1)) / nt);
      t.f = fpos ? fiber_of(lptr, fpos[s], fpos[s + 1], t.lo) : 0;
      t.slot = slot[s];
      t.nchunk = nt;
    } else {
      t.lo = a + (posoff ? posoff[s] : 0u);
      t.f = fpos ? fpos[s] : 0;
      t.slot = NOSLOT;
      t.nchunk = 1;
    }
    tasks[i] = t;
  }
}

// A run of light slices ends at its last slice (the next slice opens a task
// or belongs to the heavy layout); that slice sets the run's end.
__global__ void k_run_hi(const uint32_t* __restrict__ loff, int64_t S, uint32_t T, uint32_t H,
                         const uint32_t* __restrict__ toff, const uint32_t* __restrict__ posoff,
                         Task* __restrict__ tasks) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t m = loff[s + 1] - loff[s];
    if (m > T) continue;
    const bool last = s + 1 == S || toff[s + 2] != toff[s + 1] || loff[s + 2] - loff[s + 1] > H;
    if (last) tasks[toff[s + 1] - 1].hi = loff[s + 1] + (posoff ? posoff[s + 1] : 0u);
  }
}

// Schedule-driven CSF tasks (mttkrp_scheduled, kernels.py:256-342): one task
// per BlockSchedule unit.
__global__ void k_units_per_slice(const uint32_t* __restrict__ units, int64_t U,
                                  uint32_t* __restrict__ cnt) {
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < U;
       u += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + units[3 * u], 1u);
}
__global__ void k_slot_flags(const uint32_t* __restrict__ cnt, int64_t S,
                             uint32_t* __restrict__ f) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x)
    f[s] = cnt[s] > 1;
}
// bpos: ranges in B-position stream positions (fiber f's leaves start at
// lptr[f] + f); units are fiber-aligned, so a unit ends on a B position.
__global__ void k_units_to_tasks(const uint32_t* __restrict__ units, int64_t U,
                                 const uint32_t* __restrict__ lptr, const uint32_t* __restrict__ cnt,
                                 const uint32_t* __restrict__ slot, int bpos,
                                 Task* __restrict__ tasks) {
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < U;
       u += int64_t(gridDim.x) * blockDim.x) {
    uint32_t sp = units[3 * u], fs = units[3 * u + 1], ft = units[3 * u + 2];
    Task t{};
    t.lo = lptr[fs] + (bpos ? fs : 0u);
    t.hi = lptr[ft] + (bpos ? ft : 0u);
    t.s = sp;
    t.f = fs;
    t.slot = cnt[sp] > 1 ? slot[sp] : NOSLOT;
    t.nchunk = cnt[sp];
    tasks[u] = t;
  }
}

__global__ void k_mark_rows(const uint32_t* __restrict__ rows, int64_t n,
                            uint8_t* __restrict__ mark) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    mark[rows[i]] = 1;
}
__global__ void k_unmarked_flags(const uint8_t* __restrict__ mark, int64_t n,
                                 uint32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    f[i] = mark[i] == 0;
}
__global__ void k_unmarked_emit(const uint32_t* __restrict__ pos, int64_t n,
                                uint32_t* __restrict__ rows) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (pos[i + 1] != pos[i]) rows[pos[i]] = uint32_t(i);
}
__global__ void k_marked_flags(const uint8_t* __restrict__ mark, int64_t n,
                               uint32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    f[i] = mark[i] != 0;
}
__global__ void k_range_tasks(Task* __restrict__ tasks, int64_t ntask, uint32_t total,
                              uint32_t step) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ntask;
       i += int64_t(gridDim.x) * blockDim.x) {
    Task t{};
    t.lo = min(total, uint32_t(i) * step);
    t.hi = min(total, uint32_t(i + 1) * step);
    t.slot = NOSLOT;
    t.nchunk = 1;
    tasks[i] = t;
  }
}
__global__ void k_empty_tasks(Task* __restrict__ tasks, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    Task t{};
    t.slot = NOSLOT;
    t.nchunk = 1;
    tasks[i] = t;
  }
}

// B-position stream of a CSF bucket in tree order: fiber f's pairs start at
// position lptr[f] + f and are followed by (fidx[f] | FB, 0).
__global__ void k_bpos_stream(const uint32_t* __restrict__ lptr, const uint32_t* __restrict__ fidx,
                              const uint32_t* __restrict__ leaf, const float* __restrict__ val,
                              int64_t F, uint32_t sh, uint2* __restrict__ out) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = lptr[f], b = lptr[f + 1];
    uint2* o = out + a + f;
    for (uint32_t i = a; i < b; ++i) *o++ = make_uint2(leaf[i] << sh, __float_as_uint(val[i]));
    *o = make_uint2((fidx[f] << sh) | FB, 0u);
  }
}
// fp64 values of the same stream: each fiber's values, then 0 at its B position
__global__ void k_bpos_v64(const uint32_t* __restrict__ lptr, const double* __restrict__ val,
                           int64_t F, double* __restrict__ out) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = lptr[f], b = lptr[f + 1];
    double* o = out + a + f;
    for (uint32_t i = a; i < b; ++i) *o++ = val[i];
    *o = 0.0;
  }
}
// SEND on the B position of each slice's last fiber
__global__ void k_bpos_send(const uint32_t* __restrict__ fpos, const uint32_t* __restrict__ lptr,
                            int64_t S, uint2* __restrict__ out) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t f0 = fpos[s], f1 = fpos[s + 1];
    if (f1 > f0) out[lptr[f1] + f1 - 1].x |= SEND;
  }
}

// Kernel-native streams (built once per plan).
__global__ void k_pairs(const uint32_t* __restrict__ k, const float* __restrict__ v, int64_t M,
                        uint2* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = make_uint2(k[i], __float_as_uint(v[i]));
}
// flag the last nonzero of every segment [ptr[x], ptr[x+1])
__global__ void k_flag_ends(const uint32_t* __restrict__ ptr, int64_t n, uint32_t flag,
                            uint2* __restrict__ out) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < n;
       x += int64_t(gridDim.x) * blockDim.x) {
    uint32_t e = ptr[x + 1];
    if (e > ptr[x]) out[e - 1].x |= flag;
  }
}
__global__ void k_quads(const uint32_t* __restrict__ i0, const uint32_t* __restrict__ j0,
                        const uint32_t* __restrict__ k0, const float* __restrict__ v, int64_t M,
                        uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = make_uint4(i0[i], j0[i], k0[i], __float_as_uint(v[i]));
}

}  // namespace hbk

struct hbk_plan {
  int order = 0, mode = 0, rank = 0;
  int64_t dims[HBK_MAX_ORDER] = {0};
  int mo[HBK_MAX_ORDER] = {0};
  hbk_coo* coo = nullptr;
  hbk_csl* csl = nullptr;
  hbk_csf* csf = nullptr;
  hbk_sched* sched = nullptr;
  hbk::Buf tasks, zero_rows, csf_send, ws;
  hbk::Buf csf_pairs, csl_pairs, coo_quads;
  hbk::Work work{};      // fast kernels (light CSF tasks when the heavy layout is on)
  hbk::Work work_gen{};  // generic kernel (every CSF slice in tree order)
  hbk::Work work_heavy{};
  hbk::Buf heavy_pairs, heavy_fj, heavy_tasks, gen_tasks, probe_sink;
  // blocked CSL layout (csl_blocked_layout): B rows per block (0 = off), the
  // block-major stream, and whether the fast CSL kernel accumulates rows
  int64_t csl_bb = 0;
  bool csl_acc = false;
  hbk::Buf vcsl_pairs, vcsl_j, vcsl_sidx;
  uint32_t vcsl_S = 0;
  // fp64 fast path (built on the first fp64 execution, hbk::ensure_f64):
  // double value streams beside the kernels' index streams
  uint32_t heavy_H = 0, heavy_tau = 0, heavy_W = 0, heavy_slot_base = 0;
  mutable int f64_state = 0;  // 0 unknown, 1 fast path ready, -1 generic kernel
  mutable hbk::Buf csf_v64s, heavy_v64s, csl_v64s;
  uint32_t csl_T = 0;  // the CSL task size the plan was built with (blocked layout rebuild)
  mutable hbk::Work work64{}, work_heavy64{};
  // leaf-blocked heavy slices (csf_block_view; chosen in hbk_plan_create):
  // the fast fp32 path runs sub_blk (the heavy slices, leaf-block-major,
  // rows accumulated into their pre-zeroed rows) then sub_main (every other
  // slice, the CSL-as-CSF light slices and the COO bucket); the plan itself
  // keeps the reference buckets for the generic / fp64 kernel and the OpCount
  hbk_plan* sub_main = nullptr;
  hbk_plan* sub_blk = nullptr;
  hbk::Buf heavy_rows;          // u32 output rows of the heavy slices
  int64_t n_heavy_rows = 0;
  int64_t leaf_bb = 0, leaf_min = 0;
  bool force_generic = false;   // fast structures live in the sub-plans
  bool acc_csf = false;         // (sub_blk) CSF kernels accumulate rows, no zero-row tasks
  const hbk::Buf* extra_owned = nullptr;  // (sub_main) rows owned by sub_blk
  int64_t n_extra_owned = 0;
  // B-position plans launch their bucket kernels on forked streams so each
  // kernel's CTAs fill the tail of the one before (HBK_CONCURRENT=0: serial)
  bool concurrent = false;
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  // leaf-blocked plans: one fork over both sub-plans' kernels (up to 8)
  cudaStream_t side_all[7] = {};
  cudaEvent_t ev_join_all[7] = {};
  int grid_heavy = 0;
  bool fast = false;
  bool bpos = false;
  // R = 32 with B/C extents < 2^27: the Factors3R32 kernels, B-position
  // stream indices pre-scaled to float4 units (bshift 3)
  bool r32 = false;
  uint32_t bshift = 0;
  int grid = 0, block = 256;
  int gen_grid = 0;
  int grids[3] = {0, 0, 0};
  hbk_plan_info info{};
  // Executions of one plan share its workspace (task counters, split-slice
  // accumulators, side streams), so they are ordered: each execution's
  // stream waits for the previous execution's completion event, whatever
  // stream or host thread issued it (include/hbk.h, "Plans").
  mutable std::mutex exec_mu;
  cudaEvent_t ev_last = nullptr;
  ~hbk_plan() {
    delete sub_main;
    delete sub_blk;
    if (ev_last) cudaEventDestroy(ev_last);
    for (int i = 0; i < 3; ++i) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    for (int i = 0; i < 7; ++i) {
      if (side_all[i]) cudaStreamDestroy(side_all[i]);
      if (ev_join_all[i]) cudaEventDestroy(ev_join_all[i]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    hbk_coo_release(coo);
    hbk_csl_release(csl);
    hbk_csf_release(csf);
    hbk_sched_release(sched);
  }
};

namespace hbk {

static int64_t pad_to(int64_t n, int64_t m) { return (n + m - 1) / m * m; }

// Tasks of one slice-structured bucket (CSF with fpos/lptr, or CSL).
struct BucketTasks {
  Scratch tasks;
  int64_t n = 0;
  int64_t slots = 0;
};

// posoff (optional): per-slice offset added to nonzero offsets to obtain
// stream positions (B-position streams: the fibers before the slice).
static BucketTasks bucket_tasks(const uint32_t* loff, const uint32_t* fpos, const uint32_t* lptr,
                                int64_t S, uint32_t M, uint32_t T, cudaStream_t st,
                                uint32_t H = 0xFFFFFFFFu, const uint32_t* posoff = nullptr) {
  BucketTasks bt;
  (void)M;
  if (S == 0) return bt;
  Scratch cnt((S + 1) * sizeof(uint32_t), st), slot((S + 1) * sizeof(uint32_t), st);
  k_task_count<<<grid_for(S, 256), 256, 0, st>>>(loff, S, T, H, cnt.as<uint32_t>(),
                                                 slot.as<uint32_t>());
  check_launch("k_task_count");
  uint32_t n = exclusive_scan_total(cnt.as<uint32_t>(), S, st);
  uint32_t nslot = exclusive_scan_total(slot.as<uint32_t>(), S, st);
  bt.tasks = Scratch(size_t(std::max<uint32_t>(n, 1)) * sizeof(Task), st);
  if (n) {
    k_task_fill<<<grid_for(n, 256), 256, 0, st>>>(loff, fpos, lptr, S, T, cnt.as<uint32_t>(),
                                                  slot.as<uint32_t>(), posoff, n,
                                                  bt.tasks.as<Task>());
    check_launch("k_task_fill");
    k_run_hi<<<grid_for(S, 256), 256, 0, st>>>(loff, S, T, H, cnt.as<uint32_t>(), posoff,
                                               bt.tasks.as<Task>());
    check_launch("k_run_hi");
  }
  bt.n = n;
  bt.slots = nslot;
  return bt;
}

// ------------------------------------------------- heavy CSF slices --
// Heavy slices (nnz > H) get a kernel-native layout in which the four 8-lane
// groups of a warp walk fibers of equal length side by side.  Each fiber is
// cut into segments of <= tau nonzeros; a slice's segments are sorted by
// length (longest first, stable) and cut into warp tasks of ~W nonzeros; the
// segments of a warp task are dealt round-robin to its four groups, and each
// group's segments are laid out contiguously as a (leaf | FEND, value)
// stream with its own list of fiber coordinates.  Lockstep groups then end
// their fibers at the same batch positions, so the per-fiber work of the
// kernel (B-row fetch, fiber-partial x B-row, reset) is shared by four
// fibers instead of being paid once per fiber.  The four groups of a warp
// task belong to one slice, so their partials are combined with shuffles
// and handed over with a single vector atomic.  Reordering fibers within a
// slice does not change any output row (a row is the sum over its slice's
// fibers, kernels.py:173-184); only fp32 summation order differs.

__global__ void k_fiber_slice(const uint32_t* __restrict__ fpos, int64_t S, int64_t F,
                              uint32_t* __restrict__ fslice) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    // last s with fpos[s] <= f
    int64_t lo = 0, hi = S;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (fpos[mid] <= uint32_t(f)) lo = mid; else hi = mid;
    }
    fslice[f] = uint32_t(lo);
  }
}

__global__ void k_seg_count(const uint32_t* __restrict__ fslice, const uint32_t* __restrict__ loff,
                            const uint32_t* __restrict__ lptr, int64_t F, uint32_t H, uint32_t tau,
                            uint32_t* __restrict__ nseg) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = fslice[f];
    const uint32_t m = loff[s + 1] - loff[s];
    const uint32_t len = lptr[f + 1] - lptr[f];
    nseg[f] = m > H ? (len + tau - 1) / tau : 0u;
  }
}

__global__ void k_seg_emit(const uint32_t* __restrict__ fslice, const uint32_t* __restrict__ lptr,
                           const uint32_t* __restrict__ fidx, const uint32_t* __restrict__ segoff,
                           int64_t F, uint32_t tau, unsigned long long* __restrict__ key,
                           uint32_t* __restrict__ val, uint32_t* __restrict__ soff,
                           uint32_t* __restrict__ slen, uint32_t* __restrict__ sj,
                           uint32_t* __restrict__ ss) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = segoff[f], b = segoff[f + 1];
    if (a == b) continue;
    const uint32_t s = fslice[f], j = fidx[f];
    uint32_t off = lptr[f];
    const uint32_t end = lptr[f + 1];
    for (uint32_t q = a; q < b; ++q, off += tau) {
      const uint32_t len = min(tau, end - off);
      key[q] = (static_cast<unsigned long long>(s) << 16) | (0xFFFFu - len);
      val[q] = q;
      soff[q] = off;
      slen[q] = len;
      sj[q] = j;
      ss[q] = s;
    }
  }
}

// per sorted segment i: local warp-task index within its slice; the last
// segment of a slice records the slice's task count
__global__ void k_seg_task(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ slen,
                           const uint32_t* __restrict__ ss, const uint32_t* __restrict__ P,
                           const uint32_t* __restrict__ hoff, int64_t G, uint32_t W,
                           uint32_t* __restrict__ tloc, uint32_t* __restrict__ ntask) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < G;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = ss[perm[i]];
    const uint32_t t = (P[i] - hoff[s]) / W;
    tloc[i] = t;
    if (i + 1 == G || ss[perm[i + 1]] != s) ntask[s] = t + 1;
  }
}

__global__ void k_seg_task_first(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ ss,
                                 const uint32_t* __restrict__ tloc, const uint32_t* __restrict__ tbase,
                                 int64_t G, uint32_t* __restrict__ tfirst,
                                 uint32_t* __restrict__ tslice) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < G;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = ss[perm[i]];
    const bool first = i == 0 || ss[perm[i - 1]] != s || tloc[i - 1] != tloc[i];
    if (first) {
      const uint32_t w = tbase[s] + tloc[i];
      tfirst[w] = uint32_t(i);
      tslice[w] = s;
    }
  }
}

// per group task (w, g): segment count and stream length.  B-position
// layout (pad): the four groups of a warp task get identical structure —
// quad q (segments 4q..4q+3, longest first) is padded to the length of its
// first segment, plus one B position — so every group stream has length
// sum_q (L_q + 1) and the kernel's fiber ends are warp-uniform.
__global__ void k_group_sizes(const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ perm,
                              const uint32_t* __restrict__ slen, int64_t NW, uint32_t G,
                              bool pad, uint32_t* __restrict__ gnnz,
                              uint32_t* __restrict__ gseg) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < NW * 4;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = x >> 2;
    const uint32_t g = uint32_t(x & 3);
    const uint32_t a = tfirst[w], b = (w + 1 < NW) ? tfirst[w + 1] : G;
    uint32_t n = 0, c = 0;
    if (pad) {
      for (uint32_t i = a; i < b; i += 4) n += slen[perm[i]] + 1;
      c = (b - a + 3) / 4;
    } else {
      for (uint32_t i = a + g; i < b; i += 4) {
        n += slen[perm[i]];
        ++c;
      }
    }
    gnnz[x] = n;
    gseg[x] = c;
  }
}

// copy each group's segments into its contiguous stream: FEND on segment
// ends (smem-slot kernel), or the padded B-position layout (pad)
__global__ void k_group_fill(const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ perm,
                             const uint32_t* __restrict__ soff, const uint32_t* __restrict__ slen,
                             const uint32_t* __restrict__ sj, const uint32_t* __restrict__ gofs,
                             const uint32_t* __restrict__ fofs, int64_t NW, uint32_t G,
                             const uint32_t* __restrict__ leaf, const float* __restrict__ val,
                             bool pad, uint32_t sh, uint2* __restrict__ pairs,
                             uint32_t* __restrict__ fj, const double* __restrict__ val64,
                             double* __restrict__ v64) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < NW * 4;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = x >> 2;
    const uint32_t g = uint32_t(x & 3);
    const uint32_t a = tfirst[w], b = (w + 1 < NW) ? tfirst[w + 1] : G;
    uint32_t dst = gofs[x], fpos = fofs[x];
    if (pad) {
      for (uint32_t i0 = a; i0 < b; i0 += 4) {
        const uint32_t Lq = slen[perm[i0]];
        const uint32_t i = i0 + g;
        uint32_t len = 0, off = 0, j = 0;
        if (i < b) {
          const uint32_t q = perm[i];
          len = slen[q];
          off = soff[q];
          j = sj[q];
        }
        for (uint32_t t = 0; t < len; ++t)
          pairs[dst + t] = make_uint2(leaf[off + t] << sh, __float_as_uint(val[off + t]));
        for (uint32_t t = len; t < Lq; ++t) pairs[dst + t] = make_uint2(0u, 0u);
        if (v64) {
          for (uint32_t t = 0; t < len; ++t) v64[dst + t] = val64[off + t];
          for (uint32_t t = len; t <= Lq; ++t) v64[dst + t] = 0.0;
        }
        dst += Lq;
        pairs[dst++] = make_uint2((j << sh) | FB, 0u);
        fj[fpos++] = j;
      }
      continue;
    }
    for (uint32_t i = a + g; i < b; i += 4) {
      const uint32_t q = perm[i];
      const uint32_t off = soff[q], len = slen[q];
      for (uint32_t t = 0; t < len; ++t)
        pairs[dst + t] = make_uint2(leaf[off + t] | (t + 1 == len ? FEND : 0u),
                                    __float_as_uint(val[off + t]));
      dst += len;
      fj[fpos++] = sj[q];
    }
  }
}

__global__ void k_group_tasks(const uint32_t* __restrict__ tslice, const uint32_t* __restrict__ gofs,
                              const uint32_t* __restrict__ gnnz, const uint32_t* __restrict__ fofs,
                              const uint32_t* __restrict__ hrank, const uint32_t* __restrict__ nchunk,
                              int64_t NW, uint32_t slot_base, Task* __restrict__ tasks) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < NW * 4;
       x += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = tslice[x >> 2];
    Task t{};
    t.lo = gofs[x];
    t.hi = gofs[x] + gnnz[x];
    t.s = s;
    t.f = fofs[x];
    t.slot = slot_base + hrank[s];
    t.nchunk = nchunk[s];
    tasks[x] = t;
  }
}

__global__ void k_slice_nchunk(const uint32_t* __restrict__ tslice, const uint32_t* __restrict__ gseg,
                               int64_t NW, uint32_t* __restrict__ nchunk) {
  for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < NW;
       w += int64_t(gridDim.x) * blockDim.x) {
    uint32_t n = 0;
    for (int g = 0; g < 4; ++g) n += gseg[4 * w + g] != 0;
    atomicAdd(nchunk + tslice[w], n);
  }
}

__global__ void k_heavy_flags(const uint32_t* __restrict__ loff, int64_t S, uint32_t H,
                              uint32_t* __restrict__ hflag, uint32_t* __restrict__ hnnz) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t m = loff[s + 1] - loff[s];
    hflag[s] = m > H;
    hnnz[s] = m > H ? m : 0u;
  }
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                             int64_t n, uint32_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[perm[i]];
}

// ------------------------------------------------ CSL B-row blocking --
// In a CSL slice the nonzeros are sorted by rest[0] (the B-row index), so the
// nonzeros whose B rows fall in one block of BB rows are one contiguous
// segment of the stream.  When the B factor is larger than the L2 can keep
// beside the hot leaf rows and the plan is CSL-dominated (delicious-3d modes
// 0 and 2: B = 317 / 68 MB, near-uniform), the fast path lays the CSL stream
// out block-major: every (block, slice) segment becomes a "virtual slice"
// ordered by (block, slice), and the tasks are runs of whole virtual slices
// (or chunks of long ones), so the persistent kernel gathers B rows from about
// one block at a time, which stays L2-resident.  A slice's segments add their
// partial rows into the output with red.global.add (the output is zeroed
// first), so the blocking adds no hand-over between tasks: one 128-B vector
// atomic per segment (reference semantics unchanged: a row is the sum over its
// slice's nonzeros, kernels.py:210-214; only fp32 summation order differs).
__global__ void k_csl_segflags(const uint32_t* __restrict__ j, int64_t M, uint32_t BB,
                               uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    flag[i] = (i == 0) || (j[i] / BB != j[i - 1] / BB);
}
__global__ void k_csl_slicestarts(const uint32_t* __restrict__ sptr, int64_t S,
                                  uint32_t* __restrict__ flag) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x)
    flag[sptr[s]] = 1;
}
__global__ void k_csl_segs(const uint32_t* __restrict__ pos, int64_t M, uint32_t* __restrict__ start) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    if (pos[i + 1] != pos[i]) start[pos[i]] = uint32_t(i);
}
// per segment: its slice (last slice with sptr[s] <= start), block and length
__global__ void k_csl_seginfo(const uint32_t* __restrict__ start, int64_t G, uint32_t M,
                              const uint32_t* __restrict__ sptr, int64_t S,
                              const uint32_t* __restrict__ j, uint32_t BB,
                              uint32_t* __restrict__ sslice, uint32_t* __restrict__ sblock,
                              uint32_t* __restrict__ slen) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < G;
       g += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = start[g], b = (g + 1 < G) ? start[g + 1] : M;
    int64_t lo = 0, hi = S;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (sptr[mid] <= a) lo = mid; else hi = mid;
    }
    sslice[g] = uint32_t(lo);
    sblock[g] = j[a] / BB;
    slen[g] = b - a;
  }
}
// virtual slice r = segment order[r]: its length, output row, and the
// inverse map segment -> r
__global__ void k_csl_vslices(const uint32_t* __restrict__ order, int64_t G,
                              const uint32_t* __restrict__ slen, const uint32_t* __restrict__ sslice,
                              const uint32_t* __restrict__ slice_idx, uint32_t* __restrict__ vlen,
                              uint32_t* __restrict__ vsidx, uint32_t* __restrict__ rank_of) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < G;
       r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = order[r];
    vlen[r] = slen[g];
    vsidx[r] = slice_idx[sslice[g]];
    rank_of[g] = uint32_t(r);
  }
}
// nonzero i -> its block-major position: (k | SEND at a segment end, v), j
__global__ void k_csl_vscatter(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ start,
                               const uint32_t* __restrict__ rank_of, const uint32_t* __restrict__ vstart,
                               const uint32_t* __restrict__ k, const uint32_t* __restrict__ j,
                               const float* __restrict__ v, int64_t M, uint2* __restrict__ vpairs,
                               uint32_t* __restrict__ vj, const double* __restrict__ v64,
                               double* __restrict__ vv64) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = pos[i + 1] - 1;
    const bool last = (i + 1 == M) || (pos[i + 2] != pos[i + 1]);
    const uint32_t q = vstart[rank_of[g]] + uint32_t(i - start[g]);
    vpairs[q] = make_uint2(k[i] | (last ? SEND : 0u), __float_as_uint(v[i]));
    vj[q] = j[i];
    if (vv64) vv64[q] = v64[i];
  }
}

__global__ void k_iota_u32(uint32_t* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = uint32_t(i);
}

struct BlockedCsl {
  Buf pairs, j, sidx;
  Buf v64;  // fp64 values in the block-major order (csl_blocked_layout(..., true))
  BucketTasks tasks;
  int64_t G = 0, nblocks = 0;
};

static BlockedCsl csl_blocked_layout(const hbk_csl* c, uint32_t BB, uint32_t T, cudaStream_t st,
                                     bool with_v64 = false) {
  BlockedCsl out;
  const int64_t M = c->M, S = c->S;
  const uint32_t* j = c->rest[0].as<uint32_t>();
  const uint32_t* sptr = c->slice_ptr.as<uint32_t>();
  const uint32_t nb = uint32_t((c->dims[c->mode_order[1]] + BB - 1) / BB);
  out.nblocks = nb;
  Scratch pos((M + 2) * 4, st);
  k_csl_segflags<<<grid_for(M, 256), 256, 0, st>>>(j, M, BB, pos.as<uint32_t>());
  k_csl_slicestarts<<<grid_for(S, 256), 256, 0, st>>>(sptr, S, pos.as<uint32_t>());
  check_launch("k_csl_segflags");
  const uint32_t G = exclusive_scan_total(pos.as<uint32_t>(), M, st);
  out.G = G;
  Scratch start(size_t(G) * 4, st), sslice(size_t(G) * 4, st), sblock(size_t(G) * 4, st),
      slen(size_t(G) * 4, st);
  k_csl_segs<<<grid_for(M, 256), 256, 0, st>>>(pos.as<uint32_t>(), M, start.as<uint32_t>());
  k_csl_seginfo<<<grid_for(G, 256), 256, 0, st>>>(start.as<uint32_t>(), G, uint32_t(M), sptr, S, j,
                                                  BB, sslice.as<uint32_t>(), sblock.as<uint32_t>(),
                                                  slen.as<uint32_t>());
  check_launch("k_csl_seginfo");
  // segments are in (slice, block) order; a stable sort by block gives (block, slice)
  Scratch keys_b(size_t(G) * 4, st), order(size_t(G) * 4, st), iota(size_t(G) * 4, st);
  k_iota_u32<<<grid_for(G, 256), 256, 0, st>>>(iota.as<uint32_t>(), G);
  int bits = 1;
  while ((uint64_t(1) << bits) < nb) ++bits;
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, sblock.as<uint32_t>(), keys_b.as<uint32_t>(),
                                           iota.as<uint32_t>(), order.as<uint32_t>(), int(G), 0, bits, st));
  {
    Scratch t(tmp, st);
    HBK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, sblock.as<uint32_t>(), keys_b.as<uint32_t>(),
                                             iota.as<uint32_t>(), order.as<uint32_t>(), int(G), 0, bits,
                                             st));
  }
  Scratch vstart((size_t(G) + 1) * 4, st), rank_of(size_t(G) * 4, st);
  out.sidx = dalloc(size_t(std::max<uint32_t>(G, 1)) * 4, st);
  k_csl_vslices<<<grid_for(G, 256), 256, 0, st>>>(order.as<uint32_t>(), G, slen.as<uint32_t>(),
                                                  sslice.as<uint32_t>(), c->slice_idx.as<uint32_t>(),
                                                  vstart.as<uint32_t>(), out.sidx.as<uint32_t>(),
                                                  rank_of.as<uint32_t>());
  check_launch("k_csl_vslices");
  const uint32_t total = exclusive_scan_total(vstart.as<uint32_t>(), G, st);
  HBK_REQUIRE(total == uint32_t(M), HBK_ECUDA, "blocked CSL layout accounting mismatch");
  out.pairs = dalloc(size_t(M) * sizeof(uint2), st);
  out.j = dalloc(size_t(M) * 4, st);
  if (with_v64) out.v64 = dalloc(size_t(M) * 8, st);
  k_csl_vscatter<<<grid_for(M, 256), 256, 0, st>>>(pos.as<uint32_t>(), start.as<uint32_t>(),
                                                   rank_of.as<uint32_t>(), vstart.as<uint32_t>(),
                                                   c->rest[1].as<uint32_t>(), j, c->v32.as<float>(), M,
                                                   out.pairs.as<uint2>(), out.j.as<uint32_t>(),
                                                   with_v64 ? c->v64.as<double>() : nullptr,
                                                   with_v64 ? out.v64.as<double>() : nullptr);
  check_launch("k_csl_vscatter");
  // tasks: runs of whole virtual slices, long ones chunked (slot fields only
  // mark chunks: partial rows are added with atomics, no accumulator slots)
  out.tasks = bucket_tasks(vstart.as<uint32_t>(), nullptr, nullptr, G, uint32_t(M), T, st);
  return out;
}

struct HeavyLayout {
  Buf pairs, fj, tasks;
  Buf v64;  // fp64 values of the same stream (heavy_layout(..., val64))
  int64_t ntasks = 0;  // group tasks (4 per warp task)
  int64_t slots = 0;   // heavy slices (one accumulator slot each)
  int64_t segments = 0;
};

// Builds the heavy-slice layout of a 3rd-order CSF bucket (see above).
static HeavyLayout heavy_layout(const hbk_csf* c, const uint32_t* loff, const uint32_t* fpos,
                                uint32_t H, uint32_t tau, uint32_t W, uint32_t slot_base, bool bpos, uint32_t bshift,
                                cudaStream_t st, bool with_v64 = false) {
  HeavyLayout hl;
  const int64_t S = c->n[0], F = c->n[1];
  const uint32_t* lptr = c->ptr[1].as<uint32_t>();
  const uint32_t* fidx = c->idx[1].as<uint32_t>();
  Scratch hflag((S + 1) * 4, st), hoff((S + 1) * 4, st);
  k_heavy_flags<<<grid_for(S, 256), 256, 0, st>>>(loff, S, H, hflag.as<uint32_t>(), hoff.as<uint32_t>());
  check_launch("k_heavy_flags");
  const uint32_t nheavy = exclusive_scan_total(hflag.as<uint32_t>(), S, st);  // -> heavy rank
  if (nheavy == 0) return hl;
  const uint32_t hnnz = exclusive_scan_total(hoff.as<uint32_t>(), S, st);
  // warp-task size: W, or smaller when the heavy slices hold too few nonzeros
  // for ~8 tasks per resident warp (small shards of a multi-GPU partition:
  // the last wave of ~1024-nonzero tasks left the GPU a third idle at 1/8 of
  // nell-2)
  {
    int dev = 0, sms = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // (inputs too small to fill the GPU once keep W: one wave either way)
    const uint64_t want = uint64_t(std::max(sms, 1)) * 24 * 8;
    const uint64_t wmin = std::max<uint32_t>(4 * tau, 128u);
    if (hnnz / want >= wmin) W = uint32_t(std::min<uint64_t>(W, hnnz / want));
  }
  Scratch fslice((F + 1) * 4, st), segoff((F + 1) * 4, st);
  k_fiber_slice<<<grid_for(F, 256), 256, 0, st>>>(fpos, S, F, fslice.as<uint32_t>());
  check_launch("k_fiber_slice");
  k_seg_count<<<grid_for(F, 256), 256, 0, st>>>(fslice.as<uint32_t>(), loff, lptr, F, H, tau,
                                                segoff.as<uint32_t>());
  check_launch("k_seg_count");
  const uint32_t G = exclusive_scan_total(segoff.as<uint32_t>(), F, st);
  hl.segments = G;
  Scratch key_a(size_t(G) * 8, st), key_b(size_t(G) * 8, st), val_a(size_t(G) * 4, st),
      val_b(size_t(G) * 4, st);
  Scratch soff(size_t(G) * 4, st), slen(size_t(G) * 4, st), sj(size_t(G) * 4, st),
      ss(size_t(G) * 4, st);
  k_seg_emit<<<grid_for(F, 256), 256, 0, st>>>(
      fslice.as<uint32_t>(), lptr, fidx, segoff.as<uint32_t>(), F, tau,
      key_a.as<unsigned long long>(), val_a.as<uint32_t>(), soff.as<uint32_t>(),
      slen.as<uint32_t>(), sj.as<uint32_t>(), ss.as<uint32_t>());
  check_launch("k_seg_emit");
  int sbits = 1;
  while ((int64_t(1) << sbits) < S) ++sbits;
  cub::DoubleBuffer<unsigned long long> kb(key_a.as<unsigned long long>(),
                                           key_b.as<unsigned long long>());
  cub::DoubleBuffer<uint32_t> vb(val_a.as<uint32_t>(), val_b.as<uint32_t>());
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, int(G), 0, 16 + sbits, st));
  {
    Scratch t(tmp, st);
    HBK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, int(G), 0, 16 + sbits, st));
  }
  const uint32_t* perm = vb.Current();
  // nonzero prefix of the sorted segments -> local warp task of each segment
  Scratch P((size_t(G) + 1) * 4, st), tloc(size_t(G) * 4, st), ntask((S + 1) * 4, st);
  k_gather_u32<<<grid_for(G, 256), 256, 0, st>>>(slen.as<uint32_t>(), perm, G, P.as<uint32_t>());
  check_launch("k_gather_u32");
  exclusive_scan_total(P.as<uint32_t>(), G, st);
  HBK_CUDA(cudaMemsetAsync(ntask.p, 0, (S + 1) * 4, st));
  k_seg_task<<<grid_for(G, 256), 256, 0, st>>>(perm, slen.as<uint32_t>(), ss.as<uint32_t>(),
                                               P.as<uint32_t>(), hoff.as<uint32_t>(), G, W,
                                               tloc.as<uint32_t>(), ntask.as<uint32_t>());
  check_launch("k_seg_task");
  const uint32_t NW = exclusive_scan_total(ntask.as<uint32_t>(), S, st);  // -> task base
  Scratch tfirst(size_t(NW) * 4, st), tslice(size_t(NW) * 4, st);
  k_seg_task_first<<<grid_for(G, 256), 256, 0, st>>>(perm, ss.as<uint32_t>(), tloc.as<uint32_t>(),
                                                     ntask.as<uint32_t>(), G,
                                                     tfirst.as<uint32_t>(), tslice.as<uint32_t>());
  check_launch("k_seg_task_first");
  const int64_t NG = int64_t(NW) * 4;
  Scratch gofs((NG + 1) * 4, st), gnnz(NG * 4, st), fofs((NG + 1) * 4, st);
  k_group_sizes<<<grid_for(NG, 256), 256, 0, st>>>(tfirst.as<uint32_t>(), perm,
                                                   slen.as<uint32_t>(), NW, G, bpos,
                                                   gofs.as<uint32_t>(), fofs.as<uint32_t>());
  check_launch("k_group_sizes");
  HBK_CUDA(cudaMemcpyAsync(gnnz.p, gofs.p, NG * 4, cudaMemcpyDeviceToDevice, st));
  Scratch gseg(NG * 4, st), nchunk((S + 1) * 4, st);
  HBK_CUDA(cudaMemcpyAsync(gseg.p, fofs.p, NG * 4, cudaMemcpyDeviceToDevice, st));
  const uint32_t Mh = exclusive_scan_total(gofs.as<uint32_t>(), NG, st);
  const uint32_t Fh = exclusive_scan_total(fofs.as<uint32_t>(), NG, st);
  HBK_CUDA(cudaMemsetAsync(nchunk.p, 0, (S + 1) * 4, st));
  k_slice_nchunk<<<grid_for(NW, 256), 256, 0, st>>>(tslice.as<uint32_t>(), gseg.as<uint32_t>(), NW,
                                                    nchunk.as<uint32_t>());
  check_launch("k_slice_nchunk");
  hl.pairs = dalloc(size_t(std::max<uint32_t>(Mh, 1)) * sizeof(uint2), st);
  hl.fj = dalloc(size_t(std::max<uint32_t>(Fh, 1)) * 4, st);
  hl.tasks = dalloc(size_t(NG) * sizeof(Task), st);
  if (with_v64) hl.v64 = dalloc(size_t(std::max<uint32_t>(Mh, 1)) * 8, st);
  k_group_fill<<<grid_for(NG, 128), 128, 0, st>>>(
      tfirst.as<uint32_t>(), perm, soff.as<uint32_t>(), slen.as<uint32_t>(), sj.as<uint32_t>(),
      gofs.as<uint32_t>(), fofs.as<uint32_t>(), NW, G, c->leaf.as<uint32_t>(), c->v32.as<float>(),
      bpos, bshift, hl.pairs.as<uint2>(), hl.fj.as<uint32_t>(),
      with_v64 ? c->v64.as<double>() : nullptr, with_v64 ? hl.v64.as<double>() : nullptr);
  check_launch("k_group_fill");
  k_group_tasks<<<grid_for(NG, 256), 256, 0, st>>>(tslice.as<uint32_t>(), gofs.as<uint32_t>(),
                                                   gnnz.as<uint32_t>(), fofs.as<uint32_t>(),
                                                   hflag.as<uint32_t>(), nchunk.as<uint32_t>(), NW,
                                                   slot_base, hl.tasks.as<Task>());
  check_launch("k_group_tasks");
  hl.ntasks = NG;
  hl.slots = nheavy;
  hl.segments = Fh;
  if (getenv("HBK_DEBUG")) {
    uint32_t heavy_nnz = 0;
    HBK_CUDA(cudaMemcpyAsync(&heavy_nnz, hoff.as<uint32_t>() + S, 4, cudaMemcpyDeviceToHost, st));
    HBK_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "hbk heavy: slices %u nnz %u segments %u warp-tasks %u positions %u (x4 groups)\n",
            nheavy, heavy_nnz, G, NW, Mh);
  }
  HBK_CUDA(cudaStreamSynchronize(st));
  return hl;
}

__global__ void k_shift_slots(Task* __restrict__ t, int64_t n, uint32_t base) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (t[i].slot != NOSLOT) t[i].slot += base;
}

// Resident CTAs per SM of the fast kernel of a kind (k 0 = light CSF,
// 1 = CSL, 2 = COO, 3 = heavy CSF), for the factor shape the plan launches.
template <class FX>
static int fast_occupancy(const hbk_plan* p, int k) {
  int per_sm = 0;
  const void* fn = nullptr;
  if (k == 0)
    fn = p->acc_csf ? reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSF_BPOS4_ACC, FX>)
                    : reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSF_BPOS4, FX>);
  else if (k == 1)
    fn = p->csl_acc ? reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSL_ACC, FX>)
                    : reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSL, FX>);
  else if (k == 2)
    fn = reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_COO, FX>);
  else
    fn = p->acc_csf ? reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSF_UNI_ACC, FX>)
                    : reinterpret_cast<const void*>(k_mttkrp3_r32<KIND_CSF_UNI, FX>);
  HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p->block, 0));
  return per_sm;
}

static int fast_occupancy_any(const hbk_plan* p, int k) {
  return p->r32 ? fast_occupancy<Factors3R32>(p, k) : fast_occupancy<Factors3>(p, k);
}

static void build_plan(hbk_plan* p, cudaStream_t st) {
  const int N = p->order;
  const int R = p->rank;
  // fast path: order 3, R a multiple of 4 (float4 rows; R > 32 runs in
  // passes of 32 columns); the old-variant streams keep two flag bits in the
  // leaf coordinate, so leaf extents must stay < 2^29
  p->fast = !p->force_generic && (N == 3 && R >= 4 && R % 4 == 0 &&
                                   p->dims[p->mo[2]] < (int64_t(1) << 29) &&
                                   p->dims[p->mo[1]] < (int64_t(1) << 29));
  p->r32 = p->fast && R == 32 && p->dims[p->mo[2]] < (int64_t(1) << 27) &&
           p->dims[p->mo[1]] < (int64_t(1) << 27);
  p->bshift = p->r32 ? 3u : 0u;
  const int gpw = p->fast ? 4 : 1;  // task ranges padded so a warp never straddles kinds
  const uint32_t Tcsf = p->fast ? TASK_NNZ_CSF : GEN_TASK_NNZ;
  // CSL runs: 256 nonzeros when the CSL slices average >= 48 (delicious-3d
  // mode 2, 56 per slice: -5%), else 128 (flickr / nell-1, 4-36 per slice)
  uint32_t Tcsl = GEN_TASK_NNZ;
  if (p->fast) {
    Tcsl = (p->csl && p->csl->S && p->csl->M >= 48 * p->csl->S) ? 2 * TASK_NNZ_CSL : TASK_NNZ_CSL;
  }
  // COO / zero-row task sizes: 64-128 and 64-1024 measured within +-2%
  const uint32_t Tcoo = p->fast ? TASK_NNZ_COO : GEN_TASK_NNZ;
  const uint32_t Tzero = TASK_ROWS_ZERO;

  Work& w = p->work;
  std::memset(&w, 0, sizeof(w));
  BucketTasks tcsf, tcsl, tcsf_light, tcsl_fast;
  bool csl_blocked = false;
  // heavy-slice layout (fast path): slices with more than H nonzeros
  // B-position streams (default fast CSF path): every slice with more than
  // Tcsf nonzeros goes to the heavy layout, lighter slices form runs
  // (schedule units run through the same light-slice B-position kernel)
  p->bpos = p->fast;
  const uint32_t heavy_H = Tcsf;
  // segment length tau and warp-task size W of the heavy layout (W 1024 vs
  // 2048: nell-2 -0.9%, others +-0.2%)
  const uint32_t heavy_tau = 32, heavy_W = 1024;
  // A schedule (mttkrp_scheduled / mttkrp_hbcsf(schedule=...)) fixes the
  // OpCount and which slices are split; on the B-position path its slices run
  // through the same layout as the default plan: single-unit slices whole,
  // multi-unit slices (> block_size nonzeros) as ~1024-nonzero warp tasks of
  // the heavy layout (two 512-nonzero units' worth across four 8-lane groups)
  // instead of one light task per unit (nell-2: 1.00 -> 0.72 ms per mode).
  const bool units_as_tasks = p->sched && !p->fast;
  const bool heavy_on = p->fast && !units_as_tasks;
  int64_t heavy_ntasks = 0, heavy_segments = 0;

  int64_t n_coo = 0, n_zero = 0;
  int64_t slots = 0;
  int64_t stream_bytes = 0;
  int64_t muls = 0, adds = 0;

  if (p->csf && p->csf->M > 0) {
    hbk_csf* c = p->csf;
    const int64_t S = c->n[0];
    const int L = N - 2;
    Chain2 ch{};
    ch.nlev = N - 1;
    for (int d = 0; d < N - 1; ++d) ch.ptr[d] = c->ptr[d].as<uint32_t>();
    p->csf_send = dalloc((S + 1) * sizeof(uint32_t), st);
    Scratch fpos((S + 1) * sizeof(uint32_t), st);
    k_csf_slice_offsets<<<grid_for(S + 1, 256), 256, 0, st>>>(ch, S, fpos.as<uint32_t>(),
                                                              p->csf_send.as<uint32_t>());
    check_launch("k_csf_slice_offsets");
    int64_t sched_muls = 0, sched_adds = 0;
    if (p->sched) {
      hbk_sched* sc = p->sched;
      HBK_REQUIRE(sc->S == S && sc->F == c->n[L], HBK_EINVAL,
                  "schedule was built for a different tree");
      if (units_as_tasks) {
        Scratch cnt((S + 1) * sizeof(uint32_t), st), slot((S + 1) * sizeof(uint32_t), st);
        HBK_CUDA(cudaMemsetAsync(cnt.p, 0, (S + 1) * sizeof(uint32_t), st));
        if (sc->U) {
          k_units_per_slice<<<grid_for(sc->U, 256), 256, 0, st>>>(sc->units.as<uint32_t>(), sc->U,
                                                                  cnt.as<uint32_t>());
          check_launch("k_units_per_slice");
        }
        k_slot_flags<<<grid_for(S, 256), 256, 0, st>>>(cnt.as<uint32_t>(), S, slot.as<uint32_t>());
        check_launch("k_slot_flags");
        uint32_t nslot = exclusive_scan_total(slot.as<uint32_t>(), S, st);
        tcsf.tasks = Scratch(size_t(sc->U) * sizeof(Task), st);
        if (sc->U) {
          k_units_to_tasks<<<grid_for(sc->U, 256), 256, 0, st>>>(
              sc->units.as<uint32_t>(), sc->U, c->ptr[L].as<uint32_t>(), cnt.as<uint32_t>(),
              slot.as<uint32_t>(), 0, tcsf.tasks.as<Task>());
          check_launch("k_units_to_tasks");
        }
        tcsf.n = sc->U;
        tcsf.slots = nslot;
      }
      // OpCount of mttkrp_scheduled (kernels.py:283-298, 325-330)
      int64_t mid = 0;
      if (N > 3) {
        // mid-level nodes per unit, computed on the host from the exported
        // pointer arrays (order > 3 only; small parity cases)
        std::vector<std::vector<uint32_t>> ptr(N - 1);
        for (int d = 0; d < N - 1; ++d) {
          ptr[d].resize(c->n[d] + 1);
          HBK_CUDA(cudaMemcpyAsync(ptr[d].data(), c->ptr[d].p, (c->n[d] + 1) * 4,
                                   cudaMemcpyDeviceToHost, st));
        }
        std::vector<uint32_t> hu(sc->U * 3);
        if (sc->U)
          HBK_CUDA(cudaMemcpyAsync(hu.data(), sc->units.p, hu.size() * 4, cudaMemcpyDeviceToHost,
                                   st));
        HBK_CUDA(cudaStreamSynchronize(st));
        for (int64_t u = 0; u < sc->U; ++u) {
          uint32_t lo = hu[3 * u + 1], hi = hu[3 * u + 2];
          for (int d = N - 3; d >= 1; --d) {
            const auto& pd = ptr[d];
            int64_t a = std::upper_bound(pd.begin(), pd.end(), lo) - pd.begin() - 1;
            int64_t b = std::lower_bound(pd.begin(), pd.end(), hi) - pd.begin();
            mid += b - a;
            lo = uint32_t(a);
            hi = uint32_t(b);
          }
        }
      }
      sched_muls = (c->M + c->n[L] + mid) * R;
      sched_adds = (c->M + mid + sc->U) * R;
    }
    if (units_as_tasks) {
      muls += sched_muls;
      adds += sched_adds;
    } else {
      tcsf = bucket_tasks(p->csf_send.as<uint32_t>(), fpos.as<uint32_t>(),
                          c->ptr[L].as<uint32_t>(), S, uint32_t(c->M), Tcsf, st);
      if (heavy_on) {
        tcsf_light = bucket_tasks(p->csf_send.as<uint32_t>(), fpos.as<uint32_t>(),
                                  c->ptr[L].as<uint32_t>(), S, uint32_t(c->M), Tcsf, st, heavy_H,
                                  p->bpos ? fpos.as<uint32_t>() : nullptr);
        HeavyLayout hl = heavy_layout(c, p->csf_send.as<uint32_t>(), fpos.as<uint32_t>(), heavy_H,
                                      heavy_tau, heavy_W, uint32_t(tcsf_light.slots), p->bpos, p->bshift, st);
        p->heavy_H = heavy_H;
        p->heavy_tau = heavy_tau;
        p->heavy_W = heavy_W;
        p->heavy_slot_base = uint32_t(tcsf_light.slots);
        HBK_REQUIRE(tcsf_light.slots + hl.slots == tcsf.slots, HBK_ECUDA,
                    "heavy layout slot accounting mismatch");
        p->heavy_pairs = hl.pairs;
        p->heavy_fj = hl.fj;
        p->heavy_tasks = hl.tasks;
        heavy_ntasks = hl.ntasks;
        heavy_segments = hl.segments;
        p->info.tasks_heavy = hl.ntasks;
      }
      // OpCount of mttkrp_csf (kernels.py:173-185), or of the schedule
      int64_t m = c->M, a = c->M;
      for (int d = N - 2; d >= 1; --d) {
        m += c->n[d];
        if (d < N - 2) a += c->n[d];
      }
      a += c->n[0];
      muls += p->sched ? sched_muls : m * R;
      adds += p->sched ? sched_adds : a * R;
    }
    slots += tcsf.slots;
    w.csf_send = p->csf_send.as<uint32_t>();
    w.csf_sidx = c->idx[0].as<uint32_t>();
    w.csf_lptr = c->ptr[L].as<uint32_t>();
    w.csf_fidx = c->idx[L].as<uint32_t>();
    w.csf_leaf = c->leaf.as<uint32_t>();
    w.csf_val = c->v32.as<float>();
    w.csf_F = uint32_t(c->n[L]);
    w.csf_S = uint32_t(S);
    if (p->bpos) {
      const int64_t P = c->M + c->n[L];
      p->csf_pairs = dalloc(P * sizeof(uint2), st);
      uint2* pp = p->csf_pairs.as<uint2>();
      k_bpos_stream<<<grid_for(c->n[L], 128), 128, 0, st>>>(
          c->ptr[L].as<uint32_t>(), c->idx[L].as<uint32_t>(), c->leaf.as<uint32_t>(),
          c->v32.as<float>(), c->n[L], p->bshift, pp);
      check_launch("k_bpos_stream");
      k_bpos_send<<<grid_for(S, 256), 256, 0, st>>>(fpos.as<uint32_t>(), c->ptr[L].as<uint32_t>(),
                                                    S, pp);
      check_launch("k_bpos_send");
      w.csf_pairs = pp;
    }
    stream_bytes += p->fast ? 8 * c->M + 4 * c->n[L] + 4 * S : 8 * c->M + 8 * c->n[L] + 8 * S;
  }
  if (p->csl && p->csl->M > 0) {
    hbk_csl* s = p->csl;
    tcsl = bucket_tasks(s->slice_ptr.as<uint32_t>(), nullptr, nullptr, s->S, uint32_t(s->M), Tcsl,
                        st);
    if (tcsl.slots) {
      k_shift_slots<<<grid_for(tcsl.n, 256), 256, 0, st>>>(tcsl.tasks.as<Task>(), tcsl.n,
                                                           uint32_t(slots));
      check_launch("k_shift_slots");
    }
    // blocked CSL layout (block size chosen in hbk_plan_create): the fast
    // kernel runs the block-major virtual slices and accumulates rows, so it
    // needs no accumulator slots
    p->csl_T = Tcsl;
    if (p->fast && p->csl_bb > 0) {
      BlockedCsl bl = csl_blocked_layout(s, uint32_t(p->csl_bb), Tcsl, st);
      p->vcsl_pairs = bl.pairs;
      p->vcsl_j = bl.j;
      p->vcsl_sidx = bl.sidx;
      p->vcsl_S = uint32_t(bl.G);
      tcsl_fast = std::move(bl.tasks);
      csl_blocked = true;
      p->csl_acc = true;
      p->info.csl_blocks = bl.nblocks;
    }
    slots += tcsl.slots;
    w.csl_send = s->slice_ptr.as<uint32_t>();
    w.csl_sidx = s->slice_idx.as<uint32_t>();
    w.csl_j = s->rest[0].as<uint32_t>();
    w.csl_k = N >= 3 ? s->rest[1].as<uint32_t>() : nullptr;
    w.csl_val = s->v32.as<float>();
    w.csl_S = uint32_t(s->S);
    if (p->fast) {
      p->csl_pairs = dalloc(s->M * sizeof(uint2), st);
      uint2* pp = p->csl_pairs.as<uint2>();
      k_pairs<<<grid_for(s->M, 256), 256, 0, st>>>(s->rest[1].as<uint32_t>(), s->v32.as<float>(),
                                                   s->M, pp);
      check_launch("k_pairs");
      k_flag_ends<<<grid_for(s->S, 256), 256, 0, st>>>(s->slice_ptr.as<uint32_t>(), s->S, SEND, pp);
      check_launch("k_flag_ends");
      w.csl_pairs = pp;
    }
    muls += int64_t(N - 1) * s->M * R;
    adds += s->M * R;
    stream_bytes += 4 * int64_t(N) * s->M + (p->fast ? 4 : 8) * s->S;
  }
  if (p->coo && p->coo->nnz > 0) {
    hbk_coo* t = p->coo;
    n_coo = (t->nnz + Tcoo - 1) / Tcoo;
    w.coo_i = t->cols[p->mode].as<uint32_t>();
    w.coo_j = t->cols[p->mo[1]].as<uint32_t>();
    w.coo_k = t->cols[p->mo[2]].as<uint32_t>();
    w.coo_val = t->v32.as<float>();
    if (p->fast) {
      p->coo_quads = dalloc(t->nnz * sizeof(uint4), st);
      k_quads<<<grid_for(t->nnz, 256), 256, 0, st>>>(w.coo_i, w.coo_j, w.coo_k, w.coo_val, t->nnz,
                                                     p->coo_quads.as<uint4>());
      check_launch("k_quads");
      w.coo_quads = p->coo_quads.as<uint4>();
    }
    muls += int64_t(N - 1) * t->nnz * R;
    adds += t->nnz * R;
    stream_bytes += 4 * int64_t(N + 1) * t->nnz;
  }
  // rows owned by no bucket
  const int64_t rows = p->dims[p->mode];
  {
    Scratch mark(rows, st);
    HBK_CUDA(cudaMemsetAsync(mark.p, 0, rows, st));
    if (p->csf && p->csf->n[0]) {
      k_mark_rows<<<grid_for(p->csf->n[0], 256), 256, 0, st>>>(p->csf->idx[0].as<uint32_t>(),
                                                               p->csf->n[0], mark.as<uint8_t>());
      check_launch("k_mark_rows");
    }
    if (p->csl && p->csl->S) {
      k_mark_rows<<<grid_for(p->csl->S, 256), 256, 0, st>>>(p->csl->slice_idx.as<uint32_t>(),
                                                            p->csl->S, mark.as<uint8_t>());
      check_launch("k_mark_rows");
    }
    if (p->coo && p->coo->nnz) {
      k_mark_rows<<<grid_for(p->coo->nnz, 256), 256, 0, st>>>(
          p->coo->cols[p->mode].as<uint32_t>(), p->coo->nnz, mark.as<uint8_t>());
      check_launch("k_mark_rows");
    }
    if (p->extra_owned && p->n_extra_owned) {
      k_mark_rows<<<grid_for(p->n_extra_owned, 256), 256, 0, st>>>(
          p->extra_owned->as<uint32_t>(), p->n_extra_owned, mark.as<uint8_t>());
      check_launch("k_mark_rows");
    }
    if (p->acc_csf) HBK_CUDA(cudaMemsetAsync(mark.p, 1, rows, st));  // sub_blk writes no zero rows
    Scratch pos((rows + 1) * sizeof(uint32_t), st);
    k_unmarked_flags<<<grid_for(rows, 256), 256, 0, st>>>(mark.as<uint8_t>(), rows,
                                                          pos.as<uint32_t>());
    check_launch("k_unmarked_flags");
    uint32_t Z = exclusive_scan_total(pos.as<uint32_t>(), rows, st);
    p->zero_rows = dalloc(size_t(Z) * sizeof(uint32_t), st);
    if (Z) {
      k_unmarked_emit<<<grid_for(rows, 256), 256, 0, st>>>(pos.as<uint32_t>(), rows,
                                                           p->zero_rows.as<uint32_t>());
      check_launch("k_unmarked_emit");
    }
    n_zero = (Z + Tzero - 1) / Tzero;
    w.zero_rows = p->zero_rows.as<uint32_t>();
    p->info.tasks_zero = n_zero;
    // assemble [CSF | CSL | COO | ZERO], each padded to a multiple of gpw
    auto assemble = [&](const BucketTasks& tc, const BucketTasks& tl, Buf& store, Work& wo) {
      const int64_t a0 = pad_to(tc.n, gpw), a1 = pad_to(tl.n, gpw), a2 = pad_to(n_coo, gpw),
                    a3 = pad_to(n_zero, gpw);
      const int64_t total = a0 + a1 + a2 + a3;
      store = dalloc(std::max<int64_t>(total, 1) * sizeof(Task), st);
      Task* T = store.as<Task>();
      if (total) {
        k_empty_tasks<<<grid_for(total, 256), 256, 0, st>>>(T, total);
        check_launch("k_empty_tasks");
      }
      if (tc.n)
        HBK_CUDA(cudaMemcpyAsync(T, tc.tasks.p, tc.n * sizeof(Task), cudaMemcpyDeviceToDevice, st));
      if (tl.n)
        HBK_CUDA(cudaMemcpyAsync(T + a0, tl.tasks.p, tl.n * sizeof(Task),
                                 cudaMemcpyDeviceToDevice, st));
      if (n_coo) {
        k_range_tasks<<<grid_for(n_coo, 256), 256, 0, st>>>(T + a0 + a1, n_coo,
                                                            uint32_t(p->coo->nnz), Tcoo);
        check_launch("k_range_tasks");
      }
      if (n_zero) {
        k_range_tasks<<<grid_for(n_zero, 256), 256, 0, st>>>(T + a0 + a1 + a2, n_zero, Z,
                                                             Tzero);
        check_launch("k_range_tasks");
      }
      wo.n0 = uint32_t(a0);
      wo.n1 = uint32_t(a0 + a1);
      wo.n2 = uint32_t(a0 + a1 + a2);
      wo.n3 = uint32_t(total);
      wo.tasks = T;
    };
    if (heavy_on || csl_blocked) {
      assemble(heavy_on ? tcsf_light : tcsf, csl_blocked ? tcsl_fast : tcsl,
               p->tasks, w);
      assemble(tcsf, tcsl, p->gen_tasks, p->work_gen);
    } else {
      assemble(tcsf, tcsl, p->tasks, w);
    }
    p->info.tasks_csf = heavy_on ? tcsf_light.n : tcsf.n;
    p->info.tasks_csl = csl_blocked ? tcsl_fast.n : tcsl.n;
    p->info.tasks_coo = n_coo;
  }
  // workspace: [ctr(2) pad to 32 words][cnt slots][acc slots x R]
  const size_t cnt_off = 32 * sizeof(uint32_t);
  const size_t acc_off = pad_to(cnt_off + slots * sizeof(uint32_t), 256);
  const size_t ws_bytes = acc_off + size_t(slots) * R * sizeof(double);  // fp64 mode shares it
  p->ws = dalloc(ws_bytes, st);
  HBK_CUDA(cudaMemsetAsync(p->ws.p, 0, ws_bytes, st));
  w.ws_ctr = reinterpret_cast<uint32_t*>(p->ws.as<char>());
  w.ws_cnt = reinterpret_cast<uint32_t*>(p->ws.as<char>() + cnt_off);
  w.ws_acc = reinterpret_cast<float*>(p->ws.as<char>() + acc_off);
  if (!heavy_on && !csl_blocked) {
    p->work_gen = w;
  } else {
    Work& wg = p->work_gen;
    const Work keep = wg;
    wg = w;
    wg.n0 = keep.n0;
    wg.n1 = keep.n1;
    wg.n2 = keep.n2;
    wg.n3 = keep.n3;
    wg.tasks = keep.tasks;
  }
  if (p->csl_acc) {  // the fast kernels read the block-major CSL stream
    w.csl_pairs = p->vcsl_pairs.as<uint2>();
    w.csl_j = p->vcsl_j.as<uint32_t>();
    w.csl_sidx = p->vcsl_sidx.as<uint32_t>();
    w.csl_S = p->vcsl_S;
  }

  // persistent grid: as many CTAs as fit, a multiple of the SM count
  int dev = 0, sms = 0, per_sm = 0;
  HBK_CUDA(cudaGetDevice(&dev));
  HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  auto grid_for_tasks = [&](int64_t ntask, int per, int tasks_per_warp) {
    per = std::max(per, 1);
    const int64_t want = int64_t(sms) * per;
    const int64_t warps_needed = (ntask + tasks_per_warp - 1) / tasks_per_warp;
    const int64_t blocks_needed = std::max<int64_t>(1, (warps_needed + 7) / 8);
    return int(std::min(want, blocks_needed));
  };
  int launches = 0;
  if (p->fast) {
    p->block = FAST_BLOCK;
    const int64_t ntk[3] = {int64_t(w.n0), int64_t(w.n1) - w.n0, int64_t(w.n3) - w.n1};
    for (int k = 0; k < 3; ++k) {
      per_sm = fast_occupancy_any(p, k);
      p->grids[k] = ntk[k] > 0 ? grid_for_tasks(ntk[k], per_sm, 4) : 0;
      w.total_warps[k] = uint32_t(p->grids[k]) * (p->block / 32);
      launches += ntk[k] > 0;
    }
    if (heavy_ntasks) {
      Work& wh = p->work_heavy;
      wh = w;
      wh.n0 = uint32_t(heavy_ntasks);
      wh.n1 = wh.n2 = wh.n3 = wh.n0;
      wh.tasks = p->heavy_tasks.as<Task>();
      wh.csf_pairs = p->heavy_pairs.as<uint2>();
      wh.csf_fidx = p->heavy_fj.as<uint32_t>();
      wh.csf_F = uint32_t(heavy_segments);
      per_sm = fast_occupancy_any(p, 3);
      p->grid_heavy = grid_for_tasks(heavy_ntasks, per_sm, 4);
      wh.total_warps[0] = uint32_t(p->grid_heavy) * (p->block / 32);
      launches += 1;
    }
    // a plan with no task at all still launches once (nothing to write, but
    // keeps launch accounting uniform)
    if (launches == 0) {
      p->grids[2] = 1;
      w.total_warps[2] = p->block / 32;
      launches = 1;
    }
  } else {
    launches = 1;
  }
  // generic (any order / rank, fp32 or fp64) launch configuration, available
  // on every plan: one warp per task
  {
    int per_gen = 0;
    HBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_gen, k_mttkrp_generic<double>, 256, 0));
    p->gen_grid = grid_for_tasks(p->work_gen.n3, per_gen, 1);
  }

  p->info.mode = p->mode;
  p->info.rank = R;
  p->info.out_rows = rows;
  p->info.split_rows = slots;
  p->info.launches = p->fast ? int64_t(launches) * ((R + 31) / 32) : launches;
  {
    const char* e = getenv("HBK_CONCURRENT");
    p->concurrent = p->fast && p->bpos && launches > 1 && !(e && atoi(e) == 0);
    if (p->concurrent) {
      HBK_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
      for (int i = 0; i < 3; ++i) {
        HBK_CUDA(cudaStreamCreateWithFlags(&p->side[i], cudaStreamNonBlocking));
        HBK_CUDA(cudaEventCreateWithFlags(&p->ev_join[i], cudaEventDisableTiming));
      }
    }
  }
  p->info.fast_path = p->fast;
  int64_t nnz = 0;
  if (p->csf) nnz += p->csf->M;
  if (p->csl) nnz += p->csl->M;
  if (p->coo) nnz += p->coo->nnz;
  p->info.nnz = nnz;
  if (nnz == 0) muls = adds = 0;
  p->info.op_muls = muls;
  p->info.op_adds = adds;
  p->info.stream_bytes = stream_bytes;
  // rows one execute gathers (B-position plans): CSF positions + 2 per CSL/COO nonzero
  if (p->bpos) {
    Scratch acc(4 * 8, st);
    HBK_CUDA(cudaMemsetAsync(acc.p, 0, 4 * 8, st));
    unsigned long long* a = acc.as<unsigned long long>();
    if (w.n0) k_task_span<<<grid_for(w.n0, 256), 256, 0, st>>>(w.tasks, w.n0, a + 0);
    if (heavy_ntasks)
      k_task_span<<<grid_for(heavy_ntasks, 256), 256, 0, st>>>(p->heavy_tasks.as<Task>(),
                                                              heavy_ntasks, a + 1);
    if (w.n1 > w.n0) k_task_span<<<grid_for(w.n1 - w.n0, 256), 256, 0, st>>>(w.tasks + w.n0,
                                                                           w.n1 - w.n0, a + 2);
    check_launch("k_task_span");
    unsigned long long h[4] = {0, 0, 0, 0};
    HBK_CUDA(cudaMemcpyAsync(h, a, sizeof(h), cudaMemcpyDeviceToHost, st));
    HBK_CUDA(cudaStreamSynchronize(st));
    p->info.gather_rows = int64_t(h[0] + h[1] + 2 * h[2]) + 2 * (p->coo ? p->coo->nnz : 0);
    p->probe_sink = dalloc(size_t(sms) * 8 * FAST_BLOCK * sizeof(float4), st);
  }
  HBK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hbk

namespace hbk {
// Generic (any order, any rank) launch in fp32 or fp64.  The fp64 variant
// reads the buckets' original fp64 values and accumulates in fp64.
template <class T>
static void launch_generic(const hbk_plan* p, const T* const* factors, T* out, cudaStream_t st) {
  const int N = p->order;
  WorkN<T> wn{};
  wn.order = N;
  wn.rank = p->rank;
  wn.mode = p->mode;
  for (int d = 0; d < N; ++d) {
    wn.F[d] = factors[p->mo[d]];
    wn.Fcoo[d] = factors[d];
  }
  auto vals = [](const Buf& v32, const Buf& v64) -> const T* {
    if constexpr (sizeof(T) == 8) {
      HBK_REQUIRE(bool(v64), HBK_EINVAL, "fp64 MTTKRP needs a tensor created with fp64 values");
      return v64.as<T>();
    } else {
      (void)v64;
      return v32.as<T>();
    }
  };
  if (p->csf) {
    for (int d = 1; d < N - 2; ++d) wn.csf_anc[d] = p->csf->anc[d].as<uint32_t>();
    if (p->csf->M) wn.csf_val = vals(p->csf->v32, p->csf->v64);
  }
  if (p->csl) {
    for (int c = 0; c < N - 1; ++c) wn.csl_rest[c] = p->csl->rest[c].as<uint32_t>();
    if (p->csl->M) wn.csl_val = vals(p->csl->v32, p->csl->v64);
  }
  if (p->coo) {
    for (int d = 0; d < N; ++d) wn.coo_col[d] = p->coo->cols[d].as<uint32_t>();
    if (p->coo->nnz) wn.coo_val = vals(p->coo->v32, p->coo->v64);
  }
  wn.acc = reinterpret_cast<T*>(p->work.ws_acc);
  wn.out = out;
  Work w = p->work_gen;
  w.total_warps[0] = uint32_t(p->gen_grid) * (p->block / 32);
  // the generic kernel pulls single tasks; reuse the fp32 generic counter slot
  k_mttkrp_generic<T><<<p->gen_grid, 256, 0, st>>>(w, wn);
  check_launch("k_mttkrp_generic");
}
}  // namespace hbk

using namespace hbk;

namespace hbk {
__global__ void k_zero_rows(const uint32_t* __restrict__ rows, int64_t n, uint32_t rs,
                            float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n * rs;
       i += int64_t(gridDim.x) * blockDim.x)
    out[size_t(rows[i / rs]) * rs + i % rs] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// A plan's bucket kernels in launch order — heavy slices first (the
// longest), then light CSF, CSL, COO/zero — each on the stream `next()` hands out.
template <class FX, class Next>
static void launch_kernels(const hbk_plan* p, const FX& fx, bool skip_zero, Next&& next,
                           const Work* wl = nullptr, const Work* wh = nullptr) {
  const Work& W = wl ? *wl : p->work;          // light CSF, CSL, COO, zero rows
  const Work& WH = wh ? *wh : p->work_heavy;   // heavy slices
  if (p->grid_heavy) {
    cudaStream_t s2 = next();
    if (p->acc_csf)
      k_mttkrp3_r32<KIND_CSF_UNI_ACC, FX><<<p->grid_heavy, p->block, 0, s2>>>(WH, fx);
    else
      k_mttkrp3_r32<KIND_CSF_UNI, FX><<<p->grid_heavy, p->block, 0, s2>>>(WH, fx);
  }
  if (p->grids[0]) {
    cudaStream_t s2 = next();
    if (p->acc_csf)
      k_mttkrp3_r32<KIND_CSF_BPOS4_ACC, FX><<<p->grids[0], p->block, 0, s2>>>(W, fx);
    else
      k_mttkrp3_r32<KIND_CSF_BPOS4, FX><<<p->grids[0], p->block, 0, s2>>>(W, fx);
  }
  if (p->grids[1]) {
    cudaStream_t s2 = next();
    if (p->csl_acc)
      k_mttkrp3_r32<KIND_CSL_ACC, FX><<<p->grids[1], p->block, 0, s2>>>(W, fx);
    else
      k_mttkrp3_r32<KIND_CSL, FX><<<p->grids[1], p->block, 0, s2>>>(W, fx);
  }
  // skip_zero: the rows no bucket owns are left unwritten (COO tasks only)
  Work wc = W;
  if (skip_zero) wc.n3 = wc.n2;
  if (p->grids[2] && wc.n3 > wc.n1) {
    cudaStream_t s2 = next();
    k_mttkrp3_r32<KIND_COO, FX><<<p->grids[2], p->block, 0, s2>>>(wc, fx);
  }
  check_launch("k_mttkrp3_r32");
}

// Fork / join over `nside` side streams: the first kernel runs on st, each
// later one on its own side stream forked from st (persistent kernels with
// full-occupancy grids, so the next one's CTAs fill the SMs the previous
// one's finishing CTAs free — the launch tails overlap).
struct Forker {
  cudaStream_t st;
  const cudaStream_t* side;
  const cudaEvent_t* join;
  cudaEvent_t fork;
  int nside, n = 0;
  cudaStream_t operator()() {
    if (fork == nullptr || n == 0) {
      ++n;
      return st;
    }
    HBK_REQUIRE(n - 1 < nside, HBK_ECUDA, "not enough side streams");
    cudaStream_t s2 = side[n - 1];
    HBK_CUDA(cudaStreamWaitEvent(s2, fork, 0));
    ++n;
    return s2;
  }
  void begin() {
    if (fork) HBK_CUDA(cudaEventRecord(fork, st));
  }
  void end() {
    if (fork)
      for (int i = 0; i + 1 < n; ++i) {
        HBK_CUDA(cudaEventRecord(join[i], side[i]));
        HBK_CUDA(cudaStreamWaitEvent(st, join[i], 0));
      }
  }
};

template <class FX>
static void launch_fast(const hbk_plan* p, const FX& fx, cudaStream_t st, bool skip_zero = false) {
  Forker f{st, p->side, p->ev_join, p->concurrent ? p->ev_fork : nullptr, 3};
  f.begin();
  launch_kernels(p, fx, skip_zero, f);
  f.end();
}

// fp64 fast path: the same kernels instantiated on double2 lane vectors (a
// pass covers 16 columns), over the plan's task lists and index streams plus
// double value streams built on the first fp64 execution.  Plans whose
// layouts have no fp64 stream yet (blocked CSL, leaf-blocked sub-plans) and
// tensors without fp64 values keep the generic kernel.
static bool ensure_f64(const hbk_plan* p, cudaStream_t st) {
  if (p->f64_state) return p->f64_state > 0;
  p->f64_state = -1;
  if (p->sub_blk) {  // leaf-blocked: both sub-plans need their streams
    if (const char* e = getenv("HBK_F64_GENERIC"))
      if (atoi(e) != 0) return false;
    const bool ok = ensure_f64(p->sub_blk, st) && ensure_f64(p->sub_main, st);
    p->f64_state = ok ? 1 : -1;
    return ok;
  }
  if (!p->fast || !p->bpos || p->order != 3) return false;
  if (const char* e = getenv("HBK_F64_GENERIC"))  // A/B, and the independent fp64 check
    if (atoi(e) != 0) return false;
  if ((p->csf && p->csf->M && !p->csf->v64) || (p->csl && p->csl->M && !p->csl->v64) ||
      (p->coo && p->coo->nnz && !p->coo->v64))
    return false;
  Work w = p->work, wh = p->work_heavy;
  if (p->csf && p->csf->M) {
    const hbk_csf* c = p->csf;
    const int64_t S = c->n[0], F = c->n[1];
    p->csf_v64s = dalloc(size_t(c->M + F) * 8, st);
    k_bpos_v64<<<grid_for(F, 128), 128, 0, st>>>(c->ptr[1].as<uint32_t>(), c->v64.as<double>(), F,
                                                 p->csf_v64s.as<double>());
    check_launch("k_bpos_v64");
    w.csf_v64 = p->csf_v64s.as<double>();
    if (p->grid_heavy) {
      // the heavy layout again (deterministic), emitting its fp64 values
      Chain2 ch{};
      ch.nlev = 2;
      for (int d = 0; d < 2; ++d) ch.ptr[d] = c->ptr[d].as<uint32_t>();
      Scratch loff((S + 1) * 4, st), fpos((S + 1) * 4, st);
      k_csf_slice_offsets<<<grid_for(S + 1, 256), 256, 0, st>>>(ch, S, fpos.as<uint32_t>(),
                                                                loff.as<uint32_t>());
      check_launch("k_csf_slice_offsets");
      HeavyLayout hl = heavy_layout(c, loff.as<uint32_t>(), fpos.as<uint32_t>(), p->heavy_H, p->heavy_tau,
                                    p->heavy_W, p->heavy_slot_base, p->bpos, p->bshift, st, true);
      HBK_REQUIRE(hl.ntasks == int64_t(p->work_heavy.n0), HBK_ECUDA, "fp64 heavy layout mismatch");
      p->heavy_v64s = hl.v64;
      wh.csf_v64 = p->heavy_v64s.as<double>();
    }
  }
  if (p->csl && p->csl->M) {
    if (p->csl_acc) {  // the block-major CSL stream again (deterministic), with fp64 values
      BlockedCsl bl = csl_blocked_layout(p->csl, uint32_t(p->csl_bb), p->csl_T, st, true);
      HBK_REQUIRE(bl.G == int64_t(p->vcsl_S), HBK_ECUDA, "fp64 blocked CSL layout mismatch");
      p->csl_v64s = bl.v64;
      w.csl_v64 = p->csl_v64s.as<double>();
    } else {
      w.csl_v64 = p->csl->v64.as<double>();
    }
  }
  if (p->coo && p->coo->nnz) w.coo_v64 = p->coo->v64.as<double>();
  p->work64 = w;
  p->work_heavy64 = wh;
  HBK_CUDA(cudaStreamSynchronize(st));
  p->f64_state = 1;
  return true;
}

template <class FX>
static void launch_fast64(const hbk_plan* p, const FX& fx, cudaStream_t st) {
  Forker f{st, p->side, p->ev_join, p->concurrent ? p->ev_fork : nullptr, 3};
  f.begin();
  launch_kernels(p, fx, false, f, &p->work64, &p->work_heavy64);
  f.end();
}

template <class FX>
static void launch_blocked64(const hbk_plan* p, const FX& fx, cudaStream_t st) {
  Forker f{st, p->side_all, p->ev_join_all, p->ev_fork, 7};
  f.begin();
  launch_kernels(p->sub_blk, fx, false, f, &p->sub_blk->work64, &p->sub_blk->work_heavy64);
  launch_kernels(p->sub_main, fx, false, f, &p->sub_main->work64, &p->sub_main->work_heavy64);
  f.end();
}

// The leaf-blocked pair: the blocked sub-plan's kernels first, the main
// sub-plan's after them, all under one fork so their tails overlap too.
template <class FX>
static void launch_blocked(const hbk_plan* p, const FX& fx, cudaStream_t st, bool skip_zero) {
  Forker f{st, p->side_all, p->ev_join_all, p->ev_fork, 7};
  f.begin();
  launch_kernels(p->sub_blk, fx, false, f);
  launch_kernels(p->sub_main, fx, skip_zero, f);
  f.end();
}

// Orders executions of one plan (see hbk_plan::exec_mu).  Inside a CUDA
// graph capture the capturing stream already orders the replays, and an
// event recorded outside the capture may not be waited on, so capture skips it.
struct ExecOrder {
  const hbk_plan* p;
  cudaStream_t st;
  bool capturing = false;
  std::lock_guard<std::mutex> lk;
  ExecOrder(const hbk_plan* plan, cudaStream_t s) : p(plan), st(s), lk(plan->exec_mu) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    HBK_CUDA(cudaStreamIsCapturing(st, &cs));
    capturing = cs != cudaStreamCaptureStatusNone;
    if (!capturing) HBK_CUDA(cudaStreamWaitEvent(st, p->ev_last, 0));
  }
  void done() {
    if (!capturing) HBK_CUDA(cudaEventRecord(p->ev_last, st));
  }
};
}  // namespace hbk

extern "C" {

namespace hbk {
__global__ void k_offset_copy(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                              int64_t n, uint32_t add) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i] + add;
}
__global__ void k_iota_from(uint32_t* __restrict__ dst, int64_t n, uint32_t first) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = first + uint32_t(i);
}

// An order-3 HB-CSF plan runs its CSL slices as CSF slices with singleton
// fibers (one fiber per nonzero): the B-position stream, the light-run and
// heavy-slice layouts then cover them, which measured faster than the CSL
// kernel (B-CSF vs HB-CSF on delicious-3d).  The merged tree is plan-
// internal: CSF slices first, then the CSL slices (the kernels do not need
// slices sorted by index); the caller's parts are untouched.
static hbk_csf* merge_csl_as_csf(const hbk_csf* c, const hbk_csl* l, cudaStream_t st) {
  hbk_csf* m = new hbk_csf();
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> guard(m, [](hbk_csf* q) { hbk_csf_release(q); });
  m->order = 3;
  std::copy(l->dims, l->dims + 3, m->dims);
  std::copy(l->mode_order, l->mode_order + 3, m->mode_order);
  const int64_t S0 = c ? c->n[0] : 0, F0 = c ? c->n[1] : 0, M0 = c ? c->M : 0;
  const int64_t S1 = l->S, M1 = l->M;
  m->n[0] = S0 + S1;
  m->n[1] = F0 + M1;
  m->M = M0 + M1;
  m->split = c ? c->split : false;
  auto cat = [&](Buf& dst, const Buf* a, int64_t na, const Buf& b, int64_t nb, size_t es) {
    dst = dalloc(size_t(std::max<int64_t>(na + nb, 1)) * es, st);
    if (na) HBK_CUDA(cudaMemcpyAsync(dst.p, a->p, size_t(na) * es, cudaMemcpyDeviceToDevice, st));
    if (nb)
      HBK_CUDA(cudaMemcpyAsync(dst.as<char>() + size_t(na) * es, b.p, size_t(nb) * es,
                               cudaMemcpyDeviceToDevice, st));
  };
  // level 0: slice -> fiber offsets; CSL fibers are its nonzeros
  m->ptr[0] = dalloc(size_t(S0 + S1 + 1) * 4, st);
  if (c) HBK_CUDA(cudaMemcpyAsync(m->ptr[0].p, c->ptr[0].p, size_t(S0 + 1) * 4,
                                  cudaMemcpyDeviceToDevice, st));
  else HBK_CUDA(cudaMemsetAsync(m->ptr[0].p, 0, 4, st));
  if (S1)
    k_offset_copy<<<grid_for(S1, 256), 256, 0, st>>>(m->ptr[0].as<uint32_t>() + S0 + 1,
                                                     l->slice_ptr.as<uint32_t>() + 1, S1,
                                                     uint32_t(F0));
  cat(m->idx[0], c ? &c->idx[0] : nullptr, S0, l->slice_idx, S1, 4);
  // level 1: fiber -> leaf offsets; one leaf per CSL fiber
  m->ptr[1] = dalloc(size_t(F0 + M1 + 1) * 4, st);
  if (c) HBK_CUDA(cudaMemcpyAsync(m->ptr[1].p, c->ptr[1].p, size_t(F0 + 1) * 4,
                                  cudaMemcpyDeviceToDevice, st));
  else HBK_CUDA(cudaMemsetAsync(m->ptr[1].p, 0, 4, st));
  if (M1)
    k_iota_from<<<grid_for(M1, 256), 256, 0, st>>>(m->ptr[1].as<uint32_t>() + F0 + 1, M1,
                                                   uint32_t(M0 + 1));
  cat(m->idx[1], c ? &c->idx[1] : nullptr, F0, l->rest[0], M1, 4);
  cat(m->leaf, c ? &c->leaf : nullptr, M0, l->rest[1], M1, 4);
  cat(m->v32, c ? &c->v32 : nullptr, M0, l->v32, M1, 4);
  if ((!c || c->v64 || M0 == 0) && (l->v64 || M1 == 0))
    cat(m->v64, c ? &c->v64 : nullptr, c && c->v64 ? M0 : 0, l->v64, M1, 8);
  check_launch("merge_csl_as_csf");
  return guard.release();
}

// ------------------------------------------------- leaf-blocked view --
// csf_block_view(c, sel, want, BB): the order-3 tree of the slices with
// sel[s] == want, its nonzeros reordered leaf-block-major — (block of BB leaf
// rows, slice, fiber, leaf) — with every (block, slice) a virtual slice and
// every (block, fiber) a virtual fiber (BB = 0: no blocking, the selected
// slices in tree order).  A slice's virtual slices all name its output row,
// so a plan over the view must accumulate rows (hbk_plan::acc_csf).
__global__ void k_nz_fiber(const uint32_t* __restrict__ fptr, int64_t F, int64_t M,
                           uint32_t* __restrict__ nzf) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = F;  // last f with fptr[f] <= i
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (fptr[mid] <= uint32_t(i)) lo = mid; else hi = mid;
    }
    nzf[i] = uint32_t(lo);
  }
}
__global__ void k_view_keep(const uint32_t* __restrict__ nzf, const uint32_t* __restrict__ fslice,
                            const uint8_t* __restrict__ sel, uint8_t want, int64_t M,
                            uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    flag[i] = sel[fslice[nzf[i]]] == want;
}
__global__ void k_view_gather(const uint32_t* __restrict__ pos, int64_t M, const uint32_t* __restrict__ leaf,
                              uint32_t BB, uint32_t* __restrict__ blk, uint32_t* __restrict__ src) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    if (pos[i + 1] != pos[i]) {
      blk[pos[i]] = BB ? leaf[i] / BB : 0u;
      src[pos[i]] = uint32_t(i);
    }
}
// per kept element q (after the block sort): source nonzero src[q]; flags of
// virtual-fiber and virtual-slice starts
__global__ void k_view_flags(const uint32_t* __restrict__ src, const uint32_t* __restrict__ blk,
                             const uint32_t* __restrict__ nzf, const uint32_t* __restrict__ fslice,
                             int64_t K, uint32_t* __restrict__ ffl, uint32_t* __restrict__ sfl) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < K;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = nzf[src[q]];
    bool nf = q == 0, ns = q == 0;
    if (q > 0) {
      const uint32_t f0 = nzf[src[q - 1]];
      const bool nb = blk[q] != blk[q - 1];
      nf = nb || f != f0;
      ns = nb || fslice[f] != fslice[f0];
    }
    ffl[q] = nf;
    sfl[q] = ns;
  }
}
__global__ void k_view_fill(const uint32_t* __restrict__ src, const uint32_t* __restrict__ nzf,
                            const uint32_t* __restrict__ fslice, const uint32_t* __restrict__ fpos,
                            const uint32_t* __restrict__ spos, int64_t K,
                            const uint32_t* __restrict__ leaf, const float* __restrict__ v32,
                            const double* __restrict__ v64, const uint32_t* __restrict__ fidx,
                            const uint32_t* __restrict__ sidx, uint32_t* __restrict__ vleaf,
                            float* __restrict__ vv32, double* __restrict__ vv64,
                            uint32_t* __restrict__ vfptr, uint32_t* __restrict__ vfidx,
                            uint32_t* __restrict__ vsptr, uint32_t* __restrict__ vsidx) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < K;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t i = src[q], f = nzf[i];
    vleaf[q] = leaf[i];
    vv32[q] = v32[i];
    if (vv64) vv64[q] = v64[i];
    if (fpos[q + 1] != fpos[q]) {  // virtual fiber start
      const uint32_t vf = fpos[q];
      vfptr[vf] = uint32_t(q);
      vfidx[vf] = fidx[f];
      if (spos[q + 1] != spos[q]) {  // virtual slice start (always a fiber start)
        vsptr[spos[q]] = vf;
        vsidx[spos[q]] = sidx[fslice[f]];
      }
    }
  }
}

static hbk_csf* csf_block_view(const hbk_csf* c, const uint8_t* sel, bool want, int64_t BB,
                               cudaStream_t st) {
  HBK_REQUIRE(c->order == 3, HBK_EINVAL, "leaf-blocked view needs an order-3 tree");
  hbk_csf* m = new hbk_csf();
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> guard(m, [](hbk_csf* q) { hbk_csf_release(q); });
  m->order = 3;
  std::copy(c->dims, c->dims + 3, m->dims);
  std::copy(c->mode_order, c->mode_order + 3, m->mode_order);
  m->split = c->split;
  const int64_t S = c->n[0], F = c->n[1], M = c->M;
  Scratch nzf(size_t(std::max<int64_t>(M, 1)) * 4, st), fsl(size_t(std::max<int64_t>(F, 1)) * 4, st);
  if (M) {
    k_nz_fiber<<<grid_for(M, 256), 256, 0, st>>>(c->ptr[1].as<uint32_t>(), F, M, nzf.as<uint32_t>());
    k_fiber_slice<<<grid_for(F, 256), 256, 0, st>>>(c->ptr[0].as<uint32_t>(), S, F, fsl.as<uint32_t>());
    check_launch("k_nz_fiber");
  }
  Scratch pos((M + 1) * 4, st);
  if (M) {
    k_view_keep<<<grid_for(M, 256), 256, 0, st>>>(nzf.as<uint32_t>(), fsl.as<uint32_t>(), sel,
                                                  uint8_t(want), M, pos.as<uint32_t>());
    check_launch("k_view_keep");
  }
  const uint32_t K = M ? exclusive_scan_total(pos.as<uint32_t>(), M, st) : 0u;
  Scratch blk_a(size_t(std::max<uint32_t>(K, 1)) * 4, st), src_a(size_t(std::max<uint32_t>(K, 1)) * 4, st);
  Scratch blk_b(size_t(std::max<uint32_t>(K, 1)) * 4, st), src_b(size_t(std::max<uint32_t>(K, 1)) * 4, st);
  if (K) {
    k_view_gather<<<grid_for(M, 256), 256, 0, st>>>(pos.as<uint32_t>(), M, c->leaf.as<uint32_t>(),
                                                    uint32_t(BB), blk_a.as<uint32_t>(), src_a.as<uint32_t>());
    check_launch("k_view_gather");
  }
  const uint32_t* blk = blk_a.as<uint32_t>();
  const uint32_t* src = src_a.as<uint32_t>();
  if (K && BB > 0) {
    const int64_t nb = (c->dims[c->mode_order[2]] + BB - 1) / BB;
    int bits = 1;
    while ((int64_t(1) << bits) < nb) ++bits;
    size_t tmp = 0;
    HBK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, blk_a.as<uint32_t>(), blk_b.as<uint32_t>(),
                                             src_a.as<uint32_t>(), src_b.as<uint32_t>(), int(K), 0, bits, st));
    Scratch t(tmp, st);
    HBK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, blk_a.as<uint32_t>(), blk_b.as<uint32_t>(),
                                             src_a.as<uint32_t>(), src_b.as<uint32_t>(), int(K), 0, bits, st));
    blk = blk_b.as<uint32_t>();
    src = src_b.as<uint32_t>();
  }
  Scratch fpos((size_t(K) + 1) * 4, st), spos((size_t(K) + 1) * 4, st);
  if (K) {
    k_view_flags<<<grid_for(K, 256), 256, 0, st>>>(src, blk, nzf.as<uint32_t>(), fsl.as<uint32_t>(), K,
                                                   fpos.as<uint32_t>(), spos.as<uint32_t>());
    check_launch("k_view_flags");
  }
  const uint32_t VF = K ? exclusive_scan_total(fpos.as<uint32_t>(), K, st) : 0u;
  const uint32_t VS = K ? exclusive_scan_total(spos.as<uint32_t>(), K, st) : 0u;
  m->M = K;
  m->n[0] = VS;
  m->n[1] = VF;
  m->ptr[0] = dalloc(size_t(VS + 1) * 4, st);
  m->idx[0] = dalloc(size_t(std::max<uint32_t>(VS, 1)) * 4, st);
  m->ptr[1] = dalloc(size_t(VF + 1) * 4, st);
  m->idx[1] = dalloc(size_t(std::max<uint32_t>(VF, 1)) * 4, st);
  m->leaf = dalloc(size_t(std::max<uint32_t>(K, 1)) * 4, st);
  m->v32 = dalloc(size_t(std::max<uint32_t>(K, 1)) * 4, st);
  if (c->v64) m->v64 = dalloc(size_t(std::max<uint32_t>(K, 1)) * 8, st);
  if (K) {
    k_view_fill<<<grid_for(K, 256), 256, 0, st>>>(
        src, nzf.as<uint32_t>(), fsl.as<uint32_t>(), fpos.as<uint32_t>(), spos.as<uint32_t>(), K,
        c->leaf.as<uint32_t>(), c->v32.as<float>(), c->v64 ? c->v64.as<double>() : nullptr,
        c->idx[1].as<uint32_t>(), c->idx[0].as<uint32_t>(), m->leaf.as<uint32_t>(), m->v32.as<float>(),
        c->v64 ? m->v64.as<double>() : nullptr, m->ptr[1].as<uint32_t>(), m->idx[1].as<uint32_t>(),
        m->ptr[0].as<uint32_t>(), m->idx[0].as<uint32_t>());
    check_launch("k_view_fill");
  }
  write_u32(m->ptr[1].as<uint32_t>() + VF, K, st);
  write_u32(m->ptr[0].as<uint32_t>() + VS, VF, st);
  return guard.release();
}
}  // namespace hbk

namespace hbk {
__global__ void k_heavy_sel(const uint32_t* __restrict__ ptr0, const uint32_t* __restrict__ ptr1,
                            int64_t S, uint32_t minnz, uint8_t* __restrict__ sel,
                            unsigned long long* __restrict__ hnnz, uint32_t* __restrict__ hflag) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t m = ptr1[ptr0[s + 1]] - ptr1[ptr0[s]];
    const bool h = m >= minnz;
    sel[s] = h;
    hflag[s] = h;
    if (h) atomicAdd(hnnz, (unsigned long long)m);
  }
}
__global__ void k_heavy_rows(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ sidx,
                             int64_t S, uint32_t* __restrict__ rows) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x)
    if (pos[s + 1] != pos[s]) rows[pos[s]] = sidx[s];
}

// Leaf rows per block for leaf-blocking the heavy slices, 0 = off.  On when
// the leaf factor's rows (the 32-column slice a pass reads) exceed half the
// L2: the heavy slices' nonzeros are then visited leaf-block by leaf-block so
// the block's leaf rows are reused out of L2 (LRU replay of the real access
// streams, scripts/lru_block_sim.py: 63-MB-LRU factor traffic nell-1 mode 0
// 10.8 -> 8.0 GB, delicious-3d mode 1 24.6 -> 14.2 GB, flickr-3d -26..-38%;
// measured: delicious-3d mode 1 4.65 -> 3.77 ms, but nell-1 / flickr-3d 2-9%
// slower — their Zipf leaf heads are L2-resident already, so build_leaf_blocked
// also requires a flat leaf distribution).  Blocks of 0.18 x L2 (12/16/24/32/48
// MB measured within 1%).  HBK_LEAF_BLOCK_MB=x forces x-MB blocks (0 = off;
// forcing also skips the flatness test); HBK_LEAF_MIN sets the heavy-slice
// threshold (nonzeros), for A/B measurement.
static int64_t leaf_block_rows(const int64_t* dims, const int* mo, int rank, bool eligible) {
  if (!eligible) return 0;
  const int64_t Crows = dims[mo[2]];
  const double row_bytes = 4.0 * std::min(rank, 32);
  double mb = -1.0;
  if (const char* e = getenv("HBK_LEAF_BLOCK_MB")) mb = atof(e);
  if (mb == 0.0) return 0;
  int64_t BB = 0;
  if (mb > 0.0) {
    BB = std::max<int64_t>(1, int64_t(mb * 1e6 / row_bytes));
  } else {
    int dev = 0, l2 = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const double cbytes = double(Crows) * row_bytes;
    if (l2 <= 0 || cbytes <= 0.5 * l2) return 0;
    BB = std::max<int64_t>(1, int64_t(0.18 * l2 / row_bytes));
  }
  return BB < Crows ? BB : 0;
}

static hbk_plan* new_plan(hbk_coo* coo, hbk_csl* csl, hbk_csf* csf, hbk_sched* sched, int mode,
                          int rank, int order, const int64_t* dims, const int* mo) {
  hbk_plan* p = new hbk_plan();
  std::unique_ptr<hbk_plan> guard(p);
  HBK_CUDA(cudaEventCreateWithFlags(&p->ev_last, cudaEventDisableTiming));
  p->order = order;
  p->mode = mode;
  p->rank = rank;
  std::copy(dims, dims + order, p->dims);
  std::copy(mo, mo + order, p->mo);
  p->coo = coo;
  p->csl = csl;
  p->csf = csf;
  p->sched = sched;
  hbk_coo_retain(coo);
  hbk_csl_retain(csl);
  hbk_csf_retain(csf);
  hbk_sched_retain(sched);
  return guard.release();
}

// Split the plan's CSF (+ CSL as singleton-fiber CSF slices) into the heavy
// slices (>= minnz nonzeros, leaf-blocked, sub_blk) and the rest (sub_main);
// false (nothing built) when the heavy slices hold under a quarter of the
// plan's nonzeros.
__global__ void k_leaf_hist(const uint32_t* __restrict__ leaf, int64_t M, uint32_t* __restrict__ h) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(h + leaf[i], 1u);
}

// Share of a tree's leaf accesses that go to its K most used leaf rows.
static double leaf_head_share(const hbk_csf* c, int64_t K, cudaStream_t st) {
  const int64_t R = c->dims[c->mode_order[2]];
  if (c->M == 0 || R == 0) return 1.0;
  K = std::min(K, R);
  Scratch h(size_t(R) * 4, st), hs(size_t(R) * 4, st), sum(8, st);
  HBK_CUDA(cudaMemsetAsync(h.p, 0, size_t(R) * 4, st));
  k_leaf_hist<<<grid_for(c->M, 256), 256, 0, st>>>(c->leaf.as<uint32_t>(), c->M, h.as<uint32_t>());
  check_launch("k_leaf_hist");
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp, h.as<uint32_t>(), hs.as<uint32_t>(),
                                                    int(R), 0, 32, st));
  {
    Scratch t(tmp, st);
    HBK_CUDA(cub::DeviceRadixSort::SortKeysDescending(t.p, tmp, h.as<uint32_t>(), hs.as<uint32_t>(),
                                                      int(R), 0, 32, st));
  }
  tmp = 0;
  HBK_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, hs.as<uint32_t>(), sum.as<unsigned long long>(), int(K), st));
  {
    Scratch t(tmp, st);
    HBK_CUDA(cub::DeviceReduce::Sum(t.p, tmp, hs.as<uint32_t>(), sum.as<unsigned long long>(), int(K), st));
  }
  unsigned long long top = 0;
  HBK_CUDA(cudaMemcpyAsync(&top, sum.p, 8, cudaMemcpyDeviceToHost, st));
  HBK_CUDA(cudaStreamSynchronize(st));
  return double(top) / double(c->M);
}

static bool build_leaf_blocked(hbk_plan* p, int64_t BB, uint32_t minnz, cudaStream_t st) {
  hbk_csf* merged = nullptr;
  if (p->csl && p->csl->M > 0) {
    merged = merge_csl_as_csf(p->csf, p->csl, st);
  } else if (p->csf) {
    merged = p->csf;
    hbk_csf_retain(merged);
  }
  if (!merged || merged->M == 0) {
    hbk_csf_release(merged);
    return false;
  }
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> gm(merged, [](hbk_csf* q) { hbk_csf_release(q); });
  // Zipf-headed leaf factors already keep their hot rows in L2: blocking
  // pays only when the rows a quarter of the L2 could hold serve under half
  // of the leaf accesses (delicious-3d mode 1, alpha = 0.3: -14%; the
  // alpha = 1 leaves of nell-1 / flickr-3d measured 2-9% slower blocked)
  {
    int dev = 0, l2 = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const int64_t K = std::max<int64_t>(1, int64_t(0.25 * l2 / (4.0 * std::min(p->rank, 32))));
    const double share = leaf_head_share(merged, K, st);
    p->info.leaf_head_share_ppm = int64_t(share * 1e6);
    if (share > 0.5 && !getenv("HBK_LEAF_BLOCK_MB")) return false;
  }
  const int64_t S = merged->n[0];
  Scratch sel(size_t(S), st), cnt(8, st), pos((S + 1) * 4, st);
  HBK_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
  k_heavy_sel<<<grid_for(S, 256), 256, 0, st>>>(merged->ptr[0].as<uint32_t>(), merged->ptr[1].as<uint32_t>(),
                                               S, minnz, sel.as<uint8_t>(),
                                               cnt.as<unsigned long long>(), pos.as<uint32_t>());
  check_launch("k_heavy_sel");
  unsigned long long hnnz = 0;
  HBK_CUDA(cudaMemcpyAsync(&hnnz, cnt.p, 8, cudaMemcpyDeviceToHost, st));
  HBK_CUDA(cudaStreamSynchronize(st));
  const int64_t total = merged->M + (p->coo ? p->coo->nnz : 0);
  if (hnnz == 0 || 4 * int64_t(hnnz) < total) return false;
  const uint32_t nh = exclusive_scan_total(pos.as<uint32_t>(), S, st);
  p->heavy_rows = dalloc(size_t(std::max<uint32_t>(nh, 1)) * 4, st);
  p->n_heavy_rows = nh;
  k_heavy_rows<<<grid_for(S, 256), 256, 0, st>>>(pos.as<uint32_t>(), merged->idx[0].as<uint32_t>(), S,
                                                p->heavy_rows.as<uint32_t>());
  check_launch("k_heavy_rows");
  hbk_csf* light = csf_block_view(merged, sel.as<uint8_t>(), false, 0, st);
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> gl(light, [](hbk_csf* q) { hbk_csf_release(q); });
  hbk_csf* blk = csf_block_view(merged, sel.as<uint8_t>(), true, BB, st);
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> gb(blk, [](hbk_csf* q) { hbk_csf_release(q); });
  std::unique_ptr<hbk_plan> sb(new_plan(nullptr, nullptr, blk, nullptr, p->mode, p->rank, p->order,
                                        p->dims, p->mo));
  sb->acc_csf = true;
  build_plan(sb.get(), st);
  std::unique_ptr<hbk_plan> sm(new_plan(p->coo, nullptr, light->M ? light : nullptr, nullptr, p->mode,
                                        p->rank, p->order, p->dims, p->mo));
  if (!sm->coo && !sm->csf) {  // every slice is heavy: an empty main plan still zero-fills
    sm->csf = light;
    hbk_csf_retain(light);
  }
  sm->extra_owned = &p->heavy_rows;
  sm->n_extra_owned = nh;
  build_plan(sm.get(), st);
  p->sub_blk = sb.release();
  p->sub_main = sm.release();
  if (!getenv("HBK_CONCURRENT") || atoi(getenv("HBK_CONCURRENT")) != 0) {
    HBK_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    for (int i = 0; i < 7; ++i) {
      HBK_CUDA(cudaStreamCreateWithFlags(&p->side_all[i], cudaStreamNonBlocking));
      HBK_CUDA(cudaEventCreateWithFlags(&p->ev_join_all[i], cudaEventDisableTiming));
    }
  }
  p->leaf_bb = BB;
  p->leaf_min = minnz;
  p->info.leaf_blocks = (p->dims[p->mo[2]] + BB - 1) / BB;
  p->info.leaf_blocked_nnz = int64_t(hnnz);
  return true;
}

// B rows per block of the blocked CSL layout, 0 = unblocked.  Blocked when the
// CSL bucket holds at least half of the plan's nonzeros and its B factor's
// rows (the 32-column slice a pass reads) exceed half the L2: blocks of about
// 0.18 x L2 (delicious-3d, ms per mode for 8/12/16/20/24/32/40/60/80 MB
// blocks: mode 0 3.31/3.17/3.07/3.03/3.03/3.05/3.11/3.28/3.48 vs 4.05
// unblocked, mode 2 3.39/3.19/3.09/3.05/3.00/3.07/3.05/3.31/3.24 vs 3.22).
// The emulation before it (scripts/remap_block_probe.py) measured the
// configurations this rule leaves unblocked 2-4% slower blocked.
// HBK_CSL_BLOCK_MB=x forces x-MB blocks (0 = off), for A/B measurement.
static int64_t csl_block_rows(const hbk_csl* csl, const hbk_csf* csf, const hbk_coo* coo, int rank,
                              bool eligible) {
  if (!csl || csl->M == 0 || !eligible) return 0;
  const int64_t Brows = csl->dims[csl->mode_order[1]];
  const double row_bytes = 4.0 * std::min(rank, 32);
  double mb = -1.0;
  if (const char* e = getenv("HBK_CSL_BLOCK_MB")) mb = atof(e);
  if (mb == 0.0) return 0;
  int64_t BB = 0;
  if (mb > 0.0) {
    BB = std::max<int64_t>(1, int64_t(mb * 1e6 / row_bytes));
  } else {
    const int64_t total = csl->M + (csf ? csf->M : 0) + (coo ? coo->nnz : 0);
    int dev = 0, l2 = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const double bbytes = double(Brows) * row_bytes;
    if (2 * csl->M < total || l2 <= 0 || bbytes <= 0.5 * l2) return 0;
    const int64_t nb = int64_t(std::ceil(bbytes / (0.18 * l2)));
    BB = (Brows + nb - 1) / nb;
  }
  return BB < Brows ? BB : 0;
}
}  // namespace hbk

int hbk_plan_create(hbk_coo* coo, hbk_csl* csl, hbk_csf* csf, hbk_sched* sched, int mode, int rank,
                    void* stream, hbk_plan** out) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    HBK_REQUIRE(rank >= 1, HBK_EINVAL, "rank must be at least 1");
    HBK_REQUIRE(coo || csl || csf, HBK_EINVAL, "plan needs at least one bucket");
    HBK_REQUIRE(!sched || csf, HBK_EINVAL, "a schedule needs a CSF bucket");
    int order = 0;
    const int64_t* dims = nullptr;
    const int* mo = nullptr;
    if (csf) {
      order = csf->order;
      dims = csf->dims;
      mo = csf->mode_order;
    } else if (csl) {
      order = csl->order;
      dims = csl->dims;
      mo = csl->mode_order;
    } else {
      order = coo->order;
      dims = coo->dims;
      mo = coo->sorted_under;
    }
    HBK_REQUIRE(mode >= 0 && mode < order, HBK_EINVAL, "mode out of range");
    if (csf)
      HBK_REQUIRE(csf->mode_order[0] == mode, HBK_EINVAL,
                  "tree was built for mode " + std::to_string(csf->mode_order[0]) +
                      ", asked for mode " + std::to_string(mode));
    if (csl)
      HBK_REQUIRE(csl->mode_order[0] == mode, HBK_EINVAL,
                  "slices were built for mode " + std::to_string(csl->mode_order[0]) +
                      ", asked for mode " + std::to_string(mode));
    if (coo)
      HBK_REQUIRE(coo->unique_mode == mode && coo->has_sorted, HBK_EINVAL,
                  "a COO bucket must be an HB-CSF coo_part of this mode");
    hbk_plan* p = new hbk_plan();
    std::unique_ptr<hbk_plan> guard(p);
    HBK_CUDA(cudaEventCreateWithFlags(&p->ev_last, cudaEventDisableTiming));
    p->order = order;
    p->mode = mode;
    p->rank = rank;
    std::copy(dims, dims + order, p->dims);
    std::copy(mo, mo + order, p->mo);
    p->coo = coo;
    p->csl = csl;
    p->csf = csf;
    p->sched = sched;
    hbk_coo_retain(coo);
    hbk_csl_retain(csl);
    hbk_csf_retain(csf);
    hbk_sched_retain(sched);
    // CSL slices through the CSF kernels (see merge_csl_as_csf): the fast
    // order-3 path without a schedule; HBK_CSL_AS_CSF=0/1 forces either way
    int64_t csl_slices_merged = 0;
    {
      const char* e = getenv("HBK_CSL_AS_CSF");
      const bool fast_shape = order == 3 && rank >= 4 && rank % 4 == 0 &&
                              dims[mo[1]] < (int64_t(1) << 29) && dims[mo[2]] < (int64_t(1) << 29);
      // worth it when the CSL slices are heavy on average (> 128 nonzeros:
      // delicious-3d mode 0, 5.6% faster); lighter CSL slices stay on the CSL
      // kernel, measured 2% faster for them (delicious mode 2, 56 per slice)
      const bool heavy_csl = csl && csl->M > 128 * csl->S;
      p->csl_bb = csl_block_rows(csl, csf, coo, rank, fast_shape && !sched);
      // leaf-blocked heavy slices (build_leaf_blocked): the plan keeps the
      // reference buckets (generic / fp64 kernel), the sub-plans run the fast path
      const int64_t lbb = leaf_block_rows(dims, mo, rank,
                                          fast_shape && !sched && order == 3 && p->csl_bb == 0 &&
                                              (!csf || csf->order == 3));
      if (lbb > 0) {
        // heavy-slice threshold: delicious-3d mode 1 at 16/32/64/128/512/2048
        // nonzeros: 3.84/3.77/3.77/3.81/4.00/4.05 ms (unblocked 4.65)
        uint32_t minnz = 64;
        if (const char* e2 = getenv("HBK_LEAF_MIN")) minnz = uint32_t(std::max(1, atoi(e2)));
        if (build_leaf_blocked(p, lbb, minnz, st)) p->force_generic = true;
      }
      if (!p->sub_blk && csl && csl->M > 0 && !sched && fast_shape && (!csf || csf->order == 3) &&
          (e ? atoi(e) != 0 : heavy_csl && p->csl_bb == 0)) {
        hbk_csf* merged = merge_csl_as_csf(csf, csl, st);
        hbk_csf_release(p->csf);
        hbk_csl_release(p->csl);
        p->csf = merged;
        p->csl = nullptr;
        csl_slices_merged = csl->S;
      }
    }
    const hbk_plan_info keep_leaf = p->info;
    build_plan(p, st);
    // OpCount is the reference's (kernels.py:210-214 for the CSL bucket):
    // the CSF count of a singleton-fiber slice adds one per slice
    p->info.op_adds -= csl_slices_merged * rank;
    if (p->sub_blk) {  // what the fast path launches and gathers
      const hbk_plan_info& a = p->sub_blk->info;
      const hbk_plan_info& b = p->sub_main->info;
      p->info.fast_path = 1;
      p->info.launches = a.launches + b.launches + 1;  // + the heavy-row zeroing
      p->info.tasks_csf = a.tasks_csf + b.tasks_csf;
      p->info.tasks_heavy = a.tasks_heavy + b.tasks_heavy;
      p->info.tasks_csl = b.tasks_csl;
      p->info.tasks_coo = b.tasks_coo;
      p->info.tasks_zero = b.tasks_zero;
      p->info.split_rows = a.split_rows + b.split_rows;
      p->info.stream_bytes = a.stream_bytes + b.stream_bytes;
      p->info.gather_rows = a.gather_rows + b.gather_rows;
      p->info.leaf_blocks = keep_leaf.leaf_blocks;
      p->info.leaf_blocked_nnz = keep_leaf.leaf_blocked_nnz;
    }
    p->info.leaf_head_share_ppm = keep_leaf.leaf_head_share_ppm;
    *out = guard.release();
  });
}

int hbk_plan_info_get(const hbk_plan* p, hbk_plan_info* info) {
  return guarded([&] { *info = p->info; });
}

int hbk_plan_execute(const hbk_plan* p, const float* const* factors, float* out, void* stream) {
  return hbk_plan_execute_ex(p, factors, out, 0, stream);
}

int hbk_plan_execute_ex(const hbk_plan* p, const float* const* factors, float* out, int flags,
                        void* stream) {
  return guarded([&] {
    const bool skip_zero = (flags & HBK_EXEC_SKIP_UNOWNED) != 0;
    cudaStream_t st = to_stream(stream);
    const int N = p->order;
    for (int d = 0; d < N; ++d)
      HBK_REQUIRE(d == p->mode || factors[d] != nullptr, HBK_EINVAL, "null factor pointer");
    HBK_REQUIRE(out != nullptr || p->dims[p->mode] == 0, HBK_EINVAL, "null output pointer");
    ExecOrder order(p, st);
    if (p->sub_blk) {
      // leaf-blocked heavy slices: zero their rows, accumulate them block by
      // block (sub_blk), then every other slice (sub_main)
      Factors3 fx;
      fx.B = reinterpret_cast<const float4*>(factors[p->mo[1]]);
      fx.C = reinterpret_cast<const float4*>(factors[p->mo[2]]);
      fx.out = reinterpret_cast<float4*>(out);
      HBK_REQUIRE((reinterpret_cast<uintptr_t>(fx.B) | reinterpret_cast<uintptr_t>(fx.C) |
                   reinterpret_cast<uintptr_t>(out)) % 16 == 0,
                  HBK_EINVAL, "factor and output buffers must be 16-byte aligned");
      const int R = p->rank;
      if (p->n_heavy_rows) {
        const int64_t n4 = p->n_heavy_rows * (R / 4);
        k_zero_rows<<<grid_for(n4, 256), 256, 0, st>>>(p->heavy_rows.as<uint32_t>(), p->n_heavy_rows,
                                                       uint32_t(R / 4), fx.out);
        check_launch("k_zero_rows");
      }
      if (p->sub_blk->r32) {
        launch_blocked(p, Factors3R32(fx), st, skip_zero);
      } else {
        fx.rs = uint32_t(R / 4);
        for (int c0 = 0; c0 < R; c0 += 32) {
          fx.col4 = uint32_t(c0 / 4);
          fx.lanes = uint32_t(std::min(8, (R - c0) / 4));
          launch_blocked(p, fx, st, skip_zero);
        }
      }
    } else if (p->fast) {
      Factors3 fx;
      fx.B = reinterpret_cast<const float4*>(factors[p->mo[1]]);
      fx.C = reinterpret_cast<const float4*>(factors[p->mo[2]]);
      fx.out = reinterpret_cast<float4*>(out);
      HBK_REQUIRE((reinterpret_cast<uintptr_t>(fx.B) | reinterpret_cast<uintptr_t>(fx.C) |
                   reinterpret_cast<uintptr_t>(out)) %
                          16 ==
                      0,
                  HBK_EINVAL, "factor and output buffers must be 16-byte aligned");
      const int R = p->rank;
      // the blocked CSL layout adds its rows into the output
      if (p->csl_acc)
        HBK_CUDA(cudaMemsetAsync(out, 0, size_t(p->dims[p->mode]) * R * sizeof(float), st));
      if (p->r32) {
        launch_fast(p, Factors3R32(fx), st, skip_zero);
      } else {
        fx.rs = uint32_t(R / 4);
        for (int c0 = 0; c0 < R; c0 += 32) {  // passes of 32 columns
          fx.col4 = uint32_t(c0 / 4);
          fx.lanes = uint32_t(std::min(8, (R - c0) / 4));
          launch_fast(p, fx, st, skip_zero);
        }
      }
    } else {
      launch_generic<float>(p, factors, out, st);
    }
    order.done();
  });
}

namespace hbk {
// Finiteness scan of up to 8 fp32 buffers in one launch (the host calling
// convention's kernels.py:82-86 check, run on the uploaded copies).  float4
// loads over the 16-byte-aligned body, scalar head/tail.
struct FiniteArgs {
  const float* p[8];
  int64_t n[8];
  int count;
};
__global__ void __launch_bounds__(256) k_nonfinite(const __grid_constant__ FiniteArgs a,
                                                   int32_t* __restrict__ flags) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int i = 0; i < a.count; ++i) {
    const float* p = a.p[i];
    const int64_t n = a.n[i];
    const int64_t head = std::min<int64_t>(n, ((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4);
    const int64_t n4 = (n - head) / 4;
    const float4* q = reinterpret_cast<const float4*>(p + head);
    bool bad = false;
    for (int64_t k = tid; k < n4; k += nth) {
      const float4 v = __ldcs(q + k);
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    for (int64_t k = tid; k < head; k += nth) bad |= !isfinite(p[k]);
    for (int64_t k = head + n4 * 4 + tid; k < n; k += nth) bad |= !isfinite(p[k]);
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) flags[i] = 1;
  }
}
}  // namespace hbk

int hbk_stream_synchronize(void* stream) {
  return guarded([&] { HBK_CUDA(cudaStreamSynchronize(to_stream(stream))); });
}

int hbk_plan_rows(const hbk_plan* p, uint32_t* rows_out, int64_t* count, void* stream) {
  return guarded([&] {
    HBK_REQUIRE(p && count, HBK_EINVAL, "null pointer");
    cudaStream_t st = to_stream(stream);
    const int64_t rows = p->dims[p->mode];
    if (rows == 0) {
      *count = 0;
      return;
    }
    Scratch mark(rows, st);
    HBK_CUDA(cudaMemsetAsync(mark.p, 0, rows, st));
    if (p->csf && p->csf->n[0])
      k_mark_rows<<<grid_for(p->csf->n[0], 256), 256, 0, st>>>(p->csf->idx[0].as<uint32_t>(),
                                                               p->csf->n[0], mark.as<uint8_t>());
    if (p->csl && p->csl->S)
      k_mark_rows<<<grid_for(p->csl->S, 256), 256, 0, st>>>(p->csl->slice_idx.as<uint32_t>(),
                                                            p->csl->S, mark.as<uint8_t>());
    if (p->coo && p->coo->nnz)
      k_mark_rows<<<grid_for(p->coo->nnz, 256), 256, 0, st>>>(
          p->coo->cols[p->mode].as<uint32_t>(), p->coo->nnz, mark.as<uint8_t>());
    check_launch("k_mark_rows");
    Scratch pos((rows + 1) * sizeof(uint32_t), st);
    k_marked_flags<<<grid_for(rows, 256), 256, 0, st>>>(mark.as<uint8_t>(), rows,
                                                        pos.as<uint32_t>());
    check_launch("k_marked_flags");
    const uint32_t n = exclusive_scan_total(pos.as<uint32_t>(), rows, st);
    *count = n;
    if (rows_out && n) {
      k_unmarked_emit<<<grid_for(rows, 256), 256, 0, st>>>(pos.as<uint32_t>(), rows, rows_out);
      check_launch("k_unmarked_emit");
    }
  });
}

int hbk_nonfinite_f32(const float* const* bufs, const int64_t* counts, int n, int32_t* flags,
                      void* stream) {
  return guarded([&] {
    HBK_REQUIRE(n >= 0 && n <= 8, HBK_EINVAL, "at most 8 buffers per finiteness scan");
    HBK_REQUIRE(n == 0 || (bufs && counts && flags), HBK_EINVAL, "null pointer");
    cudaStream_t st = to_stream(stream);
    if (n == 0) return;
    FiniteArgs a{};
    a.count = n;
    int64_t total = 0;
    for (int i = 0; i < n; ++i) {
      HBK_REQUIRE(counts[i] >= 0 && (counts[i] == 0 || bufs[i]), HBK_EINVAL, "bad buffer");
      a.p[i] = bufs[i];
      a.n[i] = counts[i];
      total += counts[i];
    }
    HBK_CUDA(cudaMemsetAsync(flags, 0, size_t(n) * 4, st));
    int dev = 0, sms = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * 8, (total / 4 + 255) / 256)));
    k_nonfinite<<<grid, 256, 0, st>>>(a, flags);
    check_launch("k_nonfinite");
  });
}

namespace hbk {
static void probe_plan(const hbk_plan* p, const Factors3R32& f32, cudaStream_t st) {
  float4* sink = p->probe_sink.as<float4>();
  int dev = 0, sms = 0;
  HBK_CUDA(cudaGetDevice(&dev));
  HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = sms * 4;
  if (p->work.n0) k_gather_probe<KIND_CSF><<<grid, FAST_BLOCK, 0, st>>>(p->work, f32, sink);
  if (p->grid_heavy) k_gather_probe<KIND_CSF><<<grid, FAST_BLOCK, 0, st>>>(p->work_heavy, f32, sink);
  if (p->work.n1 > p->work.n0) k_gather_probe<KIND_CSL><<<grid, FAST_BLOCK, 0, st>>>(p->work, f32, sink);
  if (p->work.n2 > p->work.n1) k_gather_probe<KIND_COO><<<grid, FAST_BLOCK, 0, st>>>(p->work, f32, sink);
  check_launch("k_gather_probe");
}
}  // namespace hbk

namespace hbk {
// Hardware row-gather ceiling (roofline anchor for the row-gather-bound
// configurations): 8-lane groups gather whole 128-B rows at
// pseudo-random indices (an LCG, two integer instructions per row) of a
// scratch matrix of `rows` rows (a power of two), 8 rows in flight per
// group, loads L1-allocating as the kernels' factor-row loads are — the
// MTTKRP's access shape with no index streams, shuffles or arithmetic.
// Matrices within the L2 give the L2 -> SM random-row rate, larger ones the
// HBM random-row rate (scripts/l2_bw_probe.cu sweeps sizes and occupancies).
__global__ void k_row_ceiling(const float4* __restrict__ a, uint32_t mask, uint32_t per_group,
                              float* __restrict__ sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  uint32_t x = grp * 0x9E3779B9u + 0x7F4A7C15u;
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  float acc = 0.f;
  for (uint32_t it = 0; it < per_group; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      v[u] = __ldg(a + size_t((x >> 8) & mask) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) *sink = acc;  // keeps the loads; never true for the zeroed matrix
}
static std::mutex g_ceiling_mu;
static void* g_ceiling_buf = nullptr;
static size_t g_ceiling_bytes = 0;
static int g_ceiling_dev = -1;  // the device the scratch lives on
}  // namespace hbk

namespace hbk {
// The same gather driven by an index STREAM read the way the MTTKRP kernels
// read theirs: each 8-lane group walks its own contiguous span of idx (HBM,
// L1 no-allocate), one coalesced load per lane per batch of 8 positions
// (the next batch's loaded one batch ahead), 8 SHFL broadcasts, 8
// L1-allocating row loads — the kernels' access structure without their
// arithmetic, for a caller-chosen row distribution (e.g. the tensor's skew).
__global__ void k_row_ceiling_stream(const float4* __restrict__ a, const uint32_t* __restrict__ idx,
                                     uint32_t mask, uint32_t per_group, float* __restrict__ sink) {
  const uint32_t lig = threadIdx.x & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const uint32_t* my = idx + size_t(grp) * per_group;
  const uint64_t pol = policy_evict_first();
  float acc = 0.f;
  uint32_t cur = ld_stream_u32(my + lig, pol);
  for (uint32_t it = 0; it < per_group; it += 8) {
    const uint32_t nxt = it + 8 < per_group ? ld_stream_u32(my + it + 8 + lig, pol) : 0u;
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = __shfl_sync(FULL, cur, u, 8) & mask;
      v[u] = __ldg(a + size_t(r) * 8 + lig);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    cur = nxt;
  }
  if (acc == 1234.5f) *sink = acc;
}
}  // namespace hbk

int hbk_row_ceiling(int64_t rows, int ctas_per_sm, int64_t gathers, void* stream) {
  return guarded([&] {
    if (rows == 0) {  // release the scratch matrix (on its device)
      std::lock_guard<std::mutex> lk(g_ceiling_mu);
      if (g_ceiling_buf) {
        int prev = 0;
        HBK_CUDA(cudaGetDevice(&prev));
        HBK_CUDA(cudaSetDevice(g_ceiling_dev));
        HBK_CUDA(cudaFree(g_ceiling_buf));
        HBK_CUDA(cudaSetDevice(prev));
      }
      g_ceiling_buf = nullptr;
      g_ceiling_bytes = 0;
      return;
    }
    HBK_REQUIRE(rows > 0 && (rows & (rows - 1)) == 0 && rows <= (int64_t(1) << 32), HBK_EINVAL,
                "rows must be a power of two <= 2^32");
    HBK_REQUIRE(ctas_per_sm >= 1 && ctas_per_sm <= 8 && gathers > 0, HBK_EINVAL,
                "ctas_per_sm in 1..8 and gathers > 0");
    cudaStream_t st = to_stream(stream);
    std::lock_guard<std::mutex> lk(g_ceiling_mu);
    const size_t bytes = size_t(rows) * 128 + 16;
    int cur = 0;
    HBK_CUDA(cudaGetDevice(&cur));
    if (g_ceiling_buf && g_ceiling_dev != cur) {  // scratch of another device: free it there
      int prev = cur;
      HBK_CUDA(cudaSetDevice(g_ceiling_dev));
      HBK_CUDA(cudaFree(g_ceiling_buf));
      HBK_CUDA(cudaSetDevice(prev));
      g_ceiling_buf = nullptr;
      g_ceiling_bytes = 0;
    }
    if (g_ceiling_bytes < bytes) {
      if (g_ceiling_buf) HBK_CUDA(cudaFree(g_ceiling_buf));
      g_ceiling_buf = nullptr;
      g_ceiling_bytes = 0;
      HBK_CUDA(cudaMalloc(&g_ceiling_buf, bytes));
      HBK_CUDA(cudaMemsetAsync(g_ceiling_buf, 0, bytes, st));
      g_ceiling_bytes = bytes;
      g_ceiling_dev = cur;
    }
    int dev = 0, sms = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = sms * ctas_per_sm;
    const int64_t groups = int64_t(grid) * (FAST_BLOCK / 8);
    const uint32_t per_group = uint32_t(std::max<int64_t>(8, (gathers / groups + 7) / 8 * 8));
    // rows 128-byte aligned (as the factor rows are); the sink after them
    float4* a = static_cast<float4*>(g_ceiling_buf);
    k_row_ceiling<<<grid, FAST_BLOCK, 0, st>>>(a, uint32_t(rows - 1), per_group,
                                               reinterpret_cast<float*>(a + size_t(rows) * 8));
    check_launch("k_row_ceiling");
  });
}

int hbk_row_ceiling_stream(const uint32_t* idx, int64_t n, int64_t rows, int ctas_per_sm, void* stream) {
  return guarded([&] {
    HBK_REQUIRE(rows > 0 && (rows & (rows - 1)) == 0 && rows <= (int64_t(1) << 32), HBK_EINVAL,
                "rows must be a power of two <= 2^32");
    HBK_REQUIRE(ctas_per_sm >= 1 && ctas_per_sm <= 8 && idx != nullptr && n > 0, HBK_EINVAL,
                "ctas_per_sm in 1..8 and a non-empty index stream");
    int dev = 0, sms = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = sms * ctas_per_sm;
    const int64_t groups = int64_t(grid) * (FAST_BLOCK / 8);
    const int64_t per_group = n / groups / 8 * 8;
    HBK_REQUIRE(per_group >= 8, HBK_EINVAL, "index stream too short for this grid (need 8 per group)");
    cudaStream_t st = to_stream(stream);
    std::lock_guard<std::mutex> lk(g_ceiling_mu);
    HBK_REQUIRE(g_ceiling_buf && g_ceiling_dev == dev && g_ceiling_bytes >= size_t(rows) * 128 + 16,
                HBK_EINVAL, "call hbk_row_ceiling with the same rows first (it owns the matrix)");
    float4* a = static_cast<float4*>(g_ceiling_buf);
    k_row_ceiling_stream<<<grid, FAST_BLOCK, 0, st>>>(a, idx, uint32_t(rows - 1), uint32_t(per_group),
                                                      reinterpret_cast<float*>(a + size_t(rows) * 8));
    check_launch("k_row_ceiling_stream");
  });
}

int hbk_plan_probe(const hbk_plan* p, const float* const* factors, void* stream) {
  return guarded([&] {
    const hbk_plan* a = p->sub_blk ? p->sub_blk : p;
    HBK_REQUIRE(a->bpos && a->r32 && (!p->sub_main || p->sub_main->r32), HBK_EINVAL,
                "the gather probe needs a B-position (fast order-3, R=32, extents < 2^27) plan");
    cudaStream_t st = to_stream(stream);
    ExecOrder order(p, st);
    Factors3 fx;
    fx.B = reinterpret_cast<const float4*>(factors[p->mo[1]]);
    fx.C = reinterpret_cast<const float4*>(factors[p->mo[2]]);
    fx.out = nullptr;
    const Factors3R32 f32(fx);
    probe_plan(a, f32, st);
    if (p->sub_main) probe_plan(p->sub_main, f32, st);
    order.done();
  });
}

int hbk_plan_execute_f64(const hbk_plan* p, const double* const* factors, double* out,
                         void* stream) {
  return guarded([&] {
    for (int d = 0; d < p->order; ++d)
      HBK_REQUIRE(d == p->mode || factors[d] != nullptr, HBK_EINVAL, "null factor pointer");
    HBK_REQUIRE(out != nullptr, HBK_EINVAL, "null output pointer");
    HBK_REQUIRE(p->gen_grid > 0, HBK_EINVAL, "plan has no fp64 launch configuration");
    cudaStream_t st = to_stream(stream);
    ExecOrder order(p, st);
    if (ensure_f64(p, st)) {
      const int R = p->rank;
      const double2* B = reinterpret_cast<const double2*>(factors[p->mo[1]]);
      const double2* Cf = reinterpret_cast<const double2*>(factors[p->mo[2]]);
      double2* o = reinterpret_cast<double2*>(out);
      HBK_REQUIRE((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(Cf) |
                   reinterpret_cast<uintptr_t>(out)) % 16 == 0,
                  HBK_EINVAL, "factor and output buffers must be 16-byte aligned");
      const hbk_plan* q = p->sub_blk ? p->sub_blk : p;  // the kernels' shape (r32)
      if (p->csl_acc)  // the blocked CSL layout adds its rows
        HBK_CUDA(cudaMemsetAsync(out, 0, size_t(p->dims[p->mode]) * R * sizeof(double), st));
      if (p->sub_blk && p->n_heavy_rows) {  // zero the leaf-blocked rows (R doubles = R/2 x 16 B)
        const int64_t n4 = p->n_heavy_rows * (R / 2);
        k_zero_rows<<<grid_for(n4, 256), 256, 0, st>>>(p->heavy_rows.as<uint32_t>(), p->n_heavy_rows,
                                                       uint32_t(R / 2), reinterpret_cast<float4*>(out));
        check_launch("k_zero_rows");
      }
      auto run = [&](const auto& fx) {
        if (p->sub_blk) launch_blocked64(p, fx, st); else launch_fast64(p, fx, st);
      };
      if (q->r32) {
        for (uint32_t c4 = 0; c4 < 16; c4 += 8) run(Factors3DR32{B, Cf, o, c4});
      } else {
        for (int c0 = 0; c0 < R; c0 += 16)
          run(Factors3D{B, Cf, o, uint32_t(R / 2), uint32_t(c0 / 2), uint32_t(std::min(8, (R - c0) / 2))});
      }
    } else {
      launch_generic<double>(p, factors, out, st);
    }
    order.done();
  });
}

void hbk_plan_release(hbk_plan* p) { delete p; }

}  // extern "C"
