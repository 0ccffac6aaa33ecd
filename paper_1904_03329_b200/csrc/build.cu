// On-GPU HB-CSF builder: key sort, canonicalize, CSF
// level compaction, slice classification + 3-way partition, fiber split and
// the greedy slice-to-block schedule.  Every array this file produces is
// bit-identical to the reference's (tenkit formats.py / balance.py); the
// reference line each step restates is cited at the step.
#include <atomic>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace hbk {

// ------------------------------------------------------------- plumbing --
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

Buf dalloc(size_t bytes, cudaStream_t st) {
  (void)st;
  Buf b;
  b.bytes = bytes;
  void* p = nullptr;
  HBK_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
  b.p = p;
  b.owner = std::shared_ptr<void>(p, [](void* q) { cudaFree(q); });
  return b;
}

// Scratch comes from the device's default stream-ordered pool.  Its default
// release threshold (0) hands freed memory back to the driver at every
// synchronisation, so the next build re-maps it: measured 7.4 ms per
// cudaMallocAsync on average over a nell-2 CP-ALS build.  Keep up to 8 GB
// cached (set once per device; torch's allocator does not use this pool).
static void retain_scratch_pool() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  if ((done.load(std::memory_order_relaxed) >> dev) & 1u) return;
  cudaMemPool_t pool;
  uint64_t thr = uint64_t(8) << 30;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess ||
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) != cudaSuccess)
    (void)cudaGetLastError();  // best effort: leave no error pending
  done.fetch_or(uint64_t(1) << dev, std::memory_order_relaxed);
}

Scratch::Scratch(size_t bytes, cudaStream_t s) : st(s) {
  retain_scratch_pool();
  HBK_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, s));
}
Scratch::~Scratch() {
  if (p) cudaFreeAsync(p, st);
}

uint32_t read_u32(const uint32_t* dev, cudaStream_t st) {
  uint32_t v = 0;
  HBK_CUDA(cudaMemcpyAsync(&v, dev, sizeof(v), cudaMemcpyDeviceToHost, st));
  HBK_CUDA(cudaStreamSynchronize(st));
  return v;
}

void write_u32(uint32_t* dev, uint32_t v, cudaStream_t st) {
  HBK_CUDA(cudaMemcpyAsync(dev, &v, sizeof(v), cudaMemcpyHostToDevice, st));
  HBK_CUDA(cudaStreamSynchronize(st));
}

uint32_t exclusive_scan_u32(uint32_t* data, int64_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  HBK_REQUIRE(n < (int64_t(1) << 31), HBK_EINVAL, "scan length exceeds 2^31");
  uint32_t last = read_u32(data + n - 1, st);
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, data, int(n), st));
  Scratch t(tmp, st);
  HBK_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, data, data, int(n), st));
  return read_u32(data + n - 1, st) + last;
}

uint32_t exclusive_scan_total(uint32_t* data, int64_t n, cudaStream_t st) {
  HBK_REQUIRE(n + 1 < (int64_t(1) << 31), HBK_EINVAL, "scan length exceeds 2^31");
  HBK_CUDA(cudaMemsetAsync(data + n, 0, sizeof(uint32_t), st));
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, data, int(n + 1), st));
  Scratch t(tmp, st);
  HBK_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, data, data, int(n + 1), st));
  return read_u32(data + n, st);
}

static int nbits(int64_t dim) {
  if (dim <= 1) return 0;
  uint64_t v = uint64_t(dim - 1);
  return 64 - __builtin_clzll(v);
}

static void check_mode_order(const int* mo, int order) {
  HBK_REQUIRE(mo != nullptr, HBK_EINVAL, "mode_order is required");
  bool seen[HBK_MAX_ORDER] = {false};
  for (int d = 0; d < order; ++d) {
    HBK_REQUIRE(mo[d] >= 0 && mo[d] < order && !seen[mo[d]], HBK_EINVAL,
                "mode_order is not a permutation of 0..order-1");
    seen[mo[d]] = true;
  }
}

struct Cols {
  const uint32_t* c[HBK_MAX_ORDER];
};
struct MCols {
  uint32_t* c[HBK_MAX_ORDER];
};

// ------------------------------------------------------------ K1: sort --
// np.lexsort over the permuted columns (coo.py:208-211) restated as a stable
// LSD radix sort: columns are packed, minor first, into <=64-bit keys; each
// key group is one stable CUB onesweep pass carrying the permutation.

struct KeyGroup {
  int ncol;
  const uint32_t* col[HBK_MAX_ORDER];
  int shift[HBK_MAX_ORDER];
  int bits;
};

template <class K>
__global__ void k_pack_keys(KeyGroup g, const uint32_t* __restrict__ perm, int64_t M,
                            K* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t src = perm ? perm[i] : uint32_t(i);
    K k = 0;
    for (int c = 0; c < g.ncol; ++c) k |= K(g.col[c][src]) << g.shift[c];
    keys[i] = k;
    if (!perm) vals[i] = uint32_t(i);
  }
}

template <class K>
static void radix_pass(const KeyGroup& g, Scratch& perm, bool first, int64_t M, cudaStream_t st) {
  Scratch keys_a(M * sizeof(K), st), keys_b(M * sizeof(K), st);
  Scratch vals_b(M * sizeof(uint32_t), st);
  k_pack_keys<K><<<grid_for(M, 256), 256, 0, st>>>(g, first ? nullptr : perm.as<uint32_t>(), M,
                                                   keys_a.as<K>(), perm.as<uint32_t>());
  check_launch("k_pack_keys");
  cub::DoubleBuffer<K> kb(keys_a.as<K>(), keys_b.as<K>());
  cub::DoubleBuffer<uint32_t> vb(perm.as<uint32_t>(), vals_b.as<uint32_t>());
  size_t tmp = 0;
  HBK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, int(M), 0, g.bits, st));
  Scratch t(tmp, st);
  HBK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, int(M), 0, g.bits, st));
  if (vb.Current() != perm.as<uint32_t>()) {
    HBK_CUDA(cudaMemcpyAsync(perm.p, vb.Current(), M * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                             st));
  }
}

__global__ void k_iota(uint32_t* p, int64_t M) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i);
}

// Permutation that orders the entries lexicographically by
// (col[mo[0]], col[mo[1]], ...), ties kept in input order (stable).
static Scratch sort_permutation(const hbk_coo* t, const int* mo, cudaStream_t st) {
  const int64_t M = t->nnz;
  Scratch perm(M * sizeof(uint32_t), st);
  // Key groups from the least significant level upward.
  std::vector<KeyGroup> groups;
  KeyGroup cur{};
  for (int lev = t->order - 1; lev >= 0; --lev) {
    int b = nbits(t->dims[mo[lev]]);
    if (b == 0) continue;
    if (cur.bits + b > 64) {
      groups.push_back(cur);
      cur = KeyGroup{};
    }
    cur.col[cur.ncol] = t->cols[mo[lev]].as<uint32_t>();
    cur.shift[cur.ncol] = cur.bits;
    cur.ncol++;
    cur.bits += b;
  }
  if (cur.ncol) groups.push_back(cur);
  if (groups.empty() || M <= 1) {
    k_iota<<<grid_for(M, 256), 256, 0, st>>>(perm.as<uint32_t>(), M);
    check_launch("k_iota");
    return perm;
  }
  for (size_t g = 0; g < groups.size(); ++g) {
    if (groups[g].bits <= 32)
      radix_pass<uint32_t>(groups[g], perm, g == 0, M, st);
    else
      radix_pass<uint64_t>(groups[g], perm, g == 0, M, st);
  }
  return perm;
}

__global__ void k_gather_coo(Cols in, MCols out, int order, const float* __restrict__ v32,
                             const double* __restrict__ v64, const uint32_t* __restrict__ perm,
                             int64_t M, float* __restrict__ o32, double* __restrict__ o64) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t s = perm[i];
    for (int d = 0; d < order; ++d) out.c[d][i] = in.c[d][s];
    o32[i] = v32[s];
    if (o64) o64[i] = v64[s];
  }
}

static hbk_coo* new_coo_like(const hbk_coo* t, int64_t M, bool with64, cudaStream_t st) {
  hbk_coo* o = new hbk_coo();
  o->order = t->order;
  std::memcpy(o->dims, t->dims, sizeof(o->dims));
  o->nnz = M;
  for (int d = 0; d < t->order; ++d) o->cols[d] = dalloc(M * sizeof(uint32_t), st);
  o->v32 = dalloc(M * sizeof(float), st);
  if (with64) o->v64 = dalloc(M * sizeof(double), st);
  return o;
}

static Cols cols_of(const hbk_coo* t) {
  Cols c{};
  for (int d = 0; d < t->order; ++d) c.c[d] = t->cols[d].as<uint32_t>();
  return c;
}
static MCols mcols_of(hbk_coo* t) {
  MCols c{};
  for (int d = 0; d < t->order; ++d) c.c[d] = t->cols[d].as<uint32_t>();
  return c;
}

// sort_by_mode_order, coo.py:214-224.
static hbk_coo* coo_sorted(hbk_coo* t, const int* mo, cudaStream_t st, bool force = false) {
  check_mode_order(mo, t->order);
  if (!force && t->has_sorted && std::equal(mo, mo + t->order, t->sorted_under)) {
    t->ref++;
    return t;
  }
  const int64_t M = t->nnz;
  Scratch perm = sort_permutation(t, mo, st);
  hbk_coo* o = new_coo_like(t, M, bool(t->v64), st);
  k_gather_coo<<<grid_for(M, 256), 256, 0, st>>>(cols_of(t), mcols_of(o), t->order,
                                                 t->v32.as<float>(), t->v64.as<double>(),
                                                 perm.as<uint32_t>(), M, o->v32.as<float>(),
                                                 o->v64.as<double>());
  check_launch("k_gather_coo");
  o->has_sorted = true;
  std::copy(mo, mo + t->order, o->sorted_under);
  HBK_CUDA(cudaStreamSynchronize(st));
  return o;
}

// ------------------------------------------------------- canonicalize --
// coo.py:227-247.  Duplicate runs are merged with np.add.reduceat's exact
// association: first element + pairwise_sum(rest), where pairwise_sum is
// NumPy's blocked pairwise summation (8 accumulators up to 128 elements,
// recursive halving above).  Verified bitwise against NumPy in tests.

__device__ double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

__global__ void k_dup_flags(Cols c, int order, int64_t M, uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t f = 1;
    if (i > 0) {
      f = 0;
      for (int d = 0; d < order; ++d) f |= (c.c[d][i] != c.c[d][i - 1]);
    }
    flag[i] = f;
  }
}

// starts[g] = first entry of group g (flags scanned in pos).
__global__ void k_group_starts(const uint32_t* __restrict__ pos, int64_t M, uint32_t G,
                               uint32_t* __restrict__ starts) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (pos[i + 1] != pos[i]) starts[pos[i]] = uint32_t(i);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) starts[G] = uint32_t(M);
}

__global__ void k_group_reduce(const uint32_t* __restrict__ starts, uint32_t G,
                               const double* __restrict__ v64, const float* __restrict__ v32,
                               int merge, double* __restrict__ gsum,
                               uint32_t* __restrict__ keep) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < G;
       g += int64_t(gridDim.x) * blockDim.x) {
    uint32_t a = starts[g], b = starts[g + 1];
    double s;
    if (v64) {
      s = v64[a];
      if (merge == 0 && b - a > 1) s = s + np_pairwise_sum(v64 + a + 1, int64_t(b - a - 1));
    } else {
      s = double(v32[a]);
      if (merge == 0)
        for (uint32_t i = a + 1; i < b; ++i) s = double(float(s) + v32[i]);
    }
    gsum[g] = s;
    keep[g] = (merge == 1) ? 1u : uint32_t(s != 0.0);
  }
}

__global__ void k_group_emit(const uint32_t* __restrict__ starts, uint32_t G,
                             const uint32_t* __restrict__ kpos, const double* __restrict__ gsum,
                             Cols in, MCols out, int order, float* __restrict__ o32,
                             double* __restrict__ o64) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < G;
       g += int64_t(gridDim.x) * blockDim.x) {
    if (kpos[g + 1] == kpos[g]) continue;
    uint32_t dst = kpos[g], src = starts[g];
    for (int d = 0; d < order; ++d) out.c[d][dst] = in.c[d][src];
    o32[dst] = float(gsum[g]);
    if (o64) o64[dst] = gsum[g];
  }
}

static hbk_coo* coo_canonical(hbk_coo* t, int merge, cudaStream_t st) {
  int identity[HBK_MAX_ORDER];
  for (int d = 0; d < t->order; ++d) identity[d] = d;
  const int64_t M = t->nnz;
  if (M == 0) {
    hbk_coo* o = new_coo_like(t, 0, bool(t->v64), st);
    o->has_sorted = true;
    std::copy(identity, identity + t->order, o->sorted_under);
    return o;
  }
  // The reference always re-sorts (coo.py:237); so do we, even if the input
  // claims to be sorted.
  hbk_coo* s = coo_sorted(t, identity, st, /*force=*/true);
  std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> sorted(s, [](hbk_coo* p) { hbk_coo_release(p); });

  Scratch pos((M + 1) * sizeof(uint32_t), st);
  k_dup_flags<<<grid_for(M, 256), 256, 0, st>>>(cols_of(s), s->order, M, pos.as<uint32_t>());
  check_launch("k_dup_flags");
  uint32_t G = exclusive_scan_total(pos.as<uint32_t>(), M, st);
  Scratch starts((G + 1) * sizeof(uint32_t), st);
  k_group_starts<<<grid_for(M, 256), 256, 0, st>>>(pos.as<uint32_t>(), M, G,
                                                   starts.as<uint32_t>());
  check_launch("k_group_starts");
  Scratch gsum(G * sizeof(double), st);
  Scratch kpos((G + 1) * sizeof(uint32_t), st);
  k_group_reduce<<<grid_for(G, 128), 128, 0, st>>>(starts.as<uint32_t>(), G, s->v64.as<double>(),
                                                   s->v32.as<float>(), merge, gsum.as<double>(),
                                                   kpos.as<uint32_t>());
  check_launch("k_group_reduce");
  uint32_t K = exclusive_scan_total(kpos.as<uint32_t>(), G, st);
  hbk_coo* o = new_coo_like(t, K, bool(t->v64), st);
  k_group_emit<<<grid_for(G, 256), 256, 0, st>>>(starts.as<uint32_t>(), G, kpos.as<uint32_t>(),
                                                 gsum.as<double>(), cols_of(s), mcols_of(o),
                                                 t->order, o->v32.as<float>(),
                                                 o->v64.as<double>());
  check_launch("k_group_emit");
  o->has_sorted = true;
  std::copy(identity, identity + t->order, o->sorted_under);
  HBK_CUDA(cudaStreamSynchronize(st));
  return o;
}

// ---------------------------------------------------- K2: CSF levels --
// build_csf, formats.py:143-162: a node starts at level d wherever any of
// the permuted coordinates 0..d changes.  lvl[i] = first changed level
// (order-1 for an exact duplicate, 0 for entry 0); node k of level d starts
// at the k-th entry with lvl <= d.

__global__ void k_change_level(Cols pc, int nlev, int64_t M, uint8_t* __restrict__ lvl) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    int l = 0;
    if (i > 0) {
      l = nlev;
      for (int d = 0; d < nlev; ++d) {
        if (pc.c[d][i] != pc.c[d][i - 1]) {
          l = d;
          break;
        }
      }
    }
    lvl[i] = uint8_t(l);
  }
}

__global__ void k_level_flags(const uint8_t* __restrict__ lvl, int d, int64_t M,
                              uint32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    f[i] = lvl[i] <= d;
}

__global__ void k_level_scatter(const uint8_t* __restrict__ lvl, int d,
                                const uint32_t* __restrict__ pos, const uint32_t* __restrict__ col,
                                int64_t M, uint32_t* __restrict__ idx,
                                uint32_t* __restrict__ start) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (lvl[i] <= d) {
      uint32_t p = pos[i];
      idx[p] = col[i];
      start[p] = uint32_t(i);
    }
  }
}

// ptrs[d][j] = position of node j's first entry among level d+1 nodes
// (np.searchsorted(starts[d+1], starts[d] ∪ {m}), formats.py:157-160).
__global__ void k_level_ptr(const uint32_t* __restrict__ start, const uint32_t* __restrict__ pos_next,
                            int64_t n, uint32_t n_next, uint32_t* __restrict__ ptr) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= n;
       j += int64_t(gridDim.x) * blockDim.x)
    ptr[j] = (j == n) ? n_next : pos_next[start[j]];
}

__global__ void k_leaf_ptr(const uint32_t* __restrict__ start, int64_t n, uint32_t M,
                           uint32_t* __restrict__ ptr) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= n;
       j += int64_t(gridDim.x) * blockDim.x)
    ptr[j] = (j == n) ? M : start[j];
}

__global__ void k_fiber_anc(const uint32_t* __restrict__ start, int64_t F,
                            const uint32_t* __restrict__ col, uint32_t* __restrict__ anc) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x)
    anc[f] = col[start[f]];
}

struct BuildKeep {
  Scratch lvl;   // uint8 [M]
  Scratch pos0;  // uint32 [M+1] exclusive scan of level-0 starts
  bool want = false;
};

// CSF tree over entries already sorted under mo.  pc.c[d] = permuted column d
// (coordinates of mode mo[d]); leaf/v32/v64 are shared, not copied.
static hbk_csf* csf_from_sorted(int order, const int64_t* dims, const int* mo, int64_t M, Cols pc,
                                Buf leaf, Buf v32, Buf v64, cudaStream_t st, BuildKeep* keep) {
  HBK_REQUIRE(M < (int64_t(1) << 31) - 1, HBK_EINVAL, "nnz must be below 2^31-1");
  hbk_csf* c = new hbk_csf();
  std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> guard(c, [](hbk_csf* p) { hbk_csf_release(p); });
  c->order = order;
  std::memcpy(c->dims, dims, sizeof(c->dims));
  std::copy(mo, mo + order, c->mode_order);
  c->M = M;
  c->leaf = leaf;
  c->v32 = v32;
  c->v64 = v64;
  const int nlev = order - 1;
  if (M == 0) {  // formats.py:133-141
    for (int d = 0; d < nlev; ++d) {
      c->n[d] = 0;
      c->ptr[d] = dalloc(sizeof(uint32_t), st);
      HBK_CUDA(cudaMemsetAsync(c->ptr[d].p, 0, sizeof(uint32_t), st));
      c->idx[d] = dalloc(0, st);
    }
    HBK_CUDA(cudaStreamSynchronize(st));
    return guard.release();
  }
  Scratch lvl(M, st);
  k_change_level<<<grid_for(M, 256), 256, 0, st>>>(pc, nlev, M, lvl.as<uint8_t>());
  check_launch("k_change_level");
  std::vector<Scratch> pos;
  std::vector<Scratch> start;
  for (int d = 0; d < nlev; ++d) {
    pos.emplace_back((M + 1) * sizeof(uint32_t), st);
    k_level_flags<<<grid_for(M, 256), 256, 0, st>>>(lvl.as<uint8_t>(), d, M,
                                                    pos[d].as<uint32_t>());
    check_launch("k_level_flags");
    uint32_t nd = exclusive_scan_total(pos[d].as<uint32_t>(), M, st);
    c->n[d] = nd;
    c->idx[d] = dalloc(nd * sizeof(uint32_t), st);
    start.emplace_back((nd + 1) * sizeof(uint32_t), st);
    k_level_scatter<<<grid_for(M, 256), 256, 0, st>>>(lvl.as<uint8_t>(), d, pos[d].as<uint32_t>(),
                                                      pc.c[d], M, c->idx[d].as<uint32_t>(),
                                                      start[d].as<uint32_t>());
    check_launch("k_level_scatter");
  }
  for (int d = 0; d < nlev - 1; ++d) {
    c->ptr[d] = dalloc((c->n[d] + 1) * sizeof(uint32_t), st);
    k_level_ptr<<<grid_for(c->n[d] + 1, 256), 256, 0, st>>>(
        start[d].as<uint32_t>(), pos[d + 1].as<uint32_t>(), c->n[d], uint32_t(c->n[d + 1]),
        c->ptr[d].as<uint32_t>());
    check_launch("k_level_ptr");
  }
  const int L = nlev - 1;  // leaf-parent level
  c->ptr[L] = dalloc((c->n[L] + 1) * sizeof(uint32_t), st);
  k_leaf_ptr<<<grid_for(c->n[L] + 1, 256), 256, 0, st>>>(start[L].as<uint32_t>(), c->n[L],
                                                         uint32_t(M), c->ptr[L].as<uint32_t>());
  check_launch("k_leaf_ptr");
  for (int d = 1; d < L; ++d) {  // order > 3: ancestor coordinates per fiber
    c->anc[d] = dalloc(c->n[L] * sizeof(uint32_t), st);
    k_fiber_anc<<<grid_for(c->n[L], 256), 256, 0, st>>>(start[L].as<uint32_t>(), c->n[L], pc.c[d],
                                                        c->anc[d].as<uint32_t>());
    check_launch("k_fiber_anc");
  }
  if (keep && keep->want) {
    keep->lvl = std::move(lvl);
    keep->pos0 = std::move(pos[0]);
  }
  HBK_CUDA(cudaStreamSynchronize(st));
  return guard.release();
}

static Cols permuted_cols(const hbk_coo* t, const int* mo) {
  Cols pc{};
  for (int d = 0; d < t->order; ++d) pc.c[d] = t->cols[mo[d]].as<uint32_t>();
  return pc;
}

// ------------------------------------------- slice metadata / classify --
// fiber_positions / leaf_offsets (formats.py:102-111): follow the pointer
// chain from slice s down to the leaf-parent level and to the nonzeros.
struct Chain {
  const uint32_t* ptr[HBK_MAX_ORDER];
  int nlev;
};

__global__ void k_slice_meta(Chain ch, int64_t S, uint32_t* __restrict__ fpos,
                             uint32_t* __restrict__ loff) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s <= S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t p = uint32_t(s);
    for (int d = 0; d < ch.nlev - 1; ++d) p = ch.ptr[d][p];
    if (fpos) fpos[s] = p;
    if (loff) loff[s] = ch.ptr[ch.nlev - 1][p];
  }
}

static Chain chain_of(const hbk_csf* c) {
  Chain ch{};
  ch.nlev = c->order - 1;
  for (int d = 0; d < ch.nlev; ++d) ch.ptr[d] = c->ptr[d].as<uint32_t>();
  return ch;
}

// classify_slices, formats.py:194-204.
__global__ void k_classify(const uint32_t* __restrict__ fpos, const uint32_t* __restrict__ loff,
                           int64_t S, uint8_t* __restrict__ label) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t m = loff[s + 1] - loff[s];
    uint32_t f = fpos[s + 1] - fpos[s];
    uint8_t l = HBK_SLICE_CSF;
    if (m >= 2 && m == f) l = HBK_SLICE_CSL;
    if (m == 1) l = HBK_SLICE_COO;
    label[s] = l;
  }
}

// -------------------------------------------------- HB-CSF partition --
// build_hbcsf, formats.py:265-294: entry labels = slice labels repeated over
// slice nnz; each class is a stable compaction.  Offsets come from per-slice
// scans (S-long), not M-long masks.

__global__ void k_class_counts(const uint8_t* __restrict__ label, const uint32_t* __restrict__ loff,
                               int64_t S, uint32_t* __restrict__ c0, uint32_t* __restrict__ c1,
                               uint32_t* __restrict__ c2, uint32_t* __restrict__ csl_ord) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t m = loff[s + 1] - loff[s];
    uint8_t l = label[s];
    c0[s] = l == HBK_SLICE_COO ? m : 0;
    c1[s] = l == HBK_SLICE_CSL ? m : 0;
    c2[s] = l == HBK_SLICE_CSF ? m : 0;
    csl_ord[s] = l == HBK_SLICE_CSL;
  }
}

struct PartOut {
  MCols coo;   // original mode numbering
  float* coo32;
  double* coo64;
  MCols csl;   // rest columns 0..order-2
  float* csl32;
  double* csl64;
  MCols csf;   // permuted columns 0..order-1
  float* csf32;
  double* csf64;
};

__global__ void k_partition(const uint8_t* __restrict__ lvl, const uint32_t* __restrict__ pos0,
                            const uint8_t* __restrict__ label, const uint32_t* __restrict__ loff,
                            const uint32_t* __restrict__ off0, const uint32_t* __restrict__ off1,
                            const uint32_t* __restrict__ off2, Cols orig, const int* mo_unused,
                            int order, Cols pc, const float* __restrict__ v32,
                            const double* __restrict__ v64, int64_t M, PartOut o) {
  (void)mo_unused;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t s = pos0[i] + (lvl[i] == 0) - 1;
    uint32_t r = uint32_t(i) - loff[s];
    uint8_t l = label[s];
    if (l == HBK_SLICE_COO) {
      uint32_t dst = off0[s] + r;
      for (int d = 0; d < order; ++d) o.coo.c[d][dst] = orig.c[d][i];
      o.coo32[dst] = v32[i];
      if (o.coo64) o.coo64[dst] = v64[i];
    } else if (l == HBK_SLICE_CSL) {
      uint32_t dst = off1[s] + r;
      for (int d = 1; d < order; ++d) o.csl.c[d - 1][dst] = pc.c[d][i];
      o.csl32[dst] = v32[i];
      if (o.csl64) o.csl64[dst] = v64[i];
    } else {
      uint32_t dst = off2[s] + r;
      for (int d = 0; d < order; ++d) o.csf.c[d][dst] = pc.c[d][i];
      o.csf32[dst] = v32[i];
      if (o.csf64) o.csf64[dst] = v64[i];
    }
  }
}

__global__ void k_csl_slices(const uint8_t* __restrict__ label, const uint32_t* __restrict__ csl_ord,
                             const uint32_t* __restrict__ off1, const uint32_t* __restrict__ idx0,
                             int64_t S, uint32_t Scsl, uint32_t Mcsl, uint32_t* __restrict__ sptr,
                             uint32_t* __restrict__ sidx) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    if (label[s] == HBK_SLICE_CSL) {
      uint32_t k = csl_ord[s];
      sptr[k] = off1[s];
      sidx[k] = idx0[s];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sptr[Scsl] = Mcsl;
}

// ------------------------------------------------------ K4: fiber split --
// split_fibers, balance.py:65-90.

__global__ void k_nseg(const uint32_t* __restrict__ lptr, int64_t F, uint32_t tau,
                       uint32_t* __restrict__ nseg, uint32_t* __restrict__ maxseg) {
  uint32_t local = 0;
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    uint32_t sz = lptr[f + 1] - lptr[f];
    uint32_t n = (sz + tau - 1) / tau;
    nseg[f] = n;
    local = max(local, n);
  }
  if (local) atomicMax(maxseg, local);
}

__global__ void k_split_fill(const uint32_t* __restrict__ lptr, const uint32_t* __restrict__ fidx,
                             Cols anc, int nanc, const uint32_t* __restrict__ segoff, int64_t F,
                             uint32_t tau, uint32_t M, uint32_t T, uint32_t* __restrict__ nptr,
                             uint32_t* __restrict__ nidx, MCols nanc_out) {
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < F;
       f += int64_t(gridDim.x) * blockDim.x) {
    uint32_t a = segoff[f], b = segoff[f + 1];
    uint32_t base = lptr[f];
    uint32_t x = fidx[f];
    for (uint32_t s = a; s < b; ++s) {
      nptr[s] = base + (s - a) * tau;
      nidx[s] = x;
      for (int d = 1; d <= nanc; ++d) nanc_out.c[d][s] = anc.c[d][f];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) nptr[T] = M;
}

__global__ void k_remap_ptr(const uint32_t* __restrict__ ptr, int64_t n,
                            const uint32_t* __restrict__ segoff, uint32_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= n;
       j += int64_t(gridDim.x) * blockDim.x)
    out[j] = segoff[ptr[j]];
}

// ---------------------------------------------------- K5: slice schedule --
// assign_slice_blocks, balance.py:153-189.  The greedy walk is restated with
// the leaf-pointer prefix sum P: a unit starting at fiber f closes at the
// first f' in (f, end] with P[f'] >= P[f] + target (acc resets at each
// close, balance.py:176-181), else the remainder [f, end) closes it.

__device__ __forceinline__ uint32_t unit_stop(const uint32_t* __restrict__ P, uint32_t start,
                                              uint32_t end, uint32_t target) {
  uint32_t want = P[start] + target;
  // fibers are non-empty, so the stop lies within `target` fibers
  uint32_t lo = start + 1, hi = min(end, start + target);
  if (P[hi] < want) return end;  // remainder unit
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (P[mid] >= want)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__global__ void k_sched_count(const uint32_t* __restrict__ fpos, const uint32_t* __restrict__ P,
                              int64_t S, uint32_t bs, uint32_t* __restrict__ cnt,
                              uint32_t* __restrict__ mult) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t b = fpos[s], e = fpos[s + 1];
    uint32_t m = P[e] - P[b];
    uint32_t mu = m <= bs ? 1u : (m + bs - 1) / bs;
    mult[s] = mu;
    if (m <= bs) {
      cnt[s] = 1;
      continue;
    }
    uint32_t target = (m + mu - 1) / mu;
    uint32_t k = 0;
    for (uint32_t f = b; f < e; f = unit_stop(P, f, e, target)) ++k;
    cnt[s] = k;
  }
}

__global__ void k_sched_fill(const uint32_t* __restrict__ fpos, const uint32_t* __restrict__ P,
                             const uint32_t* __restrict__ mult, const uint32_t* __restrict__ uoff,
                             int64_t S, uint32_t bs, uint32_t* __restrict__ units) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < S;
       s += int64_t(gridDim.x) * blockDim.x) {
    uint32_t b = fpos[s], e = fpos[s + 1];
    uint32_t m = P[e] - P[b];
    uint32_t u = uoff[s];
    if (m <= bs) {
      units[3 * u + 0] = uint32_t(s);
      units[3 * u + 1] = b;
      units[3 * u + 2] = e;
      continue;
    }
    uint32_t target = (m + mult[s] - 1) / mult[s];
    for (uint32_t f = b; f < e;) {
      uint32_t g = unit_stop(P, f, e, target);
      units[3 * u + 0] = uint32_t(s);
      units[3 * u + 1] = f;
      units[3 * u + 2] = g;
      ++u;
      f = g;
    }
  }
}

// BlockSchedule.validate_for, balance.py:128-150.  err[0] = first bad unit,
// err[1] = reason (1 partition, 2 starts outside, 3 crosses out).
__global__ void k_sched_validate(const uint32_t* __restrict__ units, int64_t U,
                                 const uint32_t* __restrict__ fpos, int64_t S,
                                 unsigned long long* __restrict__ err) {
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < U;
       u += int64_t(gridDim.x) * blockDim.x) {
    uint32_t sp = units[3 * u], fs = units[3 * u + 1], ft = units[3 * u + 2];
    uint32_t cursor = u == 0 ? 0u : units[3 * (u - 1) + 2];
    int why = 0;
    if (fs != cursor || ft <= fs)
      why = 1;
    else if (sp >= S || !(fpos[sp] <= fs && fs < fpos[sp + 1]))
      why = 2;
    else if (ft > fpos[sp + 1])
      why = 3;
    if (why) atomicMin(err, (static_cast<unsigned long long>(u) << 8) | unsigned(why));
  }
}

}  // namespace hbk

using namespace hbk;

// =================================================================== C ABI
extern "C" {

const char* hbk_last_error(void) { return g_last_error.c_str(); }
int hbk_abi_version(void) { return HBK_ABI_VERSION; }

int hbk_device_sms(int* sms) {
  return guarded([&] {
    int dev = 0;
    HBK_CUDA(cudaGetDevice(&dev));
    HBK_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  });
}

void hbk_coo_retain(hbk_coo* t) {
  if (t) t->ref++;
}
void hbk_coo_release(hbk_coo* t) {
  if (t && --t->ref == 0) delete t;
}
void hbk_csl_retain(hbk_csl* s) {
  if (s) s->ref++;
}
void hbk_csl_release(hbk_csl* s) {
  if (s && --s->ref == 0) delete s;
}
void hbk_csf_retain(hbk_csf* c) {
  if (c) c->ref++;
}
void hbk_csf_release(hbk_csf* c) {
  if (c && --c->ref == 0) delete c;
}
void hbk_sched_retain(hbk_sched* s) {
  if (s) s->ref++;
}
void hbk_sched_release(hbk_sched* s) {
  if (s && --s->ref == 0) delete s;
}

}  // extern "C"

namespace hbk {
__global__ void k_unpack_rowmajor(const uint32_t* __restrict__ idx, int order, int64_t M,
                                  MCols out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    for (int d = 0; d < order; ++d) out.c[d][i] = idx[i * order + d];
}
__global__ void k_pack_rowmajor(Cols in, int order, int64_t M, uint32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    for (int d = 0; d < order; ++d) idx[i * order + d] = in.c[d][i];
}
__global__ void k_f64_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = float(a[i]);
}
__global__ void k_f32_to_f64(const float* __restrict__ a, int64_t n, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = double(a[i]);
}

static hbk_coo* coo_create(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx,
                           const double* v64, const float* v32, const int* sorted_under,
                           cudaStream_t st) {
  HBK_REQUIRE(order >= 3 && order <= HBK_MAX_ORDER, HBK_EINVAL,
              "tensor order must be >= 3 (and <= 8 in this build)");
  for (int d = 0; d < order; ++d)
    HBK_REQUIRE(dims[d] >= 1 && dims[d] <= 0xFFFFFFFFll, HBK_EINVAL,
                "all dimensions must be positive (and fit in uint32)");
  HBK_REQUIRE(nnz >= 0 && nnz < (int64_t(1) << 31) - 1, HBK_EINVAL, "nnz must be in [0, 2^31-1)");
  hbk_coo* t = new hbk_coo();
  std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> guard(t, [](hbk_coo* p) { hbk_coo_release(p); });
  t->order = order;
  for (int d = 0; d < order; ++d) t->dims[d] = dims[d];
  t->nnz = nnz;
  for (int d = 0; d < order; ++d) t->cols[d] = dalloc(nnz * sizeof(uint32_t), st);
  t->v32 = dalloc(nnz * sizeof(float), st);
  if (nnz) {
    k_unpack_rowmajor<<<grid_for(nnz, 256), 256, 0, st>>>(idx, order, nnz, mcols_of(t));
    check_launch("k_unpack_rowmajor");
  }
  if (v64) {
    t->v64 = dalloc(nnz * sizeof(double), st);
    if (nnz) {
      HBK_CUDA(cudaMemcpyAsync(t->v64.p, v64, nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
      k_f64_to_f32<<<grid_for(nnz, 256), 256, 0, st>>>(v64, nnz, t->v32.as<float>());
      check_launch("k_f64_to_f32");
    }
  } else if (nnz) {
    HBK_CUDA(cudaMemcpyAsync(t->v32.p, v32, nnz * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  if (sorted_under) {
    check_mode_order(sorted_under, order);
    t->has_sorted = true;
    std::copy(sorted_under, sorted_under + order, t->sorted_under);
  }
  HBK_CUDA(cudaStreamSynchronize(st));
  return guard.release();
}

static void copy_u32_as_i64(const uint32_t* dev, int64_t n, int64_t* host, cudaStream_t st) {
  std::vector<uint32_t> tmp(n);
  if (n) HBK_CUDA(cudaMemcpyAsync(tmp.data(), dev, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  HBK_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) host[i] = tmp[i];
}

static void copy_values_f64(const Buf& v64, const Buf& v32, int64_t n, double* host,
                            cudaStream_t st) {
  if (!n) return;
  if (v64) {
    HBK_CUDA(cudaMemcpyAsync(host, v64.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  } else {
    Scratch t(n * sizeof(double), st);
    k_f32_to_f64<<<grid_for(n, 256), 256, 0, st>>>(v32.as<float>(), n, t.as<double>());
    check_launch("k_f32_to_f64");
    HBK_CUDA(cudaMemcpyAsync(host, t.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  HBK_CUDA(cudaStreamSynchronize(st));
}

static hbk_csl* csl_from_sorted_slices(const hbk_coo* s, const int* mo, cudaStream_t st);

}  // namespace hbk

extern "C" {

int hbk_coo_create(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx,
                   const double* vals, const int* sorted_under, void* stream, hbk_coo** out) {
  return guarded([&] {
    HBK_REQUIRE(vals || nnz == 0, HBK_EINVAL, "values pointer is NULL");
    static const double dummy = 0;
    *out = coo_create(order, dims, nnz, idx, vals ? vals : &dummy, nullptr, sorted_under,
                      to_stream(stream));
  });
}

int hbk_coo_create_f32(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx,
                       const float* vals, const int* sorted_under, void* stream, hbk_coo** out) {
  return guarded([&] {
    *out = coo_create(order, dims, nnz, idx, nullptr, vals, sorted_under, to_stream(stream));
  });
}

int hbk_coo_info_get(const hbk_coo* t, hbk_coo_info* info) {
  return guarded([&] {
    HBK_REQUIRE(t && info, HBK_EINVAL, "null handle");
    std::memset(info, 0, sizeof(*info));
    info->order = t->order;
    std::copy(t->dims, t->dims + t->order, info->dims);
    info->nnz = t->nnz;
    info->has_sorted = t->has_sorted;
    std::copy(t->sorted_under, t->sorted_under + t->order, info->sorted_under);
    info->unique_mode = t->unique_mode;
  });
}

int hbk_coo_export(const hbk_coo* t, uint32_t* idx, double* vals, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    const int64_t M = t->nnz;
    if (idx && M) {
      Scratch tmp(M * t->order * sizeof(uint32_t), st);
      k_pack_rowmajor<<<grid_for(M, 256), 256, 0, st>>>(cols_of(t), t->order, M,
                                                        tmp.as<uint32_t>());
      check_launch("k_pack_rowmajor");
      HBK_CUDA(cudaMemcpyAsync(idx, tmp.p, M * t->order * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               st));
      HBK_CUDA(cudaStreamSynchronize(st));
    }
    if (vals) copy_values_f64(t->v64, t->v32, M, vals, st);
  });
}

int hbk_coo_export_device(const hbk_coo* t, uint32_t* idx, double* v64, float* v32, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    const int64_t M = t->nnz;
    if (!M) return;
    if (idx) {
      k_pack_rowmajor<<<grid_for(M, 256), 256, 0, st>>>(cols_of(t), t->order, M, idx);
      check_launch("k_pack_rowmajor");
    }
    if (v32)
      HBK_CUDA(cudaMemcpyAsync(v32, t->v32.p, M * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (v64) {
      if (t->v64) {
        HBK_CUDA(cudaMemcpyAsync(v64, t->v64.p, M * sizeof(double), cudaMemcpyDeviceToDevice, st));
      } else {
        k_f32_to_f64<<<grid_for(M, 256), 256, 0, st>>>(t->v32.as<float>(), M, v64);
        check_launch("k_f32_to_f64");
      }
    }
    HBK_CUDA(cudaStreamSynchronize(st));
  });
}

int hbk_coo_device_arrays(const hbk_coo* t, const uint32_t** cols, const float** vals32) {
  return guarded([&] {
    for (int d = 0; d < t->order; ++d) cols[d] = t->cols[d].as<uint32_t>();
    *vals32 = t->v32.as<float>();
  });
}

int hbk_coo_sort(hbk_coo* t, const int* mode_order, void* stream, hbk_coo** out) {
  return guarded([&] { *out = coo_sorted(t, mode_order, to_stream(stream)); });
}

int hbk_coo_canonicalize(const hbk_coo* t, int merge, void* stream, hbk_coo** out) {
  return guarded([&] {
    HBK_REQUIRE(merge == 0 || merge == 1, HBK_EINVAL, "merge must be 0 or 1");
    *out = coo_canonical(const_cast<hbk_coo*>(t), merge, to_stream(stream));
  });
}

int hbk_coo_slices(hbk_coo* t, int mode, void* stream, hbk_csl** out) {
  return guarded([&] {
    HBK_REQUIRE(mode >= 0 && mode < t->order, HBK_EINVAL, "mode out of range");
    cudaStream_t st = to_stream(stream);
    int mo[HBK_MAX_ORDER];
    // kernels.py:126-130: keep the given order if it is already mode-major,
    // else sort under (mode, *rest).
    if (t->has_sorted && t->sorted_under[0] == mode) {
      std::copy(t->sorted_under, t->sorted_under + t->order, mo);
    } else {
      int k = 0;
      mo[k++] = mode;
      for (int d = 0; d < t->order; ++d)
        if (d != mode) mo[k++] = d;
    }
    hbk_coo* s = coo_sorted(t, mo, st);
    std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> g(s, [](hbk_coo* p) { hbk_coo_release(p); });
    *out = csl_from_sorted_slices(s, mo, st);
  });
}

int hbk_csl_info_get(const hbk_csl* s, hbk_csl_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    info->order = s->order;
    std::copy(s->dims, s->dims + s->order, info->dims);
    std::copy(s->mode_order, s->mode_order + s->order, info->mode_order);
    info->num_slices = s->S;
    info->nnz = s->M;
  });
}

int hbk_csl_export(const hbk_csl* s, int which, void* host, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    switch (which) {
      case HBK_CSL_SLICE_PTR:
        copy_u32_as_i64(s->slice_ptr.as<uint32_t>(), s->S + 1, static_cast<int64_t*>(host), st);
        break;
      case HBK_CSL_SLICE_IDX:
        if (s->S)
          HBK_CUDA(cudaMemcpyAsync(host, s->slice_idx.p, s->S * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, st));
        HBK_CUDA(cudaStreamSynchronize(st));
        break;
      case HBK_CSL_REST_IDX: {
        if (s->M) {
          Cols c{};
          for (int d = 0; d < s->order - 1; ++d) c.c[d] = s->rest[d].as<uint32_t>();
          Scratch tmp(s->M * (s->order - 1) * sizeof(uint32_t), st);
          k_pack_rowmajor<<<grid_for(s->M, 256), 256, 0, st>>>(c, s->order - 1, s->M,
                                                               tmp.as<uint32_t>());
          check_launch("k_pack_rowmajor");
          HBK_CUDA(cudaMemcpyAsync(host, tmp.p, s->M * (s->order - 1) * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, st));
        }
        HBK_CUDA(cudaStreamSynchronize(st));
        break;
      }
      case HBK_CSL_VALUES:
        copy_values_f64(s->v64, s->v32, s->M, static_cast<double*>(host), st);
        break;
      default:
        throw Error(HBK_EINVAL, "unknown CSL array id");
    }
  });
}

int hbk_csf_info_get(const hbk_csf* c, hbk_csf_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    info->order = c->order;
    std::copy(c->dims, c->dims + c->order, info->dims);
    std::copy(c->mode_order, c->mode_order + c->order, info->mode_order);
    info->nnz = c->M;
    for (int d = 0; d < c->order - 1; ++d) info->level_sizes[d] = c->n[d];
    info->split = c->split;
  });
}

int hbk_csf_export(const hbk_csf* c, int which, int level, void* host, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    if (which == HBK_CSF_PTR || which == HBK_CSF_IDX)
      HBK_REQUIRE(level >= 0 && level < c->order - 1, HBK_EINVAL, "level out of range");
    switch (which) {
      case HBK_CSF_PTR:
        copy_u32_as_i64(c->ptr[level].as<uint32_t>(), c->n[level] + 1,
                        static_cast<int64_t*>(host), st);
        break;
      case HBK_CSF_IDX:
        if (c->n[level])
          HBK_CUDA(cudaMemcpyAsync(host, c->idx[level].p, c->n[level] * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, st));
        HBK_CUDA(cudaStreamSynchronize(st));
        break;
      case HBK_CSF_LEAF:
        if (c->M)
          HBK_CUDA(cudaMemcpyAsync(host, c->leaf.p, c->M * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, st));
        HBK_CUDA(cudaStreamSynchronize(st));
        break;
      case HBK_CSF_VALUES:
        copy_values_f64(c->v64, c->v32, c->M, static_cast<double*>(host), st);
        break;
      default:
        throw Error(HBK_EINVAL, "unknown CSF array id");
    }
  });
}

int hbk_build_csf(hbk_coo* t, const int* mode_order, void* stream, hbk_csf** out) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    hbk_coo* s = coo_sorted(t, mode_order, st);
    std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> g(s, [](hbk_coo* p) { hbk_coo_release(p); });
    *out = csf_from_sorted(t->order, t->dims, mode_order, s->nnz, permuted_cols(s, mode_order),
                           s->cols[mode_order[t->order - 1]], s->v32, s->v64, st, nullptr);
  });
}

int hbk_classify_slices(const hbk_csf* c, int8_t* labels, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    const int64_t S = c->n[0];
    if (S == 0) return;
    Scratch fpos((S + 1) * sizeof(uint32_t), st), loff((S + 1) * sizeof(uint32_t), st);
    Scratch lab(S, st);
    k_slice_meta<<<grid_for(S + 1, 256), 256, 0, st>>>(chain_of(c), S, fpos.as<uint32_t>(),
                                                       loff.as<uint32_t>());
    check_launch("k_slice_meta");
    k_classify<<<grid_for(S, 256), 256, 0, st>>>(fpos.as<uint32_t>(), loff.as<uint32_t>(), S,
                                                 lab.as<uint8_t>());
    check_launch("k_classify");
    HBK_CUDA(cudaMemcpyAsync(labels, lab.p, S, cudaMemcpyDeviceToHost, st));
    HBK_CUDA(cudaStreamSynchronize(st));
  });
}

namespace hbk {
// Slice and fiber population reductions (hbk_csf_population): per thread a
// grid-stride share of slices and fibers; u64 sums of squares, u32 maxima and
// class counts reduced per warp, then one atomic per warp.
// acc: [0] slice sumsq, [1] fiber sumsq, [2] COO slices, [3] CSL slices;
// mx: [0] max slice, [1] max fiber.
__global__ void k_population(const uint32_t* __restrict__ fpos, const uint32_t* __restrict__ loff,
                             int64_t S, const uint32_t* __restrict__ lptr, int64_t F,
                             unsigned long long* __restrict__ acc, unsigned int* __restrict__ mx) {
  unsigned long long sq_s = 0, sq_f = 0, n_coo = 0, n_csl = 0;
  unsigned int m_s = 0, m_f = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < S; i += stride) {
    const unsigned int x = loff[i + 1] - loff[i];
    const unsigned int nf = fpos[i + 1] - fpos[i];
    sq_s += (unsigned long long)x * x;
    m_s = max(m_s, x);
    n_coo += x == 1u;
    n_csl += (x >= 2u && x == nf);
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < F; i += stride) {
    const unsigned int x = lptr[i + 1] - lptr[i];
    sq_f += (unsigned long long)x * x;
    m_f = max(m_f, x);
  }
  for (int o = 16; o; o >>= 1) {
    sq_s += __shfl_xor_sync(0xFFFFFFFFu, sq_s, o);
    sq_f += __shfl_xor_sync(0xFFFFFFFFu, sq_f, o);
    n_coo += __shfl_xor_sync(0xFFFFFFFFu, n_coo, o);
    n_csl += __shfl_xor_sync(0xFFFFFFFFu, n_csl, o);
  }
  m_s = __reduce_max_sync(0xFFFFFFFFu, m_s);
  m_f = __reduce_max_sync(0xFFFFFFFFu, m_f);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc + 0, sq_s);
    atomicAdd(acc + 1, sq_f);
    atomicAdd(acc + 2, n_coo);
    atomicAdd(acc + 3, n_csl);
    atomicMax(mx + 0, m_s);
    atomicMax(mx + 1, m_f);
  }
}
}  // namespace hbk

int hbk_csf_population(const hbk_csf* c, hbk_population* out, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    std::memset(out, 0, sizeof(*out));
    const int64_t S = c->n[0], F = c->n[c->order - 2];
    out->slices = S;
    out->fibers = F;
    out->nnz = c->M;
    if (S == 0) return;
    Scratch fpos((S + 1) * sizeof(uint32_t), st), loff((S + 1) * sizeof(uint32_t), st);
    Scratch red(6 * sizeof(unsigned long long), st);
    HBK_CUDA(cudaMemsetAsync(red.p, 0, 6 * sizeof(unsigned long long), st));
    k_slice_meta<<<grid_for(S + 1, 256), 256, 0, st>>>(chain_of(c), S, fpos.as<uint32_t>(),
                                                       loff.as<uint32_t>());
    check_launch("k_slice_meta");
    auto* acc = red.as<unsigned long long>();
    k_population<<<grid_for(std::max(S, F), 256), 256, 0, st>>>(
        fpos.as<uint32_t>(), loff.as<uint32_t>(), S, c->ptr[c->order - 2].as<uint32_t>(), F, acc,
        reinterpret_cast<unsigned int*>(acc + 4));
    check_launch("k_population");
    unsigned long long h[6];
    HBK_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    HBK_CUDA(cudaStreamSynchronize(st));
    const unsigned int* hm = reinterpret_cast<const unsigned int*>(h + 4);
    out->sumsq_slice = h[0];
    out->sumsq_fiber = h[1];
    out->coo_slices = int64_t(h[2]);
    out->csl_slices = int64_t(h[3]);
    out->csf_slices = S - out->coo_slices - out->csl_slices;
    out->max_slice = hm[0];
    out->max_fiber = hm[1];
  });
}

int hbk_build_hbcsf(hbk_coo* t, const int* mo, void* stream, hbk_coo** coo_part,
                    hbk_csl** csl_part, hbk_csf** csf_part) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    const int order = t->order;
    hbk_coo* s = coo_sorted(t, mo, st);
    std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> gs(s, [](hbk_coo* p) { hbk_coo_release(p); });
    const int64_t M = s->nnz;
    Cols pc = permuted_cols(s, mo);
    BuildKeep keep;
    keep.want = true;
    hbk_csf* full = csf_from_sorted(order, t->dims, mo, M, pc, s->cols[mo[order - 1]], s->v32,
                                    s->v64, st, &keep);
    std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> gf(full, [](hbk_csf* p) { hbk_csf_release(p); });
    const int64_t S = full->n[0];
    const bool w64 = bool(s->v64);

    Scratch fpos((S + 1) * sizeof(uint32_t), st), loff((S + 1) * sizeof(uint32_t), st);
    Scratch label(S ? S : 1, st);
    Scratch c0((S + 1) * sizeof(uint32_t), st), c1((S + 1) * sizeof(uint32_t), st),
        c2((S + 1) * sizeof(uint32_t), st), cord((S + 1) * sizeof(uint32_t), st);
    uint32_t M0 = 0, M1 = 0, M2 = 0, S1 = 0;
    if (S) {
      k_slice_meta<<<grid_for(S + 1, 256), 256, 0, st>>>(chain_of(full), S, fpos.as<uint32_t>(),
                                                         loff.as<uint32_t>());
      check_launch("k_slice_meta");
      k_classify<<<grid_for(S, 256), 256, 0, st>>>(fpos.as<uint32_t>(), loff.as<uint32_t>(), S,
                                                   label.as<uint8_t>());
      check_launch("k_classify");
      k_class_counts<<<grid_for(S, 256), 256, 0, st>>>(label.as<uint8_t>(), loff.as<uint32_t>(),
                                                       S, c0.as<uint32_t>(), c1.as<uint32_t>(),
                                                       c2.as<uint32_t>(), cord.as<uint32_t>());
      check_launch("k_class_counts");
      M0 = exclusive_scan_total(c0.as<uint32_t>(), S, st);
      M1 = exclusive_scan_total(c1.as<uint32_t>(), S, st);
      M2 = exclusive_scan_total(c2.as<uint32_t>(), S, st);
      S1 = exclusive_scan_total(cord.as<uint32_t>(), S, st);
    }
    // COO bucket: unpermuted coordinates, sorted under mo (formats.py:273-275)
    hbk_coo* coo = new_coo_like(s, M0, w64, st);
    std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> gc(coo, [](hbk_coo* p) { hbk_coo_release(p); });
    coo->has_sorted = true;
    std::copy(mo, mo + order, coo->sorted_under);
    coo->unique_mode = mo[0];
    // CSL bucket (formats.py:277-289)
    hbk_csl* csl = new hbk_csl();
    std::unique_ptr<hbk_csl, void (*)(hbk_csl*)> gl(csl, [](hbk_csl* p) { hbk_csl_release(p); });
    csl->order = order;
    std::memcpy(csl->dims, t->dims, sizeof(csl->dims));
    std::copy(mo, mo + order, csl->mode_order);
    csl->S = S1;
    csl->M = M1;
    csl->slice_ptr = dalloc((S1 + 1) * sizeof(uint32_t), st);
    csl->slice_idx = dalloc(S1 * sizeof(uint32_t), st);
    for (int d = 0; d < order - 1; ++d) csl->rest[d] = dalloc(M1 * sizeof(uint32_t), st);
    csl->v32 = dalloc(M1 * sizeof(float), st);
    if (w64) csl->v64 = dalloc(M1 * sizeof(double), st);
    // CSF bucket entries (permuted), rebuilt as a tree below (formats.py:291-294)
    MCols csfc{};
    std::vector<Buf> csfcols;
    for (int d = 0; d < order; ++d) {
      csfcols.push_back(dalloc(M2 * sizeof(uint32_t), st));
      csfc.c[d] = csfcols.back().as<uint32_t>();
    }
    Buf csf32 = dalloc(M2 * sizeof(float), st);
    Buf csf64;
    if (w64) csf64 = dalloc(M2 * sizeof(double), st);
    if (S) {
      MCols cslc{};
      for (int d = 0; d < order - 1; ++d) cslc.c[d] = csl->rest[d].as<uint32_t>();
      PartOut po{mcols_of(coo), coo->v32.as<float>(), coo->v64.as<double>(),
                 cslc,          csl->v32.as<float>(), csl->v64.as<double>(),
                 csfc,          csf32.as<float>(),    csf64.as<double>()};
      k_partition<<<grid_for(M, 256), 256, 0, st>>>(
          keep.lvl.as<uint8_t>(), keep.pos0.as<uint32_t>(), label.as<uint8_t>(),
          loff.as<uint32_t>(), c0.as<uint32_t>(), c1.as<uint32_t>(), c2.as<uint32_t>(),
          cols_of(s), nullptr, order, pc, s->v32.as<float>(), s->v64.as<double>(), M, po);
      check_launch("k_partition");
      k_csl_slices<<<grid_for(S, 256), 256, 0, st>>>(
          label.as<uint8_t>(), cord.as<uint32_t>(), c1.as<uint32_t>(), full->idx[0].as<uint32_t>(),
          S, S1, M1, csl->slice_ptr.as<uint32_t>(), csl->slice_idx.as<uint32_t>());
      check_launch("k_csl_slices");
    } else {
      HBK_CUDA(cudaMemsetAsync(csl->slice_ptr.p, 0, sizeof(uint32_t), st));
    }
    Cols cpc{};
    for (int d = 0; d < order; ++d) cpc.c[d] = csfcols[d].as<uint32_t>();
    hbk_csf* csf = csf_from_sorted(order, t->dims, mo, M2, cpc, csfcols[order - 1], csf32, csf64,
                                   st, nullptr);
    HBK_CUDA(cudaStreamSynchronize(st));
    *coo_part = gc.release();
    *csl_part = gl.release();
    *csf_part = csf;
  });
}

int hbk_split_fibers(const hbk_csf* c, int64_t tau64, void* stream, hbk_csf** out) {
  return guarded([&] {
    HBK_REQUIRE(tau64 >= 1, HBK_EINVAL, "fiber_threshold must be at least 1");
    cudaStream_t st = to_stream(stream);
    *out = nullptr;
    const int L = c->order - 2;
    const int64_t F = c->n[L];
    if (c->M == 0 || F == 0) return;
    const uint32_t tau = tau64 > 0xFFFFFFFFll ? 0xFFFFFFFFu : uint32_t(tau64);
    Scratch nseg((F + 1) * sizeof(uint32_t), st), mx(sizeof(uint32_t), st);
    HBK_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(uint32_t), st));
    k_nseg<<<grid_for(F, 256), 256, 0, st>>>(c->ptr[L].as<uint32_t>(), F, tau, nseg.as<uint32_t>(),
                                             mx.as<uint32_t>());
    check_launch("k_nseg");
    if (read_u32(mx.as<uint32_t>(), st) <= 1) return;  // balance.py:70-71
    uint32_t T = exclusive_scan_total(nseg.as<uint32_t>(), F, st);
    hbk_csf* o = new hbk_csf();
    std::unique_ptr<hbk_csf, void (*)(hbk_csf*)> g(o, [](hbk_csf* p) { hbk_csf_release(p); });
    o->order = c->order;
    std::memcpy(o->dims, c->dims, sizeof(o->dims));
    std::copy(c->mode_order, c->mode_order + c->order, o->mode_order);
    o->M = c->M;
    for (int d = 0; d <= L; ++d) {
      o->n[d] = c->n[d];
      o->ptr[d] = c->ptr[d];
      o->idx[d] = c->idx[d];
      o->anc[d] = c->anc[d];
    }
    o->leaf = c->leaf;
    o->v32 = c->v32;
    o->v64 = c->v64;
    o->split = true;
    o->n[L] = T;
    o->ptr[L] = dalloc((T + 1) * sizeof(uint32_t), st);
    o->idx[L] = dalloc(T * sizeof(uint32_t), st);
    Cols anc{};
    MCols nanc{};
    for (int d = 1; d < L; ++d) {
      anc.c[d] = c->anc[d].as<uint32_t>();
      o->anc[d] = dalloc(T * sizeof(uint32_t), st);
      nanc.c[d] = o->anc[d].as<uint32_t>();
    }
    k_split_fill<<<grid_for(F, 128), 128, 0, st>>>(
        c->ptr[L].as<uint32_t>(), c->idx[L].as<uint32_t>(), anc, L - 1, nseg.as<uint32_t>(), F,
        tau, uint32_t(c->M), T, o->ptr[L].as<uint32_t>(), o->idx[L].as<uint32_t>(), nanc);
    check_launch("k_split_fill");
    // parents now address segment positions (balance.py:86-87)
    o->ptr[L - 1] = dalloc((c->n[L - 1] + 1) * sizeof(uint32_t), st);
    k_remap_ptr<<<grid_for(c->n[L - 1] + 1, 256), 256, 0, st>>>(
        c->ptr[L - 1].as<uint32_t>(), c->n[L - 1], nseg.as<uint32_t>(),
        o->ptr[L - 1].as<uint32_t>());
    check_launch("k_remap_ptr");
    HBK_CUDA(cudaStreamSynchronize(st));
    *out = g.release();
  });
}

int hbk_assign_slice_blocks(const hbk_csf* c, int64_t block_size, void* stream, hbk_sched** out) {
  return guarded([&] {
    HBK_REQUIRE(block_size >= 1 && block_size < (int64_t(1) << 31), HBK_EINVAL,
                "block_size must be positive");
    cudaStream_t st = to_stream(stream);
    const int64_t S = c->n[0];
    const int L = c->order - 2;
    hbk_sched* s = new hbk_sched();
    std::unique_ptr<hbk_sched, void (*)(hbk_sched*)> g(s, [](hbk_sched* p) { hbk_sched_release(p); });
    s->S = S;
    s->F = c->n[L];
    s->block_size = block_size;
    s->mult = dalloc(S * sizeof(uint32_t), st);
    if (S == 0) {
      s->units = dalloc(0, st);
      *out = g.release();
      return;
    }
    Scratch fpos((S + 1) * sizeof(uint32_t), st), cnt((S + 1) * sizeof(uint32_t), st);
    k_slice_meta<<<grid_for(S + 1, 256), 256, 0, st>>>(chain_of(c), S, fpos.as<uint32_t>(),
                                                       nullptr);
    check_launch("k_slice_meta");
    k_sched_count<<<grid_for(S, 64), 64, 0, st>>>(fpos.as<uint32_t>(), c->ptr[L].as<uint32_t>(), S,
                                                  uint32_t(block_size), cnt.as<uint32_t>(),
                                                  s->mult.as<uint32_t>());
    check_launch("k_sched_count");
    uint32_t U = exclusive_scan_total(cnt.as<uint32_t>(), S, st);
    s->U = U;
    s->units = dalloc(size_t(U) * 3 * sizeof(uint32_t), st);
    k_sched_fill<<<grid_for(S, 64), 64, 0, st>>>(fpos.as<uint32_t>(), c->ptr[L].as<uint32_t>(),
                                                 s->mult.as<uint32_t>(), cnt.as<uint32_t>(), S,
                                                 uint32_t(block_size), s->units.as<uint32_t>());
    check_launch("k_sched_fill");
    HBK_CUDA(cudaStreamSynchronize(st));
    *out = g.release();
  });
}

int hbk_sched_from_units(const hbk_csf* c, const int64_t* units, int64_t U, const int64_t* mult,
                         void* stream, hbk_sched** out) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    hbk_sched* s = new hbk_sched();
    std::unique_ptr<hbk_sched, void (*)(hbk_sched*)> g(s, [](hbk_sched* p) { hbk_sched_release(p); });
    const int64_t S = c->n[0];
    s->S = S;
    s->F = c->n[c->order - 2];
    s->U = U;
    std::vector<uint32_t> hu(U * 3), hm(S);
    for (int64_t u = 0; u < U; ++u) {
      HBK_REQUIRE(units[4 * u + 1] >= 0 && units[4 * u + 1] < 0xFFFFFFFFll &&
                      units[4 * u + 2] >= 0 && units[4 * u + 3] >= 0 &&
                      units[4 * u + 3] < 0xFFFFFFFFll,
                  HBK_EINVAL, "schedule unit field out of range");
      hu[3 * u] = uint32_t(units[4 * u + 1]);
      hu[3 * u + 1] = uint32_t(units[4 * u + 2]);
      hu[3 * u + 2] = uint32_t(units[4 * u + 3]);
    }
    for (int64_t i = 0; i < S; ++i) hm[i] = mult ? uint32_t(mult[i]) : 1u;
    s->units = dalloc(hu.size() * sizeof(uint32_t), st);
    s->mult = dalloc(hm.size() * sizeof(uint32_t), st);
    if (U)
      HBK_CUDA(cudaMemcpyAsync(s->units.p, hu.data(), hu.size() * 4, cudaMemcpyHostToDevice, st));
    if (S) HBK_CUDA(cudaMemcpyAsync(s->mult.p, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice, st));
    HBK_CUDA(cudaStreamSynchronize(st));
    *out = g.release();
  });
}

int hbk_sched_info_get(const hbk_sched* s, hbk_sched_info* info) {
  return guarded([&] {
    info->num_units = s->U;
    info->num_slices = s->S;
    info->num_fibers = s->F;
    info->block_size = s->block_size;
  });
}

int hbk_sched_export(const hbk_sched* s, int which, int64_t* host, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    if (which == HBK_SCHED_UNITS) {
      std::vector<uint32_t> hu(s->U * 3);
      if (s->U)
        HBK_CUDA(cudaMemcpyAsync(hu.data(), s->units.p, hu.size() * 4, cudaMemcpyDeviceToHost, st));
      HBK_CUDA(cudaStreamSynchronize(st));
      for (int64_t u = 0; u < s->U; ++u) {
        host[4 * u] = u;
        host[4 * u + 1] = hu[3 * u];
        host[4 * u + 2] = hu[3 * u + 1];
        host[4 * u + 3] = hu[3 * u + 2];
      }
    } else if (which == HBK_SCHED_MULT) {
      copy_u32_as_i64(s->mult.as<uint32_t>(), s->S, host, st);
    } else {
      throw Error(HBK_EINVAL, "unknown schedule array id");
    }
  });
}

int hbk_sched_validate(const hbk_sched* s, const hbk_csf* c, void* stream) {
  return guarded([&] {
    cudaStream_t st = to_stream(stream);
    const int64_t S = c->n[0], F = c->n[c->order - 2];
    if (S != s->S || F != s->F)
      throw Error(HBK_EINVAL, "schedule was built for " + std::to_string(s->S) + " slices/" +
                                  std::to_string(s->F) + " fibers, tensor has " +
                                  std::to_string(S) + "/" + std::to_string(F));
    Scratch fpos((S + 1) * sizeof(uint32_t), st), err(sizeof(unsigned long long), st);
    HBK_CUDA(cudaMemsetAsync(err.p, 0xFF, sizeof(unsigned long long), st));
    if (S) {
      k_slice_meta<<<grid_for(S + 1, 256), 256, 0, st>>>(chain_of(c), S, fpos.as<uint32_t>(),
                                                         nullptr);
      check_launch("k_slice_meta");
    }
    if (s->U) {
      k_sched_validate<<<grid_for(s->U, 256), 256, 0, st>>>(s->units.as<uint32_t>(), s->U,
                                                            fpos.as<uint32_t>(), S,
                                                            err.as<unsigned long long>());
      check_launch("k_sched_validate");
    }
    unsigned long long e = 0;
    HBK_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(e), cudaMemcpyDeviceToHost, st));
    HBK_CUDA(cudaStreamSynchronize(st));
    if (e != ~0ull) {
      uint64_t u = e >> 8;
      int why = int(e & 0xFF);
      uint32_t sp = 0;
      HBK_CUDA(cudaMemcpy(&sp, s->units.as<uint32_t>() + 3 * u, 4, cudaMemcpyDeviceToHost));
      if (why == 1) throw Error(HBK_EINVAL, "schedule units do not partition the fibers");
      if (why == 2)
        throw Error(HBK_EINVAL, "unit " + std::to_string(u) + " starts outside slice " +
                                    std::to_string(sp));
      throw Error(HBK_EINVAL,
                  "unit " + std::to_string(u) + " crosses out of slice " + std::to_string(sp));
    }
    uint32_t last = 0;
    if (s->U) {
      HBK_CUDA(cudaMemcpy(&last, s->units.as<uint32_t>() + 3 * (s->U - 1) + 2, 4,
                          cudaMemcpyDeviceToHost));
    }
    if (int64_t(last) != F) throw Error(HBK_EINVAL, "schedule does not cover all fibers");
  });
}

}  // extern "C"

// ----------------------------------------------------- COO slice view --
namespace hbk {
__global__ void k_slice_flags(const uint32_t* __restrict__ col, int64_t M,
                              uint32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    f[i] = (i == 0) || col[i] != col[i - 1];
}
__global__ void k_slice_emit(const uint32_t* __restrict__ col, const uint32_t* __restrict__ pos,
                             int64_t M, uint32_t S, uint32_t* __restrict__ sptr,
                             uint32_t* __restrict__ sidx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (pos[i + 1] != pos[i]) {
      sptr[pos[i]] = uint32_t(i);
      sidx[pos[i]] = col[i];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sptr[S] = uint32_t(M);
}

static hbk_csl* csl_from_sorted_slices(const hbk_coo* s, const int* mo, cudaStream_t st) {
  const int64_t M = s->nnz;
  hbk_csl* c = new hbk_csl();
  std::unique_ptr<hbk_csl, void (*)(hbk_csl*)> g(c, [](hbk_csl* p) { hbk_csl_release(p); });
  c->order = s->order;
  std::memcpy(c->dims, s->dims, sizeof(c->dims));
  std::copy(mo, mo + s->order, c->mode_order);
  c->M = M;
  for (int d = 1; d < s->order; ++d) c->rest[d - 1] = s->cols[mo[d]];
  c->v32 = s->v32;
  c->v64 = s->v64;
  Scratch pos((M + 1) * sizeof(uint32_t), st);
  uint32_t S = 0;
  if (M) {
    k_slice_flags<<<grid_for(M, 256), 256, 0, st>>>(s->cols[mo[0]].as<uint32_t>(), M,
                                                    pos.as<uint32_t>());
    check_launch("k_slice_flags");
    S = exclusive_scan_total(pos.as<uint32_t>(), M, st);
  }
  c->S = S;
  c->slice_ptr = dalloc((S + 1) * sizeof(uint32_t), st);
  c->slice_idx = dalloc(S * sizeof(uint32_t), st);
  if (M) {
    k_slice_emit<<<grid_for(M, 256), 256, 0, st>>>(s->cols[mo[0]].as<uint32_t>(),
                                                   pos.as<uint32_t>(), M, S,
                                                   c->slice_ptr.as<uint32_t>(),
                                                   c->slice_idx.as<uint32_t>());
    check_launch("k_slice_emit");
  } else {
    HBK_CUDA(cudaMemsetAsync(c->slice_ptr.p, 0, sizeof(uint32_t), st));
  }
  HBK_CUDA(cudaStreamSynchronize(st));
  return g.release();
}

// ------------------------------------------------------------- sharding --
__global__ void k_hist(const uint32_t* __restrict__ col, int64_t M,
                       unsigned long long* __restrict__ h) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(h + col[i], 1ull);
}
__global__ void k_row_flags(const uint32_t* __restrict__ col, int64_t M, uint32_t lo, uint32_t hi,
                            uint32_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    f[i] = col[i] >= lo && col[i] < hi;
}
__global__ void k_row_compact(const uint32_t* __restrict__ pos, Cols in, MCols out, int order,
                              const float* __restrict__ v32, const double* __restrict__ v64,
                              int64_t M, float* __restrict__ o32, double* __restrict__ o64,
                              int shift_mode, uint32_t shift) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (pos[i + 1] != pos[i]) {
      uint32_t d = pos[i];
      for (int m = 0; m < order; ++m) out.c[m][d] = in.c[m][i] - (m == shift_mode ? shift : 0u);
      o32[d] = v32[i];
      if (o64) o64[d] = v64[i];
    }
  }
}
}  // namespace hbk

extern "C" int hbk_coo_slice_histogram(const hbk_coo* t, int mode, int64_t* hist, void* stream) {
  return guarded([&] {
    HBK_REQUIRE(mode >= 0 && mode < t->order, HBK_EINVAL, "mode out of range");
    cudaStream_t st = to_stream(stream);
    HBK_CUDA(cudaMemsetAsync(hist, 0, t->dims[mode] * sizeof(int64_t), st));
    if (t->nnz) {
      k_hist<<<grid_for(t->nnz, 256), 256, 0, st>>>(t->cols[mode].as<uint32_t>(), t->nnz,
                                                    reinterpret_cast<unsigned long long*>(hist));
      check_launch("k_hist");
    }
  });
}

namespace hbk {
__global__ void k_pair_keys(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t M,
                            uint64_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    key[i] = (uint64_t(a[i]) << 32) | b[i];
}
// one count per distinct (slice, mid) pair, into its slice
__global__ void k_distinct_hist(const uint64_t* __restrict__ key, int64_t M,
                                unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M;
       i += int64_t(gridDim.x) * blockDim.x)
    if (i == 0 || key[i] != key[i - 1]) atomicAdd(hist + (key[i] >> 32), 1ull);
}
}  // namespace hbk

extern "C" int hbk_coo_fiber_histogram(const hbk_coo* t, int mode, int mid_mode, int64_t* hist,
                                       void* stream) {
  return guarded([&] {
    HBK_REQUIRE(mode >= 0 && mode < t->order && mid_mode >= 0 && mid_mode < t->order &&
                    mid_mode != mode,
                HBK_EINVAL, "mode out of range");
    cudaStream_t st = to_stream(stream);
    HBK_CUDA(cudaMemsetAsync(hist, 0, t->dims[mode] * sizeof(int64_t), st));
    const int64_t M = t->nnz;
    if (M == 0) return;
    Scratch ka(M * 8, st), kb(M * 8, st);
    k_pair_keys<<<grid_for(M, 256), 256, 0, st>>>(t->cols[mode].as<uint32_t>(),
                                                  t->cols[mid_mode].as<uint32_t>(), M,
                                                  ka.as<uint64_t>());
    check_launch("k_pair_keys");
    int hi_bits = 1;
    while ((int64_t(1) << hi_bits) < t->dims[mode]) ++hi_bits;
    size_t tmp = 0;
    cub::DoubleBuffer<uint64_t> kbuf(ka.as<uint64_t>(), kb.as<uint64_t>());
    HBK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kbuf, int(M), 0, 32 + hi_bits, st));
    Scratch t_(tmp, st);
    HBK_CUDA(cub::DeviceRadixSort::SortKeys(t_.p, tmp, kbuf, int(M), 0, 32 + hi_bits, st));
    k_distinct_hist<<<grid_for(M, 256), 256, 0, st>>>(kbuf.Current(), M,
                                                      reinterpret_cast<unsigned long long*>(hist));
    check_launch("k_distinct_hist");
  });
}

static hbk_coo* coo_rows(const hbk_coo* t, int mode, int64_t lo, int64_t hi, bool rebase,
                         cudaStream_t st) {
    HBK_REQUIRE(mode >= 0 && mode < t->order, HBK_EINVAL, "mode out of range");
    HBK_REQUIRE(0 <= lo && lo <= hi && hi <= t->dims[mode], HBK_EINVAL, "row range out of bounds");
    HBK_REQUIRE(!rebase || hi > lo, HBK_EINVAL, "a rebased shard needs at least one row");
    const int64_t M = t->nnz;
    Scratch pos((M + 1) * sizeof(uint32_t), st);
    uint32_t K = 0;
    if (M) {
      k_row_flags<<<grid_for(M, 256), 256, 0, st>>>(t->cols[mode].as<uint32_t>(), M, uint32_t(lo),
                                                    uint32_t(hi), pos.as<uint32_t>());
      check_launch("k_row_flags");
      K = exclusive_scan_total(pos.as<uint32_t>(), M, st);
    }
    std::unique_ptr<hbk_coo, void (*)(hbk_coo*)> o(new_coo_like(t, K, bool(t->v64), st),
                                                [](hbk_coo* p) { hbk_coo_release(p); });
    if (K) {
      k_row_compact<<<grid_for(M, 256), 256, 0, st>>>(pos.as<uint32_t>(), cols_of(t), mcols_of(o.get()),
                                                      t->order, t->v32.as<float>(),
                                                      t->v64.as<double>(), M, o->v32.as<float>(),
                                                      o->v64.as<double>(), rebase ? mode : -1,
                                                      uint32_t(lo));
      check_launch("k_row_compact");
    }
    if (rebase) o->dims[mode] = hi - lo;
    o->has_sorted = t->has_sorted;
    std::copy(t->sorted_under, t->sorted_under + t->order, o->sorted_under);
    HBK_CUDA(cudaStreamSynchronize(st));
    return o.release();
}

extern "C" int hbk_coo_shard_rows(const hbk_coo* t, int mode, int64_t lo, int64_t hi,
                                  void* stream, hbk_coo** out) {
  return guarded([&] { *out = coo_rows(t, mode, lo, hi, true, to_stream(stream)); });
}

extern "C" int hbk_coo_select_rows(const hbk_coo* t, int mode, int64_t lo, int64_t hi,
                                   void* stream, hbk_coo** out) {
  return guarded([&] { *out = coo_rows(t, mode, lo, hi, false, to_stream(stream)); });
}
