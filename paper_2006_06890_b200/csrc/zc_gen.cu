// Native synthetic graph generators.
//
// The reference generators (csr.py:248-317) are numpy loops that need ~20 s
// at 2^20 vertices and cannot reach scale 27; these run on the GPU, write the
// CSR straight into a handle and are deterministic in (parameters, seed)
// through a counter-based hash (no sequential RNG state).
//
// R-MAT / Kronecker (GAP "kron", Graph500 parameters a,b,c = .57,.19,.19):
// the source bit of each of the `scale` levels is Bernoulli(c+d) and,
// given it, the destination bit is Bernoulli(b/(a+b)) or Bernoulli(d/(c+d)).
// Pass 1 draws every arc's source and counts out-degrees, pass 2 scans them
// into offsets, pass 3 draws each list's destinations in CSR order -- the
// arc multiset has exactly the R-MAT distribution and no sort is needed.
// Vertex ids are scrambled by a keyed Feistel bijection (GAP permutes ids).
// Duplicates and self loops are kept, as the reference does.
// Symmetrize appends the reverse arcs (csr.py:350-359 semantics, no dedup);
// lists are then sorted ascending like the reference's lexsort.
//
// Uniform (csr.py:270-282 semantics): out-degree uniform in
// [min_degree, max_degree], destinations uniform with no duplicate inside a
// list (rejection, as csr.py:248-267).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "zc_graph.cuh"
#include "zc_internal.cuh"

namespace zc {
namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(seed ^ (stream * 0xd1b54a32d192ed03ull)) + i);
}

// Keyed Feistel bijection on [0, 2^bits) with cycle walking.
struct Feistel {
  uint32_t half;  // bits per half (domain 2^(2*half) >= 2^bits)
  uint32_t bits;
  uint64_t key;
  __device__ __forceinline__ uint64_t f(uint64_t x, int r) const {
    return hash3(key, 100 + r, x) & ((1ull << half) - 1);
  }
  __device__ __forceinline__ uint64_t round_fwd(uint64_t x) const {
    uint64_t l = x >> half, r = x & ((1ull << half) - 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t nl = r, nr = l ^ f(r, k);
      l = nl;
      r = nr;
    }
    return (l << half) | r;
  }
  __device__ __forceinline__ uint64_t round_inv(uint64_t x) const {
    uint64_t l = x >> half, r = x & ((1ull << half) - 1);
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      const uint64_t pr = l, pl = r ^ f(l, k);
      l = pl;
      r = pr;
    }
    return (l << half) | r;
  }
  __device__ __forceinline__ uint64_t fwd(uint64_t x) const {
    do x = round_fwd(x); while (x >> bits);
    return x;
  }
  __device__ __forceinline__ uint64_t inv(uint64_t x) const {
    do x = round_inv(x); while (x >> bits);
    return x;
  }
};

struct RmatParams {
  uint32_t scale;
  uint32_t thr_src;   // P(src bit = 1) = c + d, 16-bit fixed point
  uint32_t thr_dst0;  // P(dst bit = 1 | src bit 0) = b / (a + b)
  uint32_t thr_dst1;  // P(dst bit = 1 | src bit 1) = d / (c + d)
  uint64_t seed;
  Feistel perm;
};

__device__ __forceinline__ uint64_t rmat_src(const RmatParams& p, uint64_t arc) {
  uint64_t s = 0, h = 0;
  for (uint32_t l = 0; l < p.scale; ++l) {
    if ((l & 3) == 0) h = hash3(p.seed, 1 + (l >> 2), arc);
    const uint32_t u = static_cast<uint32_t>(h >> ((l & 3) * 16)) & 0xffffu;
    s |= static_cast<uint64_t>(u < p.thr_src) << l;
  }
  return s;
}

__device__ __forceinline__ uint64_t rmat_dst(const RmatParams& p, uint64_t src_old,
                                             uint64_t key) {
  uint64_t d = 0, h = 0;
  for (uint32_t l = 0; l < p.scale; ++l) {
    if ((l & 3) == 0) h = hash3(p.seed, 32 + (l >> 2), key);
    const uint32_t u = static_cast<uint32_t>(h >> ((l & 3) * 16)) & 0xffffu;
    const uint32_t thr = (src_old >> l) & 1 ? p.thr_dst1 : p.thr_dst0;
    d |= static_cast<uint64_t>(u < thr) << l;
  }
  return d;
}

// Arcs of every global source whose destination lies in [lo, lo + nl): count
// them per local destination (FILL = false), or write the source into the
// destination's in-list (FILL = true; deg = cursors).
template <bool FILL>
__global__ void k_rmat_in_arcs(RmatParams p, uint64_t nv, const uint64_t* goff, uint64_t lo,
                               uint64_t nl, uint32_t* deg, const uint64_t* in_off,
                               uint32_t* in_e) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = goff[v], e = goff[v + 1];
    if (s == e) continue;
    const uint64_t src_old = p.perm.inv(v);
    for (uint64_t k = s + lane; k < e; k += 32) {
      const uint64_t d = p.perm.fwd(rmat_dst(p, src_old, (v << 32) | (k - s)));
      if (d < lo || d >= lo + nl) continue;
      const uint32_t slot = atomicAdd(deg + (d - lo), 1u);
      if (FILL) in_e[in_off[d - lo] + slot] = static_cast<uint32_t>(v);
    }
  }
}

__global__ void k_rmat_count(RmatParams p, uint64_t narcs, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < narcs;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = p.perm.fwd(rmat_src(p, i));
    atomicAdd(deg + s, 1u);
  }
}

// Warp per (permuted) vertex: its list in CSR order, lanes strided over k.
// vbase: global id of local vertex 0 (partition generation fills one range).
// woff (optional): write list lv at woff[lv] instead of off[lv] (the out-arcs
// of a symmetric partition's lists, whose in-arcs follow them).
template <typename ET>
__global__ void k_rmat_fill(RmatParams p, uint64_t nv, const uint64_t* off, ET* edges,
                            uint64_t vbase = 0, const uint64_t* woff = nullptr) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t lv = gw; lv < nv; lv += nw) {
    const uint64_t s = off[lv], e = off[lv + 1];
    if (s == e) continue;
    const uint64_t v = vbase + lv;
    const uint64_t src_old = p.perm.inv(v);
    const uint64_t w0 = woff ? woff[lv] : s;
    for (uint64_t k = s + lane; k < e; k += 32) {
      const uint64_t d_old = rmat_dst(p, src_old, (v << 32) | (k - s));
      edges[w0 + (k - s)] = static_cast<ET>(p.perm.fwd(d_old));
    }
  }
}

__global__ void k_add_u32(uint64_t n, uint32_t* a, const uint32_t* b) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

// Symmetrize: sym list of x = out-list of x followed by the sources of its
// in-arcs, then sorted.  cursor[x] starts at out_deg[x].
template <typename ET>
__global__ void k_sym_copy_out(uint64_t nv, const uint64_t* off, const ET* edges,
                               const uint64_t* soff, ET* sedges) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], e = off[v + 1], t = soff[v];
    for (uint64_t k = s + lane; k < e; k += 32) sedges[t + (k - s)] = edges[k];
  }
}

template <typename ET>
__global__ void k_sym_scatter_in(uint64_t nv, const uint64_t* off, const ET* edges,
                                 const uint64_t* soff, uint32_t* cursor, ET* sedges) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], e = off[v + 1];
    for (uint64_t k = s + lane; k < e; k += 32) {
      const uint64_t d = edges[k];
      const uint32_t pos = atomicAdd(cursor + d, 1u);
      sedges[soff[d] + pos] = static_cast<ET>(v);
    }
  }
}

template <typename ET>
__global__ void k_count_in(uint64_t ne, const ET* edges, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + edges[i], 1u);
}

__global__ void k_deg_from_off(uint64_t nv, const uint64_t* off, uint32_t* deg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x)
    deg[v] = static_cast<uint32_t>(off[v + 1] - off[v]);
}

template <typename ET>
__global__ void k_uniform_fill(uint64_t nv, uint64_t seed, const uint64_t* off, ET* edges) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = off[v], e = off[v + 1];
    uint64_t attempt = 0;
    for (uint64_t k = s; k < e; ++k) {
      uint64_t d;
      bool dup;
      do {
        d = hash3(seed, 2, (k << 8) ^ attempt++) % nv;
        dup = false;
        for (uint64_t t = s; t < k; ++t) dup |= (static_cast<uint64_t>(edges[t]) == d);
      } while (dup);
      edges[k] = static_cast<ET>(d);
    }
  }
}

__global__ void k_uniform_deg(uint64_t nv, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* deg) {
  const uint64_t span = static_cast<uint64_t>(hi) - lo + 1;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x)
    deg[v] = lo + static_cast<uint32_t>(hash3(seed, 1, v) % span);
}

__global__ void k_weights(uint64_t ne, uint64_t seed, int64_t lo, int64_t hi, uint32_t* w,
                          uint64_t ebase = 0) {
  const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x)
    w[i] = static_cast<uint32_t>(lo + static_cast<int64_t>(hash3(seed, 3, ebase + i) % span));
}

constexpr int kGenGrid = 148 * 16;

// Frees a half-built handle on every early return (ZC_CUDA_TRY included).
struct GraphGuard {
  zc_graph* g;
  ~GraphGuard() {
    if (g) free_graph(g);
  }
  zc_graph* release() {
    zc_graph* r = g;
    g = nullptr;
    return r;
  }
};

// Device temporaries of one generator call: freed on every exit path (error
// returns included) unless handed over to the handle.
struct Temps {
  std::vector<void*> ps;
  template <typename T>
  void add(T* p) {
    ps.push_back(p);
  }
  void forget(const void* p) {
    for (auto& q : ps)
      if (q == p) q = nullptr;
  }
  void release(const void* p) {
    for (auto& q : ps)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~Temps() {
    for (void* p : ps) cudaFree(p);
  }
};

// deg (u32, device) -> offsets into g->h_off (pinned) and g's device offsets.
int offsets_from_degrees(zc_graph* g, uint32_t* d_deg, uint64_t nv, uint64_t** d_off_out) {
  Temps t;
  uint64_t* d_off = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&d_off, (nv + 1) * sizeof(uint64_t)));
  t.add(d_off);
  const size_t tb = scan_tmp_bytes(nv);
  void* tmp = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&tmp, tb));
  t.add(tmp);
  ZC_CUDA_TRY(scan_u32_to_u64(d_deg, d_off, nv, tmp, tb, 0));
  if (!g->h_off) {
    g->h_off = static_cast<int64_t*>(pinned_list_alloc(g->device, (nv + 1) * sizeof(int64_t)));
    if (!g->h_off) {
      set_error("cannot allocate pinned offsets");
      return ZC_ENOMEM;
    }
  }
  ZC_CUDA_TRY(cudaMemcpy(g->h_off, d_off, (nv + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  t.forget(d_off);  // handed to the caller
  *d_off_out = d_off;
  return ZC_OK;
}

// Any list not ascending?  A warp per list, lanes compare neighbours.
template <typename ET>
__global__ void k_lists_unsorted(uint64_t nv, const uint64_t* off, const ET* edges,
                                 unsigned* bad) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; v < nv; v += warps) {
    const uint64_t s = off[v], e = off[v + 1];
    bool b = false;
    for (uint64_t i = s + 1 + lane; i < e && !b; i += 32) b = edges[i - 1] > edges[i];
    if (__any_sync(0xffffffffu, b)) {
      if (lane == 0) atomicOr(bad, 1u);
      return;
    }
  }
}

// Offsets of a batch of lists relative to its first element (CUB takes int).
__global__ void k_rel_offsets(uint64_t n, const uint64_t* off, uint64_t base, int* rel) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x)
    rel[i] = static_cast<int>(off[i] - base);
}

// Sort every list ascending: CUB's segmented sort (segments partitioned by
// size into sub-warp / warp / CTA sorts) over batches of consecutive lists
// holding at most 2^30 keys (CUB takes int sizes), out of place into a batch
// buffer, copied back; lists already ascending are left as they are.
// t_sort_gpu_ms: the GPU time of this thread's last call's sorts and copies
// (CUDA events; the rest of its wall time is allocation and batching).
thread_local float t_sort_gpu_ms = 0;

template <typename ET>
int sort_lists(uint64_t nv, const uint64_t* d_off, ET* edges, bool radix = true) {
  t_sort_gpu_ms = 0;
  if (nv == 0) return ZC_OK;
  {  // already ascending (graphs built by a lexsort, symmetrized ones): done
    unsigned* bad = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&bad, sizeof(unsigned)));
    unsigned h = 1;
    cudaMemset(bad, 0, sizeof(unsigned));
    k_lists_unsorted<ET><<<kGenGrid, 256>>>(nv, d_off, edges, bad);
    const cudaError_t e = cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(bad);
    ZC_CUDA_TRY(e);
    if (!h) return ZC_OK;
  }
  if constexpr (std::is_same<ET, uint32_t>::value) {  // radix transposes when they fit
    uint64_t ne = 0;
    ZC_CUDA_TRY(cudaMemcpy(&ne, d_off + nv, sizeof(ne), cudaMemcpyDeviceToHost));
    if (radix && ne > 0) {
      uint32_t* mx = nullptr;
      void* tmp = nullptr;
      size_t tb = 0;
      uint32_t hmx = 0;
      ZC_CUDA_TRY(cub::DeviceReduce::Max(nullptr, tb, edges, mx, ne));
      ZC_CUDA_TRY(cudaMalloc(&mx, 256 + tb));
      tmp = reinterpret_cast<char*>(mx) + 256;
      cudaError_t e = cub::DeviceReduce::Max(tmp, tb, edges, mx, ne);
      if (e == cudaSuccess) e = cudaMemcpy(&hmx, mx, sizeof(hmx), cudaMemcpyDeviceToHost);
      cudaFree(mx);
      ZC_CUDA_TRY(e);
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, 0);
      const int rc = sort_lists_radix(nv, d_off, edges, ne, static_cast<uint64_t>(hmx) + 1);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (rc != ZC_ENOMEM) {
        t_sort_gpu_ms = ms;
        return rc;
      }
    }
  }
  std::vector<uint64_t> cut{0};
  auto off_at = [&](uint64_t v, uint64_t* x) {
    return cudaMemcpy(x, d_off + v, sizeof(*x), cudaMemcpyDeviceToHost);
  };
  const uint64_t kSpan = 1ull << 30;
  uint64_t ne = 0;
  ZC_CUDA_TRY(off_at(nv, &ne));
  while (cut.back() < nv) {  // largest v1 with off[v1] - off[v0] <= kSpan (at least v0 + 1)
    const uint64_t v0 = cut.back();
    uint64_t b0 = 0;
    ZC_CUDA_TRY(off_at(v0, &b0));
    uint64_t lo = v0 + 1, hi = nv;
    if (ne - b0 <= kSpan) {
      lo = nv;
    } else {
      while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) / 2;
        uint64_t x = 0;
        ZC_CUDA_TRY(off_at(mid, &x));
        if (x - b0 <= kSpan) lo = mid; else hi = mid - 1;
      }
    }
    uint64_t b1 = 0;
    ZC_CUDA_TRY(off_at(lo, &b1));
    if (b1 - b0 > kSpan) {
      set_error("a list longer than 2^30 elements cannot be sorted");
      return ZC_EINVAL;
    }
    cut.push_back(lo);
  }
  uint64_t maxv = 0, maxe = 0;
  for (size_t k = 0; k + 1 < cut.size(); ++k) maxv = std::max(maxv, cut[k + 1] - cut[k]);
  maxe = std::min<uint64_t>(ne, kSpan);
  int* rel = nullptr;
  ET* out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  ZC_CUDA_TRY(cudaMalloc(&rel, (maxv + 1) * sizeof(int)));
  if (cudaMalloc(&out, std::max<uint64_t>(maxe, 1) * sizeof(ET)) != cudaSuccess) {
    cudaFree(rel);
    set_error("out of device memory (list sort)");
    return ZC_ENOMEM;
  }
  int rc = ZC_OK;
  for (size_t k = 0; k + 1 < cut.size() && rc == ZC_OK; ++k) {
    const uint64_t v0 = cut[k], n = cut[k + 1] - v0;
    uint64_t base = 0, span = 0;
    if (off_at(v0, &base) != cudaSuccess || off_at(v0 + n, &span) != cudaSuccess) {
      rc = ZC_ECUDA;
      break;
    }
    span -= base;
    if (span == 0) continue;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    k_rel_offsets<<<kGenGrid, 256>>>(n, d_off + v0, base, rel);
    size_t need = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, need, edges + base, out, static_cast<int>(span),
                                       static_cast<int>(n), rel, rel + 1);
    if (need > tmp_bytes) {
      cudaFree(tmp);
      tmp = nullptr;
      tmp_bytes = need;
      if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) {
        rc = ZC_ENOMEM;
        set_error("out of device memory (list sort)");
        break;
      }
    }
    if (cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, edges + base, out,
                                           static_cast<int>(span), static_cast<int>(n), rel,
                                           rel + 1) != cudaSuccess ||
        cudaMemcpyAsync(edges + base, out, span * sizeof(ET), cudaMemcpyDeviceToDevice, 0) !=
            cudaSuccess) {
      rc = ZC_ECUDA;
      set_error(std::string("list sort: ") + cudaGetErrorString(cudaGetLastError()));
    }
    cudaEventRecord(e1, 0);
    float ms = 0;
    if (cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess)
      t_sort_gpu_ms += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  cudaFree(rel);
  cudaFree(out);
  cudaFree(tmp);
  return rc;
}

zc_graph* new_handle(int32_t placement, int32_t device, uint32_t flags) {
  zc_graph* g = new zc_graph();
  g->placement = placement;
  g->device = device;
  g->flags = flags;
  g->eb = 4;
  g->wb = 4;
  return g;
}

int attach_weights_range(zc_graph* g, uint64_t seed, int64_t wlow, int64_t whigh,
                         uint64_t ebase) {
  if (wlow > whigh) return ZC_OK;
  Temps t;
  uint32_t* d_w = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&d_w, std::max<uint64_t>(g->ne, 32) * sizeof(uint32_t)));
  t.add(d_w);
  if (g->ne) k_weights<<<kGenGrid, 256>>>(g->ne, seed, wlow, whigh, d_w, ebase);
  ZC_CUDA_TRY(cudaGetLastError());
  t.forget(d_w);  // adopt_device_list frees or keeps it
  g->has_weights = true;
  return adopt_device_list(g, d_w, 4, g->ne, &g->h_weights, &g->d_weights, &g->hbm_weights);
}

int attach_weights(zc_graph* g, uint64_t seed, int64_t wlow, int64_t whigh) {
  return attach_weights_range(g, seed, wlow, whigh, 0);
}

int check_common(int32_t placement, int32_t device, int64_t wlow, int64_t whigh) {
  int ndev = 0;
  ZC_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device not present");
    return ZC_EINVAL;
  }
  if (!placement_valid(placement)) {
    set_error("unknown placement");
    return ZC_EINVAL;
  }
  if (wlow <= whigh && (wlow < 0 || whigh > 0xffffffffll)) {
    set_error("weights must lie in [0, 2^32)");
    return ZC_EINVAL;
  }
  return ZC_OK;
}

RmatParams rmat_params(uint32_t scale, double a, double b, double c, uint64_t seed) {
  const double d = 1.0 - a - b - c;
  RmatParams p;
  p.scale = scale;
  p.thr_src = static_cast<uint32_t>((c + d) * 65536.0 + 0.5);
  p.thr_dst0 = static_cast<uint32_t>(b / (a + b) * 65536.0 + 0.5);
  p.thr_dst1 = (c + d) > 0 ? static_cast<uint32_t>(d / (c + d) * 65536.0 + 0.5) : 0;
  p.seed = seed;
  p.perm.bits = scale;
  p.perm.half = (scale + 1) / 2;
  p.perm.key = mix64(seed ^ 0x5eedull);
  return p;
}

// One edge-balanced vertex range of the directed R-MAT graph generate_rmat
// would build with the same parameters (the same arcs, lists and order).
// symmetrize: the part of the symmetrized graph (out-arcs + reverse arcs,
// csr.py:350-359 semantics, lists sorted) -- every rank enumerates all arcs
// for the global symmetric degrees (edge-balanced cuts) and for the reverse
// arcs into its range; no edge exchange between ranks.
int generate_rmat_part(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                       int symmetrize, int64_t wlow, int64_t whigh, uint32_t nparts,
                       uint32_t part, int32_t placement, int32_t device, uint64_t* bounds,
                       zc_graph** out) {
  *out = nullptr;
  int rc = check_common(placement, device, wlow, whigh);
  if (rc) return rc;
  if (scale < 1 || scale > 31 || ef < 1 || a <= 0 || b < 0 || c < 0 || 1.0 - a - b - c < 0 ||
      nparts < 1 || part >= nparts || !bounds || (symmetrize && wlow <= whigh)) {
    set_error("invalid rmat partition parameters");
    return ZC_EINVAL;
  }
  cudaSetDevice(device);
  const uint64_t nv = 1ull << scale;
  const uint64_t narcs = static_cast<uint64_t>(ef) << scale;
  const RmatParams p = rmat_params(scale, a, b, c, seed);
  Temps t;
  // global degrees -> global offsets (identical on every rank)
  uint32_t* d_deg = nullptr;
  uint64_t* d_goff = nullptr;
  if (cudaMalloc(&d_deg, nv * sizeof(uint32_t)) != cudaSuccess) {
    set_error("out of device memory");
    return ZC_ENOMEM;
  }
  t.add(d_deg);
  cudaMemset(d_deg, 0, nv * sizeof(uint32_t));
  k_rmat_count<<<kGenGrid, 256>>>(p, narcs, d_deg);
  ZC_CUDA_TRY(cudaMalloc(&d_goff, (nv + 1) * sizeof(uint64_t)));
  t.add(d_goff);
  {
    const size_t tb = scan_tmp_bytes(nv);
    void* tmp = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&tmp, tb));
    t.add(tmp);
    ZC_CUDA_TRY(scan_u32_to_u64(d_deg, d_goff, nv, tmp, tb, 0));
    ZC_CUDA_TRY(cudaDeviceSynchronize());
    t.release(tmp);
  }
  // symmetric: degrees = out + in (every arc enumerated once more), offsets d_soff
  uint64_t* d_soff = nullptr;
  if (symmetrize) {
    uint32_t* d_ideg = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&d_ideg, nv * sizeof(uint32_t)));
    t.add(d_ideg);
    ZC_CUDA_TRY(cudaMemset(d_ideg, 0, nv * sizeof(uint32_t)));
    k_rmat_in_arcs<false><<<kGenGrid, 256>>>(p, nv, d_goff, 0, nv, d_ideg, nullptr, nullptr);
    k_add_u32<<<kGenGrid, 256>>>(nv, d_deg, d_ideg);
    ZC_CUDA_TRY(cudaGetLastError());
    t.release(d_ideg);
    ZC_CUDA_TRY(cudaMalloc(&d_soff, (nv + 1) * sizeof(uint64_t)));
    t.add(d_soff);
    const size_t tb = scan_tmp_bytes(nv);
    void* tmp = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&tmp, tb));
    t.add(tmp);
    ZC_CUDA_TRY(scan_u32_to_u64(d_deg, d_soff, nv, tmp, tb, 0));
    ZC_CUDA_TRY(cudaDeviceSynchronize());
    t.release(tmp);
  }
  t.release(d_deg);
  const uint64_t* d_coff = symmetrize ? d_soff : d_goff;  // the partitioned graph's offsets
  const uint64_t ctotal = symmetrize ? 2 * narcs : narcs;
  // edge-balanced bounds: first vertex whose offset reaches E*k/nparts
  std::vector<uint64_t> cut(nparts + 1);
  cut[0] = 0;
  cut[nparts] = nv;
  for (uint32_t k = 1; k < nparts; ++k) {
    const uint64_t target = static_cast<uint64_t>(static_cast<double>(ctotal) * k / nparts);
    uint64_t lo = 0, hi = nv;  // smallest v with coff[v] >= target
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      uint64_t val = 0;
      ZC_CUDA_TRY(cudaMemcpy(&val, d_coff + mid, sizeof(val), cudaMemcpyDeviceToHost));
      if (val >= target) hi = mid; else lo = mid + 1;
    }
    cut[k] = std::max(lo, cut[k - 1]);
  }
  for (uint32_t k = 0; k <= nparts; ++k) bounds[k] = cut[k];
  const uint64_t lo = cut[part], hi = cut[part + 1], nl = hi - lo;
  uint64_t e0 = 0, e1 = 0;
  ZC_CUDA_TRY(cudaMemcpy(&e0, d_coff + lo, sizeof(e0), cudaMemcpyDeviceToHost));
  ZC_CUDA_TRY(cudaMemcpy(&e1, d_coff + hi, sizeof(e1), cudaMemcpyDeviceToHost));

  zc_graph* g = new_handle(placement, device, symmetrize ? 0u : ZC_F_DIRECTED);
  GraphGuard guard{g};
  auto fail = [](int code) { return code; };
  g->nv = nl;
  g->ne = e1 - e0;
  g->h_off = static_cast<int64_t*>(pinned_list_alloc(g->device, (nl + 1) * sizeof(int64_t)));
  if (!g->h_off) {
    set_error("cannot allocate pinned offsets");
    return fail(ZC_ENOMEM);
  }
  ZC_CUDA_TRY(cudaMemcpy(g->h_off, d_coff + lo, (nl + 1) * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost));
  for (uint64_t v = 0; v <= nl; ++v) g->h_off[v] -= static_cast<int64_t>(e0);
  uint64_t* d_loff = nullptr;
  uint32_t* d_edges = nullptr;
  if (cudaMalloc(&d_loff, (nl + 1) * sizeof(uint64_t)) != cudaSuccess) {
    set_error("out of device memory");
    return fail(ZC_ENOMEM);
  }
  t.add(d_loff);
  if (cudaMalloc(&d_edges, std::max<uint64_t>(g->ne, 32) * sizeof(uint32_t)) != cudaSuccess) {
    set_error("out of device memory");
    return fail(ZC_ENOMEM);
  }
  t.add(d_edges);
  ZC_CUDA_TRY(cudaMemcpy(d_loff, g->h_off, (nl + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice));
  if (symmetrize) {
    // list x = its out-arcs (generator order), then the sources of its in-arcs
    // (cursor from the out-degree), then sorted like generate_rmat's
    uint32_t* d_cursor = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&d_cursor, std::max<uint64_t>(nl, 1) * sizeof(uint32_t)));
    t.add(d_cursor);
    k_rmat_fill<uint32_t><<<kGenGrid, 256>>>(p, nl, d_goff + lo, d_edges, lo, d_loff);
    k_deg_from_off<<<kGenGrid, 256>>>(nl, d_goff + lo, d_cursor);
    k_rmat_in_arcs<true><<<kGenGrid, 256>>>(p, nv, d_goff, lo, nl, d_cursor, d_loff, d_edges);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      set_error(std::string("rmat symmetric part: ") + cudaGetErrorString(cudaGetLastError()));
      return fail(ZC_ECUDA);
    }
    t.release(d_cursor);
    t.release(d_soff);
    t.release(d_goff);
    if ((rc = sort_lists<uint32_t>(nl, d_loff, d_edges))) return fail(rc);
  } else {
    t.release(d_goff);
    k_rmat_fill<uint32_t><<<kGenGrid, 256>>>(p, nl, d_loff, d_edges, lo);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(std::string("rmat fill: ") + cudaGetErrorString(cudaGetLastError()));
    return fail(ZC_ECUDA);
  }
  t.release(d_loff);
  t.forget(d_edges);  // adopt_device_list frees or keeps it
  if ((rc = adopt_device_list(g, d_edges, 4, g->ne, &g->h_edges, &g->d_edges, &g->hbm_edges)))
    return fail(rc);
  if ((rc = attach_weights_range(g, seed ^ 0x77ull, wlow, whigh, e0))) return fail(rc);
  if ((rc = alloc_state(g))) return fail(rc);
  zc_part_info info;
  info.global_vertices = nv;
  info.bounds = bounds;
  info.nparts = nparts;
  info.part = part;
  uint64_t stride = 1;
  for (uint32_t k = 0; k < nparts; ++k) stride = std::max(stride, cut[k + 1] - cut[k]);
  info.stride = stride;
  if ((rc = init_partition(g, &info))) return fail(rc);
  if ((rc = finish_create(g))) return fail(rc);
  g->gen_rmat = true;
  g->gen_scale = scale;
  g->gen_ef = ef;
  g->gen_a = a;
  g->gen_b = b;
  g->gen_c = c;
  g->gen_seed = seed;
  *out = guard.release();
  return ZC_OK;
}

// In-lists of a generated R-MAT partition: every rank enumerates all arcs
// (the generator is counter-based) and keeps those whose destination it
// owns -- no edge exchange between ranks.
int rmat_part_in_lists(zc_graph* g) {
  const RmatParams p = rmat_params(g->gen_scale, g->gen_a, g->gen_b, g->gen_c, g->gen_seed);
  const uint64_t nv = 1ull << g->gen_scale;
  const uint64_t narcs = static_cast<uint64_t>(g->gen_ef) << g->gen_scale;
  const uint64_t lo = g->lo, nl = g->nv;
  Temps t;
  uint32_t* d_deg = nullptr;
  uint64_t* d_goff = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&d_deg, nv * sizeof(uint32_t)));
  t.add(d_deg);
  ZC_CUDA_TRY(cudaMemset(d_deg, 0, nv * sizeof(uint32_t)));
  k_rmat_count<<<kGenGrid, 256>>>(p, narcs, d_deg);
  ZC_CUDA_TRY(cudaMalloc(&d_goff, (nv + 1) * sizeof(uint64_t)));
  t.add(d_goff);
  const size_t tb = scan_tmp_bytes(std::max(nv, nl));
  void* tmp = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&tmp, tb));
  t.add(tmp);
  ZC_CUDA_TRY(scan_u32_to_u64(d_deg, d_goff, nv, tmp, tb, 0));
  uint32_t* d_ideg = d_deg;  // reuse: local in-degrees, then cursors
  ZC_CUDA_TRY(cudaMemset(d_ideg, 0, std::max<uint64_t>(nl, 1) * sizeof(uint32_t)));
  k_rmat_in_arcs<false><<<kGenGrid, 256>>>(p, nv, d_goff, lo, nl, d_ideg, nullptr, nullptr);
  uint64_t* d_in_off = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&d_in_off, (nl + 1) * sizeof(uint64_t)));
  t.add(d_in_off);
  ZC_CUDA_TRY(scan_u32_to_u64(d_ideg, d_in_off, nl, tmp, tb, 0));
  uint64_t ne_in = 0;
  ZC_CUDA_TRY(cudaMemcpy(&ne_in, d_in_off + nl, sizeof(ne_in), cudaMemcpyDeviceToHost));
  uint32_t* d_in = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&d_in, std::max<uint64_t>(ne_in, 32) * sizeof(uint32_t)));
  t.add(d_in);
  ZC_CUDA_TRY(cudaMemset(d_ideg, 0, std::max<uint64_t>(nl, 1) * sizeof(uint32_t)));
  k_rmat_in_arcs<true><<<kGenGrid, 256>>>(p, nv, d_goff, lo, nl, d_ideg, d_in_off, d_in);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(std::string("rmat in-lists: ") + cudaGetErrorString(cudaGetLastError()));
    return ZC_ECUDA;
  }
  t.release(d_goff);
  t.release(d_deg);
  int rc = sort_lists<uint32_t>(nl, d_in_off, d_in);
  if (rc) return rc;
  ZC_CUDA_TRY(cudaDeviceSynchronize());
  if ((rc = install_in_lists(g, d_in_off, d_in))) return rc;
  t.forget(d_in_off);  // the handle owns it
  return ZC_OK;
}

int generate_rmat(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                  int symmetrize, int64_t wlow, int64_t whigh, int32_t placement, int32_t device,
                  zc_graph** out) {
  *out = nullptr;
  int rc = check_common(placement, device, wlow, whigh);
  if (rc) return rc;
  const double d = 1.0 - a - b - c;
  if (scale < 1 || scale > 31 || ef < 1 || a <= 0 || b < 0 || c < 0 || d < 0) {
    set_error("rmat needs 1 <= scale <= 31, edge_factor >= 1, a > 0, b, c, 1-a-b-c >= 0");
    return ZC_EINVAL;
  }
  cudaSetDevice(device);
  const uint64_t nv = 1ull << scale;
  const uint64_t narcs = static_cast<uint64_t>(ef) << scale;
  if (symmetrize && 2 * narcs / nv > 0xffffffffull) {
    set_error("degree overflow");
    return ZC_EINVAL;
  }
  const RmatParams p = rmat_params(scale, a, b, c, seed);

  zc_graph* g = new_handle(placement, device, symmetrize ? 0u : ZC_F_DIRECTED);
  GraphGuard guard{g};
  Temps t;
  auto fail = [](int code) {
    if (code == ZC_ENOMEM) set_error("out of device memory");
    return code;
  };
  g->nv = nv;
  uint32_t* d_deg = nullptr;
  uint64_t* d_off = nullptr;
  uint32_t* d_edges = nullptr;
  if (cudaMalloc(&d_deg, nv * sizeof(uint32_t)) != cudaSuccess) return fail(ZC_ENOMEM);
  t.add(d_deg);
  cudaMemset(d_deg, 0, nv * sizeof(uint32_t));
  k_rmat_count<<<kGenGrid, 256>>>(p, narcs, d_deg);
  if ((rc = offsets_from_degrees(g, d_deg, nv, &d_off))) return fail(rc);
  t.add(d_off);
  if (cudaMalloc(&d_edges, std::max<uint64_t>(narcs, 32) * sizeof(uint32_t)) != cudaSuccess)
    return fail(ZC_ENOMEM);
  t.add(d_edges);
  k_rmat_fill<uint32_t><<<kGenGrid, 256>>>(p, nv, d_off, d_edges);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(std::string("rmat fill: ") + cudaGetErrorString(cudaGetLastError()));
    return fail(ZC_ECUDA);
  }
  g->ne = narcs;
  if (symmetrize) {
    // symmetric degree = out-degree + in-degree; cursor[x] starts at out-degree
    uint32_t* d_cursor = nullptr;
    uint32_t* d_sedges = nullptr;
    uint64_t* d_soff = nullptr;
    if (cudaMalloc(&d_cursor, nv * sizeof(uint32_t)) != cudaSuccess) return fail(ZC_ENOMEM);
    t.add(d_cursor);
    k_deg_from_off<<<kGenGrid, 256>>>(nv, d_off, d_deg);
    k_count_in<uint32_t><<<kGenGrid, 256>>>(narcs, d_edges, d_deg);
    if ((rc = offsets_from_degrees(g, d_deg, nv, &d_soff))) return fail(rc);
    t.add(d_soff);
    k_deg_from_off<<<kGenGrid, 256>>>(nv, d_off, d_cursor);
    if (cudaMalloc(&d_sedges, std::max<uint64_t>(2 * narcs, 32) * sizeof(uint32_t)) !=
        cudaSuccess)
      return fail(ZC_ENOMEM);
    t.add(d_sedges);
    k_sym_copy_out<uint32_t><<<kGenGrid, 256>>>(nv, d_off, d_edges, d_soff, d_sedges);
    k_sym_scatter_in<uint32_t><<<kGenGrid, 256>>>(nv, d_off, d_edges, d_soff, d_cursor, d_sedges);
    if ((rc = sort_lists<uint32_t>(nv, d_soff, d_sedges))) return fail(rc);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      set_error(std::string("symmetrize: ") + cudaGetErrorString(cudaGetLastError()));
      return fail(ZC_ECUDA);
    }
    t.release(d_cursor);
    t.release(d_edges);
    t.release(d_off);
    d_edges = d_sedges;
    d_off = d_soff;
    g->ne = 2 * narcs;
  }
  t.release(d_deg);
  g->eb = 4;
  t.forget(d_edges);  // adopt_device_list frees or keeps it
  if ((rc = adopt_device_list(g, d_edges, 4, g->ne, &g->h_edges, &g->d_edges, &g->hbm_edges)))
    return fail(rc);
  t.release(d_off);
  if ((rc = attach_weights(g, seed ^ 0x77ull, wlow, whigh))) return fail(rc);
  if ((rc = alloc_state(g))) return fail(rc);
  if ((rc = finish_create(g))) return fail(rc);
  *out = guard.release();
  return ZC_OK;
}

int generate_uniform(uint64_t nv, uint32_t dmin, uint32_t dmax, uint64_t seed, int64_t wlow,
                     int64_t whigh, int32_t placement, int32_t device, zc_graph** out) {
  *out = nullptr;
  int rc = check_common(placement, device, wlow, whigh);
  if (rc) return rc;
  // csr.py:273-274 precondition, plus the native generator's list cap
  if (!(dmin <= dmax && dmax < nv) || nv >= 0xffffffffull || dmax > 256) {
    set_error("require 0 <= min_degree <= max_degree < num_vertices, max_degree <= 256");
    return ZC_EINVAL;
  }
  cudaSetDevice(device);
  zc_graph* g = new_handle(placement, device, ZC_F_DIRECTED);
  GraphGuard guard{g};
  Temps t;
  auto fail = [](int code) {
    if (code == ZC_ENOMEM) set_error("out of device memory");
    return code;
  };
  g->nv = nv;
  uint32_t* d_deg = nullptr;
  uint64_t* d_off = nullptr;
  uint32_t* d_edges = nullptr;
  if (cudaMalloc(&d_deg, std::max<uint64_t>(nv, 1) * sizeof(uint32_t)) != cudaSuccess)
    return fail(ZC_ENOMEM);
  t.add(d_deg);
  k_uniform_deg<<<kGenGrid, 256>>>(nv, seed, dmin, dmax, d_deg);
  if ((rc = offsets_from_degrees(g, d_deg, nv, &d_off))) return fail(rc);
  t.add(d_off);
  g->ne = static_cast<uint64_t>(g->h_off[nv]);
  if (cudaMalloc(&d_edges, std::max<uint64_t>(g->ne, 32) * sizeof(uint32_t)) != cudaSuccess)
    return fail(ZC_ENOMEM);
  t.add(d_edges);
  k_uniform_fill<uint32_t><<<kGenGrid, 128>>>(nv, seed, d_off, d_edges);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(std::string("uniform fill: ") + cudaGetErrorString(cudaGetLastError()));
    return fail(ZC_ECUDA);
  }
  t.release(d_deg);
  t.release(d_off);
  t.forget(d_edges);  // adopt_device_list frees or keeps it
  if ((rc = adopt_device_list(g, d_edges, 4, g->ne, &g->h_edges, &g->d_edges, &g->hbm_edges)))
    return fail(rc);
  if ((rc = attach_weights(g, seed ^ 0x77ull, wlow, whigh))) return fail(rc);
  if ((rc = alloc_state(g))) return fail(rc);
  if ((rc = finish_create(g))) return fail(rc);
  *out = guard.release();
  return ZC_OK;
}

}  // namespace

int part_in_lists(zc_graph* g) { return rmat_part_in_lists(g); }

float last_sort_gpu_ms() { return t_sort_gpu_ms; }
void set_sort_gpu_ms(float ms) { t_sort_gpu_ms = ms; }

cudaError_t lists_ascending(uint64_t nv, const uint64_t* d_off, const uint32_t* edges, bool* yes) {
  *yes = true;
  if (nv == 0) return cudaSuccess;
  unsigned* bad = nullptr;
  cudaError_t e = cudaMalloc(&bad, sizeof(unsigned));
  if (e != cudaSuccess) return e;
  unsigned h = 1;
  cudaMemset(bad, 0, sizeof(unsigned));
  k_lists_unsorted<uint32_t><<<kGenGrid, 256>>>(nv, d_off, edges, bad);
  e = cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  *yes = h == 0;
  return e;
}

int sort_lists_device(int elem_bytes, uint64_t nv, const uint64_t* d_off, void* edges,
                      bool radix) {
  int rc = elem_bytes == 4 ? sort_lists<uint32_t>(nv, d_off, static_cast<uint32_t*>(edges), radix)
                           : sort_lists<uint64_t>(nv, d_off, static_cast<uint64_t*>(edges));
  if (rc) return rc;
  ZC_CUDA_TRY(cudaDeviceSynchronize());
  return ZC_OK;
}

}  // namespace zc

extern "C" int zc_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b,
                                double c, uint64_t seed, int symmetrize, int64_t wlow,
                                int64_t whigh, int32_t placement, int32_t device,
                                zc_graph** out) {
  if (!out) return ZC_ESTATE;
  return zc::generate_rmat(scale, edge_factor, a, b, c, seed, symmetrize, wlow, whigh, placement,
                           device, out);
}

extern "C" int zc_generate_uniform(uint64_t num_vertices, uint32_t min_degree, uint32_t max_degree,
                                   uint64_t seed, int64_t wlow, int64_t whigh, int32_t placement,
                                   int32_t device, zc_graph** out) {
  if (!out) return ZC_ESTATE;
  return zc::generate_uniform(num_vertices, min_degree, max_degree, seed, wlow, whigh, placement,
                              device, out);
}

extern "C" int zc_generate_rmat_part(uint32_t scale, uint32_t edge_factor, double a, double b,
                                     double c, uint64_t seed, int symmetrize, int64_t wlow,
                                     int64_t whigh, uint32_t nparts, uint32_t part,
                                     int32_t placement, int32_t device, uint64_t* bounds,
                                     zc_graph** out) {
  if (!out) return ZC_ESTATE;
  return zc::generate_rmat_part(scale, edge_factor, a, b, c, seed, symmetrize, wlow, whigh, nparts,
                                part, placement, device, bounds, out);
}

extern "C" int zc_part_build_in_lists(zc_graph* g, uint64_t* compressed_bytes) {
  if (!g || !g->nparts) {
    zc::set_error("not a partition handle");
    return ZC_ESTATE;
  }
  if (g->d_cpos_in) {
    if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
    return ZC_OK;
  }
  if (!(g->flags & ZC_F_DIRECTED)) return zc_graph_build_in_lists(g, compressed_bytes);
  if (!g->gen_rmat) {
    zc::set_error("in-lists of a directed partition need its generator (zc_generate_rmat_part)");
    return ZC_EINVAL;
  }
  int rc = zc_graph_build_compressed(g, nullptr);
  if (rc) return rc;
  cudaSetDevice(g->device);
  if ((rc = zc::part_in_lists(g))) return rc;
  if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
  return ZC_OK;
}
