// Compressed line stream: an optional B200-native host-store format.
//
// Zero-copy traversal is bound by the host link: ~437 M fully-used 128-byte
// line reads/s (55.9 GB/s of PCIe read bytes, profiles/ncu_summary.json), and
// about as much by the request count as by the bytes.  BFS / CC / PageRank /
// SSSP results do not depend on the order inside a list, so every list is
// sorted and stored delta-encoded in 128-byte lines (format in
// zc_internal.cuh): a hub list as whole self-describing lines (~50-100 edges
// per aligned line read instead of 32), short lists packed into shared
// 256-byte spans (one read serves every frontier list in it).  SSSP weights ride in the
// same lines as (weight - wmin) fields of the narrowest width that holds them.
//
// Build, on the GPU: sort each list (by destination, then weight), size every
// list (short: its bit length; long: the lines of a greedy fill -- as many
// deltas as fit 1024 - 48 bits at the width of the widest one, at most 255),
// place them in vertex order (first fit inside blocks of kPlaceBlock vertices,
// a thread per block: a short list moves to the next 256-byte span only when
// it does not fit the current one, a long list starts a line; every block
// starts a span, placed by a scan of the block sizes), then encode.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <future>
#include <string>
#include <vector>

#include "zc_graph.cuh"
#include "zc_internal.cuh"

namespace zc {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr uint32_t kLongSize = 1u << 31;  // size word: long list, low bits = lines

__device__ __forceinline__ uint32_t bits_of(uint32_t x) { return x ? 32 - __clz(x) : 0; }

// Sorted list element k: destination (and weight - wmin) of a u32 list or of a
// u64 (dst << 32 | weight) pair list.
struct Elems {
  const uint32_t* e32;
  const uint64_t* e64;
  uint32_t wmin;
  __device__ __forceinline__ uint32_t dst(uint64_t i) const {
    return e64 ? static_cast<uint32_t>(e64[i] >> 32) : e32[i];
  }
  __device__ __forceinline__ uint32_t wt(uint64_t i) const {
    return e64 ? static_cast<uint32_t>(e64[i]) - wmin : 0u;
  }
};

// Greedy fill of one long-list line starting at element p of the list [0, d):
// the largest K <= min(255, d-1-p) with 48 + K * max(bits(delta 1..K)) +
// (K + 1) * ww <= 1024.  Warp-cooperative, in one pass: lane l loads elements
// 8l .. 8l+8 of the line's window (all 256 candidate deltas in flight at once;
// a 32-delta chunk loop serialised ~5 load round trips per line, which set
// the build's tail on hub lists), a warp prefix-max gives every delta's
// running width, and the fitting deltas are a prefix (the cost grows with k).
// Returns count = K + 1 and width = max bits(delta 1..K).
__device__ __forceinline__ void line_fill(const Elems& x, uint64_t s, uint64_t d, uint64_t p,
                                          uint32_t ww, int lane, uint32_t* count,
                                          uint32_t* width) {
  const uint64_t rest = d - 1 - p;
  const uint32_t kmax = static_cast<uint32_t>(rest < kCmpMaxCount - 1 ? rest : kCmpMaxCount - 1);
  const uint32_t k0 = static_cast<uint32_t>(lane) * 8;  // this lane's deltas k0+1 .. k0+8
  uint32_t e[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) e[j] = k0 + j <= kmax ? x.dst(s + p + k0 + j) : 0u;
  uint32_t b[8], lm = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    b[j] = k0 + j + 1 <= kmax ? bits_of(e[j + 1] - e[j]) : 0u;
    lm = max(lm, b[j]);
  }
  uint32_t inc = lm;  // inclusive prefix max over lanes, then exclusive
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFullMask, inc, o);
    if (lane >= o) inc = max(inc, t);
  }
  uint32_t pm = __shfl_up_sync(kFullMask, inc, 1);
  if (lane == 0) pm = 0;
  uint32_t n = 0, mlast = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t k = k0 + j + 1;
    pm = max(pm, b[j]);
    if (k <= kmax && kCmpHdrBits + k * pm + (k + 1) * ww <= kLineBits) {
      ++n;
      mlast = pm;
    }
  }
  const uint32_t K = __reduce_add_sync(kFullMask, n);
  const uint32_t m = __shfl_sync(kFullMask, mlast, K ? (K - 1) / 8 : 0);
  *count = K + 1;
  *width = K ? m : 0u;
}

// Width of the widest delta of the whole list (warp-cooperative).
__device__ __forceinline__ uint32_t list_width(const Elems& x, uint64_t s, uint64_t d,
                                               int lane) {
  uint32_t mx = 0;
  for (uint64_t k = 1 + lane; k < d; k += 32) mx = max(mx, x.dst(s + k) - x.dst(s + k - 1));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFullMask, mx, o));
  return bits_of(mx);
}

__host__ __device__ __forceinline__ uint64_t short_bits(uint64_t d, uint32_t w, uint32_t ww,
                                                        uint32_t b0) {
  return kCmpShortWidthBits + b0 + (d - 1) * w + d * ww;
}

// Lists of at most kLaneList elements are sized / encoded by one lane each
// (32 lists per warp in flight: the warp-per-list loop was latency-bound,
// 15-25 % SM throughput, long-scoreboard stalls); longer lists, and the rare
// short-degree list too wide for a span, take the warp-cooperative path.
constexpr uint32_t kLaneList = 32;

// Largest delta of a list of 1 <= d <= kLaneList elements, one lane.
__device__ __forceinline__ uint32_t lane_max_delta(const Elems& x, uint64_t s, uint32_t d) {
  uint32_t prev = x.dst(s), mx = 0;
#pragma unroll 4
  for (uint32_t k = 1; k < d; ++k) {
    const uint32_t c = x.dst(s + k);
    mx = max(mx, c - prev);
    prev = c;
  }
  return mx;
}

// Size word of list [s, s + d), warp-cooperative (any d >= 1).
__device__ uint32_t size_list_warp(const Elems& x, uint64_t s, uint64_t d, uint32_t ww,
                                   uint32_t b0, int lane) {
  const uint64_t sb = short_bits(d, list_width(x, s, d, lane), ww, b0);
  if (sb <= kShortSpanBits && d <= kCmpShortMaxDeg)  // one lane decodes a short list
    return static_cast<uint32_t>(sb);
  uint32_t n = 0;
  for (uint64_t p = 0; p < d; ++n) {
    uint32_t cnt, w;
    line_fill(x, s, d, p, ww, lane, &cnt, &w);
    p += cnt;
  }
  return kLongSize | n;
}

// Size word of every list: 0 (empty), its bit length (short), or
// kLongSize | lines (long).  A warp takes 32 consecutive lists at a time.
__global__ void k_cmp_size(uint64_t nv, const uint64_t* off, Elems x, uint32_t ww, uint32_t b0,
                           uint32_t* size) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * 32; base < nv; base += nw * 32) {
    const uint64_t v = base + lane;
    uint64_t s = 0, d = 0;
    if (v < nv) {
      s = off[v];
      d = off[v + 1] - s;
    }
    uint32_t out = 0;
    bool warp_path = d > kLaneList;
    if (d && d <= kLaneList) {
      const uint64_t sb = short_bits(d, bits_of(lane_max_delta(x, s, static_cast<uint32_t>(d))),
                                     ww, b0);
      if (sb <= kShortSpanBits) out = static_cast<uint32_t>(sb);
      else warp_path = true;
    }
    for (unsigned m = __ballot_sync(kFullMask, warp_path); m; m &= m - 1) {
      const int l = __ffs(m) - 1;
      const uint32_t o = size_list_warp(x, __shfl_sync(kFullMask, s, l),
                                        __shfl_sync(kFullMask, d, l), ww, b0, lane);
      if (lane == l) out = o;
    }
    if (v < nv) size[v] = out;
  }
}

// OR `nbits` (<= 32) of `val` into the bit stream at bit position `bit`.
__device__ __forceinline__ void put_bits(uint32_t* out, uint64_t bit, uint32_t val,
                                         uint32_t nbits) {
  if (!nbits) return;
  if (nbits < 32) val &= (1u << nbits) - 1;
  const uint32_t sh = static_cast<uint32_t>(bit & 31);
  atomicOr(out + (bit >> 5), val << sh);
  if (sh + nbits > 32) atomicOr(out + (bit >> 5) + 1, val >> (32 - sh));
}

// Short list [s, s + d) at bit `pos`, one lane: width, first element, deltas,
// weights.  Lists share words at their ends, hence the OR atomics.
__device__ __forceinline__ void encode_short_lane(const Elems& x, uint64_t s, uint32_t d,
                                                  uint32_t ww, uint32_t b0, uint64_t pos,
                                                  uint32_t* out) {
  const uint32_t w = bits_of(lane_max_delta(x, s, d));
  const uint64_t hdr = pos + kCmpShortWidthBits + b0, wbase = hdr + (d - 1) * w;
  uint32_t prev = x.dst(s);
  put_bits(out, pos, w, kCmpShortWidthBits);
  put_bits(out, pos + kCmpShortWidthBits, prev, b0);
  put_bits(out, wbase, x.wt(s), ww);
#pragma unroll 4
  for (uint32_t k = 1; k < d; ++k) {
    const uint32_t c = x.dst(s + k);
    put_bits(out, hdr + (k - 1) * w, c - prev, w);
    put_bits(out, wbase + k * ww, x.wt(s + k), ww);
    prev = c;
  }
}

// List [s, s + d) with index word c, warp-cooperative (any d >= 1).  Short
// lists OR their fields into shared lines; long lists build each line in a
// shared-memory buffer (L, this warp's) and store it whole.
__device__ void encode_list_warp(const Elems& x, uint64_t s, uint64_t d, uint64_t c, uint32_t ww,
                                 uint32_t b0, uint32_t* out, uint32_t* L, int lane) {
  const uint64_t pos = cmp_pos(c);
  if (!(c & kCmpLong)) {
    const uint32_t w = list_width(x, s, d, lane);
    const uint64_t hdr = kCmpShortWidthBits + b0;
    if (lane == 0) {
      put_bits(out, pos, w, kCmpShortWidthBits);
      put_bits(out, pos + kCmpShortWidthBits, x.dst(s), b0);
    }
    const uint64_t wbase = pos + hdr + (d - 1) * w;
    for (uint64_t k = lane; k < d; k += 32) {
      if (k) put_bits(out, pos + hdr + (k - 1) * w, x.dst(s + k) - x.dst(s + k - 1), w);
      put_bits(out, wbase + k * ww, x.wt(s + k), ww);
    }
    return;
  }
  const uint64_t l0 = pos / kLineBits, nl = cmp_lines(c);
  uint64_t p = 0;
  for (uint64_t t = 0; t < nl; ++t) {
    uint32_t cnt, w;
    line_fill(x, s, d, p, ww, lane, &cnt, &w);
    L[lane] = 0;
    if (lane < 2) L[kLineWords + lane] = 0;
    __syncwarp();
    const uint32_t wb = kCmpHdrBits + (cnt - 1) * w;
    for (uint32_t k = lane; k < cnt; k += 32) {
      if (k && w) {
        const uint32_t dl = x.dst(s + p + k) - x.dst(s + p + k - 1);
        const uint32_t bit = kCmpHdrBits + (k - 1) * w;
        atomicOr(&L[bit >> 5], dl << (bit & 31));
        if ((bit & 31) + w > 32) atomicOr(&L[(bit >> 5) + 1], dl >> (32 - (bit & 31)));
      }
      if (ww) {
        const uint32_t wv = x.wt(s + p + k) & (ww < 32 ? (1u << ww) - 1 : ~0u);
        const uint32_t bit = wb + k * ww;
        atomicOr(&L[bit >> 5], wv << (bit & 31));
        if ((bit & 31) + ww > 32) atomicOr(&L[(bit >> 5) + 1], wv >> (32 - (bit & 31)));
      }
    }
    __syncwarp();
    if (lane == 0) {
      L[0] = x.dst(s + p);
      L[1] |= w | ((cnt - 1) << 6);
    }
    __syncwarp();
    out[(l0 + t) * kLineWords + lane] = L[lane];
    __syncwarp();
    p += cnt;
  }
}

// Encode: a warp takes 32 consecutive lists at a time, the short ones of at
// most kLaneList elements a lane each, the rest one by one together.
__global__ void __launch_bounds__(256) k_cmp_encode(uint64_t nv, const uint64_t* off, Elems x,
                                                    uint32_t ww, uint32_t b0, const uint64_t* cpos,
                                                    uint32_t* out) {
  __shared__ uint32_t buf[8][kLineWords + 2];
  const int lane = threadIdx.x & 31;
  uint32_t* L = buf[threadIdx.x >> 5];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * 32; base < nv; base += nw * 32) {
    const uint64_t v = base + lane;
    uint64_t s = 0, d = 0, c = 0;
    if (v < nv) {
      s = off[v];
      d = off[v + 1] - s;
      if (d) c = cpos[v];
    }
    const bool mine = d && d <= kLaneList && !(c & kCmpLong);
    if (mine) encode_short_lane(x, s, static_cast<uint32_t>(d), ww, b0, cmp_pos(c), out);
    for (unsigned m = __ballot_sync(kFullMask, d && !mine); m; m &= m - 1) {
      const int l = __ffs(m) - 1;
      encode_list_warp(x, __shfl_sync(kFullMask, s, l), __shfl_sync(kFullMask, d, l),
                       __shfl_sync(kFullMask, c, l), ww, b0, out, L, lane);
    }
  }
}

// (dst << 32 | weight) pair list of u32 edges + u32 weights; weight range.
__global__ void k_cmp_pairs(uint64_t ne, const uint32_t* e, const uint32_t* w, uint64_t* out,
                            unsigned* wmin, unsigned* wmax) {
  unsigned lo = 0xffffffffu, hi = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x) {
    out[i] = (static_cast<uint64_t>(e[i]) << 32) | w[i];
    lo = min(lo, w[i]);
    hi = max(hi, w[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFullMask, lo, o));
    hi = max(hi, __shfl_xor_sync(kFullMask, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(wmin, lo);
    atomicMax(wmax, hi);
  }
}

constexpr int kCmpGrid = 148 * 16;

// Placement, block-local first fit: block b (vertices [b B, b B + B)) is laid
// out from relative position 0; block_bits[b] = its length rounded up to a
// span, so every block starts on a span (and line) boundary.
constexpr uint64_t kPlaceBlock = 1024;
__global__ void k_cmp_place_local(uint64_t nv, const uint32_t* size, uint64_t* cpos,
                                  uint64_t* block_bits, unsigned* err) {
  const uint64_t nb = (nv + kPlaceBlock - 1) / kPlaceBlock;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
       b += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t pos = 0;
    const uint64_t v1 = min(nv, (b + 1) * kPlaceBlock);
    for (uint64_t v = b * kPlaceBlock; v < v1; ++v) {
      const uint32_t sz = size[v];
      if (sz & kLongSize) {
        const uint64_t nl = sz & ~kLongSize;
        if (nl > kCmpMaxLines) *err = 1;
        pos = (pos + kLineBits - 1) / kLineBits * kLineBits;
        cpos[v] = pos | kCmpLong | (nl << kCmpPosBits);
        pos += nl * kLineBits;
      } else {
        if (sz && (pos % kShortSpanBits) + sz > kShortSpanBits)  // next 256-byte span
          pos = (pos + kShortSpanBits - 1) / kShortSpanBits * kShortSpanBits;
        cpos[v] = pos;
        pos += sz;
      }
    }
    block_bits[b] = (pos + kShortSpanBits - 1) / kShortSpanBits * kShortSpanBits;
  }
}

// cpos[v] += the block's base (exclusive scan of block_bits); cpos[nv] = end.
__global__ void k_cmp_place_add(uint64_t nv, uint64_t* cpos, const uint64_t* base) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nv;
       v += (uint64_t)gridDim.x * blockDim.x)
    cpos[v] = v < nv ? cpos[v] + base[v / kPlaceBlock] : base[(nv + kPlaceBlock - 1) / kPlaceBlock];
}

// Transpose: in-degree count, then a scatter of every arc (v -> d) into d's
// in-list (slot from a per-vertex cursor; the lists are sorted afterwards).
__global__ void k_in_count(uint64_t ne, const uint32_t* e, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + e[i], 1u);
}

__global__ void k_in_scatter(uint64_t nv, const uint64_t* off, const uint32_t* e,
                             const uint64_t* in_off, uint32_t* cursor, uint32_t* in_e) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw)
    for (uint64_t k = off[v] + lane; k < off[v + 1]; k += 32) {
      const uint32_t d = e[k];
      in_e[in_off[d] + atomicAdd(cursor + d, 1u)] = static_cast<uint32_t>(v);
    }
}

// The owning list of every element: src[k] = v for off[v] <= k < off[v+1]
// (warp per list; a hub list's warp streams its stores).
__global__ void k_arc_sources(uint64_t nv, const uint64_t* off, uint32_t* src) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], e = off[v + 1];
    for (uint64_t k = s + lane; k < e; k += 32) src[k] = static_cast<uint32_t>(v);
  }
}

// List offsets from sorted keys: off[j] = first i with keys[i] >= j, for
// j in [0, nk]; thread i fills the offsets of the keys between keys[i-1] and
// keys[i] (i == ne: up to nk), so every offset is written once.
__global__ void k_offsets_from_sorted(uint64_t ne, const uint32_t* keys, uint64_t nk,
                                      uint64_t* off) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= ne;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = i ? static_cast<uint64_t>(keys[i - 1]) + 1 : 0;
    const uint64_t hi = i < ne ? static_cast<uint64_t>(keys[i]) : nk;
    for (uint64_t j = lo; j <= hi; ++j) off[j] = i;
  }
}

}  // namespace

// device temporaries are released on every path
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { reset(); }
  cudaError_t scratch(size_t bytes) { return cudaMalloc(&p, bytes); }
  void reset() {
    cudaFree(p);
    p = nullptr;
  }
  void* release() {  // the buffer changes owner
    void* q = p;
    p = nullptr;
    return q;
  }
  void take(DevBuf* o) {
    reset();
    p = o->release();
  }
};

namespace {
// Transpose by a stable device radix sort: the nl lists (offsets d_off) of
// element ids < nk become nk lists of list ids, ascending inside each list
// (keys = elements, values = owning list ids in ascending order; LSD radix
// sorting is stable) -- sorted in-lists from sorted or unsorted out-lists
// (two transposes sort every list: sort_lists_radix_keep).  Replaces a count
// / atomic-cursor scatter followed by a segmented sort (~0.55 s at 2^31
// arcs).  e (ne elements) is consumed; t_e / t_off (nk + 1 offsets, from the
// sorted keys) receive the result.  Returns ZC_ENOMEM with e intact and
// nothing allocated when the four ne-element buffers do not fit (callers
// fall back).
int radix_transpose(uint64_t nl, const uint64_t* d_off, DevBuf* e, uint64_t ne, uint64_t nk,
                    DevBuf* t_e, DevBuf* t_off, zc_graph* g, const char* tag) {
  auto mark = [&](const char* what) {
    if (g) build_mark(g, (std::string(tag) + what).c_str());
  };
  const uint32_t bits = nk > 1 ? 64 - __builtin_clzll(nk - 1) : 1;
  const size_t nb = std::max<uint64_t>(ne, 1) * sizeof(uint32_t);
  DevBuf src, kalt, valt, off, tmp;
  cub::DoubleBuffer<uint32_t> probe_k(nullptr, nullptr), probe_v(nullptr, nullptr);
  size_t tb = 0;
  ZC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, probe_k, probe_v, ne, 0,
                                              static_cast<int>(bits)));
  if (src.scratch(nb) != cudaSuccess || kalt.scratch(nb) != cudaSuccess ||
      valt.scratch(nb) != cudaSuccess || off.scratch((nk + 1) * sizeof(uint64_t)) != cudaSuccess ||
      tmp.scratch(tb) != cudaSuccess) {
    cudaGetLastError();  // the failed allocation is not sticky
    return ZC_ENOMEM;
  }
  mark(":alloc");
  uint32_t* ke = static_cast<uint32_t*>(e->p);
  k_arc_sources<<<kCmpGrid, 256>>>(nl, d_off, static_cast<uint32_t*>(src.p));
  ZC_CUDA_TRY(cudaGetLastError());
  mark(":sources");
  cub::DoubleBuffer<uint32_t> keys(ke, static_cast<uint32_t*>(kalt.p));
  cub::DoubleBuffer<uint32_t> vals(static_cast<uint32_t*>(src.p), static_cast<uint32_t*>(valt.p));
  ZC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, vals, ne, 0,
                                              static_cast<int>(bits)));
  k_offsets_from_sorted<<<kCmpGrid, 256>>>(ne, keys.Current(), nk, static_cast<uint64_t*>(off.p));
  ZC_CUDA_TRY(cudaGetLastError());
  mark(":radix");
  DevBuf* held = vals.Current() == src.p ? &src : &valt;
  t_e->take(held);
  t_off->take(&off);
  e->reset();
  src.reset();
  kalt.reset();
  valt.reset();
  tmp.reset();
  mark(":free");
  return ZC_OK;
}
}  // namespace

namespace {
// Every list (offsets d_off, u32 elements < nk) sorted in place by two radix
// transposes through three scratch buffers allocated once: the first leaves
// the transposed lists (the graph's in-lists, ascending) in one of them, the
// second writes the sorted lists back (into `edges` itself, or a copy).
// keep_e / keep_off (optional) receive a copy of the first transpose and its
// offsets.  ZC_ENOMEM, lists untouched, when the scratch does not fit.  g
// (optional) takes the phase marks.
int sort_lists_radix_keep(zc_graph* g, uint64_t nv, const uint64_t* d_off, uint32_t* edges,
                          uint64_t ne, uint64_t nk, DevBuf* keep_e, DevBuf* keep_off) {
  auto mark = [&](const char* what) {
    if (g) build_mark(g, what);
  };
  const uint32_t bits_k = nk > 1 ? 64 - __builtin_clzll(nk - 1) : 1;
  const uint32_t bits_v = nv > 1 ? 64 - __builtin_clzll(nv - 1) : 1;
  const size_t nb = std::max<uint64_t>(ne, 1) * sizeof(uint32_t);
  DevBuf K, S, V, toff, tmp;
  cub::DoubleBuffer<uint32_t> pk(nullptr, nullptr), pv(nullptr, nullptr);
  size_t tb = 0;
  ZC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, pk, pv, ne, 0,
                                              static_cast<int>(std::max(bits_k, bits_v))));
  if (K.scratch(nb) != cudaSuccess || S.scratch(nb) != cudaSuccess ||
      V.scratch(nb) != cudaSuccess || toff.scratch((nk + 1) * sizeof(uint64_t)) != cudaSuccess ||
      tmp.scratch(tb) != cudaSuccess) {
    cudaGetLastError();
    return ZC_ENOMEM;
  }
  mark("out:sort:alloc");
  uint32_t* E = edges;
  uint32_t* k = static_cast<uint32_t*>(K.p);
  uint32_t* sp = static_cast<uint32_t*>(S.p);
  uint32_t* vp = static_cast<uint32_t*>(V.p);
  // 1: keys = elements, values = owning lists (ascending) -> transposed lists
  k_arc_sources<<<kCmpGrid, 256>>>(nv, d_off, sp);
  cub::DoubleBuffer<uint32_t> keys(E, k), vals(sp, vp);
  ZC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, vals, ne, 0,
                                              static_cast<int>(bits_k)));
  k_offsets_from_sorted<<<kCmpGrid, 256>>>(ne, keys.Current(), nk,
                                           static_cast<uint64_t*>(toff.p));
  ZC_CUDA_TRY(cudaGetLastError());
  uint32_t* T = vals.Current();
  uint32_t* U = T == sp ? vp : sp;
  DevBuf copy;
  if (keep_e) {  // the second transpose overwrites T's buffer pair
    if (copy.scratch(nb) == cudaSuccess)
      ZC_CUDA_TRY(cudaMemcpyAsync(copy.p, T, nb, cudaMemcpyDeviceToDevice, 0));
    else
      cudaGetLastError();  // no copy: the caller transposes again later
  }
  mark("out:sort:t1");
  // 2: keys = transposed elements (list ids), values = their owners -> sorted lists
  k_arc_sources<<<kCmpGrid, 256>>>(nk, static_cast<uint64_t*>(toff.p), k);
  cub::DoubleBuffer<uint32_t> keys2(T, U), vals2(k, E);
  ZC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys2, vals2, ne, 0,
                                              static_cast<int>(bits_v)));
  if (vals2.Current() != E)
    ZC_CUDA_TRY(cudaMemcpyAsync(E, vals2.Current(), nb, cudaMemcpyDeviceToDevice, 0));
  ZC_CUDA_TRY(cudaGetLastError());
  mark("out:sort:t2");
  if (keep_e && copy.p) {
    keep_e->take(&copy);
    keep_off->take(&toff);
  }
  return ZC_OK;
}
}  // namespace

int sort_lists_radix(uint64_t nv, const uint64_t* d_off, uint32_t* edges, uint64_t ne,
                     uint64_t nk) {
  return sort_lists_radix_keep(nullptr, nv, d_off, edges, ne, nk, nullptr, nullptr);
}

// Sorted lists (x) over offsets d_off -> the line stream in device memory
// (enc) and the per-vertex bit positions (cpos).
namespace {
// Bits of the largest vertex id a list can hold (global ids for partitions).
uint32_t first_element_bits(const zc_graph* g) {
  const uint64_t maxid = (g->nparts ? g->global_nv : g->nv);
  return maxid > 1 ? 64 - __builtin_clzll(maxid - 1) : 1;
}

// enc_kept: the stream stays in HBM (an HBM-placed handle keeps it), else it
// is scratch until copied to host memory.  The encode is left running: the
// caller's host-side allocation overlaps it.
int encode_stream(uint64_t nv, const uint64_t* d_off, const Elems& x, uint32_t ww, uint32_t b0,
                  bool enc_kept, DevBuf* cpos, DevBuf* enc, size_t* bytes) {
  DevBuf size, blk, tmp, err;
  const uint64_t nb = (nv + kPlaceBlock - 1) / kPlaceBlock;
  ZC_CUDA_TRY(size.scratch(std::max<uint64_t>(nv, 1) * sizeof(uint32_t)));
  k_cmp_size<<<kCmpGrid, 256>>>(nv, d_off, x, ww, b0, static_cast<uint32_t*>(size.p));
  ZC_CUDA_TRY(cudaGetLastError());
  ZC_CUDA_TRY(cudaMalloc(&cpos->p, (nv + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(blk.scratch((nb + 1) * 2 * sizeof(uint64_t)));  // sizes, then bases
  ZC_CUDA_TRY(err.scratch(sizeof(unsigned)));
  ZC_CUDA_TRY(cudaMemset(err.p, 0, sizeof(unsigned)));
  uint64_t* bbits = static_cast<uint64_t*>(blk.p);
  uint64_t* bbase = bbits + nb + 1;
  ZC_CUDA_TRY(cudaMemset(bbits + nb, 0, sizeof(uint64_t)));
  k_cmp_place_local<<<std::max<uint64_t>((nb + 127) / 128, 1), 128>>>(
      nv, static_cast<uint32_t*>(size.p), static_cast<uint64_t*>(cpos->p), bbits,
      static_cast<unsigned*>(err.p));
  ZC_CUDA_TRY(cudaGetLastError());
  size_t tb = 0;
  ZC_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, bbits, bbase, nb + 1));
  ZC_CUDA_TRY(tmp.scratch(std::max<size_t>(tb, 1)));
  ZC_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, bbits, bbase, nb + 1));
  k_cmp_place_add<<<kCmpGrid, 256>>>(nv, static_cast<uint64_t*>(cpos->p), bbase);
  ZC_CUDA_TRY(cudaGetLastError());
  uint64_t end = 0;
  unsigned herr = 0;
  ZC_CUDA_TRY(cudaMemcpy(&end, static_cast<uint64_t*>(cpos->p) + nv, sizeof(end),
                         cudaMemcpyDeviceToHost));
  ZC_CUDA_TRY(cudaMemcpy(&herr, err.p, sizeof(herr), cudaMemcpyDeviceToHost));
  if (herr) {
    set_error("a list needs more compressed lines than the index can record");
    return ZC_EINVAL;
  }
  if (end > kCmpPosMask) {
    set_error("compressed stream exceeds the index's 2^40-bit positions");
    return ZC_EINVAL;
  }
  const uint64_t lines = end / kLineBits;  // span-aligned, so whole lines
  *bytes = std::max<uint64_t>(lines, 1) * kLineBytes;
  if (enc_kept) ZC_CUDA_TRY(cudaMalloc(&enc->p, *bytes));
  else ZC_CUDA_TRY(enc->scratch(*bytes));
  ZC_CUDA_TRY(cudaMemsetAsync(enc->p, 0, *bytes, 0));
  k_cmp_encode<<<kCmpGrid, 256>>>(nv, d_off, x, ww, b0, static_cast<uint64_t*>(cpos->p),
                                  static_cast<uint32_t*>(enc->p));
  ZC_CUDA_TRY(cudaGetLastError());
  return ZC_OK;
}

}  // namespace

// Place an encoded stream like the handle's lists: host (pinned / managed,
// read zero-copy), managed (UVM) or HBM (with a host shadow).
int place_stream(zc_graph* g, DevBuf* enc, size_t bytes, void** host_out, const void** dev_out,
                 void** hbm_out, std::future<HostMap>* pre = nullptr, const char* tag = "out") {
  void* host = nullptr;
  const void* dev = nullptr;
  void* hbm = nullptr;
  if (g->placement == ZC_PLACE_UVM) {
    ZC_CUDA_TRY(cudaMallocManaged(&host, bytes, cudaMemAttachGlobal));
    if (cudaMemcpy(host, enc->p, bytes, cudaMemcpyDefault) != cudaSuccess ||
        cudaMemAdvise(host, bytes, cudaMemAdviseSetReadMostly, g->device) != cudaSuccess) {
      cudaFree(host);
      set_error(std::string("compressed lists (uvm): ") + cudaGetErrorString(cudaGetLastError()));
      return ZC_ECUDA;
    }
    dev = host;
  } else {
    // the stream, or the HBM run's host shadow (pre: allocated in the background)
    host = pre && pre->valid() ? pinned_list_finish(pre->get(), bytes) : host_list_alloc(g, bytes);
    if (!host) {
      set_error("cannot allocate host memory for the compressed lists");
      return ZC_ENOMEM;
    }
    build_mark(g, (std::string(tag) + ":encode+pin_alloc").c_str());  // overlaps the encode
    const void* d = nullptr;
    if (cudaMemcpy(host, enc->p, bytes, cudaMemcpyDefault) != cudaSuccess ||
        (g->placement != ZC_PLACE_HBM && host_list_device_ptr(host, &d) != ZC_OK)) {
      pinned_list_free(host);
      set_error(std::string("compressed lists: ") + cudaGetErrorString(cudaGetLastError()));
      return ZC_ECUDA;
    }
    if (g->placement == ZC_PLACE_HBM) {
      hbm = enc->release();
      dev = hbm;
    } else {
      dev = d;
    }
  }
  build_mark(g, (std::string(tag) + ":d2h_copy").c_str());
  *host_out = host;
  *dev_out = dev;
  *hbm_out = hbm;
  return ZC_OK;
}

// An in-list stream encoded ahead of its placement: a fresh direction-
// optimizing build encodes the in-lists right after the out-list sort and
// allocates their pinned host stream on a background thread while the
// out-list stream is encoded and placed.
struct InPrep {
  DevBuf in_e, in_off;  // sorted in-lists (device) and their offsets
  DevBuf enc, cpos;
  size_t bytes = 0;
  std::future<HostMap> host;  // the host stream's mapping, prefaulted in the background
  ~InPrep() {
    if (host.valid()) pinned_list_unmap(host.get());
  }
};

int prepare_in_stream(zc_graph* g, uint64_t* d_in_off, uint32_t* d_in_sorted, InPrep* p,
                      bool background_alloc) {
  Elems x{d_in_sorted, nullptr, 0};
  int rc = encode_stream(g->nv, d_in_off, x, 0, first_element_bits(g),
                         g->placement == ZC_PLACE_HBM, &p->cpos, &p->enc, &p->bytes);
  if (rc) return rc;
  if (background_alloc && (g->placement == ZC_PLACE_ZEROCOPY || g->placement == ZC_PLACE_HBM)) {
    // only the mapping and first touch: registering pins pages under a driver
    // lock that would stall this thread's device calls (measured: slower)
    const size_t bytes = p->bytes;
    const int dev = g->device;
    try {
      p->host = std::async(std::launch::async,
                           [dev, bytes] { return pinned_list_map(dev, bytes); });
    } catch (...) {  // no thread: place_stream allocates on this one
    }
  }
  build_mark(g, "in:size_place");
  return ZC_OK;
}

int place_in_stream(zc_graph* g, uint64_t* d_in_off, InPrep* p) {
  void* host = nullptr;
  const void* dev = nullptr;
  void* hbm = nullptr;
  int rc = place_stream(g, &p->enc, p->bytes, &host, &dev, &hbm, &p->host, "in");
  if (rc) return rc;
  g->h_cmp_in = host;
  g->d_cmp_in = dev;
  g->hbm_cmp_in = hbm;
  g->d_cpos_in = static_cast<uint64_t*>(p->cpos.release());
  g->d_in_off = d_in_off;
  g->cmp_in_bytes = p->bytes;
  rc = alloc_pull_state(g);
  build_mark(g, "in:pull_state");
  return rc;
}

int install_in_lists(zc_graph* g, uint64_t* d_in_off, uint32_t* d_in_sorted) {
  InPrep p;
  int rc = prepare_in_stream(g, d_in_off, d_in_sorted, &p, false);
  return rc ? rc : place_in_stream(g, d_in_off, &p);
}

int alloc_pull_state(zc_graph* g) {
  if (!g->d_cand) {
    ZC_CUDA_TRY(cudaMalloc(&g->d_cand, g->vpad));
    ZC_CUDA_TRY(cudaMemset(g->d_cand, 0, g->vpad));
  }
  if (!g->d_fbits) {
    const uint64_t words = ((g->nparts ? g->global_nv : g->nv) + 31) / 32 + 1;
    ZC_CUDA_TRY(cudaMalloc(&g->d_fbits, words * sizeof(uint32_t)));
  }
  if (!g->d_hasin) {
    ZC_CUDA_TRY(cudaMalloc(&g->d_hasin, ((g->nv + 31) / 32 + 1) * sizeof(uint32_t)));
    ZC_CUDA_TRY(cudaMemset(g->d_hasin, 0, ((g->nv + 31) / 32 + 1) * sizeof(uint32_t)));
    ZC_CUDA_TRY(launch_hasin(g->nv, g->d_in_off, g->d_hasin, 0));
    ZC_CUDA_TRY(cudaDeviceSynchronize());
  }
  return ZC_OK;
}

}  // namespace zc

using namespace zc;

namespace {
// The out-list stream.  keep_lists (unweighted graphs): hand the sorted device
// copy of the raw lists to the caller (the in-list transpose reads it instead
// of copying the lists from host memory again).
// Sort the out-lists in place (sorted: the device copy, offsets g->d_off):
// two radix transposes, or the segmented sort when they do not fit.  With
// keep_in_e, the first transpose's sorted in-lists are handed over too
// (directed, unpartitioned graphs; left empty otherwise).
int sort_out_lists(zc_graph* g, DevBuf* sorted, DevBuf* keep_in_e, DevBuf* keep_in_off) {
  const uint64_t nv = g->nv, ne = g->ne;
  const uint64_t nk = g->nparts ? g->global_nv : nv;
  bool asc = false;
  ZC_CUDA_TRY(lists_ascending(nv, g->d_off, static_cast<const uint32_t*>(sorted->p), &asc));
  set_sort_gpu_ms(0);
  if (asc) return ZC_OK;
  const bool keep = keep_in_e && !g->nparts && (g->flags & ZC_F_DIRECTED);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  int rc = g->tune.seg_sort
               ? ZC_ENOMEM
               : sort_lists_radix_keep(g, nv, g->d_off, static_cast<uint32_t*>(sorted->p), ne,
                                       nk, keep ? keep_in_e : nullptr,
                                       keep ? keep_in_off : nullptr);
  if (rc == ZC_ENOMEM)  // the lists are intact: the segmented sort
    rc = sort_lists_device(4, nv, g->d_off, sorted->p, false);
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  set_sort_gpu_ms(ms);
  return rc;
}

int build_out_stream(zc_graph* g, DevBuf* keep_lists, InPrep* prep = nullptr) {
  cudaSetDevice(g->device);
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  build_start(g);
  const uint64_t nv = g->nv, ne = g->ne;
  // weights ride along when they are 4-byte (SSSP on the compressed stream)
  const bool weighted = g->has_weights && g->wb == 4 && g->h_weights;
  DevBuf sorted, wtmp, enc, cpos, range;
  Elems x{nullptr, nullptr, 0};
  uint32_t ww = 0;
  if (weighted) {
    ZC_CUDA_TRY(sorted.scratch(std::max<uint64_t>(ne, 1) * 8));
    ZC_CUDA_TRY(wtmp.scratch(std::max<uint64_t>(ne, 1) * 8));
    ZC_CUDA_TRY(range.scratch(2 * sizeof(unsigned)));
    const unsigned init[2] = {0xffffffffu, 0u};
    ZC_CUDA_TRY(cudaMemcpy(range.p, init, sizeof(init), cudaMemcpyHostToDevice));
    uint32_t* de = static_cast<uint32_t*>(wtmp.p);
    uint32_t* dw = de + std::max<uint64_t>(ne, 1);
    ZC_CUDA_TRY(cudaMemcpy(de, g->h_edges, ne * 4, cudaMemcpyDefault));
    ZC_CUDA_TRY(cudaMemcpy(dw, g->h_weights, ne * 4, cudaMemcpyDefault));
    unsigned* r = static_cast<unsigned*>(range.p);
    k_cmp_pairs<<<kCmpGrid, 256>>>(ne, de, dw, static_cast<uint64_t*>(sorted.p), r, r + 1);
    ZC_CUDA_TRY(cudaGetLastError());
    unsigned hr[2];
    ZC_CUDA_TRY(cudaMemcpy(hr, r, sizeof(hr), cudaMemcpyDeviceToHost));
    wtmp.reset();
    if (!ne) hr[0] = hr[1] = 0;
    x.e64 = static_cast<const uint64_t*>(sorted.p);
    x.wmin = hr[0];
    ww = hr[1] > hr[0] ? 32 - __builtin_clz(hr[1] - hr[0]) : 0;
    build_mark(g, "out:h2d_pairs");
    const int rc = sort_lists_device(8, nv, g->d_off, sorted.p);
    if (rc) return rc;
  } else {
    ZC_CUDA_TRY(sorted.scratch(std::max<uint64_t>(ne, 1) * 4));
    ZC_CUDA_TRY(cudaMemcpy(sorted.p, g->h_edges, ne * 4, cudaMemcpyDefault));
    build_mark(g, "out:h2d_copy");
    int rc = sort_out_lists(g, &sorted, prep ? &prep->in_e : nullptr,
                            prep ? &prep->in_off : nullptr);
    if (rc) return rc;
    x.e32 = static_cast<const uint32_t*>(sorted.p);
    if (prep && prep->in_e.p &&  // the in-lists came with the sort: encode them now
        (rc = prepare_in_stream(g, static_cast<uint64_t*>(prep->in_off.p),
                                static_cast<uint32_t*>(prep->in_e.p), prep, true)))
      return rc;
  }
  build_mark(g, "out:sort");
  g->build_log.emplace_back("out:sort[gpu]", last_sort_gpu_ms());
  size_t bytes = 0;
  const uint32_t b0 = first_element_bits(g);
  int rc = encode_stream(nv, g->d_off, x, ww, b0, g->placement == ZC_PLACE_HBM, &cpos, &enc,
                         &bytes);
  if (rc) return rc;
  if (keep_lists && !weighted) keep_lists->take(&sorted);
  sorted.reset();
  build_mark(g, "out:size_place");
  void* host = nullptr;
  const void* dev = nullptr;
  void* hbm = nullptr;
  if ((rc = place_stream(g, &enc, bytes, &host, &dev, &hbm))) return rc;
  g->h_cmp = host;
  g->d_cmp = dev;
  g->hbm_cmp = hbm;
  g->d_cpos = static_cast<uint64_t*>(cpos.release());
  g->cmp_bytes = bytes;
  g->cmp_weighted = weighted;
  g->cmp_ww = ww;
  g->cmp_b0 = b0;
  g->cmp_wmin = x.wmin;
  return ZC_OK;
}
}  // namespace

extern "C" int zc_graph_build_compressed(zc_graph* g, uint64_t* compressed_bytes) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (g->eb != 4) {
    set_error("compressed lists need 4-byte edges");
    return ZC_EINVAL;
  }
  if (!g->h_cmp) {
    const int rc = build_out_stream(g, nullptr);
    if (rc) return rc;
  }
  if (compressed_bytes) *compressed_bytes = g->cmp_bytes;
  return ZC_OK;
}

namespace {
// Sorted in-lists (device, offsets in_off) -> the handle's in-list stream.
int finish_in_lists(zc_graph* g, DevBuf* in_e, DevBuf* in_off, uint64_t* compressed_bytes) {
  int rc = install_in_lists(g, static_cast<uint64_t*>(in_off->p), static_cast<uint32_t*>(in_e->p));
  if (rc) return rc;
  in_off->release();  // owned by the handle now
  if ((rc = alloc_pull_state(g))) return rc;
  if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
  return ZC_OK;
}
}  // namespace

extern "C" int zc_graph_build_in_lists(zc_graph* g, uint64_t* compressed_bytes) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (g->d_cpos_in) {
    if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
    return ZC_OK;
  }
  if (g->eb != 4) {
    set_error("compressed lists need 4-byte edges");
    return ZC_EINVAL;
  }
  if (g->nparts && (g->flags & ZC_F_DIRECTED)) {
    set_error("a directed partition's in-lists come from zc_part_build_in_lists");
    return ZC_EINVAL;
  }
  const bool transpose = (g->flags & ZC_F_DIRECTED) != 0;
  DevBuf out_e;  // the raw lists on the device (any order inside a list)
  InPrep prep;  // or the out-list sort's transpose: the sorted, encoded in-lists
  int rc = ZC_OK;
  if (!g->h_cmp &&
      (rc = build_out_stream(g, transpose ? &out_e : nullptr, transpose ? &prep : nullptr)))
    return rc;
  cudaSetDevice(g->device);
  build_start(g);
  const uint64_t nv = g->nv, ne = g->ne;
  if (!(g->flags & ZC_F_DIRECTED)) {  // in-lists are the out-lists
    g->d_in_off = g->d_off;
    g->d_cpos_in = g->d_cpos;
    g->d_cmp_in = g->d_cmp;
    g->cmp_in_bytes = g->cmp_bytes;
    g->in_alias = true;
  } else {
    DevBuf in_e, deg, in_off, tmp;
    if (prep.enc.p) {  // transposed and encoded while the out-lists were built
      out_e.reset();
      if ((rc = place_in_stream(g, static_cast<uint64_t*>(prep.in_off.p), &prep))) return rc;
      prep.in_off.release();  // owned by the handle now
      if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
      return ZC_OK;
    }
    if (!out_e.p) {
      ZC_CUDA_TRY(out_e.scratch(std::max<uint64_t>(ne, 1) * 4));
      ZC_CUDA_TRY(cudaMemcpy(out_e.p, g->h_edges, ne * 4, cudaMemcpyDefault));
      build_mark(g, "in:h2d_copy");
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    rc = g->tune.seg_sort
             ? ZC_ENOMEM
             : radix_transpose(nv, g->d_off, &out_e, ne, nv, &in_e, &in_off, g, "in:t");
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc == ZC_OK) {
      build_mark(g, "in:transpose");
      g->build_log.emplace_back("in:transpose[gpu]", ms);
      return finish_in_lists(g, &in_e, &in_off, compressed_bytes);
    }
    if (rc != ZC_ENOMEM) return rc;
    // the radix transpose's buffers do not fit: count, scatter, segmented sort
    ZC_CUDA_TRY(deg.scratch(std::max<uint64_t>(nv, 1) * 4));
    ZC_CUDA_TRY(cudaMemset(deg.p, 0, std::max<uint64_t>(nv, 1) * 4));
    k_in_count<<<kCmpGrid, 256>>>(ne, static_cast<uint32_t*>(out_e.p),
                                  static_cast<uint32_t*>(deg.p));
    ZC_CUDA_TRY(cudaGetLastError());
    ZC_CUDA_TRY(cudaMalloc(&in_off.p, (nv + 1) * sizeof(uint64_t)));
    const size_t tb = scan_tmp_bytes(nv);
    ZC_CUDA_TRY(tmp.scratch(tb));
    ZC_CUDA_TRY(scan_u32_to_u64(static_cast<uint32_t*>(deg.p), static_cast<uint64_t*>(in_off.p),
                                nv, tmp.p, tb, 0));
    tmp.reset();
    ZC_CUDA_TRY(cudaMemset(deg.p, 0, std::max<uint64_t>(nv, 1) * 4));  // now the cursors
    ZC_CUDA_TRY(in_e.scratch(std::max<uint64_t>(ne, 1) * 4));
    k_in_scatter<<<kCmpGrid, 256>>>(nv, g->d_off, static_cast<uint32_t*>(out_e.p),
                                    static_cast<uint64_t*>(in_off.p),
                                    static_cast<uint32_t*>(deg.p), static_cast<uint32_t*>(in_e.p));
    ZC_CUDA_TRY(cudaGetLastError());
    out_e.reset();
    deg.reset();
    build_mark(g, "in:transpose");
    rc = sort_lists_device(4, nv, static_cast<uint64_t*>(in_off.p), in_e.p, !g->tune.seg_sort);
    if (rc) return rc;
    build_mark(g, "in:sort");
    g->build_log.emplace_back("in:sort[gpu]", last_sort_gpu_ms());
    if ((rc = install_in_lists(g, static_cast<uint64_t*>(in_off.p),
                               static_cast<uint32_t*>(in_e.p))))
      return rc;
    in_off.release();  // owned by the handle now
  }
  if ((rc = alloc_pull_state(g))) return rc;
  if (compressed_bytes) *compressed_bytes = g->cmp_in_bytes;
  return ZC_OK;
}

extern "C" int zc_graph_compressed_index(const zc_graph* g, uint64_t* cpos) {
  if (!g || !g->d_cpos) {
    set_error(g ? "compressed lists not built" : "null graph handle");
    return ZC_ESTATE;
  }
  if (!cpos) {
    set_error("null output buffer");
    return ZC_EINVAL;
  }
  cudaSetDevice(g->device);
  ZC_CUDA_TRY(cudaMemcpy(cpos, g->d_cpos, (g->nv + 1) * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost));
  return ZC_OK;
}
