// Line-compressed lists: an optional B200-native host-store format.
//
// Zero-copy traversal is bound by the host link: ~437 M fully-used 128-byte
// line reads/s (55.9 GB/s of PCIe read bytes, profiles/ncu_summary.json), and
// about as much by the request count as by the bytes.  BFS / CC / PageRank
// results do not depend on the order inside a list, so a list can be sorted
// and stored delta-encoded in self-describing 128-byte lines (format in
// zc_internal.cuh): one aligned line read then carries ~50-100 edges of a hub
// list instead of 32.  A list is compressed only when that needs fewer lines
// than its raw form touches; short lists stay raw (packed windows share their
// lines).  Lines are filled greedily: as many deltas as fit 1024 - 48 bits at
// the width of the widest one, at most 255.
//
// Per-vertex first-line index coff (u64[V+1]) lives in HBM next to the CSR
// offsets; the line stream lives in the handle's placement.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "zc_graph.cuh"
#include "zc_internal.cuh"

namespace zc {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint32_t bits_of(uint32_t x) { return x ? 32 - __clz(x) : 0; }

// Greedy fill of one line starting at element p of the sorted list e[0, d):
// the largest K <= min(255, d-1-p) with 48 + K * max(bits(delta 1..K)) <=
// 1024.  Warp-cooperative; returns count = K + 1 and the width.
__device__ __forceinline__ void line_fill(const uint32_t* e, uint64_t d, uint64_t p, int lane,
                                          uint32_t* count, uint32_t* width) {
  const uint64_t rest = d - 1 - p;
  const uint32_t kmax = static_cast<uint32_t>(rest < kCmpMaxCount - 1 ? rest : kCmpMaxCount - 1);
  uint32_t K = 0, m = 0;
  for (uint32_t c = 0; c < kmax; c += 32) {
    const uint32_t k = c + lane + 1;
    uint32_t pm = m;
    if (k <= kmax) pm = max(pm, bits_of(e[p + k] - e[p + k - 1]));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFullMask, pm, o);
      if (lane >= o) pm = max(pm, t);
    }
    // 48 + k * pm is non-decreasing in the lane: the fitting lanes are a prefix
    const bool ok = k <= kmax && kCmpHdrBits + k * pm <= kLineWords * 32;
    const int nok = __popc(__ballot_sync(kFullMask, ok));
    if (nok) m = __shfl_sync(kFullMask, pm, nok - 1);
    K = c + nok;
    if (nok < 32) break;
  }
  *count = K + 1;
  *width = m;
}

// Lines the list of v needs compressed, or 0 when raw is no worse.  Host
// memory is read in 32-byte sectors: a raw list costs the sectors it touches
// (and shares its partial lines with neighbouring lists under packed
// windows), a compressed one full lines -- so compress only when that reads
// strictly fewer sectors (in practice lists of more than ~28 elements).
__global__ void k_cmp_lines(uint64_t nv, const uint64_t* off, const uint32_t* e,
                            uint32_t* lines) {
  constexpr uint64_t kSectorElems = 8, kLineSectors = 4;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], d = off[v + 1] - s;
    const uint64_t raw = d ? (s + d - 1) / kSectorElems - s / kSectorElems + 1 : 0;
    uint32_t n = 0;
    if (raw > kLineSectors) {
      for (uint64_t p = 0; p < d && n * kLineSectors < raw; ++n) {
        uint32_t cnt, w;
        line_fill(e + s, d, p, lane, &cnt, &w);
        p += cnt;
      }
      if (n * kLineSectors >= raw) n = 0;
    }
    if (lane == 0) lines[v] = n;
  }
}

// Encode: warp per compressed list, one shared-memory line buffer per warp.
__global__ void __launch_bounds__(256) k_cmp_encode(uint64_t nv, const uint64_t* off,
                                                    const uint32_t* e, const uint64_t* coff,
                                                    uint32_t* out) {
  __shared__ uint32_t buf[8][kLineWords + 2];
  const int lane = threadIdx.x & 31;
  uint32_t* L = buf[threadIdx.x >> 5];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t l0 = coff[v], nl = coff[v + 1] - l0;
    if (!nl) continue;
    const uint64_t s = off[v], d = off[v + 1] - s;
    const uint32_t* x = e + s;
    uint64_t p = 0;
    for (uint64_t t = 0; t < nl; ++t) {
      uint32_t cnt, w;
      line_fill(x, d, p, lane, &cnt, &w);
      L[lane] = 0;
      if (lane < 2) L[kLineWords + lane] = 0;
      __syncwarp();
      if (w)
        for (uint32_t k = lane + 1; k < cnt; k += 32) {
          const uint32_t dl = x[p + k] - x[p + k - 1];
          const uint32_t bit = kCmpHdrBits + (k - 1) * w;
          atomicOr(&L[bit >> 5], dl << (bit & 31));
          if ((bit & 31) + w > 32) atomicOr(&L[(bit >> 5) + 1], dl >> (32 - (bit & 31)));
        }
      __syncwarp();
      if (lane == 0) {
        L[0] = x[p];
        L[1] |= w | ((cnt - 1) << 6);
      }
      __syncwarp();
      out[(l0 + t) * kLineWords + lane] = L[lane];
      __syncwarp();
      p += cnt;
    }
  }
}

constexpr int kCmpGrid = 148 * 16;

}  // namespace
}  // namespace zc

using namespace zc;

extern "C" int zc_graph_build_compressed(zc_graph* g, uint64_t* compressed_bytes) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (g->eb != 4) {
    set_error("compressed lists need 4-byte edges");
    return ZC_EINVAL;
  }
  if (g->h_cmp) {
    if (compressed_bytes) *compressed_bytes = g->cmp_bytes;
    return ZC_OK;
  }
  cudaSetDevice(g->device);
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  const uint64_t nv = g->nv, ne = g->ne;
  // device temporaries are released on every path; the handle is only
  // updated once the whole stream is built
  struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
    void* release() {
      void* q = p;
      p = nullptr;
      return q;
    }
  } sorted, lines, tmp, enc, coff;
  ZC_CUDA_TRY(cudaMalloc(&sorted.p, std::max<uint64_t>(ne, 1) * 4));
  ZC_CUDA_TRY(cudaMemcpy(sorted.p, g->h_edges, ne * 4, cudaMemcpyDefault));
  const int rc = sort_lists_device(4, nv, g->d_off, g->h_off, sorted.p);
  if (rc) return rc;
  ZC_CUDA_TRY(cudaMalloc(&coff.p, (nv + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&lines.p, std::max<uint64_t>(nv, 1) * sizeof(uint32_t)));
  k_cmp_lines<<<kCmpGrid, 256>>>(nv, g->d_off, static_cast<uint32_t*>(sorted.p),
                                 static_cast<uint32_t*>(lines.p));
  ZC_CUDA_TRY(cudaGetLastError());
  const size_t tb = scan_tmp_bytes(nv);
  ZC_CUDA_TRY(cudaMalloc(&tmp.p, tb));
  ZC_CUDA_TRY(scan_u32_to_u64(static_cast<uint32_t*>(lines.p), static_cast<uint64_t*>(coff.p), nv,
                              tmp.p, tb, 0));
  uint64_t total = 0;
  ZC_CUDA_TRY(cudaMemcpy(&total, static_cast<uint64_t*>(coff.p) + nv, sizeof(total),
                         cudaMemcpyDeviceToHost));
  const size_t bytes = std::max<uint64_t>(total, 1) * kLineBytes;
  ZC_CUDA_TRY(cudaMalloc(&enc.p, bytes));
  ZC_CUDA_TRY(cudaMemset(enc.p, 0, bytes));
  k_cmp_encode<<<kCmpGrid, 256>>>(nv, g->d_off, static_cast<uint32_t*>(sorted.p),
                                  static_cast<uint64_t*>(coff.p), static_cast<uint32_t*>(enc.p));
  ZC_CUDA_TRY(cudaDeviceSynchronize());
  // place the stream like the lists
  void* host = nullptr;
  const void* dev = nullptr;
  void* hbm = nullptr;
  if (g->placement == ZC_PLACE_UVM) {
    ZC_CUDA_TRY(cudaMallocManaged(&host, bytes, cudaMemAttachGlobal));
    if (cudaMemcpy(host, enc.p, bytes, cudaMemcpyDefault) != cudaSuccess ||
        cudaMemAdvise(host, bytes, cudaMemAdviseSetReadMostly, g->device) != cudaSuccess) {
      cudaFree(host);
      set_error(std::string("compressed lists (uvm): ") + cudaGetErrorString(cudaGetLastError()));
      return ZC_ECUDA;
    }
    dev = host;
  } else {
    host = host_list_alloc(g, bytes);  // the stream, or the HBM run's host shadow
    if (!host) {
      set_error("cannot allocate host memory for the compressed lists");
      return ZC_ENOMEM;
    }
    const void* d = nullptr;
    if (cudaMemcpy(host, enc.p, bytes, cudaMemcpyDefault) != cudaSuccess ||
        (g->placement != ZC_PLACE_HBM && host_list_device_ptr(host, &d) != ZC_OK)) {
      pinned_list_free(host);
      set_error(std::string("compressed lists: ") + cudaGetErrorString(cudaGetLastError()));
      return ZC_ECUDA;
    }
    if (g->placement == ZC_PLACE_HBM) {
      hbm = enc.release();
      dev = hbm;
    } else {
      dev = d;
    }
  }
  g->h_cmp = host;
  g->d_cmp = dev;
  g->hbm_cmp = hbm;
  g->d_coff = static_cast<uint64_t*>(coff.release());
  g->cmp_bytes = total * kLineBytes;
  if (compressed_bytes) *compressed_bytes = g->cmp_bytes;
  return ZC_OK;
}

extern "C" int zc_graph_compressed_index(const zc_graph* g, uint64_t* first_line) {
  if (!g || !g->d_coff) {
    set_error(g ? "compressed lists not built" : "null graph handle");
    return ZC_ESTATE;
  }
  if (!first_line) {
    set_error("null output buffer");
    return ZC_EINVAL;
  }
  cudaSetDevice(g->device);
  ZC_CUDA_TRY(cudaMemcpy(first_line, g->d_coff, (g->nv + 1) * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost));
  return ZC_OK;
}
