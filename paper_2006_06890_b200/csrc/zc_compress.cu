// Delta-compressed lists: an optional B200-native host-store format.
//
// Zero-copy traversal is bound by the host link (51.5 GB/s for SM-side
// reads, profiles/r01_tma_bulk_probe.txt); BFS / CC / PageRank results do not
// depend on the order inside a list, so the lists can be sorted and stored
// delta-encoded to move fewer bytes over PCIe.  Format (per list of degree d,
// sorted ascending):
//   blocks of kCmpBlock = 128 elements; block = u32 base (first element)
//   followed by the block's 127 (or count-1) deltas at the list's width w
//   bits, packed little-endian from bit 32, padded to a 4-byte word;
//   full blocks are cmp_full_bytes(w) long, the last block exactly as long
//   as its count needs.
// Per-vertex byte offset (u64[V+1]) and width (u8[V]) live in HBM next to the
// CSR offsets; the stream itself lives in the handle's placement.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "zc_graph.cuh"
#include "zc_internal.cuh"

namespace zc {
namespace {

__global__ void k_cmp_sizes(uint64_t nv, const uint64_t* off, const uint32_t* e, uint8_t* width,
                            uint32_t* bytes) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], d = off[v + 1] - s;
    uint32_t mx = 0;
    for (uint64_t k = 1 + lane; k < d; k += 32) mx = max(mx, e[s + k] - e[s + k - 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      const uint32_t w = mx ? 32 - __clz(mx) : 0;
      width[v] = static_cast<uint8_t>(w);
      bytes[v] = static_cast<uint32_t>(cmp_list_bytes(w, d));
    }
  }
}

// Warp per list, lane per block: base word, then the deltas bit-packed.
__global__ void k_cmp_encode(uint64_t nv, const uint64_t* off, const uint32_t* e,
                             const uint8_t* width, const uint64_t* coff, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = gw; v < nv; v += nw) {
    const uint64_t s = off[v], d = off[v + 1] - s;
    if (!d) continue;
    const uint32_t w = width[v];
    const uint64_t nb = (d + kCmpBlock - 1) / kCmpBlock;
    for (uint64_t b = lane; b < nb; b += 32) {
      uint32_t* dst = out + (coff[v] + b * cmp_full_bytes(w)) / 4;
      const uint64_t e0 = s + b * kCmpBlock;
      const uint64_t rem = d - b * kCmpBlock;
      const uint64_t cnt = rem < kCmpBlock ? rem : kCmpBlock;
      dst[0] = e[e0];
      uint64_t acc = 0;
      uint32_t nbits = 0, word = 1;
      for (uint64_t i = 1; i < cnt; ++i) {
        acc |= static_cast<uint64_t>(e[e0 + i] - e[e0 + i - 1]) << nbits;
        nbits += w;
        if (nbits >= 32) {
          dst[word++] = static_cast<uint32_t>(acc);
          acc >>= 32;
          nbits -= 32;
        }
      }
      if (nbits) dst[word] = static_cast<uint32_t>(acc);
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
  } sorted, sizes, tmp, enc, cw, coff;
  ZC_CUDA_TRY(cudaMalloc(&sorted.p, std::max<uint64_t>(ne, 1) * 4));
  ZC_CUDA_TRY(cudaMemcpy(sorted.p, g->h_edges, ne * 4, cudaMemcpyDefault));
  const int rc = sort_lists_device(4, nv, g->d_off, g->h_off, sorted.p);
  if (rc) return rc;
  ZC_CUDA_TRY(cudaMalloc(&cw.p, std::max<uint64_t>(nv, 1)));
  ZC_CUDA_TRY(cudaMalloc(&coff.p, (nv + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&sizes.p, std::max<uint64_t>(nv, 1) * sizeof(uint32_t)));
  k_cmp_sizes<<<kCmpGrid, 256>>>(nv, g->d_off, static_cast<uint32_t*>(sorted.p),
                                 static_cast<uint8_t*>(cw.p), static_cast<uint32_t*>(sizes.p));
  const size_t tb = scan_tmp_bytes(nv);
  ZC_CUDA_TRY(cudaMalloc(&tmp.p, tb));
  ZC_CUDA_TRY(scan_u32_to_u64(static_cast<uint32_t*>(sizes.p), static_cast<uint64_t*>(coff.p), nv,
                              tmp.p, tb, 0));
  uint64_t total = 0;
  ZC_CUDA_TRY(cudaMemcpy(&total, static_cast<uint64_t*>(coff.p) + nv, sizeof(total),
                         cudaMemcpyDeviceToHost));
  const size_t bytes = std::max<uint64_t>(total, 4) + 16;  // + slack for the decoder
  ZC_CUDA_TRY(cudaMalloc(&enc.p, bytes));
  ZC_CUDA_TRY(cudaMemset(enc.p, 0, bytes));
  k_cmp_encode<<<kCmpGrid, 256>>>(nv, g->d_off, static_cast<uint32_t*>(sorted.p),
                                  static_cast<uint8_t*>(cw.p), static_cast<uint64_t*>(coff.p),
                                  static_cast<uint32_t*>(enc.p));
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
  g->d_cw = static_cast<uint8_t*>(cw.release());
  g->d_coff = static_cast<uint64_t*>(coff.release());
  g->cmp_bytes = total;
  if (compressed_bytes) *compressed_bytes = total;
  return ZC_OK;
}
