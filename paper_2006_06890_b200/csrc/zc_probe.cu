// Host-link and HBM probes: the measured denominators for the roofline
// (pinned cudaMemcpy H2D peak, zero-copy streaming-read peak,
// next to the 63.0 GB/s PCIe Gen5 x16 theoretical figure).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/zcgraph.h"
#include "zc_internal.cuh"

namespace zc {
namespace {

// Streaming read: each lane loads 16 B, a warp covers 512 contiguous bytes
// (4 full 128-byte lines) per load, kU independent loads in flight per lane.
template <int kU>
__global__ void __launch_bounds__(256) k_stream_read(const uint4* __restrict__ p, uint64_t n16,
                                                     unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  uint64_t i = tid;
  for (; i + (kU - 1) * nt < n16; i += kU * nt) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint4* q = p + i + u * nt;
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(q));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += nt) {
    const uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

}  // namespace
}  // namespace zc

extern "C" int zc_link_probe(int32_t device, uint64_t bytes, int iters, double* memcpy_gbs,
                             double* zc_gbs, double* hbm_gbs) {
  using namespace zc;
  cudaSetDevice(device);
  bytes = std::max<uint64_t>(bytes / 512 * 512, 1 << 20);
  iters = std::max(iters, 1);
  void* h = nullptr;
  void* d = nullptr;
  unsigned long long* sink = nullptr;
  ZC_CUDA_TRY(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, bytes);
  ZC_CUDA_TRY(cudaMalloc(&d, bytes));
  ZC_CUDA_TRY(cudaMalloc(&sink, sizeof(unsigned long long)));
  void* hd = nullptr;
  ZC_CUDA_TRY(cudaHostGetDevicePointer(&hd, h, 0));
  cudaStream_t st;
  ZC_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  float ms = 0;
  // memcpy H2D
  ZC_CUDA_TRY(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
  cudaEventRecord(a, st);
  for (int k = 0; k < iters; ++k) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
  cudaEventRecord(b, st);
  ZC_CUDA_TRY(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  if (memcpy_gbs) *memcpy_gbs = bytes * (double)iters / (ms * 1e6);
  // zero-copy streaming read
  const uint64_t n16 = bytes / 16;
  const int grid = nsm * 8;
  k_stream_read<4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(hd), n16, sink);
  cudaEventRecord(a, st);
  for (int k = 0; k < iters; ++k)
    k_stream_read<4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(hd), n16, sink);
  cudaEventRecord(b, st);
  ZC_CUDA_TRY(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  if (zc_gbs) *zc_gbs = bytes * (double)iters / (ms * 1e6);
  // HBM streaming read (same kernel on device memory)
  k_stream_read<4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(d), n16, sink);
  cudaEventRecord(a, st);
  for (int k = 0; k < iters; ++k)
    k_stream_read<4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(d), n16, sink);
  cudaEventRecord(b, st);
  ZC_CUDA_TRY(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  if (hbm_gbs) *hbm_gbs = bytes * (double)iters / (ms * 1e6);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(st);
  cudaFree(sink);
  cudaFree(d);
  cudaFreeHost(h);
  return ZC_OK;
}
