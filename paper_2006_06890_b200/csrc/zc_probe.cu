// Host-link and HBM probes: the measured denominators for the roofline
// (pinned cudaMemcpy H2D peak, zero-copy streaming-read peak,
// next to the 63.0 GB/s PCIe Gen5 x16 theoretical figure).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>
#include <sys/mman.h>

#include <algorithm>
#include <string>

#include "../../include/zcgraph.h"
#include "../../include/zcprobe.h"
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

// Read microbenchmark (the paper's zero-copy toy kernel):
// every warp reads `chunk` contiguous bytes per request (32..512, lanes
// masked beyond it) at either consecutive (pattern 0) or pseudo-random
// (pattern 1) chunk-aligned offsets; kU requests in flight per warp.
template <int kU>
__global__ void __launch_bounds__(256) k_chunk_read(const uint32_t* __restrict__ p, uint64_t nchunks,
                                                    uint32_t chunk_words, int random,
                                                    uint64_t total_reqs,
                                                    unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (uint64_t r0 = gw * kU; r0 < total_reqs; r0 += nw * kU) {
    uint32_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t r = r0 + u;
      v[u] = 0;
      if (r < total_reqs) {
        uint64_t c = r % nchunks;
        if (random == 2) {  // one contiguous stream per warp
          const uint64_t per = (total_reqs + nw - 1) / nw;
          const uint64_t wi = r / kU / nw, lane_u = r % kU;  // r = (wi*nw + gw)*kU + u
          c = (gw * per + wi * kU + lane_u) % nchunks;
        } else if (random == 3) {  // one contiguous stream per CTA, warps interleaved
          const uint64_t wpc = blockDim.x >> 5, ncta = gridDim.x;
          const uint64_t per = (total_reqs + ncta - 1) / ncta;
          const uint64_t wi = r / kU / nw, lane_u = r % kU;
          const uint64_t wl = gw % wpc;
          c = (blockIdx.x * per + (wi * wpc + wl) * kU + lane_u) % nchunks;
        } else if (random) {
          uint64_t z = r * 0x9e3779b97f4a7c15ull;
          z ^= z >> 31;
          z *= 0xbf58476d1ce4e5b9ull;
          z ^= z >> 29;
          c = z % nchunks;
        }
        for (uint32_t w = lane; w < chunk_words; w += 32) {
          uint32_t x;
          asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];"
                       : "=r"(x) : "l"(p + c * chunk_words + w));
          v[u] ^= x;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// Bulk-copy (TMA engine, cp.async.bulk) streaming read: every CTA streams
// its own contiguous region chunk by chunk into a ring of shared-memory
// stages; one elected thread issues the copies, an mbarrier per stage
// tracks the transaction bytes.
constexpr int kBulkStages = 4;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes));
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
      "p; }"
      : "=r"(ok)
      : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))), "r"(phase));
  return ok;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

__global__ void __launch_bounds__(128) k_bulk_read(const char* __restrict__ src, uint64_t bytes,
                                                   uint32_t chunk,
                                                   unsigned long long* sink) {
  extern __shared__ __align__(128) char stage[];
  __shared__ __align__(8) uint64_t bar[kBulkStages];
  const uint64_t nchunks = bytes / chunk;
  const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const uint64_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
  if (threadIdx.x == 0)
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t acc = 0;
  if (threadIdx.x == 0) {
    uint64_t issued = c0;
    for (int s = 0; s < kBulkStages && issued < c1; ++s, ++issued) {
      mbar_expect_tx(&bar[s], chunk);
      bulk_g2s(stage + s * chunk, src + issued * chunk, chunk, &bar[s]);
    }
    uint32_t phase[kBulkStages] = {0, 0, 0, 0};
    for (uint64_t c = c0; c < c1; ++c) {
      const int s = static_cast<int>((c - c0) % kBulkStages);
      while (!mbar_try_wait(&bar[s], phase[s])) {
      }
      phase[s] ^= 1;
      acc ^= *reinterpret_cast<const uint32_t*>(stage + s * chunk);
      if (issued < c1) {
        mbar_expect_tx(&bar[s], chunk);
        bulk_g2s(stage + s * chunk, src + issued * chunk, chunk, &bar[s]);
        ++issued;
      }
    }
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

}  // namespace
}  // namespace zc

// TMA bulk-copy streaming read of `bytes` of pinned host memory in `chunk`-
// byte copies (multiple of 16, <= 48 KB), `ctas_per_sm` CTAs per SM.
extern "C" int zc_bulk_probe(int32_t device, uint64_t bytes, uint32_t chunk, int ctas_per_sm,
                             int iters, double* gbs) {
  using namespace zc;
  cudaSetDevice(device);
  if (chunk < 16 || chunk % 16 || chunk * kBulkStages > 200 * 1024) {
    set_error("chunk must be a multiple of 16 with 4 stages fitting in shared memory");
    return ZC_EINVAL;
  }
  bytes = std::max<uint64_t>(bytes / chunk * chunk, chunk);
  void* h = nullptr;
  ZC_CUDA_TRY(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, bytes);
  void* d = nullptr;
  ZC_CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
  unsigned long long* sink = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&sink, sizeof(unsigned long long)));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const size_t smem = static_cast<size_t>(chunk) * kBulkStages;
  ZC_CUDA_TRY(cudaFuncSetAttribute(k_bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  const int grid = nsm * std::max(1, ctas_per_sm);
  k_bulk_read<<<grid, 128, smem>>>(static_cast<const char*>(d), bytes, chunk, sink);
  ZC_CUDA_TRY(cudaGetLastError());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int k = 0; k < std::max(iters, 1); ++k)
    k_bulk_read<<<grid, 128, smem>>>(static_cast<const char*>(d), bytes, chunk, sink);
  cudaEventRecord(b);
  ZC_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  *gbs = static_cast<double>(bytes) * std::max(iters, 1) / (ms * 1e6);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  cudaFreeHost(h);
  return ZC_OK;
}

namespace zc {
namespace {
// Driver VMM entry points, fetched through the runtime (no -lcuda link).
struct Vmm {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Vmm& vmm() {
  static Vmm v = [] {
    Vmm x;
    x.ok = entry("cuMemCreate", &x.create) && entry("cuMemRelease", &x.release) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemAddressFree", &x.addr_free) &&
           entry("cuMemMap", &x.map) && entry("cuMemUnmap", &x.unmap) &&
           entry("cuMemSetAccess", &x.set_access) &&
           entry("cuMemGetAllocationGranularity", &x.granularity);
    return x;
  }();
  return v;
}

// Host-NUMA-located VMM allocation mapped for the device and the CPU at one
// address (cuMemCreate with CU_MEM_LOCATION_TYPE_HOST_NUMA).
struct VmmHost {
  CUdeviceptr va = 0;
  size_t size = 0;
  CUmemGenericAllocationHandle h = 0;
};

int vmm_host_alloc(int device, int numa, size_t bytes, VmmHost* out, size_t* gran_out) {
  const Vmm& v = vmm();
  if (!v.ok) {
    set_error("driver VMM entry points unavailable");
    return ZC_ECUDA;
  }
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = numa;
  size_t gran = 0;
  if (v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS ||
      !gran) {
    set_error("cuMemGetAllocationGranularity(HOST_NUMA) failed");
    return ZC_ECUDA;
  }
  if (gran_out) *gran_out = gran;
  bytes = (bytes + gran - 1) / gran * gran;
  CUresult r = v.create(&out->h, bytes, &prop, 0);
  if (r != CUDA_SUCCESS) {
    set_error("cuMemCreate(HOST_NUMA) failed: " + std::to_string(static_cast<int>(r)));
    return ZC_ENOMEM;
  }
  r = v.reserve(&out->va, bytes, std::max<size_t>(gran, 2u << 20), 0, 0);
  if (r == CUDA_SUCCESS) r = v.map(out->va, bytes, 0, out->h, 0);
  if (r == CUDA_SUCCESS) {
    CUmemAccessDesc acc[2] = {};
    acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[0].location.id = device;
    acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
    acc[1].location.id = numa;
    acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = v.set_access(out->va, bytes, acc, 2);
  }
  if (r != CUDA_SUCCESS) {
    set_error("cuMemMap/SetAccess(HOST_NUMA) failed: " + std::to_string(static_cast<int>(r)));
    if (out->va) v.addr_free(out->va, bytes);
    v.release(out->h);
    return ZC_ECUDA;
  }
  out->size = bytes;
  return ZC_OK;
}

void vmm_host_free(VmmHost* a) {
  const Vmm& v = vmm();
  if (!a->va) return;
  v.unmap(a->va, a->size);
  v.addr_free(a->va, a->size);
  v.release(a->h);
  a->va = 0;
}
}  // namespace
}  // namespace zc

// Granularity (bytes) of host-NUMA VMM allocations, 0 when unsupported.
extern "C" int zc_vmm_host_probe(int32_t device, uint64_t bytes, uint64_t* granularity) {
  using namespace zc;
  cudaSetDevice(device);
  cudaFree(nullptr);
  VmmHost a;
  size_t g = 0;
  const int rc = vmm_host_alloc(device, 0, bytes, &a, &g);
  if (granularity) *granularity = g;
  if (rc == ZC_OK) {
    memset(reinterpret_cast<void*>(a.va), 0, 4096);
    vmm_host_free(&a);
  }
  return rc;
}

// alloc: 0 = cudaHostAlloc(Mapped), 1 = THP (madvise) + cudaHostRegister,
// 2 = device memory, 3 = host-NUMA VMM allocation (cuMemCreate),
// 4 = hugetlbfs 2 MB pages (MAP_HUGETLB) + cudaHostRegister,
// 5 = cudaMallocManaged preferred on the CPU, accessed-by the device.
// Returns GB/s of useful bytes in *gbs.
extern "C" int zc_read_probe(int32_t device, uint64_t bytes, int pattern, uint32_t chunk_bytes,
                             int alloc, int iters, double* gbs) {
  using namespace zc;
  cudaSetDevice(device);
  if (chunk_bytes < 4 || chunk_bytes % 4 || chunk_bytes > 4096) {
    set_error("chunk_bytes must be a multiple of 4 in [4, 4096]");
    return ZC_EINVAL;
  }
  bytes = std::max<uint64_t>(bytes / 4096 * 4096, 1 << 22);
  void* h = nullptr;
  const void* dp = nullptr;
  bool registered = false;
  VmmHost vh;
  void* managed = nullptr;
  if (alloc == 0) {
    ZC_CUDA_TRY(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 1, bytes);
    void* d = nullptr;
    ZC_CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
    dp = d;
  } else if (alloc == 1) {
    const size_t huge = 2u << 20;
    bytes = (bytes + huge - 1) / huge * huge;
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (m == MAP_FAILED) {
      set_error("mmap failed");
      return ZC_ENOMEM;
    }
    madvise(m, bytes, MADV_HUGEPAGE);
    memset(m, 1, bytes);
    h = m;
    ZC_CUDA_TRY(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
    registered = true;
    void* d = nullptr;
    ZC_CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
    dp = d;
  } else if (alloc == 3) {
    const int rc = vmm_host_alloc(device, 0, bytes, &vh, nullptr);
    if (rc != ZC_OK) return rc;
    memset(reinterpret_cast<void*>(vh.va), 1, bytes);
    dp = reinterpret_cast<const void*>(vh.va);
  } else if (alloc == 4) {
    const size_t huge = 2u << 20;
    bytes = (bytes + huge - 1) / huge * huge;
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (m == MAP_FAILED) {
      set_error("mmap(MAP_HUGETLB) failed (no reserved hugepages?)");
      return ZC_ENOMEM;
    }
    memset(m, 1, bytes);
    h = m;
    ZC_CUDA_TRY(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
    registered = true;
    void* d = nullptr;
    ZC_CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
    dp = d;
  } else if (alloc == 5) {
    void* m = nullptr;
    ZC_CUDA_TRY(cudaMallocManaged(&m, bytes));
    cudaMemLocation cpu = {};
    cpu.type = cudaMemLocationTypeHost;
    cudaMemLocation gpu = {};
    gpu.type = cudaMemLocationTypeDevice;
    gpu.id = device;
    ZC_CUDA_TRY(cudaMemAdvise(m, bytes, cudaMemAdviseSetPreferredLocation, cpu));
    ZC_CUDA_TRY(cudaMemAdvise(m, bytes, cudaMemAdviseSetAccessedBy, gpu));
    memset(m, 1, bytes);
    managed = m;
    dp = m;
  } else {
    void* d = nullptr;
    ZC_CUDA_TRY(cudaMalloc(&d, bytes));
    ZC_CUDA_TRY(cudaMemset(d, 1, bytes));
    dp = d;
  }
  unsigned long long* sink = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&sink, sizeof(unsigned long long)));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const uint64_t nchunks = bytes / chunk_bytes;
  const uint64_t reqs = nchunks;  // one pass worth of requests
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = nsm * 8;
  k_chunk_read<4><<<grid, 256>>>(static_cast<const uint32_t*>(dp), nchunks, chunk_bytes / 4,
                                 pattern, reqs, sink);
  cudaEventRecord(a);
  for (int k = 0; k < std::max(iters, 1); ++k)
    k_chunk_read<4><<<grid, 256>>>(static_cast<const uint32_t*>(dp), nchunks, chunk_bytes / 4,
                                   pattern, reqs, sink);
  cudaEventRecord(b);
  ZC_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  *gbs = static_cast<double>(reqs) * chunk_bytes * std::max(iters, 1) / (ms * 1e6);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (alloc == 0) cudaFreeHost(h);
  else if (alloc == 1 || alloc == 4) {
    if (registered) cudaHostUnregister(h);
    munmap(h, bytes);
  } else if (alloc == 3) vmm_host_free(&vh);
  else if (alloc == 5) cudaFree(managed);
  else cudaFree(const_cast<void*>(dp));
  return ZC_OK;
}

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

// Pinned-allocation cost (the compressed streams' build pins ~6 GB twice):
// mode 0 cudaHostAlloc(Mapped|Portable); 1 mmap + MADV_HUGEPAGE + parallel
// first touch + cudaHostRegister; 2 the same without huge pages; 3 mmap +
// MADV_HUGEPAGE + cudaHostRegister with no prefault.  *alloc_s covers the
// mapping and first touch, *register_s the registration (mode 0: all in
// alloc_s); the buffer is freed before returning.
#include <chrono>
#include <thread>
#include <vector>
extern "C" int zc_pin_probe(uint64_t bytes, int mode, int threads, double* alloc_s,
                            double* register_s) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  *alloc_s = *register_s = 0;
  const auto t0 = clk::now();
  if (mode == 0) {
    void* p = nullptr;
    ZC_CUDA_TRY(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    *alloc_s = secs(t0, clk::now());
    cudaFreeHost(p);
    return ZC_OK;
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) {
    zc::set_error("mmap failed");
    return ZC_ENOMEM;
  }
  if (mode != 2) madvise(p, bytes, MADV_HUGEPAGE);
  if (mode != 3) {
    const int nt = std::max(1, threads);
    std::vector<std::thread> th;
    const uint64_t chunk = (bytes / nt + 4095) & ~4095ull;
    for (int k = 0; k < nt; ++k)
      th.emplace_back([=] {
        char* b = static_cast<char*>(p);
        for (uint64_t o = k * chunk; o < std::min<uint64_t>(bytes, (k + 1) * chunk); o += 4096)
          b[o] = 0;
      });
    for (auto& t : th) t.join();
  }
  const auto t1 = clk::now();
  *alloc_s = secs(t0, t1);
  const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  *register_s = secs(t1, clk::now());
  if (e == cudaSuccess) cudaHostUnregister(p);
  munmap(p, bytes);
  if (e != cudaSuccess) {
    zc::set_error(std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    return ZC_ECUDA;
  }
  return ZC_OK;
}

// Gather roofline of the HBM control run: its per-edge visited-bitmap probe
// is a random 4-byte read of a V/8-byte bitmap (16 MB at K27, L2-resident).
// Every thread issues `per` independent random word loads (counter-hashed
// indices) into a `words`-word device array and folds them into a sink.
// mode 0: plain loads; 1: plain loads + atomicOr on 1/16 of them (the claims).
__global__ void __launch_bounds__(256) k_gather_probe(uint32_t* __restrict__ bm, uint64_t words,
                                                      uint32_t per, int mode,
                                                      unsigned long long* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  uint64_t h = t * 0x9e3779b97f4a7c15ull + 1;
  for (uint32_t i = 0; i < per; i += 8) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h ^= h >> 33;
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 29;
      v[u] = bm[h % words];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += v[u];
      if (mode == 1 && ((h >> (u * 4)) & 15) == 0) atomicOr(bm + ((h >> 7) % words), 1u << u);
    }
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

extern "C" int zc_gather_probe(int32_t device, uint64_t bytes, int mode, double* gloads_per_s) {
  using namespace zc;
  cudaSetDevice(device);
  const uint64_t words = std::max<uint64_t>(bytes / 4, 1024);
  uint32_t* bm = nullptr;
  unsigned long long* sink = nullptr;
  ZC_CUDA_TRY(cudaMalloc(&bm, words * 4));
  ZC_CUDA_TRY(cudaMemset(bm, 0, words * 4));
  ZC_CUDA_TRY(cudaMalloc(&sink, sizeof(*sink)));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const int grid = nsm * 8;
  const uint32_t per = 512;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather_probe<<<grid, 256>>>(bm, words, per, mode, sink);  // warm L2
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_gather_probe<<<grid, 256>>>(bm, words, per, mode, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(bm);
  cudaFree(sink);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) {
    set_error(std::string("gather probe: ") + cudaGetErrorString(e));
    return ZC_ECUDA;
  }
  *gloads_per_s = 5.0 * grid * 256.0 * per / (ms * 1e-3) / 1e9;
  return ZC_OK;
}
