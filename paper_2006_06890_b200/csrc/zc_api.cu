// Host graph store + C ABI (include/zcgraph.h).
//
// One handle = one CSR graph resident on one GPU:
//   * edge / weight lists: pinned mapped host memory read zero-copy by the
//     kernels (EMOGI), or managed memory with
//     cudaMemAdviseSetReadMostly (the paper's UVM baseline), or
//     plain HBM (control run);
//   * offsets and every per-vertex array: HBM, allocated once at create and
//     reused by every traversal (no allocation on the run path).
// The traversal drivers restate traversal.py:98-179 as a host loop over
// levels: expand (zc_kernels.cu) -> compact -> read two counters.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <dirent.h>
#include <immintrin.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <mutex>
#include <unordered_map>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zcgraph.h"
#include "zc_graph.cuh"
#include "zc_internal.cuh"

namespace zc {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

// Run fn(lo, hi) over [0, n) on all host cores but `spare`.
// `serial_below`: item counts under it run on the calling thread.
template <typename F>
static void parallel_for(uint64_t n, F fn, unsigned spare = 0, uint64_t serial_below = 1u << 16) {
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  unsigned nt = hc > spare + 1 ? hc - spare : 1;
  if (n < serial_below) nt = 1;
  if (nt == 1) {
    fn(uint64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const uint64_t lo = std::min(n, t * chunk), hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back(fn, lo, hi);
  }
  for (auto& x : th) x.join();
}

// Copy n elements of width sw from src into dst of width dw.
static void convert_copy(void* dst, uint32_t dw, const void* src, uint32_t sw, uint64_t n) {
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    if (dw == sw) {
      memcpy(static_cast<char*>(dst) + lo * dw, static_cast<const char*>(src) + lo * sw,
             (hi - lo) * dw);
      return;
    }
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t x = sw == 8 ? static_cast<const uint64_t*>(src)[i]
                           : static_cast<const uint32_t*>(src)[i];
      if (dw == 8) static_cast<uint64_t*>(dst)[i] = x;
      else static_cast<uint32_t*>(dst)[i] = static_cast<uint32_t>(x);
    }
  });
}

void tune_params(ExpandArgs* a, const zc_graph* g) {
  // the HBM control run is bound by its state gathers, not by list loads:
  // occupancy beats loads in flight there (K27: U=4 115.7 GTEPS, U=8 102.2)
  a->unroll = g->tune.unroll ? g->tune.unroll : g->placement == ZC_PLACE_HBM ? 4 : 0;
  a->ctas_per_sm = g->tune.ctas;
  a->chunk_sched = g->tune.sched;
  a->carveout = g->tune.carveout;
  a->ld = g->tune.ld;
  a->uf_sample = g->tune.uf_sample ? static_cast<uint32_t>(g->tune.uf_sample) : kUfSample;
}

// ---------------------------------------------------------- pinned lists
// Zero-copy lists are read by the GPU across PCIe: on a multi-socket host
// they belong on the GPU's own NUMA node (the node is
// ignored with ZC_NUMA=0).  See pinned_list_alloc.
static std::mutex g_map_mu;
static std::unordered_map<void*, size_t> g_mapped;  // our registered mappings

static int gpu_numa_node(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = static_cast<char>(tolower(*c));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  int nodes = 0;
  if (DIR* d = opendir("/sys/devices/system/node")) {
    while (dirent* e = readdir(d))
      if (!strncmp(e->d_name, "node", 4) && isdigit(static_cast<unsigned char>(e->d_name[4])))
        ++nodes;
    closedir(d);
  }
  return nodes > 1 ? node : -1;
}

// Pinned mapped host memory, fast.  cudaHostAlloc pins at ~1.5 GB/s (4.35 s
// for a 6 GB line stream, profiles/r02_pin_probe.txt); an anonymous mapping
// with transparent huge pages, first-touched by 8 threads (the kernel zeroes
// 2 MB pages concurrently) and then cudaHostRegister'ed, takes 0.27 s and
// streams over the link like cudaHostAlloc memory (r01_alloc_probe.txt).  On
// a multi-node host the mapping is bound to the GPU's NUMA node first.
// Small buffers (< 64 MB) and any failure take cudaHostAlloc.
static void prefault(void* p, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = std::min(8u, hw);
  const size_t chunk = (bytes / nt + 4095) & ~static_cast<size_t>(4095);
  std::vector<std::thread> th;
  for (unsigned k = 0; k < nt; ++k)
    th.emplace_back([=] {
      volatile char* b = static_cast<char*>(p);
      for (size_t o = k * chunk; o < std::min(bytes, (k + 1) * chunk); o += 4096) b[o] = 0;
    });
  for (auto& t : th) t.join();
}

static bool numa_disabled();

HostMap pinned_list_map(int device, size_t bytes) {
  HostMap m;
  bytes = std::max<size_t>(bytes, 1);
  if (bytes < (64ull << 20)) return m;
  const int node = numa_disabled() ? -1 : gpu_numa_node(device);
  // a 2 MiB-aligned mapping of whole 2 MiB pages: an unaligned one is only
  // partly backed by huge pages, and registering 4 KiB pages is slow (a
  // 6.2 GB stream took 0.4-0.9 s in cudaHostRegister instead of ~0.15 s)
  constexpr size_t kHuge = 2ull << 20;
  bytes = (bytes + kHuge - 1) & ~(kHuge - 1);
  void* raw = mmap(nullptr, bytes + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS,
                   -1, 0);
  if (raw == MAP_FAILED) return m;
  const uintptr_t r = reinterpret_cast<uintptr_t>(raw);
  const uintptr_t a = (r + kHuge - 1) & ~(kHuge - 1);
  if (a > r) munmap(raw, a - r);
  if (r + kHuge > a) munmap(reinterpret_cast<void*>(a + bytes), r + kHuge - a);
  void* p = reinterpret_cast<void*>(a);
  if (node >= 0 && node < 64) {
    unsigned long mask = 1ul << node;
    if (syscall(SYS_mbind, p, bytes, 2 /* MPOL_BIND */, &mask, 64, 0) != 0) {
      munmap(p, bytes);
      return m;
    }
  }
  madvise(p, bytes, MADV_HUGEPAGE);
  prefault(p, bytes);
  m.p = p;
  m.bytes = bytes;
  return m;
}

void pinned_list_unmap(HostMap m) {
  if (m.p) munmap(m.p, m.bytes);
}

void* pinned_list_finish(HostMap m, size_t bytes) {
  if (m.p) {
    if (cudaHostRegister(m.p, m.bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) ==
        cudaSuccess) {
      std::lock_guard<std::mutex> lk(g_map_mu);
      g_mapped[m.p] = m.bytes;
      return m.p;
    }
    cudaGetLastError();
    munmap(m.p, m.bytes);
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocMapped | cudaHostAllocPortable) !=
      cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void* pinned_list_alloc(int device, size_t bytes) {
  return pinned_list_finish(pinned_list_map(device, bytes), bytes);
}

static bool numa_disabled() {
  static const bool off = [] {
    const char* env = getenv("ZC_NUMA");
    return env && env[0] == '0';
  }();
  return off;
}

// Host-resident managed lists (ZC_PLACE_ZEROCOPY_MANAGED).  The pages stay
// in host memory (PreferredLocation = CPU) and are mapped in the GPU's page
// tables up front (AccessedBy), so the GPU reads them over PCIe exactly like
// pinned memory -- but through the UVM driver's mappings, whose large GPU
// pages keep the scattered line reads of sparse frontiers out of the
// translation misses that cap pinned memory at ~70 M random lines/s
// (profiles/r01_alloc_probe.txt: random 128 B reads over 8 GiB, 9.0 GB/s
// pinned vs 34.0 GB/s managed-on-host).  No ReadMostly: no GPU copies.
static std::unordered_map<void*, size_t> g_managed;

static void* managed_host_alloc(int device, size_t bytes) {
  void* p = nullptr;
  if (cudaMallocManaged(&p, bytes, cudaMemAttachGlobal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, cudaCpuDeviceId) !=
          cudaSuccess ||
      cudaMemAdvise(p, bytes, cudaMemAdviseSetAccessedBy, device) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p);
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_map_mu);
  g_managed[p] = bytes;
  return p;
}

void* host_list_alloc(const zc_graph* g, size_t bytes) {
  if (g->placement == ZC_PLACE_ZEROCOPY_MANAGED) return managed_host_alloc(g->device, bytes);
  return pinned_list_alloc(g->device, bytes);
}

int host_list_device_ptr(void* p, const void** d) {
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_managed.count(p)) {
      *d = p;
      return ZC_OK;
    }
  }
  void* dp = nullptr;
  ZC_CUDA_TRY(cudaHostGetDevicePointer(&dp, p, 0));
  *d = dp;
  return ZC_OK;
}

void pinned_list_free(void* p) {
  if (!p) return;
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto m = g_managed.find(p);
    if (m != g_managed.end()) {
      g_managed.erase(m);
      cudaFree(p);
      return;
    }
    auto it = g_mapped.find(p);
    if (it != g_mapped.end()) {
      bytes = it->second;
      g_mapped.erase(it);
    }
  }
  if (bytes) {
    cudaHostUnregister(p);
    munmap(p, bytes);
  } else {
    cudaFreeHost(p);
  }
}

// int64 BFS levels from the narrowed download (0xff = unreached -> -1,
// traversal.py:22); the widen of one result runs while the caller's thread
// drives the next traversal's level loop.
// AVX2 body: 8 levels per step, streamed (non-temporal) stores so the 8 B
// per vertex written do not also cost a read-for-ownership of host memory
// the GPU is streaming lists from.
__attribute__((target("avx2"))) static void widen_levels_avx2(const uint8_t* src, int64_t* out,
                                                              uint64_t lo, uint64_t hi) {
  uint64_t i = lo;
  for (; i < hi && (reinterpret_cast<uintptr_t>(out + i) & 31); ++i)
    out[i] = src[i] == 0xffu ? -1ll : static_cast<int64_t>(src[i]);
  const __m256i ff = _mm256_set1_epi64x(0xff);
  for (; i + 8 <= hi; i += 8) {
    uint64_t b8;
    memcpy(&b8, src + i, 8);
    const __m128i b = _mm_cvtsi64_si128(static_cast<long long>(b8));
    __m256i lo4 = _mm256_cvtepu8_epi64(b);
    __m256i hi4 = _mm256_cvtepu8_epi64(_mm_srli_si128(b, 4));
    // 0xff (unreached) -> -1: OR in the all-ones mask of the equal lanes
    lo4 = _mm256_or_si256(lo4, _mm256_cmpeq_epi64(lo4, ff));
    hi4 = _mm256_or_si256(hi4, _mm256_cmpeq_epi64(hi4, ff));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i), lo4);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i + 4), hi4);
  }
  for (; i < hi; ++i) out[i] = src[i] == 0xffu ? -1ll : static_cast<int64_t>(src[i]);
  _mm_sfence();
}

static void widen_levels(const uint8_t* src, int64_t* out, uint64_t n, bool overlapped,
                         int threads = 0) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  // Overlapped (pipelined) widens run on four threads: they share the host's
  // memory bandwidth with the next traversal's zero-copy reads -- more
  // threads finish sooner but slow the traversal (tools/e2e_probe.py: 2 / 4 /
  // 16 threads: e2e 39.6 / 40.9 / 40.0 GTEPS).  A blocking call's widen uses
  // all cores but two.
  static const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  static const unsigned spare_overlap = hc > 4 ? hc - 4 : 0u;
  unsigned spare = overlapped ? spare_overlap : 2u;
  if (threads > 0) spare = hc > static_cast<unsigned>(threads) ? hc - threads : 0u;
  parallel_for(
      n,
      [&](uint64_t lo, uint64_t hi) {
        if (avx2) {
          widen_levels_avx2(src, out, lo, hi);
          return;
        }
        for (uint64_t i = lo; i < hi; ++i)
          out[i] = src[i] == 0xffu ? -1ll : static_cast<int64_t>(src[i]);
      },
      spare);
}

static double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

void build_start(zc_graph* g) { g->build_t = now_ms(); }

void build_mark(zc_graph* g, const char* phase) {
  cudaDeviceSynchronize();
  const double t = now_ms();
  g->build_log.emplace_back(phase, t - g->build_t);
  g->build_t = t;
}

}  // namespace zc

using namespace zc;

namespace {
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

void zc::free_graph(zc_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  for (auto& t : g->widen_th)
    if (t.joinable()) t.join();
  for (auto* p : g->h_stage) pinned_list_free(p);
  if (g->stream) cudaStreamSynchronize(g->stream);
  if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);
  auto free_list = [&](void*& h, bool registered, void*& hbm) {
    if (h) {
      if (registered) cudaHostUnregister(h);
      else if (g->placement == ZC_PLACE_UVM) cudaFree(h);
      else pinned_list_free(h);
    }
    h = nullptr;
    if (hbm) cudaFree(hbm);
    hbm = nullptr;
  };
  free_list(g->h_edges, g->edges_registered, g->hbm_edges);
  free_list(g->h_weights, g->weights_registered, g->hbm_weights);
  free_list(g->h_pairs, false, g->hbm_pairs);
  free_list(g->h_cmp, false, g->hbm_cmp);
  if (!g->in_alias) {
    free_list(g->h_cmp_in, false, g->hbm_cmp_in);
    cudaFree(g->d_cpos_in);
    cudaFree(g->d_in_off);
  }
  cudaFree(g->d_cand);
  cudaFree(g->d_fbits);
  cudaFree(g->d_hasin);
  cudaFree(g->d_cpos);
  pinned_list_free(g->h_off);
  cudaFree(g->d_off);
  cudaFree(g->d_state);
  cudaFree(g->d_flags);
  cudaFree(g->d_visited);
  for (int i = 0; i < 2; ++i) {
    cudaFree(g->d_front[i]);
    cudaFree(g->d_fval[i]);
    cudaFree(g->d_fs[i]);
    cudaFree(g->d_fd[i]);
  }
  cudaFree(g->d_tiles);
  cudaFree(g->d_big_s);
  cudaFree(g->d_big_e);
  cudaFree(g->d_big_val);
  cudaFree(g->d_big_prefix);
  cudaFree(g->d_ctr);
  cudaFree(g->d_part_lo);
  if (g->loop.exec) cudaGraphExecDestroy(g->loop.exec);
  if (g->loop.graph) cudaGraphDestroy(g->loop.graph);
  cudaFree(g->d_log);
  for (void* p : g->ipc_opened_sent) cudaIpcCloseMemHandle(p);
  cudaFree(g->d_peer_sent);
  for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
  cudaFree(g->d_mine);
  cudaFree(g->d_peers);
  cudaFree(g->d_sent);
  cudaFree(g->d_lbest);
  cudaFree(g->d_wcnt);
  cudaFree(g->d_wpre);
  cudaFree(g->d_scan_tmp);
  if (g->h_ctr) cudaFreeHost(g->h_ctr);
  if (g->h_small) cudaFreeHost(g->h_small);
  for (auto& e : g->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : g->iter_ev) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    cudaFree(g->d_outbuf[i]);
    if (g->out_ready[i]) cudaEventDestroy(g->out_ready[i]);
    if (g->out_done[i]) cudaEventDestroy(g->out_done[i]);
  }
  if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

namespace {
// Host-side invariant check (csr.py:80-105) on the caller's arrays.
int validate_desc(const zc_graph_desc* d, bool* negative_weight, uint64_t dest_limit = 0) {
  const uint64_t nv = d->num_vertices, ne = d->num_edges;
  const uint64_t dl = dest_limit ? dest_limit : nv;  // edge destinations must be < dl
  if (d->edge_elem_bytes != 4 && d->edge_elem_bytes != 8) {
    set_error("edge_elem_bytes must be 4 or 8, got " + std::to_string(d->edge_elem_bytes));
    return ZC_EINVAL;
  }
  if (d->weight_elem_bytes != 4 && d->weight_elem_bytes != 8) {
    set_error("weight_elem_bytes must be 4 or 8, got " + std::to_string(d->weight_elem_bytes));
    return ZC_EINVAL;
  }
  if (d->src_edge_bytes != 4 && d->src_edge_bytes != 8) {
    set_error("src_edge_bytes must be 4 or 8");
    return ZC_EINVAL;
  }
  if (d->weights && d->src_weight_bytes != 4 && d->src_weight_bytes != 8) {
    set_error("src_weight_bytes must be 4 or 8");
    return ZC_EINVAL;
  }
  if (nv >= 0xffffffffull || dl >= 0xffffffffull) {
    set_error("device path supports fewer than 2^32-1 vertices");
    return ZC_EINVAL;
  }
  if (!d->offsets || (ne && !d->edges)) {
    set_error("offsets / edges must not be NULL");
    return ZC_EINVAL;
  }
  if (!placement_valid(d->placement)) {
    set_error("unknown placement");
    return ZC_EINVAL;
  }
  *negative_weight = false;
  if (d->flags & ZC_F_NO_VALIDATE) return ZC_OK;
  const int64_t* off = d->offsets;
  if (off[0] != 0) {
    set_error("offsets[0] must be 0");
    return ZC_EINVAL;
  }
  if (static_cast<uint64_t>(off[nv]) != ne) {
    set_error("offsets[-1]=" + std::to_string(off[nv]) + " does not match num_edges=" +
              std::to_string(ne));
    return ZC_EINVAL;
  }
  std::atomic<int> bad_off{0}, bad_edge{0}, neg_w{0}, big_w{0};
  parallel_for(nv, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t v = lo; v < hi; ++v)
      if (off[v + 1] < off[v]) {
        bad_off = 1;
        return;
      }
  });
  if (bad_off) {
    set_error("offsets must be non-decreasing");
    return ZC_EINVAL;
  }
  parallel_for(ne, [&](uint64_t lo, uint64_t hi) {
    int b = 0;
    if (d->src_edge_bytes == 8) {
      const int64_t* e = static_cast<const int64_t*>(d->edges);
      for (uint64_t i = lo; i < hi; ++i) b |= (e[i] < 0) | (static_cast<uint64_t>(e[i]) >= dl);
    } else {
      const uint32_t* e = static_cast<const uint32_t*>(d->edges);
      for (uint64_t i = lo; i < hi; ++i) b |= (e[i] >= dl);
    }
    if (b) bad_edge = 1;
    if (d->weights) {
      int n = 0, big = 0;
      if (d->src_weight_bytes == 8) {
        const int64_t* w = static_cast<const int64_t*>(d->weights);
        for (uint64_t i = lo; i < hi; ++i) {
          n |= w[i] < 0;
          big |= (d->weight_elem_bytes == 4) & (w[i] > 0xffffffffll);
        }
      }
      if (n) neg_w = 1;
      if (big) big_w = 1;
    }
  });
  if (bad_edge) {
    set_error("edge destination out of range");
    return ZC_EINVAL;
  }
  if (big_w) {
    set_error("weight does not fit the 4-byte weight element width");
    return ZC_EINVAL;
  }
  *negative_weight = neg_w != 0;
  return ZC_OK;
}

// Place one list (edges or weights) according to the handle's placement.
int place_list(zc_graph* g, const void* src, uint32_t sw, uint32_t dw, uint64_t n, void** h,
               bool* registered, const void** dptr, void** hbm) {
  const size_t bytes = std::max<size_t>(n * dw, kLineBytes);
  *registered = false;
  if (g->placement == ZC_PLACE_ZEROCOPY && (g->flags & ZC_F_REGISTER)) {
    if (sw != dw || (reinterpret_cast<uintptr_t>(src) % kLineBytes)) {
      set_error("ZC_F_REGISTER needs 128-byte aligned lists already at the element width");
      return ZC_EINVAL;
    }
    void* p = const_cast<void*>(src);
    cudaError_t e = cudaHostRegister(p, n * dw, cudaHostRegisterMapped | cudaHostRegisterReadOnly);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ZC_CUDA_TRY(cudaHostRegister(p, n * dw, cudaHostRegisterMapped));
    }
    *h = p;
    *registered = true;
    void* d = nullptr;
    ZC_CUDA_TRY(cudaHostGetDevicePointer(&d, p, 0));
    *dptr = d;
    return ZC_OK;
  }
  if (g->placement == ZC_PLACE_UVM) {
    void* p = nullptr;
    ZC_CUDA_TRY(cudaMallocManaged(&p, bytes, cudaMemAttachGlobal));
    *h = p;
    if (src && n) convert_copy(p, dw, src, sw, n);
    ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseSetReadMostly, g->device));
    *dptr = p;
    return ZC_OK;
  }
  // host buffer read in place (zero-copy list), or the host shadow of HBM
  void* p = host_list_alloc(g, bytes);
  if (!p) {
    set_error("cannot allocate host memory for a list");
    return ZC_ENOMEM;
  }
  *h = p;
  if (src && n) convert_copy(p, dw, src, sw, n);
  if (g->placement == ZC_PLACE_HBM) {
    ZC_CUDA_TRY(cudaMalloc(hbm, bytes));
    ZC_CUDA_TRY(cudaMemcpy(*hbm, p, n * dw, cudaMemcpyHostToDevice));
    *dptr = *hbm;
    return ZC_OK;
  }
  return host_list_device_ptr(p, dptr);
}

}  // namespace

int zc::alloc_state(zc_graph* g) {
  const uint64_t nv = g->nv;
  const uint64_t n1 = std::max<uint64_t>(nv, 1);
  g->ntiles = std::max<uint64_t>((nv + kTileVerts - 1) / kTileVerts, 1);
  g->vpad = g->ntiles * kTileVerts;
  ZC_CUDA_TRY(cudaMalloc(&g->d_off, (nv + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMemcpy(g->d_off, g->h_off, (nv + 1) * sizeof(uint64_t),
                         cudaMemcpyHostToDevice));
  ZC_CUDA_TRY(cudaMalloc(&g->d_state, n1 * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_flags, g->vpad));
  ZC_CUDA_TRY(cudaMalloc(&g->d_visited, g->vpad / 8));
  ZC_CUDA_TRY(cudaMemset(g->d_flags, 0, g->vpad));
  for (int i = 0; i < 2; ++i) {
    ZC_CUDA_TRY(cudaMalloc(&g->d_front[i], n1 * sizeof(uint32_t)));
    ZC_CUDA_TRY(cudaMalloc(&g->d_fval[i], n1 * sizeof(uint64_t)));
    ZC_CUDA_TRY(cudaMalloc(&g->d_fs[i], n1 * sizeof(uint64_t)));
    ZC_CUDA_TRY(cudaMalloc(&g->d_fd[i], n1 * sizeof(uint32_t)));
  }
  ZC_CUDA_TRY(cudaMalloc(&g->d_tiles, g->ntiles * sizeof(uint32_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_big_s, n1 * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_big_e, n1 * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_big_val, n1 * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_big_prefix, (n1 + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_ctr, kCtrCount * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_log, 4 * kLogCap * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_wcnt, n1 * sizeof(uint32_t)));
  ZC_CUDA_TRY(cudaMalloc(&g->d_wpre, (n1 + 1) * sizeof(uint64_t)));
  g->scan_tmp_bytes = scan_tmp_bytes(n1);
  ZC_CUDA_TRY(cudaMalloc(&g->d_scan_tmp, g->scan_tmp_bytes));
  ZC_CUDA_TRY(cudaHostAlloc(&g->h_ctr, kCtrCount * sizeof(uint64_t), cudaHostAllocDefault));
  ZC_CUDA_TRY(cudaHostAlloc(&g->h_small, 4 * sizeof(uint64_t), cudaHostAllocDefault));
  ZC_CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  for (auto& e : g->ev) ZC_CUDA_TRY(cudaEventCreate(&e));
  cudaDeviceProp prop;
  ZC_CUDA_TRY(cudaGetDeviceProperties(&prop, g->device));
  g->num_sms = prop.multiProcessorCount;
  return ZC_OK;
}

int zc::init_partition(zc_graph* g, const zc_part_info* info) {
  DeviceGuard dg(g->device);
  g->nparts = info->nparts;
  g->part = info->part;
  g->global_nv = info->global_vertices;
  g->lo = info->bounds[info->part];
  g->stride = info->stride;
  ZC_CUDA_TRY(cudaMalloc(&g->d_part_lo, (info->nparts + 1) * sizeof(uint64_t)));
  ZC_CUDA_TRY(cudaMemcpy(g->d_part_lo, info->bounds, (info->nparts + 1) * sizeof(uint64_t),
                         cudaMemcpyHostToDevice));
  return ZC_OK;
}

int zc::finish_create(zc_graph* g) {
  if (g->placement == ZC_PLACE_UVM && (g->flags & ZC_F_UVM_PREFETCH) && g->ne) {
    ZC_CUDA_TRY(cudaMemPrefetchAsync(g->h_edges, g->ne * g->eb, g->device, g->stream));
    if (g->h_weights)
      ZC_CUDA_TRY(cudaMemPrefetchAsync(g->h_weights, g->ne * g->wb, g->device, g->stream));
  }
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  return ZC_OK;
}

int zc::adopt_device_list(zc_graph* g, void* d_src, uint32_t w, uint64_t n, void** h,
                          const void** dptr, void** hbm) {
  const size_t bytes = std::max<size_t>(n * w, kLineBytes);
  if (g->placement == ZC_PLACE_UVM) {
    void* p = nullptr;
    ZC_CUDA_TRY(cudaMallocManaged(&p, bytes, cudaMemAttachGlobal));
    *h = p;
    ZC_CUDA_TRY(cudaMemcpy(p, d_src, n * w, cudaMemcpyDefault));
    ZC_CUDA_TRY(cudaFree(d_src));
    // start cold: pages resident on the host, read-mostly on the GPU
    ZC_CUDA_TRY(cudaMemPrefetchAsync(p, bytes, cudaCpuDeviceId, 0));
    ZC_CUDA_TRY(cudaDeviceSynchronize());
    ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseSetReadMostly, g->device));
    *dptr = p;
    return ZC_OK;
  }
  void* p = host_list_alloc(g, bytes);
  if (!p) {
    set_error("cannot allocate host memory for a list");
    return ZC_ENOMEM;
  }
  *h = p;
  ZC_CUDA_TRY(cudaMemcpy(p, d_src, n * w, cudaMemcpyDefault));
  if (g->placement == ZC_PLACE_HBM) {
    *hbm = d_src;
    *dptr = d_src;
    return ZC_OK;
  }
  ZC_CUDA_TRY(cudaFree(d_src));
  return host_list_device_ptr(p, dptr);
}

namespace {

// Build (or reuse) the device-driven level loop of (algo, strategy): a CUDA
// graph whose conditional WHILE node repeats
//   stamp -> window counts -> scan -> sweep expansion -> stamp ->
//   compaction -> level end (log + cudaGraphSetConditional)
// with the frontier size / level read from device memory.
int build_loop_graph(zc_graph* g, int algo, int strategy, int ebytes, const ExpandArgs& base,
                     const CompactArgs& c) {
  LoopGraph& L = g->loop;
  if (L.exec && L.algo == algo && L.strategy == strategy && L.ebytes == ebytes &&
      L.unroll == base.unroll && L.ctas == base.ctas_per_sm && L.ld == base.ld &&
      L.carveout == base.carveout)
    return ZC_OK;
  if (L.exec) cudaGraphExecDestroy(L.exec);
  if (L.graph) cudaGraphDestroy(L.graph);
  L = LoopGraph{};
  cudaStream_t st = g->stream;
  ZC_CUDA_TRY(cudaGraphCreate(&L.graph, 0));
  cudaGraphConditionalHandle loop;
  ZC_CUDA_TRY(cudaGraphConditionalHandleCreate(&loop, L.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = loop;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  ZC_CUDA_TRY(cudaGraphAddNode(&node, L.graph, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  ZC_CUDA_TRY(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeRelaxed));
  ExpandArgs a = base;
  a.n = g->nv;  // sizes grids; the kernels read the live size from n_dev
  a.n_dev = g->d_ctr + kCtrCur;
  a.iter_dev = g->d_ctr + kCtrIter;
  uint64_t launches = 0;
  cudaError_t e = launch_stamp(g->d_ctr, g->d_log + 2 * kLogCap, st);
  if (e == cudaSuccess) e = launch_expand(strategy, algo, ebytes, g->wb, a, g->num_sms, st, &launches);
  if (e == cudaSuccess) e = launch_stamp(g->d_ctr, g->d_log + 3 * kLogCap, st);
  if (e == cudaSuccess) e = launch_compact(algo, c, st, &launches);
  if (e == cudaSuccess)
    e = launch_level_end(g->d_ctr, g->d_log, g->d_log + kLogCap, kLogCap, loop, st);
  cudaGraph_t captured = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(st, &captured);
  if (e != cudaSuccess || e2 != cudaSuccess) {
    set_error(std::string("level-loop capture: ") +
              cudaGetErrorString(e != cudaSuccess ? e : e2));
    return ZC_ECUDA;
  }
  ZC_CUDA_TRY(cudaGraphInstantiate(&L.exec, L.graph, 0));
  L.algo = algo;
  L.strategy = strategy;
  L.ebytes = ebytes;
  L.unroll = base.unroll;
  L.ctas = base.ctas_per_sm;
  L.ld = base.ld;
  L.carveout = base.carveout;
  L.launches_per_iter = launches + 3;
  return ZC_OK;
}

// One traversal (traversal.py:98-179) on the handle.
// Lazily created resources of the pipelined result path.
int ensure_async(zc_graph* g) {
  if (g->copy_stream) return ZC_OK;
  for (int i = 0; i < 2; ++i) {
    if (!g->d_outbuf[i] &&
        cudaMalloc(&g->d_outbuf[i], std::max<uint64_t>(g->nv, 1) * sizeof(int64_t)) !=
            cudaSuccess) {
      cudaGetLastError();
      set_error("out of device memory for the pipelined result slots");
      return ZC_ENOMEM;
    }
    if (!g->out_ready[i]) ZC_CUDA_TRY(cudaEventCreateWithFlags(&g->out_ready[i], cudaEventDisableTiming));
    if (!g->out_done[i]) ZC_CUDA_TRY(cudaEventCreateWithFlags(&g->out_done[i], cudaEventDisableTiming));
  }
  ZC_CUDA_TRY(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
  return ZC_OK;
}

int run(zc_graph* g, int algo, uint64_t src, int strategy, int64_t* out, zc_stats* stats,
        bool async = false, uint64_t nf_delta = 0) {
  const double t0 = now_ms();
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (strategy < kNaive || strategy > kDirOpt) {
    set_error("unknown access strategy " + std::to_string(strategy));
    return ZC_EINVAL;
  }
  if (strategy >= kPacked && (g->options & ZC_OPT_TRAFFIC_MODEL)) {
    set_error("the request model is defined for the reference's three strategies "
              "(naive, merged, merged-aligned), not for packed / compressed / "
              "direction-optimizing");
    return ZC_EINVAL;
  }
  if (strategy == kDirOpt && algo != kBfs) {
    set_error("direction-optimizing is a bfs strategy");
    return ZC_EINVAL;
  }
  if (strategy == kCompressed && algo == kSssp && g->has_weights && g->wb != 4) {
    set_error("compressed lists carry 4-byte weights only: use packed for 8-byte weights");
    return ZC_EINVAL;
  }
  if ((strategy == kCompressed || strategy == kDirOpt) && g->eb != 4) {
    set_error("compressed lists need 4-byte edges");
    return ZC_EINVAL;
  }
  if (algo != kCc && src >= g->nv) {  // traversal.py:93-95
    set_error("source " + std::to_string(src) + " out of range for " + std::to_string(g->nv) +
              " vertices");
    return ZC_EINVAL;
  }
  if (algo == kSssp) {  // traversal.py:133-136
    if (!g->has_weights) {
      set_error("sssp requires edge weights");
      return ZC_EINVAL;
    }
    if (g->ne && g->negative_weight) {
      set_error("sssp requires non-negative weights");
      return ZC_EINVAL;
    }
  }
  if (algo == kCc && (g->flags & ZC_F_DIRECTED)) {  // traversal.py:163-165
    set_error("connected components require an undirected graph "
              "(load with directed=False or symmetrize first)");
    return ZC_EINVAL;
  }
  if (!out && g->nv) {
    set_error("null output buffer");
    return ZC_EINVAL;
  }
  DeviceGuard dg(g->device);
  if (strategy == kCompressed && !g->d_cmp) {  // built once per handle
    const int rc = zc_graph_build_compressed(g, nullptr);
    if (rc) return rc;
  }
  if (strategy == kDirOpt && !g->d_cpos_in) {  // + the in-lists
    const int rc = zc_graph_build_in_lists(g, nullptr);
    if (rc) return rc;
  }
  // top-down steps of the direction-optimizing strategy are compressed steps
  const bool dobfs = strategy == kDirOpt;
  const int td_strategy = dobfs ? static_cast<int>(kCompressed) : strategy;
  if (async) {
    const int rc = ensure_async(g);
    if (rc) return rc;
  }
  cudaStream_t st = g->stream;
  uint64_t launches = 0;
  g->log_trav.clear();
  g->log_front.clear();
  g->log_hist.clear();
  g->log_expand_ms.clear();
  g->log_pull.clear();
  const bool model = (g->options & ZC_OPT_TRAFFIC_MODEL) != 0;

  ZC_CUDA_TRY(cudaMemsetAsync(g->d_flags, 0, g->vpad, st));
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr, 0, kCtrCount * sizeof(uint64_t), st));
  ZC_CUDA_TRY(launch_init(algo, g->d_state, g->nv, src, g->d_off, g->d_front[0], g->d_fval[0],
                          g->d_fs[0], g->d_fd[0], st, &launches));
  uint64_t n = 0, trav = 0;
  uint64_t h2d = 0;
  if (algo == kCc) {
    n = g->nv;
    trav = g->ne;
  } else {
    // state[src] = 0 (the frontier [src] was written by launch_init)
    g->h_small[1] = 0;
    const size_t sb = algo == kSssp ? 8 : 4;
    ZC_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(g->d_state) + src * sb, &g->h_small[1], sb,
                                cudaMemcpyHostToDevice, st));
    h2d += sb;
    if (algo == kBfs) {  // visited bitmap = {src}
      ZC_CUDA_TRY(cudaMemsetAsync(g->d_visited, 0, g->vpad / 8, st));
      g->h_small[2] = 1ull << (src & 31);
      ZC_CUDA_TRY(cudaMemcpyAsync(g->d_visited + (src >> 5), &g->h_small[2], sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, st));
      h2d += sizeof(uint32_t);
    }
    n = 1;
    trav = g->h_off[src + 1] - g->h_off[src];
  }
  // Frontier buffers [0] are both read by the expansion and rewritten by the
  // compaction (which only reads the marks), so the level loop has fixed
  // pointers -- the device-driven loop below is one instantiated CUDA graph.
  // SSSP over 4-byte edges and weights with a windowed raw strategy reads the
  // interleaved (dst, weight) stream (built on first use): a degree-16 list is
  // one full line instead of two half lines (U27: 0.52 -> 0.80 of the link)
  if (algo == kSssp && !model && !g->d_pairs && g->tune.pairs && g->has_weights && g->eb == 4 &&
      g->wb == 4 && !g->nparts &&
      (strategy == kMerged || strategy == kMergedAligned || strategy == kPacked)) {
    const int rc = zc_graph_build_pairs(g);
    if (rc) return rc;
  }
  const bool pairs = algo == kSssp && g->d_pairs && !model && g->tune.pairs;
  auto expand_args = [&](uint64_t nn, uint32_t iter) {
    ExpandArgs a{};
    a.front = g->d_front[0];
    a.fs = g->d_fs[0];
    a.fd = g->d_fd[0];
    a.fval = g->d_fval[0];
    a.n = nn;
    a.off = g->d_off;
    a.edges = pairs ? g->d_pairs : g->d_edges;  // interleaved (dst, weight) stream
    a.weights = pairs ? nullptr : g->d_weights;
    a.pairs = pairs ? 1 : 0;
    a.state = g->d_state;
    a.flags = g->d_flags;
    a.visited = g->d_visited;
    a.iter = iter;
    a.big_s = g->d_big_s;
    a.big_e = g->d_big_e;
    a.big_val = g->d_big_val;
    a.big_prefix = g->d_big_prefix;
    a.ctr = g->d_ctr;
    a.wcnt = g->d_wcnt;
    a.wpre = g->d_wpre;
    a.scan_tmp = g->d_scan_tmp;
    a.scan_tmp_bytes = g->scan_tmp_bytes;
    a.cmp = static_cast<const uint32_t*>(g->d_cmp);
    a.cpos = g->d_cpos;
    a.cmp_ww = g->cmp_ww;
    a.cmp_wmin = g->cmp_wmin;
    a.cmp_b0 = g->cmp_b0;
    tune_params(&a, g);
    return a;
  };
  auto compact_args = [&]() {
    CompactArgs c{};
    c.flags = g->d_flags;
    c.nv = g->nv;
    c.ntiles = g->ntiles;
    c.tiles = g->d_tiles;
    c.front_out = g->d_front[0];
    c.fs_out = g->d_fs[0];
    c.fd_out = g->d_fd[0];
    c.fval_out = g->d_fval[0];
    c.off = g->d_off;
    c.state = g->d_state;
    c.ctr = g->d_ctr;
    c.in_off = dobfs ? g->d_in_off : nullptr;  // unvisited in-edge bookkeeping
    return c;
  };
  const int ebytes = pairs ? 8 : static_cast<int>(g->eb);
  uint64_t iters = 0, total_trav = 0, max_front = 0;

  // ---- device-driven loop: the whole traversal is one graph launch
  const ExpandArgs probe = expand_args(g->nv, 0);
  // near-far SSSP (nf_delta > 0, B200 extension): the frontier holds only
  // the improved vertices below a moving threshold; the rest wait, marked
  const bool nearfar = algo == kSssp && nf_delta > 0;
  uint64_t thresh = nearfar ? nf_delta : 0;
  const bool device_loop = n > 0 && strategy != kNaive && !dobfs && !model && !nearfar &&
                           !probe.chunk_sched && !(g->options & ZC_OPT_HOST_LOOP) &&
                           !g->tune.host_loop;
  if (device_loop) {  // (re)built on the host before the timed region starts
    const int rc =
        build_loop_graph(g, algo, strategy, ebytes, expand_args(g->nv, 0), compact_args());
    if (rc) return rc;
  }
  ZC_CUDA_TRY(cudaEventRecord(g->ev[0], st));
  // direction-optimizing: in-edges of the unvisited vertices (Beamer's m_u)
  uint64_t unvisited_in = 0;
  if (dobfs && n) {
    uint64_t io[2];
    ZC_CUDA_TRY(cudaMemcpy(io, g->d_in_off + src, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    uint64_t e_in = 0;
    ZC_CUDA_TRY(cudaMemcpy(&e_in, g->d_in_off + g->nv, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    unvisited_in = e_in - (io[1] - io[0]);
  }
  const double do_alpha = g->tune.do_alpha;
  if (device_loop) {
    uint64_t* h = g->h_ctr;
    h[kCtrCur] = n;
    h[kCtrIter] = 0;
    h[20] = trav;
    h[21] = n;
    ZC_CUDA_TRY(cudaMemcpyAsync(g->d_ctr + kCtrCur, h + kCtrCur, 2 * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, st));
    ZC_CUDA_TRY(cudaMemcpyAsync(g->d_log, h + 20, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    ZC_CUDA_TRY(cudaMemcpyAsync(g->d_log + kLogCap, h + 21, sizeof(uint64_t),
                                cudaMemcpyHostToDevice, st));
    ZC_CUDA_TRY(cudaGraphLaunch(g->loop.exec, st));
    ZC_CUDA_TRY(cudaMemcpyAsync(h, g->d_ctr, kCtrCount * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    iters = h[kCtrIter];
    const uint64_t logged = std::min<uint64_t>(iters, kLogCap);
    std::vector<uint64_t> lg(4 * kLogCap);
    ZC_CUDA_TRY(cudaMemcpy(lg.data(), g->d_log, 4 * kLogCap * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < logged; ++k) {
      g->log_trav.push_back(lg[k]);
      g->log_front.push_back(lg[kLogCap + k]);
      g->log_expand_ms.push_back((lg[3 * kLogCap + k] - lg[2 * kLogCap + k]) * 1e-6);
      total_trav += lg[k];
      max_front = std::max(max_front, lg[kLogCap + k]);
    }
    launches += iters * g->loop.launches_per_iter;
    n = h[kCtrCur];  // non-zero only if the log capacity ran out: finish on the host
    trav = h[kCtrTrav];
  }

  // ---- host-driven loop (naive, request model, tuning, or the tail past the log)
  std::vector<uint64_t> host_iters;
  while (n > 0) {
    ++iters;
    g->log_trav.push_back(trav);
    g->log_front.push_back(n);
    total_trav += trav;
    max_front = std::max(max_front, n);
    if (model)
      ZC_CUDA_TRY(launch_traffic_model(strategy, g->eb, g->wb, algo == kSssp, g->d_front[0], n,
                                       g->d_off, g->d_ctr, g->num_sms, st, &launches));
    const ExpandArgs a = expand_args(n, static_cast<uint32_t>(iters));
    while (g->iter_ev.size() < 2 * (host_iters.size() + 1)) {
      cudaEvent_t e;
      ZC_CUDA_TRY(cudaEventCreate(&e));
      g->iter_ev.push_back(e);
    }
    const size_t ev = 2 * host_iters.size();
    host_iters.push_back(iters);
    // bottom-up when the frontier's out-edges outnumber the unvisited
    // vertices' in-edges / alpha (the step then reads the candidates' in-list
    // lines, stopping at the first parent, instead of the frontier's lists)
    const bool pull = dobfs && iters > 1 && static_cast<double>(trav) * do_alpha >
                                                static_cast<double>(unvisited_in);
    if (!pull) ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[ev], st));
    if (pull) {
      ZC_CUDA_TRY(launch_pull_prepare(g->d_front[0], n, g->d_fbits, g->nv, g->d_visited,
                                      g->d_hasin, g->d_cand, g->num_sms, st, &launches));
      CompactArgs cc{};
      cc.flags = g->d_cand;
      cc.nv = g->nv;
      cc.ntiles = g->ntiles;
      cc.tiles = g->d_tiles;
      cc.front_out = g->d_front[1];
      cc.fs_out = g->d_fs[1];
      cc.fd_out = g->d_fd[1];
      cc.fval_out = g->d_fval[1];
      cc.off = g->d_in_off;
      cc.state = g->d_state;
      cc.ctr = g->d_ctr;
      ZC_CUDA_TRY(launch_compact(kBfs, cc, st, &launches));
      ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      ZC_CUDA_TRY(cudaStreamSynchronize(st));
      const uint64_t ncand = g->h_ctr[kCtrNext];
      // the expansion-time events bracket the sweep only (candidate set-up is
      // compaction work, like the top-down steps' next-frontier compaction)
      ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[ev], st));
      ExpandArgs b = a;
      b.front = g->d_front[1];
      b.fs = g->d_fs[1];
      b.fd = g->d_fd[1];
      b.fval = g->d_fval[1];
      b.n = ncand;
      b.cmp = static_cast<const uint32_t*>(g->d_cmp_in);
      b.cpos = g->d_cpos_in;
      b.fbits = g->d_fbits;
      // pass 1: first lines (most candidates find their parent there); pass 2:
      // the remaining lines of long in-lists still without one
      b.pull_pass = 1;
      ZC_CUDA_TRY(launch_expand(kCompressed, kBfsPull, 4, g->wb, b, g->num_sms, st, &launches));
      b.pull_pass = 2;
      ZC_CUDA_TRY(launch_expand(kCompressed, kBfsPull, 4, g->wb, b, g->num_sms, st, &launches));
    } else {
      ZC_CUDA_TRY(launch_expand(td_strategy, algo, ebytes, g->wb, a, g->num_sms, st, &launches));
    }
    ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[ev + 1], st));
    CompactArgs ca = compact_args();
    ca.thresh = thresh;
    ZC_CUDA_TRY(launch_compact(algo, ca, st, &launches));
    const size_t nctr = model ? kCtrCount : dobfs ? kCtrLoaded + 1 : 2;
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, nctr * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
    if (model)
      ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr + kCtrHist, 0, 8 * sizeof(uint64_t), st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    n = g->h_ctr[kCtrNext];
    trav = g->h_ctr[kCtrTrav];
    while (nearfar && n == 0) {  // near set done: next non-empty bucket of the far pile
      ZC_CUDA_TRY(launch_far_min(g->d_flags, g->d_state, g->nv, g->d_ctr, st, &launches));
      ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr + kCtrFarMin, g->d_ctr + kCtrFarMin,
                                  2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      ZC_CUDA_TRY(cudaStreamSynchronize(st));
      if (g->h_ctr[kCtrFar] == 0) break;
      thresh = g->h_ctr[kCtrFarMin] + nf_delta;
      ca.thresh = thresh;
      ZC_CUDA_TRY(launch_compact(algo, ca, st, &launches));
      ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, 2 * sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, st));
      ZC_CUDA_TRY(cudaStreamSynchronize(st));
      n = g->h_ctr[kCtrNext];
      trav = g->h_ctr[kCtrTrav];
    }
    if (dobfs) {
      unvisited_in -= std::min(unvisited_in, g->h_ctr[kCtrTravIn]);
      g->log_pull.push_back(pull ? 1 : 0);
    }
    if (model) g->log_hist.insert(g->log_hist.end(), g->h_ctr + kCtrHist, g->h_ctr + kCtrHist + 8);
  }
  // compressed sweeps: the line-stream bytes they requested over the whole run
  ZC_CUDA_TRY(cudaMemcpyAsync(&g->h_small[3], g->d_ctr + kCtrLoaded, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaEventRecord(g->ev[1], st));
  // BFS levels below 255 travel as one byte each and are widened to int64 on
  // the host: the download is V bytes instead of 8 V (which, at the link's
  // speed, costs as much as a bottom-up traversal and competes with its reads)
  const bool narrow = algo == kBfs && g->nv && iters <= 255;
  if (async && narrow) {
    const uint32_t b = g->out_next;
    g->out_next ^= 1;
    if (g->widen_th[b].joinable()) g->widen_th[b].join();  // slot b's host staging is free
    ZC_CUDA_TRY(cudaStreamWaitEvent(st, g->out_done[b], 0));
    uint8_t* d_u8 = reinterpret_cast<uint8_t*>(g->d_outbuf[b]);
    ZC_CUDA_TRY(launch_narrow_levels(g->d_state, g->nv, d_u8, st, &launches));
    ZC_CUDA_TRY(cudaEventRecord(g->out_ready[b], st));
    ZC_CUDA_TRY(cudaStreamWaitEvent(g->copy_stream, g->out_ready[b], 0));
    if (!g->h_stage[b]) g->h_stage[b] = static_cast<uint8_t*>(pinned_list_alloc(g->device, g->nv));
    if (!g->h_stage[b]) return ZC_ENOMEM;
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_stage[b], d_u8, g->nv, cudaMemcpyDeviceToHost,
                                g->copy_stream));
    ZC_CUDA_TRY(cudaEventRecord(g->out_done[b], g->copy_stream));
    ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
    const cudaEvent_t done = g->out_done[b];
    const uint8_t* src8 = g->h_stage[b];
    const uint64_t nv = g->nv;
    const int dev = g->device;
    const int wthreads = g->tune.widen;
    int* err = &g->widen_err;
    g->widen_th[b] = std::thread([=] {  // widens while the caller starts the next traversal
      cudaSetDevice(dev);
      if (cudaEventSynchronize(done) != cudaSuccess) {
        *err = ZC_ECUDA;
        return;
      }
      widen_levels(src8, out, nv, true, wthreads);
    });
    ZC_CUDA_TRY(cudaEventSynchronize(g->ev[1]));
  } else if (narrow) {
    uint8_t* d_u8 = reinterpret_cast<uint8_t*>(g->d_fval[0]);
    ZC_CUDA_TRY(launch_narrow_levels(g->d_state, g->nv, d_u8, st, &launches));
    if (!g->h_stage[2]) g->h_stage[2] = static_cast<uint8_t*>(pinned_list_alloc(g->device, g->nv));
    if (!g->h_stage[2]) return ZC_ENOMEM;
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_stage[2], d_u8, g->nv, cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    widen_levels(g->h_stage[2], out, g->nv, false);
  } else if (async) {
    // widen into the slot the download two calls ago has finished with, then
    // download it on copy_stream: the D2H direction of the link is idle while
    // the next traversal streams the edge list H2D
    const uint32_t b = g->out_next;
    g->out_next ^= 1;
    if (g->widen_th[b].joinable()) g->widen_th[b].join();
    ZC_CUDA_TRY(cudaStreamWaitEvent(st, g->out_done[b], 0));
    ZC_CUDA_TRY(launch_widen(algo, g->d_state, g->nv, g->d_outbuf[b], st, &launches));
    ZC_CUDA_TRY(cudaEventRecord(g->out_ready[b], st));
    ZC_CUDA_TRY(cudaStreamWaitEvent(g->copy_stream, g->out_ready[b], 0));
    if (g->nv)
      ZC_CUDA_TRY(cudaMemcpyAsync(out, g->d_outbuf[b], g->nv * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, g->copy_stream));
    ZC_CUDA_TRY(cudaEventRecord(g->out_done[b], g->copy_stream));
    ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
    ZC_CUDA_TRY(cudaEventSynchronize(g->ev[1]));
  } else {
    // widen into an int64 staging buffer (free fval slot) and download
    int64_t* d_out = reinterpret_cast<int64_t*>(g->d_fval[0]);
    ZC_CUDA_TRY(launch_widen(algo, g->d_state, g->nv, d_out, st, &launches));
    if (g->nv)
      ZC_CUDA_TRY(cudaMemcpyAsync(out, d_out, g->nv * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
  }
  for (size_t k = 0; k < host_iters.size(); ++k) {
    float e = 0;
    cudaEventElapsedTime(&e, g->iter_ev[2 * k], g->iter_ev[2 * k + 1]);
    g->log_expand_ms.push_back(e);
  }
  double expand_ms = 0;
  for (double x : g->log_expand_ms) expand_ms += x;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->iterations = iters;
    stats->total_traversed_edges = total_trav;
    stats->max_frontier = max_front;
    float ms = 0;
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    stats->kernel_ms = ms;
    if (!async) {  // the pipelined download has not finished yet
      cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
      stats->d2h_ms = ms;
    }
    stats->h2d_bytes = h2d;
    stats->d2h_bytes = g->nv * (narrow ? 1 : sizeof(int64_t)) +
                       (device_loop ? (kCtrCount + 4 * kLogCap) : iters * (model ? kCtrCount : 2)) *
                           sizeof(uint64_t);
    stats->launches = launches;
    stats->expand_ms = expand_ms;
    stats->total_ms = now_ms() - t0;
  }
  return ZC_OK;
}

// Bucket width of near-far SSSP when the caller passes 0: measured over
// 8..256 on U27 and a weighted K27 (weights 8..72, profiles/r02_delta_ab.txt),
// 16 is within 3% of the best on every graph / strategy pair (32: up to 11%
// slower; 8 does the least work but takes more iterations).
constexpr uint64_t kNearFarDelta = 16;

// Connected components by union-find, Afforest's schedule (Sutton et al.,
// IPDPS'18) over the zero-copy lists (B200 extension; the reference's Jacobi
// label propagation is traversal.py:154-179).  Labels equal the reference's:
// parents point to smaller ids, so each root is its component's minimum id.
//   pass 1: every vertex unions with the neighbours of its first window (one
//           request per list: the merged-aligned line / the first compressed
//           line, short compressed lists whole);
//   flatten, sample 1024 roots -> the most frequent one (the giant component);
//   pass 2: only vertices outside it whose lists reach past the first window
//           union with all their neighbours -- for an undirected graph every
//           edge with an endpoint outside the giant component is seen from
//           that endpoint, so no edge is missed;
//   flatten -> labels.
// iterations = passes; traversed_edges[k] = the list elements pass k read (pass 1:
// the first windows, counted on the device; pass 2: the degree sum of its lists).
int run_afforest(zc_graph* g, int strategy, int64_t* out, zc_stats* stats) {
  const double t0 = now_ms();
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (strategy < kNaive || strategy > kCompressed) {
    set_error("afforest runs with naive / merged / merged-aligned / packed / compressed");
    return ZC_EINVAL;
  }
  if (g->flags & ZC_F_DIRECTED) {  // traversal.py:163-165
    set_error("connected components require an undirected graph "
              "(load with directed=False or symmetrize first)");
    return ZC_EINVAL;
  }
  if (g->nparts) {
    set_error("afforest runs on whole graphs, not partitions");
    return ZC_ESTATE;
  }
  if (!out && g->nv) {
    set_error("null output buffer");
    return ZC_EINVAL;
  }
  if (strategy == kCompressed && g->eb != 4) {
    set_error("compressed lists need 4-byte edges");
    return ZC_EINVAL;
  }
  DeviceGuard dg(g->device);
  if (strategy == kCompressed && !g->d_cmp) {
    const int rc = zc_graph_build_compressed(g, nullptr);
    if (rc) return rc;
  }
  // pass 1 reads one window per list: packed's shared blocks are an
  // optimisation of whole-list sweeps, so its first pass is merged-aligned
  const int s1 = strategy == kPacked ? static_cast<int>(kMergedAligned) : strategy;
  cudaStream_t st = g->stream;
  uint64_t launches = 0;
  g->log_trav.clear();
  g->log_front.clear();
  g->log_hist.clear();
  g->log_expand_ms.clear();
  g->log_pull.clear();
  uint32_t* parent = static_cast<uint32_t*>(g->d_state);
  ZC_CUDA_TRY(cudaEventRecord(g->ev[0], st));
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_flags, 0, g->vpad, st));
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr, 0, kCtrCount * sizeof(uint64_t), st));
  // parent[v] = v, frontier = every vertex (value = its id)
  ZC_CUDA_TRY(launch_init(kCc, g->d_state, g->nv, 0, g->d_off, g->d_front[0], g->d_fval[0],
                          g->d_fs[0], g->d_fd[0], st, &launches));
  while (g->iter_ev.size() < 4) {
    cudaEvent_t e;
    ZC_CUDA_TRY(cudaEventCreate(&e));
    g->iter_ev.push_back(e);
  }
  auto args = [&](uint64_t n, int pass) {
    ExpandArgs a{};
    a.front = g->d_front[0];
    a.fs = g->d_fs[0];
    a.fd = g->d_fd[0];
    a.fval = g->d_fval[0];
    a.n = n;
    a.off = g->d_off;
    a.edges = g->d_edges;
    a.state = g->d_state;
    a.flags = g->d_flags;
    a.visited = g->d_visited;
    a.ctr = g->d_ctr;
    a.big_s = g->d_big_s;
    a.big_e = g->d_big_e;
    a.big_val = g->d_big_val;
    a.big_prefix = g->d_big_prefix;
    a.wcnt = g->d_wcnt;
    a.wpre = g->d_wpre;
    a.scan_tmp = g->d_scan_tmp;
    a.scan_tmp_bytes = g->scan_tmp_bytes;
    a.cmp = static_cast<const uint32_t*>(g->d_cmp);
    a.cpos = g->d_cpos;
    a.cmp_b0 = g->cmp_b0;
    a.pull_pass = static_cast<uint32_t>(pass);
    tune_params(&a, g);
    return a;
  };
  uint64_t iters = 0;
  if (g->nv) {
    ++iters;
    g->log_trav.push_back(g->ne);  // naive reads whole lists; else replaced by kCtrVisited below
    g->log_front.push_back(g->nv);
    ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[0], st));
    ZC_CUDA_TRY(launch_expand(s1, kCcUf, g->eb, g->wb, args(g->nv, 1), g->num_sms, st, &launches));
    ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[1], st));
    ZC_CUDA_TRY(launch_uf_flatten(parent, g->nv, st, &launches));
    // the most frequent root of 1024 sampled vertices
    uint32_t* d_sample = reinterpret_cast<uint32_t*>(g->d_log);  // 4 kLogCap u64: unused here
    constexpr uint32_t kSample = 1024;
    ZC_CUDA_TRY(launch_uf_sample(parent, g->nv, d_sample, kSample, st, &launches));
    std::vector<uint32_t> roots(kSample);
    ZC_CUDA_TRY(cudaMemcpyAsync(roots.data(), d_sample, kSample * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    std::sort(roots.begin(), roots.end());
    uint32_t giant = roots[0];
    size_t best = 0;
    for (size_t i = 0; i < roots.size();) {
      size_t j = i;
      while (j < roots.size() && roots[j] == roots[i]) ++j;
      if (j - i > best) {
        best = j - i;
        giant = roots[i];
      }
      i = j;
    }
    ZC_CUDA_TRY(launch_uf_marks(parent, g->d_off, g->d_cpos, g->nv, giant, s1, g->eb,
                                args(0, 1).uf_sample, g->d_flags, st, &launches));
    CompactArgs c{};
    c.flags = g->d_flags;
    c.nv = g->nv;
    c.ntiles = g->ntiles;
    c.tiles = g->d_tiles;
    c.front_out = g->d_front[0];
    c.fs_out = g->d_fs[0];
    c.fd_out = g->d_fd[0];
    c.fval_out = g->d_fval[0];
    c.off = g->d_off;
    c.state = g->d_state;
    c.ctr = g->d_ctr;
    ZC_CUDA_TRY(launch_compact(kCc, c, st, &launches));
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, (kCtrVisited + 1) * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    const uint64_t n2 = g->h_ctr[kCtrNext], trav2 = g->h_ctr[kCtrTrav];
    // the sampling pass reads the first window (line) of every list: log the
    // elements it actually read, so work and link bytes are what crossed the link
    if (s1 != kNaive) g->log_trav[0] = g->h_ctr[kCtrVisited];
    if (n2) {
      ++iters;
      g->log_trav.push_back(trav2);
      g->log_front.push_back(n2);
      ZC_CUDA_TRY(launch_fval_ids(g->d_front[0], g->d_fval[0], n2, st, &launches));
      ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2], st));
      ZC_CUDA_TRY(launch_expand(strategy, kCcUf, g->eb, g->wb, args(n2, 0), g->num_sms, st,
                                &launches));
      ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[3], st));
      ZC_CUDA_TRY(launch_uf_flatten(parent, g->nv, st, &launches));
    }
  }
  ZC_CUDA_TRY(cudaEventRecord(g->ev[1], st));
  int64_t* d_out = reinterpret_cast<int64_t*>(g->d_fval[0]);
  ZC_CUDA_TRY(launch_widen(kCc, g->d_state, g->nv, d_out, st, &launches));
  if (g->nv)
    ZC_CUDA_TRY(cudaMemcpyAsync(out, d_out, g->nv * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  double expand_ms = 0;
  for (uint64_t k = 0; k < iters; ++k) {
    float e = 0;
    cudaEventElapsedTime(&e, g->iter_ev[2 * k], g->iter_ev[2 * k + 1]);
    g->log_expand_ms.push_back(e);
    expand_ms += e;
  }
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->iterations = iters;
    uint64_t tt = 0;
    for (uint64_t x : g->log_trav) tt += x;
    stats->total_traversed_edges = tt;
    stats->max_frontier = g->nv;
    float ms = 0;
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    stats->kernel_ms = ms;
    cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
    stats->d2h_ms = ms;
    stats->d2h_bytes = g->nv * sizeof(int64_t) + 1024 * sizeof(uint32_t) + iters * 16;
    stats->launches = launches;
    stats->expand_ms = expand_ms;
    stats->total_ms = now_ms() - t0;
  }
  return ZC_OK;
}

}  // namespace

extern "C" {

const char* zc_last_error(void) { return g_err.c_str(); }
int zc_abi_version(void) { return ZC_ABI_VERSION; }

int zc_device_count(int* count) {
  ZC_CUDA_TRY(cudaGetDeviceCount(count));
  return ZC_OK;
}

static int create_impl(const zc_graph_desc* d, zc_graph** out, uint64_t dest_limit) {
  if (!d || !out) {
    set_error("null argument");
    return ZC_ESTATE;
  }
  *out = nullptr;
  bool neg = false;
  int rc = validate_desc(d, &neg, dest_limit);
  if (rc) return rc;
  int ndev = 0;
  ZC_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) {
    set_error("device " + std::to_string(d->device) + " not present (" + std::to_string(ndev) +
              " visible)");
    return ZC_EINVAL;
  }
  DeviceGuard dg(d->device);
  zc_graph* g = new zc_graph();
  g->nv = d->num_vertices;
  g->ne = d->num_edges;
  g->eb = d->edge_elem_bytes;
  g->wb = d->weight_elem_bytes;
  g->placement = d->placement;
  g->device = d->device;
  g->flags = d->flags;
  g->has_weights = d->weights != nullptr;
  g->negative_weight = neg;
  auto fail = [&](int code) {
    free_graph(g);
    return code;
  };
  g->h_off = static_cast<int64_t*>(pinned_list_alloc(g->device, (g->nv + 1) * sizeof(int64_t)));
  if (!g->h_off) {
    cudaGetLastError();
    set_error("cannot allocate pinned offsets");
    return fail(ZC_ENOMEM);
  }
  convert_copy(g->h_off, 8, d->offsets, 8, g->nv + 1);
  rc = place_list(g, d->edges, d->src_edge_bytes, g->eb, g->ne, &g->h_edges,
                  &g->edges_registered, &g->d_edges, &g->hbm_edges);
  if (rc) return fail(rc);
  if (g->has_weights) {
    rc = place_list(g, d->weights, d->src_weight_bytes, g->wb, g->ne, &g->h_weights,
                    &g->weights_registered, &g->d_weights, &g->hbm_weights);
    if (rc) return fail(rc);
  }
  rc = alloc_state(g);
  if (rc) return fail(rc);
  rc = finish_create(g);
  if (rc) return fail(rc);
  *out = g;
  return ZC_OK;
}

int zc_graph_create(const zc_graph_desc* d, zc_graph** out) { return create_impl(d, out, 0); }

// ------------------------------------------------------------ EMGI loader
// Reads an EMGI v1 file (csr.py:17-23, 180-245) straight into the handle's
// list buffers (pinned / managed / pinned staging for HBM) with parallel
// preads: no intermediate copy of the payload.
namespace {
int pread_all(int fd, void* dst, uint64_t bytes, uint64_t off) {
  std::atomic<int> bad{0};
  const uint64_t chunk = 64ull << 20;
  const uint64_t nchunks = (bytes + chunk - 1) / chunk;
  parallel_for(nchunks, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t c = lo; c < hi && !bad; ++c) {
      uint64_t done = c * chunk;
      const uint64_t end = std::min(bytes, done + chunk);
      while (done < end) {
        const ssize_t r = pread(fd, static_cast<char*>(dst) + done, end - done, off + done);
        if (r <= 0) {
          bad = 1;
          break;
        }
        done += static_cast<uint64_t>(r);
      }
    }
  }, 0, 2);  // 64 MiB chunks on every core: page-cache copies scale with threads
  return bad ? ZC_EINVAL : ZC_OK;
}

uint64_t round_up(uint64_t n, uint64_t a) { return (n + a - 1) / a * a; }
}  // namespace

int zc_graph_open_emgi(const char* path, int32_t placement, int32_t device, uint32_t flags,
                       zc_graph** out) {
  if (!path || !out) {
    set_error("null argument");
    return ZC_ESTATE;
  }
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    set_error(std::string("cannot open ") + path);
    return ZC_EINVAL;
  }
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } guard{fd};
  struct stat stt;
  fstat(fd, &stt);
  const uint64_t size = static_cast<uint64_t>(stt.st_size);
  unsigned char hdr[28];
  if (size < sizeof(hdr) || pread(fd, hdr, sizeof(hdr), 0) != (ssize_t)sizeof(hdr)) {
    set_error("truncated file: " + std::to_string(size) + " bytes, header needs 28");
    return ZC_EINVAL;
  }
  if (memcmp(hdr, "EMGI", 4) != 0) {
    set_error("bad magic");
    return ZC_EINVAL;
  }
  uint32_t version, fl;
  uint64_t nv, ne;
  memcpy(&version, hdr + 4, 4);
  memcpy(&fl, hdr + 8, 4);
  memcpy(&nv, hdr + 12, 8);
  memcpy(&ne, hdr + 20, 8);
  if (version != 1) {
    set_error("unsupported format version " + std::to_string(version));
    return ZC_EINVAL;
  }
  const uint32_t eb = (fl & 2) ? 8 : 4, wb = (fl & 4) ? 8 : 4;
  const bool has_w = fl & 1;
  // header fields are untrusted: bound every count by the bytes that follow
  // before multiplying, so no product can wrap past the size checks
  const uint64_t off_pos = 28;
  if (nv > (size - off_pos) / 8 - 1 || (size - off_pos) / 8 == 0) {
    set_error("truncated file: offsets array incomplete");
    return ZC_EINVAL;
  }
  const uint64_t off_end = off_pos + (nv + 1) * 8;
  const uint64_t e_pos = round_up(off_end, 128);
  if (e_pos > size || ne > (size - e_pos) / eb) {
    set_error("truncated file: edge array incomplete");
    return ZC_EINVAL;
  }
  const uint64_t e_end = e_pos + ne * eb;
  const uint64_t w_pos = round_up(e_end, 128);
  const uint64_t w_end = has_w && w_pos <= size && ne <= (size - w_pos) / wb ? w_pos + ne * wb
                                                                              : UINT64_MAX;
  if (has_w && w_end > size) {
    set_error("truncated file: weight array incomplete");
    return ZC_EINVAL;
  }
  if (!placement_valid(placement)) {
    set_error("unknown placement");
    return ZC_EINVAL;
  }
  if (nv >= 0xffffffffull) {
    set_error("device path supports fewer than 2^32-1 vertices");
    return ZC_EINVAL;
  }
  int ndev = 0;
  ZC_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device not present");
    return ZC_EINVAL;
  }
  DeviceGuard dg(device);
  zc_graph* g = new zc_graph();
  g->nv = nv;
  g->ne = ne;
  g->eb = eb;
  g->wb = wb;
  g->placement = placement;
  g->device = device;
  g->flags = flags & (ZC_F_DIRECTED | ZC_F_UVM_PREFETCH | ZC_F_NO_VALIDATE);
  g->has_weights = has_w;
  auto fail = [&](int code) {
    free_graph(g);
    return code;
  };
  g->h_off = static_cast<int64_t*>(pinned_list_alloc(g->device, (nv + 1) * sizeof(int64_t)));
  if (!g->h_off) {
    set_error("cannot allocate pinned offsets");
    return fail(ZC_ENOMEM);
  }
  if (pread_all(fd, g->h_off, (nv + 1) * 8, off_pos)) {
    set_error("read error (offsets)");
    return fail(ZC_EINVAL);
  }
  // lists: read straight into their final host-side buffer
  auto load = [&](uint64_t pos, uint32_t w, void** h, const void** dptr, void** hbm) -> int {
    const size_t bytes = std::max<size_t>(ne * w, kLineBytes);
    void* p = nullptr;
    if (placement == ZC_PLACE_UVM) {
      ZC_CUDA_TRY(cudaMallocManaged(&p, bytes, cudaMemAttachGlobal));
    } else if (!(p = host_list_alloc(g, bytes))) {
      set_error("cannot allocate host memory for a list");
      return ZC_ENOMEM;
    }
    *h = p;
    if (ne && pread_all(fd, p, ne * w, pos)) {
      set_error("read error (lists)");
      return ZC_EINVAL;
    }
    if (placement == ZC_PLACE_UVM) {
      ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseSetReadMostly, device));
      *dptr = p;
    } else if (placement == ZC_PLACE_HBM) {
      ZC_CUDA_TRY(cudaMalloc(hbm, bytes));
      ZC_CUDA_TRY(cudaMemcpy(*hbm, p, ne * w, cudaMemcpyHostToDevice));
      *dptr = *hbm;
    } else {
      return host_list_device_ptr(p, dptr);
    }
    return ZC_OK;
  };
  int rc = load(e_pos, eb, &g->h_edges, &g->d_edges, &g->hbm_edges);
  if (rc) return fail(rc);
  if (has_w && (rc = load(w_pos, wb, &g->h_weights, &g->d_weights, &g->hbm_weights)))
    return fail(rc);
  // invariants (csr.py:80-105) on the loaded buffers
  zc_graph_desc d{};
  d.num_vertices = nv;
  d.num_edges = ne;
  d.offsets = g->h_off;
  d.edges = g->h_edges;
  d.weights = has_w ? g->h_weights : nullptr;
  d.src_edge_bytes = d.edge_elem_bytes = eb;
  d.src_weight_bytes = d.weight_elem_bytes = wb;
  d.placement = placement;
  d.device = device;
  d.flags = g->flags;
  bool neg = false;
  if ((rc = validate_desc(&d, &neg))) return fail(rc);
  g->negative_weight = neg;
  if ((rc = alloc_state(g))) return fail(rc);
  if ((rc = finish_create(g))) return fail(rc);
  *out = g;
  return ZC_OK;
}

void zc_graph_destroy(zc_graph* g) { free_graph(g); }

// ------------------------------------------------------------ partitions
int zc_part_create(const zc_graph_desc* local, const zc_part_info* info, zc_graph** out) {
  if (!info || !info->bounds || !info->nparts || info->part >= info->nparts) {
    set_error("invalid partition info");
    return ZC_EINVAL;
  }
  const uint64_t gv = info->global_vertices;
  for (uint32_t k = 0; k < info->nparts; ++k) {
    if (info->bounds[k] > info->bounds[k + 1] ||
        info->bounds[k + 1] - info->bounds[k] > info->stride) {
      set_error("partition bounds must be non-decreasing with ranges <= stride");
      return ZC_EINVAL;
    }
  }
  if (info->bounds[0] != 0 || info->bounds[info->nparts] != gv ||
      info->bounds[info->part + 1] - info->bounds[info->part] != local->num_vertices) {
    set_error("partition bounds do not match the global / local vertex counts");
    return ZC_EINVAL;
  }
  int rc = create_impl(local, out, gv ? gv : 1);
  if (rc) return rc;
  rc = init_partition(*out, info);
  if (rc) {
    free_graph(*out);
    *out = nullptr;
  }
  return rc;
}

size_t zc_part_exchange_elem_bytes(int algo) {
  return algo == kBfs ? 1 : algo == kSssp ? 8 : 4;
}

int zc_part_begin(zc_graph* g, int algo, uint64_t src, int strategy, uint64_t* n_local,
                  uint64_t* trav_local) {
  if (!g || !g->nparts) {
    set_error("not a partition handle");
    return ZC_ESTATE;
  }
  if (algo < kBfs || algo > kCc || strategy < kNaive || strategy > kDirOpt) {
    set_error("unknown algorithm or strategy");
    return ZC_EINVAL;
  }
  if (strategy == kDirOpt && algo != kBfs) {
    set_error("direction-optimizing is a bfs strategy");
    return ZC_EINVAL;
  }
  if ((strategy == kCompressed || strategy == kDirOpt) &&
      (g->eb != 4 || (algo == kSssp && g->has_weights && g->wb != 4))) {
    set_error("compressed lists need 4-byte edges (and 4-byte weights for sssp)");
    return ZC_EINVAL;
  }
  if ((strategy == kCompressed || strategy == kDirOpt) && !g->d_cmp) {  // built once per handle
    const int rc = zc_graph_build_compressed(g, nullptr);
    if (rc) return rc;
  }
  if (strategy == kDirOpt && !g->d_cpos_in) {  // + the owned vertices' in-lists
    const int rc = zc_part_build_in_lists(g, nullptr);
    if (rc) return rc;
  }
  if (algo != kCc && src >= g->global_nv) {
    set_error("source " + std::to_string(src) + " out of range for " +
              std::to_string(g->global_nv) + " vertices");
    return ZC_EINVAL;
  }
  if (algo == kSssp && !g->has_weights) {
    set_error("sssp requires edge weights");
    return ZC_EINVAL;
  }
  if (algo == kSssp && g->negative_weight) {
    set_error("sssp requires non-negative weights");
    return ZC_EINVAL;
  }
  if (algo == kCc && (g->flags & ZC_F_DIRECTED)) {
    set_error("connected components require an undirected graph "
              "(load with directed=False or symmetrize first)");
    return ZC_EINVAL;
  }
  if (algo == kCc && g->global_nv > 0x7fffffffull) {
    set_error("partitioned cc supports fewer than 2^31 vertices");
    return ZC_EINVAL;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  g->p_algo = algo;
  g->p_strategy = strategy;
  g->p_iter = 0;
  g->p_cur = 0;
  g->p_launches = 0;
  g->p_xbytes = 0;
  g->log_trav.clear();
  g->log_front.clear();
  g->log_expand_ms.clear();
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_flags, 0, g->vpad, st));
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr, 0, kCtrCount * sizeof(uint64_t), st));
  const bool owned = algo != kCc && src >= g->lo && src < g->lo + g->nv;
  const uint64_t lsrc = owned ? src - g->lo : 0;
  ZC_CUDA_TRY(launch_init(algo, g->d_state, g->nv, lsrc, g->d_off, g->d_front[0], g->d_fval[0],
                          g->d_fs[0], g->d_fd[0], st, &g->p_launches, g->lo, owned));
  uint64_t n = 0, trav = 0;
  if (algo == kCc) {
    n = g->nv;
    trav = g->ne;
  } else if (owned) {
    g->h_small[1] = 0;
    const size_t sb = algo == kSssp ? 8 : 4;
    ZC_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(g->d_state) + lsrc * sb, &g->h_small[1], sb,
                                cudaMemcpyHostToDevice, st));
    n = 1;
    trav = g->h_off[lsrc + 1] - g->h_off[lsrc];
  }
  if (strategy == kDirOpt) {  // owned unvisited vertices' in-edges (the source is visited)
    uint64_t e_in = 0, io[2] = {0, 0};
    ZC_CUDA_TRY(cudaMemcpy(&e_in, g->d_in_off + g->nv, sizeof(e_in), cudaMemcpyDeviceToHost));
    if (owned)
      ZC_CUDA_TRY(cudaMemcpy(io, g->d_in_off + lsrc, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    g->p_unvisited_in = e_in - (io[1] - io[0]);
  }
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  g->p_n = n;
  if (n_local) *n_local = n;
  if (trav_local) *trav_local = trav;
  return ZC_OK;
}

enum PartExchange { kExchReduceScatter = 0, kExchStore = 1, kExchBitmap = 2 };

static int part_expand_impl(zc_graph* g, void* exch, int mode) {
  if (!g || !g->nparts || g->p_algo < 0) {
    set_error("zc_part_begin first");
    return ZC_ESTATE;
  }
  const bool fused = mode == kExchStore;
  if (fused && (!g->peers_ready || g->fused_algo != g->p_algo)) {
    set_error("fused exchange not initialised for this algorithm (zc_part_fused_init/connect)");
    return ZC_ESTATE;
  }
  if (mode == kExchBitmap && (!g->peer_sent_ready || g->p_algo != kBfs)) {
    set_error("bitmap exchange: a bfs run and zc_part_bitmap_init/connect first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  const int algo = g->p_algo;
  const size_t xb = zc_part_exchange_elem_bytes(algo);
  if (mode == kExchBitmap) {
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_sent, 0, (g->global_nv + 31) / 32 * 4, st));
  } else if (!fused) {
    ZC_CUDA_TRY(launch_fill_exchange(algo, exch, g->nparts * g->stride, st, &g->p_launches));
    g->p_xbytes += (g->nparts - 1) * g->stride * xb;  // this rank's reduce-scatter send
  } else if (algo == kBfs) {
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_sent, 0, (g->global_nv + 31) / 32 * 4, st));
  } else {
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_lbest, 0xff, g->global_nv * xb, st));
  }
  ++g->p_iter;
  g->log_front.push_back(g->p_n);
  while (g->iter_ev.size() < 2 * g->p_iter) {
    cudaEvent_t e;
    ZC_CUDA_TRY(cudaEventCreate(&e));
    g->iter_ev.push_back(e);
  }
  ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (g->p_iter - 1)], st));
  ExpandArgs a{};
  a.front = g->d_front[g->p_cur];
  a.fs = g->d_fs[g->p_cur];
  a.fd = g->d_fd[g->p_cur];
  a.fval = g->d_fval[g->p_cur];
  a.n = g->p_n;
  a.off = g->d_off;
  a.edges = g->d_edges;
  a.weights = g->d_weights;
  a.state = g->d_state;
  a.flags = g->d_flags;
  a.iter = static_cast<uint32_t>(g->p_iter);
  a.big_s = g->d_big_s;
  a.big_e = g->d_big_e;
  a.big_val = g->d_big_val;
  a.big_prefix = g->d_big_prefix;
  a.ctr = g->d_ctr;
  a.exch = exch;
  a.part_lo = g->d_part_lo;
  a.nparts = g->nparts;
  a.stride = g->stride;
  a.peers = fused ? g->d_peers : nullptr;
  a.sent = (fused && algo == kBfs) || mode == kExchBitmap ? g->d_sent : nullptr;
  a.sent_only = mode == kExchBitmap;
  a.lbest = fused && algo != kBfs ? g->d_lbest : nullptr;
  a.wcnt = g->d_wcnt;
  a.wpre = g->d_wpre;
  a.scan_tmp = g->d_scan_tmp;
  a.scan_tmp_bytes = g->scan_tmp_bytes;
  a.cmp = static_cast<const uint32_t*>(g->d_cmp);
  a.cpos = g->d_cpos;
  a.cmp_ww = g->cmp_ww;
  a.cmp_wmin = g->cmp_wmin;
  a.cmp_b0 = g->cmp_b0;
  tune_params(&a, g);
  // top-down steps of the direction-optimizing strategy are compressed steps
  const int td = g->p_strategy == kDirOpt ? static_cast<int>(kCompressed) : g->p_strategy;
  ZC_CUDA_TRY(launch_expand(td, algo + kPartAlgo, g->eb, g->wb, a, g->num_sms, st,
                            &g->p_launches));
  ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (g->p_iter - 1) + 1], st));
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr + kCtrBig, 0, sizeof(uint64_t), st));
  if (fused) {  // remote destinations this rank sent to (BFS: exact stores)
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr + kCtrRemote, 0, sizeof(uint64_t), st));
    ZC_CUDA_TRY(launch_count_remote(algo == kBfs ? static_cast<const void*>(g->d_sent) : g->d_lbest,
                                    algo == kBfs ? 0 : static_cast<int>(xb), g->global_nv, g->lo,
                                    g->lo + g->nv, g->d_ctr + kCtrRemote, g->num_sms, st,
                                    &g->p_launches));
    ZC_CUDA_TRY(cudaMemcpyAsync(&g->h_small[2], g->d_ctr + kCtrRemote, sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
  }
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  if (fused) g->p_xbytes += g->h_small[2] * xb;
  float ms = 0;
  cudaEventElapsedTime(&ms, g->iter_ev[2 * (g->p_iter - 1)], g->iter_ev[2 * (g->p_iter - 1) + 1]);
  g->log_expand_ms.push_back(ms);
  return ZC_OK;
}

int zc_part_expand(zc_graph* g, void* exch) {
  return part_expand_impl(g, exch, kExchReduceScatter);
}

int zc_part_fused_init(zc_graph* g, int algo, void* ipc_handle, void** local) {
  if (!g || !g->nparts) {
    set_error("not a partition handle");
    return ZC_ESTATE;
  }
  if (algo < kBfs || algo > kCc) {
    set_error("unknown algorithm");
    return ZC_EINVAL;
  }
  DeviceGuard dg(g->device);
  if (!g->d_mine) {
    ZC_CUDA_TRY(cudaMalloc(&g->d_mine, std::max<uint64_t>(g->stride, 1) * sizeof(uint64_t)));
    ZC_CUDA_TRY(cudaMalloc(&g->d_peers, g->nparts * sizeof(void*)));
    ZC_CUDA_TRY(cudaMalloc(&g->d_sent, (g->global_nv + 31) / 32 * 4 + 4));
  }
  if (algo != kBfs && !g->d_lbest)  // the local pre-filter (u64: SSSP or CC)
    ZC_CUDA_TRY(cudaMalloc(&g->d_lbest, std::max<uint64_t>(g->global_nv, 1) * sizeof(uint64_t)));
  g->fused_algo = algo;
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    ZC_CUDA_TRY(cudaIpcGetMemHandle(&h, g->d_mine));
    memcpy(ipc_handle, &h, sizeof(h));
  }
  if (local) *local = g->d_mine;
  return ZC_OK;
}

int zc_part_fused_connect(zc_graph* g, const void* handles, void* const* ptrs) {
  if (!g || !g->d_mine) {
    set_error("zc_part_fused_init first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  g->peers_ready = false;
  for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
  g->ipc_opened.clear();
  std::vector<void*> peers(g->nparts);
  for (uint32_t k = 0; k < g->nparts; ++k) {
    if (k == g->part) {
      peers[k] = g->d_mine;
    } else if (ptrs) {
      peers[k] = ptrs[k];  // same-process device pointers (one-GPU validation)
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, static_cast<const char*>(handles) + k * sizeof(h), sizeof(h));
      void* p = nullptr;
      ZC_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      g->ipc_opened.push_back(p);
      peers[k] = p;
    }
  }
  ZC_CUDA_TRY(cudaMemcpy(g->d_peers, peers.data(), g->nparts * sizeof(void*),
                         cudaMemcpyHostToDevice));
  g->peers_ready = true;
  return ZC_OK;
}

int zc_part_fused_reset(zc_graph* g) {
  if (!g || !g->d_mine || g->fused_algo < 0) {
    set_error("zc_part_fused_init first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  ZC_CUDA_TRY(launch_fill_exchange(g->fused_algo, g->d_mine, g->stride, g->stream,
                                   &g->p_launches));
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  return ZC_OK;
}

int zc_part_fused_expand(zc_graph* g) { return part_expand_impl(g, nullptr, kExchStore); }

// Owner merge of the iteration's candidates -- a reduced slice (`mine`,
// device) or, mine == NULL, the OR of every rank's discovery bitmap (BFS
// bitmap exchange) -- then the next frontier's compaction.
static int part_apply_impl(zc_graph* g, const void* mine, uint64_t* n_next,
                           uint64_t* trav_next) {
  if (!g || !g->nparts || g->p_algo < 0 || g->p_iter == 0) {
    set_error("zc_part_expand first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  const int algo = g->p_algo;
  if (mine) {
    ZC_CUDA_TRY(launch_part_apply(algo, mine, g->nv, g->d_state, g->d_flags,
                                  static_cast<uint32_t>(g->p_iter), st, &g->p_launches));
  } else {
    ZC_CUDA_TRY(launch_part_pull_apply(g->d_peer_sent, g->nparts, g->lo, g->nv, g->d_state,
                                       g->d_flags, static_cast<uint32_t>(g->p_iter),
                                       g->num_sms, st, &g->p_launches));
    // the words of this range read from every other rank
    g->p_xbytes += (g->nparts - 1) * ((g->nv + 31) / 32 + 1) * 4;
  }
  CompactArgs c{};
  c.flags = g->d_flags;
  c.nv = g->nv;
  c.ntiles = g->ntiles;
  c.tiles = g->d_tiles;
  c.front_out = g->d_front[g->p_cur ^ 1];
  c.fs_out = g->d_fs[g->p_cur ^ 1];
  c.fd_out = g->d_fd[g->p_cur ^ 1];
  c.fval_out = g->d_fval[g->p_cur ^ 1];
  c.off = g->d_off;
  c.state = g->d_state;
  c.ctr = g->d_ctr;
  c.in_off = g->p_strategy == kDirOpt ? g->d_in_off : nullptr;
  ZC_CUDA_TRY(launch_compact(algo, c, st, &g->p_launches));
  ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, (kCtrTravIn + 1) * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  g->p_n = g->h_ctr[kCtrNext];
  g->p_cur ^= 1;
  if (c.in_off) g->p_unvisited_in -= std::min(g->p_unvisited_in, g->h_ctr[kCtrTravIn]);
  if (n_next) *n_next = g->h_ctr[kCtrNext];
  if (trav_next) *trav_next = g->h_ctr[kCtrTrav];
  return ZC_OK;
}


int zc_part_apply(zc_graph* g, const void* mine, uint64_t* n_next, uint64_t* trav_next) {
  if (!mine) {
    set_error("null exchange slice");
    return ZC_EINVAL;
  }
  return part_apply_impl(g, mine, n_next, trav_next);
}

int zc_part_bitmap_init(zc_graph* g, void* ipc_handle, void** local) {
  if (!g || !g->nparts) {
    set_error("not a partition handle");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  if (!g->d_sent) ZC_CUDA_TRY(cudaMalloc(&g->d_sent, (g->global_nv + 31) / 32 * 4 + 4));
  if (!g->d_peer_sent)
    ZC_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&g->d_peer_sent), g->nparts * sizeof(void*)));
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    ZC_CUDA_TRY(cudaIpcGetMemHandle(&h, g->d_sent));
    memcpy(ipc_handle, &h, sizeof(h));
  }
  if (local) *local = g->d_sent;
  return ZC_OK;
}

int zc_part_bitmap_connect(zc_graph* g, const void* handles, void* const* ptrs) {
  if (!g || !g->d_peer_sent) {
    set_error("zc_part_bitmap_init first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  g->peer_sent_ready = false;
  for (void* p : g->ipc_opened_sent) cudaIpcCloseMemHandle(p);
  g->ipc_opened_sent.clear();
  std::vector<const void*> peers(g->nparts);
  for (uint32_t k = 0; k < g->nparts; ++k) {
    if (k == g->part) {
      peers[k] = g->d_sent;
    } else if (ptrs) {
      peers[k] = ptrs[k];  // same-process device pointers (one-GPU validation)
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, static_cast<const char*>(handles) + k * sizeof(h), sizeof(h));
      void* p = nullptr;
      ZC_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      g->ipc_opened_sent.push_back(p);
      peers[k] = p;
    }
  }
  ZC_CUDA_TRY(cudaMemcpy(g->d_peer_sent, peers.data(), g->nparts * sizeof(void*),
                         cudaMemcpyHostToDevice));
  g->peer_sent_ready = true;
  return ZC_OK;
}

int zc_part_bitmap_expand(zc_graph* g) { return part_expand_impl(g, nullptr, kExchBitmap); }

int zc_part_bitmap_apply(zc_graph* g, uint64_t* n_next, uint64_t* trav_next) {
  if (!g || !g->peer_sent_ready) {
    set_error("zc_part_bitmap_init / connect first");
    return ZC_ESTATE;
  }
  return part_apply_impl(g, nullptr, n_next, trav_next);
}

int zc_part_unvisited_in(const zc_graph* g, uint64_t* in_edges) {
  if (!g || !g->nparts || !in_edges) {
    set_error("not a partition handle");
    return ZC_ESTATE;
  }
  *in_edges = g->p_unvisited_in;
  return ZC_OK;
}

int zc_part_frontier_bits(zc_graph* g, uint32_t* bits) {
  if (!g || !g->nparts || g->p_algo < 0 || !bits) {
    set_error("zc_part_begin first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  ZC_CUDA_TRY(launch_frontier_bits(g->d_front[g->p_cur], g->p_n, g->lo, bits,
                                   (g->global_nv + 31) / 32 + 1, g->num_sms, g->stream,
                                   &g->p_launches));
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  return ZC_OK;
}

int zc_part_pull(zc_graph* g, const uint32_t* bits, uint64_t* n_next, uint64_t* trav_next) {
  if (!g || !g->nparts || g->p_algo != kBfs || g->p_strategy != kDirOpt || !bits) {
    set_error("zc_part_pull needs a direction-optimizing bfs (zc_part_begin) and the bitmap");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  ++g->p_iter;
  g->log_front.push_back(g->p_n);
  while (g->iter_ev.size() < 2 * g->p_iter) {
    cudaEvent_t e;
    ZC_CUDA_TRY(cudaEventCreate(&e));
    g->iter_ev.push_back(e);
  }
  const int nb = g->p_cur ^ 1;
  // candidates: owned unvisited vertices with in-edges, sorted, over the in-offsets
  ZC_CUDA_TRY(launch_part_pull_prepare(g->d_state, g->nv, g->d_visited, g->d_hasin, g->d_cand,
                                       g->num_sms, st, &g->p_launches));
  CompactArgs cc{};
  cc.flags = g->d_cand;
  cc.nv = g->nv;
  cc.ntiles = g->ntiles;
  cc.tiles = g->d_tiles;
  cc.front_out = g->d_front[nb];
  cc.fs_out = g->d_fs[nb];
  cc.fd_out = g->d_fd[nb];
  cc.fval_out = g->d_fval[nb];
  cc.off = g->d_in_off;
  cc.state = g->d_state;
  cc.ctr = g->d_ctr;
  ZC_CUDA_TRY(launch_compact(kBfs, cc, st, &g->p_launches));
  ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t ncand = g->h_ctr[kCtrNext];
  ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (g->p_iter - 1)], st));
  ExpandArgs b{};
  b.front = g->d_front[nb];
  b.fs = g->d_fs[nb];
  b.fd = g->d_fd[nb];
  b.fval = g->d_fval[nb];
  b.n = ncand;
  b.off = g->d_in_off;
  b.state = g->d_state;
  b.flags = g->d_flags;
  b.visited = g->d_visited;
  b.iter = static_cast<uint32_t>(g->p_iter);
  b.ctr = g->d_ctr;
  b.wcnt = g->d_wcnt;
  b.wpre = g->d_wpre;
  b.scan_tmp = g->d_scan_tmp;
  b.scan_tmp_bytes = g->scan_tmp_bytes;
  b.cmp = static_cast<const uint32_t*>(g->d_cmp_in);
  b.cpos = g->d_cpos_in;
  b.cmp_b0 = g->cmp_b0;
  b.fbits = bits;
  tune_params(&b, g);
  for (uint32_t pass = 1; pass <= 2; ++pass) {
    b.pull_pass = pass;
    ZC_CUDA_TRY(launch_expand(kCompressed, kBfsPull, 4, g->wb, b, g->num_sms, st, &g->p_launches));
  }
  ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (g->p_iter - 1) + 1], st));
  CompactArgs c{};
  c.flags = g->d_flags;
  c.nv = g->nv;
  c.ntiles = g->ntiles;
  c.tiles = g->d_tiles;
  c.front_out = g->d_front[nb];
  c.fs_out = g->d_fs[nb];
  c.fd_out = g->d_fd[nb];
  c.fval_out = g->d_fval[nb];
  c.off = g->d_off;
  c.state = g->d_state;
  c.ctr = g->d_ctr;
  c.in_off = g->d_in_off;
  ZC_CUDA_TRY(launch_compact(kBfs, c, st, &g->p_launches));
  ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, (kCtrTravIn + 1) * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0;
  cudaEventElapsedTime(&ms, g->iter_ev[2 * (g->p_iter - 1)], g->iter_ev[2 * (g->p_iter - 1) + 1]);
  g->log_expand_ms.push_back(ms);
  g->p_n = g->h_ctr[kCtrNext];
  g->p_cur = nb;
  g->p_unvisited_in -= std::min(g->p_unvisited_in, g->h_ctr[kCtrTravIn]);
  if (n_next) *n_next = g->h_ctr[kCtrNext];
  if (trav_next) *trav_next = g->h_ctr[kCtrTrav];
  return ZC_OK;
}

int zc_part_result(zc_graph* g, int64_t* out, zc_stats* stats) {
  if (!g || !g->nparts || g->p_algo < 0) {
    set_error("zc_part_begin first");
    return ZC_ESTATE;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  if (out) {  // NULL: statistics only
    int64_t* d_out = reinterpret_cast<int64_t*>(g->d_fval[g->p_cur ^ 1]);
    ZC_CUDA_TRY(launch_widen(g->p_algo, g->d_state, g->nv, d_out, st, &g->p_launches));
    if (g->nv)
      ZC_CUDA_TRY(cudaMemcpyAsync(out, d_out, g->nv * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->iterations = g->p_iter;
    stats->launches = g->p_launches;
    double ex = 0;
    for (double x : g->log_expand_ms) ex += x;
    stats->expand_ms = ex;
    stats->d2h_bytes = out ? g->nv * sizeof(int64_t) : 0;
    stats->exchange_bytes = g->p_xbytes;
  }
  return ZC_OK;
}

int zc_graph_host_lists(zc_graph* g, void** edges, void** weights, const int64_t** offsets) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (edges) *edges = g->h_edges;
  if (weights) *weights = g->h_weights;
  if (offsets) *offsets = g->h_off;
  return ZC_OK;
}

int zc_graph_info(const zc_graph* g, uint64_t* nv, uint64_t* ne, uint32_t* eb, uint32_t* wb,
                  int32_t* placement, uint32_t* flags) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (nv) *nv = g->nv;
  if (ne) *ne = g->ne;
  if (eb) *eb = g->eb;
  if (wb) *wb = g->has_weights ? g->wb : 0;
  if (placement) *placement = g->placement;
  if (flags) *flags = g->flags;
  return ZC_OK;
}

int zc_bfs(zc_graph* g, uint64_t source, int strategy, int64_t* out, zc_stats* stats) {
  return run(g, kBfs, source, strategy, out, stats);
}
int zc_sssp(zc_graph* g, uint64_t source, int strategy, int64_t* out, zc_stats* stats) {
  return run(g, kSssp, source, strategy, out, stats);
}
int zc_bfs_async(zc_graph* g, uint64_t source, int strategy, int64_t* out, zc_stats* stats) {
  return run(g, kBfs, source, strategy, out, stats, true);
}
int zc_sssp_async(zc_graph* g, uint64_t source, int strategy, int64_t* out, zc_stats* stats) {
  return run(g, kSssp, source, strategy, out, stats, true);
}
int zc_sync(zc_graph* g) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (!g->copy_stream) return ZC_OK;
  DeviceGuard dg(g->device);
  ZC_CUDA_TRY(cudaStreamSynchronize(g->copy_stream));
  for (auto& t : g->widen_th)
    if (t.joinable()) t.join();
  if (g->widen_err) {
    g->widen_err = 0;
    set_error("pipelined result download failed");
    return ZC_ECUDA;
  }
  return ZC_OK;
}
int zc_cc(zc_graph* g, int strategy, int64_t* out, zc_stats* stats) {
  return run(g, kCc, 0, strategy, out, stats);
}
int zc_sssp_nearfar(zc_graph* g, uint64_t source, int strategy, uint64_t delta, int64_t* out,
                    zc_stats* stats) {
  return run(g, kSssp, source, strategy, out, stats, false, delta ? delta : kNearFarDelta);
}
int zc_cc_afforest(zc_graph* g, int strategy, int64_t* out, zc_stats* stats) {
  return run_afforest(g, strategy, out, stats);
}

int zc_run_log(const zc_graph* g, uint64_t* trav, uint64_t* front, uint64_t cap) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  const uint64_t n = std::min<uint64_t>(cap, g->log_trav.size());
  if (trav) std::copy(g->log_trav.begin(), g->log_trav.begin() + n, trav);
  if (front) std::copy(g->log_front.begin(), g->log_front.begin() + n, front);
  return ZC_OK;
}

int zc_pagerank(zc_graph* g, int strategy, double damping, uint64_t max_iters, double tol,
                double* out, zc_stats* stats) {
  const double t0 = now_ms();
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  // traversal.py:201-208
  if (!(damping > 0.0 && damping < 1.0)) {
    set_error("damping must be in (0, 1)");
    return ZC_EINVAL;
  }
  if (max_iters < 1) {
    set_error("max_iters must be >= 1");
    return ZC_EINVAL;
  }
  if (!(tol > 0)) {
    set_error("tol must be positive");
    return ZC_EINVAL;
  }
  if (g->nv == 0) {
    set_error("pagerank needs at least one vertex");
    return ZC_EINVAL;
  }
  if (strategy < kNaive || strategy > kCompressed) {
    set_error("unknown access strategy " + std::to_string(strategy));
    return ZC_EINVAL;
  }
  const bool model = (g->options & ZC_OPT_TRAFFIC_MODEL) != 0;
  if (strategy == kCompressed && !g->d_cmp) {
    const int rc = zc_graph_build_compressed(g, nullptr);
    if (rc) return rc;
  }
  if (strategy >= kPacked && model) {
    set_error("the request model is defined for the reference's three strategies "
              "(naive, merged, merged-aligned), not for packed");
    return ZC_EINVAL;
  }
  DeviceGuard dg(g->device);
  cudaStream_t st = g->stream;
  uint64_t launches = 0;
  g->log_trav.clear();
  g->log_front.clear();
  g->log_hist.clear();
  g->log_expand_ms.clear();
  double* rank = static_cast<double*>(g->d_state);
  double* pushed = reinterpret_cast<double*>(g->d_fval[1]);
  ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr, 0, kCtrCount * sizeof(uint64_t), st));
  ZC_CUDA_TRY(launch_pr_init(g->nv, g->d_off, g->d_front[0], g->d_fs[0], g->d_fd[0], rank, st,
                             &launches));
  std::vector<uint64_t> hist0;
  if (model) {  // the whole list is traced once and repeated (traversal.py:237-246)
    ZC_CUDA_TRY(launch_traffic_model(strategy, g->eb, g->wb, false, g->d_front[0], g->nv,
                                     g->d_off, g->d_ctr, g->num_sms, st, &launches));
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr, g->d_ctr, kCtrCount * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    hist0.assign(g->h_ctr + kCtrHist, g->h_ctr + kCtrHist + 8);
  }
  ZC_CUDA_TRY(cudaEventRecord(g->ev[0], st));
  uint64_t iters = 0;
  double expand_ms = 0;
  while (iters < max_iters) {
    ++iters;
    g->log_trav.push_back(g->ne);
    g->log_front.push_back(g->nv);
    if (model) g->log_hist.insert(g->log_hist.end(), hist0.begin(), hist0.end());
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr + kCtrPrDangling, 0, 3 * sizeof(uint64_t), st));
    ZC_CUDA_TRY(launch_pr_prepare(rank, g->d_fd[0], g->nv, g->d_fval[0], pushed, g->d_ctr, st,
                                  &launches));
    ExpandArgs a{};
    a.front = g->d_front[0];
    a.fs = g->d_fs[0];
    a.fd = g->d_fd[0];
    a.fval = g->d_fval[0];
    a.n = g->nv;
    a.off = g->d_off;
    a.edges = g->d_edges;
    a.weights = g->d_weights;
    a.state = g->d_state;
    a.flags = g->d_flags;
    a.big_s = g->d_big_s;
    a.big_e = g->d_big_e;
    a.big_val = g->d_big_val;
    a.big_prefix = g->d_big_prefix;
    a.ctr = g->d_ctr;
    a.exch = pushed;
    a.cmp = static_cast<const uint32_t*>(g->d_cmp);
    a.cpos = g->d_cpos;
    a.cmp_ww = g->cmp_ww;
    a.cmp_wmin = g->cmp_wmin;
    a.cmp_b0 = g->cmp_b0;
    a.wcnt = g->d_wcnt;
    a.wpre = g->d_wpre;
    a.scan_tmp = g->d_scan_tmp;
    a.scan_tmp_bytes = g->scan_tmp_bytes;
    tune_params(&a, g);
    while (g->iter_ev.size() < 2 * iters) {
      cudaEvent_t e;
      ZC_CUDA_TRY(cudaEventCreate(&e));
      g->iter_ev.push_back(e);
    }
    ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (iters - 1)], st));
    ZC_CUDA_TRY(launch_expand(strategy, kPr, g->eb, g->wb, a, g->num_sms, st, &launches));
    ZC_CUDA_TRY(cudaEventRecord(g->iter_ev[2 * (iters - 1) + 1], st));
    ZC_CUDA_TRY(cudaMemsetAsync(g->d_ctr + kCtrBig, 0, sizeof(uint64_t), st));
    ZC_CUDA_TRY(launch_pr_update(rank, pushed, g->nv, damping, g->d_ctr, st, &launches));
    ZC_CUDA_TRY(cudaMemcpyAsync(g->h_ctr + kCtrPrDelta, g->d_ctr + kCtrPrDelta, sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, st));
    ZC_CUDA_TRY(cudaStreamSynchronize(st));
    // the L1 change is a fixed-point sum (x 2^62, zc_kernels.cu pr_fx)
    const double delta = static_cast<double>(g->h_ctr[kCtrPrDelta]) / 4611686018427387904.0;
    if (delta < tol) break;
  }
  ZC_CUDA_TRY(cudaEventRecord(g->ev[1], st));
  ZC_CUDA_TRY(launch_pr_normalize(rank, g->nv, g->d_ctr, false, st, &launches));
  ZC_CUDA_TRY(launch_pr_normalize(rank, g->nv, g->d_ctr, true, st, &launches));
  ZC_CUDA_TRY(cudaMemcpyAsync(out, rank, g->nv * sizeof(double), cudaMemcpyDeviceToHost, st));
  ZC_CUDA_TRY(cudaEventRecord(g->ev[2], st));
  ZC_CUDA_TRY(cudaStreamSynchronize(st));
  for (uint64_t k = 0; k < iters; ++k) {
    float e = 0;
    cudaEventElapsedTime(&e, g->iter_ev[2 * k], g->iter_ev[2 * k + 1]);
    g->log_expand_ms.push_back(e);
    expand_ms += e;
  }
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->iterations = iters;
    stats->total_traversed_edges = iters * g->ne;
    stats->max_frontier = g->nv;
    float ms = 0;
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    stats->kernel_ms = ms;
    cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]);
    stats->d2h_ms = ms;
    stats->d2h_bytes = g->nv * sizeof(double) + iters * sizeof(uint64_t);
    stats->launches = launches;
    stats->expand_ms = expand_ms;
    stats->total_ms = now_ms() - t0;
  }
  return ZC_OK;
}

int zc_graph_build_pairs(zc_graph* g) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (!g->has_weights || g->eb != 4 || g->wb != 4) {
    set_error("pairs need 4-byte edges and 4-byte weights");
    return ZC_EINVAL;
  }
  if (g->h_pairs) return ZC_OK;
  DeviceGuard dg(g->device);
  ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
  const uint64_t ne = g->ne;
  const size_t bytes = std::max<size_t>(ne * 8, kLineBytes);
  void* p = nullptr;
  if (g->placement == ZC_PLACE_UVM) ZC_CUDA_TRY(cudaMallocManaged(&p, bytes, cudaMemAttachGlobal));
  else if (!(p = host_list_alloc(g, bytes))) {
    set_error("cannot allocate host memory for a list");
    return ZC_ENOMEM;
  }
  g->h_pairs = p;
  const uint32_t* e = static_cast<const uint32_t*>(g->h_edges);
  const uint32_t* w = static_cast<const uint32_t*>(g->h_weights);
  uint64_t* out = static_cast<uint64_t*>(p);
  parallel_for(ne, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = uint64_t(e[i]) | (uint64_t(w[i]) << 32);
  });
  if (g->placement == ZC_PLACE_UVM) {
    ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseSetReadMostly, g->device));
    g->d_pairs = p;
  } else if (g->placement == ZC_PLACE_HBM) {
    ZC_CUDA_TRY(cudaMalloc(&g->hbm_pairs, bytes));
    ZC_CUDA_TRY(cudaMemcpy(g->hbm_pairs, p, ne * 8, cudaMemcpyHostToDevice));
    g->d_pairs = g->hbm_pairs;
  } else {
    return host_list_device_ptr(p, &g->d_pairs);
  }
  return ZC_OK;
}

int zc_graph_multigraph(zc_graph* g, int* out) {
  if (!g || !out) {
    set_error("null argument");
    return ZC_ESTATE;
  }
  if (g->multigraph < 0) {
    if (g->ne < 2) {
      g->multigraph = 0;
    } else {
      DeviceGuard dg(g->device);
      void* scratch = nullptr;
      ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
      ZC_CUDA_TRY(cudaMalloc(&scratch, g->ne * g->eb));
      ZC_CUDA_TRY(cudaMemcpy(scratch, g->h_edges, g->ne * g->eb, cudaMemcpyDefault));
      int rc = sort_lists_device(static_cast<int>(g->eb), g->nv, g->d_off, scratch);
      if (rc) {
        cudaFree(scratch);
        return rc;
      }
      ZC_CUDA_TRY(cudaMemset(g->d_ctr + kCtrBig, 0, sizeof(uint64_t)));
      ZC_CUDA_TRY(launch_dup_flags(scratch, static_cast<int>(g->eb), g->d_off, g->nv, g->d_ctr, 0));
      uint64_t flag = 0;
      ZC_CUDA_TRY(cudaMemcpy(&flag, g->d_ctr + kCtrBig, sizeof(flag), cudaMemcpyDeviceToHost));
      ZC_CUDA_TRY(cudaMemset(g->d_ctr + kCtrBig, 0, sizeof(uint64_t)));
      cudaFree(scratch);
      g->multigraph = flag ? 1 : 0;
    }
  }
  *out = g->multigraph;
  return ZC_OK;
}

int zc_run_link_bytes(const zc_graph* g, uint64_t* bytes) {
  if (!g || !bytes) {
    set_error("null argument");
    return ZC_ESTATE;
  }
  *bytes = g->h_small ? g->h_small[3] : 0;
  return ZC_OK;
}

int zc_run_directions(const zc_graph* g, uint8_t* bottom_up, uint64_t cap) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  const uint64_t n = std::min<uint64_t>(cap, g->log_pull.size());
  if (bottom_up) std::copy(g->log_pull.begin(), g->log_pull.begin() + n, bottom_up);
  return ZC_OK;
}

int zc_run_profile(const zc_graph* g, double* expand_ms, uint64_t cap) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  const uint64_t n = std::min<uint64_t>(cap, g->log_expand_ms.size());
  if (expand_ms) std::copy(g->log_expand_ms.begin(), g->log_expand_ms.begin() + n, expand_ms);
  return ZC_OK;
}

int zc_graph_evict(zc_graph* g) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (g->placement != ZC_PLACE_UVM || !g->ne) return ZC_OK;
  DeviceGuard dg(g->device);
  // Read-mostly pages keep their GPU duplicate across a prefetch to the
  // host, so collapse the duplicates first, migrate, then re-advise.
  auto cold = [&](void* p, size_t bytes) -> int {
    ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
    ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseUnsetReadMostly, g->device));
    ZC_CUDA_TRY(cudaMemPrefetchAsync(p, bytes, cudaCpuDeviceId, g->stream));
    ZC_CUDA_TRY(cudaStreamSynchronize(g->stream));
    ZC_CUDA_TRY(cudaMemAdvise(p, bytes, cudaMemAdviseSetReadMostly, g->device));
    return ZC_OK;
  };
  int rc = cold(g->h_edges, g->ne * g->eb);
  if (rc == ZC_OK && g->h_weights) rc = cold(g->h_weights, g->ne * g->wb);
  return rc;
}

int zc_graph_prefetch(zc_graph* g, float* ms) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (ms) *ms = 0;
  if (g->placement != ZC_PLACE_UVM || !g->ne) return ZC_OK;
  DeviceGuard dg(g->device);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ZC_CUDA_TRY(cudaEventCreate(&e0));
  if (cudaEventCreate(&e1) != cudaSuccess) {
    cudaEventDestroy(e0);
    set_error("cudaEventCreate failed");
    return ZC_ECUDA;
  }
  cudaError_t e = cudaEventRecord(e0, g->stream);
  if (e == cudaSuccess) e = cudaMemPrefetchAsync(g->h_edges, g->ne * g->eb, g->device, g->stream);
  if (e == cudaSuccess && g->h_weights)
    e = cudaMemPrefetchAsync(g->h_weights, g->ne * g->wb, g->device, g->stream);
  if (e == cudaSuccess) e = cudaEventRecord(e1, g->stream);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float t = 0;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ZC_CUDA_TRY(e);
  if (ms) *ms = t;
  return ZC_OK;
}

int zc_set_tuning(zc_graph* g, const char* spec) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  zc_graph::Tuning t;
  const std::string sp = spec ? spec : "";
  size_t pos = 0;
  while (pos < sp.size()) {
    size_t end = sp.find(',', pos);
    if (end == std::string::npos) end = sp.size();
    const std::string kv = sp.substr(pos, end - pos);
    pos = end + 1;
    if (kv.empty()) continue;
    const size_t eq = kv.find('=');
    const std::string k = kv.substr(0, eq);
    const std::string v = eq == std::string::npos ? "" : kv.substr(eq + 1);
    if (k == "unroll" && (v == "2" || v == "4" || v == "8" || v == "16")) t.unroll = std::stoi(v);
    else if (k == "ctas") t.ctas = std::max(0, atoi(v.c_str()));
    else if (k == "sched" && (v == "chunk" || v == "sweep")) t.sched = v == "chunk";
    else if (k == "loop" && (v == "host" || v == "device")) t.host_loop = v == "host";
    else if (k == "do_alpha" && atof(v.c_str()) > 0) t.do_alpha = atof(v.c_str());
    else if (k == "ld" && v.size() == 1 && v[0] >= '0' && v[0] <= '4') t.ld = v[0] - '0';
    else if (k == "pairs" && (v == "0" || v == "1")) t.pairs = v == "1";
    else if (k == "widen" && atoi(v.c_str()) > 0 && atoi(v.c_str()) <= 256) t.widen = atoi(v.c_str());
    else if (k == "uf_sample" && atoi(v.c_str()) > 0 && atoi(v.c_str()) <= 1024)
      t.uf_sample = atoi(v.c_str());
    else if (k == "sort" && (v == "radix" || v == "segmented")) t.seg_sort = v == "segmented";
    else if (k == "carveout" && !v.empty() && atoi(v.c_str()) >= 0 && atoi(v.c_str()) <= 100)
      t.carveout = atoi(v.c_str());
    else {
      set_error("unknown tuning entry '" + kv + "'");
      return ZC_EINVAL;
    }
  }
  g->tune = t;
  return ZC_OK;
}

int zc_set_options(zc_graph* g, uint32_t options) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (options & ~(ZC_OPT_TRAFFIC_MODEL | ZC_OPT_HOST_LOOP)) {
    set_error("unknown option bits");
    return ZC_EINVAL;
  }
  g->options = options;
  return ZC_OK;
}

int zc_run_traffic(const zc_graph* g, uint64_t* hist, uint64_t cap) {
  if (!g) {
    set_error("null graph handle");
    return ZC_ESTATE;
  }
  if (!(g->options & ZC_OPT_TRAFFIC_MODEL)) {
    set_error("traffic model not enabled (zc_set_options)");
    return ZC_ESTATE;
  }
  const uint64_t n = std::min<uint64_t>(cap, g->log_hist.size() / 8);
  if (hist) std::copy(g->log_hist.begin(), g->log_hist.begin() + 8 * n, hist);
  return ZC_OK;
}

int zc_graph_build_log(const zc_graph* g, char* buf, size_t cap) {
  if (!g || (!buf && cap)) {
    set_error("null argument");
    return ZC_ESTATE;
  }
  std::string out;
  for (const auto& e : g->build_log) out += e.first + " " + std::to_string(e.second) + "\n";
  if (cap) {
    const size_t n = std::min(cap - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return static_cast<int>(std::min<size_t>(out.size() + 1, 0x7fffffff));
}

void* zc_host_alloc(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  void* p = pinned_list_alloc(dev, bytes);
  if (!p) set_error("cannot allocate pinned host memory");
  return p;
}

void zc_host_free(void* p) { pinned_list_free(p); }

}  // extern "C"
