// Definition of the graph handle shared by the C-ABI (zc_api.cu) and the
// native generators (zc_gen.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <thread>
#include <string>
#include <utility>
#include <vector>

#include "../../include/zcgraph.h"
#include "zc_internal.cuh"

// Instantiated device-driven level loop (zc_api.cu build_loop_graph).
struct LoopGraph {
  int algo = -1, strategy = -1, ebytes = 0, unroll = 0, ctas = 0, ld = -1, carveout = -1;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t launches_per_iter = 0;
};
// log entries per array of the device loop (trav, front, t0, t1)
constexpr uint64_t kLogCap = 4096;

struct zc_graph {
  uint64_t nv = 0, ne = 0;
  uint32_t eb = 4, wb = 4;
  int32_t placement = ZC_PLACE_ZEROCOPY;
  int32_t device = 0;
  uint32_t flags = 0;
  int num_sms = 148;
  bool has_weights = false;
  bool negative_weight = false;
  // host side
  int64_t* h_off = nullptr;  // pinned copy of the offsets (V+1)
  void* h_edges = nullptr;   // pinned / managed / pinned shadow
  void* h_weights = nullptr;
  bool edges_registered = false, weights_registered = false;
  // device-visible lists
  const void* d_edges = nullptr;
  const void* d_weights = nullptr;
  void* hbm_edges = nullptr;
  void* hbm_weights = nullptr;
  // optional compressed line stream (zc_graph_build_compressed)
  void* h_cmp = nullptr;
  const void* d_cmp = nullptr;
  void* hbm_cmp = nullptr;
  uint64_t* d_cpos = nullptr;  // per-vertex bit position (| kCmpLong), V+1
  uint64_t cmp_bytes = 0;
  uint32_t cmp_ww = 0, cmp_wmin = 0;  // weight field width / offset (0: unweighted)
  uint32_t cmp_b0 = 32;               // bits of a short list's first element
  bool cmp_weighted = false;
  // direction-optimizing BFS: in-list offsets and the compressed in-list
  // stream (undirected graphs alias the out-lists), candidate marks and the
  // frontier bitmap of the bottom-up steps
  uint64_t* d_in_off = nullptr;
  void* h_cmp_in = nullptr;
  const void* d_cmp_in = nullptr;
  void* hbm_cmp_in = nullptr;
  uint64_t* d_cpos_in = nullptr;
  uint64_t cmp_in_bytes = 0;
  bool in_alias = false;
  uint8_t* d_cand = nullptr;
  uint32_t* d_fbits = nullptr;
  uint32_t* d_hasin = nullptr;  // vertices with in-edges (bitmap)
  // R-MAT partitions remember their generator, so their in-lists (arcs from
  // any rank into the owned range) can be generated on demand
  bool gen_rmat = false;
  uint32_t gen_scale = 0, gen_ef = 0;
  double gen_a = 0, gen_b = 0, gen_c = 0;
  uint64_t gen_seed = 0;
  uint64_t p_unvisited_in = 0;  // partition: owned unvisited vertices' in-edges
  // optional interleaved (dst, weight) u32 pairs for SSSP (zc_graph_build_pairs)
  void* h_pairs = nullptr;
  const void* d_pairs = nullptr;
  void* hbm_pairs = nullptr;
  // HBM state
  uint64_t* d_off = nullptr;
  void* d_state = nullptr;
  uint8_t* d_flags = nullptr;
  uint32_t* d_visited = nullptr;
  uint64_t vpad = 0, ntiles = 0;
  uint32_t* d_front[2] = {nullptr, nullptr};
  uint64_t* d_fval[2] = {nullptr, nullptr};
  uint64_t* d_fs[2] = {nullptr, nullptr};
  uint32_t* d_fd[2] = {nullptr, nullptr};
  uint32_t* d_tiles = nullptr;
  uint64_t* d_big_s = nullptr;
  uint64_t* d_big_e = nullptr;
  uint64_t* d_big_val = nullptr;
  uint64_t* d_big_prefix = nullptr;
  uint64_t* d_ctr = nullptr;
  uint32_t* d_wcnt = nullptr;  // per-slot window counts (CTA sweep)
  uint64_t* d_wpre = nullptr;  // their exclusive prefix
  void* d_scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
  uint64_t* h_ctr = nullptr;    // pinned
  uint64_t* h_small = nullptr;  // pinned staging for the source / initial values
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // last run's per-iteration log
  std::vector<uint64_t> log_trav, log_front;
  std::vector<uint8_t> log_pull;  // direction-optimizing: 1 = bottom-up step
  std::vector<uint64_t> log_hist;  // 8 per iteration (ZC_OPT_TRAFFIC_MODEL)
  std::vector<double> log_expand_ms;
  std::vector<cudaEvent_t> iter_ev;  // 2 per iteration, grown on demand
  uint32_t options = 0;
  // launch tuning (zc_set_tuning; read by the run path, never from the environment)
  struct Tuning {
    int unroll = 0;   // windows per warp batch in the sweep (2 / 4 / 8; 0: the strategy's)
    int ctas = 0;     // sweep CTAs per SM (0: occupancy maximum)
    int sched = 0;    // 1: the round-1 chunk scheduler instead of the sweep
    int host_loop = 0;  // 1: host-driven level loop (profilers cannot see graph kernels)
    double do_alpha = 2.0;  // direction-optimizing switch factor
    int ld = -1;      // load flavour override of the raw BFS sweeps (zc_kernels.cu DefaultLd)
    int pairs = 1;    // SSSP on merged / merged-aligned / packed: build + read the pairs stream
    int carveout = -1;  // sweep kernels' preferred shared-memory carveout (%, -1: default)
    int widen = 0;      // host threads of an overlapped result widen (0: 4)
    int uf_sample = 0;  // afforest sampling pass on compressed lists (0: kUfSample)
    int seg_sort = 0;   // 1: compressed builds sort by count/scatter + segmented sort, not radix transposes
  } tune;
  int multigraph = -1;  // cached duplicate-arc check (-1 unknown)
  // one-time builds (compressed streams, pairs): wall ms per phase, in order
  std::vector<std::pair<std::string, double>> build_log;
  double build_t = 0;
  LoopGraph loop;
  uint64_t* d_log = nullptr;  // 4 * kLogCap
  // vertex-range partition (multi-GPU); nparts == 0 for a whole graph
  uint32_t nparts = 0, part = 0;
  uint64_t global_nv = 0, lo = 0, stride = 0;
  uint64_t* d_part_lo = nullptr;  // nparts + 1
  // fused exchange: own candidate buffer (stride slots of <= 8 bytes), the
  // owners' buffers (device array of nparts pointers), IPC-opened peers
  void* d_mine = nullptr;
  void** d_peers = nullptr;
  uint32_t* d_sent = nullptr;  // BFS: discoveries already sent this iteration
  // BFS bitmap exchange: the ranks' `sent` bitmaps (device array of nparts
  // pointers; peers' through CUDA IPC), read by each owner for its range
  const uint32_t** d_peer_sent = nullptr;
  bool peer_sent_ready = false;  // zc_part_bitmap_connect done
  bool peers_ready = false;      // zc_part_fused_connect done
  std::vector<void*> ipc_opened_sent;
  void* d_lbest = nullptr;     // SSSP / CC: best candidate sent per global vertex this iteration
  std::vector<void*> ipc_opened;
  int fused_algo = -1;
  // pipelined results (zc_bfs_async / zc_sssp_async / zc_sync): two int64
  // staging slots widened on the run stream, downloaded on copy_stream while
  // the next traversal streams the edge list
  cudaStream_t copy_stream = nullptr;
  int64_t* d_outbuf[2] = {nullptr, nullptr};
  cudaEvent_t out_ready[2] = {nullptr, nullptr}, out_done[2] = {nullptr, nullptr};
  uint32_t out_next = 0;
  // narrowed BFS results: pinned u8 staging per slot, widened to int64 on the
  // host by a worker thread while the next traversal runs
  uint8_t* h_stage[3] = {nullptr, nullptr, nullptr};  // [2]: the blocking path
  std::thread widen_th[2];
  int widen_err = 0;
  // stepped run state (zc_part_begin / expand / apply)
  int p_algo = -1, p_strategy = 0, p_cur = 0;
  uint64_t p_iter = 0, p_n = 0, p_launches = 0;
  uint64_t p_xbytes = 0;  // exchange bytes this rank sent since zc_part_begin
};


namespace zc {
// zc_api.cu
void free_graph(zc_graph* g);
// Build-phase timing: build_start resets the clock, build_mark(g, "x")
// synchronizes the device and logs the wall ms since the previous mark.
void build_start(zc_graph* g);
void build_mark(zc_graph* g, const char* phase);
int alloc_state(zc_graph* g);
int finish_create(zc_graph* g);  // prefetch (UVM) + sync
int init_partition(zc_graph* g, const zc_part_info* info);
// pinned mapped list buffers, NUMA-local to the GPU when the host has several nodes
void* pinned_list_alloc(int device, size_t bytes);
// pinned_list_alloc in two halves: the prefaulted huge-page mapping (no CUDA
// calls, so another thread can run it beside device work; p == nullptr when
// small or failed), then its registration (cudaHostAlloc on any failure).
struct HostMap {
  void* p = nullptr;
  size_t bytes = 0;
};
HostMap pinned_list_map(int device, size_t bytes);
void* pinned_list_finish(HostMap m, size_t bytes);
void pinned_list_unmap(HostMap m);

void pinned_list_free(void* p);
// Host-side list buffer of a handle: pinned (ZEROCOPY, and the HBM run's
// shadow) or host-resident managed memory (ZEROCOPY_MANAGED).  Freed with
// pinned_list_free; host_list_device_ptr gives the address kernels use.
void* host_list_alloc(const zc_graph* g, size_t bytes);
int host_list_device_ptr(void* p, const void** d);
// Compress the handle's sorted in-lists (device offsets + u32 lists, both
// over the handle's own vertices) into its in-list line stream; takes
// ownership of d_in_off (zc_compress.cu).
int install_in_lists(zc_graph* g, uint64_t* d_in_off, uint32_t* d_in_sorted);
// Candidate marks, frontier bitmap and in-edge bitmap of the bottom-up steps
// (once the in-lists exist).
int alloc_pull_state(zc_graph* g);
// In-lists of a generated R-MAT partition (zc_gen.cu).
int part_in_lists(zc_graph* g);
inline bool placement_valid(int32_t p) { return p >= ZC_PLACE_ZEROCOPY && p <= ZC_PLACE_ZEROCOPY_MANAGED; }
// Adopt a list generated in HBM (d_src, n elements of width w) into the
// handle's placement; frees d_src unless it becomes the HBM copy.
int adopt_device_list(zc_graph* g, void* d_src, uint32_t w, uint64_t n, void** h,
                      const void** dptr, void** hbm);
}  // namespace zc
