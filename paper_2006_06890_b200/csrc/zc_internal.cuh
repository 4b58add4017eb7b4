// Internal declarations shared by the zcgraph B200 translation units.
//
// Layout in HBM (per handle, allocated once at create, reused by every run):
//   off      u64[V+1]      CSR vertex list (the paper keeps it on the GPU,
//                          PAPER.md:452-455)
//   state    u64[V]        BFS: u32 level[V] (0xffffffff = unreached);
//                          SSSP: u64 dist[V] (UINT64_MAX = unreached);
//                          CC: u32 label[V]
//   visited  u32[V/32]     BFS visited bitmap (L2-resident filter for level[])
//   flags    u8[Vpad]      "improved / discovered this iteration" marks,
//                          Vpad = V rounded up to the compaction tile
//   front    u32[V] x2     frontier (sorted ascending, like traversal.py:117/150)
//   fval     u64[V] x2     start-of-iteration value of each frontier vertex
//                          (Jacobi snapshot, traversal.py:147,175)
//   fs, fd   u64[V], u32[V] x2  list start / degree of each frontier vertex
//                          (written by the compaction: expansion needs no
//                          dependent offsets gather)
//   tiles    u32[ntiles]   per-tile counts / offsets of the compaction
//   big_*    u64[V] x3 + u64[V+1]  lists split across all warps
//                          (degree-binned scheduling): start, end, value,
//                          exclusive prefix of their window counts
//   ctr      u64[8]        device counters (next size, traversed sum, ...)
// Edge / weight lists: pinned mapped host memory (zero-copy), managed memory
// (UVM) or HBM (control), all 128-byte aligned.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

struct zc_graph;

namespace zc {

constexpr int kWarp = 32;
constexpr int kLineBytes = 128;
constexpr int kTileThreads = 256;
constexpr int kTileVerts = kTileThreads * 16;  // 16 flag bytes (one uint4) per thread
constexpr uint32_t kUnreached32 = 0xffffffffu;
constexpr uint64_t kUnreached64 = ~0ull;
// "no candidate" in the partition exchange buffers: signed maxima, so the
// buffers reduce correctly as int64 / int32 MIN in NCCL and gloo.
constexpr uint64_t kExchNone64 = 0x7fffffffffffffffull;
constexpr uint32_t kExchNone32 = 0x7fffffffu;
// A frontier vertex whose list needs more than kBigSteps warp steps is not
// expanded by its chunk warp but queued and split across all warps.
constexpr uint32_t kBigSteps = 16;

enum Strategy : int {
  kNaive = 0,
  kMerged = 1,
  kMergedAligned = 2,
  kPacked = 3,
  kCompressed = 4,
  kDirOpt = 5  // BFS: compressed top-down + bottom-up steps over the compressed in-lists
};
// kCompressed (B200 host-store option, zc_compress.cu): every list is stored
// sorted and delta-encoded in a stream of 128-byte lines, in vertex order.
//   short list (encoding <= 2048 bits, <= 96 elements): packed with its
//     neighbours into a shared 256-byte span (two lines), never straddling
//     one -- 6-bit delta width w, the first element in cmp_b0 bits (bits of
//     the largest vertex id), d-1 deltas of w bits, then (weighted) d weights
//     of ww bits (weight - wmin);
//   long list: whole self-describing lines -- word 0 base, word 1 [0,6) w,
//     [6,14) count - 1 (<= 255); from bit 48: count-1 deltas of w bits, then
//     (weighted) count weights of ww bits.
// Per-vertex cpos (u64[V+1], HBM): bit position of the list in the stream,
// kCmpLong and the line count for long lists (layout below).
// A window is one long-list line, or one shared span of short lists fetched
// once for all its frontier lists.
constexpr uint32_t kCmpHdrBits = 48;
// A short list's header: the 6-bit delta width, then the first element in
// b0 = bits(largest vertex id) bits (cmp_b0; at most 32).
constexpr uint32_t kCmpShortWidthBits = 6;
constexpr uint32_t kCmpMaxCount = 256;
constexpr uint32_t kLineWords = 32;
constexpr uint32_t kLineBits = 1024;
constexpr uint32_t kCmpShortMaxDeg = 96;
// Afforest's sampling pass over compressed lists reads this many elements of
// each short list and one per lane of a long list's first line (the rest of a
// list outside the giant component is read by the second pass).
constexpr uint32_t kUfSample = 4;
// Short lists are packed into 256-byte spans (two lines) and never straddle
// one: a U27 SSSP list (540 bits) then shares its span with two others.
constexpr uint32_t kShortSpanBits = 2 * kLineBits;
constexpr uint32_t kShortSpanWords = 2 * kLineWords;
// cpos word: bit 63 = long list; bits [40, 63) = a long list's line count
// (padding may follow it, so it is not the gap to the next list); bits
// [0, 40) = the bit position in the stream (streams up to 128 GiB).
constexpr uint64_t kCmpLong = 1ull << 63;
constexpr int kCmpPosBits = 40;
constexpr uint64_t kCmpPosMask = (1ull << kCmpPosBits) - 1;
constexpr uint64_t kCmpMaxLines = (1ull << (63 - kCmpPosBits)) - 1;
__host__ __device__ __forceinline__ uint64_t cmp_pos(uint64_t c) { return c & kCmpPosMask; }
__host__ __device__ __forceinline__ uint64_t cmp_lines(uint64_t c) {
  return (c & ~kCmpLong) >> kCmpPosBits;
}
// kPacked (B200 extension, not one of the paper's three): a window is an
// aligned 32-element block touched by any frontier list, fetched once for all
// the lists that share it (see k_window_counts / k_expand_sweep).
enum Algo : int { kBfs = 0, kSssp = 1, kCc = 2, kPr = 3 };
// Partitioned (multi-GPU) variants: the visit writes candidates for any
// global vertex into the exchange buffer instead of updating local state.
constexpr int kPartAlgo = 4;  // algo + kPartAlgo
// Bottom-up BFS step (direction-optimizing strategy): the slots are the
// unvisited candidates, their in-lists are scanned for a parent in the
// current frontier (frontier bitmap), the slot's vertex is the value.
constexpr int kBfsPull = 8;
// Connected components by union-find (the "afforest" schedule, B200
// extension): the slot's value is its vertex id, the visit unions the two
// endpoints' trees (parents in the u32 state, always pointing to smaller ids,
// so every root is its component's minimum id -- the reference's label).
constexpr int kCcUf = 9;
template <int A>
struct AlgoTraits {
  static constexpr bool pull = A == kBfsPull;
  static constexpr bool uf = A == kCcUf;
  static constexpr int base = pull ? kBfs : uf ? kCc : A % kPartAlgo;
  static constexpr bool part = A >= kPartAlgo && !pull && !uf;
  static constexpr bool has_val = base != kBfs || pull;  // slot carries a value
  static constexpr bool weighted = base == kSssp;
};

// device counter slots
enum Ctr : int {
  kCtrNext = 0,      // size of the next frontier
  kCtrTrav = 1,      // sum of degrees of the next frontier
  kCtrBig = 2,       // entries in the big-list queue
  kCtrBigSteps = 3,  // total warp steps of the big-list queue
  kCtrPrDangling = 4,  // PageRank: dangling mass (double bits)
  kCtrPrDelta = 5,     //   L1 change of the iteration
  kCtrPrSum = 6,       //   sum of ranks
  kCtrTravIn = 7,    // sum of in-degrees of the next frontier (compaction with in_off)
  kCtrHist = 8,      // 8..11 modelled edge requests of 1..4 sectors, 12..15 weights
  kCtrCur = 16,      // device level loop: size of the current frontier
  kCtrIter = 17,     //   completed iterations
  kCtrLoaded = 18,   // compressed sweeps: bytes requested from the line streams
  kCtrVisited = 19,  // union-find sweeps: list elements actually read (afforest pass 1)
  kCtrRemote = 20,   // fused partitions: remote destinations sent to (launch_count_remote)
  kCtrFarMin = 22,   // near-far SSSP: smallest distance in the far pile
  kCtrFar = 23,      //   vertices in the far pile
  kCtrCount = 24
};

struct ExpandArgs {
  const uint32_t* front;  // frontier vertex ids
  const uint64_t* fs;     // list start of each frontier vertex
  const uint32_t* fd;     // degree of each frontier vertex
  const uint64_t* fval;   // snapshot values (SSSP dist / CC label)
  uint64_t n;             // frontier size
  const uint64_t* off;    // CSR offsets (HBM)
  const void* edges;      // edge list (zero-copy / managed / HBM)
  const void* weights;    // weight list (SSSP)
  void* state;            // level / dist / label
  uint8_t* flags;         // next-frontier marks
  uint32_t* visited;      // BFS visited bitmap ((V + 31) / 32 words)
  uint32_t iter;          // BFS: level assigned to newly reached vertices
  uint64_t* big_s;        // big-list queue: list start,
  uint64_t* big_e;        //   list end,
  uint64_t* big_val;      //   snapshot value
  uint64_t* big_prefix;   // exclusive prefix of big-list steps (nbig+1)
  uint64_t* ctr;          // device counters
  // partitioned mode: exchange buffer of nparts * stride slots; global
  // vertex w of part k lives in slot k * stride + (w - part_lo[k])
  void* exch;
  const uint64_t* part_lo;  // nparts + 1 range starts (device)
  uint32_t nparts;
  uint64_t stride;
  // fused mode: owners' buffers reached directly (NVLink peer pointers);
  // `sent` dedups BFS discoveries per iteration (global V bits)
  void* const* peers;
  uint32_t* sent;
  int sent_only;  // BFS bitmap exchange: discoveries only set `sent` bits
  // fused SSSP / CC: this rank's best candidate per global vertex this
  // iteration (u64 / u32, all ones = none); only improvements go to the owner
  void* lbest;
  // CTA-sweep scheduling: per-slot window counts, their exclusive prefix
  uint32_t* wcnt;
  uint64_t* wpre;  // n + 1
  void* scan_tmp;
  size_t scan_tmp_bytes;
  // launch tuning (host side only; zc_set_tuning)
  int unroll;
  int ctas_per_sm;
  int carveout;     // sweep kernels' preferred shared-memory carveout (%, -1: driver default)
  int chunk_sched;  // 1: the per-warp chunk + big-list scheduler instead of the sweep
  int ld;           // load flavour override of the raw BFS sweeps (-1: the strategy's default)
  int pairs;        // SSSP: `edges` is the interleaved (dst, weight) u32-pair list
  // device-driven level loop: frontier size / completed iterations in device
  // memory (then `n` is only the maximum, used to size grids)
  const uint64_t* n_dev;
  const uint64_t* iter_dev;
  // compressed lists (kCompressed): the line stream, each vertex's bit
  // position (kCmpLong: whole lines), the weight field width and offset
  const uint32_t* cmp;
  const uint64_t* cpos;
  uint32_t cmp_ww;
  uint32_t cmp_wmin;
  uint32_t cmp_b0;  // bits of a short list's first element
  // bottom-up step (kBfsPull): bitmap of the current frontier; pass 1 reads
  // every candidate's first line (short lists whole), pass 2 the remaining
  // lines of the long in-lists still without a parent (0: one pass, all)
  const uint32_t* fbits;
  uint32_t pull_pass;
  // union-find sampling pass (kCcUf, pull_pass 1) over compressed lists:
  // elements read per short list, and per lane of a long list's first line
  // when below kCmpShortMaxDeg (>= kCmpShortMaxDeg: short lists and the first
  // line whole)
  uint32_t uf_sample;
};

// Expansion tuning knobs of a handle (zc_set_tuning "unroll=8,ctas=6,sched=chunk").
void tune_params(ExpandArgs* a, const ::zc_graph* g);

struct CompactArgs {
  uint8_t* flags;
  uint64_t nv;
  uint64_t ntiles;
  uint32_t* tiles;          // per-tile counts, then offsets
  uint32_t* front_out;
  uint64_t* fs_out;
  uint32_t* fd_out;
  uint64_t* fval_out;
  const uint64_t* off;
  const void* state;
  uint64_t* ctr;
  const uint64_t* in_off;  // optional: also sum the in-degrees into ctr[kCtrTravIn]
  // near-far SSSP: only marked vertices with dist < thresh join the frontier;
  // the others stay marked (the far pile).  0 = every marked vertex.
  uint64_t thresh;
};

// Launchers (zc_kernels.cu).  All launch on `st`; return cudaError_t.
cudaError_t launch_expand(int strategy, int algo, int edge_bytes, int weight_bytes,
                          const ExpandArgs& a, int num_sms, cudaStream_t st, uint64_t* launches);
// The reference's request model (coalesce.py:165-207) of one frontier,
// accumulated into ctr[kCtrHist..kCtrHist+7].
cudaError_t launch_traffic_model(int strategy, int edge_bytes, int weight_bytes, bool weights,
                                 const uint32_t* front, uint64_t n, const uint64_t* off,
                                 uint64_t* ctr, int num_sms, cudaStream_t st, uint64_t* launches);
cudaError_t launch_compact(int algo, const CompactArgs& c, cudaStream_t st, uint64_t* launches);
// Bottom-up step inputs: zero + set the frontier bitmap from front[0, n), and
// mark (u8 per vertex, padded to 16) every unvisited vertex with in-edges.
cudaError_t launch_pull_prepare(const uint32_t* front, uint64_t n, uint32_t* fbits, uint64_t nv,
                                const uint32_t* visited, const uint32_t* hasin, uint8_t* cand,
                                int num_sms, cudaStream_t st, uint64_t* launches);
// Bitmap of the vertices with in-edges ((nv + 31) / 32 words).
cudaError_t launch_hasin(uint64_t nv, const uint64_t* in_off, uint32_t* bits, cudaStream_t st);
cudaError_t launch_init(int algo, void* state, uint64_t nv, uint64_t src, const uint64_t* off,
                        uint32_t* front, uint64_t* fval, uint64_t* fs, uint32_t* fd,
                        cudaStream_t st, uint64_t* launches, uint64_t label_base = 0,
                        bool with_source = true);
// Partitioned mode: owner-side merge of this part's reduced exchange slice
// (BFS: flags / SSSP: u64 candidates / CC: u32 candidates) into the local
// state, marking improved vertices for the compaction.
cudaError_t launch_fill_exchange(int algo, void* x, uint64_t n, cudaStream_t st,
                                 uint64_t* launches);
cudaError_t launch_part_apply(int algo, const void* mine, uint64_t nlocal, void* state,
                              uint8_t* flags, uint32_t iter, cudaStream_t st, uint64_t* launches);
// BFS bitmap exchange: OR the nparts ranks' discovery bitmaps over this
// part's range [lo, lo + nlocal) (peer memory) and apply them like
// launch_part_apply.
cudaError_t launch_part_pull_apply(const uint32_t* const* sent, uint32_t nparts, uint64_t lo,
                                   uint64_t nlocal, void* state, uint8_t* flags, uint32_t iter,
                                   int num_sms, cudaStream_t st, uint64_t* launches);
// Fused exchange accounting: how many global vertices outside [lo, hi) this
// rank sent a candidate to this iteration -- set bits of the BFS `sent`
// bitmap (elem_bytes 0) or entries of `lbest` other than all-ones (4 / 8) --
// added to *out (device).
cudaError_t launch_count_remote(const void* x, int elem_bytes, uint64_t global_nv, uint64_t lo,
                                uint64_t hi, uint64_t* out, int num_sms, cudaStream_t st,
                                uint64_t* launches);
// Frontier bitmap over global ids: zero `words` words, set vbase + front[j].
cudaError_t launch_frontier_bits(const uint32_t* front, uint64_t n, uint64_t vbase,
                                 uint32_t* bits, uint64_t words, int num_sms, cudaStream_t st,
                                 uint64_t* launches);
// Partition bottom-up inputs: the owned range's visited bitmap from its
// levels, then the candidate marks.
cudaError_t launch_part_pull_prepare(const void* level, uint64_t nv, uint32_t* visited,
                                     const uint32_t* hasin, uint8_t* cand, int num_sms,
                                     cudaStream_t st, uint64_t* launches);
// Near-far SSSP: ctr[kCtrFarMin] = min dist over the marked vertices,
// ctr[kCtrFar] = their count (both reset first).
cudaError_t launch_far_min(const uint8_t* flags, const void* dist, uint64_t nv, uint64_t* ctr,
                           cudaStream_t st, uint64_t* launches);
// Union-find CC helpers: parent[v] = root (full compression); `sample`
// roots of hashed vertices into out[sample]; marks of the vertices outside
// component `giant` whose lists reach past the first window (pass 2);
// fval[j] = front[j].
cudaError_t launch_uf_flatten(uint32_t* parent, uint64_t nv, cudaStream_t st, uint64_t* launches);
cudaError_t launch_uf_sample(const uint32_t* parent, uint64_t nv, uint32_t* out, uint32_t sample,
                             cudaStream_t st, uint64_t* launches);
cudaError_t launch_uf_marks(const uint32_t* parent, const uint64_t* off, const uint64_t* cpos,
                            uint64_t nv, uint32_t giant, int strategy, int edge_bytes,
                            uint32_t uf_sample, uint8_t* flags, cudaStream_t st,
                            uint64_t* launches);
cudaError_t launch_fval_ids(const uint32_t* front, uint64_t* fval, uint64_t n, cudaStream_t st,
                            uint64_t* launches);
// BFS levels (all below 255) as u8, 0xff = unreached.
cudaError_t launch_narrow_levels(const void* state, uint64_t nv, uint8_t* out, cudaStream_t st,
                                 uint64_t* launches);
cudaError_t launch_widen(int algo, const void* state, uint64_t nv, int64_t* out, cudaStream_t st,
                         uint64_t* launches);
cudaError_t launch_check_edges(const void* edges, int edge_bytes, uint64_t ne, uint64_t nv,
                               uint64_t* bad, cudaStream_t st);

// PageRank (traversal.py:191-249) per-iteration helpers.
cudaError_t launch_pr_init(uint64_t nv, const uint64_t* off, uint32_t* front, uint64_t* fs,
                           uint32_t* fd, double* rank, cudaStream_t st, uint64_t* launches);
cudaError_t launch_pr_prepare(const double* rank, const uint32_t* deg, uint64_t nv, uint64_t* fval,
                              double* pushed, uint64_t* ctr, cudaStream_t st, uint64_t* launches);
cudaError_t launch_pr_update(double* rank, const double* pushed, uint64_t nv, double damping,
                             uint64_t* ctr, cudaStream_t st, uint64_t* launches);
cudaError_t launch_pr_normalize(double* rank, uint64_t nv, uint64_t* ctr, bool divide,
                                cudaStream_t st, uint64_t* launches);
cudaError_t launch_dup_flags(const void* sorted, int elem_bytes, const uint64_t* off, uint64_t nv,
                             uint64_t* ctr, cudaStream_t st);
// Sort every list ascending in place (device array, zc_gen.cu).
// (u32 lists: radix transposes first unless radix == false, then the segmented sort)
int sort_lists_device(int elem_bytes, uint64_t nv, const uint64_t* d_off, void* edges,
                      bool radix = true);
float last_sort_gpu_ms();  // GPU time of this thread's last list sort
void set_sort_gpu_ms(float ms);
// Lists sorted in place by two radix transposes (zc_compress.cu); ZC_ENOMEM
// (untouched) when the three edge-sized scratch buffers do not fit.
int sort_lists_radix(uint64_t nv, const uint64_t* d_off, uint32_t* edges, uint64_t ne,
                     uint64_t nk);
// *yes = every list (offsets d_off, device) ascending
cudaError_t lists_ascending(uint64_t nv, const uint64_t* d_off, const uint32_t* edges, bool* yes);

// Exclusive scan of u32 counts into u64 offsets (n+1 outputs), device-wide.
cudaError_t scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp,
                            size_t tmp_bytes, cudaStream_t st, const uint64_t* n_dev = nullptr);
// device level loop (CUDA graph with a conditional while node)
cudaError_t launch_level_end(uint64_t* ctr, uint64_t* log_trav, uint64_t* log_front, uint64_t cap,
                             cudaGraphConditionalHandle loop, cudaStream_t st);
cudaError_t launch_stamp(const uint64_t* ctr, uint64_t* log_t, cudaStream_t st);
size_t scan_tmp_bytes(uint64_t n);

// error plumbing (zc_api.cu)
void set_error(const std::string& msg);

}  // namespace zc

#define ZC_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::zc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
      return ZC_ECUDA;                                                                 \
    }                                                                                  \
  } while (0)
