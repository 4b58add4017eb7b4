// Traversal kernels for sm_100a: frontier expansion under the three EMOGI
// access strategies, frontier compaction, init / widen helpers.
//
// The lane -> element maps follow the reference access engine exactly
// (/root/reference/pkg/src/zcgraph/access.py):
//   naive           access.py:146-156, 195-216: lane i of warp w carries
//                   frontier[32w+i]; each lane walks its own list one element
//                   per step.
//   merged          access.py:70-97, 171-192: one warp per list, step k covers
//                   elements [s+32k, s+32k+32) & [s,e).
//   merged-aligned  same with the first window floored to a 128-byte line:
//                   a = s & ~0x1F (4-byte elements) / s & ~0xF (8-byte),
//                   access.py:34-37; lanes outside [s,e) are masked.
// Weight reads (SSSP) reuse the edge windows (access.py:100-106, 183).
//
// What is B200-specific here (not in the reference, which has no GPU code):
//   * a warp owns a chunk of 32 consecutive frontier slots, loads their
//     (v, s, e, value) with one coalesced gather and then walks the flattened
//     sequence of their warp steps, keeping kUnroll independent 128-byte
//     line requests in flight per warp (memory-level parallelism for the
//     ~1-2 us PCIe round trip);
//   * lists longer than kBigSteps steps are queued and their steps are spread
//     evenly over every warp of the grid (degree-binned scheduling, so a
//     Kronecker hub does not serialise one warp);
//   * Jacobi semantics of the reference SSSP / CC (cand computed from the
//     start-of-iteration values, traversal.py:147,175) are kept by carrying
//     each frontier vertex's value in the frontier itself; results, iteration
//     counts and per-iteration traversed edges equal the reference's.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "zc_internal.cuh"

namespace zc {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kExpandThreads = 256;
constexpr int kUnroll = 4;

// ---------------------------------------------------------------- loads
// Edge / weight reads: the lists are read exactly once per expansion, so
// keep them out of L1 (.L1::no_allocate).  Works for host-mapped (sysmem),
// managed and device pointers alike.
__device__ __forceinline__ uint32_t ld_list(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_list(const uint64_t* p) {
  uint64_t v;
  asm("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// Load flavours of the raw-list sweep: 0 = L1::no_allocate, 1 = cached in L1
// (.ca), 2 = the read-only path (.nc), 3 = L1::evict_first.  Merged and
// merged-aligned read the reference's per-list windows, so two adjacent
// frontier lists that share a 128-byte line each request it; cached in L1 the
// second request is served on the SM while the line stays there (K27 BFS,
// merged-aligned: 234 -> 212 ms; the tiny-list level 46.6 -> 32.0 ms).
// Packed / compressed fetch each line once by construction: no_allocate.
// zc_set_tuning "ld=N" overrides the flavour of the BFS u32 sweeps for A/B.
template <int STRAT>
struct DefaultLd {
  static constexpr int value = STRAT == kMerged || STRAT == kMergedAligned ? 1 : 0;
};
template <int LD>
__device__ __forceinline__ uint32_t ld_list_f(const uint32_t* p) {
  uint32_t v;
  if constexpr (LD == 1) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if constexpr (LD == 2) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if constexpr (LD == 3) asm volatile("ld.global.L1::evict_first.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else v = ld_list(p);
  return v;
}
template <int LD, typename T>
__device__ __forceinline__ T ld_list_f(const T* p) {
  return ld_list(p);
}

// Interleaved (destination, weight) u32 pairs in one 8-byte element stream
// (zc_graph_build_pairs): the weight rides in the high half, no second load.
struct PairW {};
template <typename WT>
struct IsPair {
  static constexpr bool value = false;
};
template <>
struct IsPair<PairW> {
  static constexpr bool value = true;
};

// ---------------------------------------------------------------- visitors
// Apply one traversed edge (v -> w, weight wt) whose source carries the
// start-of-iteration value `val`.
template <int ALGO>
struct Visit;

template <>
struct Visit<kBfs> {
  // traversal.py:116-118: unvisited neighbours get level = iteration.  The
  // check goes to a visited bitmap (V/8 bytes, L2-resident) instead of the
  // level array, and the atomicOr elects the one writer of each new level.
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t) {
    uint32_t* word = a.visited + (w >> 5);
    const uint32_t bit = 1u << (w & 31);
    if (!(*word & bit) && !(atomicOr(word, bit) & bit)) {
      static_cast<uint32_t*>(a.state)[w] = a.iter;
      a.flags[w] = 1;
    }
  }
};

template <>
struct Visit<kBfsPull> {
  // Bottom-up: w is an in-neighbour of the candidate u; u joins the next
  // level when w is in the current frontier (the same level traversal.py
  // :116-118 gives it top-down).  The visited bitmap elects one writer.
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t u) {
    if (!(a.fbits[w >> 5] & (1u << (w & 31)))) return;
    uint32_t* word = a.visited + (u >> 5);
    const uint32_t bit = 1u << (u & 31);
    if (!(*word & bit) && !(atomicOr(word, bit) & bit)) {
      static_cast<uint32_t*>(a.state)[u] = a.iter;
      a.flags[u] = 1;
    }
  }
};

__device__ __forceinline__ bool is_visited(const ExpandArgs& a, uint64_t u) {
  return (a.visited[u >> 5] >> (u & 31)) & 1u;
}

template <>
struct Visit<kSssp> {
  // traversal.py:146-150: cand = dist_old[v] + w; dist = min(dist, cand);
  // improved vertices form the next frontier.
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t wt,
                                               uint64_t val) {
    unsigned long long* dist = static_cast<unsigned long long*>(a.state);
    const unsigned long long cand = val + wt;
    if (cand < dist[w]) {
      const unsigned long long old = atomicMin(dist + w, cand);
      if (cand < old) a.flags[w] = 1;
    }
  }
};

template <>
struct Visit<kCc> {
  // traversal.py:174-178: cand = label_old[v]; label = min(label, cand).
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t val) {
    unsigned* label = static_cast<unsigned*>(a.state);
    const unsigned cand = static_cast<unsigned>(val);
    if (cand < label[w]) {
      const unsigned old = atomicMin(label + w, cand);
      if (cand < old) a.flags[w] = 1;
    }
  }
};

// PageRank sums are fixed point (value x 2^62 in a u64): integer atomics add
// in any order to the same bits, so ranks, the L1 change and with it the
// iteration count do not depend on the schedule (a float64 atomicAdd does).
// Every PageRank sum is below 4 (ranks sum to 1); the quantum 2^-62 ~ 2e-19.
constexpr double kPrFx = 4611686018427387904.0;  // 2^62
__device__ __forceinline__ unsigned long long pr_fx(double x) { return __double2ull_rn(x * kPrFx); }
__device__ __forceinline__ double pr_unfx(unsigned long long v) {
  return __ull2double_rn(v) * (1.0 / kPrFx);
}

// Union-find with min-hooking (lock-free: a root is hooked by one CAS; path
// halving stores only move non-roots closer to their root).  Parents always
// point to smaller ids, so a root is the minimum id of its tree.
__device__ __forceinline__ uint32_t uf_find(uint32_t* p, uint32_t x) {
  uint32_t par = __ldcg(p + x);
  if (par == x) return x;
  uint32_t prev = x, next;
  while (par > (next = __ldcg(p + par))) {
    __stcg(p + prev, next);
    prev = par;
    par = next;
  }
  return par;
}

__device__ __forceinline__ void uf_union(uint32_t* p, uint32_t u, uint32_t v) {
  uint32_t ru = uf_find(p, u), rv = uf_find(p, v);
  while (ru != rv) {
    if (ru < rv) {
      const uint32_t t = ru;
      ru = rv;
      rv = t;
    }
    const uint32_t old = atomicCAS(p + ru, ru, rv);  // hook the larger root
    if (old == ru) return;
    ru = uf_find(p, old);
    rv = uf_find(p, rv);
  }
}

template <>
struct Visit<kCcUf> {
  // edge v -> w of an undirected graph: v and w are connected
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t v) {
    uf_union(static_cast<uint32_t*>(a.state), static_cast<uint32_t>(v),
             static_cast<uint32_t>(w));
  }
};

template <>
struct Visit<kPr> {
  // traversal.py:229: pushed[d] += rank[s] / out[s]; the contribution rides in
  // the frontier value slot (fixed point, pr_fx); pushed (u64) lives in a.exch.
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t val) {
    atomicAdd(static_cast<unsigned long long*>(a.exch) + w, static_cast<unsigned long long>(val));
  }
};

// Owner part of global vertex w.
__device__ __forceinline__ uint32_t part_of(const ExpandArgs& a, uint64_t w) {
  uint32_t lo = 0, hi = a.nparts;  // part_lo[lo] <= w < part_lo[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a.part_lo[mid] <= w) lo = mid; else hi = mid;
  }
  return lo;
}

// Candidate slot of w: in the local exchange buffer (reduce-scatter mode) or,
// fused mode, directly in the owner's buffer (peer pointer over NVLink).
template <typename T>
__device__ __forceinline__ T* cand_slot(const ExpandArgs& a, uint64_t w) {
  const uint32_t k = part_of(a, w);
  if (a.peers) return static_cast<T*>(a.peers[k]) + (w - a.part_lo[k]);
  return static_cast<T*>(a.exch) + (k * a.stride + (w - a.part_lo[k]));
}

template <>
struct Visit<kBfs + kPartAlgo> {
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t) {
    if (a.sent) {  // send each discovery once per iteration
      uint32_t* word = a.sent + (w >> 5);
      const uint32_t bit = 1u << (w & 31);
      if ((*word & bit) || (atomicOr(word, bit) & bit)) return;
      if (a.sent_only) return;  // bitmap exchange: the owner reads the bit
    }
    *cand_slot<uint8_t>(a, w) = 1;
  }
};

// Fused mode sends a candidate to its owner only when it improves this rank's
// best for w this iteration (local pre-filter in HBM): the owner still gets
// every rank's minimum, with one remote reduction per improvement instead of
// one per edge.
template <typename T>
__device__ __forceinline__ bool improves_local(const ExpandArgs& a, uint64_t w, T cand) {
  if (!a.lbest) return true;
  T* lb = static_cast<T*>(a.lbest) + w;
  if (cand >= *lb) return false;
  return cand < atomicMin(lb, cand);
}

template <>
struct Visit<kSssp + kPartAlgo> {
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t wt,
                                               uint64_t val) {
    const unsigned long long cand = val + wt;
    if (a.peers) {  // remote: reduction, no read-back
      if (improves_local<unsigned long long>(a, w, cand))
        atomicMin(cand_slot<unsigned long long>(a, w), cand);
      return;
    }
    unsigned long long* x = cand_slot<unsigned long long>(a, w);
    if (cand < *x) atomicMin(x, cand);
  }
};

template <>
struct Visit<kCc + kPartAlgo> {
  static __device__ __forceinline__ void apply(const ExpandArgs& a, uint64_t w, uint64_t,
                                               uint64_t val) {
    const unsigned cand = static_cast<unsigned>(val);
    if (a.peers) {
      if (improves_local<unsigned>(a, w, cand)) atomicMin(cand_slot<unsigned>(a, w), cand);
      return;
    }
    unsigned* x = cand_slot<unsigned>(a, w);
    if (cand < *x) atomicMin(x, cand);
  }
};

template <typename ET>
struct LineElems {
  static constexpr uint64_t value = kLineBytes / sizeof(ET);
};

template <int STRAT, typename ET>
__device__ __forceinline__ uint64_t window_base(uint64_t s) {
  if (STRAT == kMergedAligned) return s & ~(LineElems<ET>::value - 1);
  if (STRAT == kPacked) return s & ~static_cast<uint64_t>(kWarp - 1);
  return s;
}

// ------------------------------------------------ merged / merged-aligned
// A batch of kUnroll windows of one warp: each lane holds the element it
// loaded from each window (ok = lane inside the list).
template <int ALGO, typename ET, typename WT, int U, bool CMP = false>
struct Batch {
  ET dst[U];
  WT wt[U];
  uint64_t sval[U];
  bool ok[U];
  // kCompressed only (warp-uniform): window u is 1 = a long-list line, 2 = a
  // shared span of the staged short lists [k0, k1), dst2 its second line
  static constexpr int C = CMP ? U : 1;
  uint8_t line[C];
  int16_t k0[C], k1[C];
  uint32_t dst2[C];
};

template <int ALGO, typename ET, typename WT, int U, bool CMP = false>
__device__ __forceinline__ void visit_batch(const ExpandArgs& a,
                                            const Batch<ALGO, ET, WT, U, CMP>& b) {
  if constexpr (ALGO == kBfs) {
    // The batch's visits in three independent phases -- all bitmap probes,
    // then the claims of the unvisited, then the winners' writes -- so the
    // U windows' L2 round trips overlap instead of chaining probe -> atomic ->
    // store window after window (a store to level[] may alias the next
    // window's bitmap word, which pins the per-window order otherwise).
    uint32_t probe[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      probe[u] = b.ok[u] ? a.visited[static_cast<uint64_t>(b.dst[u]) >> 5] : ~0u;
    uint32_t old[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t bit = 1u << (static_cast<uint32_t>(b.dst[u]) & 31);
      old[u] = ~0u;
      if (!(probe[u] & bit))
        old[u] = atomicOr(a.visited + (static_cast<uint64_t>(b.dst[u]) >> 5), bit);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t w = static_cast<uint64_t>(b.dst[u]);
      if (!(old[u] & (1u << (w & 31)))) {
        static_cast<uint32_t*>(a.state)[w] = a.iter;
        a.flags[w] = 1;
      }
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!b.ok[u]) continue;
    if constexpr (IsPair<WT>::value)
      Visit<ALGO>::apply(a, uint64_t(b.dst[u]) & 0xffffffffull, uint64_t(b.dst[u]) >> 32,
                         b.sval[u]);
    else
      Visit<ALGO>::apply(a, b.dst[u], AlgoTraits<ALGO>::weighted ? uint64_t(b.wt[u]) : 0,
                         b.sval[u]);
  }
}

// Per-lane metadata of one 32-slot chunk of the frontier.
struct Chunk {
  uint64_t s, e, val;
  uint32_t nst;
};

template <int STRAT, int ALGO, typename ET>
__device__ __forceinline__ Chunk load_chunk(const ExpandArgs& a, uint64_t c0, int lane) {
  Chunk c{0, 0, 0, 0};
  const uint64_t j = c0 + lane;
  if (j < a.n) {
    c.s = a.fs[j];
    c.e = c.s + a.fd[j];
    if (AlgoTraits<ALGO>::has_val) c.val = a.fval[j];
  }
  return c;
}

// Tier 1: a warp takes 32 consecutive frontier slots (their list start and
// degree were written by the compaction, so no dependent offsets gather),
// then walks the flattened sequence of their 32-element windows, kUnroll
// windows at a time, issuing the loads of batch k+1 before visiting batch k
// (so the HBM-side visit overlaps the next PCIe round trip) and prefetching
// the next chunk's metadata.  Lists needing more than kBigSteps windows go to
// the tier-2 queue.
template <int STRAT, int ALGO, typename ET, typename WT, int U>
__global__ void __launch_bounds__(kExpandThreads) k_expand_warp(ExpandArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * kExpandThreads + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * kExpandThreads) >> 5;
  const ET* __restrict__ E = static_cast<const ET*>(a.edges);
  const WT* __restrict__ W = static_cast<const WT*>(a.weights);

  uint64_t c0 = gw * kWarp;
  Chunk nextc = load_chunk<STRAT, ALGO, ET>(a, c0, lane);
  for (; c0 < a.n; c0 += nw * kWarp) {
    const Chunk c = nextc;
    if (c0 + nw * kWarp < a.n) nextc = load_chunk<STRAT, ALGO, ET>(a, c0 + nw * kWarp, lane);
    uint32_t nst = 0;
    const uint64_t base = window_base<STRAT, ET>(c.s);
    if (c.e > c.s) {
      const uint64_t steps = (c.e - base + kWarp - 1) / kWarp;
      if (steps > kBigSteps) {
        const unsigned long long slot =
            atomicAdd(reinterpret_cast<unsigned long long*>(a.ctr + kCtrBig), 1ull);
        a.big_s[slot] = c.s;
        a.big_e[slot] = c.e;
        if (AlgoTraits<ALGO>::has_val) a.big_val[slot] = c.val;
        a.big_prefix[slot] = steps;
      } else {
        nst = static_cast<uint32_t>(steps);
      }
    }
    // warp-inclusive scan of the per-slot window counts
    uint32_t incl = nst;
#pragma unroll
    for (int d = 1; d < kWarp; d <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    const uint32_t excl = incl - nst;
    const uint32_t total = __shfl_sync(kFull, incl, kWarp - 1);

    auto issue = [&](Batch<ALGO, ET, WT, U>& b, uint32_t q0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + u;
        b.ok[u] = false;
        b.sval[u] = 0;
        if (q < total) {  // warp-uniform
          // owner slot of window q: highest lane whose exclusive prefix <= q
          const unsigned m = __ballot_sync(kFull, excl <= q);
          const int k = 31 - __clz(m);
          const uint64_t bk = __shfl_sync(kFull, base, k);
          const uint64_t sk = __shfl_sync(kFull, c.s, k);
          const uint64_t ek = __shfl_sync(kFull, c.e, k);
          const uint32_t t = q - __shfl_sync(kFull, excl, k);
          if (AlgoTraits<ALGO>::has_val) b.sval[u] = __shfl_sync(kFull, c.val, k);
          const uint64_t idx = bk + static_cast<uint64_t>(t) * kWarp + lane;
          b.ok[u] = idx >= sk && idx < ek;
          if (b.ok[u]) {
            b.dst[u] = ld_list(E + idx);
            if constexpr (AlgoTraits<ALGO>::weighted && !IsPair<WT>::value)
              b.wt[u] = ld_list(W + idx);
          }
        }
      }
    };
    if (total == 0) continue;
    Batch<ALGO, ET, WT, U> cur, nxt;
    issue(cur, 0);
    for (uint32_t q0 = 0; q0 < total; q0 += U) {
      if (q0 + U < total) issue(nxt, q0 + U);
      visit_batch<ALGO, ET, WT, U>(a, cur);
      cur = nxt;
    }
  }
}

// Tier 2: every warp takes an equal contiguous range of the big lists'
// flattened window sequence (same windows as tier 1), software-pipelined
// the same way.
template <int STRAT, int ALGO, typename ET, typename WT, int U>
__global__ void __launch_bounds__(kExpandThreads) k_expand_big(ExpandArgs a) {
  const uint64_t nbig = a.ctr[kCtrBig];
  if (nbig == 0) return;
  const uint64_t total = a.big_prefix[nbig];
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * kExpandThreads + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * kExpandThreads) >> 5;
  uint64_t per = (total + nw - 1) / nw;
  per = (per + U - 1) / U * U;
  const uint64_t q_begin = gw * per;
  if (q_begin >= total) return;
  const uint64_t q_end = min(total, q_begin + per);
  const ET* __restrict__ E = static_cast<const ET*>(a.edges);
  const WT* __restrict__ W = static_cast<const WT*>(a.weights);

  // entry i owning q_begin: last i with prefix[i] <= q_begin
  uint64_t lo = 0, hi = nbig;  // invariant prefix[lo] <= q < prefix[hi]
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a.big_prefix[mid] <= q_begin) lo = mid; else hi = mid;
  }
  uint64_t i = lo;
  uint64_t p_i = a.big_prefix[i], p_next = a.big_prefix[i + 1];
  uint64_t s = a.big_s[i], e = a.big_e[i];
  uint64_t b = window_base<STRAT, ET>(s);
  uint64_t val = AlgoTraits<ALGO>::has_val ? a.big_val[i] : 0;

  auto issue = [&](Batch<ALGO, ET, WT, U>& bt, uint64_t q0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t q = q0 + u;
      bt.ok[u] = false;
      bt.sval[u] = val;
      if (q < q_end) {
        while (q >= p_next) {  // warp-uniform
          ++i;
          p_i = p_next;
          p_next = a.big_prefix[i + 1];
          s = a.big_s[i];
          e = a.big_e[i];
          b = window_base<STRAT, ET>(s);
          if (AlgoTraits<ALGO>::has_val) val = a.big_val[i];
        }
        bt.sval[u] = val;
        const uint64_t idx = b + (q - p_i) * kWarp + lane;
        bt.ok[u] = idx >= s && idx < e;
        if (bt.ok[u]) {
          bt.dst[u] = ld_list(E + idx);
          if constexpr (AlgoTraits<ALGO>::weighted && !IsPair<WT>::value)
            bt.wt[u] = ld_list(W + idx);
        }
      }
    }
  };
  Batch<ALGO, ET, WT, U> cur, nxt;
  issue(cur, q_begin);
  for (uint64_t q0 = q_begin; q0 < q_end; q0 += U) {
    if (q0 + U < q_end) issue(nxt, q0 + U);
    visit_batch<ALGO, ET, WT, U>(a, cur);
    cur = nxt;
  }
}

// ------------------------------------------------- CTA sweep (default)
// Scheduling measured on B200 (tools/read_probe.py): zero-copy reads reach
// the link rate only while the number of concurrently streamed address
// regions stays around one per CTA (~1.2 K); one stream per warp (~9.5 K)
// caps at ~35 GB/s -- the GPU/IOMMU translation reach.  So every CTA takes
// an equal contiguous range of the frontier's flattened window sequence
// (windows are equal-cost line requests, so static ranges balance) and its
// 8 warps take interleaved batches of U windows inside it: the CTA streams
// ~4 KB at a time through its region.  Windows (lane -> element maps) are
// exactly those of the strategy; only their schedule changes.
constexpr int kSweepThreads = 256;
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kStage = 256;  // frontier slots staged in shared memory at a time
// Resident CTAs per SM the register allocation must allow: the compressed
// decode is latency-bound, so occupancy beats a few spilled registers.
// Measured on K27 / U27 (compressed): SSSP 96 registers / 2 CTAs 1,305 ms,
// 80 / 3 CTAs 976 ms; CC 80 / 3 CTAs 1,074 ms, 64 / 4 CTAs 1,006 ms.
// The raw strategies keep the compiler's choice (the HBM control run is
// occupancy-sensitive the other way: 117 vs 94 GTEPS).
template <int STRAT, int ALGO>
struct SweepMinBlocks {
  static constexpr int value = STRAT != kCompressed ? 0 : AlgoTraits<ALGO>::weighted ? 3 : 4;
};

// Windows per frontier slot.  Packed: the slot's 32-element blocks minus its
// first block when the nearest earlier non-empty slot of the same aligned
// group of kStage slots (one shared-memory stage of the sweep) already
// touches it -- so every block is fetched once per group and the lists that
// share it are always staged together.  Compressed: a long list's windows
// are its lines; a short list's line is one window unless the nearest earlier
// non-empty slot of the group has its list in the same line.
template <int STRAT, typename ET>
__global__ void k_window_counts(ExpandArgs a) {
  const uint64_t n = a.n_dev ? *a.n_dev : a.n;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = a.fs[j], d = a.fd[j];
    if (!d) {
      a.wcnt[j] = 0;
      continue;
    }
    const uint64_t group0 = j - j % kStage;
    if (STRAT == kCompressed) {
      const uint32_t v = a.front[j];
      const uint64_t c = a.cpos[v];
      if (a.pull_pass == 2) {  // the rest of the long in-lists still without a parent
        a.wcnt[j] = (c & kCmpLong) && !((a.visited[v >> 5] >> (v & 31)) & 1u)
                        ? static_cast<uint32_t>(cmp_lines(c) - 1)
                        : 0u;
        continue;
      }
      if (c & kCmpLong) {
        a.wcnt[j] = a.pull_pass == 1 ? 1u : static_cast<uint32_t>(cmp_lines(c));
        continue;
      }
      uint32_t w = 1;
      for (uint64_t i = j; i > group0; --i) {
        if (!a.fd[i - 1]) continue;
        const uint64_t ci = a.cpos[a.front[i - 1]];
        w = (ci & kCmpLong) || cmp_pos(ci) / kShortSpanBits != cmp_pos(c) / kShortSpanBits;
        break;
      }
      a.wcnt[j] = w;
      continue;
    }
    uint64_t w = (s + d - window_base<STRAT, ET>(s) + kWarp - 1) / kWarp;
    if (a.pull_pass == 1 && w > 1) w = 1;  // first window only (union-find sampling pass)
    if (STRAT == kPacked) {
      for (uint64_t i = j; i > group0; --i) {
        const uint32_t di = a.fd[i - 1];
        if (!di) continue;
        w -= ((a.fs[i - 1] + di - 1) / kWarp) == (s / kWarp);
        break;
      }
    }
    a.wcnt[j] = static_cast<uint32_t>(w);
  }
}

// `nbits` (<= 32) of the staged line L at bit position `bit` (< 1024).
__device__ __forceinline__ uint32_t line_bits(const uint32_t* L, uint32_t bit, uint32_t nbits) {
  const uint64_t pair = (static_cast<uint64_t>(L[(bit >> 5) + 1]) << 32) | L[bit >> 5];
  return static_cast<uint32_t>((pair >> (bit & 31)) & (nbits >= 32 ? 0xffffffffull
                                                                    : ((1ull << nbits) - 1)));
}

// Decode one long-list line (this lane's word in x) and visit its elements:
// lane l takes elements [l m, l m + m), m = ceil(count / 32); values are the
// base plus a warp prefix sum of the deltas (u32 exact: ids < 2^32).
template <int ALGO>
__device__ __forceinline__ uint32_t visit_line(const ExpandArgs& a, uint32_t x, uint64_t sval,
                                               uint32_t* L, int lane) {
  L[lane] = x;
  if (lane < 2) L[kLineWords + lane] = 0;
  __syncwarp();
  const uint32_t hdr = L[1];
  const uint32_t w = hdr & 63, cnt = ((hdr >> 6) & 255) + 1;
  const uint32_t m = (cnt + 31) >> 5;
  const uint32_t e0 = lane * m, e1 = min(cnt, e0 + m);
  uint32_t run = 0;
  for (uint32_t e = e0; e < e1; ++e)
    run += e == 0 ? L[0] : line_bits(L, kCmpHdrBits + (e - 1) * w, w);
  uint32_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t val = incl - run;
  const uint32_t wb = kCmpHdrBits + (cnt - 1) * w;
  uint32_t e1v = e1;  // union-find sampling pass: one element per lane
  if constexpr (ALGO == kCcUf)
    if (a.pull_pass == 1 && a.uf_sample < kCmpShortMaxDeg) e1v = min(e1, e0 + 1);
  for (uint32_t e = e0; e < e1v; ++e) {
    val += e == 0 ? L[0] : line_bits(L, kCmpHdrBits + (e - 1) * w, w);
    uint64_t wt = 0;
    if constexpr (AlgoTraits<ALGO>::weighted) wt = a.cmp_wmin + line_bits(L, wb + e * a.cmp_ww, a.cmp_ww);
    Visit<ALGO>::apply(a, val, wt, sval);
  }
  __syncwarp();
  return e1v > e0 ? e1v - e0 : 0u;  // elements this lane visited
}

// Decode the short lists of staged slots [k0, k1) from their shared line
// (this lane's word in x): a lane per list, elements in order.  Every slot
// in [k0, k1) is in the frontier; empty lists take no bits, so there can be
// more than 32 of them.
template <int ALGO>
__device__ __forceinline__ uint32_t visit_short(const ExpandArgs& a, uint32_t x, uint32_t x2, int k0,
                                            int k1, const uint64_t* sh_c, const uint64_t* sh_s,
                                            const uint64_t* sh_e, const uint64_t* sh_v,
                                            uint32_t* L, int lane) {
  L[lane] = x;
  L[kLineWords + lane] = x2;
  if (lane < 2) L[kShortSpanWords + lane] = 0;
  __syncwarp();
  uint32_t seen = 0;  // elements this lane visited
  // more than 32 staged slots can share a line when empty lists sit between
  for (int i = k0 + lane; i < k1; i += 32) {
    const uint32_t d = static_cast<uint32_t>(sh_e[i] - sh_s[i]);
    const uint32_t p = static_cast<uint32_t>(cmp_pos(sh_c[i]) % kShortSpanBits);
    const uint64_t sval = AlgoTraits<ALGO>::has_val ? sh_v[i] : 0;
    const uint32_t hdr = kCmpShortWidthBits + a.cmp_b0;
    const uint32_t w = d ? line_bits(L, p, kCmpShortWidthBits) : 0;
    uint32_t val = d ? line_bits(L, p + kCmpShortWidthBits, a.cmp_b0) : 0;
    const uint32_t wb = p + hdr + (d - 1) * w;
    uint32_t dv = d;  // union-find sampling pass: the first uf_sample elements
    if constexpr (ALGO == kCcUf)
      if (a.pull_pass == 1) dv = min(d, a.uf_sample);
    for (uint32_t e = 0; e < dv; ++e) {
      // bottom-up: stop at the first parent (or a candidate found elsewhere)
      if (AlgoTraits<ALGO>::pull && is_visited(a, sval)) break;
      if (e) val += line_bits(L, p + hdr + (e - 1) * w, w);
      uint64_t wt = 0;
      if constexpr (AlgoTraits<ALGO>::weighted) wt = a.cmp_wmin + line_bits(L, wb + e * a.cmp_ww, a.cmp_ww);
      Visit<ALGO>::apply(a, val, wt, sval);
      ++seen;
    }
  }
  __syncwarp();
  return seen;
}

template <int STRAT, int ALGO, typename ET, typename WT, int U, int LD = DefaultLd<STRAT>::value>
__global__ void __launch_bounds__(kSweepThreads, SweepMinBlocks<STRAT, ALGO>::value)
    k_expand_sweep(ExpandArgs a) {
  if (a.n_dev) {  // device-driven level loop: size and level live in device memory
    a.n = *a.n_dev;
    a.iter = static_cast<uint32_t>(*a.iter_dev) + 1;
  }
  constexpr bool kCmp = STRAT == kCompressed;
  __shared__ uint64_t sh_s[kStage], sh_e[kStage], sh_v[kStage];
  __shared__ uint64_t sh_w[kStage + 1];
  __shared__ uint64_t sh_c[kCmp ? kStage : 1];  // list position (| kCmpLong)
  __shared__ uint64_t sh_n[kCmp ? kStage : 1];  // next vertex's position (list end bound)
  __shared__ uint32_t sh_line[kCmp ? kSweepWarps : 1][kShortSpanWords + 2];  // decode buffer
  __shared__ uint64_t sh_j;
  const uint64_t n = a.n;
  const uint64_t T = a.wpre[n];
  const uint64_t G = gridDim.x, b = blockIdx.x;
  const uint64_t Wb = T / G * b + min(b, T % G);
  const uint64_t We = Wb + T / G + (b < T % G ? 1 : 0);
  if (Wb >= We) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const ET* __restrict__ E = static_cast<const ET*>(a.edges);
  const WT* __restrict__ Wt = static_cast<const WT*>(a.weights);

  // slot owning window Wb: the last j with wpre[j] <= Wb (32-ary search)
  if (warp == 0) {
    uint64_t lo = 0, hi = n;  // wpre[lo] <= Wb < wpre[hi] (wpre[n] = T > Wb)
    while (hi - lo > 1) {
      const uint64_t step = (hi - lo + 31) / 32;
      const uint64_t probe = lo + step * (lane + 1);
      const bool le = probe < hi && a.wpre[probe] <= Wb;
      const unsigned m = __ballot_sync(kFull, le);
      const int k = m ? 31 - __clz(m) : -1;  // predicates are monotone in the lane
      const uint64_t nlo = k >= 0 ? lo + step * (k + 1) : lo;
      hi = min(hi, nlo + step);
      lo = nlo;
    }
    if (lane == 0) sh_j = lo - lo % kStage;  // stages are aligned groups of kStage slots
  }
  __syncthreads();
  uint64_t j = sh_j;
  uint64_t W = Wb;
  uint64_t words = 0;  // compressed: 4-byte words this warp requested (warp-uniform)
  uint64_t seen = 0;   // union-find: list elements this thread visited
  while (W < We) {
    // stage slots [j, j + kStage)
    for (int i = threadIdx.x; i <= kStage; i += kSweepThreads) {
      const uint64_t jj = j + i;
      sh_w[i] = jj <= n ? a.wpre[jj] : T;
      if (i < kStage && jj < n) {
        const uint64_t s0 = a.fs[jj];
        sh_s[i] = s0;
        sh_e[i] = s0 + a.fd[jj];
        if (AlgoTraits<ALGO>::has_val)
          sh_v[i] = AlgoTraits<ALGO>::pull ? a.front[jj] : a.fval[jj];
        if constexpr (kCmp) {
          const uint32_t v = a.front[jj];
          sh_c[i] = a.cpos[v];
          sh_n[i] = cmp_pos(a.cpos[v + 1]);
        }
      }
    }
    __syncthreads();
    const uint64_t Wend = min(We, sh_w[kStage]);
    const int stage_n = static_cast<int>(n - j < kStage ? n - j : kStage);  // staged slots

    int k = 0;  // per-warp slot cursor, monotone within this stage
    auto issue = [&](Batch<ALGO, ET, WT, U, kCmp>& bt, uint64_t q0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t q = q0 + u;
        bt.ok[u] = false;
        bt.sval[u] = 0;
        if constexpr (kCmp) bt.line[u] = 0;
        if (q < Wend) {  // warp-uniform
          if (u == 0) {  // binary search for the batch head, then walk
            int lo = 0, hi = kStage;  // sh_w[lo] <= q < sh_w[hi]
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (sh_w[mid] <= q) lo = mid; else hi = mid;
            }
            k = lo;
          } else {
            while (sh_w[k + 1] <= q) ++k;
          }
          const uint64_t s0 = sh_s[k], e0 = sh_e[k];
          uint64_t idx;
          if constexpr (kCmp) {
            const uint64_t c = sh_c[k];
            if (c & kCmpLong) {  // line t of a long list: a word per lane
              // bottom-up: a candidate found earlier in this level needs no more lines
              if (AlgoTraits<ALGO>::pull && is_visited(a, sh_v[k])) continue;
              bt.line[u] = 1;
              if (AlgoTraits<ALGO>::has_val) bt.sval[u] = sh_v[k];
              const uint64_t line = cmp_pos(c) / kLineBits + (q - sh_w[k]) + (a.pull_pass == 2);
              bt.dst[u] = ld_list(a.cmp + line * kLineWords + lane);
              words += kLineWords;
            } else {  // a shared span: the words of its staged frontier lists
              bt.line[u] = 2;
              const uint64_t L = cmp_pos(c) / kShortSpanBits;
              int m = k + 1;
              while (m < stage_n && !(sh_c[m] & kCmpLong) && cmp_pos(sh_c[m]) / kShortSpanBits == L)
                ++m;
              if constexpr (AlgoTraits<ALGO>::pull) {  // all candidates of the line found?
                bool open = false;
                for (int i = k + lane; i < m && !open; i += 32) open = !is_visited(a, sh_v[i]);
                if (!__any_sync(kFull, open)) continue;
              }
              const uint32_t w0 = static_cast<uint32_t>(cmp_pos(c) % kShortSpanBits) / 32;
              const uint64_t endb = min(sh_n[m - 1], (L + 1) * kShortSpanBits);
              const uint32_t w1 = static_cast<uint32_t>(endb - 1 - L * kShortSpanBits) / 32;
              bt.k0[u] = static_cast<int16_t>(k);
              bt.k1[u] = static_cast<int16_t>(m);
              const uint32_t* sp = a.cmp + L * kShortSpanWords;
              bt.dst[u] = lane >= w0 && lane <= w1 ? ld_list(sp + lane) : 0u;
              bt.dst2[u] = lane + 32 >= w0 && lane + 32 <= w1 ? ld_list(sp + 32 + lane) : 0u;
              words += w1 - w0 + 1;
            }
            continue;
          }
          if (STRAT == kPacked) {
            // block t of slot k's new blocks; the lane's element may belong to
            // any staged list that shares the block: search its owner
            const uint64_t fb = s0 / kWarp;
            const bool shared = (sh_w[k + 1] - sh_w[k]) < ((e0 - 1) / kWarp - fb + 1);
            idx = (fb + shared + (q - sh_w[k])) * kWarp + lane;
            int lo = 0, hi = stage_n;  // last m with sh_s[m] <= idx
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (sh_s[mid] <= idx) lo = mid; else hi = mid;
            }
            bt.ok[u] = idx >= sh_s[lo] && idx < sh_e[lo];
            if (AlgoTraits<ALGO>::has_val) bt.sval[u] = sh_v[lo];
          } else {
            if (AlgoTraits<ALGO>::has_val) bt.sval[u] = sh_v[k];
            idx = window_base<STRAT, ET>(s0) + (q - sh_w[k]) * kWarp + lane;
            bt.ok[u] = idx >= s0 && idx < e0;
          }
          if constexpr (ALGO == kCcUf) seen += bt.ok[u];
          bool promote = false;  // ld=4: a window of 3 sectors loads its whole line
          if constexpr (LD == 4 && STRAT == kMergedAligned && sizeof(ET) == 4) {
            // only over a 128-byte-aligned list array (every allocation here;
            // a caller-registered buffer may not be): then the window is one
            // memory line holding list elements, inside mapped pages
            const uint64_t base = idx - lane;
            const uint64_t lo = max(s0, base), hi = min(e0, base + kWarp);
            promote = (reinterpret_cast<uintptr_t>(E) & 127) == 0 && hi > lo &&
                      ((hi - 1 - base) >> 3) - ((lo - base) >> 3) == 2;
          }
          if (bt.ok[u] || promote) {
            bt.dst[u] = ld_list_f<LD == 4 ? 1 : LD>(E + idx);
            if constexpr (AlgoTraits<ALGO>::weighted && !IsPair<WT>::value)
              bt.wt[u] = ld_list_f<LD>(Wt + idx);
          }
        }
      }
    };
    // warps interleave batches of U windows: warp w takes [W + (i*8 + w)*U, +U)
    uint64_t q0 = W + static_cast<uint64_t>(warp) * U;
    if (q0 < Wend) {
      Batch<ALGO, ET, WT, U, kCmp> cur, nxt;
      issue(cur, q0);
      for (; q0 < Wend; q0 += kSweepWarps * U) {
        const uint64_t qn = q0 + kSweepWarps * U;
        if (qn < Wend) issue(nxt, qn);
        if constexpr (kCmp) {
#pragma unroll
          for (int u = 0; u < U; ++u) {  // line kinds are warp-uniform
            if (cur.line[u] == 1)
              seen += visit_line<ALGO>(a, static_cast<uint32_t>(cur.dst[u]), cur.sval[u],
                                       sh_line[warp], lane);
            else if (cur.line[u] == 2)
              seen += visit_short<ALGO>(a, static_cast<uint32_t>(cur.dst[u]), cur.dst2[u],
                                        cur.k0[u], cur.k1[u], sh_c, sh_s, sh_e, sh_v,
                                        sh_line[warp], lane);
          }
        } else {
          visit_batch<ALGO, ET, WT, U, kCmp>(a, cur);
        }
        cur = nxt;
      }
    }
    __syncthreads();
    W = Wend;
    j += kStage;
  }
  if constexpr (ALGO == kCcUf) {  // elements read (the sampling pass reads part of each list)
    __shared__ unsigned long long sh_seen;
    if (threadIdx.x == 0) sh_seen = 0;
    __syncthreads();
    for (int o = 16; o; o >>= 1) seen += __shfl_xor_sync(kFull, seen, o);
    if (lane == 0 && seen) atomicAdd(&sh_seen, static_cast<unsigned long long>(seen));
    __syncthreads();
    if (threadIdx.x == 0 && sh_seen)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.ctr + kCtrVisited), sh_seen);
  }
  if constexpr (kCmp) {  // link bytes requested: one atomic per CTA
    __shared__ unsigned long long sh_words;
    if (threadIdx.x == 0) sh_words = 0;
    __syncthreads();
    if (lane == 0 && words) atomicAdd(&sh_words, static_cast<unsigned long long>(words));
    __syncthreads();
    if (threadIdx.x == 0 && sh_words)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.ctr + kCtrLoaded), sh_words * 4ull);
  }
}

// In-place exclusive scan of the big-list step counts (single CTA; the
// queue holds only lists longer than kBigSteps windows).
__global__ void __launch_bounds__(1024) k_big_scan(uint64_t* prefix, const uint64_t* ctr) {
  const uint64_t n = ctr[kCtrBig];
  if (n == 0) return;
  __shared__ uint64_t warp_sums[32];
  const int tid = threadIdx.x;
  const uint64_t chunk = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min(n, tid * chunk), hi = min(n, lo + chunk);
  uint64_t sum = 0;
  for (uint64_t k = lo; k < hi; ++k) sum += prefix[k];
  // block exclusive scan of `sum`
  uint64_t incl = sum;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint64_t ws = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
    uint64_t wi = ws;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t t = __shfl_up_sync(kFull, wi, d);
      if (lane >= d) wi += t;
    }
    warp_sums[lane] = wi - ws;
  }
  __syncthreads();
  uint64_t run = warp_sums[wid] + incl - sum;
  for (uint64_t k = lo; k < hi; ++k) {
    const uint64_t c = prefix[k];
    prefix[k] = run;
    run += c;
  }
  if (hi == n && lo < hi) prefix[n] = run;
}

// ------------------------------------------------------------------ naive
// access.py:195-216: thread per frontier vertex, lockstep one element per
// step.  Slot j is lane j%32 of warp j/32 in the first grid-stride round.
template <int ALGO, typename ET, typename WT>
__global__ void __launch_bounds__(kExpandThreads) k_expand_naive(ExpandArgs a) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kExpandThreads + threadIdx.x;
  const uint64_t nt = static_cast<uint64_t>(gridDim.x) * kExpandThreads;
  const ET* __restrict__ E = static_cast<const ET*>(a.edges);
  const WT* __restrict__ W = static_cast<const WT*>(a.weights);
  for (uint64_t j = tid; j < a.n; j += nt) {
    const uint64_t s = a.fs[j], e = s + a.fd[j];
    const uint64_t val = AlgoTraits<ALGO>::has_val ? a.fval[j] : 0;
    for (uint64_t k = s; k < e; ++k) {
      const ET w = ld_list(E + k);
      if constexpr (IsPair<WT>::value) {
        Visit<ALGO>::apply(a, uint64_t(w) & 0xffffffffull, uint64_t(w) >> 32, val);
      } else {
        const uint64_t wt = AlgoTraits<ALGO>::weighted ? uint64_t(ld_list(W + k)) : 0;
        Visit<ALGO>::apply(a, w, wt, val);
      }
    }
  }
}

// ------------------------------------------------------------ traffic model
// Device restatement of the reference's request model (coalesce.py:88-207):
// every warp memory instruction is split into runs of consecutive touched
// 32-byte sectors inside one 128-byte line; each run is one request of
// 32/64/96/128 bytes.  No cache is modelled.  It reads only the
// frontier and the offsets (HBM), never the lists themselves.

// Requests of one contiguous element window [lo, hi) of width eb.
__device__ __forceinline__ void model_window(uint64_t lo, uint64_t hi, uint32_t eb,
                                             uint32_t* cnt) {
  const uint64_t first = lo * eb / 32, last = (hi * eb - 1) / 32;
  for (uint64_t line = first >> 2; line <= (last >> 2); ++line) {
    const uint64_t a = max(first, line << 2), b = min(last, (line << 2) + 3);
    cnt[b - a] += 1;
  }
}

__device__ __forceinline__ void flush_counts(uint32_t* cnt, uint64_t* ctr, int slot0) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    unsigned long long c = cnt[i];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(kFull, c, d);
    if ((threadIdx.x & 31) == 0 && c)
      atomicAdd(reinterpret_cast<unsigned long long*>(ctr + slot0 + i), c);
  }
}

// merged / merged-aligned: windows of access.py:171-192, one per warp step.
template <int STRAT>
__global__ void __launch_bounds__(256) k_model_merged(const uint32_t* front, uint64_t n,
                                                      const uint64_t* off, uint32_t eb,
                                                      uint32_t wb, int weights, uint64_t* ctr) {
  uint32_t ce[4] = {0, 0, 0, 0}, cw[4] = {0, 0, 0, 0};
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t rounds = (n + nt - 1) / nt;  // keep the warp converged for the shuffles
  for (uint64_t r = 0; r < rounds; ++r) {
    const uint64_t j = tid0 + r * nt;
    if (j >= n) continue;
    const uint32_t v = front[j];
    const uint64_t s = off[v], e = off[v + 1];
    if (e <= s) continue;
    const uint64_t a = STRAT == kMergedAligned ? (s & ~(uint64_t)(kLineBytes / eb - 1)) : s;
    for (uint64_t base = a; base < e; base += kWarp) {
      const uint64_t lo = max(base, s), hi = min(base + kWarp, e);
      model_window(lo, hi, eb, ce);
      if (weights) model_window(lo, hi, wb, cw);
    }
  }
  flush_counts(ce, ctr, kCtrHist);
  if (weights) flush_counts(cw, ctr, kCtrHist + 4);
}

// Runs of one warp step: each lane holds one sector id (or ~0 if masked).
__device__ __forceinline__ void model_lanes(uint64_t sec, uint32_t* cnt) {
  const int lane = threadIdx.x & 31;
  // bitonic sort of the 32 sector ids across the warp (ascending)
  for (int k = 2; k <= 32; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(kFull, sec, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      const uint64_t lo = sec < o ? sec : o, hi = sec < o ? o : sec;
      sec = (lower == up) ? lo : hi;
    }
  }
  const uint64_t prev = __shfl_up_sync(kFull, sec, 1);
  const bool valid = sec != ~0ull;
  const bool uniq = valid && (lane == 0 || prev != sec);
  const unsigned umask = __ballot_sync(kFull, uniq);
  // previous unique sector (for run breaks): nearest unique lane below
  const unsigned below = umask & ((1u << lane) - 1);
  const int pl = below ? 31 - __clz(below) : -1;
  const uint64_t psec = __shfl_sync(kFull, sec, pl < 0 ? 0 : pl);
  const bool start = uniq && (pl < 0 || psec + 1 != sec || (psec >> 2) != (sec >> 2));
  const unsigned smask = __ballot_sync(kFull, start);
  if (start) {
    const unsigned above = smask & ~((2u << lane) - 1);  // starts after this lane
    const int next = above ? __ffs(above) - 1 : 32;
    const unsigned span = (next == 32 ? 0xffffffffu : ((1u << next) - 1)) & ~((1u << lane) - 1);
    cnt[__popc(umask & span) - 1] += 1;
  }
}

// naive: access.py:195-216 -- lane i of warp w is frontier[32w+i], lanes
// step through their lists in lockstep; edge and weight accesses are
// separate instructions (coalesce.py:182-191).
__global__ void __launch_bounds__(256) k_model_naive(const uint32_t* front, uint64_t n,
                                                     const uint64_t* off, uint32_t eb,
                                                     uint32_t wb, int weights, uint64_t* ctr) {
  uint32_t ce[4] = {0, 0, 0, 0}, cw[4] = {0, 0, 0, 0};
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = gw; w * kWarp < n; w += nw) {
    const uint64_t j = w * kWarp + lane;
    uint64_t s = 0, d = 0;
    if (j < n) {
      const uint32_t v = front[j];
      s = off[v];
      d = off[v + 1] - s;
    }
    uint64_t steps = d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x = __shfl_xor_sync(kFull, steps, o);
      steps = x > steps ? x : steps;
    }
    for (uint64_t k = 0; k < steps; ++k) {
      const bool act = k < d;
      const unsigned am = __ballot_sync(kFull, act);
      if (__popc(am) == 1) {  // one lane left: one 1-sector request per step
        const int only = __ffs(am) - 1;
        const uint64_t rem = __shfl_sync(kFull, d, only) - k;
        if (lane == 0) {
          ce[0] += static_cast<uint32_t>(rem);
          if (weights) cw[0] += static_cast<uint32_t>(rem);
        }
        break;
      }
      model_lanes(act ? (s + k) * eb / 32 : ~0ull, ce);
      if (weights) model_lanes(act ? (s + k) * wb / 32 : ~0ull, cw);
    }
  }
  flush_counts(ce, ctr, kCtrHist);
  if (weights) flush_counts(cw, ctr, kCtrHist + 4);
}

// ------------------------------------------------------------ compaction
// Next frontier = marked vertices in ascending order (the reference's
// frontiers are sorted: np.unique / np.flatnonzero, traversal.py:116,150,178).
// Three passes over 4096-vertex tiles: count, scan, write (+ snapshot value,
// + degree sum for traversed_edges, + clearing of the marks).

__device__ __forceinline__ uint32_t block_reduce_u32(uint32_t x, uint32_t* sh) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_down_sync(kFull, x, d);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = x;
  __syncthreads();
  uint32_t r = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[w];
  return r;  // valid in thread 0
}

// Near-far SSSP: of 16 marked vertices from v0, keep the marks of those with
// dist < thresh (the near set); the others stay in the far pile.
__device__ __forceinline__ uint4 select_near(uint4 f, uint64_t v0, const CompactArgs& c) {
  if (!c.thresh || !(f.x | f.y | f.z | f.w)) return f;
  const uint64_t* dist = static_cast<const uint64_t*>(c.state);
  uint32_t w[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const uint32_t m = 0xffu << ((b & 3) * 8);
    if ((w[b >> 2] & m) && dist[v0 + b] >= c.thresh) w[b >> 2] &= ~m;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kTileThreads) k_tile_count(CompactArgs c) {
  __shared__ uint32_t sh[kTileThreads / 32];
  for (uint64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
    const uint4 f = select_near(
        reinterpret_cast<const uint4*>(c.flags)[t * kTileThreads + threadIdx.x],
        t * kTileVerts + static_cast<uint64_t>(threadIdx.x) * 16, c);
    uint32_t cnt = __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);
    cnt = block_reduce_u32(cnt, sh);
    if (threadIdx.x == 0) c.tiles[t] = cnt;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_tile_scan(CompactArgs c) {
  __shared__ uint64_t warp_sums[32];
  const int tid = threadIdx.x;
  const uint64_t n = c.ntiles;
  // chunks of whole uint4 groups: the per-thread sums read 16 bytes at a time
  const uint64_t chunk = (n + blockDim.x * 4 - 1) / (blockDim.x * 4) * 4;
  const uint64_t lo = min(n, tid * chunk), hi = min(n, lo + chunk);
  uint64_t sum = 0;
  if (hi - lo == chunk) {
    const uint4* q = reinterpret_cast<const uint4*>(c.tiles + lo);
#pragma unroll 4
    for (uint64_t k = 0; k < chunk / 4; ++k) {
      const uint4 x = q[k];
      sum += static_cast<uint64_t>(x.x) + x.y + x.z + x.w;
    }
  } else {
    for (uint64_t k = lo; k < hi; ++k) sum += c.tiles[k];
  }
  uint64_t incl = sum;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint64_t ws = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
    uint64_t wi = ws;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t t = __shfl_up_sync(kFull, wi, d);
      if (lane >= d) wi += t;
    }
    warp_sums[lane] = wi - ws;
    if (lane == 31) {
      c.ctr[kCtrNext] = wi;  // grand total
      c.ctr[kCtrTrav] = 0;
      c.ctr[kCtrTravIn] = 0;
      c.ctr[kCtrBig] = 0;
    }
  }
  __syncthreads();
  uint64_t run = warp_sums[wid] + incl - sum;
  if (hi - lo == chunk) {  // frontier positions fit u32 (V < 2^32)
    uint4* q = reinterpret_cast<uint4*>(c.tiles + lo);
#pragma unroll 4
    for (uint64_t k = 0; k < chunk / 4; ++k) {
      const uint4 x = q[k];
      uint4 y;
      y.x = static_cast<uint32_t>(run);
      y.y = static_cast<uint32_t>(run += x.x);
      y.z = static_cast<uint32_t>(run += x.y);
      y.w = static_cast<uint32_t>(run += x.z);
      run += x.w;
      q[k] = y;
    }
  } else {
    for (uint64_t k = lo; k < hi; ++k) {
      const uint32_t cnt = c.tiles[k];
      c.tiles[k] = static_cast<uint32_t>(run);
      run += cnt;
    }
  }
}

// One tile (kTileVerts vertices) per iteration: the marked vertices' tile
// offsets are staged in shared memory in vertex order (a block prefix over
// the threads' 16-flag groups), then the block writes the tile's frontier
// entries with consecutive threads on consecutive positions -- coalesced
// stores, and coalesced offset gathers for the sorted ids -- instead of each
// thread scattering its own 16 vertices' entries.
template <int ALGO>
__global__ void __launch_bounds__(kTileThreads) k_tile_write(CompactArgs c) {
  __shared__ uint16_t sh_v[kTileVerts];  // tile offsets of the marked vertices
  __shared__ uint32_t warp_tot[kTileThreads / 32];
  __shared__ unsigned long long deg_sh[kTileThreads / 32], indeg_sh[kTileThreads / 32];
  static_assert(kTileVerts <= 65536, "tile offsets are u16");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t t = blockIdx.x; t < c.ntiles; t += gridDim.x) {
    uint4* fp = reinterpret_cast<uint4*>(c.flags) + t * kTileThreads + threadIdx.x;
    const uint4 f_all = *fp;
    const uint64_t tile0 = t * kTileVerts;
    const uint4 f = select_near(f_all, tile0 + static_cast<uint64_t>(threadIdx.x) * 16, c);
    const uint32_t words[4] = {f.x, f.y, f.z, f.w};
    const uint32_t cnt = __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += x;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kTileThreads / 32; ++w) {
      before += w < wid ? warp_tot[w] : 0u;
      total += warp_tot[w];
    }
    if (cnt) {
      uint32_t lpos = before + incl - cnt;
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if ((words[b >> 2] >> ((b & 3) * 8)) & 0xffu)
          sh_v[lpos++] = static_cast<uint16_t>(threadIdx.x * 16 + b);
      // selected marks are consumed; far-pile marks (near-far SSSP) stay
      *fp = make_uint4(f_all.x ^ f.x, f_all.y ^ f.y, f_all.z ^ f.z, f_all.w ^ f.w);
    }
    __syncthreads();
    const uint64_t base = c.tiles[t];
    unsigned long long deg = 0, indeg = 0;
    for (uint32_t i = threadIdx.x; i < total; i += kTileThreads) {
      const uint64_t v = tile0 + sh_v[i], pos = base + i;
      const uint64_t s0 = c.off[v], d0 = c.off[v + 1] - s0;
      c.front_out[pos] = static_cast<uint32_t>(v);
      c.fs_out[pos] = s0;
      c.fd_out[pos] = static_cast<uint32_t>(d0);
      if (ALGO == kSssp) c.fval_out[pos] = static_cast<const uint64_t*>(c.state)[v];
      if (ALGO == kCc) c.fval_out[pos] = static_cast<const uint32_t*>(c.state)[v];
      deg += d0;
      if (c.in_off) indeg += c.in_off[v + 1] - c.in_off[v];
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      deg += __shfl_down_sync(kFull, deg, d);
      indeg += __shfl_down_sync(kFull, indeg, d);
    }
    if (lane == 0) {
      deg_sh[wid] = deg;
      indeg_sh[wid] = indeg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long tot = 0, tin = 0;
      for (int w = 0; w < kTileThreads / 32; ++w) {
        tot += deg_sh[w];
        tin += indeg_sh[w];
      }
      if (tot) atomicAdd(reinterpret_cast<unsigned long long*>(c.ctr + kCtrTrav), tot);
      if (tin) atomicAdd(reinterpret_cast<unsigned long long*>(c.ctr + kCtrTravIn), tin);
    }
    __syncthreads();
  }
}

// ------------------------------------------------- near-far / union-find
__global__ void __launch_bounds__(256) k_far_min(const uint8_t* flags, const uint64_t* dist,
                                                 uint64_t nv, uint64_t* ctr) {
  unsigned long long mn = ~0ull, cnt = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (flags[v]) {
      ++cnt;
      mn = min(mn, static_cast<unsigned long long>(dist[v]));
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = min(mn, __shfl_down_sync(kFull, mn, d));
    cnt += __shfl_down_sync(kFull, cnt, d);
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicMin(reinterpret_cast<unsigned long long*>(ctr + kCtrFarMin), mn);
    atomicAdd(reinterpret_cast<unsigned long long*>(ctr + kCtrFar), cnt);
  }
}

__global__ void k_far_reset(uint64_t* ctr) {
  ctr[kCtrFarMin] = ~0ull;
  ctr[kCtrFar] = 0;
}

__global__ void k_uf_flatten(uint32_t* parent, uint64_t nv) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = uf_find(parent, static_cast<uint32_t>(v));
    if (parent[v] != r) parent[v] = r;
  }
}

__global__ void k_uf_sample(const uint32_t* parent, uint64_t nv, uint32_t* out, uint32_t sample) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < sample; i += gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9e3779b97f4a7c15ull;
    z ^= z >> 31;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 29;
    out[i] = parent[z % nv];  // flattened: the root
  }
}

// Pass-2 marks: vertices outside the giant component whose list has
// elements beyond the window(s) pass 1 read (the first window; for the
// compressed stream the first line of a long list, short lists whole).
__global__ void k_uf_marks(const uint32_t* parent, const uint64_t* off, const uint64_t* cpos,
                           uint64_t nv, uint32_t giant, int strategy, int eb,
                           uint32_t uf_sample, uint8_t* flags) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = off[v], e = off[v + 1];
    bool rest;
    if (strategy == kCompressed) {
      // the sampling pass read uf_sample elements of a short list, one per
      // lane of a long list's first line (uf_sample >= kCmpShortMaxDeg: short
      // lists and the first line whole)
      const uint64_t c = cpos[v];
      rest = uf_sample < kCmpShortMaxDeg ? (c & kCmpLong) || e - s > uf_sample
                                         : (c & kCmpLong) && cmp_lines(c) > 1;
    } else if (strategy == kNaive) {
      rest = false;  // the naive sweep reads whole lists in pass 1
    } else {
      const uint64_t line = kLineBytes / static_cast<uint64_t>(eb);
      const uint64_t base = strategy == kMerged ? s : strategy == kPacked ? (s & ~31ull)
                                                                         : (s & ~(line - 1));
      rest = e > base + kWarp;
    }
    flags[v] = rest && parent[v] != giant ? 1 : 0;
  }
}

__global__ void k_fval_ids(const uint32_t* front, uint64_t* fval, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    fval[j] = front[j];
}

// ------------------------------------------------------- device level loop
// One body of the CUDA-graph while loop ends here: log the next frontier,
// make it current, and keep looping while it is non-empty (and the log has
// room).  Single thread.
__global__ void k_level_end(uint64_t* ctr, uint64_t* log_trav, uint64_t* log_front, uint64_t cap,
                            cudaGraphConditionalHandle loop) {
  const uint64_t it = ctr[kCtrIter] + 1;  // completed iterations
  const uint64_t n = ctr[kCtrNext], t = ctr[kCtrTrav];
  ctr[kCtrIter] = it;
  ctr[kCtrCur] = n;
  const bool more = n > 0 && it < cap;
  if (more) {
    log_trav[it] = t;
    log_front[it] = n;
  }
  cudaGraphSetConditional(loop, more ? 1u : 0u);
}

// %globaltimer stamp of the current iteration (per-level expansion time).
__global__ void k_stamp(const uint64_t* ctr, uint64_t* log_t) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  log_t[ctr[kCtrIter]] = t;
}

// ---------------------------------------------------------------- helpers
__global__ void k_init_cc(uint32_t* label, uint64_t nv, uint32_t* front, uint64_t* fval,
                          const uint64_t* off, uint64_t* fs, uint32_t* fd, uint64_t base) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    label[v] = static_cast<uint32_t>(base + v);
    front[v] = static_cast<uint32_t>(v);
    fval[v] = base + v;
    const uint64_t s0 = off[v];
    fs[v] = s0;
    fd[v] = static_cast<uint32_t>(off[v + 1] - s0);
  }
}

// frontier = every vertex with its list bounds (PageRank); rank = 1/V
__global__ void k_init_all(uint64_t nv, const uint64_t* off, uint32_t* front, uint64_t* fs,
                           uint32_t* fd, double* rank) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    front[v] = static_cast<uint32_t>(v);
    const uint64_t s0 = off[v];
    fs[v] = s0;
    fd[v] = static_cast<uint32_t>(off[v + 1] - s0);
    rank[v] = 1.0 / static_cast<double>(nv);
  }
}

// frontier = [src] with its list bounds (BFS / SSSP)
__global__ void k_init_source(uint64_t src, const uint64_t* off, uint32_t* front, uint64_t* fval,
                              uint64_t* fs, uint32_t* fd) {
  front[0] = static_cast<uint32_t>(src);
  fval[0] = 0;
  fs[0] = off[src];
  fd[0] = static_cast<uint32_t>(off[src + 1] - off[src]);
}

__global__ void k_fill_exchange(void* x, uint64_t n, int elem_bytes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (elem_bytes == 8) static_cast<uint64_t*>(x)[i] = kExchNone64;
    else static_cast<uint32_t*>(x)[i] = kExchNone32;
  }
}

template <int ALGO>
__global__ void k_part_apply(const void* mine, uint64_t n, void* state, uint8_t* flags,
                             uint32_t iter) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (ALGO == kBfs) {
      uint32_t* level = static_cast<uint32_t*>(state);
      if (static_cast<const uint8_t*>(mine)[v] && level[v] == kUnreached32) {
        level[v] = iter;
        flags[v] = 1;
      }
    } else if (ALGO == kSssp) {
      uint64_t* dist = static_cast<uint64_t*>(state);
      const uint64_t m = static_cast<const uint64_t*>(mine)[v];
      if (m != kExchNone64 && m < dist[v]) {
        dist[v] = m;
        flags[v] = 1;
      }
    } else {
      uint32_t* label = static_cast<uint32_t*>(state);
      const uint32_t m = static_cast<const uint32_t*>(mine)[v];
      if (m < label[v]) {
        label[v] = m;
        flags[v] = 1;
      }
    }
  }
}

// ---------------------------------------------------------------- PageRank
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long x,
                                                            unsigned long long* sh) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_down_sync(kFull, x, d);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = x;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ void add_ctr_fx(uint64_t* ctr, int slot, unsigned long long t) {
  if (t) atomicAdd(reinterpret_cast<unsigned long long*>(ctr + slot), t);
}

// contrib[v] = rank[v] / out[v] (fixed point) into the frontier value slot,
// dangling mass, pushed[] = 0 (traversal.py:218-230).
__global__ void k_pr_prepare(const double* rank, const uint32_t* deg, uint64_t nv, uint64_t* fval,
                             unsigned long long* pushed, uint64_t* ctr) {
  __shared__ unsigned long long sh[32];
  unsigned long long dang = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t rounds = (nv + stride - 1) / stride;
  for (uint64_t r = 0; r < rounds; ++r) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + r * stride;
    if (v < nv) {
      const double rv = rank[v];
      const uint32_t d = deg[v];
      fval[v] = d ? pr_fx(rv * (1.0 / d)) : 0ull;
      if (!d) dang += pr_fx(rv);
      pushed[v] = 0ull;
    }
  }
  const unsigned long long t = block_sum_u64(dang, sh);
  if (threadIdx.x == 0) add_ctr_fx(ctr, kCtrPrDangling, t);
}

// new = (1-d)/V + d (pushed + dangling/V); delta += |new - rank| (traversal.py:231-233)
__global__ void k_pr_update(double* rank, const unsigned long long* pushed, uint64_t nv,
                            double damping, uint64_t* ctr) {
  __shared__ unsigned long long sh[32];
  const double dang = pr_unfx(ctr[kCtrPrDangling]);
  const double base = (1.0 - damping) / static_cast<double>(nv);
  unsigned long long delta = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t rounds = (nv + stride - 1) / stride;
  for (uint64_t r = 0; r < rounds; ++r) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + r * stride;
    if (v < nv) {
      const double nr = base + damping * (pr_unfx(pushed[v]) + dang / static_cast<double>(nv));
      delta += pr_fx(fabs(nr - rank[v]));
      rank[v] = nr;
    }
  }
  const unsigned long long t = block_sum_u64(delta, sh);
  if (threadIdx.x == 0) add_ctr_fx(ctr, kCtrPrDelta, t);
}

// sum of ranks (divide == false) or rank /= sum (divide == true) (traversal.py:248)
__global__ void k_pr_normalize(double* rank, uint64_t nv, uint64_t* ctr, int divide) {
  __shared__ unsigned long long sh[32];
  const double total = pr_unfx(ctr[kCtrPrSum]);
  unsigned long long acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t rounds = (nv + stride - 1) / stride;
  for (uint64_t r = 0; r < rounds; ++r) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + r * stride;
    if (v < nv) {
      if (divide) rank[v] = rank[v] / total;
      else acc += pr_fx(rank[v]);
    }
  }
  if (!divide) {
    const unsigned long long t = block_sum_u64(acc, sh);
    if (threadIdx.x == 0) add_ctr_fx(ctr, kCtrPrSum, t);
  }
}

// any list with a repeated destination (lists sorted): ctr[kCtrBig] = 1
template <typename ET>
__global__ void k_dup_flags(const ET* e, const uint64_t* off, uint64_t nv, uint64_t* ctr) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    for (uint64_t k = off[v] + 1; k < off[v + 1]; ++k)
      if (e[k] == e[k - 1]) {
        ctr[kCtrBig] = 1;
        break;
      }
  }
}

template <int ALGO>
__global__ void k_widen(const void* state, uint64_t nv, int64_t* out) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (ALGO == kBfs) {
      const uint32_t x = static_cast<const uint32_t*>(state)[v];
      out[v] = x == kUnreached32 ? -1ll : static_cast<int64_t>(x);
    } else if (ALGO == kSssp) {
      const uint64_t x = static_cast<const uint64_t*>(state)[v];
      out[v] = x == kUnreached64 ? INT64_MAX : static_cast<int64_t>(x);
    } else {
      out[v] = static_cast<const uint32_t*>(state)[v];
    }
  }
}

template <typename ET>
__global__ void k_check_edges(const ET* edges, uint64_t ne, uint64_t nv,
                              unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (static_cast<uint64_t>(edges[i]) >= nv) atomicAdd(bad, 1ull);
  }
}

// ------------------------------------------------- device-wide u32 -> u64 scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr uint64_t kScanChunk = kScanThreads * kScanItems;

// The size may live in device memory (n_dev, device-driven level loop): the
// kernels then loop over chunks with a fixed grid.
__device__ __forceinline__ uint64_t scan_n(uint64_t n, const uint64_t* n_dev) {
  return n_dev ? *n_dev : n;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* in, uint64_t n0,
                                                              const uint64_t* n_dev,
                                                              uint64_t* part) {
  __shared__ unsigned long long sh[kScanThreads / 32];
  const uint64_t n = scan_n(n0, n_dev), nb = (n + kScanChunk - 1) / kScanChunk;
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint64_t base = b * kScanChunk + threadIdx.x * (uint64_t)kScanItems;
    unsigned long long sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < n) sum += in[base + i];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_down_sync(kFull, sum, d);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < kScanThreads / 32; ++w) t += sh[w];
      part[b] = t;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_scan_partials(uint64_t* part, uint64_t nb0,
                                                        const uint64_t* n_dev) {
  __shared__ uint64_t warp_sums[32];
  const uint64_t nb = n_dev ? (*n_dev + kScanChunk - 1) / kScanChunk : nb0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t chunk = (nb + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min(nb, tid * chunk), hi = min(nb, lo + chunk);
  uint64_t sum = 0;
  for (uint64_t k = lo; k < hi; ++k) sum += part[k];
  uint64_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint64_t ws = warp_sums[lane];
    uint64_t wi = ws;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t t = __shfl_up_sync(kFull, wi, d);
      if (lane >= d) wi += t;
    }
    warp_sums[lane] = wi - ws;
  }
  __syncthreads();
  uint64_t run = warp_sums[wid] + incl - sum;
  for (uint64_t k = lo; k < hi; ++k) {
    const uint64_t c = part[k];
    part[k] = run;
    run += c;
  }
  if (hi == nb && lo < hi) part[nb] = run;
  if (nb == 0 && tid == 0) part[0] = 0;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* in, uint64_t n0,
                                                            const uint64_t* n_dev,
                                                            const uint64_t* part, uint64_t* out) {
  __shared__ unsigned long long warp_tot[kScanThreads / 32];
  const uint64_t n = scan_n(n0, n_dev), nb = (n + kScanChunk - 1) / kScanChunk;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (nb == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint64_t base = b * kScanChunk + threadIdx.x * (uint64_t)kScanItems;
    uint32_t vals[kScanItems];
    unsigned long long sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      vals[i] = base + i < n ? in[base + i] : 0;
      sum += vals[i];
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    unsigned long long run = part[b] + incl - sum;
    for (int w = 0; w < wid; ++w) run += warp_tot[w];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < n) out[base + i] = run;
      run += vals[i];
    }
    if (b == nb - 1 && threadIdx.x == kScanThreads - 1) out[n] = part[nb];
    __syncthreads();
  }
}

int grid_for(uint64_t work, int threads, int num_sms, int per_sm) {
  uint64_t g = (work + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

template <typename K>
int resident_ctas(K kernel, int threads, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  return num_sms * (per_sm > 0 ? per_sm : 1);
}

template <int STRAT, int ALGO, typename ET, typename WT, int U,
          int LD = DefaultLd<STRAT>::value>
cudaError_t expand_sweep(const ExpandArgs& a, int num_sms, cudaStream_t st,
                         uint64_t* launches) {
  // window counts -> global exclusive prefix (wpre[n] = total windows)
  const int g1 = grid_for(a.n, 256, num_sms, 16);
  k_window_counts<STRAT, ET><<<g1, 256, 0, st>>>(a);
  cudaError_t e =
      scan_u32_to_u64(a.wcnt, a.wpre, a.n, a.scan_tmp, a.scan_tmp_bytes, st, a.n_dev);
  if (e != cudaSuccess) return e;
  static int carve = -2;  // per instantiation: the carveout last set
  if (a.carveout != carve && a.carveout >= -1) {
    cudaFuncSetAttribute(k_expand_sweep<STRAT, ALGO, ET, WT, U, LD>,
                         cudaFuncAttributePreferredSharedMemoryCarveout,
                         a.carveout < 0 ? -1 : a.carveout);
    carve = a.carveout;
  }
  static int grid = 0;  // per instantiation: all CTAs resident at once
  if (!grid)
    grid = resident_ctas(k_expand_sweep<STRAT, ALGO, ET, WT, U, LD>, kSweepThreads, num_sms);
  const int g = a.ctas_per_sm > 0 ? num_sms * a.ctas_per_sm : grid;
  k_expand_sweep<STRAT, ALGO, ET, WT, U, LD><<<g, kSweepThreads, 0, st>>>(a);
  *launches += 5;
  return cudaGetLastError();
}

template <int STRAT, int ALGO, typename ET, typename WT, int U>
cudaError_t expand_u(const ExpandArgs& a, int num_sms, cudaStream_t st, uint64_t* launches) {
  if constexpr (ALGO == kPr && STRAT == kMergedAligned && sizeof(ET) == 4) {
    // PageRank's full-list passes: whole-line 3-sector windows like BFS / CC
    if (!a.chunk_sched && (a.ld < 0 || a.ld == 4))
      return expand_sweep<STRAT, ALGO, ET, WT, U, 4>(a, num_sms, st, launches);
  }
  if (!a.chunk_sched || STRAT == kPacked)
    return expand_sweep<STRAT, ALGO, ET, WT, U>(a, num_sms, st, launches);
  // default: 8 resident 256-thread CTAs per SM = 64 warps/SM (register-limited below)
  const int per_sm = a.ctas_per_sm > 0 ? a.ctas_per_sm : 2048 / kExpandThreads;
  const int g = grid_for((a.n + kWarp - 1) / kWarp * kWarp, kExpandThreads, num_sms, per_sm);
  k_expand_warp<STRAT, ALGO, ET, WT, U><<<g, kExpandThreads, 0, st>>>(a);
  k_big_scan<<<1, 1024, 0, st>>>(a.big_prefix, a.ctr);
  k_expand_big<STRAT, ALGO, ET, WT, U><<<num_sms * per_sm, kExpandThreads, 0, st>>>(a);
  *launches += 3;
  return cudaGetLastError();
}

// Unroll variants of the raw-list sweeps (u32 lists, or SSSP's interleaved
// pairs): `value` = the default windows per warp batch.
template <int STRAT, int ALGO, typename ET, typename WT>
struct SweepUnroll {
  static constexpr bool tunable =
      (STRAT == kMergedAligned || STRAT == kMerged || STRAT == kPacked) &&
      !AlgoTraits<ALGO>::pull && ALGO != kPr &&
      ((sizeof(ET) == 4 && sizeof(WT) == 4) || IsPair<WT>::value);
  static constexpr bool raw_line = STRAT == kMergedAligned || STRAT == kMerged;
  static constexpr int value =
      raw_line && ALGO == kBfs ? 16
      : raw_line && (AlgoTraits<ALGO>::base == kBfs || AlgoTraits<ALGO>::base == kCc) &&
              !AlgoTraits<ALGO>::uf
          ? 8
          : 4;
};

template <int STRAT, int ALGO, typename ET, typename WT>
cudaError_t expand_t(const ExpandArgs& a, int num_sms, cudaStream_t st, uint64_t* launches) {
  if (STRAT == kNaive) {
    const int per_sm = a.ctas_per_sm > 0 ? a.ctas_per_sm : 2048 / kExpandThreads;
    const int g = grid_for(a.n, kExpandThreads, num_sms, per_sm);
    k_expand_naive<ALGO, ET, WT><<<g, kExpandThreads, 0, st>>>(a);
    *launches += 1;
    return cudaGetLastError();
  }
  // Windows per warp batch of the raw-list sweeps.  Merged / merged-aligned
  // BFS take 16 by default, CC (and partitioned BFS) 8: more loads in flight
  // per warp, and adjacent lists' windows (which share lines) issued back to
  // back by one warp, so the L1 / L2 merge more of the reference's duplicate
  // line requests (profiles/r02_unroll_ab.txt, K27 BFS merged-aligned: 4 -> 8
  // +1.8 %, 8 -> 16 +2.1 % (108 registers then, 127-128 now; 2 CTAs / SM); merged +8 %, +7 %;
  // CC-K27-sym merged-aligned 4 -> 8 +2.3 %, 8 -> 16 -0.9 %; SSSP and packed
  // unchanged or slower above 4).  zc_set_tuning unroll=2|4|8|16 and ld=0..3
  // are A/B variants.
  if constexpr (SweepUnroll<STRAT, ALGO, ET, WT>::tunable) {
    if (!a.chunk_sched) {
      const int u = a.unroll ? a.unroll : SweepUnroll<STRAT, ALGO, ET, WT>::value;
      if (u == 2) return expand_sweep<STRAT, ALGO, ET, WT, 2>(a, num_sms, st, launches);
      if constexpr ((STRAT == kMergedAligned || STRAT == kMerged) &&
                    (ALGO == kBfs || ALGO == kCc)) {
        if (u == 16) {
          // merged-aligned BFS reads a window of 3 sectors as its whole line by
          // default (ld=4; ld=1 = the plain window loads): one 128-byte request
          // instead of a 96-byte one, which the link serves at 0.33 G/s against
          // 0.39 G/s for full lines (+1.0-1.2 % over K27 sources, r02_promote_ab)
          if constexpr (ALGO == kBfs && STRAT == kMergedAligned) {
            if (a.ld < 0 || a.ld == 4)
              return expand_sweep<STRAT, ALGO, ET, WT, 16, 4>(a, num_sms, st, launches);
          }
          return expand_sweep<STRAT, ALGO, ET, WT, 16>(a, num_sms, st, launches);
        }
      }
      if (u == 8) {
        if constexpr (ALGO == kCc && STRAT == kMergedAligned) {  // whole-line 3-sector windows
          if (a.ld < 0 || a.ld == 4)
            return expand_sweep<STRAT, ALGO, ET, WT, 8, 4>(a, num_sms, st, launches);
        }
        if constexpr (ALGO == kBfs && STRAT != kPacked) {
          if (a.ld == 0) return expand_sweep<STRAT, ALGO, ET, WT, 8, 0>(a, num_sms, st, launches);
          if (a.ld == 2) return expand_sweep<STRAT, ALGO, ET, WT, 8, 2>(a, num_sms, st, launches);
          if (a.ld == 3) return expand_sweep<STRAT, ALGO, ET, WT, 8, 3>(a, num_sms, st, launches);
        }
        return expand_sweep<STRAT, ALGO, ET, WT, 8>(a, num_sms, st, launches);
      }
    }
  }
  return expand_u<STRAT, ALGO, ET, WT, kUnroll>(a, num_sms, st, launches);
}

template <int STRAT, int ALGO>
cudaError_t expand_w(int eb, int wb, const ExpandArgs& a, int num_sms, cudaStream_t st,
                     uint64_t* l) {
  constexpr bool W = AlgoTraits<ALGO>::weighted;
  if constexpr (W) {
    if (a.pairs) return expand_t<STRAT, ALGO, uint64_t, PairW>(a, num_sms, st, l);
  }
  if (eb == 4) {
    if (W && wb == 8) return expand_t<STRAT, ALGO, uint32_t, uint64_t>(a, num_sms, st, l);
    return expand_t<STRAT, ALGO, uint32_t, uint32_t>(a, num_sms, st, l);
  }
  if (W && wb == 8) return expand_t<STRAT, ALGO, uint64_t, uint64_t>(a, num_sms, st, l);
  return expand_t<STRAT, ALGO, uint64_t, uint32_t>(a, num_sms, st, l);
}

template <int STRAT>
cudaError_t expand_a(int algo, int eb, int wb, const ExpandArgs& a, int num_sms, cudaStream_t st,
                     uint64_t* l) {
  switch (algo) {
    case kBfs: return expand_w<STRAT, kBfs>(eb, wb, a, num_sms, st, l);
    case kSssp: return expand_w<STRAT, kSssp>(eb, wb, a, num_sms, st, l);
    case kCc: return expand_w<STRAT, kCc>(eb, wb, a, num_sms, st, l);
    case kPr: return expand_w<STRAT, kPr>(eb, wb, a, num_sms, st, l);
    case kCcUf: return expand_w<STRAT, kCcUf>(eb, wb, a, num_sms, st, l);
    case kBfs + kPartAlgo: return expand_w<STRAT, kBfs + kPartAlgo>(eb, wb, a, num_sms, st, l);
    case kSssp + kPartAlgo: return expand_w<STRAT, kSssp + kPartAlgo>(eb, wb, a, num_sms, st, l);
    default: return expand_w<STRAT, kCc + kPartAlgo>(eb, wb, a, num_sms, st, l);
  }
}

}  // namespace

template <int ALGO>
cudaError_t expand_cmp(const ExpandArgs& a, int num_sms, cudaStream_t st, uint64_t* launches) {
  return expand_sweep<kCompressed, ALGO, uint32_t, uint32_t, kUnroll>(a, num_sms, st, launches);
}

cudaError_t launch_expand(int strategy, int algo, int edge_bytes, int weight_bytes,
                          const ExpandArgs& a, int num_sms, cudaStream_t st, uint64_t* launches) {
  if (a.n == 0) return cudaSuccess;
  if (strategy == kCompressed) {
    switch (algo) {
      case kBfs: return expand_cmp<kBfs>(a, num_sms, st, launches);
      case kSssp: return expand_cmp<kSssp>(a, num_sms, st, launches);
      case kCc: return expand_cmp<kCc>(a, num_sms, st, launches);
      case kPr: return expand_cmp<kPr>(a, num_sms, st, launches);
      case kBfs + kPartAlgo: return expand_cmp<kBfs + kPartAlgo>(a, num_sms, st, launches);
      case kSssp + kPartAlgo: return expand_cmp<kSssp + kPartAlgo>(a, num_sms, st, launches);
      case kCc + kPartAlgo: return expand_cmp<kCc + kPartAlgo>(a, num_sms, st, launches);
      case kBfsPull: return expand_cmp<kBfsPull>(a, num_sms, st, launches);
      case kCcUf: return expand_cmp<kCcUf>(a, num_sms, st, launches);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (strategy) {
    case kNaive: return expand_a<kNaive>(algo, edge_bytes, weight_bytes, a, num_sms, st, launches);
    case kMerged: return expand_a<kMerged>(algo, edge_bytes, weight_bytes, a, num_sms, st, launches);
    case kPacked: return expand_a<kPacked>(algo, edge_bytes, weight_bytes, a, num_sms, st, launches);
    default:
      return expand_a<kMergedAligned>(algo, edge_bytes, weight_bytes, a, num_sms, st, launches);
  }
}

cudaError_t launch_traffic_model(int strategy, int edge_bytes, int weight_bytes, bool weights,
                                 const uint32_t* front, uint64_t n, const uint64_t* off,
                                 uint64_t* ctr, int num_sms, cudaStream_t st, uint64_t* launches) {
  if (n == 0) return cudaSuccess;
  const int g = grid_for(n, 256, num_sms, 8);
  if (strategy == kNaive)
    k_model_naive<<<g, 256, 0, st>>>(front, n, off, edge_bytes, weight_bytes, weights, ctr);
  else if (strategy == kMerged)
    k_model_merged<kMerged><<<g, 256, 0, st>>>(front, n, off, edge_bytes, weight_bytes, weights,
                                               ctr);
  else
    k_model_merged<kMergedAligned><<<g, 256, 0, st>>>(front, n, off, edge_bytes, weight_bytes,
                                                      weights, ctr);
  *launches += 1;
  return cudaGetLastError();
}

namespace {
// Bottom-up step inputs: the current frontier as a bitmap, and the candidate
// marks (unvisited vertices with in-edges), 16 vertices per thread.
__global__ void k_fbits_set(const uint32_t* front, uint64_t n, uint64_t vbase, uint32_t* fbits) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vbase + front[j];
    atomicOr(fbits + (v >> 5), 1u << (v & 31));
  }
}

// Visited bitmap of a partition's owned range from its levels.
__global__ void k_visited_from_levels(const uint32_t* level, uint64_t nv, uint32_t* visited) {
  const uint64_t nw = (nv + 31) / 32;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const uint64_t v = w * 32 + b;
      if (v < nv && level[v] != kUnreached32) bits |= 1u << b;
    }
    visited[w] = bits;
  }
}

__global__ void k_cand_marks(uint64_t nv, const uint32_t* visited, const uint32_t* hasin,
                             uint8_t* cand) {
  const uint64_t ngroups = (nv + 15) / 16;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ngroups;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v0 = t * 16;
    const uint32_t sh = static_cast<uint32_t>(v0 & 31);
    const uint32_t c = ~(visited[v0 >> 5] >> sh) & (hasin[v0 >> 5] >> sh) & 0xffffu;
    uint32_t m[4] = {0, 0, 0, 0};
#pragma unroll
    for (int b = 0; b < 16; ++b)
      if ((c >> b) & 1u) m[b >> 2] |= 1u << ((b & 3) * 8);
    reinterpret_cast<uint4*>(cand)[t] = make_uint4(m[0], m[1], m[2], m[3]);
  }
}

// Bitmap of the vertices with in-edges (bits past nv stay 0).
__global__ void k_hasin(uint64_t nv, const uint64_t* in_off, uint32_t* bits) {
  const uint64_t nw = (nv + 31) / 32;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = 0;
    for (int b = 0; b < 32; ++b) {
      const uint64_t v = w * 32 + b;
      if (v < nv && in_off[v + 1] > in_off[v]) x |= 1u << b;
    }
    bits[w] = x;
  }
}
}  // namespace

cudaError_t launch_pull_prepare(const uint32_t* front, uint64_t n, uint32_t* fbits,
                                uint64_t nv, const uint32_t* visited, const uint32_t* hasin,
                                uint8_t* cand, int num_sms, cudaStream_t st, uint64_t* launches) {
  cudaError_t e = cudaMemsetAsync(fbits, 0, ((nv + 31) / 32 + 1) * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  if (n) k_fbits_set<<<grid_for(n, 256, num_sms, 16), 256, 0, st>>>(front, n, 0, fbits);
  k_cand_marks<<<grid_for((nv + 15) / 16, 256, num_sms, 16), 256, 0, st>>>(nv, visited, hasin,
                                                                            cand);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_hasin(uint64_t nv, const uint64_t* in_off, uint32_t* bits, cudaStream_t st) {
  k_hasin<<<grid_for((nv + 31) / 32 + 1, 256, 148, 16), 256, 0, st>>>(nv, in_off, bits);
  return cudaGetLastError();
}

cudaError_t launch_frontier_bits(const uint32_t* front, uint64_t n, uint64_t vbase,
                                 uint32_t* bits, uint64_t words, int num_sms, cudaStream_t st,
                                 uint64_t* launches) {
  cudaError_t e = cudaMemsetAsync(bits, 0, words * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  if (n) {
    k_fbits_set<<<grid_for(n, 256, num_sms, 16), 256, 0, st>>>(front, n, vbase, bits);
    *launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t launch_part_pull_prepare(const void* level, uint64_t nv, uint32_t* visited,
                                     const uint32_t* hasin, uint8_t* cand, int num_sms,
                                     cudaStream_t st, uint64_t* launches) {
  k_visited_from_levels<<<grid_for((nv + 31) / 32, 256, num_sms, 16), 256, 0, st>>>(
      static_cast<const uint32_t*>(level), nv, visited);
  k_cand_marks<<<grid_for((nv + 15) / 16, 256, num_sms, 16), 256, 0, st>>>(nv, visited, hasin,
                                                                            cand);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_compact(int algo, const CompactArgs& c, cudaStream_t st, uint64_t* launches) {
  const int g = static_cast<int>(c.ntiles < (1u << 20) ? c.ntiles : (1u << 20));
  k_tile_count<<<g, kTileThreads, 0, st>>>(c);
  k_tile_scan<<<1, 1024, 0, st>>>(c);
  switch (algo) {
    case kBfs: k_tile_write<kBfs><<<g, kTileThreads, 0, st>>>(c); break;
    case kSssp: k_tile_write<kSssp><<<g, kTileThreads, 0, st>>>(c); break;
    default: k_tile_write<kCc><<<g, kTileThreads, 0, st>>>(c); break;
  }
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_far_min(const uint8_t* flags, const void* dist, uint64_t nv, uint64_t* ctr,
                           cudaStream_t st, uint64_t* launches) {
  k_far_reset<<<1, 1, 0, st>>>(ctr);
  k_far_min<<<grid_for(nv, 256, 148, 8), 256, 0, st>>>(flags, static_cast<const uint64_t*>(dist),
                                                       nv, ctr);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_uf_flatten(uint32_t* parent, uint64_t nv, cudaStream_t st, uint64_t* launches) {
  if (!nv) return cudaSuccess;
  k_uf_flatten<<<grid_for(nv, 256, 148, 8), 256, 0, st>>>(parent, nv);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_uf_sample(const uint32_t* parent, uint64_t nv, uint32_t* out, uint32_t sample,
                             cudaStream_t st, uint64_t* launches) {
  if (!nv) return cudaSuccess;
  k_uf_sample<<<(sample + 255) / 256, 256, 0, st>>>(parent, nv, out, sample);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_uf_marks(const uint32_t* parent, const uint64_t* off, const uint64_t* cpos,
                            uint64_t nv, uint32_t giant, int strategy, int edge_bytes,
                            uint32_t uf_sample, uint8_t* flags, cudaStream_t st,
                            uint64_t* launches) {
  if (!nv) return cudaSuccess;
  k_uf_marks<<<grid_for(nv, 256, 148, 8), 256, 0, st>>>(parent, off, cpos, nv, giant, strategy,
                                                        edge_bytes, uf_sample, flags);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_fval_ids(const uint32_t* front, uint64_t* fval, uint64_t n, cudaStream_t st,
                            uint64_t* launches) {
  if (!n) return cudaSuccess;
  k_fval_ids<<<grid_for(n, 256, 148, 8), 256, 0, st>>>(front, fval, n);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_init(int algo, void* state, uint64_t nv, uint64_t src, const uint64_t* off,
                        uint32_t* front, uint64_t* fval, uint64_t* fs, uint32_t* fd,
                        cudaStream_t st, uint64_t* launches, uint64_t label_base,
                        bool with_source) {
  if (algo == kCc) {
    if (nv == 0) return cudaSuccess;
    const int g = grid_for(nv, 256, 148, 16);
    k_init_cc<<<g, 256, 0, st>>>(static_cast<uint32_t*>(state), nv, front, fval, off, fs, fd,
                                 label_base);
    *launches += 1;
    return cudaGetLastError();
  }
  const size_t bytes = nv * (algo == kSssp ? 8 : 4);
  cudaError_t e = cudaMemsetAsync(state, 0xff, bytes, st);
  if (e != cudaSuccess || !with_source) return e;
  k_init_source<<<1, 1, 0, st>>>(src, off, front, fval, fs, fd);
  *launches += 1;
  return cudaGetLastError();
}

// elem_bytes 0: x is a bitmap of global ids (count set bits); 4 / 8: an
// array (count entries other than all-ones); only ids outside [lo, hi).
__global__ void k_count_remote(const void* x, int eb, uint64_t n, uint64_t lo, uint64_t hi,
                               unsigned long long* out) {
  unsigned long long c = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (eb == 0) {
    const uint32_t* b = static_cast<const uint32_t*>(x);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n + 31) / 32;
         i += stride) {
      uint32_t m = b[i];
      const uint64_t v0 = i * 32;
      if (v0 + 32 > lo && v0 < hi) {  // clear the owned ids of this word
        const uint64_t a0 = max(lo, v0) - v0, a1 = min(hi, v0 + 32) - v0;
        const uint32_t own = (a1 - a0 == 32) ? 0xffffffffu : (((1u << (a1 - a0)) - 1u) << a0);
        m &= ~own;
      }
      c += __popc(m);
    }
  } else {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      if (i >= lo && i < hi) continue;
      c += eb == 4 ? static_cast<const uint32_t*>(x)[i] != 0xffffffffu
                   : static_cast<const unsigned long long*>(x)[i] != ~0ull;
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_remote(const void* x, int elem_bytes, uint64_t global_nv, uint64_t lo,
                                uint64_t hi, uint64_t* out, int num_sms, cudaStream_t st,
                                uint64_t* launches) {
  if (global_nv == 0) return cudaSuccess;
  k_count_remote<<<num_sms * 8, 256, 0, st>>>(x, elem_bytes, global_nv, lo, hi,
                                               reinterpret_cast<unsigned long long*>(out));
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_fill_exchange(int algo, void* x, uint64_t n, cudaStream_t st,
                                 uint64_t* launches) {
  if (algo == kBfs) return cudaMemsetAsync(x, 0, n, st);
  if (n == 0) return cudaSuccess;
  const int g = grid_for(n, 256, 148, 16);
  k_fill_exchange<<<g, 256, 0, st>>>(x, n, algo == kSssp ? 8 : 4);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_part_apply(int algo, const void* mine, uint64_t nlocal, void* state,
                              uint8_t* flags, uint32_t iter, cudaStream_t st, uint64_t* launches) {
  if (nlocal == 0) return cudaSuccess;
  const int g = grid_for(nlocal, 256, 148, 16);
  switch (algo) {
    case kBfs: k_part_apply<kBfs><<<g, 256, 0, st>>>(mine, nlocal, state, flags, iter); break;
    case kSssp: k_part_apply<kSssp><<<g, 256, 0, st>>>(mine, nlocal, state, flags, iter); break;
    default: k_part_apply<kCc><<<g, 256, 0, st>>>(mine, nlocal, state, flags, iter); break;
  }
  *launches += 1;
  return cudaGetLastError();
}

// Thread per 32-vertex word of the owned range: OR of every rank's bit word
// (peer loads over NVLink, coalesced across threads), applied like
// k_part_apply<kBfs>.
__global__ void k_part_pull_apply(const uint32_t* const* sent, uint32_t nparts, uint64_t lo,
                                  uint64_t n, uint32_t* level, uint8_t* flags, uint32_t iter) {
  const uint64_t w0 = lo >> 5, w1 = (lo + n + 31) >> 5;
  for (uint64_t w = w0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < w1;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = 0;
    for (uint32_t k = 0; k < nparts; ++k) x |= sent[k][w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      const uint64_t v = (w << 5) + b;
      if (v < lo || v >= lo + n) continue;
      const uint64_t lv = v - lo;
      if (level[lv] == kUnreached32) {
        level[lv] = iter;
        flags[lv] = 1;
      }
    }
  }
}

cudaError_t launch_part_pull_apply(const uint32_t* const* sent, uint32_t nparts, uint64_t lo,
                                   uint64_t nlocal, void* state, uint8_t* flags, uint32_t iter,
                                   int num_sms, cudaStream_t st, uint64_t* launches) {
  if (nlocal == 0) return cudaSuccess;
  k_part_pull_apply<<<num_sms * 8, 256, 0, st>>>(sent, nparts, lo, nlocal,
                                                  static_cast<uint32_t*>(state), flags, iter);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_level_end(uint64_t* ctr, uint64_t* log_trav, uint64_t* log_front, uint64_t cap,
                             cudaGraphConditionalHandle loop, cudaStream_t st) {
  k_level_end<<<1, 1, 0, st>>>(ctr, log_trav, log_front, cap, loop);
  return cudaGetLastError();
}

cudaError_t launch_stamp(const uint64_t* ctr, uint64_t* log_t, cudaStream_t st) {
  k_stamp<<<1, 1, 0, st>>>(ctr, log_t);
  return cudaGetLastError();
}

cudaError_t launch_pr_init(uint64_t nv, const uint64_t* off, uint32_t* front, uint64_t* fs,
                           uint32_t* fd, double* rank, cudaStream_t st, uint64_t* launches) {
  if (nv == 0) return cudaSuccess;
  const int g = grid_for(nv, 256, 148, 16);
  k_init_all<<<g, 256, 0, st>>>(nv, off, front, fs, fd, rank);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_pr_prepare(const double* rank, const uint32_t* deg, uint64_t nv, uint64_t* fval,
                              double* pushed, uint64_t* ctr, cudaStream_t st, uint64_t* launches) {
  // pushed holds fixed-point sums (pr_fx): same 8 bytes per vertex
  const int g = grid_for(nv, 256, 148, 8);
  k_pr_prepare<<<g, 256, 0, st>>>(rank, deg, nv, fval,
                                   reinterpret_cast<unsigned long long*>(pushed), ctr);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_pr_update(double* rank, const double* pushed, uint64_t nv, double damping,
                             uint64_t* ctr, cudaStream_t st, uint64_t* launches) {
  const int g = grid_for(nv, 256, 148, 8);
  k_pr_update<<<g, 256, 0, st>>>(rank, reinterpret_cast<const unsigned long long*>(pushed), nv,
                                  damping, ctr);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_pr_normalize(double* rank, uint64_t nv, uint64_t* ctr, bool divide,
                                cudaStream_t st, uint64_t* launches) {
  const int g = grid_for(nv, 256, 148, 8);
  k_pr_normalize<<<g, 256, 0, st>>>(rank, nv, ctr, divide ? 1 : 0);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_dup_flags(const void* sorted, int elem_bytes, const uint64_t* off, uint64_t nv,
                             uint64_t* ctr, cudaStream_t st) {
  if (nv == 0) return cudaSuccess;
  const int g = grid_for(nv, 256, 148, 16);
  if (elem_bytes == 4)
    k_dup_flags<uint32_t><<<g, 256, 0, st>>>(static_cast<const uint32_t*>(sorted), off, nv, ctr);
  else
    k_dup_flags<uint64_t><<<g, 256, 0, st>>>(static_cast<const uint64_t*>(sorted), off, nv, ctr);
  return cudaGetLastError();
}

cudaError_t launch_widen(int algo, const void* state, uint64_t nv, int64_t* out, cudaStream_t st,
                         uint64_t* launches) {
  if (nv == 0) return cudaSuccess;
  const int g = grid_for(nv, 256, 148, 16);
  switch (algo) {
    case kBfs: k_widen<kBfs><<<g, 256, 0, st>>>(state, nv, out); break;
    case kSssp: k_widen<kSssp><<<g, 256, 0, st>>>(state, nv, out); break;
    default: k_widen<kCc><<<g, 256, 0, st>>>(state, nv, out); break;
  }
  *launches += 1;
  return cudaGetLastError();
}

namespace {
// BFS levels below 255 as one byte each (0xff = unreached): the download is
// V bytes instead of 8 V; the host widens to the reference's int64.
__global__ void k_narrow_levels(const uint32_t* level, uint64_t nv, uint8_t* out) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = level[v];
    out[v] = x == kUnreached32 ? 0xffu : static_cast<uint8_t>(x);
  }
}
}  // namespace

cudaError_t launch_narrow_levels(const void* state, uint64_t nv, uint8_t* out, cudaStream_t st,
                                 uint64_t* launches) {
  if (nv == 0) return cudaSuccess;
  k_narrow_levels<<<grid_for(nv, 256, 148, 16), 256, 0, st>>>(static_cast<const uint32_t*>(state),
                                                             nv, out);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_check_edges(const void* edges, int edge_bytes, uint64_t ne, uint64_t nv,
                               uint64_t* bad, cudaStream_t st) {
  if (ne == 0) return cudaSuccess;
  const int g = grid_for(ne, 256, 148, 16);
  if (edge_bytes == 4)
    k_check_edges<uint32_t><<<g, 256, 0, st>>>(static_cast<const uint32_t*>(edges), ne, nv,
                                               reinterpret_cast<unsigned long long*>(bad));
  else
    k_check_edges<uint64_t><<<g, 256, 0, st>>>(static_cast<const uint64_t*>(edges), ne, nv,
                                               reinterpret_cast<unsigned long long*>(bad));
  return cudaGetLastError();
}

size_t scan_tmp_bytes(uint64_t n) {
  const uint64_t nb = (n + kScanChunk - 1) / kScanChunk;
  return (nb + 1) * sizeof(uint64_t);
}

cudaError_t scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp,
                            size_t tmp_bytes, cudaStream_t st, const uint64_t* n_dev) {
  // n: the size, or with n_dev the maximum size (the grid is sized for it)
  if (n == 0 && !n_dev) return cudaMemsetAsync(out, 0, sizeof(uint64_t), st);
  const uint64_t nb = (n + kScanChunk - 1) / kScanChunk;
  if (tmp_bytes < (nb + 1) * sizeof(uint64_t)) return cudaErrorInvalidValue;
  uint64_t* part = static_cast<uint64_t*>(tmp);
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(nb, 148 * 8)));
  k_scan_reduce<<<grid, kScanThreads, 0, st>>>(in, n, n_dev, part);
  k_scan_partials<<<1, 1024, 0, st>>>(part, nb, n_dev);
  k_scan_down<<<grid, kScanThreads, 0, st>>>(in, n, n_dev, part, out);
  return cudaGetLastError();
}

}  // namespace zc
