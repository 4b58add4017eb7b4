/*
 * zcgraph.h -- C ABI of the B200-native EMOGI zero-copy traversal library
 * (libzcgraph_b200.so, built from paper_2006_06890_b200/csrc/).
 *
 * The reference (arxiv 2006.06890, package `zcgraph`, pure Python) has no FFI
 * layer; its boundary is the Python library API.  Each entry point below
 * replaces one reference interface, cited as path:line relative to
 * /root/reference/pkg/src/zcgraph/:
 *
 *   zc_graph_create   <- CsrGraph (csr.py:34-77) + validate (csr.py:80-105):
 *                        the caller's CSR arrays become a handle whose edge /
 *                        weight lists live in pinned mapped host memory
 *                        (ZC_PLACE_ZEROCOPY), host-resident managed memory
 *                        (ZC_PLACE_ZEROCOPY_MANAGED), migrating managed
 *                        memory (ZC_PLACE_UVM) or HBM (ZC_PLACE_HBM);
 *                        offsets and all per-vertex state
 *                        live in HBM.
 *   zc_bfs            <- bfs(g, source, strategy, ...)   traversal.py:98-120
 *   zc_sssp           <- sssp(g, source, strategy, ...)  traversal.py:123-151
 *   zc_cc             <- cc(g, strategy, ...)            traversal.py:154-179
 *   zc_bfs_async / zc_sssp_async / zc_sync
 *                     <- the per-source loop of run_experiment
 *                        (report.py:168-170: one bfs/sssp per picked source)
 *   zc_pagerank       <- pagerank(g, strategy, ...)      traversal.py:191-249
 *   zc_graph_multigraph <- _is_multigraph(g)             traversal.py:182-188
 *   zc_run_log        <- TraversalResult.traversed_edges traversal.py:26-45,63-65
 *   zc_run_traffic    <- TraversalResult.per_iteration_traffic (the modelled
 *                        request histogram, coalesce.py:44-85,165-207)
 *   strategy ids      <- AccessStrategy                  access.py:28-31
 *   ZC_UNREACHED_*    <- UNREACHED_LEVEL / UNREACHED_DIST traversal.py:22-23
 *
 * Conventions
 *   - Every function returning int returns ZC_OK (0) on success and a
 *     negative ZC_E* code otherwise; zc_last_error() then returns a message
 *     (thread-local, valid until the next call on that thread).
 *   - ZC_EINVAL is returned for exactly the conditions the reference raises
 *     ValueError for (source out of range, missing / negative weights, CC on
 *     a directed graph, invariant violations); the Python wrapper maps it to
 *     ValueError and every other code to RuntimeError.
 *   - Results are written as int64 into caller-owned buffers of length V
 *     (the reference's result dtype).  Calls on one handle are serialised by
 *     the caller; different handles may be used from different threads.
 *   - No torch / C++ types cross this boundary.
 */
#ifndef ZCGRAPH_H_
#define ZCGRAPH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZC_ABI_VERSION 1

/* status codes */
#define ZC_OK 0
#define ZC_EINVAL (-1)   /* reference ValueError conditions */
#define ZC_ECUDA (-2)    /* CUDA runtime / driver error */
#define ZC_ENOMEM (-3)   /* host or device allocation failed */
#define ZC_ESTATE (-4)   /* API misuse (null handle, wrong placement, ...) */

/* access strategies (access.py:28-31, report.py:31-35 names) */
#define ZC_NAIVE 0          /* "naive": thread per frontier vertex          */
#define ZC_MERGED 1         /* "merged": warp per vertex, 32-element steps  */
#define ZC_MERGED_ALIGNED 2 /* "merged-aligned": first step floored to 128 B */
#define ZC_PACKED 3         /* B200 extension (not in the reference): windows are
                               aligned 32-element blocks of the union of the
                               frontier's lists, each fetched once           */
#define ZC_COMPRESSED 4     /* B200 host-store option: lists sorted and stored
                               delta-encoded in 128-byte lines
                               (zc_graph_build_compressed)                   */
#define ZC_DIRECTION_OPT 5  /* B200 extension, BFS only: compressed top-down
                               steps, switching to bottom-up steps (unvisited
                               vertices scan their compressed in-lists for a
                               parent in the frontier) when the frontier's
                               out-edges outnumber half the unvisited
                               vertices' in-edges.  Same levels, iterations and
                               traversed_edges (the frontier's out-degrees)  */

/* where the edge / weight lists live */
#define ZC_PLACE_ZEROCOPY 0 /* cudaHostAlloc(Mapped|Portable) or cudaHostRegister */
#define ZC_PLACE_UVM 1      /* cudaMallocManaged + cudaMemAdviseSetReadMostly     */
#define ZC_PLACE_HBM 2      /* cudaMalloc: in-HBM control run                     */
#define ZC_PLACE_ZEROCOPY_MANAGED 3 /* B200 host mapping (not in the reference):
                               host-resident cudaMallocManaged lists
                               (PreferredLocation = CPU, AccessedBy = the GPU),
                               never migrated; the GPU reads them over PCIe with
                               the same zero-copy loads, through the UVM
                               driver's large-page GPU mappings             */

/* zc_graph_desc.flags */
#define ZC_F_DIRECTED 1u        /* CsrGraph.directed (csr.py:45)                     */
#define ZC_F_REGISTER 2u        /* ZEROCOPY: cudaHostRegister the caller's edge /
                                   weight buffers in place instead of copying; they
                                   must outlive the handle, be 128 B aligned and
                                   already have the device element width          */
#define ZC_F_UVM_PREFETCH 4u    /* UVM: cudaMemPrefetchAsync the lists before runs   */
#define ZC_F_NO_VALIDATE 8u     /* skip the O(V+E) invariant check (trusted input)   */

/* unreached markers in the int64 results (traversal.py:22-23) */
#define ZC_UNREACHED_LEVEL (-1LL)
#define ZC_UNREACHED_DIST (0x7fffffffffffffffLL)

typedef struct zc_graph zc_graph;

typedef struct zc_graph_desc {
  uint64_t num_vertices;       /* V (device path requires V < 2^32 - 1)        */
  uint64_t num_edges;          /* E                                            */
  const int64_t *offsets;      /* V+1 entries, offsets[0]=0, offsets[V]=E      */
  const void *edges;           /* E entries of src_edge_bytes each             */
  const void *weights;         /* NULL or E entries of src_weight_bytes each   */
  uint32_t src_edge_bytes;     /* width of the caller's edge array: 4 or 8     */
  uint32_t src_weight_bytes;   /* width of the caller's weight array: 4 or 8   */
  uint32_t edge_elem_bytes;    /* CsrGraph.edge_elem_bytes: 4 or 8 (device)    */
  uint32_t weight_elem_bytes;  /* CsrGraph.weight_elem_bytes: 4 or 8 (device)  */
  int32_t placement;           /* ZC_PLACE_*                                   */
  int32_t device;              /* CUDA device ordinal                          */
  uint32_t flags;              /* ZC_F_*                                       */
  uint32_t reserved;
} zc_graph_desc;

/* Per-run statistics.  traversed_edges / frontier sizes per iteration are
 * retrieved with zc_run_log (the count can exceed any fixed array). */
typedef struct zc_stats {
  uint64_t iterations;             /* TraversalResult.iterations            */
  uint64_t total_traversed_edges;  /* sum of traversed_edges                */
  uint64_t max_frontier;           /* largest frontier                      */
  double kernel_ms;                /* device time of the traversal loop     */
  double total_ms;                 /* host wall time of the whole call      */
  double d2h_ms;                   /* device time of the result download    */
  uint64_t h2d_bytes;              /* bytes copied host->device in the call */
  uint64_t d2h_bytes;              /* bytes copied device->host in the call */
  uint64_t launches;               /* kernels launched by the call          */
  double expand_ms;                /* device time of the expansion kernels
                                      (the zero-copy edge stream) alone     */
  uint64_t exchange_bytes;         /* partitions: bytes this rank sent to the
                                      others since zc_part_begin (reduce-
                                      scatter share, or fused remote sends) */
  uint64_t reserved[5];
} zc_stats;

const char *zc_last_error(void);
int zc_abi_version(void);
int zc_device_count(int *count);

/* Graph handle lifecycle. */
int zc_graph_create(const zc_graph_desc *desc, zc_graph **out);
void zc_graph_destroy(zc_graph *g);
/* Open an EMGI v1 file (csr.py:17-23, 180-245: 28-byte header, u64 offsets,
 * 128-byte aligned edge / weight payloads) straight into a handle: the
 * payloads are read in parallel directly into their pinned (zero-copy),
 * managed (UVM) or staging (HBM) buffers.  Same errors as load_csr_binary
 * (ZC_EINVAL: truncated / bad magic / version).  flags: ZC_F_DIRECTED (the
 * reference's directed argument), ZC_F_UVM_PREFETCH, ZC_F_NO_VALIDATE. */
int zc_graph_open_emgi(const char *path, int32_t placement, int32_t device, uint32_t flags,
                       zc_graph **out);

/* Host pointers of the handle's edge / weight lists (pinned, managed or a
 * host shadow for HBM placement) -- used by checkers and generators. */
int zc_graph_host_lists(zc_graph *g, void **edges, void **weights, const int64_t **offsets);
int zc_graph_info(const zc_graph *g, uint64_t *num_vertices, uint64_t *num_edges,
                  uint32_t *edge_elem_bytes, uint32_t *weight_elem_bytes,
                  int32_t *placement, uint32_t *flags);

/* Traversals (reference traversal.py:98-179).  out: caller buffer, V int64. */
int zc_bfs(zc_graph *g, uint64_t source, int strategy, int64_t *out, zc_stats *stats);
int zc_sssp(zc_graph *g, uint64_t source, int strategy, int64_t *out, zc_stats *stats);
int zc_cc(zc_graph *g, int strategy, int64_t *out, zc_stats *stats);

/* Work-efficient schedules (B200 extensions; the reference's SSSP and CC are
 * Jacobi iterations, traversal.py:123-179).  The values are identical -- the
 * distances and min-id labels are unique fixpoints -- while iteration counts
 * and per-iteration traversed edges follow the schedule:
 *   zc_sssp_nearfar: the frontier holds only the improved vertices with
 *     dist < threshold (near set); the others wait marked (far pile); when
 *     the near set runs dry the threshold moves to the smallest waiting
 *     distance + delta (delta = 0: the default, 16).
 *   zc_cc_afforest: union-find (Afforest's schedule): pass 1 unions every
 *     vertex with the neighbours of its list's first window (compressed: the
 *     first 4 elements of a short list, 32 samples of a long list's first
 *     line), pass 2 only the
 *     vertices outside the largest component whose lists reach further;
 *     iterations = passes.  Strategies naive .. compressed. */
int zc_sssp_nearfar(zc_graph *g, uint64_t source, int strategy, uint64_t delta, int64_t *out,
                    zc_stats *stats);
int zc_cc_afforest(zc_graph *g, int strategy, int64_t *out, zc_stats *stats);
/* Pipelined variants for a batch of sources on one handle: return as soon as
 * the traversal has finished (stats and zc_run_log are final), while the
 * int64 result is still being downloaded to `out` on a second stream -- so
 * the D2H of source k overlaps the edge-list reads of source k+1.  `out`
 * must stay valid and untouched until zc_sync(g) returns; stats->d2h_ms is 0.
 * Up to two downloads are in flight; a third call waits for the oldest. */
int zc_bfs_async(zc_graph *g, uint64_t source, int strategy, int64_t *out, zc_stats *stats);
int zc_sssp_async(zc_graph *g, uint64_t source, int strategy, int64_t *out, zc_stats *stats);
int zc_sync(zc_graph *g);

/* PageRank (traversal.py:191-249): synchronous push over the whole edge list
 * every iteration, float64, dangling mass redistributed uniformly, stop when
 * the L1 change < tol or after max_iters; ranks normalised to sum 1.  out:
 * caller buffer of V doubles.  Same ValueError conditions (ZC_EINVAL). */
int zc_pagerank(zc_graph *g, int strategy, double damping, uint64_t max_iters, double tol,
                double *out, zc_stats *stats);
/* Build (once) the line-compressed copy of the lists in the handle's
 * placement: every list that reads fewer 32-byte sectors that way is sorted
 * and stored as self-describing 128-byte lines (u32 base, 6-bit delta width,
 * 8-bit count, deltas); the other lists stay in the raw edge list.
 * *compressed_bytes (may be NULL) receives the line stream's size.  Built
 * automatically by the first ZC_COMPRESSED run. */
int zc_graph_build_compressed(zc_graph *g, uint64_t *compressed_bytes);
/* Build (once) the in-lists of the graph as a compressed line stream (the
 * transpose, built on the GPU; an undirected graph reuses its out-lists) for
 * the bottom-up steps of ZC_DIRECTION_OPT.  *compressed_bytes (may be NULL)
 * receives its size.  Built automatically by the first ZC_DIRECTION_OPT run. */
int zc_graph_build_in_lists(zc_graph *g, uint64_t *compressed_bytes);
/* Copy the compressed-line index to the caller's V+1 u64 buffer: vertex v's
 * list is lines [first_line[v], first_line[v+1]) of the stream (none: read
 * raw).  ZC_ESTATE before zc_graph_build_compressed. */
int zc_graph_compressed_index(const zc_graph *g, uint64_t *first_line);
/* Build (once) an interleaved copy of the lists as 8-byte (dst, weight) u32
 * pairs in the handle's placement; SSSP then reads one stream instead of two,
 * so a list of n edges costs ceil(8n/128) line requests instead of two
 * half-used ones.  A B200 layout choice; results are identical.  zc_sssp /
 * zc_sssp_nearfar build it on first use for the merged, merged-aligned and
 * packed strategies (4-byte edges and weights; +8 bytes per edge of host
 * memory; tuning "pairs=0" opts out).  The request model
 * (ZC_OPT_TRAFFIC_MODEL) keeps describing the reference's separate arrays, so
 * modelled runs read those. */
int zc_graph_build_pairs(zc_graph *g);
/* Wall-time log of the handle's one-time builds (compressed out / in streams):
 * "phase milliseconds" lines in build order, NUL-terminated in buf (at most
 * cap bytes); returns the bytes the whole log needs (>= 1). */
int zc_graph_build_log(const zc_graph *g, char *buf, size_t cap);
/* 1 if some list repeats a destination (traversal.py:182-188), cached. */
int zc_graph_multigraph(zc_graph *g, int *out);

/* Per-iteration log of the handle's most recent run: traversed_edges[k] =
 * sum of frontier degrees of iteration k (traversal.py:63-65) and the
 * frontier size.  Copies min(capacity, iterations) entries; either pointer
 * may be NULL. */
int zc_run_log(const zc_graph *g, uint64_t *traversed_edges, uint64_t *frontier_sizes,
               uint64_t capacity);

/* Bytes of the compressed line streams (out- and in-lists) the expansion
 * kernels of the last ZC_COMPRESSED / ZC_DIRECTION_OPT run requested over the
 * link (4 bytes per loaded word; 0 for the other strategies). */
int zc_run_link_bytes(const zc_graph *g, uint64_t *bytes);
/* Direction of each iteration of the last ZC_DIRECTION_OPT run: 1 = bottom-up
 * step, 0 = top-down; at most `cap` entries (the run's iterations). */
int zc_run_directions(const zc_graph *g, uint8_t *bottom_up, uint64_t cap);
/* Device time (ms, CUDA events on the handle's stream) of each iteration's
 * expansion kernels in the most recent run. */
int zc_run_profile(const zc_graph *g, double *expand_ms, uint64_t capacity);

/* UVM placement: migrate the lists back to host memory so the next run
 * starts cold (the paper's UVM timing).  No-op otherwise. */
int zc_graph_evict(zc_graph *g);

/* UVM placement: migrate the lists to the device now (cudaMemPrefetchAsync on
 * the handle's stream; the lists stay read-mostly) -- the paper's UVM
 * comparison with prefetch, after zc_graph_evict for a cold start.  *ms (may
 * be NULL) = the migration's device time.  No-op (ms 0) on other placements. */
int zc_graph_prefetch(zc_graph *g, float *ms);

/* Per-handle run options. */
#define ZC_OPT_TRAFFIC_MODEL 1u /* also evaluate the reference's request model
                                   (coalesce.py:165-207) on every frontier */
#define ZC_OPT_HOST_LOOP 2u     /* drive the levels from the host instead of the
                                   device-driven CUDA-graph loop (default for the
                                   merged / merged-aligned / packed strategies) */
int zc_set_options(zc_graph *g, uint32_t options);

/* Launch tuning of a handle (B200 extension, no reference counterpart):
 * comma-separated "unroll=2|4|8", "ctas=N" (sweep CTAs per SM),
 * "sched=chunk|sweep", "loop=host|device" (host-driven level loop, e.g. under
 * a profiler, which cannot see kernels inside conditional graph nodes),
 * "do_alpha=X" (direction-optimizing switch factor), "ld=0..4" (load flavour of
 * the raw-list BFS sweeps: L1::no_allocate, L1-cached, read-only path,
 * L1::evict_first; 4 = L1-cached with a 3-sector merged-aligned window read
 * as its whole 128-byte line, the merged-aligned BFS default -- ld=1 gives
 * its plain windows), "pairs=0|1" (SSSP reads the separate edge and weight
 * arrays / the interleaved pairs stream), "carveout=0..100" (the sweeps'
 * preferred shared-memory carveout; no measurable effect on K27 BFS),
 * "widen=N" (host threads widening a pipelined result; more slow the next
 * traversal's zero-copy reads: K27, 2 / 4 / 8 / 12 threads, e2e 45.8 / 45.6 /
 * 45.5 / 45.0 GTEPS direction-optimizing), "uf_sample=N" (afforest's
 * sampling pass over compressed lists: elements per short list, default 4;
 * >= 96 reads short lists and long lists' first lines whole), "sort=radix|
 * segmented" (compressed builds sort the lists by two stable radix-sort
 * transposes, which also yield the in-lists, or -- the fallback when their four
 * edge-sized device buffers do not fit -- a count / scatter transpose and a
 * segmented sort).
 * "unroll" also takes 16 (merged / merged-aligned BFS and CC).  NULL or "" resets the
 * defaults; an unknown entry is ZC_EINVAL.  Read by the run path; nothing is
 * taken from the environment. */
int zc_set_tuning(zc_graph *g, const char *spec);

/* Modelled request histogram of the most recent run (needs
 * ZC_OPT_TRAFFIC_MODEL): for iteration k, hist[8k+i] = edge-list requests of
 * (i+1)*32 bytes and hist[8k+4+i] = weight-list requests (SSSP), i = 0..3 --
 * TrafficStats.hist of traversal.py:66-73.  Copies min(capacity, iterations)
 * iterations. */
int zc_run_traffic(const zc_graph *g, uint64_t *hist, uint64_t capacity);

/* Pinned host memory for result buffers (D2H at link speed). */
void *zc_host_alloc(size_t bytes);
void zc_host_free(void *p);

/* Native synthetic graph generators.  The graph is
 * generated on `device`, written straight into a new handle with the given
 * placement; deterministic in (parameters, seed).
 *   rmat:    R-MAT / Kronecker (a,b,c; d = 1-a-b-c), 2^scale vertices,
 *            edge_factor * 2^scale arcs, Feistel vertex permutation,
 *            duplicates / self loops kept; symmetrize!=0 adds reverse arcs
 *            (csr.py:350-359 semantics, lists sorted by destination).
 *   uniform: out-degree in [min_degree, max_degree], destinations uniform
 *            without in-list duplicates (csr.py:248-282 semantics).
 *   weights (both): uniform integers in [wlow, whigh] when wlow <= whigh,
 *            none when wlow > whigh. */
int zc_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                     uint64_t seed, int symmetrize, int64_t wlow, int64_t whigh,
                     int32_t placement, int32_t device, zc_graph **out);
int zc_generate_uniform(uint64_t num_vertices, uint32_t min_degree, uint32_t max_degree,
                        uint64_t seed, int64_t wlow, int64_t whigh, int32_t placement,
                        int32_t device, zc_graph **out);

/* ---------------------------------------------------------------------------
 * Vertex-range partitions (multi-GPU; no reference counterpart --
 * the paper lists multi-GPU as future work).
 * Rank k owns global vertices [bounds[k], bounds[k+1]) and holds only their
 * lists (offsets rebased to its edge slice, destinations global), streamed
 * over its own host link.  One iteration = zc_part_expand (writes candidates
 * for ANY global vertex into the caller's device exchange buffer of
 * nparts*stride slots; global w of part j -> slot j*stride + w - bounds[j]),
 * a reduce-scatter of that buffer by the caller (BFS: u8 flags, MAX; SSSP:
 * int64 candidate distances, MIN, none = INT64_MAX; CC: int32 candidate
 * labels, MIN, none = INT32_MAX), and
 * zc_part_apply with this rank's reduced slice.  Iterates, per-iteration
 * traversed edges (summed over ranks) and results equal the single-graph run.
 * ------------------------------------------------------------------------- */
typedef struct zc_part_info {
  uint64_t global_vertices;
  uint64_t stride;         /* slots per part in the exchange buffer (>= max range) */
  const uint64_t *bounds;  /* nparts + 1 range starts, bounds[nparts] = global V */
  uint32_t nparts, part;
} zc_part_info;

/* local: this part's CSR (V = its range, offsets rebased, global destinations). */
int zc_part_create(const zc_graph_desc *local, const zc_part_info *info, zc_graph **out);
size_t zc_part_exchange_elem_bytes(int algo); /* algo: 0 bfs, 1 sssp, 2 cc */
int zc_part_begin(zc_graph *g, int algo, uint64_t source, int strategy, uint64_t *n_local,
                  uint64_t *traversed_local);
int zc_part_expand(zc_graph *g, void *exchange /* device pointer */);
int zc_part_apply(zc_graph *g, const void *mine /* device pointer, stride slots */,
                  uint64_t *n_next, uint64_t *traversed_next);
/* Direction-optimizing partitions (strategy ZC_DIRECTION_OPT, bfs):
 *   zc_part_build_in_lists  the owned vertices' in-lists as a compressed line
 *                           stream: an undirected partition reuses its
 *                           out-lists; a directed one must come from
 *                           zc_generate_rmat_part (every rank enumerates the
 *                           counter-based arcs into its range; no exchange).
 *                           Built by zc_part_begin when needed.
 *   zc_part_unvisited_in    in-edges of the owned, still unvisited vertices
 *                           (sum over ranks = the switch test's denominator).
 *   zc_part_frontier_bits   zero the caller's device bitmap of
 *                           (global_vertices + 31) / 32 + 1 words and set the
 *                           owned frontier's bits (global ids).  Ranks own
 *                           disjoint bits, so a SUM all-reduce of the words
 *                           is their OR.
 *   zc_part_pull            a bottom-up step with the all-reduced bitmap in
 *                           place of zc_part_expand + zc_part_apply: the
 *                           owned unvisited vertices scan their in-lists. */
int zc_part_build_in_lists(zc_graph *g, uint64_t *compressed_bytes);
int zc_part_unvisited_in(const zc_graph *g, uint64_t *in_edges);
int zc_part_frontier_bits(zc_graph *g, uint32_t *bits);
int zc_part_pull(zc_graph *g, const uint32_t *bits, uint64_t *n_next, uint64_t *trav_next);
int zc_part_result(zc_graph *g, int64_t *out_local /* range size, or NULL: stats only */,
                   zc_stats *stats);
/* Fused exchange (no reduce-scatter): the expand kernel writes each candidate
 * straight into its owner's buffer -- peer memory over NVLink (CUDA IPC) --
 * BFS: byte stores, deduplicated per iteration; SSSP / CC: atomicMin
 * reductions.  Per iteration: every rank zc_part_fused_reset; barrier;
 * zc_part_fused_expand; barrier; zc_part_apply(g, local, ...).
 * init allocates this rank's buffer (stride slots) and exports its IPC
 * handle (64 bytes, may be NULL); connect opens the other ranks' handles
 * (nparts * 64 bytes, own slot ignored) or, for parts sharing one device and
 * process, takes raw device pointers (ptrs, nparts entries). */
int zc_part_fused_init(zc_graph *g, int algo, void *ipc_handle_out, void **local_buffer);
int zc_part_fused_connect(zc_graph *g, const void *ipc_handles, void *const *ptrs);
int zc_part_fused_reset(zc_graph *g);
int zc_part_fused_expand(zc_graph *g);
/* BFS bitmap exchange (no collective, no remote stores): every rank marks its
 * discoveries in its own global-V bitmap; each owner then ORs the ranks'
 * words over its range, reading the peers' bitmaps through CUDA IPC (NVLink),
 * and applies them -- V/8 bytes read per rank and level, coalesced.  Per
 * iteration: zc_part_bitmap_expand; barrier; zc_part_bitmap_apply; barrier
 * (the termination all-reduce).  init exports this rank's bitmap handle (64
 * bytes, may be NULL) and its device address (may be NULL); connect opens the
 * others' (nparts * 64 bytes, own slot ignored) or takes raw device pointers
 * for parts in one process. */
int zc_part_bitmap_init(zc_graph *g, void *ipc_handle_out, void **local_bitmap);
int zc_part_bitmap_connect(zc_graph *g, const void *ipc_handles, void *const *ptrs);
int zc_part_bitmap_expand(zc_graph *g);
int zc_part_bitmap_apply(zc_graph *g, uint64_t *n_next, uint64_t *trav_next);

/* Part `part` of the graph zc_generate_rmat builds with the same parameters
 * (same arcs, same lists), edge-balanced across nparts; bounds (nparts+1)
 * receives the vertex ranges of all parts.  symmetrize != 0: the part of the
 * symmetrized graph (reverse arcs added, csr.py:350-359 semantics, lists
 * sorted; no weights), cut at 2E*k/nparts of its arcs -- every rank
 * enumerates the counter-based arcs into its range, no edge exchange. */
int zc_generate_rmat_part(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                          uint64_t seed, int symmetrize, int64_t wlow, int64_t whigh,
                          uint32_t nparts, uint32_t part, int32_t placement, int32_t device,
                          uint64_t *bounds, zc_graph **out);

#ifdef __cplusplus
}
#endif
#endif /* ZCGRAPH_H_ */
