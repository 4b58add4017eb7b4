"""BFS / SSSP / CC over zero-copy CSR on a B200 -- drop-in for the reference's
traversal entry points (/root/reference/pkg/src/zcgraph/traversal.py:98-179).

Same signatures, same argument checks (same ValueError conditions and
messages), same ``TraversalResult`` (int64 values with -1 / INT64_MAX for
unreached, iteration count, per-iteration traversed edges, per-iteration
modelled traffic).  The work runs in the CUDA library through the C ABI;
there is no CPU path.  Extra keyword-only arguments select the placement of
the edge list (``placement="zerocopy" | "zerocopy-managed" | "uvm" | "hbm"``)
and the GPU.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .access import AccessStrategy, strategy_id
from .device import DeviceGraph, _pagerank_run, device_graph, is_multigraph
from .traffic import TrafficStats

UNREACHED_LEVEL = -1
UNREACHED_DIST = np.iinfo(np.int64).max

# Schedules beyond the reference's Jacobi iteration (B200 extensions): the
# values are the same unique fixpoints (distances, min-id labels); iteration
# counts and per-iteration traversed edges follow the schedule.
SCHEDULES = {"sssp": ("near-far",), "cc": ("afforest",)}


def _check_schedule(algo: str, schedule: str, collect_traffic) -> None:
    if schedule == "jacobi":
        return
    if schedule not in SCHEDULES[algo]:
        raise ValueError(f"unknown {algo} schedule {schedule!r}: 'jacobi' or "
                         + " / ".join(repr(x) for x in SCHEDULES[algo]))
    if collect_traffic:
        raise ValueError("the request model follows the reference's Jacobi schedule; "
                         f"run schedule={schedule!r} with collect_traffic=False")


@dataclass
class TraversalResult:
    """Reference traversal.py:26-45, plus the device run statistics."""

    algo: str
    values: np.ndarray
    iterations: int
    per_iteration_traffic: list
    traversed_edges: list
    flags: tuple = ()
    page_streams: Optional[list] = None
    frontier_sizes: list = field(default_factory=list)
    kernel_ms: float = 0.0
    total_ms: float = 0.0
    d2h_ms: float = 0.0
    expand_ms: float = 0.0
    launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    @property
    def total_traffic(self) -> TrafficStats:
        total = TrafficStats.zero()
        for s in self.per_iteration_traffic:
            total = total.merged_with(s)
        return total

    @property
    def total_traversed_edges(self) -> int:
        return sum(self.traversed_edges)


def _check_source(g, source: int) -> None:
    # traversal.py:93-95
    if not 0 <= source < g.num_vertices:
        raise ValueError(f"source {source} out of range for {g.num_vertices} vertices")


def _has_weights(g) -> bool:
    if isinstance(g, DeviceGraph):
        return g.has_weights
    return g.weights is not None


def _model_wanted(collect_traffic: Optional[bool], sid: int) -> bool:
    """The reference's request model (coalesce.py:165-207) is defined for its
    three strategies only.  ``collect_traffic=None`` (the default) means "if
    the strategy has a model": on for naive / merged / merged-aligned (the
    reference's default, traversal.py:99), off for the B200 extensions, which
    then return zero TrafficStats.  An explicit True with an extension raises."""
    if collect_traffic is None:
        return sid <= 2
    return bool(collect_traffic)


def _run(algo: str, g, source: int, strategy, collect_traffic: Optional[bool], want_pages: bool,
         placement: str, device: int, schedule: str = "jacobi", delta: int = 0) -> TraversalResult:
    sid = strategy_id(strategy)
    if schedule != "jacobi" and collect_traffic is None:
        collect_traffic = False
    if algo != "bfs":
        _check_schedule(algo, schedule, collect_traffic)
    collect_traffic = _model_wanted(collect_traffic, sid)
    if want_pages:
        # The page streams feed the reference's LRU page-migration simulator
        # (uvm.py), which this build replaces with a real managed-memory run.
        raise NotImplementedError(
            "page streams are a simulator artefact; run with placement='uvm' for the real "
            "cudaMallocManaged comparison")
    dg = device_graph(g, placement, device)
    out, st, trav, front, hist = dg.run(algo, int(source), sid, traffic=collect_traffic,
                                        schedule=schedule, delta=delta)
    if hist is not None:
        per_iter = [TrafficStats.from_device_hist(h) for h in hist]
    else:
        per_iter = [TrafficStats.zero() for _ in range(st.iterations)]
    return TraversalResult(
        algo=algo, values=out, iterations=int(st.iterations), per_iteration_traffic=per_iter,
        traversed_edges=[int(x) for x in trav], frontier_sizes=[int(x) for x in front],
        kernel_ms=st.kernel_ms, total_ms=st.total_ms, d2h_ms=st.d2h_ms, expand_ms=st.expand_ms,
        launches=int(st.launches), h2d_bytes=int(st.h2d_bytes), d2h_bytes=int(st.d2h_bytes))


def bfs(g, source: int, strategy=AccessStrategy.MERGED_ALIGNED, *,
        collect_traffic: Optional[bool] = None, want_pages: bool = False,
        page_bytes: int = 4096, placement: str = "zerocopy", device: int = 0) -> TraversalResult:
    """Unweighted hop distances from source; unreached vertices get -1.

    One iteration per level including the final empty expansion, so
    iterations = max reached level + 1 (reference traversal.py:98-120).
    """
    _check_source(g, source)
    return _run("bfs", g, source, strategy, collect_traffic, want_pages, placement, device)


def sssp(g, source: int, strategy=AccessStrategy.MERGED_ALIGNED, *,
         collect_traffic: Optional[bool] = None, want_pages: bool = False,
         page_bytes: int = 4096, placement: str = "zerocopy", device: int = 0,
         schedule: str = "jacobi", delta: Optional[int] = None) -> TraversalResult:
    """Exact shortest distances by frontier-restricted (Jacobi) relaxation
    (reference traversal.py:123-151); unreached vertices get INT64_MAX.

    ``schedule="near-far"`` (B200 extension) expands only the improved
    vertices below a threshold that advances by ``delta`` (default 16) once
    they run out: the same distances with less work; iteration counts differ
    from the reference's.

    With 4-byte edges and weights, the merged / merged-aligned / packed
    strategies read an interleaved (dst, weight) copy of the lists, built on
    first use in the graph's placement (+8 bytes per edge of host memory;
    ``DeviceGraph.set_tuning("pairs=0")`` reads the separate arrays)."""
    _check_source(g, source)
    if not _has_weights(g):
        raise ValueError("sssp requires edge weights")
    if not isinstance(g, DeviceGraph) and g.num_edges and int(np.min(g.weights)) < 0:
        raise ValueError("sssp requires non-negative weights")
    if delta is not None and delta < 1:
        raise ValueError("delta must be >= 1")
    return _run("sssp", g, source, strategy, collect_traffic, want_pages, placement, device,
                schedule, delta or 0)


def cc(g, strategy=AccessStrategy.MERGED_ALIGNED, *, collect_traffic: Optional[bool] = None,
       want_pages: bool = False, page_bytes: int = 4096, placement: str = "zerocopy",
       device: int = 0, schedule: str = "jacobi") -> TraversalResult:
    """Connected-component labels (min vertex id) by minimum-label propagation,
    all vertices active at the start (reference traversal.py:154-179).

    ``schedule="afforest"`` (B200 extension) computes the same labels by
    union-find in at most two passes over the lists (iterations = passes;
    ``traversed_edges[k]`` = the list elements pass k read: the first window
    of every list (compressed: a sample, ``DeviceGraph.set_tuning("uf_sample=N")``),
    then the whole lists of the vertices outside the giant component)."""
    if g.directed:
        raise ValueError("connected components require an undirected graph "
                         "(load with directed=False or symmetrize first)")
    return _run("cc", g, 0, strategy, collect_traffic, want_pages, placement, device, schedule)


def _run_many(algo: str, g, sources, strategy, collect_traffic: bool, placement: str,
              device: int) -> list:
    srcs = [int(s) for s in sources]
    collect_traffic = bool(collect_traffic)
    for s in srcs:
        _check_source(g, s)
    if collect_traffic:  # the request model runs per level on the host loop
        return [_run(algo, g, s, strategy, True, False, placement, device) for s in srcs]
    dg = device_graph(g, placement, device)
    return [
        TraversalResult(
            algo=algo, values=out, iterations=int(st.iterations),
            per_iteration_traffic=[TrafficStats.zero() for _ in range(st.iterations)],
            traversed_edges=[int(x) for x in trav], frontier_sizes=[int(x) for x in front],
            kernel_ms=st.kernel_ms, total_ms=st.total_ms, d2h_ms=st.d2h_ms,
            expand_ms=st.expand_ms, launches=int(st.launches), h2d_bytes=int(st.h2d_bytes),
            d2h_bytes=int(st.d2h_bytes))
        for out, st, trav, front in dg.run_many(algo, srcs, strategy_id(strategy))]


def bfs_many(g, sources, strategy=AccessStrategy.MERGED_ALIGNED, *,
             collect_traffic: bool = False, placement: str = "zerocopy",
             device: int = 0) -> list:
    """bfs() from each source, in order -- the per-source loop of the
    reference's run_experiment (report.py:168-170) as one pipelined call: the
    int64 levels of source k download while source k+1 streams the edge list.
    Same results as calling bfs() per source."""
    return _run_many("bfs", g, sources, strategy, collect_traffic, placement, device)


def sssp_many(g, sources, strategy=AccessStrategy.MERGED_ALIGNED, *,
              collect_traffic: bool = False, placement: str = "zerocopy",
              device: int = 0) -> list:
    """sssp() from each source, pipelined like bfs_many."""
    if not _has_weights(g):
        raise ValueError("sssp requires edge weights")
    if not isinstance(g, DeviceGraph) and g.num_edges and int(np.min(g.weights)) < 0:
        raise ValueError("sssp requires non-negative weights")
    return _run_many("sssp", g, sources, strategy, collect_traffic, placement, device)


def pagerank(g, strategy=AccessStrategy.MERGED_ALIGNED, damping: float = 0.85,
             max_iters: int = 100, tol: float = 1e-6, *, collect_traffic: Optional[bool] = None,
             want_pages: bool = False, page_bytes: int = 4096, placement: str = "zerocopy",
             device: int = 0) -> TraversalResult:
    """Synchronous push PageRank over the full edge list each iteration
    (reference traversal.py:191-249): rank' = (1-d)/V + d (pushed + dangling/V),
    stop when the L1 change < tol or after max_iters, ranks normalised to 1.
    float64 ranks; the pushes are summed in 2^-62 fixed point (u64 atomics, so
    the sums and the iteration count do not depend on the order), matching the
    reference to ~1e-15 (criterion: L-inf <= 1e-8, test_acceptance.py:169-180)."""
    if not 0.0 < damping < 1.0:
        raise ValueError("damping must be in (0, 1)")
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    if tol <= 0:
        raise ValueError("tol must be positive")
    if g.num_vertices == 0:
        raise ValueError("pagerank needs at least one vertex")
    sid = strategy_id(strategy)
    collect_traffic = _model_wanted(collect_traffic, sid)
    if want_pages:
        raise NotImplementedError(
            "page streams are a simulator artefact; run with placement='uvm' for the real "
            "cudaMallocManaged comparison")
    dg = device_graph(g, placement, device)
    flags: tuple = ()
    if is_multigraph(dg):
        flags = ("multigraph",)
        warnings.warn("multigraph input: pagerank treats each duplicate edge as an edge",
                      stacklevel=2)
    out, st, hist = _pagerank_run(dg, sid, damping, max_iters, tol, collect_traffic)
    it = int(st.iterations)
    if hist is not None:
        per_iter = [TrafficStats.from_device_hist(h) for h in hist]
    else:
        per_iter = [TrafficStats.zero() for _ in range(it)]
    return TraversalResult(
        algo="pagerank", values=out, iterations=it, per_iteration_traffic=per_iter,
        traversed_edges=[int(dg.num_edges)] * it, flags=flags,
        frontier_sizes=[int(dg.num_vertices)] * it, kernel_ms=st.kernel_ms,
        total_ms=st.total_ms, d2h_ms=st.d2h_ms, expand_ms=st.expand_ms,
        launches=int(st.launches), h2d_bytes=int(st.h2d_bytes), d2h_bytes=int(st.d2h_bytes))
