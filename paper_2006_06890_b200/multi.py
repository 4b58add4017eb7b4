"""Vertex-range partitioned BFS / SSSP / CC across GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink).  Rank k owns
the global vertices [bounds[k], bounds[k+1]) -- ranges cut so every rank
holds ~E/p edges -- and keeps only their lists in its pinned host memory, so
each GPU streams its own edge slice over its own host link.  Per iteration the
rank's CUDA kernels read its frontier's lists (zero-copy) and produce a
candidate for every touched global vertex, delivered to the owners by one of:

* ``fused=True`` (no collective on the data path; CUDA-IPC peer pointers,
  NVLink between GPUs):
  - BFS, ``bfs_exchange="bitmap"`` (default): every rank marks its
    discoveries in its own global bitmap; after a barrier each owner ORs the
    ranks' words over its range and applies them (V/8 bytes read per rank);
  - BFS ``"store"`` / SSSP / CC: the expansion stores each discovery, or
    atomicMin's each candidate that improves the rank's local best, straight
    into the owner's buffer;
* ``fused=False``: a dense exchange buffer of ``nparts * stride`` slots and a
  ``reduce_scatter`` (MAX on u8 flags for BFS -- NCCL has no bitwise OR --,
  MIN on int64 distances / int32 labels).

The owner merges its candidates into its state (Jacobi: computed from
start-of-iteration values) and compacts its next frontier; an ``all_reduce``
of (frontier size, traversed edges, unvisited in-edges) decides termination
and, for direction-optimizing BFS, the step direction (bottom-up steps
all-reduce the owned frontiers' disjoint bitmaps and scan owned in-lists).

Because every step is the reference's level-synchronous / Jacobi iteration
(traversal.py:98-179), values, iteration counts and per-iteration traversed
edges (summed over ranks) are identical to the single-GPU run.

The reference has no multi-device code (PAPER.md:1051-1054 lists
multi-GPU as future work).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Protocol, Sequence

import numpy as np

from . import _native as N
from .access import strategy_id
from .csr import CsrGraph

ALGO_IDS = {"bfs": 0, "sssp": 1, "cc": 2}
# exchange element types (numpy names; torch dtypes resolved lazily)
EXCH_NP = {"bfs": np.uint8, "sssp": np.int64, "cc": np.int32}
EXCH_NONE = {"bfs": 0, "sssp": np.iinfo(np.int64).max, "cc": np.iinfo(np.int32).max}


def edge_balanced_bounds(offsets: np.ndarray, nparts: int) -> np.ndarray:
    """nparts+1 vertex boundaries cutting the CSR at ~E*k/nparts edges."""
    off = np.asarray(offsets)
    nv = off.size - 1
    ne = int(off[-1])
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    targets = (np.arange(1, nparts, dtype=np.float64) * ne / nparts).astype(np.int64)
    cuts = np.searchsorted(off, targets, side="left")
    bounds = np.concatenate(([0], np.minimum(cuts, nv), [nv])).astype(np.uint64)
    return np.maximum.accumulate(bounds)


def exchange_stride(bounds: np.ndarray) -> int:
    return max(1, int(np.max(np.diff(np.asarray(bounds, dtype=np.int64)))))


def local_part(g, bounds: np.ndarray, part: int) -> CsrGraph:
    """Part `part` of g: its vertex range, offsets rebased, global destinations."""
    lo, hi = int(bounds[part]), int(bounds[part + 1])
    off = np.asarray(g.offsets)
    e0, e1 = int(off[lo]), int(off[hi])
    loc_off = (off[lo:hi + 1] - e0).astype(np.int64)
    edges = np.asarray(g.edges)[e0:e1]
    weights = None if g.weights is None else np.asarray(g.weights)[e0:e1]
    return CsrGraph(hi - lo, e1 - e0, loc_off, edges, weights, g.edge_elem_bytes,
                    g.weight_elem_bytes, g.directed)


class Engine(Protocol):
    """One partition's traversal steps (CUDA: CudaPartition; tests: a numpy model)."""

    lo: int
    num_local: int

    def begin(self, algo: str, source: int, strategy) -> tuple[int, int]: ...
    def expand(self, exch) -> None: ...
    def apply(self, mine) -> tuple[int, int]: ...
    def result(self) -> np.ndarray: ...


class CudaPartition:
    """One vertex range of a graph on one GPU (zc_part_* of the C ABI)."""

    def __init__(self, g_local, bounds: np.ndarray, part: int, placement: str = "zerocopy",
                 device: int = 0, validate: bool = True, _handle: Optional[int] = None):
        self.bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        self.nparts = self.bounds.size - 1
        self.part = part
        self.lo = int(self.bounds[part])
        self.num_local = int(self.bounds[part + 1]) - self.lo
        self.stride = exchange_stride(self.bounds)
        self.device = device
        self.global_vertices = int(self.bounds[-1])
        self.stats = N.Stats()
        if _handle is not None:
            self._h = C.c_void_p(_handle)
            return
        from .device import _list_arg
        offsets = np.ascontiguousarray(np.asarray(g_local.offsets), dtype=np.int64)
        edges, eb_src = _list_arg(g_local.edges)
        weights, wb_src = (None, 8) if g_local.weights is None else _list_arg(g_local.weights)
        d = N.GraphDesc()
        d.num_vertices, d.num_edges = g_local.num_vertices, g_local.num_edges
        d.offsets = offsets.ctypes.data
        d.edges = edges.ctypes.data if edges.size else None
        d.weights = None if weights is None else (weights.ctypes.data or None)
        d.src_edge_bytes, d.src_weight_bytes = eb_src, wb_src
        d.edge_elem_bytes, d.weight_elem_bytes = g_local.edge_elem_bytes, g_local.weight_elem_bytes
        d.placement, d.device = N.PLACEMENTS[placement], device
        d.flags = ((N.ZC_F_DIRECTED if g_local.directed else 0)
                   | (0 if validate else N.ZC_F_NO_VALIDATE))
        info = N.PartInfo()
        info.global_vertices = self.global_vertices
        info.stride = self.stride
        info.bounds = self.bounds.ctypes.data
        info.nparts, info.part = self.nparts, part
        h = C.c_void_p()
        N.check(N.lib().zc_part_create(C.byref(d), C.byref(info), C.byref(h)))
        self._h = h

    def close(self):
        if self._h is not None and self._h.value:
            N.lib().zc_graph_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def begin(self, algo: str, source: int, strategy) -> tuple[int, int]:
        n, t = C.c_uint64(), C.c_uint64()
        N.check(N.lib().zc_part_begin(self._h, ALGO_IDS[algo], int(source), strategy_id(strategy),
                                      C.byref(n), C.byref(t)))
        return n.value, t.value

    def expand(self, exch) -> None:
        N.check(N.lib().zc_part_expand(self._h, exch.data_ptr()))

    def apply(self, mine) -> tuple[int, int]:
        n, t = C.c_uint64(), C.c_uint64()
        N.check(N.lib().zc_part_apply(self._h, mine.data_ptr(), C.byref(n), C.byref(t)))
        return n.value, t.value

    # -- direction-optimizing bfs: bottom-up steps against the global frontier bitmap
    @property
    def bitmap_words(self) -> int:
        return (int(self.bounds[-1]) + 31) // 32 + 1

    def unvisited_in(self) -> int:
        x = C.c_uint64()
        N.check(N.lib().zc_part_unvisited_in(self._h, C.byref(x)))
        return x.value

    def frontier_bits(self, bits) -> None:
        """Zero `bits` (device, bitmap_words int32) and set the owned frontier's bits."""
        N.check(N.lib().zc_part_frontier_bits(self._h, bits.data_ptr()))

    def pull(self, bits) -> tuple[int, int]:
        n, t = C.c_uint64(), C.c_uint64()
        N.check(N.lib().zc_part_pull(self._h, bits.data_ptr(), C.byref(n), C.byref(t)))
        return n.value, t.value

    def graph_view(self):
        """DeviceGraph-style host views (offsets, edges, weights) of this part."""
        from .device import DeviceGraph
        dg = DeviceGraph.__new__(DeviceGraph)
        dg._h = self._h
        nv, ne = C.c_uint64(), C.c_uint64()
        eb, wb, pl, fl = C.c_uint32(), C.c_uint32(), C.c_int32(), C.c_uint32()
        N.check(N.lib().zc_graph_info(self._h, C.byref(nv), C.byref(ne), C.byref(eb), C.byref(wb),
                                      C.byref(pl), C.byref(fl)))
        dg.num_vertices, dg.num_edges = nv.value, ne.value
        dg.edge_elem_bytes, dg.weight_elem_bytes = eb.value, wb.value or 4
        dg.has_weights = wb.value != 0
        dg.directed = bool(fl.value & N.ZC_F_DIRECTED)
        off, edges, weights = DeviceGraph.host_arrays(dg)
        dg._h = None  # the view does not own the handle
        return CsrGraph(dg.num_vertices, dg.num_edges, off, edges, weights, dg.edge_elem_bytes,
                        dg.weight_elem_bytes, dg.directed)

    # -- fused exchange (candidates written straight into the owners' buffers)
    def fused_init(self, algo: str) -> tuple[bytes, int]:
        handle = (C.c_char * 64)()
        local = C.c_void_p()
        N.check(N.lib().zc_part_fused_init(self._h, ALGO_IDS[algo], handle, C.byref(local)))
        return bytes(handle), local.value

    def fused_connect(self, handles: Optional[Sequence[bytes]] = None,
                      ptrs: Optional[Sequence[int]] = None) -> None:
        if ptrs is not None:
            arr = (C.c_void_p * len(ptrs))(*ptrs)
            N.check(N.lib().zc_part_fused_connect(self._h, None, arr))
        else:
            blob = b"".join(handles)
            N.check(N.lib().zc_part_fused_connect(self._h, blob, None))

    def fused_reset(self) -> None:
        N.check(N.lib().zc_part_fused_reset(self._h))

    def fused_expand(self) -> None:
        N.check(N.lib().zc_part_fused_expand(self._h))

    # -- BFS bitmap exchange (each owner ORs the ranks' discovery bitmaps)
    def bitmap_init(self) -> tuple[bytes, int]:
        """(IPC handle, device address) of this part's discovery bitmap."""
        handle = (C.c_char * 64)()
        local = C.c_void_p()
        N.check(N.lib().zc_part_bitmap_init(self._h, handle, C.byref(local)))
        return bytes(handle), local.value

    def bitmap_connect(self, handles: Optional[Sequence[bytes]] = None,
                       ptrs: Optional[Sequence[int]] = None) -> None:
        if ptrs is not None:
            arr = (C.c_void_p * len(ptrs))(*ptrs)
            N.check(N.lib().zc_part_bitmap_connect(self._h, None, arr))
        else:
            N.check(N.lib().zc_part_bitmap_connect(self._h, b"".join(handles), None))

    def bitmap_expand(self) -> None:
        N.check(N.lib().zc_part_bitmap_expand(self._h))

    def bitmap_apply(self) -> tuple[int, int]:
        n, t = C.c_uint64(), C.c_uint64()
        N.check(N.lib().zc_part_bitmap_apply(self._h, C.byref(n), C.byref(t)))
        return n.value, t.value

    def apply_ptr(self, ptr: int) -> tuple[int, int]:
        n, t = C.c_uint64(), C.c_uint64()
        N.check(N.lib().zc_part_apply(self._h, ptr, C.byref(n), C.byref(t)))
        return n.value, t.value

    def build_stores(self) -> None:
        """The compressed out-lists and the owned vertices' in-lists the
        direction-optimizing strategy reads (built on first use otherwise)."""
        nb = C.c_uint64()
        N.check(N.lib().zc_graph_build_compressed(self._h, C.byref(nb)))
        N.check(N.lib().zc_part_build_in_lists(self._h, C.byref(nb)))

    def launches(self) -> int:
        """Kernels launched since the last begin (this rank)."""
        return self.run_stats()["launches"]

    def run_stats(self) -> dict:
        """This rank's counters since the last begin: kernel launches, the
        expansion kernels' device time, and the exchange bytes it sent
        (reduce-scatter share, or fused remote sends)."""
        N.check(N.lib().zc_part_result(self._h, None, C.byref(self.stats)))
        return {"launches": int(self.stats.launches), "expand_ms": float(self.stats.expand_ms),
                "exchange_bytes": int(self.stats.exchange_bytes)}

    def result(self) -> np.ndarray:
        from .device import pinned_empty
        out = pinned_empty(self.num_local, np.int64)
        N.check(N.lib().zc_part_result(self._h, out.ctypes.data, C.byref(self.stats)))
        return out


def generate_rmat_part(scale: int, nparts: int, part: int, edge_factor: int = 16,
                       a: float = 0.57, b: float = 0.19, c: float = 0.19, seed: int = 27, *,
                       symmetrize: bool = False, weights=None, placement: str = "zerocopy",
                       device: int = 0) -> CudaPartition:
    """This rank's edge-balanced part of generate_rmat(scale, ..., symmetrize)
    (same arcs, same sorted lists when symmetrized), generated on the GPU
    straight into a partition handle: every rank enumerates the counter-based
    arcs itself, so no edges move between ranks."""
    if symmetrize and weights is not None:
        raise ValueError("symmetrized partitions carry no weights")
    lo, hi = weights if weights is not None else (1, 0)
    bounds = np.zeros(nparts + 1, np.uint64)
    h = C.c_void_p()
    N.check(N.lib().zc_generate_rmat_part(scale, edge_factor, a, b, c, seed, int(bool(symmetrize)),
                                          lo, hi, nparts, part, N.PLACEMENTS[placement], device,
                                          bounds.ctypes.data, C.byref(h)))
    return CudaPartition(None, bounds, part, placement, device, _handle=h.value)


@dataclass
class PartResult:
    """This rank's share of a partitioned traversal."""

    algo: str
    lo: int
    values: np.ndarray          # int64 values of the owned range
    iterations: int             # global (same on every rank)
    traversed_edges: list       # global, summed over ranks
    frontier_sizes: list = field(default_factory=list)  # global
    local_traversed: int = 0    # edges this rank streamed over its own host link
    expand_ms: float = 0.0      # this rank's expansion kernels (device time)
    exchange_bytes: int = 0     # bytes this rank sent: candidates + frontier bitmaps
    bottom_up_steps: int = 0

    @property
    def total_traversed_edges(self) -> int:
        return sum(self.traversed_edges)


def _torch_dtype(algo: str):
    import torch
    return {"bfs": torch.uint8, "sssp": torch.int64, "cc": torch.int32}[algo]


def run_partition(engine: Engine, algo: str, source: int, strategy, *, group=None,
                  tensor_device=None, stage_host: bool = False, fetch: bool = True,
                  buffers=None, fused: bool = False, bfs_exchange: str = "bitmap"
                  ) -> PartResult:
    """SPMD driver: call on every rank of `group` with that rank's engine.

    stage_host: run the collectives on host copies of the exchange buffers
    (gloo; lets several ranks share one GPU in tests).  fetch=False skips the
    download of the owned values (timing of the traversal loop alone).
    buffers: reusable (exch, mine) tensors from exchange_buffers().
    fused: no collective on the data path -- BFS: each owner ORs the ranks'
    discovery bitmaps over its range through peer memory (bfs_exchange
    "bitmap") or the expansion stores each discovery into its owner's buffer
    ("store"); SSSP / CC: remote atomicMin of each locally improved candidate.
    """
    import torch
    import torch.distributed as dist

    if algo not in ALGO_IDS:
        raise ValueError(f"unknown algorithm {algo!r}")
    if bfs_exchange not in ("bitmap", "store"):
        raise ValueError("bfs_exchange must be 'bitmap' or 'store'")
    if fused:
        return _run_partition_fused(engine, algo, source, strategy, group, fetch,
                                    algo == "bfs" and bfs_exchange == "bitmap")
    nparts = dist.get_world_size(group)
    stride = engine.stride
    dev = tensor_device if tensor_device is not None else torch.device("cuda", engine.device)
    if buffers is None:
        buffers = exchange_buffers(algo, nparts, stride, dev)
    exch, mine = buffers
    if stage_host:
        h_exch, h_mine = exch.cpu(), mine.cpu()
    op = dist.ReduceOp.MAX if algo == "bfs" else dist.ReduceOp.MIN
    cdev = torch.device("cpu") if stage_host else dev
    counts = torch.zeros(3, dtype=torch.int64, device=cdev)
    dobfs = is_direction_optimizing(strategy)

    local = [0, 0, 0]  # edges streamed by this rank, bitmap all-reduce bytes, bottom-up steps

    def global_counts(n: int, t: int) -> tuple[int, int, int]:
        local[0] += t
        counts[0], counts[1] = n, t
        counts[2] = engine.unvisited_in() if dobfs else 0
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
        return int(counts[0]), int(counts[1]), int(counts[2])

    def pull_step():
        # the owned frontiers' disjoint bits, OR-ed by a SUM all-reduce
        local[1] += allreduce_send_bytes(engine.bitmap_words * 4, nparts)
        local[2] += 1
        bits = torch.empty(engine.bitmap_words, dtype=torch.int32, device=dev)
        engine.frontier_bits(bits)
        if stage_host:
            hb = bits.cpu()
            dist.all_reduce(hb, op=dist.ReduceOp.SUM, group=group)
            bits.copy_(hb)
        else:
            dist.all_reduce(bits, op=dist.ReduceOp.SUM, group=group)
        if dev.type == "cuda":
            torch.cuda.current_stream(dev).synchronize()
        return engine.pull(bits)

    n, t, m = global_counts(*engine.begin(algo, source, strategy))
    iters, trav, front = 0, [], []
    while n > 0:
        iters += 1
        trav.append(t)
        front.append(n)
        if dobfs and pull_now(iters, t, m):
            n, t, m = global_counts(*pull_step())
            continue
        engine.expand(exch)                      # device work done when this returns
        if stage_host:
            h_exch.copy_(exch)
            dist.reduce_scatter_tensor(h_mine, h_exch, op=op, group=group)
            mine.copy_(h_mine)
        else:
            dist.reduce_scatter_tensor(mine, exch, op=op, group=group)
        if dev.type == "cuda":
            torch.cuda.current_stream(dev).synchronize()
        n, t, m = global_counts(*engine.apply(mine))
    values = engine.result() if fetch else None
    return _finish(PartResult(algo, engine.lo, values, iters, trav, front), engine, local)


def allreduce_send_bytes(nbytes: int, nparts: int) -> int:
    """Bytes one rank sends in a ring all-reduce of nbytes."""
    return 2 * (nparts - 1) * nbytes // max(nparts, 1)


def _finish(res: PartResult, engine, local) -> PartResult:
    """Attach this rank's counters: traversed edges of the frontiers it owned
    (the reference's work units), expansion time, exchange bytes sent."""
    res.local_traversed = local[0]
    stats = engine.run_stats() if hasattr(engine, "run_stats") else {}
    res.expand_ms = stats.get("expand_ms", 0.0)
    res.exchange_bytes = stats.get("exchange_bytes", 0) + local[1]
    res.bottom_up_steps = local[2]
    return res


def is_direction_optimizing(strategy) -> bool:
    return strategy_id(strategy) == 5


DO_ALPHA = 2.0  # the direction switch factor, zc_graph::Tuning::do_alpha's default


def pull_now(iteration: int, frontier_out_edges: int, unvisited_in_edges: int,
             alpha: float = DO_ALPHA) -> bool:
    """Bottom-up when the frontier's out-edges exceed the unvisited vertices'
    in-edges / alpha (never the source's own expansion) -- zc_api.cu's rule."""
    return iteration > 1 and frontier_out_edges * alpha > unvisited_in_edges


def _run_partition_fused(engine, algo, source, strategy, group, fetch, bitmap) -> PartResult:
    """Fused exchange over peer memory (CUDA IPC pointers; NVLink between
    GPUs).  bitmap (BFS): every rank marks discoveries in its own global
    bitmap, each owner ORs the ranks' words over its range -- one barrier and
    the counts all-reduce per level.  Otherwise the expand kernel stores /
    atomicMin's each candidate into its owner's buffer; two barriers per
    level replace the reduce-scatter."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", engine.device)
    key = "bitmap" if bitmap else algo
    if getattr(engine, "_fused_for", None) == key:  # peers opened by an earlier run
        mine = engine._fused_mine
    else:  # once per (engine, mode): export, exchange and open the IPC handles
        handle, mine = engine.bitmap_init() if bitmap else engine.fused_init(algo)
        connect = engine.bitmap_connect if bitmap else engine.fused_connect
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, handle, group=group)
        err = None
        try:
            connect(handles=handles)
        except RuntimeError as exc:  # e.g. no peer access between these GPUs
            err = exc
        # every rank learns whether all peers opened, so none waits on a dead exchange
        status = [None] * dist.get_world_size(group)
        dist.all_gather_object(status, None if err is None else str(err), group=group)
        failed = [m for m in status if m is not None]
        if failed:
            raise RuntimeError(f"fused exchange unavailable: {failed[0]}")
        engine._fused_for, engine._fused_mine = key, mine
    cdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else dev
    counts = torch.zeros(2, dtype=torch.int64, device=cdev)

    def sync_all():
        counts.zero_()
        dist.all_reduce(counts, group=group)  # doubles as a barrier
        if cdev.type == "cuda":
            torch.cuda.current_stream(dev).synchronize()

    dobfs = is_direction_optimizing(strategy)
    counts3 = torch.zeros(3, dtype=torch.int64, device=cdev)
    nparts = dist.get_world_size(group)
    local = [0, 0, 0]

    def global_counts3(n: int, t: int) -> tuple[int, int, int]:
        local[0] += t
        counts3[0], counts3[1] = n, t
        counts3[2] = engine.unvisited_in() if dobfs else 0
        dist.all_reduce(counts3, op=dist.ReduceOp.SUM, group=group)
        return int(counts3[0]), int(counts3[1]), int(counts3[2])

    n, t, m = global_counts3(*engine.begin(algo, source, strategy))
    iters, trav, front = 0, [], []
    while n > 0:
        iters += 1
        trav.append(t)
        front.append(n)
        if dobfs and pull_now(iters, t, m):
            local[1] += allreduce_send_bytes(engine.bitmap_words * 4, nparts)
            local[2] += 1
            bits = torch.empty(engine.bitmap_words, dtype=torch.int32, device=dev)
            engine.frontier_bits(bits)
            hb = bits.cpu() if cdev.type == "cpu" else bits
            dist.all_reduce(hb, op=dist.ReduceOp.SUM, group=group)
            if cdev.type == "cpu":
                bits.copy_(hb)
            torch.cuda.current_stream(dev).synchronize()
            n, t, m = global_counts3(*engine.pull(bits))
            continue
        if bitmap:
            engine.bitmap_expand()  # own bitmap zeroed, then this rank's discoveries
            sync_all()              # every rank's bitmap complete
            # the counts all-reduce is the barrier before the bitmaps are reused
            n, t, m = global_counts3(*engine.bitmap_apply())
            continue
        engine.fused_reset()
        sync_all()              # every owner buffer reset before anyone writes
        engine.fused_expand()   # kernel done (its peer stores performed) on return
        sync_all()              # every rank's candidates delivered
        n, t, m = global_counts3(*engine.apply_ptr(mine))
    values = engine.result() if fetch else None
    return _finish(PartResult(algo, engine.lo, values, iters, trav, front), engine, local)


def exchange_buffers(algo: str, nparts: int, stride: int, device):
    """(exchange, owned-slice) tensors for run_partition."""
    import torch
    dt = _torch_dtype(algo)
    return (torch.empty(nparts * stride, dtype=dt, device=device),
            torch.empty(stride, dtype=dt, device=device))


def run_partitions_local(engines: Sequence[Engine], algo: str, source: int, strategy,
                         fused: bool = False, bfs_exchange: str = "bitmap"
                         ) -> tuple[np.ndarray, int, list]:
    """All partitions in one process (one device): the reduce-scatter becomes a
    host-driven reduction over the stacked exchange buffers (or, fused, the
    expand kernels write into each other's buffers by device pointer).  Used to
    validate the partitioned kernels on a single GPU."""
    import torch

    dobfs = is_direction_optimizing(strategy)

    def unvisited_in() -> int:
        return sum(e.unvisited_in() for e in engines) if dobfs else 0

    def pull_all() -> tuple[int, int]:
        """Bottom-up step of every partition against the OR of their frontiers."""
        dev = torch.device("cuda", engines[0].device)
        parts = []
        for e in engines:
            b = torch.empty(e.bitmap_words, dtype=torch.int32, device=dev)
            e.frontier_bits(b)
            parts.append(b)
        bits = parts[0]
        for b in parts[1:]:
            bits = torch.bitwise_or(bits, b)
        torch.cuda.synchronize(dev)
        nt = [e.pull(bits) for e in engines]
        return sum(x[0] for x in nt), sum(x[1] for x in nt)

    if fused and algo == "bfs" and bfs_exchange == "bitmap":
        ptrs = [e.bitmap_init()[1] for e in engines]
        for e in engines:
            e.bitmap_connect(ptrs=ptrs)
        nt = [e.begin(algo, source, strategy) for e in engines]
        n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
        iters, trav = 0, []
        while n > 0:
            iters += 1
            trav.append(t)
            if dobfs and pull_now(iters, t, unvisited_in()):
                n, t = pull_all()
                continue
            for e in engines:
                e.bitmap_expand()
            nt = [e.bitmap_apply() for e in engines]
            n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
        values = np.concatenate([e.result() for e in engines])
        return values, iters, trav
    if fused:
        locals_ = [e.fused_init(algo)[1] for e in engines]
        for e in engines:
            e.fused_connect(ptrs=locals_)
        nt = [e.begin(algo, source, strategy) for e in engines]
        n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
        iters, trav = 0, []
        while n > 0:
            iters += 1
            trav.append(t)
            if dobfs and pull_now(iters, t, unvisited_in()):
                n, t = pull_all()
                continue
            for e in engines:
                e.fused_reset()
            for e in engines:
                e.fused_expand()
            nt = [e.apply_ptr(p) for e, p in zip(engines, locals_)]
            n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
        values = np.concatenate([e.result() for e in engines])
        return values, iters, trav

    p = len(engines)
    stride = engines[0].stride
    dev = torch.device("cuda", engines[0].device)
    dt = _torch_dtype(algo)
    bufs = [torch.empty(p * stride, dtype=dt, device=dev) for _ in range(p)]
    nt = [e.begin(algo, source, strategy) for e in engines]
    n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
    iters, trav = 0, []
    while n > 0:
        iters += 1
        trav.append(t)
        if dobfs and pull_now(iters, t, unvisited_in()):
            n, t = pull_all()
            continue
        for e, b in zip(engines, bufs):
            e.expand(b)
        st = torch.stack(bufs)
        red = st.max(dim=0).values if algo == "bfs" else st.min(dim=0).values
        slices = [red[k * stride:(k + 1) * stride].contiguous() for k in range(p)]
        torch.cuda.synchronize(dev)
        nt = [e.apply(sl) for e, sl in zip(engines, slices)]
        n, t = sum(x[0] for x in nt), sum(x[1] for x in nt)
    values = np.concatenate([e.result() for e in engines]) if engines else np.zeros(0, np.int64)
    return values, iters, trav
