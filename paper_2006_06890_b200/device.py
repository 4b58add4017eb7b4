"""Device-resident graph handles (the B200 host graph store).

``DeviceGraph`` owns one ``zc_graph`` handle of the C ABI: the edge / weight
lists live in pinned mapped host memory (``placement="zerocopy"``, EMOGI),
in host-resident managed memory read in place (``"zerocopy-managed"``, the
same zero-copy loads through the UVM driver's large-page GPU mappings),
in managed memory with read-mostly advice (``"uvm"``, the paper's baseline,
PAPER.md:593) or in HBM (``"hbm"``, control run); offsets and all per-vertex
state live in HBM.  Building a handle pins and copies the lists once;
:func:`device_graph` caches it per (graph object, placement, device) so the
reference-style ``bfs(g, ...)`` calls reuse it (CsrGraph is immutable by
convention, reference csr.py:36).

The native generators build handles directly on the GPU
(:func:`generate_rmat`, :func:`generate_uniform_device`).
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref
from typing import Optional

import numpy as np

from . import _native as N
from .csr import CsrGraph


# ------------------------------------------------------------ pinned results
class _PinnedPool:
    """Recycles pinned host buffers of result arrays (D2H at link speed
    without paying cudaHostAlloc on every call)."""

    def __init__(self, cap_bytes: int = 16 << 30):
        self.free: dict[int, list[int]] = {}
        self.pooled = 0
        self.cap = cap_bytes
        self.lock = threading.Lock()

    def get(self, nbytes: int) -> int:
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                self.pooled -= nbytes
                return lst.pop()
        ptr = N.lib().zc_host_alloc(max(nbytes, 8))
        if not ptr:
            raise MemoryError(N.last_error())
        return ptr

    def put(self, nbytes: int, ptr: int) -> None:
        with self.lock:
            if self.pooled + nbytes <= self.cap:
                self.free.setdefault(nbytes, []).append(ptr)
                self.pooled += nbytes
                return
        N.lib().zc_host_free(ptr)


_POOL = _PinnedPool()


class _PinnedArrayOwner:
    """numpy base object of a pinned array; returns the buffer to the pool."""

    def __init__(self, count: int, dtype):
        dt = np.dtype(dtype)
        self.nbytes = count * dt.itemsize
        self.ptr = _POOL.get(self.nbytes)
        self.__array_interface__ = {"shape": (count,), "typestr": dt.str,
                                    "data": (self.ptr, False), "version": 3}

    def __del__(self):
        try:
            _POOL.put(self.nbytes, self.ptr)
        except Exception:  # interpreter shutdown
            pass


def pinned_empty(count: int, dtype=np.int64) -> np.ndarray:
    """Uninitialised numpy array in pinned (page-locked) host memory."""
    return np.asarray(_PinnedArrayOwner(count, dtype))


# --------------------------------------------------------------- the handle
def _list_arg(arr) -> tuple[np.ndarray, int]:
    """Contiguous array with 4- or 8-byte integer elements + its width."""
    a = np.asarray(arr)
    if a.dtype.kind not in "iu":
        a = a.astype(np.int64)
    if a.dtype.itemsize not in (4, 8):
        a = a.astype(np.int64)
    return np.ascontiguousarray(a), a.dtype.itemsize


class DeviceGraph:
    """A CSR graph resident for traversal on one GPU."""

    def __init__(self, g=None, placement: str = "zerocopy", device: int = 0, *,
                 register: bool = False, uvm_prefetch: bool = False, validate: bool = True,
                 _handle: Optional[int] = None):
        if placement not in N.PLACEMENTS:
            raise ValueError(f"placement must be one of {sorted(N.PLACEMENTS)}")
        self.placement = placement
        self.device = device
        self._h = None
        self._keep = None
        self._lock = threading.Lock()
        lib = N.lib()
        if _handle is not None:
            self._h = C.c_void_p(_handle)
        else:
            offsets = np.ascontiguousarray(np.asarray(g.offsets), dtype=np.int64)
            edges, eb_src = _list_arg(g.edges)
            weights, wb_src = (None, 8) if g.weights is None else _list_arg(g.weights)
            d = N.GraphDesc()
            d.num_vertices, d.num_edges = g.num_vertices, g.num_edges
            d.offsets = offsets.ctypes.data
            d.edges = edges.ctypes.data if edges.size else None
            d.weights = None if weights is None else (weights.ctypes.data or None)
            d.src_edge_bytes, d.src_weight_bytes = eb_src, wb_src
            d.edge_elem_bytes, d.weight_elem_bytes = g.edge_elem_bytes, g.weight_elem_bytes
            d.placement, d.device = N.PLACEMENTS[placement], device
            d.flags = ((N.ZC_F_DIRECTED if g.directed else 0)
                       | (N.ZC_F_REGISTER if register else 0)
                       | (N.ZC_F_UVM_PREFETCH if uvm_prefetch else 0)
                       | (0 if validate else N.ZC_F_NO_VALIDATE))
            h = C.c_void_p()
            N.check(lib.zc_graph_create(C.byref(d), C.byref(h)))
            self._h = h
            if register:  # the registered caller buffers must outlive the handle
                self._keep = (edges, weights)
        nv, ne = C.c_uint64(), C.c_uint64()
        eb, wb, pl, fl = C.c_uint32(), C.c_uint32(), C.c_int32(), C.c_uint32()
        N.check(lib.zc_graph_info(self._h, C.byref(nv), C.byref(ne), C.byref(eb), C.byref(wb),
                                  C.byref(pl), C.byref(fl)))
        self.num_vertices, self.num_edges = nv.value, ne.value
        self.edge_elem_bytes = eb.value
        self.weight_elem_bytes = wb.value or 4
        self.has_weights = wb.value != 0
        self.directed = bool(fl.value & N.ZC_F_DIRECTED)
        self._options = 0

    # -- lifecycle
    def close(self) -> None:
        if self._h is not None and self._h.value:
            N.lib().zc_graph_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise RuntimeError("DeviceGraph is closed")
        return self._h

    # -- host views of the handle's own memory (valid while the handle lives)
    def host_arrays(self):
        e, w, o = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(N.lib().zc_graph_host_lists(self.handle, C.byref(e), C.byref(w), C.byref(o)))
        nv, ne = self.num_vertices, self.num_edges
        off = np.ctypeslib.as_array((C.c_int64 * (nv + 1)).from_address(o.value))
        et = C.c_uint32 if self.edge_elem_bytes == 4 else C.c_uint64
        edges = (np.ctypeslib.as_array((et * ne).from_address(e.value)) if ne
                 else np.zeros(0, np.uint32))
        weights = None
        if self.has_weights:
            wt = C.c_uint32 if self.weight_elem_bytes == 4 else C.c_uint64
            weights = (np.ctypeslib.as_array((wt * ne).from_address(w.value)) if ne
                       else np.zeros(0, np.uint32))
        return off, edges, weights

    def as_csr(self) -> CsrGraph:
        """CsrGraph whose arrays are views of this handle's host memory."""
        off, edges, weights = self.host_arrays()
        g = CsrGraph(self.num_vertices, self.num_edges, off, edges, weights,
                     self.edge_elem_bytes, self.weight_elem_bytes, self.directed)
        g._device_graph_owner = self  # keep the memory alive with the view
        return g

    def evict(self) -> None:
        """UVM: move the lists back to host memory so the next run is cold."""
        N.check(N.lib().zc_graph_evict(self.handle))

    def prefetch(self) -> float:
        """UVM: migrate the lists to the GPU now (cudaMemPrefetchAsync; the
        paper's UVM-with-prefetch comparison, after evict() for a cold
        start).  Returns the migration's device time in ms (0 otherwise)."""
        ms = C.c_float(0)
        N.check(N.lib().zc_graph_prefetch(self.handle, C.byref(ms)))
        return float(ms.value)

    def build_sssp_pairs(self) -> None:
        """Interleave (dst, weight) into one 8-byte stream for SSSP (extra
        8 B/edge of host memory); results are identical."""
        N.check(N.lib().zc_graph_build_pairs(self.handle))

    def build_compressed(self) -> int:
        """Build the line-compressed list stream (strategy "compressed");
        returns its size in bytes."""
        nbytes = C.c_uint64()
        N.check(N.lib().zc_graph_build_compressed(self.handle, C.byref(nbytes)))
        return nbytes.value

    def compressed_index(self) -> np.ndarray:
        """Every vertex's entry of the compressed line stream's index (V+1
        u64): bits [0, 40) the list's bit position; bit 63 set: a long list
        stored as whole lines, their count in bits [40, 63)."""
        out = np.empty(self.num_vertices + 1, np.uint64)
        N.check(N.lib().zc_graph_compressed_index(self.handle, out.ctypes.data))
        return out

    def stored_list_bytes(self, strategy: str = "compressed") -> np.ndarray:
        """Bytes each vertex's list occupies in the stream a strategy reads:
        edge width x degree for the raw lists (+ weight width x degree when
        `weights`), the list's span of the compressed line stream (its lines,
        or its share of a shared line including padding) for "compressed"."""
        if strategy != "compressed":
            return np.diff(self.as_csr().offsets).astype(np.int64) * self.edge_elem_bytes
        idx = self.compressed_index()
        pos = (idx & np.uint64((1 << 40) - 1)).astype(np.int64)
        lines = ((idx[:-1] & np.uint64((1 << 63) - 1)) >> np.uint64(40)).astype(np.int64)
        long_ = (idx[:-1] >> np.uint64(63)).astype(bool)
        return np.where(long_, lines * 128, np.diff(pos) // 8)

    def build_in_lists(self) -> int:
        """Build the compressed in-list stream (the transpose; an undirected
        graph reuses its out-lists) used by "direction-optimizing"; returns
        its size in bytes."""
        nbytes = C.c_uint64()
        N.check(N.lib().zc_graph_build_in_lists(self.handle, C.byref(nbytes)))
        return nbytes.value

    def build_log(self) -> list:
        """[(phase, wall ms)] of this handle's one-time builds (compressed out /
        in-list streams), in order (zc_graph_build_log); "…[gpu]" entries are
        the GPU time inside the phase before them, not phases of their own."""
        need = N.lib().zc_graph_build_log(self.handle, None, 0)
        if need < 0:
            N.check(need)
        buf = C.create_string_buffer(max(need, 1))
        N.lib().zc_graph_build_log(self.handle, buf, len(buf))
        return [(ln.split()[0], float(ln.split()[1]))
                for ln in buf.value.decode().splitlines() if ln.strip()]

    def link_bytes_requested(self) -> int:
        """Line-stream bytes the last compressed / direction-optimizing run's
        expansion kernels requested over the link (0 for other strategies)."""
        out = C.c_uint64()
        N.check(N.lib().zc_run_link_bytes(self.handle, C.byref(out)))
        return out.value

    def directions(self, iterations: int) -> np.ndarray:
        """Per-iteration direction of the last "direction-optimizing" run
        (True = bottom-up step)."""
        out = np.zeros(iterations, np.uint8)
        N.check(N.lib().zc_run_directions(self.handle, out.ctypes.data, iterations))
        return out.astype(bool)

    def expand_profile(self, iterations: int) -> np.ndarray:
        """Per-iteration device time (ms) of the expansion kernels of the last run."""
        out = np.zeros(iterations, np.float64)
        N.check(N.lib().zc_run_profile(self.handle, out.ctypes.data, iterations))
        return out

    # -- run plumbing
    def set_tuning(self, spec: str = "") -> None:
        """Launch tuning of this handle (zc_set_tuning): comma-separated
        unroll=2|4|8|16, ctas=N, sched=chunk|sweep, loop=host|device,
        do_alpha=X, ld=0..4, pairs=0|1, carveout=0..100, widen=1..256,
        uf_sample=1..1024; "" restores the defaults."""
        N.check(N.lib().zc_set_tuning(self.handle, spec.encode()))

    def set_traffic_model(self, on: bool) -> None:
        opt = N.ZC_OPT_TRAFFIC_MODEL if on else 0
        if opt != self._options:
            N.check(N.lib().zc_set_options(self.handle, opt))
            self._options = opt

    def run(self, algo: str, source: int, strategy_id: int, traffic: bool = False,
            schedule: str = "jacobi", delta: int = 0):
        """Run one traversal; returns (values int64[V] pinned, Stats, traversed, frontier, hist)."""
        lib = N.lib()
        with self._lock:
            self.set_traffic_model(traffic)
            out = pinned_empty(self.num_vertices, np.int64)
            st = N.Stats()
            ptr = out.ctypes.data
            if algo == "bfs":
                rc = lib.zc_bfs(self.handle, source, strategy_id, ptr, C.byref(st))
            elif algo == "sssp" and schedule == "near-far":
                rc = lib.zc_sssp_nearfar(self.handle, source, strategy_id, int(delta), ptr,
                                         C.byref(st))
            elif algo == "sssp":
                rc = lib.zc_sssp(self.handle, source, strategy_id, ptr, C.byref(st))
            elif algo == "cc" and schedule == "afforest":
                rc = lib.zc_cc_afforest(self.handle, strategy_id, ptr, C.byref(st))
            elif algo == "cc":
                rc = lib.zc_cc(self.handle, strategy_id, ptr, C.byref(st))
            else:
                raise ValueError(f"unknown algorithm {algo!r}")
            N.check(rc)
            it = st.iterations
            trav = np.zeros(it, np.uint64)
            front = np.zeros(it, np.uint64)
            N.check(lib.zc_run_log(self.handle, trav.ctypes.data, front.ctypes.data, it))
            hist = None
            if traffic:
                hist = np.zeros((it, 8), np.uint64)
                N.check(lib.zc_run_traffic(self.handle, hist.ctypes.data, it))
        return out, st, trav, front, hist


    def run_many(self, algo: str, sources, strategy_id: int):
        """Traverse from each source with the result downloads pipelined behind
        the next traversal (zc_bfs_async / zc_sssp_async + zc_sync); returns a
        list of (values, Stats, traversed, frontier)."""
        lib = N.lib()
        fn = {"bfs": lib.zc_bfs_async, "sssp": lib.zc_sssp_async}.get(algo)
        if fn is None:
            raise ValueError(f"no pipelined runner for {algo!r}")
        done = []
        with self._lock:
            self.set_traffic_model(False)
            try:
                for s in sources:
                    out = pinned_empty(self.num_vertices, np.int64)
                    st = N.Stats()
                    N.check(fn(self.handle, int(s), strategy_id, out.ctypes.data, C.byref(st)))
                    # `out` is still being written: keep it referenced until zc_sync
                    done.append((out, st))
                    it = st.iterations
                    trav = np.zeros(it, np.uint64)
                    front = np.zeros(it, np.uint64)
                    N.check(lib.zc_run_log(self.handle, trav.ctypes.data, front.ctypes.data, it))
                    done[-1] = (out, st, trav, front)
            finally:
                N.check(lib.zc_sync(self.handle))
        return done


# id(graph) -> (weakref to graph, {key: DeviceGraph}); CsrGraph defines __eq__
# without __hash__ (like the reference), so it cannot key a WeakKeyDictionary.
def _pagerank_run(dg: "DeviceGraph", sid: int, damping: float, max_iters: int, tol: float,
                  traffic: bool):
    lib = N.lib()
    with dg._lock:
        dg.set_traffic_model(traffic)
        out = pinned_empty(dg.num_vertices, np.float64)
        st = N.Stats()
        N.check(lib.zc_pagerank(dg.handle, sid, float(damping), int(max_iters), float(tol),
                                out.ctypes.data, C.byref(st)))
        it = st.iterations
        hist = None
        if traffic:
            hist = np.zeros((it, 8), np.uint64)
            N.check(lib.zc_run_traffic(dg.handle, hist.ctypes.data, it))
    return out, st, hist


def is_multigraph(dg: "DeviceGraph") -> bool:
    flag = C.c_int()
    N.check(N.lib().zc_graph_multigraph(dg.handle, C.byref(flag)))
    return bool(flag.value)


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()
HANDLES_PER_GRAPH = 2


def _drop(gid: int) -> None:
    with _CACHE_LOCK:
        entry = _CACHE.pop(gid, None)
    if entry:
        for dg in entry[1].values():
            dg.close()


def device_graph(g, placement: str = "zerocopy", device: int = 0) -> DeviceGraph:
    """The cached DeviceGraph of a CsrGraph (or g itself if already one)."""
    if isinstance(g, DeviceGraph):
        return g
    owner = getattr(g, "_device_graph_owner", None)
    if isinstance(owner, DeviceGraph) and owner.placement == placement and owner.device == device:
        return owner
    key = (placement, device, g.num_vertices, g.num_edges, g.edge_elem_bytes,
           g.weight_elem_bytes, bool(g.directed), id(g.offsets), id(g.edges), id(g.weights))
    gid = id(g)
    with _CACHE_LOCK:
        entry = _CACHE.get(gid)
        if entry is None or entry[0]() is not g:
            entry = (weakref.ref(g, lambda _r, gid=gid: _drop(gid)), {})
            _CACHE[gid] = entry
        per = entry[1]
        dg = per.pop(key, None)
        if dg is None:
            # at most HANDLES_PER_GRAPH live handles per graph object (each holds
            # a full copy of the lists): switching back and forth between two
            # placements does not re-pin, a third evicts the least recent
            while len(per) >= HANDLES_PER_GRAPH:
                per.pop(next(iter(per))).close()
            dg = DeviceGraph(g, placement, device)
        per[key] = dg  # most recently used last
    return dg


def release(g) -> None:
    """Drop the cached device handle of g (frees pinned / HBM memory)."""
    _drop(id(g))


# --------------------------------------------------------------- generators
def generate_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                  c: float = 0.19, seed: int = 27, *, symmetrize: bool = False,
                  weights: Optional[tuple[int, int]] = None, placement: str = "zerocopy",
                  device: int = 0) -> DeviceGraph:
    """R-MAT / Kronecker graph generated on the GPU straight into a handle."""
    lo, hi = weights if weights is not None else (1, 0)
    h = C.c_void_p()
    N.check(N.lib().zc_generate_rmat(scale, edge_factor, a, b, c, seed, int(symmetrize), lo, hi,
                                     N.PLACEMENTS[placement], device, C.byref(h)))
    return DeviceGraph(placement=placement, device=device, _handle=h.value)


def generate_uniform_device(num_vertices: int, min_degree: int, max_degree: int,
                            seed: int = 3, *, weights: Optional[tuple[int, int]] = None,
                            placement: str = "zerocopy", device: int = 0) -> DeviceGraph:
    """Uniform random graph (generate_uniform semantics) generated on the GPU."""
    lo, hi = weights if weights is not None else (1, 0)
    h = C.c_void_p()
    N.check(N.lib().zc_generate_uniform(num_vertices, min_degree, max_degree, seed, lo, hi,
                                        N.PLACEMENTS[placement], device, C.byref(h)))
    return DeviceGraph(placement=placement, device=device, _handle=h.value)


def open_emgi(path: str, directed: bool = True, placement: str = "zerocopy",
              device: int = 0, validate: bool = True) -> DeviceGraph:
    """EMGI file -> DeviceGraph, the payloads read straight into the handle's
    pinned / managed / staging buffers (reference load_csr_binary semantics,
    csr.py:204-245, without the int64 widening or a second copy)."""
    if placement not in N.PLACEMENTS:
        raise ValueError(f"placement must be one of {sorted(N.PLACEMENTS)}")
    flags = (N.ZC_F_DIRECTED if directed else 0) | (0 if validate else N.ZC_F_NO_VALIDATE)
    h = C.c_void_p()
    N.check(N.lib().zc_graph_open_emgi(str(path).encode(), N.PLACEMENTS[placement], device,
                                       flags, C.byref(h)))
    return DeviceGraph(placement=placement, device=device, _handle=h.value)


def evict(dg: DeviceGraph) -> None:
    dg.evict()


def read_probe(nbytes: int, chunk_bytes: int, random, alloc: str = "pinned",
               device: int = 0, iters: int = 3) -> float:
    """GB/s of warps reading chunk_bytes per request (zero-copy toy kernel)."""
    a = {"pinned": 0, "thp": 1, "hbm": 2, "vmm": 3, "hugetlb": 4, "managed_host": 5}[alloc]
    out = C.c_double()
    N.check(N.probe_lib().zc_read_probe(device, nbytes, int(random), chunk_bytes, a, iters,
                                  C.byref(out)))
    return out.value


def gather_probe(nbytes: int = 16 << 20, mode: int = 1, device: int = 0) -> float:
    """G random 4-byte loads/s into an nbytes device array (mode 1: with an
    atomicOr per 16 loads) -- the in-HBM control run's gather roofline."""
    out = C.c_double()
    N.check(N.probe_lib().zc_gather_probe(device, nbytes, mode, C.byref(out)))
    return out.value


def link_probe(device: int = 0, nbytes: int = 1 << 30, iters: int = 5) -> dict:
    """Measured host-link and HBM read bandwidths (GB/s)."""
    m, z, h = C.c_double(), C.c_double(), C.c_double()
    N.check(N.probe_lib().zc_link_probe(device, nbytes, iters, C.byref(m), C.byref(z), C.byref(h)))
    return {"memcpy_h2d_gbs": m.value, "zerocopy_read_gbs": z.value, "hbm_read_gbs": h.value}
