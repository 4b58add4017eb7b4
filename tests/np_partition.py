"""TEST INFRASTRUCTURE: a numpy model of one partition's steps (the zc_part_*
protocol of include/zcgraph.h), so the SPMD driver
paper_2006_06890_b200.multi.run_partition and its collectives can be tested
with gloo on CPU.  Never used by the product."""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2006_06890_b200.multi import EXCH_NONE, exchange_stride  # noqa: E402

INF = np.iinfo(np.uint64).max


def owned_in_lists(g, lo, hi):
    """In-lists (global source ids) of the owned destinations [lo, hi) of g."""
    off = np.asarray(g.offsets, np.int64)
    dst = np.asarray(g.edges, np.int64)
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(off))
    keep = (dst >= lo) & (dst < hi)
    order = np.argsort(dst[keep], kind="stable")
    d, s = dst[keep][order], src[keep][order]
    in_off = np.zeros(hi - lo + 1, np.int64)
    np.add.at(in_off, d - lo + 1, 1)
    return np.cumsum(in_off), s


class NumpyPartition:
    def __init__(self, g_local, bounds, part, in_lists=None):
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.lo = int(self.bounds[part])
        self.num_local = int(self.bounds[part + 1]) - self.lo
        self.stride = exchange_stride(self.bounds)
        self.device = "cpu"
        self.off = np.asarray(g_local.offsets, np.int64)
        self.edges = np.asarray(g_local.edges, np.int64)
        self.w = None if g_local.weights is None else np.asarray(g_local.weights, np.int64)
        # direction-optimizing bfs: the owned vertices' in-lists (zc_part_build_in_lists)
        self.in_off, self.in_src = in_lists if in_lists is not None else (None, None)
        self.unvisited = 0

    # -- zc_part_unvisited_in / zc_part_frontier_bits / zc_part_pull
    @property
    def bitmap_words(self):
        return (int(self.bounds[-1]) + 31) // 32 + 1

    def _indeg(self, f):
        return int((self.in_off[f + 1] - self.in_off[f]).sum()) if self.in_off is not None else 0

    def unvisited_in(self):
        return self.unvisited

    def frontier_bits(self, bits):
        b = bits.numpy().view(np.uint32)
        b[:] = 0
        g = self.lo + self.front
        np.bitwise_or.at(b, g >> 5, (np.uint32(1) << (g & 31).astype(np.uint32)))

    def pull(self, bits):
        b = bits.numpy().view(np.uint32)
        self.iter += 1
        cand = np.flatnonzero((self.state == -1) & (np.diff(self.in_off) > 0))
        new = []
        for u in cand:
            srcs = self.in_src[self.in_off[u]:self.in_off[u + 1]]
            if ((b[srcs >> 5] >> (srcs & 31).astype(np.uint32)) & 1).any():
                new.append(u)
        self.front = np.asarray(new, np.int64)
        self.state[self.front] = self.iter
        self.unvisited -= self._indeg(self.front)
        self.fval = self.state[self.front].astype(np.int64)
        return self.front.size, self._degsum(self.front)

    def _degsum(self, f):
        return int((self.off[f + 1] - self.off[f]).sum())

    def begin(self, algo, source, strategy):
        self.algo, self.iter = algo, 0
        R = self.num_local
        if algo == "bfs":
            self.state = np.full(R, -1, np.int64)
        elif algo == "sssp":
            self.state = np.full(R, INF, np.uint64)
        else:
            self.state = self.lo + np.arange(R, dtype=np.int64)
        if algo == "cc":
            self.front = np.arange(R, dtype=np.int64)
        elif self.lo <= source < self.lo + R:
            self.front = np.array([source - self.lo], np.int64)
            self.state[source - self.lo] = 0
        else:
            self.front = np.zeros(0, np.int64)
        self.fval = self.state[self.front].astype(np.int64)
        if self.in_off is not None:
            self.unvisited = int(self.in_off[-1]) - self._indeg(self.front)
        return self.front.size, self._degsum(self.front)

    def expand(self, exch):
        a = exch.numpy()
        a[:] = EXCH_NONE[self.algo]
        self.iter += 1
        f = self.front
        degs = self.off[f + 1] - self.off[f]
        rep = np.repeat(np.arange(f.size), degs)
        eidx = self.off[f][rep] + (np.arange(rep.size) - np.repeat(np.cumsum(degs) - degs, degs))
        dst = self.edges[eidx]
        owner = np.searchsorted(self.bounds, dst, side="right") - 1
        slot = owner * self.stride + (dst - self.bounds[owner])
        if self.algo == "bfs":
            a[slot] = 1
        elif self.algo == "sssp":
            np.minimum.at(a, slot, self.fval[rep] + self.w[eidx])
        else:
            np.minimum.at(a, slot, self.fval[rep].astype(np.int32))

    def apply(self, mine):
        m = mine.numpy()[:self.num_local]
        if self.algo == "bfs":
            new = (m != 0) & (self.state == -1)
            self.state[new] = self.iter
        elif self.algo == "sssp":
            mm = m.astype(np.int64)
            new = (mm != EXCH_NONE["sssp"]) & (mm.astype(np.uint64) < self.state)
            self.state[new] = mm[new].astype(np.uint64)
        else:
            new = m.astype(np.int64) < self.state
            self.state[new] = m[new]
        self.front = np.flatnonzero(new)
        self.fval = self.state[self.front].astype(np.int64)
        self.unvisited -= self._indeg(self.front)
        return self.front.size, self._degsum(self.front)

    def result(self):
        if self.algo == "sssp":
            out = self.state.astype(np.int64)
            out[self.state == INF] = np.iinfo(np.int64).max
            return out
        return self.state.astype(np.int64)


def gloo_worker(rank, world, port, graph, algo, source, q, strategy="merged-aligned"):
    """One rank of a gloo world: partition, run the SPMD driver, report."""
    import torch
    import torch.distributed as dist
    from paper_2006_06890_b200.multi import edge_balanced_bounds, local_part, run_partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for g, al, src in zip(graph, algo, source):
            bounds = edge_balanced_bounds(g.offsets, world)
            lo, hi = int(bounds[rank]), int(bounds[rank + 1])
            eng = NumpyPartition(local_part(g, bounds, rank), bounds, rank,
                                 owned_in_lists(g, lo, hi))
            r = run_partition(eng, al, src, strategy, tensor_device=torch.device("cpu"))
            results.append((r.lo, r.values, r.iterations, r.traversed_edges, r.local_traversed,
                            r.exchange_bytes, r.bottom_up_steps))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()
