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


class NumpyPartition:
    def __init__(self, g_local, bounds, part):
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.lo = int(self.bounds[part])
        self.num_local = int(self.bounds[part + 1]) - self.lo
        self.stride = exchange_stride(self.bounds)
        self.device = "cpu"
        self.off = np.asarray(g_local.offsets, np.int64)
        self.edges = np.asarray(g_local.edges, np.int64)
        self.w = None if g_local.weights is None else np.asarray(g_local.weights, np.int64)

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
        return self.front.size, self._degsum(self.front)

    def result(self):
        if self.algo == "sssp":
            out = self.state.astype(np.int64)
            out[self.state == INF] = np.iinfo(np.int64).max
            return out
        return self.state.astype(np.int64)


def gloo_worker(rank, world, port, graph, algo, source, q):
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
            eng = NumpyPartition(local_part(g, bounds, rank), bounds, rank)
            r = run_partition(eng, al, src, "merged-aligned", tensor_device=torch.device("cpu"))
            results.append((r.lo, r.values, r.iterations, r.traversed_edges))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()
