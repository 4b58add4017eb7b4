"""The partitioned (multi-GPU) driver with world_size 2 and 3 over gloo on CPU:
partitioning, exchange protocol, termination and result assembly must give
the reference's values, iteration counts and traversed edges."""
import multiprocessing as mp
import random

import numpy as np
import pytest

import oracle
from fixtures import small_cases
from np_partition import gloo_worker

import paper_2006_06890_b200 as zc
from paper_2006_06890_b200.multi import edge_balanced_bounds, exchange_stride, local_part


def _run_world(world, graphs, algos, sources, strategy="merged-aligned"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=gloo_worker,
                      args=(r, world, port, graphs, algos, sources, q, strategy))
          for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    merged = []
    for k in range(len(graphs)):
        parts = [out[r][k] for r in range(world)]  # rank order = range order
        vals = np.concatenate([p[1] for p in parts])
        iters = {p[2] for p in parts}
        trav = {tuple(p[3]) for p in parts}
        assert len(iters) == 1 and len(trav) == 1  # every rank agrees
        # each rank streamed its own frontiers' lists: together the global work
        assert sum(p[4] for p in parts) == sum(parts[0][3])
        # bottom-up steps all-reduce the frontier bitmap: counted as sent bytes
        assert all((p[5] > 0) == (p[6] > 0) for p in parts)
        merged.append((vals, iters.pop(), list(trav.pop())))
    return merged


def _cases():
    cases = [c for c in small_cases() if c.tag.startswith(("c8_", "pl_")) or c.index < 11]
    return cases


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_driver_matches_reference(world):
    cases = _cases()
    got = _run_world(world, [c.graph for c in cases], [c.algo for c in cases],
                     [max(c.source, 0) for c in cases])
    for c, (vals, iters, trav) in zip(cases, got):
        assert np.array_equal(vals, c.values), c.tag
        assert iters == c.iterations, c.tag
        assert trav == c.traversed, c.tag


def test_partitioned_driver_uniform_graph():
    g = zc.with_uniform_weights(zc.generate_uniform(3000, 2, 12, seed=4))
    gu = zc.symmetrized(g)
    got = _run_world(2, [g, g, gu], ["bfs", "sssp", "cc"], [5, 5, 0])
    for (vals, iters, trav), ref in zip(got, [oracle.bfs(g, 5), oracle.sssp(g, 5), oracle.cc(gu)]):
        assert np.array_equal(vals, ref.values)
        assert iters == ref.iterations and trav == ref.traversed_edges


def test_edge_balanced_bounds():
    g = zc.generate_powerlaw(5000, 10.0, 2.0, seed=2)
    for p in (1, 2, 4, 8):
        b = edge_balanced_bounds(g.offsets, p).astype(np.int64)
        assert b[0] == 0 and b[-1] == g.num_vertices and np.all(np.diff(b) >= 0)
        per = np.diff(np.asarray(g.offsets)[b])
        assert per.sum() == g.num_edges
        assert per.max() <= g.num_edges / p + g.degrees.max()  # balanced up to one list
        parts = [local_part(g, b, k) for k in range(p)]
        assert sum(x.num_vertices for x in parts) == g.num_vertices
        assert exchange_stride(b) == int(np.diff(b).max())


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_direction_optimizing_driver(world):
    """Direction-optimizing SPMD protocol: top-down steps by reduce-scatter,
    bottom-up steps against the SUM-all-reduced (= OR) owned-frontier bitmaps,
    switch test on all-reduced unvisited in-edges -- reference levels,
    iterations and traversed edges on directed and undirected graphs."""
    g = zc.generate_powerlaw(4000, 12.0, 2.0, seed=6)
    gu = zc.symmetrized(g)
    cases = [c for c in _cases() if c.algo == "bfs"]
    graphs = [g, gu] + [c.graph for c in cases]
    srcs = [int(zc.pick_sources(g, 1)[0]), int(zc.pick_sources(gu, 1)[0])] + \
           [max(c.source, 0) for c in cases]
    got = _run_world(world, graphs, ["bfs"] * len(graphs), srcs, "direction-optimizing")
    for gr, s, (vals, iters, trav) in zip(graphs, srcs, got):
        ref = oracle.bfs(gr, s)
        assert np.array_equal(vals, ref.values)
        assert iters == ref.iterations and trav == ref.traversed_edges


def test_pull_rule():
    from paper_2006_06890_b200.multi import DO_ALPHA, pull_now
    assert DO_ALPHA == 2.0
    assert not pull_now(1, 10**9, 1)          # never the source's own expansion
    assert pull_now(2, 600, 1000) and not pull_now(2, 400, 1000)


def test_driver_argument_errors_and_accounting():
    from paper_2006_06890_b200.multi import allreduce_send_bytes, run_partition
    with pytest.raises(ValueError, match="bfs_exchange"):
        run_partition(None, "bfs", 0, "merged-aligned", bfs_exchange="ring")
    with pytest.raises(ValueError, match="unknown algorithm"):
        run_partition(None, "pagerank", 0, "merged-aligned")
    # a ring all-reduce sends 2 (p - 1) / p of the buffer per rank; nothing alone
    assert allreduce_send_bytes(1000, 1) == 0
    assert allreduce_send_bytes(1000, 2) == 1000
    assert allreduce_send_bytes(800, 4) == 1200
