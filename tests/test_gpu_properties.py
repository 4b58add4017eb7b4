"""Property-based parity (hypothesis, like the reference's acceptance
criterion 6 stream): arbitrary small CSR graphs -- duplicate arcs, self
loops, isolated vertices, empty lists, 4- and 8-byte elements, zero and
large weights -- traversed by every strategy and schedule equal the CPU
oracle: values, iterations and per-iteration traversed edges (values only
for the work-efficient schedules)."""
import numpy as np
import pytest
from hypothesis import given, settings, HealthCheck
from hypothesis import strategies as st

import oracle
import paper_2006_06890_b200 as zc

pytestmark = pytest.mark.gpu

STRATS = ["naive", "merged", "merged-aligned", "packed", "compressed"]


@st.composite
def graphs(draw):
    nv = draw(st.integers(1, 90))
    degs = draw(st.lists(st.integers(0, 70), min_size=nv, max_size=nv))
    dst = draw(st.lists(st.integers(0, nv - 1), min_size=sum(degs), max_size=sum(degs)))
    eb = draw(st.sampled_from([4, 8]))
    wmax = draw(st.sampled_from([0, 9, 1000, 2 ** 31 - 1, 2 ** 40]))
    w = draw(st.lists(st.integers(0, wmax), min_size=sum(degs), max_size=sum(degs)))
    off = np.concatenate([[0], np.cumsum(degs)]).astype(np.int64)
    g = zc.CsrGraph(nv, int(off[-1]), off, np.asarray(dst, np.int64), np.asarray(w, np.int64),
                    eb, 4 if wmax < 2 ** 32 else 8, True)
    src = draw(st.integers(0, nv - 1))
    return g, src


def _same(r, ref, full=True):
    ok = np.array_equal(r.values, ref.values)
    if full:
        ok = ok and r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges
    return ok


@settings(max_examples=int(__import__("os").environ.get("ZC_HYP_EXAMPLES", "200")), deadline=None, derandomize=__import__("os").environ.get("ZC_HYP_RANDOM") != "1",
          suppress_health_check=list(HealthCheck))
@given(graphs())
def test_random_graphs_match_oracle(case):
    g, src = case
    ref_b, ref_s = oracle.bfs(g, src), oracle.sssp(g, src)
    gu = zc.symmetrized(g)
    ref_c = oracle.cc(gu)
    for s in STRATS:
        if s == "compressed" and g.edge_elem_bytes != 4:
            continue
        assert _same(zc.bfs(g, src, s, collect_traffic=False), ref_b), ("bfs", s)
        if s != "compressed" or g.weight_elem_bytes == 4:
            assert _same(zc.sssp(g, src, s, collect_traffic=False), ref_s), ("sssp", s)
            assert _same(zc.sssp(g, src, s, collect_traffic=False, schedule="near-far",
                                 delta=3), ref_s, False), ("near-far", s)
        assert _same(zc.cc(gu, s, collect_traffic=False), ref_c), ("cc", s)
        assert _same(zc.cc(gu, s, collect_traffic=False, schedule="afforest"), ref_c,
                     False), ("afforest", s)
    if g.edge_elem_bytes == 4:
        r = zc.bfs(g, src, "direction-optimizing", collect_traffic=False)
        assert _same(r, ref_b), "direction-optimizing"
    for s in ("naive", "merged", "merged-aligned"):  # the request model on every graph
        r = zc.bfs(g, src, s, collect_traffic=True)
        assert _same(r, ref_b) and len(r.per_iteration_traffic) == r.iterations
    zc.release(g)
    zc.release(gu)


@settings(max_examples=int(__import__("os").environ.get("ZC_HYP_EXAMPLES", "200")) // 4,
          deadline=None, derandomize=__import__("os").environ.get("ZC_HYP_RANDOM") != "1",
          suppress_health_check=list(HealthCheck))
@given(graphs(), st.integers(1, 4), st.sampled_from(["merged-aligned", "packed"]),
       st.sampled_from([(False, "bitmap"), (True, "bitmap"), (True, "store")]))
def test_random_partitions_match_oracle(case, nparts, strategy, exchange):
    """Vertex-range partitions of arbitrary graphs (ranges may be empty) with
    every exchange: identical values, iterations and traversed edges."""
    from paper_2006_06890_b200.multi import (CudaPartition, edge_balanced_bounds, local_part,
                                             run_partitions_local)
    g, src = case
    g = zc.CsrGraph(g.num_vertices, g.num_edges, g.offsets, g.edges,
                    np.minimum(np.asarray(g.weights), 2 ** 31), g.edge_elem_bytes, 4, True)
    gu = zc.symmetrized(g)
    fused, bx = exchange
    for algo, graph in (("bfs", g), ("sssp", g), ("cc", gu)):
        ref = oracle.run(algo, graph, src)
        b = edge_balanced_bounds(graph.offsets, nparts)
        engines = [CudaPartition(local_part(graph, b, k), b, k) for k in range(nparts)]
        vals, iters, trav = run_partitions_local(engines, algo, src, strategy, fused=fused,
                                                 bfs_exchange=bx)
        assert np.array_equal(vals, ref.values), (algo, nparts, strategy, exchange)
        assert iters == ref.iterations and trav == ref.traversed_edges
        for e in engines:
            e.close()
