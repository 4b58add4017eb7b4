"""Parity of the CUDA path (through the C ABI) with the reference's outputs and
the CPU oracle.  Bit-exact: values (int64), iteration counts and per-iteration
traversed-edge counts; modelled traffic histograms too.
"""
import os

import numpy as np
import pytest

import oracle
from fixtures import crc, goldens, small_cases, traffic_cases

import paper_2006_06890_b200 as zc

pytestmark = pytest.mark.gpu

STRATS = list(zc.AccessStrategy)
# the reference's three + the B200 "packed" extension (identical results)
ALL = STRATS + ["packed"]
ALL_IDS = [getattr(s, "value", s) for s in ALL]
CASES = small_cases()


def _run(c, strategy, placement="zerocopy", traffic=False):
    fn = {"bfs": lambda: zc.bfs(c.graph, c.source, strategy, collect_traffic=traffic,
                                placement=placement),
          "sssp": lambda: zc.sssp(c.graph, c.source, strategy, collect_traffic=traffic,
                                  placement=placement),
          "cc": lambda: zc.cc(c.graph, strategy, collect_traffic=traffic,
                              placement=placement)}[c.algo]
    return fn()


@pytest.mark.parametrize("strategy", ALL, ids=ALL_IDS)
def test_small_graphs_match_reference(strategy):
    bad = []
    for c in CASES:
        r = _run(c, strategy)
        if not (np.array_equal(r.values, c.values) and r.iterations == c.iterations
                and r.traversed_edges == c.traversed):
            bad.append((c.index, c.tag))
    assert not bad, f"{len(bad)} mismatches, first {bad[:8]}"


@pytest.mark.parametrize("placement", ["uvm", "hbm", "zerocopy-managed"])
def test_small_graphs_other_placements(placement):
    """Every fixture on the other placements: values, iterations and
    per-iteration traversed edges."""
    bad = []
    for c in CASES:
        r = _run(c, zc.AccessStrategy.MERGED_ALIGNED, placement)
        if not (np.array_equal(r.values, c.values) and r.iterations == c.iterations
                and r.traversed_edges == c.traversed):
            bad.append((c.index, c.tag))
        zc.release(c.graph)
    assert not bad, bad[:8]


def test_host_rmat_generator_matches_device():
    """oracle.generate_rmat (host C, the bench's reference arm input) builds
    byte-identical CSR to the product's GPU generator."""
    for scale, ef, seed in ((10, 16, 27), (16, 16, 5), (17, 8, 27)):
        dg = zc.generate_rmat(scale, ef, seed=seed)
        off, edges = oracle.generate_rmat(scale, ef, seed=seed, threads=4)
        g = dg.as_csr()
        assert np.array_equal(np.asarray(g.offsets, np.int64), off)
        assert np.array_equal(np.asarray(g.edges, np.uint32), edges)
        dg.close()


def test_reference_built_graphs_traverse_like_the_reference():
    """Graphs built by the unmodified reference (oracle.reference(): the
    /root/reference tree or its oracle/_ref zip on the GPU box) traversed by
    the CUDA path equal the reference's own bfs / sssp / cc results."""
    try:
        ref = oracle.reference()
    except ImportError:
        pytest.skip("reference package unavailable")
    g = ref.with_uniform_weights(ref.generate_powerlaw(3000, 6.0, seed=11))
    gu = ref.symmetrized(ref.generate_uniform(2000, 0, 5, seed=12))
    for src in [int(x) for x in ref.pick_sources(g, 3, seed=7)]:
        for algo in ("bfs", "sssp"):
            want = getattr(ref, algo)(g, src, collect_traffic=False)
            for s in ALL + ["compressed"] + (["direction-optimizing"] if algo == "bfs" else []):
                got = getattr(zc, algo)(g, src, s, collect_traffic=False)
                assert np.array_equal(got.values, want.values), (algo, s, src)
                assert got.iterations == want.iterations, (algo, s, src)
                assert got.traversed_edges == [int(x) for x in want.traversed_edges], (algo, s)
    want = ref.cc(gu, collect_traffic=False)
    for s in ALL + ["compressed"]:
        got = zc.cc(gu, s, collect_traffic=False)
        assert np.array_equal(got.values, want.values) and got.iterations == want.iterations


def test_traffic_model_matches_reference():
    bad = []
    for idx, sid, hist in traffic_cases():
        c = CASES[idx]
        r = _run(c, STRATS[sid], traffic=True)
        got = np.array([[t.hist[s] for s in (32, 64, 96, 128)] for t in r.per_iteration_traffic],
                       np.int64).reshape(-1, 4)
        if not np.array_equal(got, hist):
            bad.append((idx, c.tag, STRATS[sid].value))
    assert not bad, f"{len(bad)} traffic mismatches, first {bad[:8]}"


def _mid(name, g):
    gold = goldens()[name]
    gw = zc.with_uniform_weights(g)
    gu = zc.symmetrized(g)
    for s in ALL:
        for algo, graph in (("bfs", g), ("sssp", gw), ("cc", gu)):
            if algo == "cc":
                r = zc.cc(graph, s, collect_traffic=False)
            else:
                r = getattr(zc, algo)(graph, gold["src"], s, collect_traffic=False)
            assert crc(r.values) == gold[algo]["crc"], (algo, s)
            assert r.iterations == gold[algo]["iterations"], (algo, s)
            assert r.traversed_edges == gold[algo]["traversed_edges"], (algo, s)


def test_uniform_2p16_all_strategies():
    _mid("uniform_2p16_d16", zc.generate_uniform(2 ** 16, 16, 16, seed=3))


def test_powerlaw_100k_all_strategies():
    _mid("powerlaw_100k_d8", zc.generate_powerlaw(100000, 8.0, 2.0, seed=3))


def test_config1_goldens():
    """Config 1: uniform 2^20 deg 16 seed 3 -- BFS src 0 crc 171fbc8b (8
    levels), SSSP 2e5f7c3e (16 iterations), CC 1ad2bc45 (6 iterations)."""
    g = zc.generate_uniform(2 ** 20, 16, 16, seed=3)
    gold = goldens()["c1"]
    r = zc.bfs(g, 0, collect_traffic=False)
    assert crc(r.values) == gold["bfs"]["crc"] == "171fbc8b"
    assert r.traversed_edges == gold["bfs"]["traversed_edges"]
    for s, rec in gold["bfs_sources"].items():
        assert crc(zc.bfs(g, int(s), collect_traffic=False).values) == rec["crc"]
    gw = zc.with_uniform_weights(g)
    r = zc.sssp(gw, 0, collect_traffic=False)
    assert crc(r.values) == gold["sssp"]["crc"] and r.iterations == 16
    r = zc.cc(zc.symmetrized(g), collect_traffic=False)
    assert crc(r.values) == gold["cc"]["crc"] and r.iterations == 6


@pytest.mark.parametrize("symmetrize", [False, True])
def test_rmat_generator_vs_oracle(symmetrize):
    dg = zc.generate_rmat(16, 16, seed=5, symmetrize=symmetrize, weights=(8, 72))
    g = dg.as_csr()
    zc.validate(g)
    assert g.num_edges == (2 if symmetrize else 1) * 16 * 2 ** 16
    src = int(zc.pick_sources(g, 1)[0])
    algos = [("cc", None)] if symmetrize else [("bfs", src), ("sssp", src)]
    for algo, s in algos:
        ref = oracle.run(algo, g, s or 0, threads=8)
        for st in ALL:
            r = zc.cc(dg, st, collect_traffic=False) if algo == "cc" else \
                getattr(zc, algo)(dg, s, st, collect_traffic=False)
            assert np.array_equal(r.values, ref.values), (algo, st)
            assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges


def test_rmat_generator_deterministic_and_symmetric():
    a = zc.generate_rmat(14, 8, seed=9)
    b = zc.generate_rmat(14, 8, seed=9)
    ga, gb = a.as_csr(), b.as_csr()
    assert np.array_equal(ga.offsets, gb.offsets) and np.array_equal(ga.edges, gb.edges)
    s = zc.generate_rmat(14, 8, seed=9, symmetrize=True).as_csr()
    ref = zc.symmetrized(ga)  # reference csr.py:350-359 semantics
    assert np.array_equal(s.offsets, ref.offsets)
    assert np.array_equal(np.asarray(s.edges, np.int64), ref.edges)


def test_uniform_generator_device():
    dg = zc.generate_uniform_device(50000, 16, 16, seed=4, weights=(8, 72))
    g = dg.as_csr()
    zc.validate(g)
    assert np.all(np.diff(g.offsets) == 16)
    lists = np.sort(np.asarray(g.edges).reshape(-1, 16), axis=1)
    assert not np.any(lists[:, 1:] == lists[:, :-1])  # no in-list duplicates
    assert int(g.weights.min()) >= 8 and int(g.weights.max()) <= 72
    ref = oracle.sssp(g, 0, threads=8)
    r = zc.sssp(dg, 0, collect_traffic=False)
    assert np.array_equal(r.values, ref.values) and r.iterations == ref.iterations


def test_edge_cases():
    empty = zc.CsrGraph(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), directed=False)
    r = zc.cc(empty, collect_traffic=False)
    assert r.values.size == 0 and r.iterations == 0
    single = zc.CsrGraph(1, 1, np.array([0, 1]), np.array([0]), weights=np.array([0]))
    assert zc.bfs(single, 0).values.tolist() == [0]
    assert zc.sssp(single, 0).values.tolist() == [0]
    # a hub whose list spans many lines, unaligned start: big-list path
    n = 40000
    off = np.array([0, 3] + [3 + n] * (n - 1), np.int64)
    edges = np.concatenate([[1, 2, 3], np.arange(1, n + 1) % n]).astype(np.int64)
    g = zc.CsrGraph(n, int(off[-1]), off, edges)
    for s in ALL + ["compressed", "direction-optimizing"]:
        r = zc.bfs(g, 1, s, collect_traffic=False)
        assert np.array_equal(r.values, oracle.bfs(g, 1).values)
    # compressed / direction-optimizing on the degenerate graphs
    for s in ("compressed", "direction-optimizing"):
        assert zc.bfs(single, 0, s, collect_traffic=False).values.tolist() == [0]
        nolinks = zc.CsrGraph(5, 0, np.zeros(6, np.int64), np.zeros(0, np.int64))
        r = zc.bfs(nolinks, 2, s, collect_traffic=False)
        assert r.values.tolist() == [-1, -1, 0, -1, -1] and r.iterations == 1
    assert zc.sssp(single, 0, "compressed", collect_traffic=False).values.tolist() == [0]
    assert zc.cc(empty, "compressed", collect_traffic=False).values.size == 0


def test_packed_many_empty_and_shared_blocks():
    """Dense runs of tiny / empty lists sharing blocks, across the 256-slot
    stage groups (packed windows and their owner search)."""
    rng = np.random.default_rng(3)
    n = 20000
    deg = rng.choice([0, 0, 1, 2, 3, 40], size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=off[1:])
    edges = rng.integers(0, n, off[-1])
    w = rng.integers(0, 9, off[-1])
    g = zc.CsrGraph(n, int(off[-1]), off, edges, w)
    gu = zc.symmetrized(g)
    src = int(np.flatnonzero(deg)[0])
    for algo, graph in (("bfs", g), ("sssp", g), ("cc", gu)):
        ref = oracle.run(algo, graph, src, threads=8)
        r = zc.cc(graph, "packed", collect_traffic=False) if algo == "cc" else \
            getattr(zc, algo)(graph, src, "packed", collect_traffic=False)
        assert np.array_equal(r.values, ref.values), algo
        assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges
    with pytest.raises(ValueError, match="request model"):
        zc.bfs(g, src, "packed", collect_traffic=True)  # model undefined for packed
    # the default (collect_traffic=None) skips the model for the extensions
    r = zc.bfs(g, src, "packed")
    assert r.total_traffic.request_count == 0 and len(r.per_iteration_traffic) == r.iterations


def test_link_probe_sane():
    p = zc.link_probe(nbytes=256 << 20, iters=3)
    assert 5 < p["memcpy_h2d_gbs"] < 200
    assert 1 < p["zerocopy_read_gbs"] < 200
    assert p["hbm_read_gbs"] > 500


# ------------------------------------------------------------ partitions
from paper_2006_06890_b200.multi import (CudaPartition, edge_balanced_bounds, generate_rmat_part,
                                         local_part, run_partitions_local)


@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_cuda_partitions_match_reference(nparts):
    """Several CUDA partitions on one GPU, host-side reduction in place of the
    reduce-scatter: identical values / iterations / traversed edges."""
    bad = []
    for c in [c for c in CASES if c.tag.startswith(("c8_", "pl_", "e8_")) or c.index < 11]:
        b = edge_balanced_bounds(c.graph.offsets, nparts)
        engines = [CudaPartition(local_part(c.graph, b, k), b, k) for k in range(nparts)]
        for s in ALL:
            vals, iters, trav = run_partitions_local(engines, c.algo, max(c.source, 0), s)
            if not (np.array_equal(vals, c.values) and iters == c.iterations
                    and trav == c.traversed):
                bad.append((c.tag, c.index, s.value))
        for e in engines:
            e.close()
    assert not bad, bad[:8]


@pytest.mark.parametrize("nparts,bfs_exchange", [(2, "bitmap"), (3, "bitmap"), (2, "store"),
                                                 (3, "store")])
def test_cuda_partitions_fused_exchange(nparts, bfs_exchange):
    """Fused exchanges on one GPU (peer pointers within the device): BFS
    bitmap OR or candidate stores, SSSP / CC remote atomicMin after the local
    pre-filter -- identical values / iterations / traversed edges."""
    bad = []
    for c in [c for c in CASES if c.tag.startswith(("c8_", "pl_")) or c.index < 11]:
        b = edge_balanced_bounds(c.graph.offsets, nparts)
        engines = [CudaPartition(local_part(c.graph, b, k), b, k) for k in range(nparts)]
        for s in ("merged-aligned", "packed"):
            vals, iters, trav = run_partitions_local(engines, c.algo, max(c.source, 0), s,
                                                     fused=True, bfs_exchange=bfs_exchange)
            if not (np.array_equal(vals, c.values) and iters == c.iterations
                    and trav == c.traversed):
                bad.append((c.tag, c.index, s))
        for e in engines:
            e.close()
    assert not bad, bad[:8]


def test_rmat_partition_generator_matches_whole_graph():
    whole = zc.generate_rmat(16, 16, seed=11, weights=(8, 72)).as_csr()
    parts = [generate_rmat_part(16, 4, k, seed=11, weights=(8, 72)) for k in range(4)]
    b = parts[0].bounds
    assert np.array_equal(b, edge_balanced_bounds(whole.offsets, 4))
    for k, p in enumerate(parts):
        ref = local_part(whole, b, k)
        got = p.graph_view()
        assert np.array_equal(got.offsets, ref.offsets)
        assert np.array_equal(np.asarray(got.edges), np.asarray(ref.edges))
        assert np.array_equal(np.asarray(got.weights), np.asarray(ref.weights))
    src = int(zc.pick_sources(whole, 1)[0])
    for algo in ("bfs", "sssp"):
        ref = oracle.run(algo, whole, src, threads=8)
        vals, iters, trav = run_partitions_local(parts, algo, src, "merged-aligned")
        assert np.array_equal(vals, ref.values) and iters == ref.iterations
        assert trav == ref.traversed_edges


def test_symmetric_rmat_partition_generator_matches_whole_graph():
    """Partitions of the symmetrized R-MAT graph (every rank enumerates the
    reverse arcs into its range): the whole graph's slices, edge-balanced over
    its 2E arcs; BFS and CC over them (both exchanges) equal the oracle."""
    whole = zc.generate_rmat(15, 16, seed=5, symmetrize=True)
    g = whole.as_csr()  # views of the handle's pinned lists: closed at the end
    src = int(zc.pick_sources(g, 1, seed=7)[0])
    for nparts in (1, 2, 3):
        parts = [generate_rmat_part(15, nparts, k, seed=5, symmetrize=True)
                 for k in range(nparts)]
        b = parts[0].bounds
        assert np.array_equal(b, edge_balanced_bounds(g.offsets, nparts))
        for k, p in enumerate(parts):
            ref = local_part(g, b, k)
            got = p.graph_view()
            assert not got.directed
            assert np.array_equal(got.offsets, ref.offsets)
            assert np.array_equal(np.asarray(got.edges), np.asarray(ref.edges))
        for algo in ("bfs", "cc"):
            ref = oracle.run(algo, g, src, threads=8)
            for fused, bx in ((False, "bitmap"), (True, "bitmap"), (True, "store")):
                vals, iters, trav = run_partitions_local(parts, algo, src, "merged-aligned",
                                                         fused=fused, bfs_exchange=bx)
                assert np.array_equal(vals, ref.values), (nparts, algo, fused)
                assert iters == ref.iterations and trav == ref.traversed_edges
        for p in parts:
            p.close()
    with pytest.raises(ValueError):
        generate_rmat_part(10, 2, 0, symmetrize=True, weights=(1, 5))
    whole.close()


def test_sssp_pairs_stream_default_and_opt_out():
    """SSSP with 4-byte edges and weights reads the interleaved (dst, weight)
    stream for the windowed raw strategies (built on first use); "pairs=0"
    reads the separate arrays.  Both equal the oracle exactly."""
    u = zc.generate_uniform_device(1 << 15, 2, 24, seed=8, weights=(1, 90))
    g = u.as_csr()
    src = int(zc.pick_sources(g, 1, seed=7)[0])
    ref = oracle.sssp(g, src, threads=8)
    for tune in ("", "pairs=0", "pairs=1"):
        u.set_tuning(tune)
        for s in ALL:
            r = zc.sssp(u, src, s, collect_traffic=False)
            assert np.array_equal(r.values, ref.values), (tune, s)
            assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges
        r = zc.sssp(u, src, "merged-aligned", collect_traffic=False, schedule="near-far")
        assert np.array_equal(r.values, ref.values), tune
    u.close()


def test_pagerank_matches_reference():
    """Reference pagerank outputs (incl. acceptance criterion 6's PR stream):
    L-inf <= 1e-8 (test_acceptance.py:169-180), the same iteration count (the
    push sums are fixed point, so the count does not depend on the atomic
    order), the multigraph flag; all strategies."""
    import warnings
    from fixtures import pagerank_cases
    bad = []
    for k, (g, (dmp, mi, tol), ranks, iters, multi, derr) in enumerate(pagerank_cases()):
        for s in ALL:
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                r = zc.pagerank(g, s, dmp, mi, tol, collect_traffic=False)
            err = float(np.abs(r.values - ranks).max())
            if err > 1e-8 or r.iterations != iters or ("multigraph" in r.flags) != multi:
                bad.append((k, getattr(s, "value", s), err, r.iterations, iters))
            if multi:
                assert any("multigraph" in str(w.message) for w in caught)
    assert not bad, bad[:8]


def test_pagerank_traffic_and_validation():
    g = zc.symmetrized(zc.generate_uniform(300, 1, 6, seed=4))
    r = zc.pagerank(g)
    assert len(r.per_iteration_traffic) == r.iterations
    assert all(n == g.num_edges for n in r.traversed_edges)
    assert r.total_traffic.request_count > 0
    with pytest.raises(ValueError):
        zc.pagerank(g, damping=1.0)
    with pytest.raises(ValueError):
        zc.pagerank(g, max_iters=0)
    with pytest.raises(ValueError):
        zc.pagerank(g, tol=-1.0)


def test_report_rows_join_reference_checksums(tmp_path):
    """Rows carry the reference's columns; levels_checksum and the modelled
    histogram equal the reference's for the same run (config-1 style graph)."""
    from paper_2006_06890_b200.report import COLUMNS, measure, write_rows_csv
    g = zc.generate_uniform(2 ** 16, 16, 16, seed=3)
    gold = goldens()["uniform_2p16_d16"]
    rows = measure(g, "bfs", ("merged-aligned", "packed"), sources=[gold["src"]], label="u16")
    assert {r["levels_checksum"] for r in rows} == {gold["bfs"]["crc"]}
    assert rows[0]["requests_total"] > 0 and rows[1]["requests_total"] == ""
    p = tmp_path / "results.csv"
    write_rows_csv(rows, str(p))
    lines = p.read_text().splitlines()
    assert lines[0].startswith("# emogi-b200") and lines[1].split(",") == COLUMNS


@pytest.mark.parametrize("placement", ["zerocopy", "uvm", "hbm", "zerocopy-managed"])
def test_open_emgi_roundtrip(tmp_path, placement):
    g = zc.with_uniform_weights(zc.generate_uniform(2 ** 16, 16, 16, seed=3))
    gold = goldens()["uniform_2p16_d16"]
    p = tmp_path / "u16.emgi"
    zc.store_csr_binary(g, str(p))
    dg = zc.open_emgi(str(p), placement=placement)
    h = dg.as_csr()
    assert crc(h.edges, "<u4") == gold["graph"]["edges_crc_u4"]
    assert crc(zc.bfs(dg, gold["src"], collect_traffic=False).values) == gold["bfs"]["crc"]
    assert crc(zc.sssp(dg, gold["src"], collect_traffic=False).values) == gold["sssp"]["crc"]
    dg.close()


def test_sssp_pairs_layout_identical():
    """Interleaved (dst, weight) stream: same SSSP results, all strategies."""
    bad = []
    for c in [c for c in CASES if c.algo == "sssp" and c.graph.edge_elem_bytes == 4]:
        dg = zc.DeviceGraph(c.graph)
        dg.build_sssp_pairs()
        for s in ALL:
            r = zc.sssp(dg, c.source, s, collect_traffic=False)
            if not (np.array_equal(r.values, c.values) and r.iterations == c.iterations
                    and r.traversed_edges == c.traversed):
                bad.append((c.tag, c.index, getattr(s, "value", s)))
        dg.close()
    assert not bad, bad[:8]
    u = zc.generate_uniform_device(1 << 16, 16, 16, seed=9, weights=(8, 72))
    ref = zc.sssp(u, 5, "packed", collect_traffic=False)
    u.build_sssp_pairs()
    for s in ALL:
        r = zc.sssp(u, 5, s, collect_traffic=False)
        assert np.array_equal(r.values, ref.values) and r.iterations == ref.iterations


def test_scale_parity_k24():
    """2^28-arc Kronecker graphs (2^29 symmetrized): GPU vs the oracle on the
    same in-memory graph, every strategy but naive (hubs make it slow)."""
    dg = zc.generate_rmat(24, 16, seed=31, weights=(8, 72))
    g = dg.as_csr()
    src = int(zc.pick_sources(g, 1, seed=7)[0])
    for algo in ("bfs", "sssp"):
        ref = oracle.run(algo, g, src, threads=os.cpu_count())
        for s in ("merged", "merged-aligned", "packed"):
            r = getattr(zc, algo)(dg, src, s, collect_traffic=False)
            assert np.array_equal(r.values, ref.values), (algo, s)
            assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges
    dg.close()
    sg = zc.generate_rmat(23, 16, seed=31, symmetrize=True)
    ref = oracle.cc(sg.as_csr(), threads=os.cpu_count())
    for s in ("merged-aligned", "packed"):
        r = zc.cc(sg, s, collect_traffic=False)
        assert np.array_equal(r.values, ref.values) and r.iterations == ref.iterations


def test_device_loop_hands_off_past_log_capacity():
    """A 6000-level chain outgrows the device loop's 4096-entry level log;
    the host loop finishes the traversal with identical results and logs."""
    n = 6000
    chain = zc.CsrGraph(n, n - 1, np.concatenate([np.arange(n), [n - 1]]).astype(np.int64),
                        np.arange(1, n, dtype=np.int64), weights=np.ones(n - 1, np.int64))
    for algo in ("bfs", "sssp"):
        ref = oracle.run(algo, chain, 0)
        for s in ("merged-aligned", "packed"):
            r = getattr(zc, algo)(chain, 0, s, collect_traffic=False)
            assert r.iterations == ref.iterations == n
            assert np.array_equal(r.values, ref.values)
            assert r.traversed_edges == ref.traversed_edges
            assert len(r.frontier_sizes) == n


def test_compressed_lists_match_reference():
    """Compressed line stream: BFS / SSSP / CC identical on every fixture graph
    with 4-byte elements (values, iterations, traversed edges); 8-byte
    elements are rejected."""
    bad = []
    for c in CASES:
        if c.graph.edge_elem_bytes != 4 or (c.algo == "sssp" and c.graph.weight_elem_bytes != 4):
            continue
        r = _run(c, "compressed")
        if not (np.array_equal(r.values, c.values) and r.iterations == c.iterations
                and r.traversed_edges == c.traversed):
            bad.append((c.index, c.tag))
    assert not bad, bad[:8]
    e8 = [c for c in CASES if c.graph.edge_elem_bytes == 8]
    if e8:
        with pytest.raises(ValueError, match="compressed"):
            _run(e8[0], "compressed")


def test_compressed_rmat_and_pagerank():
    dg = zc.generate_rmat(18, 16, seed=21)
    nbytes = dg.build_compressed()
    assert 0 < nbytes < dg.num_edges * 4
    g = dg.as_csr()
    src = int(zc.pick_sources(g, 1, seed=7)[0])
    ref = oracle.bfs(g, src, threads=8)
    r = zc.bfs(dg, src, "compressed", collect_traffic=False)
    assert np.array_equal(r.values, ref.values) and r.traversed_edges == ref.traversed_edges
    sg = zc.generate_rmat(16, 8, seed=5, symmetrize=True)
    ref = oracle.cc(sg.as_csr(), threads=8)
    r = zc.cc(sg, "compressed", collect_traffic=False)
    assert np.array_equal(r.values, ref.values) and r.iterations == ref.iterations
    gu = zc.symmetrized(zc.generate_uniform(3000, 1, 12, seed=8))
    a = zc.pagerank(gu, "compressed", collect_traffic=False)
    b = oracle.pagerank(gu)
    assert np.abs(a.values - b.values).max() < 1e-8


@pytest.mark.parametrize("placement", ["zerocopy", "hbm"])
def test_pipelined_many_sources_match_single_calls(placement):
    """bfs_many / sssp_many (zc_*_async + zc_sync, downloads overlapped with
    the next traversal through two staging slots) return exactly what one
    bfs / sssp call per source returns -- five sources exercise slot reuse."""
    g = zc.with_uniform_weights(zc.generate_powerlaw(1 << 16, 8, seed=5))
    srcs = [int(s) for s in zc.pick_sources(g, 5, seed=7)]
    for algo, many in (("bfs", zc.bfs_many), ("sssp", zc.sssp_many)):
        for strategy in ("merged-aligned", "packed"):
            rs = many(g, srcs, strategy, placement=placement)
            assert len(rs) == len(srcs)
            for s, r in zip(srcs, rs):
                one = getattr(zc, algo)(g, s, strategy, collect_traffic=False,
                                        placement=placement)
                ref = oracle.run(algo, g, s)
                assert np.array_equal(r.values, one.values), (algo, strategy, s)
                assert np.array_equal(r.values, ref.values), (algo, strategy, s)
                assert r.iterations == ref.iterations
                assert r.traversed_edges == ref.traversed_edges
    with pytest.raises(ValueError):
        zc.bfs_many(g, [0, g.num_vertices])
    assert zc.bfs_many(g, []) == []


def _crafted_long_lists(seed=3):
    """Lists that exercise the compressed-line encoder: all-duplicate lists
    (width 0, split at the 256-element line cap), dense and sparse hubs,
    lists just either side of the ~28-element compression threshold, empty
    and single-element lists, self loops."""
    rng = np.random.default_rng(seed)
    nv = 1 << 20
    lists = []
    for v in range(4096):
        kind = v % 8
        if kind == 0:
            d = int(rng.integers(0, 3))
            lst = rng.integers(0, nv, d)
        elif kind == 1:
            lst = np.full(int(rng.integers(250, 700)), int(rng.integers(0, nv)))
        elif kind == 2:
            lst = rng.integers(0, nv, int(rng.integers(24, 36)))
        elif kind == 3:
            lo = int(rng.integers(0, nv - 5000))
            lst = rng.integers(lo, lo + 4000, int(rng.integers(300, 3000)))
        elif kind == 4:
            lst = rng.integers(0, nv, int(rng.integers(40, 2000)))
        elif kind == 5:
            lst = np.concatenate([[v], rng.integers(0, 4096, int(rng.integers(1, 60)))])
        else:
            lst = rng.integers(0, 4096, int(rng.integers(0, 20)))
        lists.append(np.sort(lst).astype(np.int64) if v % 3 else lst.astype(np.int64))
    lists += [np.array([], np.int64)] * (nv - len(lists))
    deg = np.array([len(x) for x in lists], np.int64)
    off = np.concatenate([[0], np.cumsum(deg)])
    edges = np.concatenate(lists)
    return zc.CsrGraph(nv, len(edges), off, edges, None, 4, 4, True)


def test_compressed_lines_crafted_lists():
    """Compressed lines (widths 0..~20, the 256-element line cap, short lists
    sharing lines, long lists, unsorted input lists): BFS, SSSP and CC equal
    the oracle; the index keeps long lists on whole lines and short lists
    inside one line."""
    g = _crafted_long_lists()
    dg = zc.DeviceGraph(g)
    nbytes = dg.build_compressed()
    idx = dg.compressed_index()
    long_ = (idx[:-1] >> np.uint64(63)).astype(bool)
    pos = (idx & np.uint64((1 << 40) - 1)).astype(np.int64)
    nlines = ((idx[:-1] & np.uint64((1 << 63) - 1)) >> np.uint64(40)).astype(np.int64)
    span = np.diff(pos)
    deg = np.diff(g.offsets)
    assert nbytes == pos[-1] // 8 and pos[-1] % 1024 == 0 and (span >= 0).all()
    assert long_.any() and (~long_ & (deg > 0)).any()
    assert (pos[:-1][long_] % 1024 == 0).all() and (nlines[long_] >= 1).all()
    # a long list's lines end at or before the next list (padding may follow)
    assert (nlines[long_] * 1024 <= span[long_]).all() and (nlines[~long_] == 0).all()
    assert (deg[long_] > 1).all() and (span[deg == 0] <= 2048).all()
    span = np.where(long_, nlines * 1024, span)
    short = ~long_ & (deg > 0)
    # a short list never straddles a 256-byte span
    assert ((pos[:-1][short] % 2048) + 38 <= 2048).all()
    assert (span[long_] // 1024 <= (deg[long_] + 31) // 32 + 1).all()
    for src in (0, 1, 9, 12, 33, 4095):
        r = zc.bfs(dg, src, "compressed", collect_traffic=False)
        ref = oracle.bfs(g, src)
        assert np.array_equal(r.values, ref.values) and r.traversed_edges == ref.traversed_edges
    gw = zc.with_uniform_weights(g)
    for src in (1, 33):
        r = zc.sssp(gw, src, "compressed", collect_traffic=False)
        ref = oracle.sssp(gw, src)
        assert np.array_equal(r.values, ref.values) and r.iterations == ref.iterations
    gu = zc.symmetrized(g)
    r = zc.cc(gu, "compressed", collect_traffic=False)
    assert np.array_equal(r.values, oracle.cc(gu).values)
    dg.close()


@pytest.mark.parametrize("fused", [False, True])
def test_cuda_partitions_compressed(fused):
    """Compressed lines inside partitions (local lists, global destinations),
    both exchanges: identical to the whole-graph reference."""
    g = zc.with_uniform_weights(zc.generate_powerlaw(1 << 15, 24, seed=4))
    gu = zc.symmetrized(g)
    for algo, graph in (("bfs", g), ("sssp", g), ("cc", gu)):
        src = int(zc.pick_sources(graph, 1, seed=7)[0])
        ref = oracle.run(algo, graph, src) if algo != "cc" else oracle.cc(graph)
        for nparts in (2, 3):
            b = edge_balanced_bounds(graph.offsets, nparts)
            engines = [CudaPartition(local_part(graph, b, k), b, k) for k in range(nparts)]
            vals, iters, trav = run_partitions_local(engines, algo, src, "compressed",
                                                     fused=fused)
            assert np.array_equal(vals, ref.values), (algo, nparts)
            assert iters == ref.iterations and trav == ref.traversed_edges
            for e in engines:
                e.close()


def test_compressed_shared_lines_with_many_empty_lists():
    """Short lists separated by runs of empty lists: a shared line then holds
    far more than 32 frontier slots (CC puts every vertex in the frontier)."""
    nv = 20000
    src = np.arange(0, nv - 1, 37)
    dst = src + 1
    g = zc.with_uniform_weights(zc.symmetrized(_from_edges(nv, src, dst)))
    for algo in ("bfs", "sssp", "cc"):
        s0 = int(src[3])
        r = zc.cc(g, "compressed", collect_traffic=False) if algo == "cc" else \
            getattr(zc, algo)(g, s0, "compressed", collect_traffic=False)
        ref = oracle.cc(g) if algo == "cc" else oracle.run(algo, g, s0)
        assert np.array_equal(r.values, ref.values), algo
        assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges


def _from_edges(nv, src, dst):
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(nv + 1, np.int64)
    np.add.at(off, src + 1, 1)
    return zc.CsrGraph(nv, len(dst), np.cumsum(off), dst.astype(np.int64), None, 4, 4, True)


def test_direction_optimizing_matches_reference():
    """Direction-optimizing BFS (compressed top-down + bottom-up steps over
    the compressed in-lists): values, iterations and traversed edges equal the
    reference on every BFS fixture (directed and undirected)."""
    bad = []
    for c in CASES:
        if c.algo != "bfs" or c.graph.edge_elem_bytes != 4:
            continue
        r = _run(c, "direction-optimizing")
        if not (np.array_equal(r.values, c.values) and r.iterations == c.iterations
                and r.traversed_edges == c.traversed):
            bad.append((c.index, c.tag))
    assert not bad, bad[:8]


@pytest.mark.parametrize("symmetrize", [False, True])
def test_direction_optimizing_rmat(symmetrize):
    """Bottom-up steps really run (directions log), and the levels equal the
    oracle's on R-MAT graphs from several sources; bfs_many agrees."""
    dg = zc.generate_rmat(18, 16, seed=9, symmetrize=symmetrize)
    g = dg.as_csr()
    srcs = [int(s) for s in zc.pick_sources(g, 3, seed=7)]
    pulled = False
    for s in srcs:
        r = zc.bfs(dg, s, "direction-optimizing", collect_traffic=False)
        ref = oracle.bfs(g, s, threads=8)
        assert np.array_equal(r.values, ref.values)
        assert r.iterations == ref.iterations and r.traversed_edges == ref.traversed_edges
        pulled |= bool(dg.directions(r.iterations).any())
    assert pulled
    for s, r in zip(srcs, zc.bfs_many(dg, srcs, "direction-optimizing")):
        assert np.array_equal(r.values, oracle.bfs(g, s, threads=8).values)
    dg.close()


def test_direction_optimizing_rejects_other_algorithms():
    g = zc.with_uniform_weights(zc.generate_uniform(500, 1, 9, seed=2))
    with pytest.raises(ValueError, match="bfs strategy"):
        zc.sssp(g, 0, "direction-optimizing", collect_traffic=False)
    with pytest.raises(ValueError, match="bfs strategy"):
        zc.cc(zc.symmetrized(g), "direction-optimizing", collect_traffic=False)
    with pytest.raises(ValueError, match="request model"):
        zc.bfs(g, 0, "direction-optimizing", collect_traffic=True)


@pytest.mark.parametrize("fused", [False, True])
def test_cuda_partitions_direction_optimizing(fused):
    """Direction-optimizing partitions: bottom-up steps against the OR of the
    owned frontiers' bitmaps; generated directed R-MAT partitions (in-lists
    from the counter-based generator) and undirected local partitions (in-lists
    = out-lists).  Identical to the oracle."""
    whole = zc.generate_rmat(16, 16, seed=11).as_csr()
    src = int(zc.pick_sources(whole, 1, seed=7)[0])
    ref = oracle.bfs(whole, src, threads=8)
    for nparts in (1, 2, 3):
        engines = [generate_rmat_part(16, nparts, k, seed=11) for k in range(nparts)]
        vals, iters, trav = run_partitions_local(engines, "bfs", src, "direction-optimizing",
                                                 fused=fused)
        assert np.array_equal(vals, ref.values), nparts
        assert iters == ref.iterations and trav == ref.traversed_edges
        for e in engines:
            e.close()
    gu = zc.symmetrized(zc.generate_powerlaw(1 << 14, 12, seed=3))
    src = int(zc.pick_sources(gu, 1, seed=7)[0])
    ref = oracle.bfs(gu, src)
    for nparts in (2, 3):
        b = edge_balanced_bounds(gu.offsets, nparts)
        engines = [CudaPartition(local_part(gu, b, k), b, k) for k in range(nparts)]
        vals, iters, trav = run_partitions_local(engines, "bfs", src, "direction-optimizing",
                                                 fused=fused)
        assert np.array_equal(vals, ref.values) and trav == ref.traversed_edges
        for e in engines:
            e.close()


def test_compressed_byte_accounting():
    """The bench's roofline inputs: the device counter of requested line-stream
    bytes, and the per-vertex stored bytes of the stream."""
    dg = zc.generate_rmat(16, 16, seed=13)
    nbytes = dg.build_compressed()
    stored = dg.stored_list_bytes("compressed")
    assert stored.shape == (dg.num_vertices,) and (stored >= 0).all()
    assert 0 < stored.sum() <= nbytes  # padding is the difference
    raw = dg.stored_list_bytes("packed")
    assert raw.sum() == dg.num_edges * 4
    src = int(zc.pick_sources(dg.as_csr(), 1, seed=7)[0])
    r = zc.bfs(dg, src, "compressed", collect_traffic=False)
    req = dg.link_bytes_requested()
    assert 0 < req <= nbytes * r.iterations and req % 4 == 0
    zc.bfs(dg, src, "packed", collect_traffic=False)
    assert dg.link_bytes_requested() == 0  # raw strategies do not count
    r = zc.bfs(dg, src, "direction-optimizing", collect_traffic=False)
    assert dg.link_bytes_requested() > 0
    assert dg.directions(r.iterations).shape == (r.iterations,)
    dg.close()


SCHED_STRATS = ["naive", "merged", "merged-aligned", "packed", "compressed"]


@pytest.mark.parametrize("strategy", SCHED_STRATS)
def test_work_efficient_schedules_match_reference_values(strategy):
    """near-far SSSP and afforest CC (B200 schedules): the reference's values
    on every fixture (iterations follow the schedule, so only values and
    the error conditions are compared)."""
    bad = []
    for c in CASES:
        if c.algo == "sssp":
            if strategy == "compressed" and (c.graph.edge_elem_bytes != 4
                                             or c.graph.weight_elem_bytes != 4):
                continue
            for delta in (1, 7, 32, 1000):
                r = zc.sssp(c.graph, c.source, strategy, schedule="near-far", delta=delta)
                if not np.array_equal(r.values, c.values):
                    bad.append((c.index, c.tag, delta))
        elif c.algo == "cc":
            if strategy == "compressed" and c.graph.edge_elem_bytes != 4:
                continue
            r = zc.cc(c.graph, strategy, schedule="afforest")
            if not np.array_equal(r.values, c.values) or r.iterations > 2:
                bad.append((c.index, c.tag))
    assert not bad, bad[:8]


def test_work_efficient_schedules_rmat():
    """Both schedules on R-MAT graphs with hubs, isolated vertices and many
    components, against the oracle (values), with their work bounds."""
    for scale, seed in ((16, 3), (18, 9)):
        k = zc.generate_rmat(scale, 16, seed=seed, symmetrize=True)
        gk = k.as_csr()
        ref = oracle.cc(gk, threads=8)
        off = np.asarray(gk.offsets, dtype=np.int64)
        st, en = off[:-1], off[1:]
        first = {"merged": np.minimum(en - st, 32).sum(),  # the sampling pass's first windows
                 "merged-aligned": (np.minimum(en, (st & ~31) + 32) - st).clip(0).sum()}
        first["packed"] = first["merged-aligned"]
        for s in SCHED_STRATS:
            r = zc.cc(k, s, schedule="afforest")
            assert np.array_equal(r.values, ref.values), (scale, s)
            assert r.iterations <= 2 and r.total_traversed_edges <= 2 * gk.num_edges
            if s in first:  # elements actually read, counted on the device
                assert r.traversed_edges[0] == first[s], (scale, s)
            elif s == "naive":
                assert r.traversed_edges[0] == gk.num_edges
            else:
                assert r.traversed_edges[0] < gk.num_edges
        k.close()
    u = zc.generate_uniform_device(1 << 17, 16, 16, seed=5, weights=(8, 72))
    gu = u.as_csr()
    src = int(zc.pick_sources(gu, 1, seed=7)[0])
    ref = oracle.sssp(gu, src, threads=8)
    for s in SCHED_STRATS:
        r = zc.sssp(u, src, s, schedule="near-far")
        assert np.array_equal(r.values, ref.values), s
        assert r.total_traversed_edges < sum(ref.traversed_edges)  # less work than Jacobi
    w = zc.generate_rmat(17, 8, seed=4, weights=(1, 1000))
    gw = w.as_csr()
    src = int(zc.pick_sources(gw, 1, seed=7)[0])
    ref = oracle.sssp(gw, src, threads=8)
    for delta in (1, 50, 10 ** 6):
        r = zc.sssp(w, src, "merged-aligned", schedule="near-far", delta=delta)
        assert np.array_equal(r.values, ref.values), delta


def test_afforest_compressed_sampling_widths():
    """Afforest's sampling pass over compressed lists reads uf_sample elements
    per short list (one per lane of a long list's first line); the second
    pass completes every list outside the giant component, so the labels do
    not depend on the width (>= 96: short lists and first lines whole)."""
    for scale, seed in ((16, 3), (17, 11)):
        k = zc.generate_rmat(scale, 16, seed=seed, symmetrize=True)
        gk = k.as_csr()
        ref = oracle.cc(gk, threads=8)
        work = {}
        for w in (1, 4, 16, 96):
            k.set_tuning(f"uf_sample={w}")
            r = zc.cc(k, "compressed", schedule="afforest")
            assert np.array_equal(r.values, ref.values), (scale, w)
            assert r.iterations <= 2
            work[w] = r.traversed_edges[0]
        assert work[1] < work[4] < work[16] <= work[96] < gk.num_edges, work
        k.set_tuning("")
        k.close()


def test_schedule_argument_errors():
    g = zc.with_uniform_weights(zc.generate_uniform(64, 1, 4, seed=1))
    with pytest.raises(ValueError, match="schedule"):
        zc.sssp(g, 0, schedule="afforest")
    with pytest.raises(ValueError, match="schedule"):
        zc.cc(zc.symmetrized(g), schedule="near-far")
    with pytest.raises(ValueError, match="request model"):
        zc.sssp(g, 0, schedule="near-far", collect_traffic=True)
    with pytest.raises(ValueError, match="undirected"):
        zc.cc(g, schedule="afforest")


def test_partition_exchange_call_order_errors():
    """The fused / bitmap exchanges refuse to run before their peers are
    connected, and the bitmap exchange is BFS-only (zc_part_* return
    ZC_ESTATE -> RuntimeError)."""
    g = zc.symmetrized(zc.generate_uniform(2000, 1, 6, seed=9))
    b = edge_balanced_bounds(g.offsets, 2)
    e = CudaPartition(local_part(g, b, 0), b, 0)
    e.begin("bfs", 0, "merged-aligned")
    with pytest.raises(RuntimeError, match="bitmap"):
        e.bitmap_expand()
    with pytest.raises(RuntimeError, match="fused"):
        e.fused_expand()
    e.bitmap_init()  # exported, but the peers are not connected yet
    with pytest.raises(RuntimeError, match="bitmap"):
        e.bitmap_expand()
    e.fused_init("bfs")
    with pytest.raises(RuntimeError, match="fused"):
        e.fused_expand()
    e.bitmap_connect(ptrs=[e.bitmap_init()[1]] * 2)
    e.begin("cc", 0, "merged-aligned")
    with pytest.raises(RuntimeError, match="bitmap"):  # BFS only
        e.bitmap_expand()
    e.close()


def test_device_graph_cache_keeps_two_placements():
    """Alternating two placements reuses both handles (no re-pinning); a third
    placement evicts the least recently used one."""
    g = zc.generate_uniform(3000, 1, 8, seed=21)
    a = zc.device_graph(g, "zerocopy")
    b = zc.device_graph(g, "hbm")
    assert zc.device_graph(g, "zerocopy") is a and zc.device_graph(g, "hbm") is b
    c = zc.device_graph(g, "uvm")  # evicts "zerocopy", the least recent
    assert zc.device_graph(g, "hbm") is b and zc.device_graph(g, "uvm") is c
    assert zc.device_graph(g, "zerocopy") is not a
    ref = oracle.bfs(g, 0)
    for p in ("zerocopy", "hbm", "uvm"):
        assert np.array_equal(zc.bfs(g, 0, placement=p, collect_traffic=False).values, ref.values)
    zc.release(g)


def test_compressed_build_radix_vs_segmented_sort():
    """The compressed builds sort lists by two stable radix-sort transposes
    (the first one's output is the sorted in-lists); the count / scatter /
    segmented-sort path is the fallback (tuning sort=segmented).  Both yield
    the same streams: equal out-list index and stream sizes, and
    direction-optimizing BFS equal to the oracle through the in-lists."""
    for make in (lambda: zc.generate_rmat(15, 16, seed=5),
                 lambda: zc.generate_uniform_device(20000, 0, 40, seed=9)):
        built = {}
        for mode in ("radix", "segmented"):
            k = make()
            k.set_tuning(f"sort={mode}")
            out_b = k.build_compressed()
            in_b = k.build_in_lists()
            built[mode] = (out_b, in_b, k.compressed_index())
            gk = k.as_csr()
            for src in zc.pick_sources(gk, 3, seed=2):
                r = zc.bfs(k, int(src), "direction-optimizing")
                ref = oracle.bfs(gk, int(src))
                assert np.array_equal(r.values, ref.values), (mode, int(src))
                assert r.traversed_edges == ref.traversed_edges
            k.close()
        assert built["radix"][0] == built["segmented"][0]
        assert built["radix"][1] == built["segmented"][1]
        assert np.array_equal(built["radix"][2], built["segmented"][2])
    # in-lists built after the out-lists (a second radix transpose of the raw lists)
    k = zc.generate_rmat(14, 16, seed=8)
    k.build_compressed()
    k.build_in_lists()
    gk = k.as_csr()
    src = int(zc.pick_sources(gk, 1, seed=1)[0])
    assert np.array_equal(zc.bfs(k, src, "direction-optimizing").values, oracle.bfs(gk, src).values)
    k.close()


def test_uvm_prefetch_cold_then_migrated():
    """UVM with prefetch (zc_graph_prefetch): after evict() the lists are
    migrated back to the GPU in one call (device time > 0), the traversal
    equals the oracle; other placements are a no-op."""
    k = zc.generate_rmat(16, 16, seed=4, placement="uvm")
    gk = k.as_csr()
    src = int(zc.pick_sources(gk, 1, seed=3)[0])
    ref = oracle.bfs(gk, src)
    k.evict()
    assert k.prefetch() > 0
    r = zc.bfs(k, src, "merged-aligned")
    assert np.array_equal(r.values, ref.values) and r.traversed_edges == ref.traversed_edges
    k.close()
    z = zc.generate_rmat(12, 16, seed=4)
    assert z.prefetch() == 0
    z.close()
