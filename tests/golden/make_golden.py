"""Generate the golden fixtures for the parity tests FROM THE REFERENCE ITSELF.

Run in the build container only (needs /root/reference, which does not exist on
the GPU box):

    python tests/golden/make_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``) and
its test oracles' graph generator, runs the reference's ``bfs`` / ``sssp`` /
``cc`` (traversal.py:98-179) and writes:

* ``small_graphs.npz`` -- many small graphs (the acceptance-criterion seeds,
  test_acceptance.py:139-227, plus the known-answer graphs from
  test_traversal.py) together with the reference's values, iteration counts and
  per-iteration traversed-edge counts;
* ``golden.json`` -- crc32 goldens for config 1 (uniform 2^20 deg 16 seed 3,
  SURVEY.md 8c) and for mid-size uniform / power-law graphs, plus byte crcs
  of the generator outputs that pin our generator restatement.

Goldens are tied to numpy's PCG64 stream; numpy version is recorded.
"""
from __future__ import annotations

import json
import os
import sys
import time
import zlib

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import zcgraph as zc  # noqa: E402
from reference import random_csr  # noqa: E402  (reference tests/reference.py:157-174)

HERE = os.path.dirname(os.path.abspath(__file__))


def crc(a: np.ndarray, dtype: str) -> str:
    return f"{zlib.crc32(np.ascontiguousarray(a).astype(dtype).tobytes()):08x}"


def run(algo, g, src=None, strategy=zc.AccessStrategy.MERGED_ALIGNED):
    if algo == "bfs":
        r = zc.bfs(g, src, strategy, collect_traffic=False)
    elif algo == "sssp":
        r = zc.sssp(g, src, strategy, collect_traffic=False)
    else:
        r = zc.cc(g, strategy, collect_traffic=False)
    return r


class Pack:
    """Concatenates many small graphs + results into flat arrays."""

    def __init__(self):
        self.cols = {k: [] for k in ("nv", "ne", "offsets", "edges", "weights", "has_w",
                                      "directed", "algo", "src", "values", "iters",
                                      "trav", "trav_len", "tag")}

    def add(self, tag, algo, g, src, r):
        c = self.cols
        c["nv"].append(g.num_vertices)
        c["ne"].append(g.num_edges)
        c["offsets"].append(np.asarray(g.offsets, np.int64))
        c["edges"].append(np.asarray(g.edges, np.int64))
        has_w = g.weights is not None
        c["has_w"].append(has_w)
        c["weights"].append(np.asarray(g.weights, np.int64) if has_w
                            else np.zeros(g.num_edges, np.int64))
        c["directed"].append(bool(g.directed))
        c["algo"].append({"bfs": 0, "sssp": 1, "cc": 2}[algo])
        c["src"].append(-1 if src is None else int(src))
        c["values"].append(np.asarray(r.values, np.int64))
        c["iters"].append(r.iterations)
        c["trav"].append(np.asarray(r.traversed_edges, np.int64))
        c["trav_len"].append(len(r.traversed_edges))
        c["tag"].append(tag)

    def save(self, path):
        c = self.cols
        np.savez_compressed(
            path,
            nv=np.array(c["nv"], np.int64), ne=np.array(c["ne"], np.int64),
            offsets=np.concatenate(c["offsets"]), edges=np.concatenate(c["edges"]),
            weights=np.concatenate(c["weights"]), has_w=np.array(c["has_w"]),
            directed=np.array(c["directed"]), algo=np.array(c["algo"], np.int8),
            src=np.array(c["src"], np.int64), values=np.concatenate(c["values"]),
            iters=np.array(c["iters"], np.int64), trav=np.concatenate(c["trav"]),
            trav_len=np.array(c["trav_len"], np.int64), tag=np.array(c["tag"]))


def known_answer_graphs():
    """Graphs from test_traversal.py (chain :194-197, path, star :204-208, ...)."""
    def chain(n):
        return zc.CsrGraph(n, n - 1, np.concatenate([np.arange(n), [n - 1]]).astype(np.int64),
                           np.arange(1, n, dtype=np.int64))
    out = []
    out.append(("path4", "bfs", zc.symmetrized(chain(4)), 0))
    star = zc.symmetrized(zc.CsrGraph(7, 6, np.concatenate([[0], np.full(7, 6)]).astype(np.int64),
                                      np.arange(1, 7, dtype=np.int64)))
    out.append(("star6", "bfs", star, 0))
    out.append(("chain3_src2", "bfs", chain(3), 2))
    c3 = chain(3)
    out.append(("wpath", "sssp", zc.CsrGraph(3, 2, c3.offsets, c3.edges, weights=np.array([5, 7])), 0))
    out.append(("twohop", "sssp", zc.CsrGraph(3, 3, np.array([0, 2, 3, 3]), np.array([1, 2, 2]),
                                              weights=np.array([3, 10, 3])), 0))
    out.append(("unreach_sssp", "sssp", zc.CsrGraph(3, 2, c3.offsets, c3.edges,
                                                    weights=np.array([1, 1])), 2))
    out.append(("two_triangles", "cc", zc.CsrGraph(6, 12, np.array([0, 2, 4, 6, 8, 10, 12]),
                                                   np.array([1, 2, 0, 2, 0, 1, 4, 5, 3, 5, 3, 4]),
                                                   directed=False), None))
    out.append(("edgeless", "cc", zc.CsrGraph(5, 0, np.zeros(6, np.int64), np.zeros(0, np.int64),
                                              directed=False), None))
    out.append(("path5_cc", "cc", zc.symmetrized(chain(5)), None))
    out.append(("single_vertex", "bfs", zc.CsrGraph(1, 0, np.zeros(2, np.int64),
                                                    np.zeros(0, np.int64)), 0))
    # self loops + duplicate edges + zero weights
    out.append(("selfloop_dup", "sssp", zc.CsrGraph(4, 6, np.array([0, 3, 4, 6, 6]),
                                                    np.array([0, 1, 1, 2, 3, 3]),
                                                    weights=np.array([0, 4, 2, 0, 1, 1])), 0))
    return out


def small(pack):
    for tag, algo, g, src in known_answer_graphs():
        pack.add(tag, algo, g, src, run(algo, g, src))
    # acceptance criterion 6 stream (test_acceptance.py:139-166): rng(1234)
    rng = np.random.default_rng(1234)
    for _ in range(100):
        g = random_csr(rng, 200)
        src = int(rng.integers(g.num_vertices))
        pack.add("c6_bfs", "bfs", g, src, run("bfs", g, src))
    for _ in range(100):
        g = random_csr(rng, 200, weighted=True)
        src = int(rng.integers(g.num_vertices))
        pack.add("c6_sssp", "sssp", g, src, run("sssp", g, src))
    for _ in range(100):
        g = random_csr(rng, 200, undirected=True)
        pack.add("c6_cc", "cc", g, None, run("cc", g))
    # criterion 8 stream (test_acceptance.py:207-227): rng(4321)
    rng = np.random.default_rng(4321)
    for _ in range(20):
        g = zc.with_uniform_weights(random_csr(rng, 120, allow_empty=False))
        gu = zc.symmetrized(g)
        src = int(zc.pick_sources(g, 1)[0])
        pack.add("c8_bfs", "bfs", g, src, run("bfs", g, src))
        pack.add("c8_sssp", "sssp", g, src, run("sssp", g, src))
        pack.add("c8_cc", "cc", gu, None, run("cc", gu))
    # 8-byte-element graphs (layout differs only in the device element width)
    rng = np.random.default_rng(88)
    for _ in range(10):
        g = zc.with_uniform_weights(random_csr(rng, 150, allow_empty=False))
        g.edge_elem_bytes = 8
        src = int(zc.pick_sources(g, 1)[0])
        pack.add("e8_bfs", "bfs", g, src, run("bfs", g, src))
        pack.add("e8_sssp", "sssp", g, src, run("sssp", g, src))
    # skewed small graphs: long lists cross several 128 B lines
    for seed in range(5):
        g = zc.with_uniform_weights(zc.generate_powerlaw(3000, 12.0, 2.0, seed=seed))
        src = int(zc.pick_sources(g, 1)[0])
        pack.add("pl_bfs", "bfs", g, src, run("bfs", g, src))
        pack.add("pl_sssp", "sssp", g, src, run("sssp", g, src))
        gu = zc.symmetrized(g)
        pack.add("pl_cc", "cc", gu, None, run("cc", gu))


def traffic_goldens():
    """Per-iteration modelled request histograms (collect_traffic=True) of the
    reference for every strategy, on a subset of the small graphs."""
    data = np.load(os.path.join(HERE, "small_graphs.npz"))
    nv, ne = data["nv"], data["ne"]
    o_off = np.concatenate(([0], np.cumsum(nv + 1)))
    o_e = np.concatenate(([0], np.cumsum(ne)))
    idx, strat, hist_len, hists = [], [], [], []
    for i, tag in enumerate(data["tag"]):
        if not (str(tag).startswith(("c8_", "pl_", "e8_")) or i < 11):
            continue
        offs = data["offsets"][o_off[i]:o_off[i + 1]]
        edges = data["edges"][o_e[i]:o_e[i + 1]]
        w = data["weights"][o_e[i]:o_e[i + 1]] if data["has_w"][i] else None
        eb = 8 if str(tag).startswith("e8_") else 4
        g = zc.CsrGraph(int(nv[i]), int(ne[i]), offs, edges, w, edge_elem_bytes=eb,
                        directed=bool(data["directed"][i]))
        algo = int(data["algo"][i])
        src = int(data["src"][i])
        for sid, st in enumerate(zc.AccessStrategy):
            if algo == 0:
                r = zc.bfs(g, src, st)
            elif algo == 1:
                r = zc.sssp(g, src, st)
            else:
                r = zc.cc(g, st)
            h = np.array([[t.hist[s] for s in (32, 64, 96, 128)]
                          for t in r.per_iteration_traffic], np.int64).reshape(-1, 4)
            idx.append(i)
            strat.append(sid)
            hist_len.append(h.shape[0])
            hists.append(h)
    np.savez_compressed(os.path.join(HERE, "traffic.npz"), idx=np.array(idx),
                        strategy=np.array(strat), hist_len=np.array(hist_len),
                        hist=np.concatenate(hists))
    print("traffic goldens:", len(idx), flush=True)


def pagerank_goldens():
    """Reference pagerank (traversal.py:191-249) outputs: the acceptance
    criterion 6 PR stream (its rng(1234) position after the bfs/sssp/cc
    streams, tol 1e-13 / 600 iterations) plus the test_traversal.py cases."""
    import warnings
    from reference import pagerank_dense  # reference tests/reference.py:118-137
    out = {"nv": [], "offsets": [], "edges": [], "ranks": [], "iters": [], "multi": [],
           "dense_err": [], "args": []}

    def add(g, damping=0.85, max_iters=100, tol=1e-6, dense=False):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = zc.pagerank(g, damping=damping, max_iters=max_iters, tol=tol,
                            collect_traffic=False)
        out["nv"].append(g.num_vertices)
        out["offsets"].append(np.asarray(g.offsets, np.int64))
        out["edges"].append(np.asarray(g.edges, np.int64))
        out["ranks"].append(np.asarray(r.values, np.float64))
        out["iters"].append(r.iterations)
        out["multi"].append("multigraph" in r.flags)
        out["args"].append((damping, max_iters, tol))
        out["dense_err"].append(float(np.abs(r.values - pagerank_dense(g)).max()) if dense
                                else -1.0)

    rng = np.random.default_rng(1234)
    for _ in range(100):  # bfs stream
        g = random_csr(rng, 200)
        rng.integers(g.num_vertices)
    for _ in range(100):  # sssp stream
        g = random_csr(rng, 200, weighted=True)
        rng.integers(g.num_vertices)
    for _ in range(100):  # cc stream
        random_csr(rng, 200, undirected=True)
    for _ in range(100):  # pr stream (test_acceptance.py:168-180)
        add(random_csr(rng, 200), tol=1e-13, max_iters=600, dense=True)
    add(zc.symmetrized(zc.CsrGraph(2, 1, np.array([0, 1, 1]), np.array([1]))))
    add(zc.CsrGraph(1, 0, np.zeros(2, np.int64), np.zeros(0, np.int64)))
    add(zc.CsrGraph(2, 2, np.array([0, 2, 2]), np.array([1, 1])))  # multigraph
    add(random_csr(np.random.default_rng(17), 5, allow_empty=False), tol=1e-13, max_iters=500,
        dense=True)
    add(zc.generate_powerlaw(3000, 12.0, 2.0, seed=2), damping=0.9, max_iters=50, tol=1e-9)
    add(zc.generate_uniform(5000, 0, 9, seed=5))
    np.savez_compressed(os.path.join(HERE, "pagerank.npz"),
                        nv=np.array(out["nv"]), offsets=np.concatenate(out["offsets"]),
                        edges=np.concatenate(out["edges"]), ranks=np.concatenate(out["ranks"]),
                        iters=np.array(out["iters"]), multi=np.array(out["multi"]),
                        dense_err=np.array(out["dense_err"]), args=np.array(out["args"]))
    print("pagerank goldens:", len(out["nv"]), "max dense err",
          max(e for e in out["dense_err"]), flush=True)


def result_record(r):
    return {"crc": crc(r.values, "<i8"), "iterations": r.iterations,
            "traversed_edges": [int(x) for x in r.traversed_edges]}


def graph_record(g):
    rec = {"V": g.num_vertices, "E": g.num_edges,
           "offsets_crc_u8": crc(g.offsets, "<u8"),
           "edges_crc_u4": crc(g.edges, "<u4")}
    if g.weights is not None:
        rec["weights_crc_u4"] = crc(g.weights, "<u4")
    return rec


def mid(gold, name, g, src, do_cc=True):
    t = time.time()
    gw = zc.with_uniform_weights(g)
    entry = {"graph": graph_record(gw)}
    entry["bfs"] = result_record(run("bfs", g, src))
    entry["sssp"] = result_record(run("sssp", gw, src))
    entry["src"] = int(src)
    if do_cc:
        gu = zc.symmetrized(g)
        entry["sym_graph"] = graph_record(gu)
        entry["cc"] = result_record(run("cc", gu))
    gold[name] = entry
    print(name, "done in", round(time.time() - t, 1), "s", flush=True)


def main():
    pack = Pack()
    small(pack)
    pack.save(os.path.join(HERE, "small_graphs.npz"))
    print("small graphs:", len(pack.cols["nv"]), flush=True)
    traffic_goldens()
    pagerank_goldens()
    if os.environ.get("GOLDEN_TRAFFIC_ONLY"):
        return

    gold = {"numpy": np.__version__, "generator": {}}
    # generator pins (fast)
    for args in [(1000, 16, 48, 7), (300, 1, 5, 9), (4096, 0, 9, 3), (65536, 16, 16, 3)]:
        g = zc.generate_uniform(args[0], args[1], args[2], seed=args[3])
        gold["generator"][f"uniform_{args[0]}_{args[1]}_{args[2]}_s{args[3]}"] = graph_record(
            zc.with_uniform_weights(g))
    for args in [(100000, 8.0, 2.0, 3), (3000, 12.0, 2.0, 1)]:
        g = zc.generate_powerlaw(args[0], args[1], args[2], seed=args[3])
        gold["generator"][f"powerlaw_{args[0]}_{args[1]}_{args[2]}_s{args[3]}"] = graph_record(g)
    g = zc.generate_uniform(2 ** 10, 2, 6, seed=5)
    gold["generator"]["sym_uniform_1024_2_6_s5"] = graph_record(zc.symmetrized(g))
    gold["pick_sources_1000_16_48_s7"] = [int(x) for x in zc.pick_sources(
        zc.generate_uniform(1000, 16, 48, seed=7), 4)]

    mid(gold, "uniform_2p16_d16", zc.generate_uniform(2 ** 16, 16, 16, seed=3), 0)
    gpl = zc.generate_powerlaw(100000, 8.0, 2.0, seed=3)
    mid(gold, "powerlaw_100k_d8", gpl, int(zc.pick_sources(gpl, 1)[0]))
    # config 1
    g1 = zc.generate_uniform(2 ** 20, 16, 16, seed=3)
    srcs = zc.pick_sources(g1, 4)
    gold["c1_pick_sources"] = [int(x) for x in srcs]
    mid(gold, "c1", g1, 0)
    gold["c1"]["bfs_sources"] = {str(int(s)): result_record(run("bfs", g1, int(s)))
                                 for s in srcs}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(gold, fh, indent=1, sort_keys=True)
    print("wrote golden.json")


if __name__ == "__main__":
    main()
