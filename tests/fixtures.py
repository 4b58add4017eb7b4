"""Loaders for the committed reference fixtures (tests/golden/, produced by
tests/golden/make_golden.py from the unmodified reference)."""
from __future__ import annotations

import json
import os
import zlib
from dataclasses import dataclass

import numpy as np

from paper_2006_06890_b200 import CsrGraph

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ALGOS = ("bfs", "sssp", "cc")


@dataclass
class Case:
    index: int
    tag: str
    algo: str
    graph: CsrGraph
    source: int
    values: np.ndarray
    iterations: int
    traversed: list


def small_cases() -> list[Case]:
    d = np.load(os.path.join(GOLDEN, "small_graphs.npz"))
    nv, ne, tl = d["nv"], d["ne"], d["trav_len"]
    o_off = np.concatenate(([0], np.cumsum(nv + 1)))
    o_e = np.concatenate(([0], np.cumsum(ne)))
    o_v = np.concatenate(([0], np.cumsum(nv)))
    o_t = np.concatenate(([0], np.cumsum(tl)))
    out = []
    for i in range(nv.size):
        tag = str(d["tag"][i])
        w = d["weights"][o_e[i]:o_e[i + 1]] if d["has_w"][i] else None
        g = CsrGraph(int(nv[i]), int(ne[i]), d["offsets"][o_off[i]:o_off[i + 1]],
                     d["edges"][o_e[i]:o_e[i + 1]], w,
                     edge_elem_bytes=8 if tag.startswith("e8_") else 4,
                     directed=bool(d["directed"][i]))
        out.append(Case(i, tag, ALGOS[int(d["algo"][i])], g, int(d["src"][i]),
                        d["values"][o_v[i]:o_v[i + 1]], int(d["iters"][i]),
                        [int(x) for x in d["trav"][o_t[i]:o_t[i + 1]]]))
    return out


def traffic_cases() -> list[tuple[int, int, np.ndarray]]:
    """(small-case index, strategy id, per-iteration hist [iters, 4])."""
    d = np.load(os.path.join(GOLDEN, "traffic.npz"))
    off = np.concatenate(([0], np.cumsum(d["hist_len"])))
    return [(int(d["idx"][k]), int(d["strategy"][k]), d["hist"][off[k]:off[k + 1]])
            for k in range(d["idx"].size)]


def goldens() -> dict:
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


def crc(a: np.ndarray, dtype: str = "<i8") -> str:
    return f"{zlib.crc32(np.ascontiguousarray(np.asarray(a).astype(dtype)).tobytes()):08x}"


def pagerank_cases():
    """(graph, (damping, max_iters, tol), ranks, iterations, multigraph, dense_err)."""
    d = np.load(os.path.join(GOLDEN, "pagerank.npz"))
    nv = d["nv"]
    ne = np.array([0] * nv.size)
    o_off = np.concatenate(([0], np.cumsum(nv + 1)))
    offs = [d["offsets"][o_off[i]:o_off[i + 1]] for i in range(nv.size)]
    ne = np.array([int(o[-1]) for o in offs])
    o_e = np.concatenate(([0], np.cumsum(ne)))
    o_v = np.concatenate(([0], np.cumsum(nv)))
    out = []
    for i in range(nv.size):
        g = CsrGraph(int(nv[i]), int(ne[i]), offs[i], d["edges"][o_e[i]:o_e[i + 1]])
        dmp, mi, tol = d["args"][i]
        out.append((g, (float(dmp), int(mi), float(tol)), d["ranks"][o_v[i]:o_v[i + 1]],
                    int(d["iters"][i]), bool(d["multi"][i]), float(d["dense_err"][i])))
    return out
