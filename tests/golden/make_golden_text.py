"""Fixtures for load_edge_list_text (reference csr.py:123-177), produced by
the unmodified reference: run here with /root/reference present.

    python tests/golden/make_golden_text.py

Writes tests/golden/edge_list_text.npz: every case's text, the load
arguments, and the reference's CSR (or its error message).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import zcgraph as R  # noqa: E402


def cases():
    rng = np.random.default_rng(2006)
    out = [
        "0 1\n0 2\n1 2\n", "1 2\n0 2\n0 1\n1 0\n", "# header\n% matrix-market style\n\n0 1\n",
        "0 1 5\n1 2 7\n", "0 1 5\n1 2\n", "0 1\nx 2\n", "0 1 # trailing\n", "  # indented\n0 1\n",
        "+5 1\n", "1_000 2\n", "1.0 2\n", "007 3\n", "0 1\r\n2 3\r\n", "0\t1\n", "", "\n\n",
        "0 -1\n", "0 1 -3\n", "0 1 2 3\n", "5 5\n5 5\n", "%\n0 1\n", "0\n",
        f"{2**32} 0\n",
    ]
    for n in (50, 400):  # random multigraphs with self loops, weighted and not
        s = rng.integers(0, n // 3, size=n)
        d = rng.integers(0, n // 3, size=n)
        out.append("".join(f"{a} {b}\n" for a, b in zip(s, d)))
        w = rng.integers(0, 100, size=n)
        out.append("# weighted\n" + "".join(f"{a}\t{b} {c}\n" for a, b, c in zip(s, d, w)))
    return out


def main():
    rows = []
    for i, text in enumerate(cases()):
        path = os.path.join("/tmp", f"zc_golden_text_{i}.txt")
        with open(path, "w") as fh:
            fh.write(text)
        for directed in (True, False):
            for nv in (None, 600):
                entry = {"text": text, "directed": directed, "num_vertices": nv}
                try:
                    g = R.load_edge_list_text(path, directed=directed, num_vertices=nv)
                    entry.update(nv_out=g.num_vertices, offsets=g.offsets.tolist(),
                                 edges=g.edges.tolist(),
                                 weights=None if g.weights is None else g.weights.tolist())
                except ValueError as exc:
                    entry["error"] = str(exc)
                rows.append(entry)
    np.savez_compressed(os.path.join(HERE, "edge_list_text.npz"),
                        cases=np.array(json.dumps(rows)))
    print(len(rows), "cases")


if __name__ == "__main__":
    main()
