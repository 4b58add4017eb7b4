"""Measured result rows in the reference's CSV schema.

The reference's ``run_experiment`` (report.py:137-207) writes one row per
(strategy, source) with modelled traffic and a priced estimate.  These rows
keep its columns, in its order (report.py:37-44), filled from the B200 run:

* the request histogram columns come from the GPU evaluation of the
  reference's own request model, which is bit-exact with ``frontier_traffic``;
* ``levels_checksum`` is crc32 of the int64 values (report.py:113-114), so
  reference rows and B200 rows join on it;
* the link-model columns (``payload_efficiency`` … ``teps``) and the UVM
  simulator columns are simulator outputs and are left empty;
* measured columns are appended: device time, GTEPS, achieved link GB/s and
  wall time of the call.
"""
from __future__ import annotations

import zlib
from typing import Iterable, Optional

import numpy as np

from .csr import pick_sources
from .traversal import bfs, cc, pagerank, sssp

SCHEMA_LINE = "# emogi-b200 v1"
REFERENCE_COLUMNS = [
    "graph", "algo", "strategy", "source", "iterations", "traversed_edges",
    "requests_total", "h32", "h64", "h96", "h128", "payload_bytes", "dram_bytes",
    "zc_amplification", "mean_request_bytes", "payload_efficiency",
    "efficiency_bound_gibs", "latency_bound_gibs", "effective_gibs",
    "est_seconds", "teps", "uvm_faults", "uvm_pages_evicted",
    "uvm_bytes_migrated", "uvm_amplification", "levels_checksum",
]
MEASURED_COLUMNS = ["placement", "kernel_ms", "gteps", "link_gbs", "call_ms"]
COLUMNS = REFERENCE_COLUMNS + MEASURED_COLUMNS
_SIMULATOR_ONLY = {"payload_efficiency", "efficiency_bound_gibs", "latency_bound_gibs",
                   "effective_gibs", "est_seconds", "teps", "uvm_faults",
                   "uvm_pages_evicted", "uvm_bytes_migrated", "uvm_amplification"}


def checksum(values: np.ndarray) -> str:
    """Same convention as the reference (report.py:113-114)."""
    return f"{zlib.crc32(np.ascontiguousarray(values).tobytes()):08x}"


def _bytes_per_edge(g, algo: str) -> int:
    n = g.edge_elem_bytes
    if algo == "sssp":
        n += g.weight_elem_bytes
    return n


def measure(g, algo: str, strategies: Iterable[str] = ("naive", "merged", "merged-aligned"),
            sources: Optional[Iterable[int]] = None, num_sources: int = 4, *,
            label: str = "graph", placement: str = "zerocopy", traffic: bool = True
            ) -> list[dict]:
    """One row per (strategy, source); cc / pagerank use source -1."""
    if algo in ("bfs", "sssp"):
        srcs = [int(s) for s in (sources if sources is not None
                                 else pick_sources(g, num_sources))]
    else:
        srcs = [-1]
    dataset = g.num_edges * _bytes_per_edge(g, algo)
    rows = []
    for name in strategies:
        model = traffic and name != "packed"  # the model covers the reference's three
        for s in srcs:
            if algo == "bfs":
                r = bfs(g, s, name, collect_traffic=model, placement=placement)
            elif algo == "sssp":
                r = sssp(g, s, name, collect_traffic=model, placement=placement)
            elif algo == "cc":
                r = cc(g, name, collect_traffic=model, placement=placement)
            elif algo == "pr":
                r = pagerank(g, name, collect_traffic=model, placement=placement)
            else:
                raise ValueError(f"unknown algorithm {algo!r}")
            t = r.total_traffic
            row = {c: "" for c in COLUMNS}
            row.update({
                "graph": label, "algo": algo, "strategy": name, "source": s,
                "iterations": r.iterations, "traversed_edges": r.total_traversed_edges,
                "levels_checksum": checksum(r.values), "placement": placement,
                "kernel_ms": r.kernel_ms, "call_ms": r.total_ms,
                "gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9
                if r.kernel_ms else 0.0,
                "link_gbs": r.total_traversed_edges * _bytes_per_edge(g, algo)
                / (r.expand_ms * 1e-3) / 1e9 if r.expand_ms else 0.0,
            })
            if model:
                row.update({
                    "requests_total": t.request_count, "h32": t.hist[32], "h64": t.hist[64],
                    "h96": t.hist[96], "h128": t.hist[128], "payload_bytes": t.payload_bytes,
                    "dram_bytes": t.dram_bytes,
                    "zc_amplification": t.payload_bytes / dataset if dataset else 0.0,
                    "mean_request_bytes": t.mean_request_bytes,
                })
            rows.append(row)
    rows.sort(key=lambda r: (r["graph"], r["algo"], r["strategy"], r["source"]))
    return rows


def _fmt(x) -> str:
    if isinstance(x, float):
        return f"{x:.9g}"
    return str(x)


def write_rows_csv(rows: list[dict], path: str) -> None:
    """CSV with a schema line, the reference's columns, then measured ones."""
    with open(path, "w", newline="") as fh:
        fh.write(SCHEMA_LINE + "\n")
        fh.write(",".join(COLUMNS) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(row.get(c, "")) for c in COLUMNS) + "\n")
