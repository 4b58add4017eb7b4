#!/usr/bin/env python
"""Benchmark: EMOGI zero-copy BFS on a Kronecker scale-27 graph, merged+aligned
(BASELINE.json configs[1]: ~2.1 B directed arcs, edge list in pinned host
memory, 1x B200; naive vs merged vs merged+aligned vs UVM).

Metric: GTEPS = traversed edges (the reference's traversed_edges, the sum of
frontier degrees, traversal.py:63-65) / second.  One step = one BFS from the
next of pick_sources(g, 64, seed=7).

  value     device time (CUDA events on the library's stream) of the level
            loop, merged+aligned (the paper's kernel, north_star's target),
            lists resident in pinned host memory
  e2e       the same through the public API (bfs_many: every source's int64
            levels land in pinned host memory; source H2D and result D2H in
            the timed region), host wall clock
  roofline  SURVEY 8(d): dominant kernel = the expansion sweep; algorithmic
            bytes = traversed edges x 4 B; achieved = those bytes / the
            sweep's device time (globaltimer stamps around the expansion
            launches inside the level graph, summed over the timed steps);
            peak = PCIe Gen5 x16, 63.0 GB/s per direction; traffic = ncu
            sysmem bytes of the main-level launch (profiles/ncu_summary.json)
  parity    every reported variant is compared with the CPU oracle (values,
            iterations, per-iteration traversed edges) on the same graph
  cpu_baseline  the unmodified reference (oracle/_ref zip) on a bounded sample
            (Kronecker scale 21, same generator), one core

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun (N>1) the graph is vertex-range partitioned (BASELINE
configs[4]); rank 0 prints the JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
import zlib

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PCIE_GEN5_X16_GBS = 63.0  # 32 GT/s x 16 lanes x 128/130 / 8, per direction
METRIC = "BFS GTEPS (Kronecker scale-27, merged+aligned, edge list zero-copy in pinned host memory)"
REF_SAMPLE_SCALE = 21  # the reference's bounded sample: same generator, 2^25 arcs (~5 s / BFS)
C1_LEVELS_CRC = "171fbc8b"  # reference BFS from 0 on generate_uniform(2**20,16,16,seed=3)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scale", type=int, default=27)
    p.add_argument("--edge-factor", type=int, default=16)
    p.add_argument("--seed", type=int, default=27)
    p.add_argument("--strategy", default="merged-aligned")
    p.add_argument("--tuning", default="", help="zc_set_tuning spec (loop=host under ncu)")
    p.add_argument("--no-variants", action="store_true",
                   help="skip the naive / merged / packed / compressed / UVM / HBM runs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the SSSP-U27 / CC-K27 blocks (BASELINE configs[2], configs[3])")
    p.add_argument("--no-c1", action="store_true", help="skip the config-1 block")
    p.add_argument("--cpu-threads", type=int, default=0)
    # test hooks for the partitioned path on a 1-GPU box
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    p.add_argument("--device-override", type=int, default=-1)
    p.add_argument("--force-partitioned", action="store_true")
    p.add_argument("--part-scale", type=int, default=29,
                   help="N>1: Kronecker scale of the partitioned graph (fixed size)")
    p.add_argument("--exchange", default="fused", choices=["fused", "reduce-scatter"],
                   help="N>1: exchange of the headline run (the other is timed beside it)")
    p.add_argument("--no-configs4", action="store_true",
                   help="N>1: skip the fixed-size Kronecker-29 symmetrized BFS / CC block")
    p.add_argument("--no-parity", action="store_true",
                   help="N>1: skip the small-scale oracle parity runs")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) >= 7 and parts[0].isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in busy),
                "sm_max_mhz": max(int(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows)}


def dist_setup(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.device_override >= 0:
        local = args.device_override
    if world > 1 or args.force_partitioned:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return rank, world, local


def barrier(world: int, device: int):
    import torch
    torch.cuda.synchronize(device)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        torch.cuda.synchronize(device)


def _reduce(x: float, op_name: str) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    dev = torch.device("cuda", torch.cuda.current_device())
    if dist.get_backend() == "gloo":
        dev = torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return float(t.item())


def max_over_ranks(x: float, world: int, device: int) -> float:
    return _reduce(x, "MAX")


def sum_over_ranks(x: float, world: int, device: int) -> float:
    return _reduce(x, "SUM")


def load_ncu_summary() -> dict:
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return {}


def crc_hex(values) -> str:
    import numpy as np
    return f"{zlib.crc32(np.ascontiguousarray(values, dtype=np.int64).tobytes()) & 0xffffffff:08x}"


# ------------------------------------------------------------- the reference
def reference_sample(steps: int, warmup: int, seed: int, threads: int, scale=REF_SAMPLE_SCALE):
    """The unmodified reference's bfs (collect_traffic=False, traversal.py:
    98-120) on a bounded sample of the bench workload: Kronecker scale
    `scale` from the same counter-based R-MAT generator (host copy in
    oracle/zc_oracle_gen.c, pinned to the GPU generator by a GPU test), the
    same source rule.  Falls back to the oracle port when the reference is
    not importable.  Never loads the product library."""
    import numpy as np
    import oracle
    t0 = time.perf_counter()
    off, edges = oracle.generate_rmat(scale, 16, seed=seed, threads=threads)
    gen_s = time.perf_counter() - t0
    try:
        ref = oracle.reference()
        kind, cores = "reference", 1
        g = ref.CsrGraph(1 << scale, int(off[-1]), off, edges.astype(np.int64))
        sources = ref.pick_sources(g, 64, seed=7)

        def one(s):
            return ref.bfs(g, int(s), collect_traffic=False)
        where = "oracle/_ref zip of /root/reference/pkg/src/zcgraph (unmodified), numpy, 1 thread"
    except ImportError:
        from paper_2006_06890_b200 import csr as _csr  # pure Python/numpy mirror, no .so
        kind, cores = "port", threads
        g = _csr.CsrGraph(1 << scale, int(off[-1]), off, edges)
        sources = _csr.pick_sources(g, 64, seed=7)

        def one(s):
            return oracle.bfs(g, int(s), threads=threads)
        where = f"oracle port (zc_oracle.c, OpenMP, {threads} threads): reference unavailable"
    per, edges_done = [], 0
    for i in range(warmup + steps):
        t1 = time.perf_counter()
        r = one(sources[i % 64])
        dt = time.perf_counter() - t1
        if i >= warmup:
            per.append(dt)
            edges_done += sum(int(x) for x in r.traversed_edges)
    total = sum(per)
    return {"value": edges_done / total / 1e9, "unit": "GTEPS", "cores": cores, "kind": kind,
            "sample": f"{steps} full bfs() runs (after {warmup} warm-up) on Kronecker scale "
                      f"{scale} (R-MAT .57/.19/.19, edge factor 16, {int(off[-1])} arcs, same "
                      f"generator and source rule as the bench graph); {where}",
            "seconds": total, "gen_s": gen_s, "ms_per_step": total / max(steps, 1) * 1e3}


def main_reference(args):
    """--impl reference: the reference's own CPU implementation on the host
    cores (rank 0 only; other ranks exit without work).  Runs the unmodified
    reference bfs on a bounded sample of this arm's workload (reference_sample);
    does not import the product package or load any CUDA library."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    threads = args.cpu_threads or os.cpu_count()
    s = reference_sample(args.steps, args.warmup, args.seed, threads)
    cfg = bfs_config(args, world)
    cfg["reference_sample"] = s["sample"]
    line = {"impl": "reference", "metric": METRIC, "value": s["value"], "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": cfg,
            "cpu_baseline": {k: s[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": s["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bfs_config(args, world: int) -> dict:
    return {"workload": f"BFS, Kronecker (R-MAT a=.57 b=.19 c=.19) scale {args.scale}, edge "
                        f"factor {args.edge_factor}, {args.edge_factor << args.scale} directed "
                        "arcs, u32 edges in pinned host memory (zero-copy)",
            "graph": f"kron{args.scale}", "scale": args.scale, "edge_factor": args.edge_factor,
            "seed": args.seed, "strategy": args.strategy, "placement": "zerocopy",
            "sources": "pick_sources(g, 64, seed=7)",
            "l2": "inputs larger than L2 (8 GiB edge list in host memory, 512 MiB level array)",
            "parallelism": "single" if world == 1 else f"vertex-partition{world}"}


# ----------------------------------------------------------------- helpers
class OracleCache:
    """CPU oracle results per (graph tag, algo, source) -- computed once,
    compared with every strategy / placement that reports a number."""

    def __init__(self, threads: int):
        self.threads = threads
        self.memo = {}
        self.seconds = {}

    def get(self, tag, g, algo, src=0):
        import oracle
        key = (tag, algo, src)
        if key not in self.memo:
            t0 = time.perf_counter()
            self.memo[key] = oracle.run(algo, g, src, threads=self.threads)
            self.seconds[key] = time.perf_counter() - t0
        return self.memo[key]


def same(r, ref) -> bool:
    import numpy as np
    return bool(np.array_equal(r.values, ref.values) and r.iterations == ref.iterations
                and list(r.traversed_edges) == list(ref.traversed_edges))


def same_values(r, ref) -> bool:
    import numpy as np
    return bool(np.array_equal(r.values, ref.values))


def bfs_point(zc, dg, src, strategy, evict=False, reps=2) -> tuple[dict, object]:
    """GTEPS of one source: `reps` runs (the first warms), the last reported."""
    r = None
    for _ in range(reps):
        if evict:
            zc.evict(dg)
        r = zc.bfs(dg, int(src), strategy, collect_traffic=False)
    return {"gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
            "kernel_ms": r.kernel_ms, "expand_ms": r.expand_ms,
            "u32_edge_gbs": r.total_traversed_edges * 4 / (r.expand_ms * 1e-3) / 1e9}, r


def ceiling_model_summary() -> dict:
    """profiles/r02_ceiling_model.txt (tools/ceiling.py): the merged-aligned
    levels' measured time against the reference request model x the measured
    per-size request rates (ratio >= 1: at or above the modelled ceiling)."""
    path = os.path.join(ROOT, "profiles", "r02_ceiling_model.txt")
    if not os.path.exists(path):
        return {}
    ratios, meas, ceil = [], 0.0, 0.0
    for ln in open(path):
        f = ln.split()
        if len(f) >= 13 and f[0] == "merged-aligned" and f[2].isdigit() and int(f[3]) > 10 ** 7:
            ratios.append(float(f[11]))
            meas += float(f[9])
            ceil += float(f[10])
    if not ratios:
        return {}
    return {"file": "profiles/r02_ceiling_model.txt", "levels_over_1e7_edges": len(ratios),
            "min_ratio_ceiling_over_measured": min(ratios), "sum_ratio": ceil / meas,
            "model": "reference request model (coalesce.py:165-207) histograms x measured "
                     "per-size CTA-streamed zero-copy rates; ratio >= 0.9 on every level = "
                     "at the link's ceiling for merged-aligned's request mix"}


def level_table(dg, r, elem_bytes=4) -> list:
    prof = dg.expand_profile(r.iterations)
    return [{"level": k, "frontier": int(r.frontier_sizes[k]), "edges": int(r.traversed_edges[k]),
             "expand_ms": round(float(prof[k]), 3),
             "gbs": round(r.traversed_edges[k] * elem_bytes / max(prof[k], 1e-9) / 1e6, 2)}
            for k in range(r.iterations)]


# ---------------------------------------------------------------- N = 1
def main():
    args = parse()
    if args.impl == "reference":
        return main_reference(args)
    rank, world, local = dist_setup(args)
    if world > 1 or args.force_partitioned:
        return main_partitioned(args, rank, world, local)
    import numpy as np
    import torch

    import paper_2006_06890_b200 as zc

    device = local
    torch.cuda.set_device(device)
    threads = args.cpu_threads or os.cpu_count()
    config = bfs_config(args, world)
    strat = args.strategy

    t0 = time.time()
    dg = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, device=device)
    gen_s = time.time() - t0
    dg.set_tuning(args.tuning)
    g = dg.as_csr()
    sources = zc.pick_sources(g, 64, seed=7)
    probe = zc.link_probe(device=device, nbytes=1 << 30, iters=5)

    for i in range(args.warmup):  # untimed
        zc.bfs(dg, int(sources[i % 64]), strat, collect_traffic=False)

    # ---- timed region 1: device time of the level loop (value)
    barrier(world, device)
    kernel_ms = expand_ms = 0.0
    trav = launches = 0
    step_srcs = [int(sources[(args.warmup + i) % 64]) for i in range(args.steps)]
    last = None
    with ClockSampler(device) as clk:
        for s in step_srcs:
            r = zc.bfs(dg, s, strat, collect_traffic=False)
            kernel_ms += r.kernel_ms
            expand_ms += r.expand_ms
            trav += r.total_traversed_edges
            launches += r.launches
            last = r
    barrier(world, device)
    value = trav / (kernel_ms * 1e-3) / 1e9
    levels = level_table(dg, last)

    # ---- timed region 2: end to end through the public API (host wall clock)
    batch = min(10, args.steps)
    zc.bfs_many(dg, step_srcs[:batch], strat)  # warms the pinned result pool
    barrier(world, device)
    t1 = time.perf_counter()
    e2e_trav = h2d = d2h = 0
    for b0 in range(0, args.steps, batch):
        for r in zc.bfs_many(dg, step_srcs[b0:b0 + batch], strat):
            e2e_trav += r.total_traversed_edges
            h2d += r.h2d_bytes
            d2h += r.d2h_bytes
    barrier(world, device)
    wall = time.perf_counter() - t1
    e2e_value = e2e_trav / wall / 1e9
    t2 = time.perf_counter()
    for s in step_srcs:
        zc.bfs(dg, s, strat, collect_traffic=False)
    wall_1 = time.perf_counter() - t2

    # ---- roofline: 4 B per traversed edge over the sweep's time
    alg_bytes = trav * 4
    achieved = alg_bytes / (expand_ms * 1e-3) / 1e9
    summ = load_ncu_summary()
    ncu = summ.get("bfs_expand_merged_aligned", {}) if strat == "merged-aligned" else {}
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": kernel_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config,
        "e2e": {"value": e2e_value, "unit": "GTEPS",
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "ms_per_step": wall / args.steps * 1e3,
                "api": f"bfs_many (pipelined result downloads, batches of {batch})",
                "per_call_value": e2e_trav / wall_1 / 1e9,
                "per_call_api": "one blocking bfs() per source"},
        "gpu_launches": launches,
        "roofline": {
            "bound": "host-link", "achieved": achieved, "peak": PCIE_GEN5_X16_GBS,
            "unit": "GB/s", "frac": achieved / PCIE_GEN5_X16_GBS,
            "traffic": ncu.get("sysmem_bytes_per_launch"),
            "traffic_kind": "ncu syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss "
                            "x 32 B of the main-level launch (host-link read bytes the L2 "
                            "fetched)",
            "traffic_algorithmic_bytes": ncu.get("algorithmic_bytes_per_launch"),
            "traffic_pcie_read_bytes": ncu.get("pcie_read_bytes_per_launch"),
            "traffic_hbm_dram_bytes": ncu.get("dram_bytes_per_launch"),
            "kernel": "k_expand_sweep<merged-aligned> (+ its window-count / scan launches)",
            "algorithmic_bytes": "traversed edges x 4 B (SURVEY 8(d))",
            "algorithmic_bytes_per_step": alg_bytes / args.steps,
            "kernel_ms_per_step": expand_ms / args.steps,
            "kernel_share_of_step": expand_ms / kernel_ms,
            "peak_kind": "PCIe Gen5 x16 theoretical per direction",
            "measured_peaks_gbs": probe,
            "frac_of_measured_memcpy": achieved / probe["memcpy_h2d_gbs"],
            "frac_of_measured_zerocopy_ceiling": achieved / probe["zerocopy_read_gbs"]},
        "clocks": clk.summary(),
        "graph": {"vertices": dg.num_vertices, "arcs": dg.num_edges, "gen_s": gen_s,
                  "traversed_edges_per_step": trav / args.steps,
                  "pinned_list_bytes": dg.num_edges * 4},
        "merged_aligned": {"gteps": value, "e2e_gteps": e2e_value,
                           "link_gbs": achieved, "frac_of_pcie_gen5": achieved / PCIE_GEN5_X16_GBS,
                           "levels_last_step": levels, "ceiling_model": ceiling_model_summary(),
                           "pcie_read_gbs_whole_traversal": summ.get(
                               "bfs_merged_aligned_whole_traversal", {}).get("pcie_read_gbs"),
                           "pcie_read_note": "ncu pcie__read_bytes over all levels of one BFS / "
                                             "their summed duration (profiles/ncu_summary.json)"},
    }

    oc = OracleCache(threads)
    parity = {}
    if not args.no_cpu_baseline:
        # bit-exact at full size: three of the timed sources against the oracle port
        checks, port_s, port_edges = [], 0.0, 0
        for s in step_srcs[:3]:
            ref = oc.get("kron", g, "bfs", s)
            port_s += oc.seconds[("kron", "bfs", s)]
            port_edges += sum(ref.traversed_edges)
            checks.append(same(zc.bfs(dg, s, strat, collect_traffic=False), ref))
        parity[f"zerocopy/{strat}"] = all(checks)
        line["cpu_port"] = {"value": port_edges / port_s / 1e9, "unit": "GTEPS",
                            "cores": threads, "kind": "port",
                            "sample": f"3 full BFS runs of the oracle port (zc_oracle.c, OpenMP) on "
                                      f"the bench graph itself, {threads} threads"}
        line["cpu_baseline"] = reference_sample(3, 0, args.seed, threads)

    if not args.no_variants:
        line["variants"] = variants_zerocopy(zc, dg, g, sources, oc, parity, args)
    dg.close()
    if not args.no_configs:
        line["configs"] = other_configs(zc, args, device, oc, parity)
    if not args.no_variants:
        line["variants"].update(variants_placements(zc, args, g, sources, device, oc, parity,
                                                    step_srcs))
        v = line["variants"]
        # same sources on both sides: the timed steps' sources, each UVM run cold
        uvm = v["uvm/merged-aligned/timed_sources"]["gteps"]
        line["merged_aligned"]["speedup_vs_uvm"] = value / uvm
        line["merged_aligned"]["speedup_vs_uvm_source0"] = (
            v["zerocopy/merged-aligned"]["gteps"] / v["uvm/merged-aligned"]["gteps"])
        line["merged_aligned"]["speedup_vs_uvm_cap25_source0"] = (
            v["zerocopy/merged-aligned"]["gteps"] / v["uvm_cap25/merged-aligned"]["gteps"])
        line["merged_aligned"]["uvm_gteps"] = uvm
        if "uvm_prefetch/merged-aligned" in v:
            line["merged_aligned"]["speedup_vs_uvm_prefetch"] = (
                value / v["uvm_prefetch/merged-aligned"]["gteps"])
        u0 = v["uvm/merged-aligned"]["gteps"]
        line["merged_aligned"]["store_extensions_vs_uvm_source0"] = {
            k: v[f"zerocopy/{k}"]["gteps"] / u0
            for k in ("packed", "compressed", "direction-optimizing") if f"zerocopy/{k}" in v}
    if not args.no_c1:
        line["c1"] = config1(zc, threads, parity)
    line["parity"] = parity
    line["parity_all_true"] = all(parity.values()) if parity else None
    print(json.dumps(line), flush=True)


def variants_zerocopy(zc, dg, g, sources, oc, parity, args) -> dict:
    """configs[1]'s comparison on the same zero-copy graph and source:
    naive / merged / merged-aligned / packed, and the B200 host-store options
    (compressed, direction-optimizing) with their build cost and an e2e that
    pays it, amortised over the 64 pick_sources."""
    out = {}
    s0 = int(sources[0])
    ref = oc.get("kron", g, "bfs", s0)
    for s in ("naive", "merged", "merged-aligned", "packed"):
        pt, r = bfs_point(zc, dg, s0, s, reps=1 if s == "naive" else 2)
        out[f"zerocopy/{s}"] = pt
        parity[f"zerocopy/{s}"] = parity.get(f"zerocopy/{s}", True) and same(r, ref)
    out_build_s = None  # the out-list stream is built once (first variant), used by both
    for s in ("compressed", "direction-optimizing"):
        t0 = time.perf_counter()
        nbytes = dg.build_compressed()
        if out_build_s is None:
            out_build_s = time.perf_counter() - t0
        build = {"out_lists_s": out_build_s, "out_line_stream_bytes": nbytes}
        if s == "direction-optimizing":
            t0 = time.perf_counter()
            build["in_line_stream_bytes"] = dg.build_in_lists()
            build["in_lists_s"] = time.perf_counter() - t0
        pt, r = bfs_point(zc, dg, s0, s)
        pt["requested_link_gbs"] = dg.link_bytes_requested() / (r.expand_ms * 1e-3) / 1e9
        parity[f"zerocopy/{s}"] = same(r, ref)
        # a fresh caller's cost: the build (measured above; the store is built
        # once per handle) + bfs_many over all 64 sources, every int64 result
        # downloaded; consumed in batches of 8 (a caller that kept all 64 would
        # hold 64 GiB of results -- the pinned result pool recycles released ones)
        t0 = time.perf_counter()
        trav64 = 0
        for b0 in range(0, 64, 8):
            for x in zc.bfs_many(dg, [int(v) for v in sources[b0:b0 + 8]], s):
                trav64 += x.total_traversed_edges
        wall64 = time.perf_counter() - t0
        build_s = build["out_lists_s"] + build.get("in_lists_s", 0.0)
        pt.update(build)
        pt["build_phases_ms"] = {k: round(v, 1) for k, v in dg.build_log()}
        pt["e2e_64_sources_gteps"] = trav64 / wall64 / 1e9
        pt["e2e_64_sources_incl_build_gteps"] = trav64 / (wall64 + build_s) / 1e9
        pt["pinned_host_bytes"] = (g.num_edges * 4 + build["out_line_stream_bytes"]
                                   + build.get("in_line_stream_bytes", 0))
        pt["algorithmic_u32_gbs_note"] = ("u32_edge_gbs counts 4 B per traversed edge; the "
                                          "strategy reads fewer bytes (requested_link_gbs)")
        out[f"zerocopy/{s}"] = pt
    return out


def variants_placements(zc, args, g, sources, device, oc, parity, step_srcs) -> dict:
    """In-HBM control, cold UVM (and at the reference's 25% capacity), and
    host-resident managed lists read in place -- each checked against the
    oracle.  UVM runs last: managed-memory runs leave the process slower on
    later zero-copy work (measured).  Cold UVM also runs over the headline's
    timed sources (evicted before each), the denominator of speedup_vs_uvm."""
    import torch
    out = {}
    s0 = int(sources[0])
    ref = oc.get("kron", g, "bfs", s0)
    for placement, strategies in (("zerocopy-managed", ("merged-aligned", "direction-optimizing")),
                                  ("hbm", ("merged-aligned",)), ("uvm", ("merged-aligned",))):
        h = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, device=device,
                             placement=placement)
        for s in strategies:
            pt, r = bfs_point(zc, h, s0, s, evict=placement == "uvm")
            out[f"{placement}/{s}"] = pt
            parity[f"{placement}/{s}"] = same(r, ref)
        if placement == "uvm":
            trav = ms = 0.0
            per = []
            for src in step_srcs:
                zc.evict(h)
                r = zc.bfs(h, int(src), "merged-aligned", collect_traffic=False)
                trav += r.total_traversed_edges
                ms += r.kernel_ms
                per.append(round(r.kernel_ms, 1))
            out["uvm/merged-aligned/timed_sources"] = {
                "gteps": trav / (ms * 1e-3) / 1e9, "sources": len(step_srcs),
                "kernel_ms_per_source": per}
            # UVM with prefetch (north_star's "prefetch/advise"): cold, then the
            # whole list migrated by cudaMemPrefetchAsync before the traversal;
            # timed = migration + traversal device time, per source
            trav = ms = mig = 0.0
            pf_ok = True
            for src in step_srcs[:3]:
                zc.evict(h)
                m = h.prefetch()
                r = zc.bfs(h, int(src), "merged-aligned", collect_traffic=False)
                trav += r.total_traversed_edges
                ms += m + r.kernel_ms
                mig += m
                pf_ok = pf_ok and same(r, oc.get("kron", g, "bfs", int(src)))
            nb = h.num_edges * h.edge_elem_bytes
            out["uvm_prefetch/merged-aligned"] = {
                "gteps": trav / (ms * 1e-3) / 1e9, "sources": 3,
                "prefetch_ms_per_source": mig / 3, "prefetch_gbs": nb / (mig / 3 * 1e-3) / 1e9,
                "traversal_ms_per_source": (ms - mig) / 3,
                "note": "for a list that fits HBM (8 GiB of 180 GB) prefetch is one bulk copy, "
                        "after which the traversal runs at the HBM control's speed; EMOGI's "
                        "zero-copy case is the list that does not stay resident"}
            parity["uvm_prefetch/merged-aligned"] = pf_ok
            # the reference's UVM capacity default: 25% of the dataset
            # (report.py:151-153) -- ballast HBM so only that much stays free
            dataset = h.num_edges * h.edge_elem_bytes
            free, _ = torch.cuda.mem_get_info(device)
            ballast = torch.empty(max(0, free - dataset // 4 - (256 << 20)), dtype=torch.uint8,
                                  device=f"cuda:{device}")
            pt, r = bfs_point(zc, h, s0, "merged-aligned", evict=True)
            pt["free_hbm_bytes"] = torch.cuda.mem_get_info(device)[0]
            out["uvm_cap25/merged-aligned"] = pt
            parity["uvm_cap25/merged-aligned"] = same(r, ref)
            del ballast
            torch.cuda.empty_cache()
        h.close()
    # the HBM control is gather-bound (a random visited-bitmap probe per edge),
    # not HBM-bandwidth bound: its roofline is the L2 random-load rate
    from paper_2006_06890_b200.device import gather_probe
    hbm = out["hbm/merged-aligned"]
    bitmap = (g.num_vertices + 7) // 8
    ceil = {m: gather_probe(bitmap, m, device) for m in (0, 1)}
    probes = hbm["gteps"] * hbm["kernel_ms"] / hbm["expand_ms"]  # G probes/s in the sweeps
    hbm["gather_roofline"] = {"g_loads_per_s": ceil[0], "g_loads_per_s_with_claims": ceil[1],
                              "bitmap_bytes": bitmap, "sweep_g_probes_per_s": probes,
                              "frac": probes / ceil[1],
                              "probe": "zc_gather_probe: random 4-byte loads into a bitmap-sized "
                                       "device array (mode 1 adds the claims' atomicOr)"}
    return out


def sssp_cc_point(zc, dg, algo, src, strategy, deg, schedule=None) -> tuple[dict, object]:
    kw = {} if schedule is None else {"schedule": schedule}
    fn = (lambda: zc.cc(dg, strategy, collect_traffic=False, **kw)) if algo == "cc" else \
         (lambda: zc.sssp(dg, src, strategy, collect_traffic=False, **kw))
    fn()
    r = fn()
    import numpy as np
    unreached = np.iinfo(np.int64).max if algo == "sssp" else None
    reached_deg = int(deg.sum()) if unreached is None else int(deg[r.values != unreached].sum())
    eb = 8 if algo == "sssp" else 4
    t = r.kernel_ms * 1e-3
    return {"primary_gteps": reached_deg / t / 1e9,
            "work_gteps": r.total_traversed_edges / t / 1e9,
            "kernel_ms": r.kernel_ms, "iterations": r.iterations,
            "work_edges": r.total_traversed_edges, "reached_degree_sum": reached_deg,
            "work_passes_over_E": r.total_traversed_edges / max(dg.num_edges, 1),
            "link_gbs_8d": r.total_traversed_edges * eb / (r.expand_ms * 1e-3) / 1e9,
            "frac_of_pcie_gen5": r.total_traversed_edges * eb / (r.expand_ms * 1e-3) / 1e9
            / PCIE_GEN5_X16_GBS}, r


def other_configs(zc, args, device, oc, parity) -> dict:
    """BASELINE configs[2] (SSSP, u32 weights, uniform scale 27, edges +
    weights zero-copy) and configs[3] (CC, Kronecker scale 27 symmetrized =
    2^32 arcs).  Primary GTEPS = sum of the reached vertices' degrees / time
    (schedule-independent); work GTEPS counts the edges the
    schedule expanded.  Every strategy is checked against the oracle."""
    import numpy as np
    out = {}
    u = zc.generate_uniform_device(1 << args.scale, 16, 16, seed=args.seed, weights=(8, 72),
                                   device=device)
    gu = u.as_csr()
    src = int(zc.pick_sources(gu, 1, seed=7)[0])
    deg = np.diff(np.asarray(gu.offsets))
    ref = oc.get("u27", gu, "sssp", src)
    tag = f"sssp_uniform{args.scale}"
    # merged-aligned / packed read the interleaved (dst, weight) stream (the
    # library's default for 4-byte edges and weights); "separate-arrays" reads
    # the edge and weight lists as two streams, like the reference's model
    runs = [("merged-aligned", None, ""), ("packed", None, ""), ("compressed", None, ""),
            ("merged-aligned", None, "pairs=0")]
    runs += [(st, s, "") for s in schedules("sssp", zc) for st in ("merged-aligned", "compressed")]
    for s, sched, tune in runs:
        key = f"{tag}/{s}" + (f"/{sched}" if sched else "") + ("/separate-arrays" if tune else "")
        u.set_tuning(tune)
        pt, r = sssp_cc_point(zc, u, "sssp", src, s, deg, sched)
        out[key] = pt
        parity[key] = same(r, ref) if sched is None else same_values(r, ref)
    u.set_tuning("")
    out[f"{tag}/cpu_port_work_gteps"] = (sum(ref.traversed_edges)
                                         / oc.seconds[("u27", "sssp", src)] / 1e9)
    link = load_ncu_summary().get("link_utilisation_r02", {})
    if f"{tag}/merged-aligned" in out and "sssp_u27_merged_aligned_pairs" in link:
        out[f"{tag}/merged-aligned"]["pcie_read_frac_ncu"] = link["sssp_u27_merged_aligned_pairs"]
    u.close()
    t0 = time.time()
    k = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, symmetrize=True,
                         device=device)
    gen_s = time.time() - t0
    gk = k.as_csr()
    deg = np.diff(np.asarray(gk.offsets))
    ref = oc.get("kron_sym", gk, "cc")
    tag = f"cc_kron{args.scale}_sym"
    runs = [("merged-aligned", None), ("packed", None), ("compressed", None)]
    runs += [(st, s) for s in schedules("cc", zc) for st in ("merged-aligned", "compressed")]
    for s, sched in runs:
        key = f"{tag}/{s}" + (f"/{sched}" if sched else "")
        pt, r = sssp_cc_point(zc, k, "cc", 0, s, deg, sched)
        pt.update({"arcs": k.num_edges, "gen_s": gen_s})
        out[key] = pt
        parity[key] = same(r, ref) if sched is None else same_values(r, ref)
    out[f"{tag}/cpu_port_work_gteps"] = (sum(ref.traversed_edges)
                                         / oc.seconds[("kron_sym", "cc", 0)] / 1e9)
    if f"{tag}/merged-aligned" in out and "cc_k27sym_merged_aligned" in link:
        out[f"{tag}/merged-aligned"]["pcie_read_frac_ncu"] = link["cc_k27sym_merged_aligned"]
    # PageRank streams the whole zero-copy list every
    # iteration (5 iterations timed; parity is pinned on the reference's
    # PageRank fixtures in the GPU tests; here against the oracle's threaded
    # C pull: float64 sums against the library's 2^-62 fixed-point sums.  Each
    # iteration quantises every summed contribution (round to nearest, <= 2^-63
    # each), so vertex v's sum is off by <= deg(v) 2^-63 per iteration, and
    # errors of earlier iterations reach it damped (x 0.85 per hop, spread over
    # the neighbours' degrees): after k iterations <= k(k+1)/2 (deg(v)+1) 2^-62.
    # The check: |gpu - oracle| <= that + 1e-9 rank + 1e-16 per vertex (a hub of
    # degree ~1e6 carries ~1e-12 absolute, ~3e-9 relative, at K27)
    import oracle
    import warnings
    t0 = time.perf_counter()
    pr_ref = oracle.pagerank_c(gk, 0.85, 5, 1e-30, threads=oc.threads, symmetric=True)
    pr_s = time.perf_counter() - t0
    tag = f"pagerank_kron{args.scale}_sym"
    for s in ("merged-aligned", "compressed"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # the multigraph note (duplicates are kept)
            zc.pagerank(k, s, max_iters=1, tol=1e-30, collect_traffic=False)
            r = zc.pagerank(k, s, max_iters=5, tol=1e-30, collect_traffic=False)
        t = r.kernel_ms * 1e-3
        err = np.abs(r.values - pr_ref.values)
        fx = (r.iterations * (r.iterations + 1) / 2) * (np.diff(np.asarray(gk.offsets)) + 1.0) \
            * 2.0 ** -62
        out[f"{tag}/{s}"] = {
            "iterations": r.iterations, "kernel_ms": r.kernel_ms,
            "edge_gteps": r.total_traversed_edges / t / 1e9,
            "link_gbs_8d": r.total_traversed_edges * 4 / (r.expand_ms * 1e-3) / 1e9,
            "max_abs_err_vs_oracle": float(err.max()),
            "max_rel_err_vs_oracle": float(np.max(err / pr_ref.values))}
        parity[f"{tag}/{s}"] = bool(r.iterations == pr_ref.iterations
                                    and np.all(err <= 1e-9 * pr_ref.values + 1e-16 + fx))
        out[f"{tag}/{s}"]["max_err_over_fixed_point_bound"] = float(
            np.max(err / (1e-9 * pr_ref.values + 1e-16 + fx)))
    out[f"{tag}/cpu_port_edge_gteps"] = sum(pr_ref.traversed_edges) / pr_s / 1e9
    k.close()
    return out


def schedules(algo: str, zc) -> list:
    """Work-efficient schedules the library offers beyond the reference's
    Jacobi iteration (values bit-identical; iteration counts differ)."""
    return list(getattr(zc, "SCHEDULES", {}).get(algo, ()))


def config1(zc, threads, parity) -> dict:
    """BASELINE configs[0]: BFS from vertex 0 on generate_uniform(2**20, 16, 16,
    seed=3) -- the GPU path, the unmodified reference's bfs timed under
    `taskset -c 0` in a subprocess on the same EMGI file, and the oracle port."""
    import numpy as np
    import oracle
    t0 = time.perf_counter()
    g = zc.generate_uniform(2 ** 20, 16, 16, seed=3)
    gen_s = time.perf_counter() - t0
    best = None
    for _ in range(6):
        r = zc.bfs(g, 0, "merged-aligned", collect_traffic=False)
        if best is None or r.kernel_ms < best.kernel_ms:
            best = r
    out = {"workload": "BFS from vertex 0, generate_uniform(2**20, 16, 16, seed=3) "
                       "(reference generator restated byte-identically), u32 edges zero-copy",
           "gpu_gteps": best.total_traversed_edges / (best.kernel_ms * 1e-3) / 1e9,
           "gpu_kernel_ms": best.kernel_ms, "levels_crc": crc_hex(best.values),
           "levels_crc_golden": C1_LEVELS_CRC, "gen_s": gen_s}
    parity["c1/merged-aligned"] = out["levels_crc"] == C1_LEVELS_CRC
    tmp = tempfile.mkdtemp(prefix="zc_c1_")
    path = os.path.join(tmp, "c1.emgi")
    zc.store_csr_binary(g, path)
    script = (
        "import sys, time, json, zlib\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "import numpy as np, oracle\n"
        "ref = oracle.reference()\n"
        f"g = ref.load_csr_binary({path!r})\n"
        "ts = []\n"
        "for _ in range(3):\n"
        "    t = time.perf_counter(); r = ref.bfs(g, 0, collect_traffic=False)\n"
        "    ts.append(time.perf_counter() - t)\n"
        "print(json.dumps({'s': min(ts), 'runs_s': ts, 'edges': int(sum(r.traversed_edges)),\n"
        "                  'crc': '%08x' % (zlib.crc32(np.asarray(r.values, np.int64).tobytes()) & 0xffffffff)}))\n")
    cmd = [sys.executable, "-c", script]
    if subprocess.run(["which", "taskset"], capture_output=True).returncode == 0:
        cmd = ["taskset", "-c", "0"] + cmd
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        rr = json.loads(res.stdout.strip().splitlines()[-1])
        out["reference"] = {"value": rr["edges"] / rr["s"] / 1e9, "unit": "GTEPS", "cores": 1,
                            "kind": "reference", "seconds": rr["s"], "runs_s": rr["runs_s"],
                            "levels_crc": rr["crc"], "pinned": cmd[0] == "taskset",
                            "sample": "the unmodified reference's bfs(g, 0, collect_traffic="
                                      "False) on the C1 EMGI file (load_csr_binary), best of 3, "
                                      "`taskset -c 0`, 1 core of " + str(os.cpu_count())}
        parity["c1/reference_crc"] = rr["crc"] == C1_LEVELS_CRC
    except Exception as exc:  # report, keep the line
        out["reference"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    finally:
        try:
            os.remove(path)
            os.rmdir(tmp)
        except OSError:
            pass
    t0 = time.perf_counter()
    port = oracle.bfs(g, 0, threads=threads)
    dt = time.perf_counter() - t0
    out["cpu_port"] = {"value": sum(port.traversed_edges) / dt / 1e9, "unit": "GTEPS",
                       "cores": threads, "kind": "port"}
    parity["c1/port_crc"] = crc_hex(port.values) == C1_LEVELS_CRC
    if "value" in out["reference"]:
        out["gpu_over_reference"] = out["gpu_gteps"] / out["reference"]["value"]
    return out


# ------------------------------------------------------------------ N > 1
def _part_series(part, algo, sources, strat, steps, warmup, world, device, *, exchange, bufs,
                 stage, fetch=False):
    """`steps` traversals of a partitioned graph after `warmup`: the loop's
    device time (CUDA events on this rank, max over ranks), the whole job's
    traversed edges, this rank's expansion time / streamed edges / exchange
    bytes, summed or maxed over ranks."""
    import torch
    from paper_2006_06890_b200.multi import run_partition

    fused = exchange in ("fused", "fused-store")

    def one(i):
        return run_partition(part, algo, int(sources[i % len(sources)]), strat, stage_host=stage,
                             fetch=fetch, buffers=None if fused else bufs, fused=fused,
                             bfs_exchange="store" if exchange == "fused-store" else "bitmap")

    for i in range(warmup):
        one(i)
    barrier(world, device)
    trav = launches = local_trav = xbytes = bu = 0
    expand_ms = 0.0
    results = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    d2h = 0
    for i in range(steps):
        r = one(warmup + i)
        trav += r.total_traversed_edges
        local_trav += r.local_traversed
        expand_ms += r.expand_ms
        xbytes += r.exchange_bytes
        bu += r.bottom_up_steps
        launches += part.launches()
        if r.values is not None:
            d2h += r.values.nbytes
        # keep the first result only: a rank's int64 slice is 1 GiB at K30 / 8
        if not results:
            results.append(r)
    ev1.record()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    barrier(world, device)
    loop_ms = max_over_ranks(ev0.elapsed_time(ev1), world, device)
    # per-rank link rate (its streamed edges x 4 B over its expansion time), summed
    link = local_trav * 4 / max(expand_ms * 1e-3, 1e-12) / 1e9
    return {"gteps": trav / (loop_ms * 1e-3) / 1e9, "ms_per_step": loop_ms / steps,
            "traversed_edges_per_step": trav / steps,
            "iterations": results[-1].iterations if results else 0,
            "aggregate_link_gbs": sum_over_ranks(link, world, device),
            "max_rank_expand_ms_per_step": max_over_ranks(expand_ms, world, device) / steps,
            "sum_rank_expand_ms_per_step": sum_over_ranks(expand_ms, world, device) / steps,
            "exchange_bytes_per_step": sum_over_ranks(xbytes, world, device) / steps,
            "bottom_up_steps_per_step": bu / steps,
            "gpu_launches": int(sum_over_ranks(launches, world, device)),
            "wall_s": max_over_ranks(wall, world, device), "_results": results,
            "_trav": trav, "_d2h": d2h}


def _gather_values_crc(r, world, device) -> str:
    """The ranks' crc32s of their owned int64 slices, in rank (= range) order
    (only the 8-character digests travel, not the slices)."""
    import numpy as np
    import torch.distributed as dist
    mine = (f"{zlib.crc32(np.ascontiguousarray(r.values, dtype='<i8')) & 0xffffffff:08x}"
            if r.values is not None else "none")
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    return "-".join(parts)


def _strip(d: dict) -> dict:
    return {k: v for k, v in d.items() if not k.startswith("_")}


def _part_parity_small(args, rank, world, device, stage) -> dict:
    """Partitioned BFS / CC at a small scale, every exchange, against the
    CPU oracle on rank 0 (values, iterations, traversed edges)."""
    import numpy as np
    import torch.distributed as dist
    import paper_2006_06890_b200 as zc
    from paper_2006_06890_b200.multi import generate_rmat_part, run_partition, exchange_buffers
    out = {}
    scale = 18
    for sym, algo in ((False, "bfs"), (True, "cc"), (True, "bfs")):
        part = generate_rmat_part(scale, world, rank, args.edge_factor, seed=args.seed,
                                  symmetrize=sym, device=device)
        ref = None
        if rank == 0:
            import oracle
            whole = zc.generate_rmat(scale, args.edge_factor, seed=args.seed, symmetrize=sym,
                                     device=device)
            g = whole.as_csr()
            src = int(zc.pick_sources(g, 1, seed=7)[0])
            ref = oracle.run(algo, g, src, threads=args.cpu_threads or os.cpu_count())
            whole.close()
        else:
            src = 0
        box = [src]
        dist.broadcast_object_list(box, 0)
        src = box[0]
        bufs = exchange_buffers(algo, world, part.stride,
                                __import__("torch").device("cuda", device))
        for exch in ("reduce-scatter", "fused"):
            r = run_partition(part, algo, src, "merged-aligned", stage_host=stage, fetch=True,
                              buffers=None if exch == "fused" else bufs, fused=exch == "fused")
            parts = [None] * world
            dist.all_gather_object(parts, r.values)
            if rank == 0:
                vals = np.concatenate(parts)
                out[f"{'sym_' if sym else ''}{algo}/{exch}"] = bool(
                    np.array_equal(vals, ref.values) and r.iterations == ref.iterations
                    and list(r.traversed_edges) == list(ref.traversed_edges))
        part.close()
    return out


def main_partitioned(args, rank, world, device):
    """N>1 (BASELINE configs[4]).  One process per GPU, vertex-range
    partitions (edge-balanced), each rank streaming its own edge slice over its
    own host link.

    headline  weak scaling: directed Kronecker scale 27 + log2(N) (2^31 arcs
              per rank, as the N=1 line; K29 at N=4), BFS merged+aligned, the
              fused bitmap exchange (every rank marks its discoveries in its
              own bitmap, each owner ORs the ranks' words over its range
              through peer memory / NVLink); the NCCL reduce-scatter exchange
              and direction-optimizing partitions timed beside it
    configs4  fixed size: Kronecker 29 symmetrized (2^34 arcs) BFS and CC
    parity    small-scale BFS / CC against the oracle for both exchanges;
              full size: the exchanges and direction-optimizing give the same
              levels (per-rank crcs), iterations and traversed edges"""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2006_06890_b200 as zc
    from paper_2006_06890_b200.multi import exchange_buffers, generate_rmat_part, run_partition

    stage = args.backend == "gloo"
    dev = torch.device("cuda", device)
    strat = args.strategy
    scale = args.scale + max(0, int(round(np.log2(world))))
    parity = {}
    if not args.no_parity:
        parity.update(_part_parity_small(args, rank, world, device, stage))

    t0 = time.time()
    part = generate_rmat_part(scale, world, rank, args.edge_factor, seed=args.seed, device=device)
    gen_s = max_over_ranks(time.time() - t0, world, device)
    # sources: pick_sources semantics on rank 0's range, broadcast
    src = [None]
    if rank == 0:
        src = [zc.pick_sources(part.graph_view(), 64, seed=7).astype(np.int64)
               + int(part.bounds[0])]
    dist.broadcast_object_list(src, 0)
    sources = src[0]
    bufs = exchange_buffers("bfs", world, part.stride, dev)
    fused_error = None
    if args.exchange == "fused":
        try:  # peer access between the ranks' GPUs is a property of the box
            run_partition(part, "bfs", int(sources[0]), strat, fetch=False, fused=True)
        except RuntimeError as exc:
            fused_error = str(exc)[:300]
            args.exchange = "reduce-scatter"
    with ClockSampler(device) as clk:
        head = _part_series(part, "bfs", sources, strat, args.steps, args.warmup, world, device,
                            exchange=args.exchange, bufs=bufs, stage=stage)
    other = "reduce-scatter" if args.exchange == "fused" else "fused"
    if fused_error is None:
        alt = _part_series(part, "bfs", sources, strat, min(args.steps, 5), 1, world, device,
                           exchange=other, bufs=bufs, stage=stage)
    else:
        alt = {"error": fused_error, "exchange_bytes_per_step": None}
        other = "reduce-scatter"
    # e2e: the public partitioned API with every rank's int64 levels downloaded
    e2e = _part_series(part, "bfs", sources, strat, args.steps, 0, world, device,
                       exchange=args.exchange, bufs=bufs, stage=stage, fetch=True)
    d2h = sum_over_ranks(e2e["_d2h"], world, device)
    ra = e2e["_results"][0]  # sources[0] (e2e runs without warm-up)
    crc_a = _gather_values_crc(ra, world, device)
    if fused_error is None:
        r_alt = _part_series(part, "bfs", sources[:1], strat, 1, 0, world, device,
                             exchange=other, bufs=bufs, stage=stage,
                             fetch=True)  # e2e's first run: sources[0]
        crc_b = _gather_values_crc(r_alt["_results"][0], world, device)
        rb = r_alt["_results"][0]
        parity[f"kron{scale}/fused_vs_reduce_scatter"] = bool(
            crc_a == crc_b and ra.iterations == rb.iterations
            and list(ra.traversed_edges) == list(rb.traversed_edges))
    e2e_value = e2e["_trav"] / e2e["wall_s"] / 1e9
    # B200 store extension at N>1: direction-optimizing partitions (compressed
    # out-lists, per-rank generated in-lists, bottom-up steps against the
    # all-reduced frontier bitmap), same graph and sources; build time apart
    dobfs = None
    ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    lists = (args.edge_factor << scale) * 4  # all ranks' raw lists, on this node
    if not args.no_variants and ram < 3 * lists:  # + ~1.5x for the two line streams
        dobfs = {"skipped": f"host memory {ram >> 30} GiB < 3 x the {lists >> 30} GiB of lists"}
    elif not args.no_variants:
        t0 = time.time()
        part.build_stores()
        build_s = max_over_ranks(time.time() - t0, world, device)
        d = _part_series(part, "bfs", sources, "direction-optimizing", min(args.steps, 5), 1,
                         world, device, exchange=args.exchange, bufs=bufs, stage=stage)
        dobfs = dict(_strip(d), build_s=build_s)
        # the same levels, iterations and work as merged-aligned from sources[0]
        r_do = _part_series(part, "bfs", sources[:1], "direction-optimizing", 1, 0, world,
                            device, exchange=args.exchange, bufs=bufs, stage=stage,
                            fetch=True)["_results"][0]
        parity[f"kron{scale}/direction-optimizing_vs_merged-aligned"] = bool(
            _gather_values_crc(r_do, world, device) == crc_a
            and r_do.iterations == ra.iterations
            and list(r_do.traversed_edges) == list(ra.traversed_edges))
    part_arcs = part.graph_view().num_edges
    part.close()
    del bufs
    torch.cuda.empty_cache()

    peak = world * PCIE_GEN5_X16_GBS
    line = {
        "metric": METRIC, "value": head["gteps"], "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": dict(bfs_config(args, world), **{
            "workload": f"BFS, Kronecker (R-MAT a=.57 b=.19 c=.19) scale {scale}, edge factor "
                        f"{args.edge_factor}, {args.edge_factor << scale} directed arcs, "
                        f"vertex-range partitioned over {world} ranks (edge-balanced), each "
                        "rank's u32 edge slice zero-copy in pinned host memory",
            "graph": f"kron{scale}", "scale": scale, "parallelism": f"vertex-partition{world}",
            "exchange": ("fused (bitmap OR over peer memory): every rank marks its "
                         "discoveries in its own V-bit bitmap, each owner ORs the ranks' words "
                         "over its range through CUDA-IPC peer pointers (NVLink) and applies "
                         "them; one barrier + the counts all-reduce per level"
                         if args.exchange == "fused" else
                         "per level: NCCL reduce-scatter of u8 flags (MAX); all-reduce of counts"),
            "backend": args.backend}),
        "e2e": {"value": e2e_value, "unit": "GTEPS", "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": int(d2h) // max(args.steps, 1),
                "ms_per_step": e2e["wall_s"] / max(args.steps, 1) * 1e3,
                "api": "run_partition(fetch=True) on every rank: owned int64 levels in host memory"},
        "gpu_launches": head["gpu_launches"],
        "roofline": {
            "bound": "host-link", "achieved": head["aggregate_link_gbs"], "peak": peak,
            "unit": "GB/s", "frac": head["aggregate_link_gbs"] / peak, "traffic": None,
            "kernel": "k_expand_sweep<merged-aligned, partitioned bfs> on every rank",
            "algorithmic_bytes": "each rank's traversed edges x 4 B over its expansion time, "
                                 "summed over ranks (SURVEY 8e aggregate host-link GB/s)",
            "peak_kind": f"{world} x PCIe Gen5 x16 theoretical per direction",
            "kernel_share_of_step": head["max_rank_expand_ms_per_step"] / head["ms_per_step"]},
        "clocks": clk.summary(),
        "exchange": {"bytes_per_step": head["exchange_bytes_per_step"],
                     "bytes_per_level": head["exchange_bytes_per_step"] / max(head["iterations"], 1),
                     "kind": args.exchange,
                     other.replace("-", "_") + "_bytes_per_step": alt["exchange_bytes_per_step"]},
        "variants": {other: _strip(alt), "direction-optimizing": dobfs},
        "fused_error": fused_error,
        "headline": _strip(head),
        "graph": {"vertices": 1 << scale, "arcs": args.edge_factor << scale,
                  "local_arcs_rank0": part_arcs, "gen_s": gen_s},
    }
    if not args.no_configs4:
        line["configs4"] = configs4(args, rank, world, device, stage, parity,
                                    fused_ok=fused_error is None)
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = reference_sample(3, 0, args.seed, args.cpu_threads or os.cpu_count())
    barrier(world, device)
    line["parity"] = parity
    line["parity_all_true"] = all(parity.values()) if parity else None
    if rank == 0:
        print(json.dumps(line), flush=True)


def configs4(args, rank, world, device, stage, parity, fused_ok=True) -> dict:
    """BASELINE configs[4] at fixed size: Kronecker `part_scale` symmetrized
    (2^34 arcs at 29), BFS and CC (Jacobi label propagation), vertex-range
    partitioned over the N ranks (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2006_06890_b200 as zc
    from paper_2006_06890_b200.multi import exchange_buffers, generate_rmat_part
    scale = args.part_scale
    dev = torch.device("cuda", device)
    t0 = time.time()
    part = generate_rmat_part(scale, world, rank, args.edge_factor, seed=args.seed,
                              symmetrize=True, device=device)
    gen_s = max_over_ranks(time.time() - t0, world, device)
    src = [None]
    if rank == 0:
        src = [zc.pick_sources(part.graph_view(), 8, seed=7).astype(np.int64)
               + int(part.bounds[0])]
    dist.broadcast_object_list(src, 0)
    sources = src[0]
    arcs = 2 * (args.edge_factor << scale)
    out = {"workload": f"Kronecker (R-MAT a=.57 b=.19 c=.19) scale {scale} symmetrized "
                       f"({arcs} arcs, {arcs * 4 >> 30} GiB u32), vertex-range partitioned over "
                       f"{world} ranks, each slice zero-copy in its rank's pinned host memory",
           "scaling": "strong", "gen_s": gen_s, "arcs": arcs}
    peak = world * PCIE_GEN5_X16_GBS
    for algo, exch, steps in (("bfs", "fused", 2), ("bfs", "fused-store", 2),
                              ("bfs", "reduce-scatter", 2), ("cc", "reduce-scatter", 1),
                              ("cc", "fused", 1)):
        if exch.startswith("fused") and not fused_ok:
            continue
        bufs = exchange_buffers(algo, world, part.stride, dev) if exch == "reduce-scatter" else None
        r = _part_series(part, algo, sources, "merged-aligned", steps, 1, world, device,
                         exchange=exch, bufs=bufs, stage=stage)
        key = f"{algo}/{exch}"
        res = _strip(r)
        res["aggregate_link_frac"] = r["aggregate_link_gbs"] / peak
        if algo == "cc":  # primary GTEPS: every vertex reached, Sigma deg = arcs
            res["primary_gteps"] = arcs / (r["ms_per_step"] * 1e-3) / 1e9
            res["work_gteps"] = r["gteps"]
        out[key] = res
        del bufs
        torch.cuda.empty_cache()
    for algo, ex in (("bfs", "fused"), ("bfs", "fused-store"), ("cc", "fused")) if fused_ok else ():
        a, b = out[f"{algo}/{ex}"], out[f"{algo}/reduce-scatter"]  # same iterations and work
        parity[f"k{scale}sym_{algo}/{ex}_vs_reduce_scatter_work"] = (
            a["iterations"] == b["iterations"]
            and a["traversed_edges_per_step"] == b["traversed_edges_per_step"])
    part.close()
    return out


if __name__ == "__main__":
    main()
