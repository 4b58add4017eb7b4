#!/usr/bin/env python
"""Benchmark: EMOGI zero-copy BFS on a Kronecker scale-27 graph (BASELINE.json
configs[1]: ~2.1 B directed arcs, edge list in pinned host memory, 1x B200,
naive vs merged vs merged+aligned vs UVM).

Metric: GTEPS = traversed edges (sum of frontier degrees, the reference's
traversed_edges, traversal.py:63-65) / second, whole job.  One step = one BFS
from the next of pick_sources(g, 64, seed=7).

  value  device time (CUDA events on the library stream) of the traversal
         loop, graph resident in its placement (edges in pinned host memory)
  e2e    the same through the public API (paper_2006_06890_b200.bfs_many on
         a DeviceGraph, the reference's per-source loop as one call): source
         H2D, traversal, D2H of every source's int64 levels into pinned host
         memory (overlapped with the next source's traversal) -- host wall
         clock; per_call_value = one blocking bfs() per source
  roofline  dominant kernel = the expansion kernels (the zero-copy edge
         stream): algorithmic bytes = traversed edges x 4 B, over their
         CUDA-event time, against PCIe Gen5 x16 (63.0 GB/s per direction)

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun (N>1) each rank generates and traverses its own replica
(scaling "weak"); rank 0 prints the JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PCIE_GEN5_X16_GBS = 63.0  # 32 GT/s x 16 lanes x 128/130 / 8, per direction
METRIC = "BFS GTEPS (Kronecker scale-27, edge list zero-copy in pinned host memory)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scale", type=int, default=27)
    p.add_argument("--edge-factor", type=int, default=16)
    p.add_argument("--seed", type=int, default=27)
    # compressed: lists that read fewer sectors that way are stored as
    # self-describing 128-byte delta lines, the rest read raw with packed
    # windows (merged-aligned line windows shared across adjacent frontier
    # lists) -- B200 host-store extension, bit-identical results; variants
    # report naive / merged / merged-aligned / packed beside it
    # direction-optimizing: compressed top-down steps, bottom-up steps over the
    # compressed in-lists once the frontier is large (B200 extension; levels,
    # iterations and traversed_edges identical to the reference)
    p.add_argument("--strategy", default="direction-optimizing")
    p.add_argument("--no-variants", action="store_true",
                   help="skip the naive / merged / UVM / HBM comparison runs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the SSSP-U27 / CC-K27 lines (BASELINE configs[2], configs[3])")
    p.add_argument("--cpu-threads", type=int, default=0)
    # test hooks for the partitioned path on a 1-GPU box
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    p.add_argument("--device-override", type=int, default=-1)
    p.add_argument("--force-partitioned", action="store_true")
    p.add_argument("--no-fused", action="store_true",
                   help="N>1: skip the fused (NVLink peer-store) exchange variant")
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
        import torch.distributed as dist
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


def cpu_baseline(g, sources, threads: int, budget_s: float = 25.0, check=None) -> dict:
    """The oracle port (oracle/zc_oracle.c, OpenMP) on the same graph: BFS from
    the bench sources until ~budget_s of CPU work.  check(source, oracle
    result) -> bool compares the GPU's result for the same source (parity at
    the full bench size)."""
    import oracle
    done, edges, t_total = 0, 0, 0.0
    parity = []
    for s in sources:
        t0 = time.perf_counter()
        r = oracle.bfs(g, int(s), threads=threads)
        t_total += time.perf_counter() - t0
        edges += sum(r.traversed_edges)
        done += 1
        if check is not None and len(parity) < 3:
            parity.append(bool(check(int(s), r)))
        if t_total > budget_s:
            break
    return {"value": edges / t_total / 1e9, "unit": "GTEPS", "cores": threads, "kind": "port",
            "sample": f"{done} full BFS run(s) of the oracle port (OpenMP C restatement of "
                      f"traversal.py:98-120) on the same in-memory graph, {threads} threads",
            "seconds": t_total,
            "gpu_bit_exact_vs_oracle": parity}


def main():
    args = parse()
    if args.impl == "reference":
        # the CPU reference arm runs on rank 0 only, without a process group
        if int(os.environ.get("RANK", "0")) != 0:
            return
        rank, world = 0, int(os.environ.get("WORLD_SIZE", "1"))
        local = max(args.device_override, 0)
    else:
        rank, world, local = dist_setup(args)
    import numpy as np

    import paper_2006_06890_b200 as zc
    import torch

    device = local
    torch.cuda.set_device(device)
    config = {"workload": f"BFS, Kronecker (R-MAT a=.57 b=.19 c=.19) scale {args.scale}, "
                          f"edge factor {args.edge_factor}, "
                          f"{args.edge_factor << args.scale} directed arcs, u32 edges in "
                          "pinned host memory (zero-copy)",
              "graph": f"kron{args.scale}", "scale": args.scale, "edge_factor": args.edge_factor,
              "seed": args.seed + rank, "strategy": args.strategy, "placement": "zerocopy",
              "list_store": ("compressed line streams in pinned host memory (B200 host-store "
                             "extension): every list sorted and delta-encoded in 128 B lines, "
                             "hub lists on whole lines, short lists sharing lines; the raw u32 "
                             "lists stay beside them"
                             + ("; out-lists and the in-lists (transpose, built on the GPU)"
                                if args.strategy == "direction-optimizing" else "")
                             if args.strategy in COMPRESSED_STRATEGIES else "raw u32 lists"),
              "direction": ("top-down steps, bottom-up steps (unvisited vertices scan their "
                            "in-lists for a parent in the frontier) once the frontier's "
                            "out-edges exceed twice the unvisited vertices' in-edges; levels, "
                            "iterations and traversed_edges are the reference's"
                            if args.strategy == "direction-optimizing" else "top-down"),
              "sources": "pick_sources(g, 64, seed=7)",
              "l2": "inputs larger than L2 (8 GiB edge list in host memory, 512 MiB level "
                    "array)",
              "parallelism": f"replicas{world}" if world > 1 else "single"}

    if args.impl == "reference":
        return main_reference(args, world, device, config)
    if world > 1 or args.force_partitioned:
        return main_partitioned(args, rank, world, device, config)

    t0 = time.time()
    dg = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed + rank, device=device)
    gen_s = time.time() - t0
    g = dg.as_csr()
    sources = zc.pick_sources(g, 64, seed=7)

    strat = args.strategy
    probe = zc.link_probe(device=device, nbytes=1 << 30, iters=5)
    cmp_info = None
    if strat in COMPRESSED_STRATEGIES:  # host-store build, like pinning: outside the timed region
        t0 = time.time()
        nbytes = dg.build_compressed()
        cmp_info = {"build_s": time.time() - t0, "line_stream_bytes": nbytes}
        if strat == "direction-optimizing":
            t0 = time.time()
            cmp_info["in_line_stream_bytes"] = dg.build_in_lists()
            cmp_info["in_build_s"] = time.time() - t0
    link = LinkBytes(dg, strat)

    # warm-up (untimed)
    for i in range(args.warmup):
        zc.bfs(dg, int(sources[i % 64]), strat, collect_traffic=False)

    # timed region 1: device time of the traversal loop (value)
    barrier(world, device)
    kernel_ms = expand_ms = 0.0
    trav = launches = link_bytes = 0
    bottom_up = []
    with ClockSampler(device) as clk:
        for i in range(args.steps):
            r = zc.bfs(dg, int(sources[(args.warmup + i) % 64]), strat, collect_traffic=False)
            kernel_ms += r.kernel_ms
            expand_ms += r.expand_ms
            trav += r.total_traversed_edges
            launches += r.launches
            link_bytes += link(r)
            if strat == "direction-optimizing":
                bottom_up.append([int(x) for x in np.flatnonzero(dg.directions(r.iterations))])
    barrier(world, device)
    kernel_ms_max = max_over_ranks(kernel_ms, world, device)
    trav_all = sum_over_ranks(trav, world, device)
    value = trav_all / (kernel_ms_max * 1e-3) / 1e9

    # timed region 2: end to end through the public API (host wall clock).
    # bfs_many = the reference's per-source loop (report.py:168-170) as one
    # call: each source's int64 levels download to pinned host memory while
    # the next source streams the edge list.  Batches of <= 10 sources keep
    # the result buffers inside the pinned pool (warmed here, untimed).
    step_srcs = [int(sources[(args.warmup + i) % 64]) for i in range(args.steps)]
    batch = min(10, args.steps)
    r = None
    zc.bfs_many(dg, step_srcs[:batch], strat)
    barrier(world, device)
    t1 = time.perf_counter()
    e2e_trav = h2d = d2h = 0
    for b0 in range(0, args.steps, batch):
        rs = zc.bfs_many(dg, step_srcs[b0:b0 + batch], strat)
        for r in rs:
            e2e_trav += r.total_traversed_edges
            h2d += r.h2d_bytes
            d2h += r.d2h_bytes
        rs = r = None
    barrier(world, device)
    wall = max_over_ranks(time.perf_counter() - t1, world, device)
    e2e_value = sum_over_ranks(e2e_trav, world, device) / wall / 1e9

    # the same, one blocking bfs() call per source (no download overlap)
    barrier(world, device)
    t2 = time.perf_counter()
    for src in step_srcs:
        r = zc.bfs(dg, src, strat, collect_traffic=False)
        r = None
    barrier(world, device)
    wall_1 = max_over_ranks(time.perf_counter() - t2, world, device)
    e2e_per_call = sum_over_ranks(e2e_trav, world, device) / wall_1 / 1e9

    # GB/s of list data the expansion kernels must read over the link
    achieved = link_bytes / (expand_ms * 1e-3) / 1e9
    summ = load_ncu_summary()
    ncu = summ.get("bfs_expand_dobfs" if strat == "direction-optimizing" else "bfs_expand", {})
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": kernel_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config,
        "e2e": {"value": e2e_value, "unit": "GTEPS",
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "ms_per_step": wall / args.steps * 1e3,
                "api": f"bfs_many (pipelined result downloads, batches of {batch})",
                "per_call_value": e2e_per_call,
                "per_call_api": "one blocking bfs() per source"},
        "gpu_launches": launches,
        "roofline": {"bound": "host-link", "achieved": achieved,
                     "peak": PCIE_GEN5_X16_GBS, "unit": "GB/s",
                     "frac": achieved / PCIE_GEN5_X16_GBS,
                     "traffic": ncu.get("dram_bytes_per_launch"),
                     "kernel": "k_expand_sweep (zero-copy edge stream)",
                     "algorithmic_bytes": link.describe,
                     "algorithmic_bytes_per_step": link_bytes / args.steps,
                     "u32_equivalent_gbs": trav * 4 / (expand_ms * 1e-3) / 1e9,
                     "peak_kind": "PCIe Gen5 x16 theoretical per direction",
                     "measured_peaks_gbs": probe,
                     "frac_of_measured_memcpy": achieved / probe["memcpy_h2d_gbs"],
                     # SM-side sysmem reads (ld or TMA cp.async.bulk) cap at the
                     # zero-copy streaming peak (profiles/r01_tma_bulk_probe.txt)
                     "frac_of_measured_zerocopy_ceiling": achieved / probe["zerocopy_read_gbs"],
                     "sysmem_bytes_per_launch": ncu.get("sysmem_bytes_per_launch")},
        "clocks": clk.summary(),
        "graph": {"vertices": dg.num_vertices, "arcs": dg.num_edges, "gen_s": gen_s,
                  "traversed_edges_per_step": trav / args.steps},
    }
    if cmp_info:
        line["graph"]["compressed"] = cmp_info
    if bottom_up:
        line["bottom_up_iterations_per_step"] = bottom_up

    if rank == 0 and not args.no_cpu_baseline:
        threads = args.cpu_threads or os.cpu_count()
        def check(src, ref):
            r = zc.bfs(dg, src, strat, collect_traffic=False)
            return (np.array_equal(r.values, ref.values) and r.iterations == ref.iterations
                    and r.traversed_edges == ref.traversed_edges)
        line["cpu_baseline"] = cpu_baseline(g, sources, threads, check=check)

    # configs before the UVM variants: managed-memory runs leave the process
    # slower on later zero-copy work (measured), so UVM goes last
    if rank == 0 and not args.no_variants and world == 1:
        line["variants"] = variants(zc, args, dg, sources, device, phase="zerocopy")
    dg.close()
    if rank == 0 and not args.no_configs and world == 1:
        line["configs"] = other_configs(zc, args, device)
    if rank == 0 and not args.no_variants and world == 1:
        line["variants"].update(variants(zc, args, None, sources, device, phase="placements"))
        finish_variants(line["variants"])
    if rank == 0:
        print(json.dumps(line), flush=True)


def main_reference(args, world, device, config):
    """--impl reference: the reference's algorithm on the host cores -- the
    oracle port (oracle/zc_oracle.c, OpenMP restatement of traversal.py:98-120;
    the reference itself is a Python package absent from the GPU box) -- on
    this arm's workload (same graph: scale 27 + log2(N), same sources).  Rank 0
    only; the input graph is built by the GPU generator (not timed)."""
    import numpy as np
    import oracle
    import paper_2006_06890_b200 as zc

    scale = args.scale + max(0, int(round(np.log2(world))))
    threads = args.cpu_threads or os.cpu_count()
    dg = zc.generate_rmat(scale, args.edge_factor, seed=args.seed, device=device)
    g = dg.as_csr()
    sources = zc.pick_sources(g, 64, seed=7)
    per, edges = [], 0
    for i in range(args.warmup + args.steps):
        t1 = time.perf_counter()
        r = oracle.bfs(g, int(sources[i % 64]), threads=threads)
        dt = time.perf_counter() - t1
        if i >= args.warmup:
            per.append(dt)
            edges += sum(r.traversed_edges)
    total = sum(per)
    val = edges / total / 1e9
    cfg = dict(config)
    cfg.update({"graph": f"kron{scale}", "scale": scale})
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": val, "unit": "GTEPS", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} full BFS runs (after {args.warmup} warm-up) "
                                       "of the oracle port on the whole graph"},
            "e2e": {"value": val, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    dg.close()


def main_partitioned(args, rank, world, device, config):
    """N>1: weak scaling -- Kronecker scale 27 + log2(N) (K29 at N=4, BASELINE
    configs[4]), vertex-range partitioned, each rank streaming its own 2^31-arc
    slice over its own host link; NCCL reduce-scatter of the u8 frontier flags
    (MAX) over NVLink every level."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2006_06890_b200 as zc
    from paper_2006_06890_b200.multi import (exchange_buffers, generate_rmat_part,
                                             run_partition)

    scale = args.scale + max(0, int(round(np.log2(world))))
    stage = args.backend == "gloo"
    t0 = time.time()
    part = generate_rmat_part(scale, world, rank, args.edge_factor, seed=args.seed,
                              device=device)
    gen_s = time.time() - t0
    # sources: pick_sources semantics on rank 0's range, broadcast
    src = torch.zeros(64, dtype=torch.int64)
    if rank == 0:
        src = torch.from_numpy(zc.pick_sources(part.graph_view(), 64, seed=7).astype(np.int64))
    src = src.to(torch.device("cpu") if stage else torch.device("cuda", device))
    dist.broadcast(src, 0)
    sources = src.cpu().numpy()
    bufs = exchange_buffers("bfs", world, part.stride, torch.device("cuda", device))
    strat = args.strategy

    def one(i, fetch):
        return run_partition(part, "bfs", int(sources[i % 64]), strat, stage_host=stage,
                             fetch=fetch, buffers=bufs)

    for i in range(args.warmup):
        one(i, False)
    barrier(world, device)
    trav = 0
    launches = 0
    expand_ms = 0.0
    with ClockSampler(device) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for i in range(args.steps):
            r = one(args.warmup + i, False)
            trav += r.total_traversed_edges
            launches += part.launches()
        ev1.record()
        torch.cuda.synchronize(device)
    barrier(world, device)
    loop_ms = max_over_ranks(ev0.elapsed_time(ev1), world, device)
    value = trav / (loop_ms * 1e-3) / 1e9  # traversed edges are global (summed over ranks)

    barrier(world, device)
    t1 = time.perf_counter()
    d2h = 0
    for i in range(args.steps):
        r = one(args.warmup + i, True)
        d2h += r.values.nbytes
        del r
    barrier(world, device)
    wall = max_over_ranks(time.perf_counter() - t1, world, device)
    e2e_value = trav / wall / 1e9
    fused = None
    if not args.no_fused:
        # variant: fused exchange -- the expand kernel writes candidates straight
        # into the owners' buffers (CUDA IPC peer pointers over NVLink)
        try:
            for i in range(args.warmup):
                run_partition(part, "bfs", int(sources[i % 64]), strat, fetch=False, fused=True)
            barrier(world, device)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ftrav = 0
            for i in range(args.steps):
                r = run_partition(part, "bfs", int(sources[(args.warmup + i) % 64]), strat,
                                  fetch=False, fused=True)
                ftrav += r.total_traversed_edges
            e1.record()
            torch.cuda.synchronize(device)
            barrier(world, device)
            fms = max_over_ranks(e0.elapsed_time(e1), world, device)
            fused = {"gteps": ftrav / (fms * 1e-3) / 1e9, "ms_per_step": fms / args.steps,
                     "same_traversed": ftrav == trav}
        except Exception as exc:  # report, keep the headline
            fused = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    cfg = dict(config)
    cfg.update({"workload": f"BFS, Kronecker (R-MAT a=.57 b=.19 c=.19) scale {scale}, edge factor "
                            f"{args.edge_factor}, {args.edge_factor << scale} directed arcs, "
                            f"vertex-range partitioned over {world} ranks (edge-balanced), each "
                            "rank's u32 edge slice zero-copy in pinned host memory",
                "graph": f"kron{scale}", "scale": scale, "seed": args.seed,
                "parallelism": f"vertex-partition{world}",
                "exchange": ("per level: reduce-scatter of u8 flags (MAX) for top-down steps; "
                             "bottom-up steps all-reduce (SUM of disjoint bits = OR) the "
                             "owned-frontier bitmaps and scan the owned vertices' in-lists "
                             "(generated per rank, no edge exchange); all-reduce of counts"
                             if strat == "direction-optimizing" else
                             "per level: reduce-scatter of u8 flags (MAX), all-reduce of counts"),
                "backend": args.backend})
    line = {"metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": loop_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": cfg,
            "e2e": {"value": e2e_value, "unit": "GTEPS", "h2d_bytes_per_step": 8,
                    "d2h_bytes_per_step": int(sum_over_ranks(d2h, world, device)) // args.steps,
                    "ms_per_step": wall / args.steps * 1e3},
            "gpu_launches": int(sum_over_ranks(launches, world, device)),
            "variants": {"fused_exchange": fused},
            "clocks": clk.summary(),
            "graph": {"vertices": 1 << scale, "arcs": args.edge_factor << scale,
                      "local_arcs_rank0": part.graph_view().num_edges, "gen_s": gen_s,
                      "traversed_edges_per_step": trav / args.steps}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    part.close()


COMPRESSED_STRATEGIES = ("compressed", "direction-optimizing")


class LinkBytes:
    """Algorithmic link bytes of a BFS step: the list data the expansion
    kernels must read -- 4 B per traversed edge of the raw u32 lists, or, for
    the compressed strategies, the line-stream bytes the kernels requested
    (counted on the device: whole lines of long lists, the spanned words of
    shared lines; bottom-up steps read candidates' in-lists up to the first
    parent)."""

    def __init__(self, dg, strategy: str):
        self.dg = dg
        self.compressed = strategy in COMPRESSED_STRATEGIES
        self.describe = ("line-stream bytes requested by the expansion kernels (device counter: "
                         "128 B per long-list line, the spanned words of shared lines)"
                         if self.compressed else
                         f"traversed edges x {dg.edge_elem_bytes} B (raw u32 lists)")

    def __call__(self, r) -> int:
        if self.compressed:
            return self.dg.link_bytes_requested()
        return r.total_traversed_edges * self.dg.edge_elem_bytes


def _gteps(zc, dg, sources, strategy, reps=1, evict=False):
    best = None
    for i in range(reps):
        if evict:
            zc.evict(dg)
        r = zc.bfs(dg, int(sources[i % 64]), strategy, collect_traffic=False)
        gbs = r.total_traversed_edges * 4 / (r.expand_ms * 1e-3) / 1e9
        cur = {"gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
               "kernel_ms": r.kernel_ms,
               ("u32_equivalent_gbs" if strategy in COMPRESSED_STRATEGIES else "expand_gbs"): gbs}
        if strategy in COMPRESSED_STRATEGIES:
            cur["requested_link_gbs"] = dg.link_bytes_requested() / (r.expand_ms * 1e-3) / 1e9
        if best is None or cur["gteps"] > best["gteps"]:
            best = cur
    return best


def other_configs(zc, args, device) -> dict:
    """BASELINE configs[2] (SSSP, u32 weights, uniform scale 27, edges + weights
    zero-copy) and configs[3] (CC, Kronecker scale 27 symmetrized = 2^32 arcs),
    one source / run each after a warm-up, merged-aligned and packed."""
    out = {}
    import oracle
    u = zc.generate_uniform_device(1 << args.scale, 16, 16, seed=args.seed, weights=(8, 72),
                                   device=device)
    src = int(zc.pick_sources(u.as_csr(), 1, seed=7)[0])
    for s in ("merged-aligned", "packed"):
        zc.sssp(u, src, s, collect_traffic=False)
        r = zc.sssp(u, src, s, collect_traffic=False)
        out[f"sssp_uniform{args.scale}/{s}"] = {
            "work_gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
            "kernel_ms": r.kernel_ms, "iterations": r.iterations,
            "link_gbs": r.total_traversed_edges * 8 / (r.expand_ms * 1e-3) / 1e9,
            "work_edges": r.total_traversed_edges}
    # B200 host-store option: compressed lines with the weights alongside
    zc.sssp(u, src, "compressed", collect_traffic=False)
    r = zc.sssp(u, src, "compressed", collect_traffic=False)
    out[f"sssp_uniform{args.scale}/compressed"] = {
        "work_gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
        "kernel_ms": r.kernel_ms, "iterations": r.iterations,
        "u32_pair_equivalent_gbs": r.total_traversed_edges * 8 / (r.expand_ms * 1e-3) / 1e9,
        "work_edges": r.total_traversed_edges}
    u.build_sssp_pairs()  # B200 layout option: one interleaved (dst, weight) stream
    for s in ("merged-aligned", "packed"):
        zc.sssp(u, src, s, collect_traffic=False)
        r = zc.sssp(u, src, s, collect_traffic=False)
        out[f"sssp_uniform{args.scale}/{s}+pairs"] = {
            "work_gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
            "kernel_ms": r.kernel_ms, "iterations": r.iterations,
            "link_gbs": r.total_traversed_edges * 8 / (r.expand_ms * 1e-3) / 1e9,
            "work_edges": r.total_traversed_edges}
    t0 = time.perf_counter()
    ref = oracle.sssp(u.as_csr(), src, threads=os.cpu_count())
    out[f"sssp_uniform{args.scale}/cpu_port_work_gteps"] = (
        sum(ref.traversed_edges) / (time.perf_counter() - t0) / 1e9)
    out[f"sssp_uniform{args.scale}/bit_exact_vs_oracle"] = bool(
        (r.values == ref.values).all() and r.iterations == ref.iterations)
    u.close()
    t0 = time.time()
    k = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, symmetrize=True,
                         device=device)
    gen_s = time.time() - t0
    for s in ("merged-aligned", "packed", "compressed"):
        zc.cc(k, s, collect_traffic=False)
        r = zc.cc(k, s, collect_traffic=False)
        out[f"cc_kron{args.scale}_sym/{s}"] = {
            "work_gteps": r.total_traversed_edges / (r.kernel_ms * 1e-3) / 1e9,
            "kernel_ms": r.kernel_ms, "iterations": r.iterations,
            ("u32_equivalent_gbs" if s == "compressed" else "link_gbs"):
                r.total_traversed_edges * 4 / (r.expand_ms * 1e-3) / 1e9,
            "work_edges": r.total_traversed_edges, "arcs": k.num_edges, "gen_s": gen_s}
    t0 = time.perf_counter()
    ref = oracle.cc(k.as_csr(), threads=os.cpu_count())
    out[f"cc_kron{args.scale}_sym/cpu_port_work_gteps"] = (
        sum(ref.traversed_edges) / (time.perf_counter() - t0) / 1e9)
    out[f"cc_kron{args.scale}_sym/bit_exact_vs_oracle"] = bool(
        (r.values == ref.values).all() and r.iterations == ref.iterations)
    k.close()
    return out


def variants(zc, args, dg, sources, device, phase: str) -> dict:
    """configs[1]'s comparison: naive vs merged vs merged+aligned vs packed
    (zero-copy), then the in-HBM control and UVM (cold; and at the reference's
    25% capacity)."""
    out = {}
    if phase == "zerocopy":
        for s in ("naive", "merged", "merged-aligned", "packed", "compressed",
                  "direction-optimizing"):
            # naive walks each hub list with one thread (seconds per BFS): one rep
            out[f"zerocopy/{s}"] = _gteps(zc, dg, sources, s, reps=1 if s == "naive" else 2)
        return out
    import torch
    # host-resident managed lists read in place (zerocopy-managed): the same
    # zero-copy loads through the UVM driver's large-page GPU mappings
    h = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, device=device,
                         placement="zerocopy-managed")
    out["zerocopy-managed/direction-optimizing"] = _gteps(zc, h, sources, "direction-optimizing",
                                                          reps=2)
    h.close()
    for placement in ("hbm", "uvm"):
        h = zc.generate_rmat(args.scale, args.edge_factor, seed=args.seed, device=device,
                             placement=placement)
        out[f"{placement}/merged-aligned"] = _gteps(zc, h, sources, "merged-aligned", reps=2,
                                                    evict=placement == "uvm")
        if placement == "uvm":
            # the reference's UVM capacity default: 25% of the dataset
            # (report.py:151-153) -- ballast HBM so only that much stays free
            dataset = h.num_edges * h.edge_elem_bytes
            free, _ = torch.cuda.mem_get_info(device)
            ballast_bytes = max(0, free - dataset // 4 - (256 << 20))
            ballast = torch.empty(ballast_bytes, dtype=torch.uint8, device=f"cuda:{device}")
            r = _gteps(zc, h, sources, "merged-aligned", reps=2, evict=True)
            r["free_hbm_bytes"] = torch.cuda.mem_get_info(device)[0]
            out["uvm_cap25/merged-aligned"] = r
            del ballast
            torch.cuda.empty_cache()
        h.close()
    return out


def finish_variants(v: dict) -> None:
    ma = v["zerocopy/merged-aligned"]["gteps"]
    v["speedup_vs_uvm"] = ma / v["uvm/merged-aligned"]["gteps"]
    v["speedup_vs_uvm_cap25"] = ma / v["uvm_cap25/merged-aligned"]["gteps"]
    for s in ("packed", "compressed", "direction-optimizing"):
        v[f"{s}_speedup_vs_uvm_cap25"] = (v[f"zerocopy/{s}"]["gteps"]
                                          / v["uvm_cap25/merged-aligned"]["gteps"])


if __name__ == "__main__":
    main()
