"""CPU checks of bench.py's host-side helpers (no GPU): the clocks summary the
driver's rejection rules read, the ceiling-model summary the headline block
quotes, and the workload description."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_clock_summary_parses_nvidia_smi_rows():
    c = bench.ClockSampler(0)
    c.lines = ["1965, 1965, Not Active, Not Active, Not Active, Not Active, 97",
               "1950, 1965, Not Active, Not Active, Not Active, Active, 99",
               "645, 1965, Not Active, Not Active, Not Active, Not Active, 0",
               "garbage"]
    s = c.summary()
    assert s["sm_max_mhz"] == 1965 and s["sm_mhz"] == 1957.5  # busy samples only
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 3
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]


def test_ceiling_model_summary_reads_the_committed_profile():
    s = bench.ceiling_model_summary()
    assert s["file"] == "profiles/r02_ceiling_model.txt"
    assert s["levels_over_1e7_edges"] >= 3 and s["min_ratio_ceiling_over_measured"] >= 0.9


def test_workload_config_names_the_baseline_graph():
    a = argparse.Namespace(scale=27, edge_factor=16, seed=27, strategy="merged-aligned")
    cfg = bench.bfs_config(a, 1)
    assert cfg["graph"] == "kron27" and cfg["parallelism"] == "single"
    assert "2147483648 directed arcs" in cfg["workload"]
    assert bench.bfs_config(a, 4)["parallelism"] == "vertex-partition4"
