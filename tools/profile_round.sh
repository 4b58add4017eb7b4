#!/bin/bash
# Round profile (run under gpurun): ncu launch list of the bench command and
# full ncu captures of the headline expansion kernel at the main BFS levels.
# ncu cannot see kernel nodes of graphs with conditional nodes: the profiled
# runs use the host-driven level loop (same kernels).
set -x
R=${1:-r01}
STRAT=${2:-compressed}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --tuning loop=host --steps 2 --warmup 3 --no-variants --no-cpu-baseline --no-configs \
    > gpurun_out/bench_ncu_$R.log 2>&1
bash tools/ncu_levels.sh ${R}_$STRAT $STRAT "2 3 4"
