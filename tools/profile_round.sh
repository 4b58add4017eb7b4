#!/bin/bash
# Round profile: bench line, ncu launch list of the bench, one full ncu capture
# of the main-level expansion kernel.  Run under gpurun.
set -x
R=${1:-r01}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
# ncu cannot see kernel nodes of graphs with conditional nodes: profile the
# same kernels launched by the host-driven level loop
export ZC_TUNE=loop=host
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline > gpurun_out/bench_ncu_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expand_sweep -s 3 -c 1 \
    -o gpurun_out/prof_sweep_$R python tools/levels.py --scale 27 --strategies packed \
    > gpurun_out/prof_sweep_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expand_sweep -s 4 -c 1 \
    -o gpurun_out/prof_sweep_L4_$R python tools/levels.py --scale 27 --strategies packed \
    > gpurun_out/prof_sweep_L4_$R.log 2>&1
