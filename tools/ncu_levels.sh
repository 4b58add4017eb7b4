#!/bin/bash
# ncu --set full of the expansion kernel at chosen levels of a K27 traversal;
# exports the raw and details pages as CSV (the .ncu-rep files are too big to
# bring back) -- usage: tools/ncu_levels.sh TAG STRATEGY "2 3 4" [extra levels.py args]
TAG=$1; STRAT=$2; LEVELS=$3; shift 3
mkdir -p gpurun_out
for L in $LEVELS; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_expand_sweep -s $L -c 1 \
      -o /tmp/prof_${TAG}_L$L python tools/levels.py --scale 27 --strategies $STRAT --tuning loop=host "$@" \
      > gpurun_out/prof_${TAG}_L$L.log 2>&1
  ncu -i /tmp/prof_${TAG}_L$L.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_L${L}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_${TAG}_L$L.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_L${L}_details.csv 2>/dev/null
  ncu -i /tmp/prof_${TAG}_L$L.ncu-rep --page source --csv > gpurun_out/prof_${TAG}_L${L}_source.csv 2>/dev/null
  rm -f /tmp/prof_${TAG}_L$L.ncu-rep
done
