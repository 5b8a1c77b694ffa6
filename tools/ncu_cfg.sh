#!/bin/bash
# ncu --set full captures of kernels (regexes in KS) in one bench config's step.
# Usage (on the box): CFG=c5 KS="row_emit tile_scatter" bash tools/ncu_cfg.sh
set -u
CFG=${CFG:-c3}
OUT=gpurun_out/ncu_$CFG
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-configs"
timeout 600 $CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for K in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $OUT/prof_$K -f $CMD > $OUT/ncu_$K.log 2>&1
  echo "$K=$?" >> $OUT/status.txt
  python tools/ncu_summary.py $OUT/prof_$K.ncu-rep > $OUT/sum_$K.txt 2>&1
done
