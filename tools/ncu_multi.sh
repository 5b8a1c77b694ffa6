#!/bin/bash
# ncu full captures of several kernels of one short bench command (one GPU).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for K in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done
