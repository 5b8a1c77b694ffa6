#!/bin/bash
set -u
mkdir -p gpurun_out/prof2
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $CMD > gpurun_out/prof2/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof2/launches.csv $CMD > gpurun_out/prof2/ncu_list.log 2>&1
echo "list=$?" >> gpurun_out/prof2/status.txt
for K in blend_bwd blend_fwd; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o gpurun_out/prof2/prof_$K -f $CMD > gpurun_out/prof2/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/prof2/status.txt
done
