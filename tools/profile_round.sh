#!/bin/bash
# Launch list + full ncu captures of the main kernels for profiles/ (one GPU).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list=$?" > gpurun_out/status.txt
for K in blend_bwd blend_fwd preprocess_bwd preprocess_fwd merge_rows duplicate; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done
