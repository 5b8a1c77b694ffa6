#!/bin/bash
# Launch list + full ncu captures of every kernel family for profiles/ (one GPU).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1
echo "bench=$?" > gpurun_out/status.txt
timeout 300 python tools/window_stats.py c3 > gpurun_out/window_stats.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list=$?" >> gpurun_out/status.txt
for K in blend_bwd blend_fwd preprocess_bwd preprocess_fwd merge_rows duplicate \
         loss_stats loss_grad adam_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done
# one density-control event per bench run: the first launch
for K in densify_classify densify_emit; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 \
    -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done
timeout 300 python tools/io_bench.py > gpurun_out/io_bench.json 2> gpurun_out/io_bench.err
echo "io=$?" >> gpurun_out/status.txt
for K in ply_pack ply_unpack; do
  timeout 600 ncu --set full --clock-control none -k regex:$K -s 0 -c 1 \
    -o gpurun_out/prof_$K -f python tools/io_bench.py > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done
