#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full capture.
# Usage (on the box): bash tools/gpu_round.sh [kernel-regex-for-full-capture]
set -u
K=${1:-blend_bwd}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" > gpurun_out/status.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "ncu_list=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu_full=$?" >> gpurun_out/status.txt
