#!/bin/bash
# A/B of an environment toggle on the full bench (all configs), one GPU.
# Usage (on the box): VAR=HS_LPT A=0 B=1 bash tools/ab_env.sh
set -u
mkdir -p gpurun_out/ab
for V in $A $B; do
  env $VAR=$V timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/ab/bench_${VAR}_$V.log 2>&1
  python tools/show_configs.py gpurun_out/ab/bench_${VAR}_$V.log > gpurun_out/ab/sum_${VAR}_$V.txt
  echo "== $VAR=$V"; cat gpurun_out/ab/sum_${VAR}_$V.txt
done
