#!/bin/bash
# Quick check on one GPU: GPU tests (optionally a subset) + a short bench (stage times).
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -q -m gpu -p no:cacheprovider -x > gpurun_out/pt.txt 2>&1
echo "pytest=$?" > gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS:---no-e2e --no-cpu-baseline} > gpurun_out/bench.log 2>&1
echo "bench=$?" >> gpurun_out/status.txt
