#!/bin/bash
# Launch list (ncu gpu__time_duration per launch) of a few bench steps of one config.
# Usage (on the box): CFG=c5 bash tools/launch_list_cfg.sh
set -u
CFG=${CFG:-c3}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-configs"
timeout 600 $CMD > gpurun_out/plain_$CFG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-120} --csv \
  --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_list_$CFG.log 2>&1
python tools/launch_list.py gpurun_out/launches_$CFG.csv ${WHICH:-3} > gpurun_out/launch_list_$CFG.txt
