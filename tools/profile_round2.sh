#!/bin/bash
# profiles/round2 evidence on one GPU: the full bench line, launch lists of one c3 / c4 /
# c5 step, and ncu --set full captures (summaries + per-line tables) of the step's
# kernels at c3.  Every ncu command profiles a program that first ran plainly and
# exited 0.  Output: gpurun_out/r2/ (copy the summaries into profiles/round2/).
set -u
O=gpurun_out/r2
mkdir -p $O
timeout 1200 python bench.py --steps 20 --warmup 3 > $O/bench_full.log 2>&1
echo "bench=$?" > $O/status.txt
for CFG in c3 c4 c5; do
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-configs --no-graph"
  timeout 600 $CMD > $O/plain_$CFG.log 2>&1 || { echo "plain $CFG failed" >> $O/status.txt; continue; }
  N=150; W=3
  # c4: a step is 8 views (K1-K7a each) and one multi-view K7
  if [ $CFG = c4 ]; then N=1500; W=3; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c $N --csv \
    --log-file $O/launches_$CFG.csv $CMD > $O/ncu_list_$CFG.log 2>&1
  python tools/launch_list.py $O/launches_$CFG.csv $W $CFG > $O/launch_list_$CFG.txt 2>&1
  echo "list_$CFG=$?" >> $O/status.txt
done
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-configs --no-graph"
for K in blend_bwd blend_fwd preprocess_bwd_kernel preprocess_fwd_kernel merge_rows seg_emit \
         seg_fill gather_counts depth_run_rank; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
    -o $O/prof_$K -f $CMD > $O/ncu_$K.log 2>&1
  echo "$K=$?" >> $O/status.txt
  python tools/ncu_summary.py $O/prof_$K.ncu-rep > $O/ncu_$K.txt 2>&1
  python tools/ncu_lines.py $O/prof_$K.ncu-rep 30 > $O/lines_$K.txt 2>&1
done
# c4: the split backward and the multi-view K7
CMD4="python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-configs --no-graph"
for K in blend_bwd preprocess_bwd_views preprocess_fwd_views blend_fwd; do
  S=24; case $K in preprocess_*_views) S=3;; esac  # one multi-view K1 and K7 per step
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $O/prof_c4_$K -f $CMD4 > $O/ncu_c4_$K.log 2>&1
  echo "c4_$K=$?" >> $O/status.txt
  python tools/ncu_summary.py $O/prof_c4_$K.ncu-rep > $O/ncu_c4_$K.txt 2>&1
  python tools/ncu_lines.py $O/prof_c4_$K.ncu-rep 30 > $O/lines_c4_$K.txt 2>&1
done
# the reports are large (gpurun copies back at most 64 MiB): keep the summaries only
rm -f $O/*.ncu-rep $O/launches_*.csv
