CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
mkdir -p gpurun_out
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || exit 1
for K in $KS; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
done
