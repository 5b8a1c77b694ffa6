#!/bin/bash
# On the GPU box: bench each library variant (tools/build_variant.sh) against the base build.
mkdir -p gpurun_out
L=paper_2406_02720_b200/lib
cp $L/libhalfsplat_b200.so /tmp/base.so
for V in base $VARIANTS; do
  if [ "$V" = base ]; then cp /tmp/base.so $L/libhalfsplat_b200.so; else cp $L/variants/$V/libhalfsplat_b200.so $L/libhalfsplat_b200.so; fi
  timeout 600 python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/vb_$V.log 2>&1
  echo "== $V" >> gpurun_out/variants.txt
  python tools/show_configs.py gpurun_out/vb_$V.log >> gpurun_out/variants.txt 2>&1
done
cp /tmp/base.so $L/libhalfsplat_b200.so
