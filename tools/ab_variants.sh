#!/bin/bash
# On the GPU box: the main library against variants built with tools/build_variant.sh,
# twice each, on some configs (plus a parity subset first).
#   VARS="name1 name2" CFGS="c3 c4" bash tools/ab_variants.sh
L=paper_2406_02720_b200/lib
python -m pytest tests -q -m gpu -x -k "parity or golden or split or windows or multiview or view_batch" 2>&1 | tail -2
cp $L/libhalfsplat_b200.so $L/main.so
for V in main $VARS main $VARS; do
  if [ $V = main ]; then cp $L/main.so $L/libhalfsplat_b200.so; else cp $L/variants/$V/libhalfsplat_b200.so $L/libhalfsplat_b200.so; fi
  for C in $CFGS; do
    timeout 300 python bench.py --config $C --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --no-clocks > gpurun_out/ab_${V}_$C.log 2>&1
    python tools/show_configs.py gpurun_out/ab_${V}_$C.log 2>&1 | sed "s/^/$V $C /" | cut -c1-250
  done
done
cp $L/main.so $L/libhalfsplat_b200.so
