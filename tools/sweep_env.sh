#!/bin/bash
# On the GPU box: one config's stage times under several environment settings.
#   CFG=c2 SETS="HS_SUBTILE=1 HS_SUBTILE=2,HS_LPT=0" bash tools/sweep_env.sh
mkdir -p gpurun_out
for S in base $SETS; do
  ENVS=""
  [ "$S" != base ] && ENVS=$(echo $S | tr ',' ' ')
  env $ENVS timeout 300 python bench.py --config ${CFG:-c3} --steps ${STEPS:-20} --warmup 3 --no-e2e \
    --no-cpu-baseline --no-configs --no-clocks > gpurun_out/sw_$S.log 2>&1
  python - "$S" gpurun_out/sw_$S.log <<'PY'
import json, sys
ln = [x for x in open(sys.argv[2]) if x.startswith("{")]
if not ln:
    print(sys.argv[1], "FAILED"); sys.exit()
d = json.loads(ln[-1])
st = d["roofline"]["stage_ms"]
print(f"{sys.argv[1]:28s} {d['value']:.1f} {d['unit']} " + " ".join(f"{k}={v:.3f}" for k, v in st.items()))
PY
done
