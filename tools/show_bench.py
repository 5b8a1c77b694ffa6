"""Print the headline numbers of gpurun_out/bench.log."""
import json, sys
d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log").read().strip().splitlines()[-1])
r = d.get("roofline", {})
print(f"value {d['value']:.1f} {d['unit']}  fwd {d.get('fwd_fps', 0):.1f} fps  ms/step {d['ms_per_step']:.3f}")
print("stages", {k: round(v, 3) for k, v in r.get("stage_ms", {}).items()})
print("roofline frac", round(r.get("frac", 0), 3), "e2e", (d.get("e2e") or {}).get("value"))
