"""One line per config of a bench.py JSON line: value, stage ms per view, blend fractions."""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(line)
st = d["roofline"]["stage_ms"]
print(f"c3 {d['value']:.1f} {d['unit']} ({d.get('launch_mode', '')}; eager "
      f"{d.get('eager_ms_per_step')}) fwd {d['fwd_fps']:.0f} fps "
      + " ".join(f"{k}={v:.3f}" for k, v in st.items())
      + f" K6 frac {d['roofline']['frac']:.3f} K5 {d['roofline']['blend_fwd']['achieved_tflops'] / d['roofline']['peak']:.3f}")
for k, v in d.get("configs", {}).items():
    print(f"{k} {v['value']:.1f} {v['unit']} "
          + " ".join(f"{a}={b:.3f}" for a, b in v["stage_ms_per_view"].items())
          + f" K5 {v['blend_fwd_frac']:.3f} K6 {v['blend_bwd_frac']:.3f}")
