"""K5's (or K6's) work units on one view, from a library built with -DHS_K5_PROBE
(or -DHS_K6_PROBE; tools/build_variant.sh probe -DHS_K5_PROBE, copied over the
in-tree library): when each unit started and ended, how many splats it evaluated,
and the critical units' nanoseconds per splat.

    python tools/k5_probe.py c2 [view] [bwd]   (on a GPU box)
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_02720_b200 import _native, device, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel, Scene  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sa = scenes.make_config(cfg)
cam = CameraModel(**sa.cameras[view])
sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
           background_color=sa.background_color, device="cuda", dtype=torch.float32)
rast = device.Rasterizer("cuda")
bwd = len(sys.argv) > 3
d_color = torch.as_tensor(scenes.cotangent(cam.height, cam.width), dtype=torch.float32,
                          device="cuda")
for _ in range(3):
    out = rast.render(sc, cam)
    if bwd:
        rast.render_backward(sc, cam, out, d_color)
torch.cuda.synchronize()
lib = _native.load()
n = 65536
buf = np.zeros(4 * n, dtype=np.int64)
assert lib.hs_k5_probe_read(ctypes.c_void_p(buf.ctypes.data), n) == 0
u = buf.reshape(n, 4)
u = u[u[:, 1] > 0]
t0 = u[:, 0].min()
start, end = (u[:, 0] - t0) / 1e3, (u[:, 1] - t0) / 1e3
spl = u[:, 2]
sm = u[:, 3] & 0xffff
tile = u[:, 3] >> 16
print(f"{cfg} view {view}: {len(u)} units, kernel span {end.max():.1f} us, "
      f"mean unit {np.mean(end - start):.2f} us, splats/unit mean {spl.mean():.0f} max {spl.max()}")
order = np.argsort(-end)[:12]
print(" unit  tile  sm  start_us  end_us  splats  ns/splat  units on its SM still running at its start+50%")
for i in order:
    mid = start[i] + 0.5 * (end[i] - start[i])
    busy = int(((sm == sm[i]) & (start <= mid) & (end >= mid)).sum())
    print(f"{i:5d} {tile[i]:5d} {sm[i]:3d} {start[i]:8.1f} {end[i]:7.1f} {spl[i]:7d} "
          f"{1e3 * (end[i] - start[i]) / max(spl[i], 1):8.1f}  {busy}")
# time profile: units running over time
for q in (0.25, 0.5, 0.75, 0.9):
    tq = q * end.max()
    print(f"  at {100 * q:.0f}% of the span: {int(((start <= tq) & (end >= tq)).sum())} units running")
