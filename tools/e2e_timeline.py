"""Where the end-to-end step's time goes (the bench's e2e headline: pinned float32
host scene, float32 outputs): wall time of render and render_backward through the
drop-in numpy API, against their device work alone.

    python tools/e2e_timeline.py   (on a GPU box)
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_02720_b200 import rasterizer as R, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel  # noqa: E402

sa = scenes.make_config("c3")
cam = CameraModel(**sa.cameras[0])


class HostScene:
    pass


hs = HostScene()
for f in sa.FIELDS:
    setattr(hs, f, torch.from_numpy(np.ascontiguousarray(getattr(sa, f), np.float32)).pin_memory())
hs.sh_degree = sa.sh_degree
hs.background_color = sa.background_color
d_color = torch.from_numpy(scenes.cotangent(cam.height, cam.width).astype(np.float32)).pin_memory()
R.set_output_dtype(np.float32)
for _ in range(3):
    out = R.render(hs, cam)
    g = R.render_backward(hs, cam, out, d_color)
torch.cuda.synchronize()
n = 10
tr = tb = 0.0
for _ in range(n):
    t0 = time.perf_counter()
    out = R.render(hs, cam)
    t1 = time.perf_counter()
    g = R.render_backward(hs, cam, out, d_color)
    t2 = time.perf_counter()
    tr += t1 - t0
    tb += t2 - t1
print(f"render {1e3 * tr / n:.2f} ms, render_backward {1e3 * tb / n:.2f} ms, "
      f"step {1e3 * (tr + tb) / n:.2f} ms")
# PCIe alone: the same bytes as pinned copies
dev = torch.empty(sum(getattr(hs, f).numel() for f in sa.FIELDS), dtype=torch.float32,
                  device="cuda")
host = torch.empty(dev.shape, dtype=torch.float32).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(n):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
t2 = time.perf_counter()
nb = dev.numel() * 4
print(f"scene-sized copies: H2D {1e3 * (t1 - t0) / n:.2f} ms ({nb / ((t1 - t0) / n) / 1e9:.1f} "
      f"GB/s), D2H {1e3 * (t2 - t1) / n:.2f} ms ({nb / ((t2 - t1) / n) / 1e9:.1f} GB/s)")
