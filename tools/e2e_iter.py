"""Per-iteration wall time of the drop-in numpy API (render + render_backward) at c3:
shows the warm-up iterations that allocate pinned staging and workspaces."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_02720_b200 import scenes
from paper_2406_02720_b200 import rasterizer as R
from paper_2406_02720_b200.geometry import CameraModel
sa = scenes.make_config("c3")
cam = CameraModel(**sa.cameras[0])
class H: pass
hs = H()
for f in sa.FIELDS:
    setattr(hs, f, torch.from_numpy(getattr(sa, f)).pin_memory())
hs.sh_degree = sa.sh_degree; hs.background_color = sa.background_color
dc = scenes.cotangent(1080, 1920)
out = g = None
for it in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = R.render(hs, cam)
    t1 = time.perf_counter()
    g = R.render_backward(hs, cam, out, dc)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"it {it}: render {1e3*(t1-t0):7.2f} ms  backward {1e3*(t2-t1):7.2f} ms")
