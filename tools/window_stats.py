"""Histogram of the blend's strip window codes (hs_blend_window_stats) on a config."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2406_02720_b200 import _native, device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
sa = scenes.make_config(cfg)
cam = CameraModel(**sa.cameras[0])
scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
              background_color=sa.background_color, device="cuda", dtype=torch.float32)
fr = device.prepare(scene, cam)
hist = torch.zeros(4, dtype=torch.int64, device="cuda")
lib = _native.load()
import ctypes
st = lib.hs_blend_window_stats(ctypes.byref(fr.st), ctypes.c_void_p(hist.data_ptr()),
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
_native.check(st, "hs_blend_window_stats")
h = hist.cpu().numpy()
tot = h.sum()
print(cfg, "pairs", tot, "none/lower/upper/all", (h / tot).round(4).tolist(),
      "pair-work kept", round(float((2 * h[1] + 2 * h[2] + 4 * h[3]) / (4 * tot)), 4))
