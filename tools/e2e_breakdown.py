"""Time the pieces of one drop-in (numpy in/out) fwd+bwd call at c3."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200 import rasterizer as R
from paper_2406_02720_b200.geometry import CameraModel, Scene

sa = scenes.make_config("c3")
cam = CameraModel(**sa.cameras[0])
class H: pass
hs = H()
for f in sa.FIELDS:
    setattr(hs, f, torch.from_numpy(getattr(sa, f)).pin_memory())
hs.sh_degree = sa.sh_degree; hs.background_color = sa.background_color
dc = scenes.cotangent(1080, 1920)
for _ in range(3):
    out = R.render(hs, cam); g = R.render_backward(hs, cam, out, dc)
torch.cuda.synchronize()
def t(label, fn):
    torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print("%-28s %8.2f ms" % (label, 1e3 * (time.perf_counter() - a))); return r
for _ in range(2):
    sc = t("upload scene (pinned)", lambda: Scene.from_any(hs))
    fr = t("prepare", lambda: device.prepare(sc, cam))
    do = t("blend fwd", lambda: device.render(sc, cam, frame=fr))
    host = t("D2H image outputs", lambda: R._to_host([do.color, do.alpha, do.depth, do.transmittance, do.terminal, do.radii]))
    dcd = t("upload d_color (pinned f32 staging)", lambda: R._upload_f32(dc, "cuda"))
    gg = t("backward", lambda: device.render_backward(sc, cam, do, dcd))
    hg = t("D2H grads", lambda: R._to_host([getattr(gg, n) for n in R.GradientSet.NAMES]))
    t("backward + bucketed D2H", lambda: R._backward_to_host(sc, cam, do, dcd))
    t("full render()", lambda: R.render(hs, cam))
    t("full render+backward", lambda: R.render_backward(hs, cam, R.render(hs, cam), dc))
