import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200 import rasterizer as R
from paper_2406_02720_b200.geometry import CameraModel, Scene
sa = scenes.make_config("c3"); cam = CameraModel(**sa.cameras[0])
class H: pass
hs = H()
for f in sa.FIELDS: setattr(hs, f, torch.from_numpy(getattr(sa, f)).pin_memory())
hs.sh_degree = sa.sh_degree; hs.background_color = sa.background_color
dc = scenes.cotangent(1080, 1920)
sc = Scene.from_any(hs); fr = device.prepare(sc, cam); do = device.render(sc, cam, frame=fr)
dcd = R._upload_f32(dc, "cuda")
for nb in (1, 2, 4, 8, 16, 4):
    R.D2H_BUCKETS = nb
    for _ in range(2): R._backward_to_host(sc, cam, do, dcd)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        a = time.perf_counter(); R._backward_to_host(sc, cam, do, dcd); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    print(nb, "%.2f ms" % (1e3 * min(ts)), flush=True)
