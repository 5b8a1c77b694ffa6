import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene
sa = scenes.ball(4000, 2, 96, 72, views=4, seed=3)
scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree, background_color=sa.background_color, device="cuda", dtype=torch.float32)
cams = [CameraModel(**c) for c in sa.cameras]
dcs = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=i), dtype=torch.float32, device="cuda") for i, c in enumerate(cams)]
rast = device.Rasterizer("cuda")
for views in ((0,), (0, 2)):
    ref = device.DeviceGradientSet.empty_flat(scene)
    red = device.DeviceGradientSet.empty_flat(scene)
    red.flat.zero_(); red.touch_count.zero_()
    ptrs = {n: getattr(red, n).data_ptr() for n in device.DeviceGradientSet.NAMES}; ptrs["mode"] = 2
    for j, v in enumerate(views):
        out = rast.render(scene, cams[v]); rast.render_backward(scene, cams[v], out, dcs[v], grads=ref, accumulate=j > 0)
        out = rast.render(scene, cams[v]); rast.render_backward(scene, cams[v], out, dcs[v], grads=red, reduce_ptrs=ptrs)
    torch.cuda.synchronize()
    for n in device.DeviceGradientSet.NAMES:
        a, b = getattr(ref, n).double(), getattr(red, n).double()
        d = (a - b).abs()
        bad = torch.nonzero(d.reshape(len(scene), -1).amax(1)).flatten()
        print(views, n, float(d.max()), int(bad.numel()), bad[:8].tolist(), float(a.abs().max()))
