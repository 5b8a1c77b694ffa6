import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import adam_cases as A
from conftest import load_golden
from oracle import oracle as O
from paper_2406_02720_b200 import rasterizer as R, loss as L
from paper_2406_02720_b200.geometry import CameraModel, Scene
gold = load_golden("train")
deg = int(gold["deg"])
f = A.split(gold["scene"], A.FIELDS, deg)
class S: pass
s = S()
for k in A.FIELDS: setattr(s, k, f[k])
s.sh_degree = deg; s.background_color = gold["background"]
fx, fy, cx, cy, w, h = gold["cam"]
order = list(np.random.default_rng(3).permutation(3))
v = order[-1]
cam = CameraModel(world_to_cam=gold[f"w2c{v}"], fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
out = R.render(s, cam)
ro = O.render(s, cam)
print("view", v, "max color diff gpu vs oracle", np.abs(out.color - ro.color).max())
t = gold[f"target{v}"]
print("gpu loss", L.compute_loss(out.color, t, 0.2)[0], "oracle loss", O.compute_loss(ro.color, t, 0.2)[0])
for vv in range(3):
    cam = CameraModel(world_to_cam=gold[f"w2c{vv}"], fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    ro = O.render(s, cam)
    print(vv, O.compute_loss(ro.color, gold[f"target{vv}"], 0.2)[0])
