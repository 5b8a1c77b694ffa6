"""Compare the device Trainer.run with the reference fixture row by row (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import adam_cases as A  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2406_02720_b200 import trainer as T  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel, Scene  # noqa: E402

gold = load_golden("train")
deg = int(gold["deg"])
f = A.split(gold["scene"], A.FIELDS, deg)
scene = Scene(*(f[k] for k in A.FIELDS), sh_degree=deg, background_color=gold["background"],
              device="cuda", dtype=torch.float64)
fx, fy, cx, cy, w, h = gold["cam"]
views = [(f"v{v}", CameraModel(world_to_cam=gold[f"w2c{v}"], fx=fx, fy=fy, cx=cx, cy=cy,
                               width=int(w), height=int(h)), gold[f"target{v}"]) for v in range(3)]
cfg = T.TrainConfig(total_iters=40, densify_until=35, densify_interval=10, opacity_reset_start=30,
                    opacity_reset_interval=30, opacity_reset_until=35,
                    densify_grad_threshold=2e-5, seed=3, prune_extent_factor=5.0,
                    percent_dense=0.02)
tr = T.Trainer(scene, views, cfg)
tr.run()
fields = [str(x) for x in gold["fields"]]
for r, g in zip(tr.metrics_rows, gold["rows"]):
    print(" ".join(f"{k}={r[k]:.6g}/{g[i]:.6g}" for i, k in enumerate(fields)
                   if k in ("iteration", "loss", "num_primitives", "cloned", "split", "pruned",
                            "opacity_reset")))
