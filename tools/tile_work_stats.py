"""Per-tile K5 work against list length on one view (what an order estimate can use).

    python tools/tile_work_stats.py c4 [view]   (on a GPU box)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel, Scene  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sa = scenes.make_config(cfg)
cam = CameraModel(**sa.cameras[view])
sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
           background_color=sa.background_color, device="cuda", dtype=torch.float32)
out = device.render(sc, cam)
term = out.terminal.to(torch.int64).cpu().numpy()
ex = out.frame.export()
starts = np.asarray(ex["tile_starts"])
ty, tx = out.frame.tiles_y, out.frame.tiles_x
lens = (starts[1:] - starts[:-1]).reshape(ty, tx)
t = np.full((ty * 16, tx * 16), -1, np.int64)
t[:cam.height, :cam.width] = term
tt = t.reshape(ty, 16, tx, 16).transpose(0, 2, 1, 3).reshape(ty, tx, 256)
L = np.repeat(lens[:, :, None], 256, axis=2)
valid = tt >= 0
done = (tt < L) & valid            # pixel terminated before the list ended
work = np.minimum(lens, tt.max(axis=2) + 1)
frac_done = done.sum(axis=2) / np.maximum(valid.sum(axis=2), 1)
lw = lens.reshape(-1).astype(float)
ww = work.reshape(-1).astype(float)
rank = lambda a: np.argsort(np.argsort(a))
print(f"{cfg} view {view}: tiles {lens.size}, spearman(len, work) "
      f"{np.corrcoef(rank(lw), rank(ww))[0, 1]:.3f}")
print(f"  work: mean {ww.mean():.0f} max {ww.max():.0f}; tiles with every pixel terminated "
      f"{(frac_done.reshape(-1) == 1).mean():.2f}")
top = np.argsort(-ww)[:15]
print("  tile (y,x)   len  work  frac_terminated")
for i in top:
    y, x = divmod(int(i), tx)
    print(f"  ({y:3d},{x:3d}) {int(lw[i]):5d} {int(ww[i]):5d}  {frac_done.reshape(-1)[i]:.2f}")
# work of never-terminating tiles vs len
nt = frac_done.reshape(-1) < 1
print(f"  tiles with a live pixel at the end: {nt.sum()}, their work = len: "
      f"{np.mean(ww[nt] == lw[nt]):.2f}; work sum share {ww[nt].sum() / ww.sum():.2f}")
