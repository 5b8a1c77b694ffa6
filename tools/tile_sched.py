"""Where the blends' time goes on a config: per-tile work (K5: a warp runs its tile's
list up to the last pixel's termination; K6: up to the largest terminal) and the
makespan of a persistent queue of `slots` warps taking tiles in a given order,
against the perfectly balanced sum / slots.

    python tools/tile_sched.py c4 c2 c3   (on a GPU box)
"""
import heapq
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_02720_b200 import _native, device, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel, Scene  # noqa: E402


def makespan(work, order, slots):
    h = [0.0] * slots
    for t in order:
        heapq.heapreplace(h, h[0] + work[t])
    return max(h)


def report(name, work, lens, slots):
    w = work.tolist()
    n = len(w)
    natural = list(range(n))
    by_len = sorted(natural, key=lambda t: -lens[t])
    by_work = sorted(natural, key=lambda t: -w[t])
    ideal = sum(w) / slots
    print(f"  {name}: tiles {n} slots {slots} max tile {max(w):.0f} mean/slot {ideal:.0f} | "
          f"natural {makespan(w, natural, slots) / ideal:.2f}x  by-length "
          f"{makespan(w, by_len, slots) / ideal:.2f}x  by-work {makespan(w, by_work, slots) / ideal:.2f}x",
          flush=True)


lib = _native.load()
for cfg in sys.argv[1:] or ["c4", "c2", "c3"]:
    sa = scenes.make_config(cfg)
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    term = out.terminal.to(torch.int64)
    starts = torch.as_tensor(out.frame.export()["tile_starts"], device="cuda")
    ty, tx = out.frame.tiles_y, out.frame.tiles_x
    lens = (starts[1:] - starts[:-1])
    th, tw = ty * 16, tx * 16
    t = torch.full((th, tw), -1, dtype=torch.int64, device="cuda")
    t[:cam.height, :cam.width] = term
    mx = t.reshape(ty, 16, tx, 16).amax(dim=(1, 3)).reshape(-1)
    k5 = torch.minimum(lens, mx + 1).clamp(min=0).double()
    k6 = (mx + 1).clamp(min=0).double()
    print(f"{cfg}: pairs {int(lens.sum()):,}  max/mean list {int(lens.max())}/{float(lens.float().mean()):.0f}")
    l = lens.tolist()
    report("K5 16x16", k5, l, 148 * 16)
    report("K6 16x16", k6, l, 148 * 12)
