"""How much of the forward blend's per-warp work is spent on pixels that already
terminated: for each config, the reference's evaluations sum_px min(terminal+1, len)
against the work of a warp that runs every pixel of its 16x16 tile (or 16x8 / 8x8
sub-tile) until the tile's last pixel terminates, 256 * min(len, max terminal + 1).

    python tools/dead_work.py c3 c4 c2   (on a GPU box)
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import CameraModel, Scene  # noqa: E402


def unit_work(term, lens, uh, uw):
    """sum over (uh x uw) units of uh*uw*min(len, max term + 1)."""
    h, w = term.shape
    th, tw = (h + 15) // 16 * 16, (w + 15) // 16 * 16
    t = torch.full((th, tw), -1, dtype=torch.int64, device=term.device)
    t[:h, :w] = term
    mx = t.reshape(th // uh, uh, tw // uw, uw).amax(dim=(1, 3))
    ln = lens.repeat_interleave(16 // uh, 0).repeat_interleave(16 // uw, 1)
    live = (mx >= 0).to(torch.int64)
    return int((torch.minimum(ln, mx + 1) * live).sum()) * uh * uw


for cfg in sys.argv[1:] or ["c3", "c4", "c2"]:
    sa = scenes.make_config(cfg)
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    term = out.terminal.to(torch.int64)
    starts = torch.as_tensor(out.frame.export()["tile_starts"], device="cuda")
    lens = (starts[1:] - starts[:-1]).reshape(out.frame.tiles_y, out.frame.tiles_x)
    lens_px = lens.repeat_interleave(16, 0).repeat_interleave(16, 1)[:cam.height, :cam.width]
    ref = int(torch.minimum(term + 1, lens_px).sum())
    full = int((lens_px).sum())
    print(f"{cfg}: ref evals {ref:,}  full lists {full / ref:.2f}x  "
          f"16x16 {unit_work(term, lens, 16, 16) / ref:.2f}x  "
          f"16x8 {unit_work(term, lens, 8, 16) / ref:.2f}x  "
          f"8x8 {unit_work(term, lens, 8, 8) / ref:.2f}x  "
          f"16x4 {unit_work(term, lens, 4, 16) / ref:.2f}x", flush=True)
