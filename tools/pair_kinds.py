"""Share of a view's pairs by splat kind (large r > 256 px -> the scalar generic blend path, sign mode, plain).

    python tools/pair_kinds.py c3 c5   (on a GPU box)
"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene
for cfg in sys.argv[1:]:
    sa = scenes.make_config(cfg)
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    ex = out.frame.export()
    radii = out.radii.cpu().numpy()
    rect = np.asarray(ex["tile_rect"]); valid = np.asarray(ex["valid"]); mode = np.asarray(ex["mode"])
    m = int(np.asarray(ex["m_out"]).reshape(-1)[0]) if "m_out" in ex else len(valid)
    cnt = (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1)
    r = radii[valid]
    P = cnt.sum()
    sig = lambda x: 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))
    a1, a2 = sig(sa.raw_opacity_a)[valid], sig(sa.raw_opacity_b)[valid]
    c1, c2 = 0.5 * (a1 + a2), 0.5 * (a1 - a2)
    clamp = (c1 + np.abs(c2)) > 0.989
    print(cfg, "may-clamp pair share", cnt[clamp].sum() / P)
    print(cfg, "pairs", P, "large (r>256) pair share", cnt[r > 256].sum() / P,
          "sign-mode pair share", cnt[mode == 1].sum() / P, "plain", cnt[mode == 2].sum() / P,
          "radius p50/p90/max", np.percentile(r, 50), np.percentile(r, 90), r.max())
