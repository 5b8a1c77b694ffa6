"""Diagnostic: where do GPU-vs-oracle gradient differences come from?

Runs on a GPU box.  For a scene/view: (1) per-group norm-wise errors of the full
pipeline, (2) the blend backward alone through Seam 1 on the oracle's own packed
splats (per-splat merged 12-column rows vs the oracle's FP64 merge), (3) the
d_normal error split by |n_ray.z| of the splat.
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2406_02720_b200 import device, scenes, cuda_blend
from paper_2406_02720_b200.geometry import CameraModel, Scene

def main():
    sa = scenes.ball(20_000, 3, 256, 192, views=8, seed=21)
    s64 = sa.as_float64()
    for idx in (0, 3, 6):
        cam = CameraModel(**sa.cameras[idx])
        dc = scenes.cotangent(cam.height, cam.width, seed=idx)
        ref = O.render(s64, cam)
        rg, merged = O.render_backward(s64, cam, ref, dc, return_merged=True)
        sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                   background_color=sa.background_color, device="cuda", dtype=torch.float64)
        out = device.render(sc, cam)
        g = device.render_backward(sc, cam, out, torch.as_tensor(dc, dtype=torch.float32))
        rep = {}
        for k in ("d_mu", "d_normal", "d_rotation", "pos_grad_norm"):
            a = getattr(g, k).double().cpu().numpy(); b = rg[k]
            rep[k] = np.linalg.norm(a - b) / np.linalg.norm(b)
        print("view", idx, "pipeline", {k: "%.2e" % v for k, v in rep.items()})
        # seam 1 on the oracle's packed
        f = ref.frame
        pg = np.zeros((f.pair_splat.shape[0], 12))
        cuda_blend.backward_tiles(f.packed, f.mode, f.pair_splat, f.tile_starts, cam.height,
                                  cam.width, f.tiles_x, np.asarray(sa.background_color, np.float64),
                                  dc, ref.transmittance, ref.per_pixel_terminal_index, pg, 0,
                                  f.tiles_x * f.tiles_y)
        m = np.zeros_like(merged)
        np.add.at(m, f.pair_splat, pg)
        cols = np.linalg.norm(m - merged, axis=0) / np.maximum(np.linalg.norm(merged, axis=0), 1e-300)
        print("  seam1 per-col normwise", " ".join("%.1e" % c for c in cols))
        # d_normal error by splat
        dn = getattr(g, "d_normal").double().cpu().numpy()[f.valid]
        rn = rg["d_normal"][f.valid]
        err = np.linalg.norm(dn - rn, axis=1)
        top = np.argsort(-err)[:5]
        print("  worst d_normal splats: err", err[top], "|ref|", np.linalg.norm(rn[top], axis=1))
        print("  za,zb of those", f.packed[top][:, 5:7], "mode", f.mode[top])
        print("  share of err^2 in top 10:", (np.sort(err**2)[::-1][:10].sum() / (err**2).sum()))

if __name__ == "__main__":
    main()
