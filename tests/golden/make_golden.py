"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs only in the build container (needs /root/reference): copies the reference
package to a scratch dir, builds its Cython blend core exactly as its setup.py
does, imports `halfsplat` from there and records its outputs on the canonical
synthetic scenes (paper_2406_02720_b200/scenes.py).  Nothing here is imported at
test time; the fixtures are plain .npz files.

    python tests/golden/make_golden.py [--build-dir /tmp/hs_refbuild] [--only c1,mini,...]

Fixture kinds
  full     every FrameGeometry integer array, packed, images, terminal and (if
           backward) the d_color and GradientSet -- small scenes only
  summary  full-size configs: sha256 of each integer array, counts, a seeded
           sample of pixels and of gradient rows, per-group gradient norms
"""

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2406_02720_b200 import scenes  # noqa: E402

REF_PKG = "/root/reference/pkg"
GRAD_GROUPS = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
               "d_raw_opacity_b", "pos_grad_norm", "touch_count")
INT_ARRAYS = {"valid": np.int64, "mode": np.int8, "tile_rect": np.int32,
              "pair_splat": np.int32, "tile_starts": np.int64}


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def scene_sha(sa):
    h = hashlib.sha256()
    for f in sa.FIELDS:
        h.update(np.ascontiguousarray(getattr(sa, f), dtype=np.float32).tobytes())
    return h.hexdigest()


def build_reference(build_dir):
    if not os.path.exists(os.path.join(build_dir, "src", "halfsplat")):
        shutil.rmtree(build_dir, ignore_errors=True)
        shutil.copytree(REF_PKG, build_dir)
        subprocess.run(["chmod", "-R", "u+w", build_dir], check=True)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=build_dir,
                       check=True, capture_output=True)
    sys.path.insert(0, os.path.join(build_dir, "src"))
    import halfsplat.backend as backend
    backend.set_backend("cython")
    return backend


def ref_scene(sa):
    from halfsplat.geometry import Scene
    s64 = sa.as_float64()
    return Scene(**{f: getattr(s64, f) for f in s64.FIELDS}, sh_degree=s64.sh_degree,
                 background_color=s64.background_color)


def ref_camera(c):
    from halfsplat.geometry import CameraModel
    return CameraModel(**c)


def run_reference(sa, cam_idx, backward, threads, kernel="half"):
    from halfsplat.rasterizer import prepare, render, render_backward
    sc = ref_scene(sa)
    cam = ref_camera(sa.cameras[cam_idx])
    t0 = time.time()
    frame = prepare(sc, cam, kernel)
    out = render(sc, cam, kernel=kernel, threads=threads, frame=frame)
    t1 = time.time()
    grads, d_color = None, None
    if backward:
        d_color = scenes.cotangent(cam.height, cam.width)
        grads = render_backward(sc, cam, out, d_color, threads=threads)
    t2 = time.time()
    return frame, out, grads, d_color, (t1 - t0, t2 - t1)


def ref_radii(frame):
    """(N,) int32 radii from the reference's own frame: r = RADIUS_SIGMAS * sqrt(lam_max)
    of the dilated screen covariance, recomputed from frame.cov_ray with the expression
    of rasterizer.py:194-200 (elementwise, so bit-identical to prepare's), then ceil;
    0 for culled primitives.  The reference never materialises radii itself; SURVEY.md
    8(b) defines them this way."""
    from halfsplat import rasterizer as R
    cov = frame.cov_ray
    a = cov[:, 0, 0] + R.LOWPASS_DILATION
    b = cov[:, 0, 1]
    c = cov[:, 1, 1] + R.LOWPASS_DILATION
    det = a * c - b * b
    mid = 0.5 * (a + c)
    lam_max = mid + np.sqrt(np.maximum(mid * mid - det, 0.0))
    radius = R.RADIUS_SIGMAS * np.sqrt(np.maximum(lam_max, 0.0))
    out = np.zeros(frame.n_total, np.int32)
    out[frame.valid] = np.ceil(radius).astype(np.int32)
    return out


def full_fixture(name, sa, cam_idx, backward, threads, kernel="half"):
    frame, out, grads, d_color, secs = run_reference(sa, cam_idx, backward, threads, kernel)
    d = dict(scene_sha=scene_sha(sa), cam_idx=cam_idx, kernel=kernel,
             packed=frame.packed, color=out.color, alpha=out.alpha, depth=out.depth,
             transmittance=out.transmittance, terminal=out.per_pixel_terminal_index,
             tiles_x=frame.tiles_x, tiles_y=frame.tiles_y)
    for k, dt in INT_ARRAYS.items():
        d[k] = np.asarray(getattr(frame, k), dtype=dt)
    d["radii"] = ref_radii(frame)
    if backward:
        d["d_color"] = d_color
        for g in GRAD_GROUPS:
            d[g] = getattr(grads, g)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"{name}: M={frame.valid.shape[0]} P={frame.pair_splat.shape[0]} "
          f"ref fwd {secs[0]:.2f}s bwd {secs[1]:.2f}s")


def summary_fixture(name, sa, cam_idx, backward, threads, n_px=4096, n_rows=2048):
    frame, out, grads, d_color, secs = run_reference(sa, cam_idx, backward, threads)
    cam = sa.cameras[cam_idx]
    h, w = cam["height"], cam["width"]
    rng = np.random.default_rng(12345)
    px = rng.choice(h * w, size=min(n_px, h * w), replace=False)
    d = dict(scene_sha=scene_sha(sa), cam_idx=cam_idx, M=frame.valid.shape[0],
             P=frame.pair_splat.shape[0], tiles_x=frame.tiles_x, tiles_y=frame.tiles_y,
             mode_counts=np.bincount(frame.mode, minlength=3), px_index=px,
             px_color=out.color.reshape(-1, 3)[px], px_alpha=out.alpha.reshape(-1)[px],
             px_depth=out.depth.reshape(-1)[px],
             px_transmittance=out.transmittance.reshape(-1)[px],
             px_terminal=out.per_pixel_terminal_index.reshape(-1)[px],
             terminal_sha=sha(out.per_pixel_terminal_index, np.int32),
             terminal_sum=int(out.per_pixel_terminal_index.astype(np.int64).sum()),
             color_sum=out.color.sum(axis=(0, 1)), alpha_sum=float(out.alpha.sum()),
             fwd_evals=int(np.minimum(out.per_pixel_terminal_index.astype(np.int64) + 1,
                                      _list_len_per_px(frame, h, w)).sum()),
             ref_seconds=np.array(secs))
    for k, dt in INT_ARRAYS.items():
        d[f"sha_{k}"] = sha(getattr(frame, k), dt)
    radii = ref_radii(frame)
    d["sha_radii"] = sha(radii, np.int32)
    d["radii_sum"] = int(radii.astype(np.int64).sum())
    d["packed_sample_rows"] = rng.choice(frame.valid.shape[0], size=min(n_rows, frame.valid.shape[0]),
                                         replace=False)
    d["packed_sample"] = frame.packed[d["packed_sample_rows"]]
    if backward:
        n = len(sa)
        rows = rng.choice(n, size=min(n_rows, n), replace=False)
        d["grad_rows"] = rows
        for g in GRAD_GROUPS:
            arr = getattr(grads, g)
            d[f"norm_{g}"] = float(np.linalg.norm(arr.astype(np.float64)))
            d[f"sample_{g}"] = arr[rows]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"{name}: M={d['M']} P={d['P']} ref fwd {secs[0]:.1f}s bwd {secs[1]:.1f}s")


def _list_len_per_px(frame, h, w):
    lens = np.diff(frame.tile_starts).reshape(frame.tiles_y, frame.tiles_x)
    full = np.repeat(np.repeat(lens, 16, axis=0), 16, axis=1)
    return full[:h, :w].astype(np.int64)


def erf_fixture():
    from halfsplat.kernels import fast_erf
    rng = np.random.default_rng(7)
    z = np.concatenate([np.linspace(-6, 6, 4001), rng.normal(0, 2, 4000),
                        np.array([0.0, -0.0, 1.0, -1.0, 2.4, -2.4, 4.5, -4.5, 1e-300, 50.0])])
    np.savez_compressed(os.path.join(HERE, "erf.npz"), z=z, erf=fast_erf(z))
    print("erf: ", z.shape[0], "points")


def loss_fixture():
    """compute_loss / ssim_with_grad (loss.py:48-106) on float32-representable
    images: ragged sizes against the 32x16 tiles, 1/3/4 channels and 2-D images,
    lambda 0 / 0.2 / 1, identical images and exact ties (sign 0)."""
    from halfsplat import loss as ref_loss
    rng = np.random.default_rng(21)
    f32 = lambda a: np.asarray(a, dtype=np.float32)  # noqa: E731
    x = f32(rng.random((37, 53, 3)))
    y = f32(np.clip(x + rng.normal(0, 0.1, x.shape), 0, 1))
    y[::3, ::4] = x[::3, ::4]  # exact ties: sign(0) = 0
    g2 = f32(rng.random((64, 48)))
    cases = {
        "rgb_l02": (x, y, 0.2),
        "rgb_l0": (x, y, 0.0),
        "rgb_l1": (x, y, 1.0),
        "small_l0": (f32(rng.random((7, 9, 3))), f32(rng.random((7, 9, 3))), 0.0),
        "gray2d_l05": (g2, f32(np.roll(g2, 3, axis=1)), 0.5),
        "rgba_l02": (f32(rng.random((24, 40, 4))), f32(rng.random((24, 40, 4))), 0.2),
        "same_l02": (x, x.copy(), 0.2),
        "edge_11": (f32(rng.random((11, 11, 3))), f32(rng.random((11, 11, 3))), 0.2),
    }
    d = {}
    for name, (a, b, lam) in cases.items():
        loss, grad = ref_loss.compute_loss(a.astype(np.float64), b.astype(np.float64), lam)
        d[f"{name}_a"], d[f"{name}_b"], d[f"{name}_lambda"] = a, b, np.float64(lam)
        d[f"{name}_loss"], d[f"{name}_grad"] = np.float64(loss), grad
        if lam > 0:
            s, sg = ref_loss.ssim_with_grad(a.astype(np.float64), b.astype(np.float64))
            d[f"{name}_ssim"], d[f"{name}_ssim_grad"] = np.float64(s), sg
    d["cases"] = np.array(list(cases))
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **d)
    print("loss:", len(cases), "cases")


def loss64_fixture():
    """compute_loss / ssim_with_grad / metrics.psnr on float64 images that float32
    cannot hold: a render in float64 against a uint8/255 target, a pair whose
    differences sit below float32 resolution (sign(diff) must stay non-zero), and
    a float64 2-D pair."""
    from halfsplat import loss as ref_loss
    from halfsplat import metrics as ref_metrics
    rng = np.random.default_rng(33)
    x = rng.random((41, 57, 3))
    tgt8 = rng.integers(0, 256, (41, 57, 3)).astype(np.uint8)
    tiny = x + rng.choice([-1.0, 1.0], x.shape) * 1e-12  # below float32's ulp near 0.5
    g = rng.random((33, 29))
    cases = {
        "u8_target_l02": (x, tgt8, 0.2),
        "tiny_diff_l02": (x, tiny, 0.2),
        "tiny_diff_l0": (x, tiny, 0.0),
        "gray_f64_l05": (g, np.roll(g, 2, axis=0) * 0.9, 0.5),
    }
    d = {}
    for name, (a, b, lam) in cases.items():
        loss, grad = ref_loss.compute_loss(a, b, lam)
        d[f"{name}_a"], d[f"{name}_b"], d[f"{name}_lambda"] = a, b, np.float64(lam)
        d[f"{name}_loss"], d[f"{name}_grad"] = np.float64(loss), grad
        d[f"{name}_psnr"] = np.float64(ref_metrics.psnr(a, b))
        if lam > 0:
            s, sg = ref_loss.ssim_with_grad(a, b)
            d[f"{name}_ssim"], d[f"{name}_ssim_grad"] = np.float64(s), sg
    d["cases"] = np.array(list(cases))
    np.savez_compressed(os.path.join(HERE, "loss64.npz"), **d)
    print("loss64:", len(cases), "cases")


def adam_fixture():
    """The optimizer part of trainer.step (trainer.py:179-226), driven through the
    reference's own step() with render / compute_loss / render_backward replaced
    by stubs that hand it preset gradients, so only its Adam / normal / tie code
    runs.  Cases: modes, 'full' kernel, frozen normal (lr 0), SH degree 0 and 3,
    rows with all-zero gradients (must stay bit-identical), 3 steps each."""
    from halfsplat import geometry, rasterizer
    from halfsplat import trainer as T
    d = {}
    cases = {
        "half_sh3": dict(kw={}, deg=3),
        "full_sh1": dict(kw={"kernel": "full"}, deg=1),
        "finetune_no": dict(kw={"mode": "finetune_normals_opacities"}, deg=2),
        "frozen_normal_sh0": dict(kw={"lr_normal": 0.0}, deg=0),
    }
    for ci, (name, c) in enumerate(cases.items()):
        rng = np.random.default_rng(100 + ci)
        n, k = 97, (c["deg"] + 1) ** 2
        f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
        nrm = rng.normal(size=(n, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        sc = geometry.Scene(mu=f32(rng.uniform(-1, 1, (n, 3))),
                            log_scale=f32(rng.uniform(-4, -2, (n, 3))),
                            rotation=f32(rng.normal(size=(n, 4))),
                            sh_coeffs=f32(rng.normal(0, 0.3, (n, k, 3))),
                            normal=f32(nrm), raw_opacity_a=f32(rng.normal(size=n)),
                            raw_opacity_b=f32(rng.normal(size=n)), sh_degree=c["deg"])
        cfg = T.TrainConfig(total_iters=100, densify_until=50, **c["kw"])
        state = T.AdamState(sc)
        d[f"{name}_init"] = np.concatenate([getattr(sc, f).reshape(n, -1) for f in SCENE_FIELDS],
                                           axis=1)
        for it in range(3):
            g = rasterizer.GradientSet.zeros(n, k)
            for gname in ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal",
                          "d_raw_opacity_a", "d_raw_opacity_b"):
                arr = getattr(g, gname)
                arr[...] = f32(rng.normal(0, 1e-3, arr.shape))
                arr[: 8 + it] = 0.0  # untouched rows
            d[f"{name}_grad{it}"] = np.concatenate(
                [getattr(g, gn).reshape(n, -1) for gn in ("d_mu", "d_log_scale", "d_rotation",
                                                          "d_sh", "d_normal", "d_raw_opacity_a",
                                                          "d_raw_opacity_b")], axis=1)
            saved = (T.render, T.compute_loss, T.render_backward)
            T.render = lambda scene, cam, kernel="half", threads=None: rasterizer.RenderOutput(
                color=None, alpha=None, depth=None, per_pixel_terminal_index=None)
            T.compute_loss = lambda color, target, lam: (0.5, None)
            T.render_backward = lambda scene, cam, out, d_color, threads=None, _g=g: _g
            try:
                T.step(sc, (None, None), cfg, state, iteration=10 * it + 5, spatial_scale=2.5)
            finally:
                T.render, T.compute_loss, T.render_backward = saved
            d[f"{name}_after{it}"] = np.concatenate(
                [getattr(sc, f).reshape(n, -1) for f in SCENE_FIELDS], axis=1)
        d[f"{name}_t"] = np.array([state.t[gname] for gname in T.GROUPS])
        d[f"{name}_deg"] = np.int64(c["deg"])
        d[f"{name}_kw"] = np.array(repr(c["kw"]))
    d["cases"] = np.array(list(cases))
    np.savez_compressed(os.path.join(HERE, "adam.npz"), **d)
    print("adam:", len(cases), "cases")


def densify_fixture():
    """densify_and_prune + reset_opacity (trainer.py:229-350) of the reference on a
    random float32-representable scene with random statistics and Adam moments:
    unlimited, a budget that accepts some clones and no splits, a budget that
    splits part of the candidates, and zero accumulated gradients (clone
    direction 0).  The split offsets come from rng = default_rng(seed)."""
    from halfsplat import geometry
    from halfsplat import trainer as T
    d = {}
    cases = {"unlimited": 0, "budget_clones": 10**9, "budget_split": 10**9, "zero_grad": 0}
    for ci, (name, maxp) in enumerate(cases.items()):
        rng = np.random.default_rng(300 + ci)
        f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
        n, deg = 160, 2
        k = (deg + 1) ** 2
        nrm = rng.normal(size=(n, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        ls = f32(rng.uniform(-5.0, -3.0, (n, 3)))
        ls[:5] = f32(rng.uniform(-1.2, -1.0, (5, 3)))  # too large: pruned by extent
        ra = f32(rng.normal(0, 3, n))
        sc = geometry.Scene(mu=f32(rng.uniform(-1, 1, (n, 3))), log_scale=ls,
                            rotation=f32(rng.normal(size=(n, 4))),
                            sh_coeffs=f32(rng.normal(0, 0.3, (n, k, 3))), normal=f32(nrm),
                            raw_opacity_a=ra, raw_opacity_b=f32(rng.normal(0, 3, n)),
                            sh_degree=deg)
        stats = T.DensifyStats.zeros(n)
        stats.count[:] = rng.integers(0, 5, n)
        stats.grad_sum[:] = f32(rng.uniform(0, 1.2e-3, n)) * stats.count
        stats.mu_grad_sum[:] = f32(rng.normal(0, 1e-3, (n, 3)))
        if name == "zero_grad":
            stats.mu_grad_sum[:] = 0.0
        opt = T.AdamState(sc)
        for g in T.GROUPS:
            opt.m[g][...] = f32(rng.normal(size=opt.m[g].shape))
            opt.v[g][...] = f32(rng.uniform(0, 1, opt.v[g].shape))
            opt.t[g] = 7
        # budgets relative to this scene's counts
        avg = np.where(stats.count > 0, stats.grad_sum / np.maximum(stats.count, 1), 0.0)
        a1, a2 = sc.alphas()
        mx = np.exp(sc.log_scale).max(axis=1)
        extent = 2.0
        prune = (np.maximum(a1, a2) < 0.005) | (mx > 0.1 * extent)
        hot = (avg >= 2e-4) & ~prune
        nclone = int((hot & (mx <= 0.01 * extent)).sum())
        nsplit = int((hot & (mx > 0.01 * extent)).sum())
        base = int((~prune & ~(hot & (mx > 0.01 * extent))).sum()) + nsplit
        if name == "budget_clones":
            maxp = base + nclone // 2
        elif name == "budget_split":
            maxp = base + nclone + nsplit // 3
        cfg = T.TrainConfig(total_iters=100, densify_until=50, max_primitives=maxp)
        # float32-representable inputs (and their copies) are stored as float32
        d[f"{name}_scene"] = np.concatenate([getattr(sc, f).reshape(n, -1) for f in SCENE_FIELDS],
                                            axis=1).astype(np.float32)
        d[f"{name}_stats"] = np.concatenate([stats.grad_sum[:, None], stats.mu_grad_sum,
                                             stats.count[:, None].astype(np.float64)], axis=1)
        d[f"{name}_m"] = np.concatenate([opt.m[g].reshape(n, -1) for g in T.GROUPS],
                                        axis=1).astype(np.float32)
        d[f"{name}_v"] = np.concatenate([opt.v[g].reshape(n, -1) for g in T.GROUPS],
                                        axis=1).astype(np.float32)
        d[f"{name}_seed"] = np.int64(1000 + ci)
        d[f"{name}_max_primitives"] = np.int64(maxp)
        new, _, report = T.densify_and_prune(sc, stats, cfg, opt, np.random.default_rng(1000 + ci),
                                             extent)
        m = len(new)
        d[f"{name}_out"] = np.concatenate([getattr(new, f).reshape(m, -1) for f in SCENE_FIELDS],
                                          axis=1)
        d[f"{name}_out_m"] = np.concatenate([opt.m[g].reshape(m, -1) for g in T.GROUPS],
                                            axis=1).astype(np.float32)
        d[f"{name}_out_v"] = np.concatenate([opt.v[g].reshape(m, -1) for g in T.GROUPS],
                                            axis=1).astype(np.float32)
        d[f"{name}_report"] = np.array([report["cloned"], report["split"], report["pruned"]])
        T.reset_opacity(new, opt, 0.01)
        d[f"{name}_reset"] = np.stack([new.raw_opacity_a, new.raw_opacity_b], axis=1)
        print(f"densify {name}: n {n} -> {m}, report {report}, max_primitives {maxp}")
    d["cases"] = np.array(list(cases))
    d["extent"] = np.float64(2.0)
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **d)


def io_fixture():
    """scene_io.py:136-269 of the reference: native save/load, 3D-GS export
    (mean / first) and import (both normal inits), and a mixed-type native file
    (float / double / uchar / int properties) read by load_scene."""
    import tempfile
    from halfsplat import geometry, scene_io
    rng = np.random.default_rng(77)
    n, deg = 45, 3
    k = (deg + 1) ** 2
    nrm = rng.normal(size=(n, 3))
    sc = geometry.Scene(mu=rng.uniform(-1, 1, (n, 3)), log_scale=rng.uniform(-5, -2, (n, 3)),
                        rotation=rng.normal(size=(n, 4)), sh_coeffs=rng.normal(0, 0.3, (n, k, 3)),
                        normal=nrm / np.linalg.norm(nrm, axis=1, keepdims=True),
                        raw_opacity_a=rng.normal(0, 3, n), raw_opacity_b=rng.normal(0, 3, n),
                        sh_degree=deg, background_color=np.array([0.1, 0.25, 0.5]))
    d = {"scene": np.concatenate([getattr(sc, f).reshape(n, -1) for f in SCENE_FIELDS], 1)}
    tmp = tempfile.mkdtemp()

    def file_bytes(fn):
        with open(fn, "rb") as fh:
            return np.frombuffer(fh.read(), dtype=np.uint8)

    scene_io.save_scene(sc, f"{tmp}/native.ply")
    d["native_ply"] = file_bytes(f"{tmp}/native.ply")
    for mode in ("mean", "first"):
        scene_io.export_3dgs(sc, f"{tmp}/gs_{mode}.ply", opacity=mode)
        d[f"gs_{mode}_ply"] = file_bytes(f"{tmp}/gs_{mode}.ply")
    for init in ("zero_plus_jitter", "random_unit"):
        imp = scene_io.import_3dgs(f"{tmp}/gs_mean.ply", normal_init=init, seed=5,
                                   background_color=(0.2, 0.2, 0.2))
        d[f"import_{init}"] = np.concatenate([getattr(imp, f).reshape(n, -1)
                                              for f in SCENE_FIELDS], 1)
    # mixed property types, degree 1
    m = 20
    props = [("x", "f4"), ("y", "f8"), ("z", "i4"), ("nx", "f8"), ("ny", "f4"), ("nz", "u1"),
             ("f_dc_0", "f4"), ("f_dc_1", "f8"), ("f_dc_2", "f4")]
    props += [(f"f_rest_{i}", "f8" if i % 2 else "f4") for i in range(9)]
    props += [("opacity", "f4"), ("opacity_2", "f8"), ("scale_0", "f8"), ("scale_1", "f4"),
              ("scale_2", "f8"), ("rot_0", "i4"), ("rot_1", "f4"), ("rot_2", "f8"), ("rot_3", "u1")]
    arr = np.zeros(m, dtype=[(nm, "<" + t) for nm, t in props])
    for nm, t in props:
        if t in ("i4", "u1"):
            arr[nm] = rng.integers(1, 5, m)
        else:
            arr[nm] = rng.normal(size=m)
    tname = {"f4": "float", "f8": "double", "i4": "int", "u1": "uchar"}
    header = ["ply", "format binary_little_endian 1.0", "comment sh_degree 1",
              f"element vertex {m}"] + [f"property {tname[t]} {nm}" for nm, t in props]
    header.append("end_header")
    with open(f"{tmp}/mixed.ply", "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(arr.tobytes())
    d["mixed_ply"] = file_bytes(f"{tmp}/mixed.ply")
    mixed = scene_io.load_scene(f"{tmp}/mixed.ply")
    d["mixed_scene"] = np.concatenate([getattr(mixed, f).reshape(m, -1) for f in SCENE_FIELDS], 1)
    np.savez_compressed(os.path.join(HERE, "io.npz"), **d)
    print("io: native", d["native_ply"].size, "bytes; mixed", d["mixed_ply"].size, "bytes")


def train_fixture():
    """A short Trainer.run of the reference (trainer.py:365-449): 40 iterations
    over 3 views of a small scene towards targets rendered from a perturbed copy,
    densify every 10 iterations, opacity reset at 30; the metrics rows."""
    from halfsplat import geometry, rasterizer
    from halfsplat import trainer as T
    sa = scenes.frustum(400, 1, 48, 40, seed=11)
    sc = geometry.Scene(**{f: getattr(sa, f).astype(np.float64) for f in SCENE_FIELDS},
                        sh_degree=sa.sh_degree, background_color=sa.background_color)
    base = sa.cameras[0]
    views = []
    rng = np.random.default_rng(5)
    tgt_scene = geometry.Scene(**{f: getattr(sa, f).astype(np.float64) for f in SCENE_FIELDS},
                               sh_degree=sa.sh_degree, background_color=sa.background_color)
    tgt_scene.sh_coeffs[:, 0, :] += 0.4
    cams = []
    for v in range(3):
        w2c = np.array(base["world_to_cam"], dtype=np.float64)
        w2c[0, 3] += 0.5 * (v - 1)
        cam = geometry.CameraModel(world_to_cam=w2c, fx=base["fx"], fy=base["fy"], cx=base["cx"],
                                   cy=base["cy"], width=base["width"], height=base["height"])
        target = rasterizer.render(tgt_scene, cam).color.astype(np.float32).astype(np.float64)
        views.append((f"v{v}", cam, target))
        cams.append(dict(world_to_cam=w2c, target=target))
    cfg = T.TrainConfig(total_iters=40, densify_until=35, densify_interval=10,
                        opacity_reset_start=30, opacity_reset_interval=30,
                        opacity_reset_until=35, densify_grad_threshold=2e-5, seed=3,
                        prune_extent_factor=5.0, percent_dense=0.02)
    # the initial scene (the run updates it in place until the first densify)
    d = {"scene": np.concatenate([getattr(sc, f).reshape(len(sc), -1) for f in SCENE_FIELDS], 1),
         "deg": np.int64(sa.sh_degree), "background": np.asarray(sa.background_color)}
    tr = T.Trainer(sc, views, cfg)
    tr.run()
    for v, c in enumerate(cams):
        d[f"w2c{v}"] = c["world_to_cam"]
        d[f"target{v}"] = c["target"].astype(np.float32)
    d["cam"] = np.array([base["fx"], base["fy"], base["cx"], base["cy"], base["width"],
                         base["height"]], dtype=np.float64)
    fields = T.METRICS_FIELDS
    d["fields"] = np.array(fields)
    d["rows"] = np.array([[float(r[f]) for f in fields] for r in tr.metrics_rows])
    np.savez_compressed(os.path.join(HERE, "train.npz"), **d)
    print("train: final prims", len(tr.scene), "rows", len(tr.metrics_rows))
    for r in tr.metrics_rows[::5]:
        print({k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()})


def radii_patch(threads):
    """Adds the reference's radii to the existing scene fixtures without re-running
    the blend: only prepare() runs (the scene hash is checked first)."""
    from halfsplat.rasterizer import prepare
    gens = {name: (gen, kernel) for name, (gen, kernel) in RADII_SCENES.items()}
    for name, (gen, kernel) in gens.items():
        path = os.path.join(HERE, f"{name}.npz")
        old = dict(np.load(path, allow_pickle=False))
        sa = gen()
        assert scene_sha(sa) == str(old["scene_sha"]), name
        frame = prepare(ref_scene(sa), ref_camera(sa.cameras[int(old["cam_idx"])]), kernel)
        radii = ref_radii(frame)
        if "sha_valid" in old:
            old["sha_radii"] = sha(radii, np.int32)
            old["radii_sum"] = np.int64(radii.astype(np.int64).sum())
        else:
            old["radii"] = radii
        np.savez_compressed(path, **old)
        print(f"{name}: radii max {radii.max()} sum {int(radii.astype(np.int64).sum())}")


RADII_SCENES = {
    "c1": (lambda: scenes.make_config("c1"), "half"),
    "mini": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "half"),
    "mini_full": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "full"),
    "ball_small": (lambda: scenes.ball(3000, 3, 96, 72, views=4, seed=9), "half"),
    "ties": (lambda: scenes.frustum(2000, 1, 96, 80, seed=5, clustered=True, dup=0.3), "half"),
    "c2": (lambda: scenes.make_config("c2"), "half"),
    "c3": (lambda: scenes.make_config("c3"), "half"),
    "c5": (lambda: scenes.make_config("c5"), "half"),
    "c4v0": (lambda: scenes.make_config("c4"), "half"),
}

SCENE_FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
                "raw_opacity_b")

JOBS = {
    "radii": radii_patch,
    "erf": lambda t: erf_fixture(),
    "adam": lambda t: adam_fixture(),
    "densify": lambda t: densify_fixture(),
    "io": lambda t: io_fixture(),
    "train": lambda t: train_fixture(),
    "loss": lambda t: loss_fixture(),
    "loss64": lambda t: loss64_fixture(),
    # small scenes, every array
    "c1": lambda t: full_fixture("c1", scenes.make_config("c1"), 0, True, t),
    "mini": lambda t: full_fixture("mini", scenes.frustum(300, 2, 64, 48, seed=3), 0, True, t),
    "mini_full": lambda t: full_fixture("mini_full", scenes.frustum(300, 2, 64, 48, seed=3), 0,
                                        True, t, kernel="full"),
    "ball_small": lambda t: full_fixture("ball_small", scenes.ball(3000, 3, 96, 72, views=4, seed=9),
                                         1, True, t),
    "ties": lambda t: full_fixture("ties", scenes.frustum(2000, 1, 96, 80, seed=5, clustered=True,
                                                          dup=0.3), 0, True, t),
    # full-size configs, summaries
    "c2": lambda t: summary_fixture("c2", scenes.make_config("c2"), 0, True, t),
    "c3": lambda t: summary_fixture("c3", scenes.make_config("c3"), 0, True, t),
    "c5": lambda t: summary_fixture("c5", scenes.make_config("c5"), 0, True, t),
    "c4v0": lambda t: summary_fixture("c4v0", scenes.make_config("c4"), 0, True, t),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build-dir", default="/tmp/hs_refbuild")
    ap.add_argument("--only", default=",".join(j for j in JOBS if j != "radii"))
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    build_reference(args.build_dir)
    for name in args.only.split(","):
        JOBS[name](args.threads)


if __name__ == "__main__":
    main()
