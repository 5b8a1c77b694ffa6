"""Decoding of tests/golden/adam.npz (made by make_golden.adam_fixture from the
reference's trainer.step) shared by the CPU and GPU optimizer tests."""

import ast

import numpy as np

FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
          "raw_opacity_b")
GRADS = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
         "d_raw_opacity_b")


def widths(deg):
    k = (deg + 1) ** 2
    return [3, 3, 4, 3 * k, 3, 1, 1], k


def split(mat, names, deg):
    w, k = widths(deg)
    out, c = {}, 0
    n = mat.shape[0]
    for name, wd in zip(names, w):
        a = np.ascontiguousarray(mat[:, c:c + wd])
        c += wd
        if name in ("sh_coeffs", "d_sh"):
            a = a.reshape(n, k, 3)
        elif wd == 1:
            a = a.reshape(n)
        out[name] = a
    return out


def case(gold, name):
    deg = int(gold[f"{name}_deg"])
    kw = ast.literal_eval(str(gold[f"{name}_kw"]))
    steps = []
    for it in range(3):
        steps.append((10 * it + 5, split(gold[f"{name}_grad{it}"], GRADS, deg),
                      split(gold[f"{name}_after{it}"], FIELDS, deg)))
    return deg, kw, split(gold[f"{name}_init"], FIELDS, deg), steps, gold[f"{name}_t"]


def config(kw):
    from paper_2406_02720_b200.trainer import TrainConfig
    return TrainConfig(total_iters=100, densify_until=50, **kw)


SPATIAL_SCALE = 2.5


def densify_case(gold, name):
    """Inputs and reference outputs of one densify.npz case (float64 dicts)."""
    deg = 2
    f64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
    params = split(f64(gold[f"{name}_scene"]), FIELDS, deg)
    st = f64(gold[f"{name}_stats"])
    stats = (st[:, 0].copy(), np.ascontiguousarray(st[:, 1:4]), st[:, 4].astype(np.int64))
    groups_w = widths_groups(deg)
    m = merge_groups(f64(gold[f"{name}_m"]), groups_w, deg)
    v = merge_groups(f64(gold[f"{name}_v"]), groups_w, deg)
    out = split(f64(gold[f"{name}_out"]), FIELDS, deg)
    out_m = merge_groups(f64(gold[f"{name}_out_m"]), groups_w, deg)
    out_v = merge_groups(f64(gold[f"{name}_out_v"]), groups_w, deg)
    report = dict(zip(("cloned", "split", "pruned"), (int(x) for x in gold[f"{name}_report"])))
    return dict(deg=deg, params=params, stats=stats, m=m, v=v, out=out, out_m=out_m,
                out_v=out_v, report=report, seed=int(gold[f"{name}_seed"]),
                max_primitives=int(gold[f"{name}_max_primitives"]),
                reset=f64(gold[f"{name}_reset"]), extent=float(gold["extent"]))


def widths_groups(deg):
    k = (deg + 1) ** 2
    # the reference's AdamState groups: mu, log_scale, rotation, sh_dc, sh_rest, normal, a, b
    return [3, 3, 4, 3, 3 * (k - 1), 3, 1, 1]


def merge_groups(mat, w, deg):
    """Reference per-group moment columns -> per-field arrays (sh_dc + sh_rest joined)."""
    k = (deg + 1) ** 2
    n = mat.shape[0]
    cols, c = [], 0
    for wd in w:
        cols.append(mat[:, c:c + wd])
        c += wd
    return {"mu": cols[0].copy(), "log_scale": cols[1].copy(), "rotation": cols[2].copy(),
            "sh_coeffs": np.concatenate([cols[3], cols[4]], axis=1).reshape(n, k, 3),
            "normal": cols[5].copy(), "raw_opacity_a": cols[6].reshape(n).copy(),
            "raw_opacity_b": cols[7].reshape(n).copy()}


DENSIFY_CFG = dict(densify_grad_threshold=2e-4, prune_opacity_threshold=0.005,
                   percent_dense=0.01, prune_extent_factor=0.1, split_scale_factor=1.6)
