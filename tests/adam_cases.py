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
