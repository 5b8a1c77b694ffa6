"""Canonical synthetic scenes and cameras.

The numpy call order is part of the definition: the same seed must give the same
scene as the survey's reference measurements (M, P and evaluation counts of the
configs table), so that the golden fixtures, the oracle and the GPU all see one
input.  All seven parameter arrays are rounded to float32 so a float32 device
scene and the float64 oracle/reference hold identical values.

    c1  frustum(10_000, 0, 128, 128, seed=0)                     forward only
    c2  ball(100_000, 3, 800, 800, views=8, seed=0), view 0      fwd + bwd
    c3  frustum(1_000_000, 3, 1920, 1080, seed=0)                fwd + bwd (headline)
    c4  ball(3_000_000, 3, 1297, 840, views=8, seed=0)           8-view batch
    c5  frustum(500_000, 3, 3840, 2160, seed=0, sig 8-40,
                clustered, dup=0.1)                              adversarial
"""

from dataclasses import dataclass, field

import numpy as np

BACKGROUND = (0.1, 0.15, 0.2)  # tests/test_rasterizer.py:18


@dataclass
class SceneArrays:
    """Host float32 scene (reference Scene field names) plus its cameras."""

    mu: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    sh_coeffs: np.ndarray
    normal: np.ndarray
    raw_opacity_a: np.ndarray
    raw_opacity_b: np.ndarray
    sh_degree: int
    background_color: np.ndarray = field(default_factory=lambda: np.array(BACKGROUND))
    cameras: list = field(default_factory=list)  # dicts for CameraModel(**cam)

    FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
              "raw_opacity_b")

    def __len__(self):
        return self.mu.shape[0]

    def as_float64(self):
        """Same values as float64 arrays (exact: every value is a float32)."""
        out = SceneArrays(**{f: getattr(self, f).astype(np.float64) for f in self.FIELDS},
                          sh_degree=self.sh_degree,
                          background_color=np.asarray(self.background_color, dtype=np.float64),
                          cameras=self.cameras)
        return out


def _logit(p):
    return np.log(p) - np.log1p(-p)  # geometry.py:355-358


def _unit(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _common_tail(rng, n, sh):
    k = (sh + 1) ** 2
    rotation = rng.normal(size=(n, 4))
    normal = _unit(rng.normal(size=(n, 3)))
    dc = rng.uniform(-0.8, 0.8, (n, 1, 3))
    rest = rng.uniform(-0.2, 0.2, (n, k - 1, 3))
    sh_coeffs = np.concatenate([dc, rest], axis=1)
    raw_a = _logit(rng.uniform(0.05, 0.95, n))
    raw_b = _logit(rng.uniform(0.05, 0.95, n))
    return rotation, normal, sh_coeffs, raw_a, raw_b


def _pack(mu, log_scale, rest, sh, cameras):
    rotation, normal, sh_coeffs, raw_a, raw_b = rest
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return SceneArrays(mu=f32(mu), log_scale=f32(log_scale), rotation=f32(rotation),
                       sh_coeffs=f32(sh_coeffs), normal=f32(normal), raw_opacity_a=f32(raw_a),
                       raw_opacity_b=f32(raw_b), sh_degree=sh,
                       background_color=np.array(BACKGROUND), cameras=cameras)


def frustum(n, sh, width, height, seed=0, sig_lo=0.5, sig_hi=4.0, clustered=False, dup=0.0):
    """Gaussians filling the view frustum of an identity camera, depth 2..6."""
    rng = np.random.default_rng(seed)
    f = 0.9 * width
    if clustered:
        z = rng.choice([3.0, 3.5, 4.0, 4.5], n) + rng.normal(0.0, 1e-3, n)
    else:
        z = rng.uniform(2.0, 6.0, n)
    x = rng.uniform(-1.1, 1.1, n) * z * (width / 2.0) / f
    y = rng.uniform(-1.1, 1.1, n) * z * (height / 2.0) / f
    mu = np.stack([x, y, z], axis=1)
    if dup > 0:
        m = int(dup * n)
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        mu[dst] = mu[src]
    sigma = np.exp(rng.uniform(np.log(sig_lo), np.log(sig_hi), (n, 3)))
    log_scale = np.log(sigma * mu[:, 2:3] / f)
    rest = _common_tail(rng, n, sh)
    cam = dict(world_to_cam=np.eye(4), fx=f, fy=f, cx=width / 2.0, cy=height / 2.0,
               width=width, height=height)
    return _pack(mu, log_scale, rest, sh, [cam])


def look_at_matrix(position, target, up=(0.0, 1.0, 0.0)):
    """world_to_cam of CameraModel.look_at (geometry.py:237-256)."""
    position = np.asarray(position, dtype=np.float64)
    forward = np.asarray(target, dtype=np.float64) - position
    forward = forward / np.linalg.norm(forward)
    up = np.asarray(up, dtype=np.float64)
    right = np.cross(forward, up)
    if np.linalg.norm(right) < 1e-9:
        up = np.array([0.0, 0.0, 1.0])
        right = np.cross(forward, up)
    right = right / np.linalg.norm(right)
    down = np.cross(forward, right)
    w2c = np.eye(4)
    w2c[:3, :3] = np.stack([right, down, forward])
    w2c[:3, 3] = -w2c[:3, :3] @ position
    return w2c


def ball(n, sh, width, height, views=8, seed=0):
    """Gaussians filling the unit ball, seen by `views` cameras on a ring of radius 3."""
    rng = np.random.default_rng(seed)
    f = 0.9 * width
    v = _unit(rng.normal(size=(n, 3)))
    mu = v * rng.uniform(0.0, 1.0, (n, 1)) ** (1.0 / 3.0)
    log_scale = np.log(np.exp(rng.uniform(np.log(0.5), np.log(4.0), (n, 3))) * 3.0 / f)
    rest = _common_tail(rng, n, sh)
    cams = []
    for i in range(views):
        th = 2.0 * np.pi * i / views
        w2c = look_at_matrix((3.0 * np.cos(th), -0.5, 3.0 * np.sin(th)), (0.0, 0.0, 0.0))
        cams.append(dict(world_to_cam=w2c, fx=f, fy=f, cx=width / 2.0, cy=height / 2.0,
                         width=width, height=height))
    return _pack(mu, log_scale, rest, sh, cams)


CONFIGS = {
    "c1": dict(kind="frustum", args=(10_000, 0, 128, 128), kw=dict(seed=0), backward=False),
    "c2": dict(kind="ball", args=(100_000, 3, 800, 800), kw=dict(views=8, seed=0), backward=True),
    "c3": dict(kind="frustum", args=(1_000_000, 3, 1920, 1080), kw=dict(seed=0), backward=True),
    "c4": dict(kind="ball", args=(3_000_000, 3, 1297, 840), kw=dict(views=8, seed=0),
               backward=True),
    "c5": dict(kind="frustum", args=(500_000, 3, 3840, 2160),
               kw=dict(seed=0, sig_lo=8.0, sig_hi=40.0, clustered=True, dup=0.1), backward=True),
}


def make_config(name):
    cfg = CONFIGS[name]
    fn = frustum if cfg["kind"] == "frustum" else ball
    return fn(*cfg["args"], **cfg["kw"])


def cotangent(height, width, seed=1):
    """Fixed cotangent d_color (tests/test_rasterizer.py:180 convention)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (height, width, 3))
