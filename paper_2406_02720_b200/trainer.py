"""Device-resident training step: render -> loss -> backward -> Adam, all on the GPU.

Mirror of the reference's optimizer path (trainer.py:22-226): the same names
(`TrainConfig`, `GROUPS`, `AdamState`, `mu_learning_rate`, `learning_rates`,
`active_groups`, `camera_extent`, `step`) with the same argument meaning, but
the scene, its gradients and the Adam moments are CUDA tensors and the update is
one `hs_adam_step` launch (csrc/hs_adam.cu).  The learning-rate schedule is
scalar host arithmetic, evaluated exactly as the reference does.

Density control (trainer.py:229-350) runs on the device too: `DensifyStats`,
`densify_and_prune` (hs_densify_plan_compute + hs_densify_apply) and
`reset_opacity`.  The run loop / metrics / checkpoints are not part of this module.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, device
from .errors import NonFiniteLoss
from .loss import DeviceLoss

ADAM_BETA1 = 0.9    # trainer.py:23
ADAM_BETA2 = 0.999  # trainer.py:24
ADAM_EPS = 1e-15    # trainer.py:25

MODES = ("from_scratch", "finetune_all", "finetune_all_with_densify",
         "finetune_normals_opacities")

# parameter groups (trainer.py:81-82) and the scene field each lives in
GROUPS = ("mu", "log_scale", "rotation", "sh_dc", "sh_rest", "normal",
          "opacity_a", "opacity_b")
_STATE_FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
                 "raw_opacity_b")
_GROUP_FIELD = {"mu": 0, "log_scale": 1, "rotation": 2, "sh_dc": 3, "sh_rest": 3, "normal": 4,
                "opacity_a": 5, "opacity_b": 6}


@dataclass
class TrainConfig:
    """trainer.py:31-76 (same fields, defaults and validation)."""

    total_iters: int = 30000
    densify_until: int = 20000
    densify_interval: int = 100
    opacity_reset_start: int = 3000
    opacity_reset_interval: int = 3000
    opacity_reset_until: int = 20000
    opacity_reset_ceiling: float = 0.01
    lambda_ssim: float = 0.2
    lr_normal: float = 0.003
    lr_mu_init: float = 1.6e-4
    lr_mu_final: float = 1.6e-6
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    lr_sh_dc: float = 2.5e-3
    sh_rest_divisor: float = 20.0
    lr_opacity: float = 5e-2
    densify_grad_threshold: float = 2e-4
    prune_opacity_threshold: float = 0.005
    percent_dense: float = 0.01
    prune_extent_factor: float = 0.1
    split_scale_factor: float = 1.6
    max_primitives: int = 0
    mode: str = "from_scratch"
    kernel: str = "half"
    seed: int = 0
    threads: int = 0
    checkpoint_interval: int = 0

    def __post_init__(self):
        if not (0 < self.densify_until <= self.total_iters):
            raise ValueError("require 0 < densify_until <= total_iters")
        if not (0.0 <= self.lambda_ssim <= 1.0):
            raise ValueError("lambda_ssim must lie in [0, 1]")
        for name in ("lr_mu_init", "lr_mu_final", "lr_scale", "lr_rotation",
                     "lr_sh_dc", "lr_opacity"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.lr_normal < 0:
            raise ValueError("lr_normal must be >= 0")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.kernel not in ("half", "full"):
            raise ValueError("kernel must be 'half' or 'full'")


class AdamState:
    """First/second moments per parameter group, row-aligned with the scene
    (trainer.py:110-136).  Moments are device tensors shaped like the scene
    fields; `m[name]` / `v[name]` give the group's view (sh_dc / sh_rest are
    slices of the sh_coeffs moments)."""

    def __init__(self, scene):
        self._m = [torch.zeros_like(getattr(scene, f)) for f in _STATE_FIELDS]
        self._v = [torch.zeros_like(getattr(scene, f)) for f in _STATE_FIELDS]
        self.t = {name: 0 for name in GROUPS}

    @staticmethod
    def _view(arrays, name):
        a = arrays[_GROUP_FIELD[name]]
        if name == "sh_dc":
            return a[:, :1, :]
        if name == "sh_rest":
            return a[:, 1:, :]
        return a

    @property
    def m(self):
        return {name: self._view(self._m, name) for name in GROUPS}

    @property
    def v(self):
        return {name: self._view(self._v, name) for name in GROUPS}

    def select(self, keep):
        keep = torch.as_tensor(keep, device=self._m[0].device)
        self._m = [a[keep].contiguous() for a in self._m]
        self._v = [a[keep].contiguous() for a in self._v]

    def append_zeros(self, count):
        self._m = [torch.cat([a, a.new_zeros((count,) + a.shape[1:])]) for a in self._m]
        self._v = [torch.cat([a, a.new_zeros((count,) + a.shape[1:])]) for a in self._v]

    def zero_group(self, name):
        self._view(self._m, name).zero_()
        self._view(self._v, name).zero_()
        self.t[name] = 0

    def struct(self):
        s = _native.HsAdamState()
        for k in range(7):
            s.m[k] = self._m[k].data_ptr()
            s.v[k] = self._v[k].data_ptr()
        for k, name in enumerate(GROUPS):
            s.t[k] = self.t[name]
        return s


def mu_learning_rate(config, iteration, spatial_scale):
    """Exponential decay from lr_mu_init to lr_mu_final (trainer.py:139-143)."""
    frac = min(max(iteration / config.total_iters, 0.0), 1.0)
    lr = config.lr_mu_init * (config.lr_mu_final / config.lr_mu_init) ** frac
    return lr * spatial_scale


def learning_rates(config, iteration, spatial_scale):
    """trainer.py:146-156."""
    return {
        "mu": mu_learning_rate(config, iteration, spatial_scale),
        "log_scale": config.lr_scale,
        "rotation": config.lr_rotation,
        "sh_dc": config.lr_sh_dc,
        "sh_rest": config.lr_sh_dc / config.sh_rest_divisor,
        "normal": config.lr_normal,
        "opacity_a": config.lr_opacity,
        "opacity_b": config.lr_opacity,
    }


def active_groups(config):
    """trainer.py:159-166."""
    if config.mode == "finetune_normals_opacities":
        groups = {"normal", "opacity_a", "opacity_b"}
    else:
        groups = set(GROUPS)
    if config.kernel == "full":
        groups.discard("normal")
    return groups


def camera_extent(cameras):
    """Radius of the camera-centre bounding sphere (trainer.py:169-176)."""
    centers = np.stack([np.asarray(cam.center, dtype=np.float64) for cam in cameras])
    if centers.shape[0] < 2:
        return 1.0
    centroid = centers.mean(axis=0)
    radius = np.linalg.norm(centers - centroid, axis=1).max()
    return float(radius) if radius > 0 else 1.0


def adam_step(scene, grads, config, opt_state, iteration, spatial_scale=1.0):
    """The Adam part of step() (trainer.py:192-224) as one device launch."""
    lrs = learning_rates(config, iteration, spatial_scale)
    enabled = active_groups(config)
    lr = (ctypes.c_double * 8)(*[(lrs[g] if g in enabled else 0.0) for g in GROUPS])
    g = _grads_struct(grads)
    st = opt_state.struct()
    sc = device.scene_struct(scene)
    lib = _native.load()
    _native.check(lib.hs_adam_step(ctypes.byref(sc), ctypes.byref(g), ctypes.byref(st), lr,
                                   1 if config.kernel == "full" else 0, device._stream()),
                  "hs_adam_step")
    for k, name in enumerate(GROUPS):
        opt_state.t[name] = int(st.t[k])


def _grads_struct(grads):
    g = _native.HsGrads()
    for name in device.DeviceGradientSet.NAMES:
        setattr(g, name, getattr(grads, name).data_ptr())
    return g


class DensifyStats:
    """Screen-space gradient statistics between densify events (trainer.py:229-244),
    float64 / int64 device tensors."""

    def __init__(self, grad_sum, mu_grad_sum, count):
        self.grad_sum, self.mu_grad_sum, self.count = grad_sum, mu_grad_sum, count

    @classmethod
    def zeros(cls, n, device="cuda"):
        return cls(torch.zeros(n, dtype=torch.float64, device=device),
                   torch.zeros((n, 3), dtype=torch.float64, device=device),
                   torch.zeros(n, dtype=torch.int64, device=device))

    def struct(self):
        s = _native.HsDensifyStats()
        s.grad_sum = self.grad_sum.data_ptr()
        s.mu_grad_sum = self.mu_grad_sum.data_ptr()
        s.count = self.count.data_ptr()
        return s

    def update(self, grads):
        """DensifyStats.update (trainer.py:241-244), one launch."""
        n = self.grad_sum.shape[0]
        dt = _native.HS_DTYPE_F64 if grads.d_mu.dtype == torch.float64 else _native.HS_DTYPE_F32
        st = self.struct()
        _native.check(_native.load().hs_densify_stats_update(
            ctypes.byref(st), ctypes.byref(_grads_struct(grads)), n, dt, device._stream()),
            "hs_densify_stats_update")


def densify_and_prune(scene, stats, config, opt_state, rng, scene_extent):
    """Clone small / split large high-gradient primitives, prune weak ones
    (trainer.py:247-340).  Returns (scene, stats, report); `opt_state` is re-aligned
    with the new rows in place.

    `rng`: a numpy Generator draws the split offsets exactly as the reference
    does (two rng.normal((k, 3)) calls, only when k > 0), so a float64 scene
    densifies bit-identically; an int (or None) seeds the device Philox draw."""
    from .geometry import Scene
    lib = _native.load()
    n = len(scene)
    ws = torch.empty(max(lib.hs_densify_workspace_size(n), 1), dtype=torch.uint8,
                     device=scene.device)
    cfg = _native.HsDensifyConfig(
        config.densify_grad_threshold, config.prune_opacity_threshold, config.percent_dense,
        config.prune_extent_factor, float(scene_extent),
        float(np.log(config.split_scale_factor)), int(config.max_primitives))
    sc = device.scene_struct(scene)
    st = stats.struct()
    plan = _native.HsDensifyPlan()
    s = device._stream()
    _native.check(lib.hs_densify_plan_compute(ctypes.byref(sc), ctypes.byref(st),
                                              ctypes.byref(cfg), ctypes.byref(plan),
                                              ws.data_ptr(), ws.numel(), s),
                  "hs_densify_plan_compute")
    m = int(plan.n_out)
    k = (scene.sh_degree + 1) ** 2
    def alloc(*shape):
        return torch.empty(shape, dtype=scene.dtype, device=scene.device)

    new = Scene(alloc(m, 3), alloc(m, 3), alloc(m, 4), alloc(m, k, 3), alloc(m, 3), alloc(m),
                alloc(m), sh_degree=scene.sh_degree, background_color=scene.background_color,
                device=scene.device, dtype=scene.dtype, validate=False)
    offsets, seed = None, 0
    if isinstance(rng, np.random.Generator):
        if plan.split:
            draws = [rng.normal(size=(int(plan.split), 3)) for _ in range(2)]
            offsets = torch.as_tensor(np.stack(draws), dtype=torch.float64, device=scene.device)
    else:
        seed = int(rng or 0)
    new_state = None
    sin = sout = None
    if opt_state is not None:
        new_m = [torch.empty((m,) + a.shape[1:], dtype=a.dtype, device=a.device)
                 for a in opt_state._m]
        new_v = [torch.empty_like(a) for a in new_m]
        sin = opt_state.struct()
        sout = _native.HsAdamState()
        for f in range(7):
            sout.m[f] = new_m[f].data_ptr()
            sout.v[f] = new_v[f].data_ptr()
        new_state = (new_m, new_v)
    out = device.scene_struct(new)
    _native.check(lib.hs_densify_apply(
        ctypes.byref(sc), ctypes.byref(st), ctypes.byref(cfg), ctypes.byref(plan),
        ws.data_ptr(), ws.numel(), offsets.data_ptr() if offsets is not None else None, seed,
        ctypes.byref(sin) if sin is not None else None, ctypes.byref(out),
        ctypes.byref(sout) if sout is not None else None, s), "hs_densify_apply")
    if new_state is not None:
        opt_state._m, opt_state._v = new_state
    report = {"cloned": int(plan.cloned), "split": int(plan.split), "pruned": int(plan.pruned)}
    return new, DensifyStats.zeros(m, scene.device), report


def reset_opacity(scene, opt_state=None, ceiling=0.01):
    """Clamp both opacity logits so sigmoid <= ceiling (trainer.py:343-350)."""
    p = np.float64(ceiling)
    cap = float(np.log(p) - np.log1p(-p))  # logit, geometry.py:355-358
    st = opt_state.struct() if opt_state is not None else None
    sc = device.scene_struct(scene)
    _native.check(_native.load().hs_reset_opacity(
        ctypes.byref(sc), cap, ctypes.byref(st) if st is not None else None, device._stream()),
        "hs_reset_opacity")
    if opt_state is not None:
        opt_state.t["opacity_a"] = 0
        opt_state.t["opacity_b"] = 0


def opacity_disparity(scene):
    """Mean |alpha1 - alpha2| over the scene (trainer.py:353-358), one device reduction."""
    from .errors import EmptyScene
    n = len(scene)
    if n == 0:
        raise EmptyScene("opacity_disparity of an empty scene")
    lib = _native.load()
    ws = torch.empty(max(lib.hs_opacity_disparity_workspace_size(n), 1), dtype=torch.uint8,
                     device=scene.device)
    out = torch.empty(1, dtype=torch.float64, device=scene.device)
    sc = device.scene_struct(scene)
    _native.check(lib.hs_opacity_disparity(ctypes.byref(sc), ctypes.c_void_p(out.data_ptr()),
                                           ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                           device._stream()), "hs_opacity_disparity")
    return float(out.item()) / n


class StepRunner:
    """Persistent buffers for repeated steps: one rasterizer workspace, one
    gradient set (re-allocated when density control changes N), one loss
    workspace."""

    def __init__(self, scene, config):
        self.config = config
        self.rast = device.Rasterizer(scene.device, slots=1, kernel=config.kernel)
        self.grads = device.DeviceGradientSet.empty_flat(scene)
        self.loss = DeviceLoss(config.lambda_ssim)
        self.last_stats = None  # [loss, L1, SSIM, MSE] of the last step (device)

    def step(self, scene, batch_view, opt_state, iteration, spatial_scale=1.0,
             check_finite=True):
        cam, target = batch_view
        if not isinstance(target, torch.Tensor):
            target = torch.as_tensor(np.asarray(target, dtype=np.float32))
        target = target.to(device=scene.device, dtype=torch.float32)
        if self.grads.d_mu.shape[0] != len(scene):
            self.grads = device.DeviceGradientSet.empty_flat(scene)
        out = self.rast.render(scene, cam)
        stats, d_color = self.loss(out.color, target)
        loss = stats[0]
        if check_finite:
            loss = float(loss)  # trainer.py:189-190 (one 8-byte read)
            if out.frame.resolve():
                # binned with P on the device past the workspace's capacity (e.g. right
                # after density control grew the scene): re-binned, blend it again
                out = self.rast.render(scene, cam)
                stats, d_color = self.loss(out.color, target)
                loss = float(stats[0])
            if not math.isfinite(loss):
                raise NonFiniteLoss(iteration, loss)
        self.last_stats = stats
        self.rast.render_backward(scene, cam, out, d_color, grads=self.grads)
        adam_step(scene, self.grads, self.config, opt_state, iteration, spatial_scale)
        return loss, self.grads, out


def step(scene, batch_view, config, opt_state, iteration, spatial_scale=1.0, threads=None):
    """One optimisation step on a (camera, target image) pair (trainer.py:179-226).

    Returns (loss, grads, out) like the reference; grads/out are device objects.
    `threads` is accepted and ignored.  Repeated callers should hold a StepRunner."""
    runner = getattr(opt_state, "_runner", None)
    if runner is None or runner.config is not config:
        runner = StepRunner(scene, config)
        opt_state._runner = runner
    return runner.step(scene, batch_view, opt_state, iteration, spatial_scale)


METRICS_FIELDS = ("iteration", "loss", "psnr", "num_primitives",
                  "opacity_disparity", "cloned", "split", "pruned",
                  "opacity_reset")


class Trainer:
    """Drives the full schedule over a fixed set of training views (trainer.py:365-449),
    every tensor on the GPU.

    Same constructor, `run`, `write_metrics` and `metrics_rows` as the reference.
    The view order and the split offsets come from one numpy Generator seeded with
    config.seed, consumed in the reference's order, so a run makes the same
    density-control decisions as the reference would on the same gradients.
    Targets are uploaded once."""

    def __init__(self, scene, views, config, metrics_path=None, checkpoint_fn=None):
        from .geometry import Scene
        self.scene = Scene.from_any(scene)
        self.views = list(views)  # (name, CameraModel, target image)
        if not self.views:
            raise ValueError("need at least one training view")
        self.config = config
        self.rng = np.random.default_rng(config.seed)
        self.opt = AdamState(self.scene)
        self.stats = DensifyStats.zeros(len(self.scene), self.scene.device)
        self.spatial_scale = camera_extent([v[1] for v in self.views])
        self.metrics_path = metrics_path
        self.checkpoint_fn = checkpoint_fn
        self._metrics_rows = []
        self._order = []
        self._targets = [torch.as_tensor(np.asarray(t, dtype=np.float32)).to(self.scene.device)
                         for _, _, t in self.views]
        self._runner = StepRunner(self.scene, config)

    def _next_view(self):
        if not self._order:
            self._order = list(self.rng.permutation(len(self.views)))
        return self._order.pop()

    def densify_enabled(self):
        return self.config.mode in ("from_scratch", "finetune_all_with_densify")

    def run(self, progress=None):
        cfg = self.config
        for iteration in range(1, cfg.total_iters + 1):
            v = self._next_view()
            _, cam, _ = self.views[v]
            loss, grads, out = self._runner.step(
                self.scene, (cam, self._targets[v]), self.opt, iteration, self.spatial_scale)
            self.stats.update(grads)
            report = {"cloned": 0, "split": 0, "pruned": 0}
            did_reset = 0
            if (self.densify_enabled() and iteration % cfg.densify_interval == 0
                    and iteration < cfg.densify_until):
                self.scene, self.stats, report = densify_and_prune(
                    self.scene, self.stats, cfg, self.opt, self.rng, self.spatial_scale)
            if (cfg.opacity_reset_start <= iteration <= cfg.opacity_reset_until
                    and iteration % cfg.opacity_reset_interval == 0):
                reset_opacity(self.scene, self.opt, cfg.opacity_reset_ceiling)
                did_reset = 1
            mse = float(self._runner.last_stats[3])
            row = {
                "iteration": iteration,
                "loss": loss,
                "psnr": math.inf if mse == 0.0 else float(10.0 * np.log10(1.0 / mse)),
                "num_primitives": len(self.scene),
                "opacity_disparity": opacity_disparity(self.scene),
                "cloned": report["cloned"],
                "split": report["split"],
                "pruned": report["pruned"],
                "opacity_reset": did_reset,
            }
            self._metrics_rows.append(row)
            if progress and iteration % progress == 0:
                print(f"iter {iteration:>6}  loss {loss:.5f}  prims {len(self.scene)}")
            if (self.checkpoint_fn and cfg.checkpoint_interval
                    and iteration % cfg.checkpoint_interval == 0):
                self.checkpoint_fn(self.scene, iteration)
        if self.metrics_path:
            self.write_metrics(self.metrics_path)
        if self.checkpoint_fn:
            self.checkpoint_fn(self.scene, cfg.total_iters)
        return self.scene

    def write_metrics(self, path):
        import csv
        with open(path, "w", newline="") as fh:
            writer = csv.DictWriter(fh, fieldnames=METRICS_FIELDS)
            writer.writeheader()
            writer.writerows(self._metrics_rows)

    @property
    def metrics_rows(self):
        return self._metrics_rows
