"""PyTorch autograd front end: rasterization settings + a differentiable forward
over means, half-Gaussian splitting normals, the two opacity logits, log-scales,
quaternions and SH coefficients, returning the image and radii.

The backward is the exact analytic backward of the reference (render_backward,
rasterizer.py:386-575) for the colour output, run by the same sm_100a kernels
as ``device.render_backward`` (K6 blend backward + K7 geometry backward).  As in
the reference, alpha and depth are outputs without gradients.

Parameters follow the reference Scene (geometry.py:364-378): log-scales and
opacity logits are the optimised quantities (no activation is applied here),
the quaternion is (w, x, y, z) and need not be normalised.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .geometry import CameraModel, Scene


@dataclass
class HalfGaussianRasterizationSettings:
    """Camera + render settings (CameraModel, geometry.py:210-235, plus the
    scene-level background / SH degree and the kernel switch)."""

    image_height: int
    image_width: int
    world_to_cam: np.ndarray  # (4, 4) row-major, +z forward, y down
    fx: float
    fy: float
    cx: float
    cy: float
    sh_degree: int
    background: tuple = (0.0, 0.0, 0.0)
    kernel: str = "half"      # "half" | "full" (plain Gaussians, rasterizer.py:259-262)
    near_clip: float = 0.01

    def camera(self):
        return CameraModel(self.world_to_cam, self.fx, self.fy, self.cx, self.cy,
                           self.image_width, self.image_height, self.near_clip)


class _RasterizeHalfGaussians(torch.autograd.Function):
    @staticmethod
    def forward(ctx, means3D, log_scales, rotations, shs, normals, raw_opacity_a, raw_opacity_b,
                settings):
        scene = Scene(means3D, log_scales, rotations, shs, normals, raw_opacity_a, raw_opacity_b,
                      sh_degree=settings.sh_degree, background_color=settings.background,
                      device=means3D.device, dtype=means3D.dtype, validate=False)
        scene.check_shapes()  # shape-only: no device sync on the autograd path
        cam = settings.camera()
        out = device.render(scene, cam, settings.kernel)
        ctx.scene, ctx.cam, ctx.out = scene, cam, out
        ctx.mark_non_differentiable(out.radii, out.alpha, out.depth)
        return out.color, out.radii, out.alpha, out.depth

    @staticmethod
    def backward(ctx, d_color, _d_radii, _d_alpha, _d_depth):
        if d_color is None:
            return (None,) * 8
        g = device.render_backward(ctx.scene, ctx.cam, ctx.out, d_color)
        ctx.scene = ctx.out = None
        return (g.d_mu, g.d_log_scale, g.d_rotation, g.d_sh, g.d_normal, g.d_raw_opacity_a,
                g.d_raw_opacity_b, None)


def rasterize_half_gaussians(means3D, normals, raw_opacity_a, raw_opacity_b, log_scales,
                             rotations, shs, settings):
    """Differentiable render of one view.

    Shapes: means3D (N,3), normals (N,3), raw_opacity_a/b (N,), log_scales
    (N,3), rotations (N,4), shs (N,(deg+1)^2,3), all on one CUDA device, float32
    or float64.  Returns color (H,W,3), radii (N,) int32 (0 = culled), alpha
    (H,W), depth (H,W)."""
    return _RasterizeHalfGaussians.apply(
        means3D.contiguous(), log_scales.contiguous(), rotations.contiguous(), shs.contiguous(),
        normals.contiguous(), raw_opacity_a.contiguous(), raw_opacity_b.contiguous(), settings)


class HalfGaussianRasterizer(torch.nn.Module):
    """Module form: settings at construction, parameters per call."""

    def __init__(self, raster_settings):
        super().__init__()
        self.raster_settings = raster_settings

    def forward(self, means3D, normals, raw_opacity_a, raw_opacity_b, log_scales, rotations, shs):
        color, radii, _, _ = rasterize_half_gaussians(means3D, normals, raw_opacity_a,
                                                      raw_opacity_b, log_scales, rotations, shs,
                                                      self.raster_settings)
        return color, radii
