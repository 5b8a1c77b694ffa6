"""Camera and scene containers for the device rasterizer.

Conventions are the reference's (geometry.py:3-10): world_to_cam maps into a
right-handed camera frame with +z forward, x right, y down; pixel (row i, col j)
has its centre at (j + 0.5, i + 0.5); scales are logs, opacities logits, the
quaternion is (w, x, y, z) and need not be normalised.

`Scene` keeps the seven parameter arrays as contiguous CUDA tensors (float32 or
float64).  Any object with the reference Scene's attributes (for instance a
``halfsplat.geometry.Scene``) can be passed where a Scene is expected; it is
uploaded once with ``Scene.from_any``.
"""

import numpy as np
import torch

DEFAULT_NEAR_CLIP = 0.01  # geometry.py:21
_SH_COUNTS = {0: 1, 1: 4, 2: 9, 3: 16}  # geometry.py:361


class CameraModel:
    """Pinhole camera, same fields and validation as geometry.py:210-273."""

    def __init__(self, world_to_cam, fx, fy, cx, cy, width, height, near_clip=DEFAULT_NEAR_CLIP):
        self.world_to_cam = np.asarray(world_to_cam, dtype=np.float64)
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.width, self.height = int(width), int(height)
        self.near_clip = float(near_clip)
        if self.world_to_cam.shape != (4, 4):
            raise ValueError("world_to_cam must be 4x4")
        r = self.world_to_cam[:3, :3]
        if np.abs(r.T @ r - np.eye(3)).max() >= 1e-6:
            raise ValueError("world_to_cam rotation block is not orthonormal")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point outside the image")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image dimensions must be positive")

    @classmethod
    def look_at(cls, position, target, width, height, focal, up=(0, 1, 0),
                near_clip=DEFAULT_NEAR_CLIP):
        """Camera at `position` aimed at `target`, y-down image (geometry.py:237-256)."""
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
        return cls(world_to_cam=w2c, fx=focal, fy=focal, cx=width / 2.0, cy=height / 2.0,
                   width=width, height=height, near_clip=near_clip)

    @classmethod
    def from_any(cls, cam):
        if isinstance(cam, cls):
            return cam
        return cls(cam.world_to_cam, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                   getattr(cam, "near_clip", DEFAULT_NEAR_CLIP))

    @property
    def rotation(self):
        return self.world_to_cam[:3, :3]

    @property
    def translation(self):
        return self.world_to_cam[:3, 3]

    @property
    def center(self):
        return -self.rotation.T @ self.translation


def _to_tensor(x, dtype, device):
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        # pinned host fields upload asynchronously (one DMA per field, no sync between
        # them); Scene.__init__ synchronises once after the last one
        return t.to(device, non_blocking=t.is_pinned()).contiguous()
    a = np.asarray(x)
    if dtype is None:
        dtype = torch.float64 if a.dtype == np.float64 else torch.float32
    src = torch.as_tensor(np.ascontiguousarray(a))
    if device.type != "cuda" or src.numel() * src.element_size() < _STAGE_MIN_BYTES:
        return src.to(dtype).to(device).contiguous()
    return _staged_upload(src, dtype, device)


# Host arrays above this size go up through pinned staging (pageable H2D copies run at
# about a third of the pinned rate on the B200 boxes: 19 vs 55 GB/s).
_STAGE_MIN_BYTES = 1 << 20
_STAGE_CHUNK_BYTES = 16 << 20


def _staged_upload(src, dtype, device):
    """Pageable host tensor -> device, through pinned staging in chunks: the host
    copy (and dtype conversion) of one chunk overlaps the DMA of the previous one.
    The staging blocks come from torch's caching host allocator, which recycles a
    block only after its copy has completed, and the caller's array is free to change
    as soon as this returns (the host copies are synchronous), so no sync is needed."""
    flat = src.reshape(-1)
    dst = torch.empty(src.shape, dtype=dtype, device=device)
    dflat = dst.view(-1)
    step = max(1, _STAGE_CHUNK_BYTES // max(src.element_size(), dst.element_size()))
    for i in range(0, flat.numel(), step):
        chunk = flat[i:i + step]
        stage = torch.empty(chunk.shape, dtype=dtype, pin_memory=True)
        stage.copy_(chunk)
        dflat[i:i + step].copy_(stage, non_blocking=True)
    return dst


class Scene:
    """Struct-of-arrays half-Gaussian scene resident on one GPU (geometry.py:364-407)."""

    FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
              "raw_opacity_b")

    def __init__(self, mu, log_scale, rotation, sh_coeffs, normal, raw_opacity_a, raw_opacity_b,
                 sh_degree, background_color=(0.0, 0.0, 0.0), device="cuda", dtype=None,
                 validate=True):
        if dtype is None:
            probe = mu if isinstance(mu, torch.Tensor) else np.asarray(mu)
            dtype = torch.float64 if probe.dtype in (np.float64, torch.float64) else torch.float32
        self.device = torch.device(device)
        self.dtype = dtype
        self.mu = _to_tensor(mu, dtype, self.device)
        self.log_scale = _to_tensor(log_scale, dtype, self.device)
        self.rotation = _to_tensor(rotation, dtype, self.device)
        self.sh_coeffs = _to_tensor(sh_coeffs, dtype, self.device)
        self.normal = _to_tensor(normal, dtype, self.device)
        self.raw_opacity_a = _to_tensor(raw_opacity_a, dtype, self.device)
        self.raw_opacity_b = _to_tensor(raw_opacity_b, dtype, self.device)
        self.sh_degree = int(sh_degree)
        self.background_color = np.asarray(background_color, dtype=np.float64).reshape(3)
        srcs = (mu, log_scale, rotation, sh_coeffs, normal, raw_opacity_a, raw_opacity_b)
        if self.device.type == "cuda" and any(isinstance(x, torch.Tensor) and x.is_pinned()
                                              for x in srcs):
            # the caller may reuse its host buffers as soon as the scene exists
            torch.cuda.current_stream(self.device).synchronize()
        if validate:
            self._validate()

    def _validate(self):
        self.check_shapes()
        if self.mu.shape[0] and bool((self.normal.norm(dim=1) == 0).any()):
            raise ValueError("zero-length splitting normal")
        if self.mu.shape[0] and bool((self.rotation.norm(dim=1) == 0).any()):
            raise ValueError("zero quaternion")
        bg = self.background_color
        if np.any((bg < 0) | (bg > 1)):
            raise ValueError("background_color must be a 3-vector in [0, 1]")

    def check_shapes(self):
        """The shape part of the validation (geometry.py:385-407): reads only
        .shape, so it costs no device work.  K1/K7 index SH with the stride of
        sh_degree, so a mismatch here would be an out-of-bounds device read."""
        n = self.mu.shape[0]
        if self.sh_degree not in _SH_COUNTS:
            raise ValueError("sh_degree must be 0..3")
        want = _SH_COUNTS[self.sh_degree]
        if tuple(self.sh_coeffs.shape) != (n, want, 3):
            raise ValueError(f"sh_coeffs shape {tuple(self.sh_coeffs.shape)} does not match "
                             f"degree {self.sh_degree} (expected {(n, want, 3)})")
        for name, width in (("mu", 3), ("log_scale", 3), ("rotation", 4), ("normal", 3)):
            if tuple(getattr(self, name).shape) != (n, width):
                raise ValueError(f"{name} must have shape {(n, width)}")
        if tuple(self.raw_opacity_a.shape) != (n,) or tuple(self.raw_opacity_b.shape) != (n,):
            raise ValueError("opacity logits must be 1D of length N")

    def __len__(self):
        return int(self.mu.shape[0])

    @classmethod
    def from_any(cls, scene, device="cuda", dtype=None):
        """Upload a reference-style scene (numpy SoA) or return a device Scene as is."""
        if isinstance(scene, cls) and (dtype is None or scene.dtype == dtype):
            return scene
        return cls(*(getattr(scene, f) for f in cls.FIELDS), sh_degree=scene.sh_degree,
                   background_color=getattr(scene, "background_color", (0.0, 0.0, 0.0)),
                   device=device, dtype=dtype)

    def numpy(self):
        """Host float64 copies of the parameter arrays (for oracles and I/O)."""
        return {f: getattr(self, f).detach().double().cpu().numpy() for f in self.FIELDS}
