"""Device-resident rasterizer: the staged C-ABI pipeline driven from PyTorch.

prepare -> render -> render_backward here mirror rasterizer.py:159-421 of the
reference, but every tensor stays in HBM and every stage is one or more
sm_100a kernels of libhalfsplat_b200.so:

    prepare          hs_preprocess_fwd (K1 + depth-rank sort + count scan),
                     hs_read_pairs_and_bin (the one host sync: P, then K2 duplicate,
                     K3 stable tile sort, K4 ranges; hs_bin_and_sort after sizing the
                     binning workspace when it is too small)
    render           hs_blend_fwd (K5)
    render_backward  hs_blend_bwd (K6) + hs_preprocess_bwd (K7)

PyTorch only provides device memory (caching allocator) and the stream.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import EmptyScene, ImageTooLarge, MismatchedForward, WorkspaceError
from .geometry import CameraModel, Scene

MAX_PIXELS = 2**31  # rasterizer.py:40
TILE = 16


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def camera_struct(cam):
    c = _native.HsCamera()
    w2c = np.ascontiguousarray(cam.world_to_cam, dtype=np.float64).reshape(16)
    for k in range(16):
        c.world_to_cam[k] = float(w2c[k])
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.near_clip = cam.near_clip
    center = -cam.rotation.T @ cam.translation  # geometry.py:266-269
    for k in range(3):
        c.center[k] = float(center[k])
    c.width, c.height = cam.width, cam.height
    return c


def scene_struct(scene):
    s = _native.HsScene()
    s.n = len(scene)
    s.sh_degree = scene.sh_degree
    if scene.dtype == torch.float32:
        s.dtype = _native.HS_DTYPE_F32
    elif scene.dtype == torch.float64:
        s.dtype = _native.HS_DTYPE_F64
    else:
        raise TypeError(f"unsupported scene dtype {scene.dtype}")
    for f in Scene.FIELDS:
        setattr(s, f, getattr(scene, f).data_ptr())
    for k in range(3):
        s.background[k] = float(scene.background_color[k])
    return s


class Workspace:
    """Persistent device buffers for one in-flight view: the frame and binning
    workspaces, the image outputs and radii.  Reused across calls (grown when a
    larger scene/image/pair count needs it), so a steady training or benchmark
    loop performs no device allocation at all."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self._bufs = {}
        # asynchronous binning (hs_bin_async): the pair capacity the binning
        # workspace is laid out for, the last P read back, and the status copy of
        # the frame binned last (checked by the next prepare into this workspace)
        self.pair_capacity = 0
        self.last_pairs = -1
        self.pending = None
        self.generation = 0
        self._status_host = None
        self.depth_sort_full = 0  # sticky once a view needed the full depth sort
        self.capturing = False    # inside a CUDA-graph capture (CapturedStep)

    def status_buffer(self):
        """Pinned host memory for hs_frame_status_async (4 int64 words)."""
        if self._status_host is None:
            self._status_host = torch.zeros(4, dtype=torch.int64, pin_memory=True)
        return self._status_host

    def check_previous(self):
        """Status of the frame this workspace binned asynchronously last: waits
        for that frame's binning (the GPU is normally still busy with its blends,
        so this does not idle it) and raises BinningOverflow if its P exceeded the
        capacity -- its outputs were then empty.  The capacity grows either way
        when P comes near it."""
        pend, self.pending = self.pending, None
        if pend is None:
            return
        event, host, frame = pend
        event.synchronize()
        p, flags, depth = int(host[0]), int(host[2]) & 0xffffffff, int(host[3]) & 0xffffffff
        frame._status_seen(p, flags, depth)
        if flags or depth:
            raise BinningOverflow(
                f"an asynchronously binned view had P={p} pairs for a capacity of "
                f"{frame.capacity} (flags {flags}, depth fallback {depth}); its outputs were "
                "incomplete -- the capacity has grown, re-run that view")

    def tensor(self, name, shape, dtype):
        t = self._bufs.get(name)
        numel = int(np.prod(shape)) if len(shape) else 1
        if t is None or t.dtype != dtype or t.numel() < numel:
            t = torch.empty(numel, dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[:numel].view(shape)

    def bytes(self, name, nbytes):
        return self.tensor(name, (nbytes,), torch.uint8)


class BinningOverflow(RuntimeError):
    """An asynchronously binned view needed more pair capacity than its workspace
    had (see Workspace.check_previous)."""


# Capacity headroom of a binning workspace: P * 5/4 + 64K pairs, grown again once a
# view's P passes 90% of it.
def _capacity_for(p):
    return int(p) * 5 // 4 + 65536


class DeviceFrame:
    """One view's binned splats (the device counterpart of FrameGeometry)."""

    def __init__(self, scene, cam, kernel, ws=None):
        lib = _native.load()
        self.lib = lib
        self.kernel = kernel
        self.camera = cam
        self.st = _native.HsFrame()
        kcode = {"half": _native.HS_KERNEL_HALF, "full": _native.HS_KERNEL_FULL}[kernel]
        _native.check(lib.hs_frame_init(ctypes.byref(self.st), len(scene), cam.width,
                                        cam.height, kcode), "hs_frame_init")
        dev = scene.device
        self.ws = ws
        nbytes = lib.hs_frame_workspace_size(len(scene), cam.width, cam.height)
        if ws is not None:
            self.frame_ws = ws.bytes("frame_ws", nbytes)
            self.radii = ws.tensor("radii", (len(scene),), torch.int32)
        else:
            self.frame_ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self.radii = torch.empty(len(scene), dtype=torch.int32, device=dev)
        self.st.frame_ws = self.frame_ws.data_ptr()
        self.st.frame_ws_bytes = nbytes
        self.bin_ws = None
        self.device = dev
        self.pending = False   # binned asynchronously, P not read back yet
        self.capacity = 0
        if ws is not None:
            ws.generation += 1
            self.generation = ws.generation
            self.st.depth_sort_full = ws.depth_sort_full

    @property
    def n_total(self):
        return int(self.st.n)

    @property
    def num_pairs(self):
        self.resolve()
        if self.st.num_pairs < 0 and self.stale():
            raise WorkspaceError("this frame's workspace was reused by a later view")
        return int(self.st.num_pairs)

    def _status_seen(self, p, flags, depth):
        if self.ws is not None and depth:
            self.ws.depth_sort_full = 1
        if self.ws is not None:
            self.ws.last_pairs = max(self.ws.last_pairs, p) if flags or depth else p
            if p > 0.9 * self.ws.pair_capacity:
                self.ws.pair_capacity = 0  # re-lay the workspace out at the next prepare
                self.ws.last_pairs = p

    def resolve(self):
        """For an asynchronously binned frame: read P and the status (a host sync);
        if the frame overflowed its capacity (or its depth ranks needed the full
        sort) grow the workspace and bin it again synchronously.  Returns True when
        it re-binned, i.e. any blend already run on this frame must be redone."""
        if not self.pending:
            return False
        if self.ws is not None and self.ws.generation != self.generation:
            # the workspace was reused since: this frame's buffers (and its status)
            # belong to a later view, whose prepare checked this one's status
            self.pending = False
            return False
        self.pending = False
        if self.ws is not None and self.ws.pending is not None and self.ws.pending[2] is self:
            self.ws.pending = None
        p, flags = ctypes.c_int64(), ctypes.c_int32()
        _native.check(self.lib.hs_frame_status(ctypes.byref(self.st), ctypes.byref(p),
                                               ctypes.byref(flags), _stream()), "hs_frame_status")
        self._status_seen(p.value, flags.value & _native.HS_FRAME_PAIR_OVERFLOW,
                          flags.value & _native.HS_FRAME_DEPTH_FALLBACK)
        if flags.value == 0:
            return False
        if flags.value & _native.HS_FRAME_DEPTH_FALLBACK:
            # redoes the ranks with the full sort and re-reads P
            _native.check(self.lib.hs_frame_read_num_pairs(ctypes.byref(self.st), _stream()),
                          "hs_frame_read_num_pairs")
        else:
            self.st.num_pairs = p.value
        self.alloc_binning()
        _native.check(self.lib.hs_bin_and_sort(ctypes.byref(self.st), _stream()),
                      "hs_bin_and_sort")
        return True

    @property
    def tiles_x(self):
        return int(self.st.tiles_x)

    @property
    def tiles_y(self):
        return int(self.st.tiles_y)

    def reuse_binning(self):
        """Point the frame at the workspace's binning buffer and pair capacity (set
        by an earlier view), so it can bin without reading P first.  Returns the
        capacity (0: none yet, read P)."""
        if self.ws is None:
            return 0
        buf = self.ws._bufs.get("bin_ws")
        cap = self.ws.pair_capacity
        if buf is None or cap <= 0:
            return 0
        if buf.numel() < self.lib.hs_binning_workspace_size(self.st.n, cap, self.st.width,
                                                            self.st.height):
            return 0
        self.bin_ws = buf
        self.st.bin_ws = buf.data_ptr()
        self.st.bin_ws_bytes = buf.numel()
        self.st.pair_capacity = cap
        self.capacity = cap
        return cap

    def alloc_binning(self):
        """A binning workspace for the known P, with headroom for later views."""
        lib = self.lib
        p = int(self.st.num_pairs)
        cap = max(_capacity_for(p), self.ws.pair_capacity if self.ws is not None else 0)
        if self.ws is None:
            cap = p
        nbytes = lib.hs_binning_workspace_size(self.st.n, cap, self.st.width, self.st.height)
        if self.ws is not None:
            self.bin_ws = self.ws.bytes("bin_ws", nbytes)
            self.ws.pair_capacity = cap
            self.ws.last_pairs = p
        elif self.bin_ws is None or self.bin_ws.numel() < nbytes:
            self.bin_ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.st.bin_ws = self.bin_ws.data_ptr()
        self.st.bin_ws_bytes = self.bin_ws.numel()
        self.st.pair_capacity = cap
        self.capacity = cap

    def stale(self):
        """True once a later view was prepared into this frame's workspace."""
        return self.ws is not None and self.ws.generation != self.generation

    def export(self):
        """FrameGeometry integers/packed columns as host numpy arrays (parity)."""
        if self.stale():
            raise WorkspaceError("this frame's workspace was reused by a later view")
        self.resolve()
        n, p, t = self.n_total, self.num_pairs, int(self.st.n_tiles)
        dev = self.device
        valid = torch.empty(n, dtype=torch.int32, device=dev)
        m_out = torch.zeros(1, dtype=torch.int64, device=dev)
        packed = torch.empty((n, 13), dtype=torch.float32, device=dev)
        mode = torch.empty(n, dtype=torch.int8, device=dev)
        rect = torch.empty((n, 4), dtype=torch.int32, device=dev)
        pair_splat = torch.empty(max(p, 1), dtype=torch.int32, device=dev)
        tile_starts = torch.empty(t + 1, dtype=torch.int64, device=dev)
        _native.check(self.lib.hs_frame_export(
            ctypes.byref(self.st), _ptr(valid), _ptr(m_out), _ptr(packed), _ptr(mode),
            _ptr(rect), _ptr(pair_splat), _ptr(tile_starts), _stream()), "hs_frame_export")
        m = int(m_out.item())
        return {
            "valid": valid[:m].cpu().numpy().astype(np.int64),
            "packed": packed[:m].cpu().numpy(),
            "mode": mode[:m].cpu().numpy(),
            "tile_rect": rect[:m].cpu().numpy(),
            "pair_splat": pair_splat[:p].cpu().numpy(),
            "tile_starts": tile_starts.cpu().numpy(),
            "radii": self.radii.cpu().numpy(),
        }


def _validate(scene, cam, kernel):
    if len(scene) == 0:
        raise EmptyScene("cannot render an empty scene")
    if cam.width * cam.height > MAX_PIXELS:
        raise ImageTooLarge(f"{cam.width}x{cam.height} exceeds {MAX_PIXELS} pixels")
    if kernel not in ("half", "full"):
        raise ValueError("kernel must be 'half' or 'full'")


def prepare(scene, cam, kernel="half", timer=None, ws=None):
    """Project + bin one view on the GPU (rasterizer.py:159-341)."""
    timer = timer or _NO_TIMER
    scene = Scene.from_any(scene)
    cam = CameraModel.from_any(cam)
    _validate(scene, cam, kernel)
    if ws is not None and not ws.capturing:
        ws.check_previous()
    frame = DeviceFrame(scene, cam, kernel, ws)
    lib = frame.lib
    s = _stream()
    sc = scene_struct(scene)
    cs = camera_struct(cam)
    with timer.span("preprocess_fwd"):
        st = lib.hs_preprocess_fwd(ctypes.byref(frame.st), ctypes.byref(sc), ctypes.byref(cs),
                                   _ptr(frame.radii), s)
    _native.check(st, "hs_preprocess_fwd")
    return _bin(frame, ws, timer)


def prepare_views(scene, cams, kernel="half", timer=None, workspaces=None, bin=True):
    """prepare() for a batch of views of one scene with ONE K1 pass
    (hs_preprocess_fwd_views): each Gaussian is staged once and its
    camera-independent state (rotation, covariance, normal, opacities) computed once
    for all the views.  `workspaces`: one Workspace per view (distinct, since the
    frames live together).  Returns the binned frames, as prepare() does per view;
    with bin=False the frames are only preprocessed (bin each with bin_frame)."""
    timer = timer or _NO_TIMER
    scene = Scene.from_any(scene)
    cams = [CameraModel.from_any(c) for c in cams]
    if workspaces is None:
        workspaces = [None] * len(cams)
    if len(workspaces) != len(cams) or not cams:
        raise ValueError("one workspace per view is required")
    real = [ws for ws in workspaces if ws is not None]
    if len({id(ws) for ws in real}) != len(real):
        raise ValueError("the views of one batch need distinct workspaces")
    for cam in cams:
        _validate(scene, cam, kernel)
    for ws in real:
        if not ws.capturing:
            ws.check_previous()
    frames = [DeviceFrame(scene, cam, kernel, ws) for cam, ws in zip(cams, workspaces)]
    lib = frames[0].lib
    n = len(frames)
    ptrs = (ctypes.c_void_p * n)(*[ctypes.addressof(f.st) for f in frames])
    radii = (ctypes.c_void_p * n)(*[f.radii.data_ptr() for f in frames])
    cs = (_native.HsCamera * n)(*[camera_struct(c) for c in cams])
    sc = scene_struct(scene)
    with timer.span("preprocess_fwd"):
        st = lib.hs_preprocess_fwd_views(ptrs, n, ctypes.byref(sc), cs, radii, 1 if bin else 0,
                                         _stream())
    _native.check(st, "hs_preprocess_fwd_views")
    if not bin:
        return frames
    return [_bin(f, ws, timer) for f, ws in zip(frames, workspaces)]


def bin_frame(frame, ws=None, timer=None):
    """The depth ranks, pair counts and binning of a frame K1 left with
    prepare_views(bin=False), on the current stream (e.g. one stream per view, after
    an event on the K1 stream)."""
    timer = timer or _NO_TIMER
    with timer.span("preprocess_fwd"):
        st = frame.lib.hs_frame_rank(ctypes.byref(frame.st), _stream())
    _native.check(st, "hs_frame_rank")
    return _bin(frame, ws, timer)


def _bin(frame, ws, timer):
    """The binning of a preprocessed frame (prepare's second half)."""
    lib = frame.lib
    s = _stream()
    if frame.reuse_binning() > 0:
        # the workspace has a pair capacity from an earlier view: bin with P on the
        # device (no host round trip); the status is copied back behind the binning
        # and checked by the next prepare into this workspace (or frame.resolve())
        with timer.span("bin_and_sort"):
            st = lib.hs_bin_async(ctypes.byref(frame.st), s)
        if st == _native.HS_ERR_WORKSPACE:  # large-image path: P was read, too big
            frame.alloc_binning()
            st = lib.hs_bin_and_sort(ctypes.byref(frame.st), s)
        _native.check(st, "hs_bin_async")
        if frame.st.num_pairs < 0:
            frame.pending = True
            pinned = ws.status_buffer()
            _native.check(lib.hs_frame_status_async(ctypes.byref(frame.st),
                                                    ctypes.c_void_p(pinned.data_ptr()), s),
                          "hs_frame_status_async")
            if not ws.capturing:  # a graph replays the copy; CapturedStep.check reads it
                ev = torch.cuda.Event()
                ev.record()
                ws.pending = (ev, pinned, frame)
        return frame
    # first view of this workspace (or no workspace): read P (a host sync), size the
    # binning workspace with headroom, then bin
    with timer.span("bin_and_sort"):
        st = lib.hs_read_pairs_and_bin(ctypes.byref(frame.st), s)
        if st == _native.HS_ERR_WORKSPACE:
            frame.alloc_binning()
            st = lib.hs_bin_and_sort(ctypes.byref(frame.st), s)
    _native.check(st, "hs_read_pairs_and_bin")
    if ws is not None and frame.st.depth_sort_full:
        ws.depth_sort_full = 1  # the fixup overflowed: rank later views with the full sort
    return frame


@dataclass
class DeviceRenderOutput:
    """Forward result on the device (RenderOutput, rasterizer.py:59-69)."""

    color: torch.Tensor          # (H, W, 3) float32
    alpha: torch.Tensor          # (H, W)
    depth: torch.Tensor          # (H, W)
    transmittance: torch.Tensor  # (H, W)
    terminal: torch.Tensor       # (H, W) int32, per_pixel_terminal_index
    radii: torch.Tensor          # (N,) int32, ceil of the 3.5-sigma radius, 0 if culled
    frame: DeviceFrame = None
    camera: object = None

    @property
    def per_pixel_terminal_index(self):
        return self.terminal


class StageTimer:
    """CUDA-event brackets around individual library calls on the current stream.

    ``timer.span(name)`` is a context manager; durations (ms) accumulate per name
    and are read after a synchronize with ``timer.totals()``."""

    def __init__(self):
        self.events = {}

    def span(self, name):
        timer = self

        class _Span:
            def __enter__(self_):
                self_.a = torch.cuda.Event(enable_timing=True)
                self_.b = torch.cuda.Event(enable_timing=True)
                self_.a.record()

            def __exit__(self_, *exc):
                self_.b.record()
                timer.events.setdefault(name, []).append((self_.a, self_.b))

        return _Span()

    def totals(self):
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.events.items()}

    def reset(self):
        self.events = {}


class _NoTimer:
    def span(self, name):
        import contextlib
        return contextlib.nullcontext()


_NO_TIMER = _NoTimer()


def render(scene, cam, kernel="half", frame=None, out=None, timer=None, ws=None):
    """Render one view (rasterizer.py:351-383); outputs stay on the device.

    With a Workspace `ws`, every buffer (frame, binning, outputs) is reused."""
    timer = timer or _NO_TIMER
    scene = Scene.from_any(scene)
    cam = CameraModel.from_any(cam)
    if frame is None:
        frame = prepare(scene, cam, kernel, timer=timer, ws=ws)
    h, w = cam.height, cam.width
    dev = scene.device
    if out is None and ws is not None:
        out = DeviceRenderOutput(
            color=ws.tensor("color", (h, w, 3), torch.float32),
            alpha=ws.tensor("alpha", (h, w), torch.float32),
            depth=ws.tensor("depth", (h, w), torch.float32),
            transmittance=ws.tensor("transmittance", (h, w), torch.float32),
            terminal=ws.tensor("terminal", (h, w), torch.int32),
            radii=frame.radii, frame=frame, camera=cam)
    if out is None:
        out = DeviceRenderOutput(
            color=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
            alpha=torch.empty((h, w), dtype=torch.float32, device=dev),
            depth=torch.empty((h, w), dtype=torch.float32, device=dev),
            transmittance=torch.empty((h, w), dtype=torch.float32, device=dev),
            terminal=torch.empty((h, w), dtype=torch.int32, device=dev),
            radii=frame.radii, frame=frame, camera=cam)
    else:
        out.frame, out.radii, out.camera = frame, frame.radii, cam
    bg = (ctypes.c_double * 3)(*scene.background_color.tolist())
    with timer.span("blend_fwd"):
        st = frame.lib.hs_blend_fwd(
            ctypes.byref(frame.st), bg, _ptr(out.color), _ptr(out.alpha), _ptr(out.depth),
            _ptr(out.transmittance), _ptr(out.terminal), _stream())
    _native.check(st, "hs_blend_fwd")
    return out


@dataclass
class DeviceGradientSet:
    """Per-primitive gradients on the device (GradientSet, rasterizer.py:72-105)."""

    d_mu: torch.Tensor
    d_log_scale: torch.Tensor
    d_rotation: torch.Tensor
    d_sh: torch.Tensor
    d_normal: torch.Tensor
    d_raw_opacity_a: torch.Tensor
    d_raw_opacity_b: torch.Tensor
    pos_grad_norm: torch.Tensor
    touch_count: torch.Tensor

    NAMES = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
             "d_raw_opacity_b", "pos_grad_norm", "touch_count")

    @classmethod
    def empty_like_scene(cls, scene):
        n, k, dev, dt = len(scene), scene.sh_coeffs.shape[1], scene.device, scene.dtype
        return cls(
            d_mu=torch.empty((n, 3), dtype=dt, device=dev),
            d_log_scale=torch.empty((n, 3), dtype=dt, device=dev),
            d_rotation=torch.empty((n, 4), dtype=dt, device=dev),
            d_sh=torch.empty((n, k, 3), dtype=dt, device=dev),
            d_normal=torch.empty((n, 3), dtype=dt, device=dev),
            d_raw_opacity_a=torch.empty(n, dtype=dt, device=dev),
            d_raw_opacity_b=torch.empty(n, dtype=dt, device=dev),
            pos_grad_norm=torch.empty(n, dtype=dt, device=dev),
            touch_count=torch.empty(n, dtype=torch.int32, device=dev))

    @classmethod
    def empty_flat(cls, scene):
        """All float groups as views of one flat buffer (one all-reduce per step)."""
        n, k, dev, dt = len(scene), scene.sh_coeffs.shape[1], scene.device, scene.dtype
        sizes = [3 * n, 3 * n, 4 * n, 3 * k * n, 3 * n, n, n, n]
        # each group starts 16-B aligned so K7 stores it with vector accesses
        padded = [(sz + 3) // 4 * 4 for sz in sizes]
        flat = torch.empty(sum(padded), dtype=dt, device=dev)
        parts = [p[:sz] for p, sz in zip(torch.split(flat, padded), sizes)]
        g = cls(d_mu=parts[0].view(n, 3), d_log_scale=parts[1].view(n, 3),
                d_rotation=parts[2].view(n, 4), d_sh=parts[3].view(n, k, 3),
                d_normal=parts[4].view(n, 3), d_raw_opacity_a=parts[5], d_raw_opacity_b=parts[6],
                pos_grad_norm=parts[7],
                touch_count=torch.empty(n, dtype=torch.int32, device=dev))
        g.flat = flat
        return g

    def add_(self, other):
        """Accumulate another view's gradients (GradientSet.add, rasterizer.py:100-105)."""
        for name in self.NAMES:
            getattr(self, name).add_(getattr(other, name))
        return self

    def flat_views(self):
        return [getattr(self, name) for name in self.NAMES]


def grads_struct(grads, accumulate=0):
    """hs_grads over a DeviceGradientSet's buffers."""
    g = _native.HsGrads()
    for name in DeviceGradientSet.NAMES:
        setattr(g, name, getattr(grads, name).data_ptr())
    g.accumulate = accumulate
    return g


class CapturedStep:
    """A steady-state step (e.g. Rasterizer render + render_backward of fixed views)
    captured once as a CUDA graph and replayed: one launch for the whole step, no
    per-kernel host work.  Possible because binning needs no host round trip
    (hs_bin_async): `fn` runs eagerly `warmup` times first, which sizes every
    workspace (pair capacities, cached attributes), then once under capture.
    The binning status of each replay lands in the workspaces' pinned status words;
    check() (after a synchronisation) raises BinningOverflow if a replayed view ever
    outgrew its capacity.  The captured buffers must not be reallocated afterwards:
    replay only while the scene and views keep their sizes."""

    def __init__(self, fn, workspaces, warmup=2):
        self.workspaces = list(workspaces)
        for _ in range(max(1, warmup)):
            fn()
        torch.cuda.synchronize()
        for ws in self.workspaces:
            ws.check_previous()
            ws.status_buffer().zero_()
        self.graph = torch.cuda.CUDAGraph()
        for ws in self.workspaces:
            ws.capturing = True
        try:
            with torch.cuda.graph(self.graph):
                fn()
        finally:
            for ws in self.workspaces:
                ws.capturing = False

    def replay(self):
        self.graph.replay()

    def check(self):
        """Call after synchronising: the status of the last replay of every view."""
        for ws in self.workspaces:
            host = ws.status_buffer()
            flags, depth = int(host[2]) & 0xffffffff, int(host[3]) & 0xffffffff
            if flags or depth:
                raise BinningOverflow(f"a replayed view overflowed its binning workspace "
                                      f"(P={int(host[0])}, capacity {ws.pair_capacity})")


class Rasterizer:
    """Allocation-free rendering loop: `slots` persistent workspaces used round
    robin.  An output stays valid until its slot is reused `slots` renders later
    (slots=1 suits render -> render_backward -> next render)."""

    def __init__(self, device="cuda", slots=1, kernel="half"):
        self.slots = [Workspace(device) for _ in range(slots)]
        self.next = 0
        self.kernel = kernel

    def render(self, scene, cam, timer=None):
        ws = self.slots[self.next]
        self.next = (self.next + 1) % len(self.slots)
        return render(scene, cam, self.kernel, timer=timer, ws=ws)

    def render_backward(self, scene, cam, out, d_color, grads=None, timer=None, accumulate=False,
                        reduce_ptrs=None, buckets=None, on_bucket=None):
        return render_backward(scene, cam, out, d_color, grads=grads, timer=timer,
                               accumulate=accumulate, reduce_ptrs=reduce_ptrs, buckets=buckets,
                               on_bucket=on_bucket)


def render_backward(scene, cam, out, d_color, grads=None, timer=None, accumulate=False,
                    reduce_ptrs=None, buckets=None, on_bucket=None):
    """Gradients of sum(d_color * color) for every parameter (rasterizer.py:386-421).

    accumulate=True adds this view's gradients into `grads` (GradientSet.add,
    rasterizer.py:100-105) inside the K7 kernel instead of overwriting them."""
    scene = Scene.from_any(scene)
    cam = CameraModel.from_any(cam)
    timer = timer or _NO_TIMER
    frame, lib, s = _blend_backward(scene, cam, out, d_color, timer)
    if grads is None:
        grads = DeviceGradientSet.empty_like_scene(scene)
    g = grads_struct(grads, 1 if accumulate else 0)
    _reduction_targets(g, reduce_ptrs)
    sc = scene_struct(scene)
    cs = camera_struct(cam)
    with timer.span("preprocess_bwd"):
        if buckets is None:
            st = lib.hs_preprocess_bwd(ctypes.byref(frame.st), ctypes.byref(sc),
                                       ctypes.byref(cs), ctypes.byref(g), s)
            _native.check(st, "hs_preprocess_bwd")
        else:
            # K7 in primitive buckets; on_bucket(b, e) runs right after each launch (e.g.
            # an async all-reduce of that bucket, overlapping the next bucket's K7)
            for b, e in buckets:
                st = lib.hs_preprocess_bwd_range(ctypes.byref(frame.st), ctypes.byref(sc),
                                                 ctypes.byref(cs), ctypes.byref(g), b, e, s)
                _native.check(st, "hs_preprocess_bwd_range")
                if on_bucket is not None:
                    on_bucket(b, e)
    return grads


def _reduction_targets(g, reduce_ptrs):
    if reduce_ptrs is not None:
        # reduction stores: {name: address} (NVLS multicast addresses -> mode 3, or the
        # buffers' own addresses with reduce_ptrs["mode"] == 2 for device atomics)
        for name in DeviceGradientSet.NAMES:
            setattr(g, name, reduce_ptrs[name])
        g.accumulate = reduce_ptrs.get("mode", 3)


def _blend_backward(scene, cam, out, d_color, timer):
    """K6 of one rendered view (hs_blend_bwd); returns (frame, lib, stream)."""
    frame = out.frame
    if frame is None or frame.n_total != len(scene):
        raise MismatchedForward("forward bookkeeping does not match the scene")
    if tuple(d_color.shape) != (cam.height, cam.width, 3):
        raise MismatchedForward(
            f"cotangent shape {tuple(d_color.shape)} != {(cam.height, cam.width, 3)}")
    if tuple(out.terminal.shape) != (cam.height, cam.width):
        raise MismatchedForward("terminal-index shape mismatch")
    if not isinstance(d_color, torch.Tensor):
        d_color = torch.as_tensor(np.asarray(d_color))
    d_color = d_color.to(device=scene.device, dtype=torch.float32).contiguous()
    lib = frame.lib
    s = _stream()
    bg = (ctypes.c_double * 3)(*scene.background_color.tolist())
    with timer.span("blend_bwd"):
        st = lib.hs_blend_bwd(ctypes.byref(frame.st), bg, _ptr(d_color),
                              _ptr(out.transmittance), _ptr(out.terminal), s)
    _native.check(st, "hs_blend_bwd")
    return frame, lib, s


MERGED_ROW_FLOATS = 16  # one 64-B merged blend-gradient row per primitive (hs_merge_rows)


def blend_backward_rows(scene, cam, out, d_color, merged=None, timer=None):
    """The first half of render_backward for the multi-view geometry backward: K6 of
    one view, then that view's per-primitive merged blend gradients (K7a) copied
    into `merged` ((n, 16) float32, allocated if None), so the view's workspace can
    be reused by the next view.  Pass the rows of a batch of views to
    geometry_backward_views."""
    scene = Scene.from_any(scene)
    cam = CameraModel.from_any(cam)
    timer = timer or _NO_TIMER
    frame, lib, s = _blend_backward(scene, cam, out, d_color, timer)
    if merged is None:
        merged = torch.empty((len(scene), MERGED_ROW_FLOATS), dtype=torch.float32,
                             device=scene.device)
    if (tuple(merged.shape) != (len(scene), MERGED_ROW_FLOATS) or
            merged.dtype != torch.float32 or not merged.is_contiguous()):
        raise ValueError(f"merged rows must be a contiguous float32 ({len(scene)}, 16) tensor")
    with timer.span("merge_rows"):
        _native.check(lib.hs_merge_rows(ctypes.byref(frame.st), _ptr(merged), s),
                      "hs_merge_rows")
    return merged


def geometry_backward_views(scene, cams, merged, grads=None, kernel="half", timer=None,
                            accumulate=False, reduce_ptrs=None, buckets=None, on_bucket=None):
    """Sum over views of the geometry backward (K7) in ONE pass over the scene
    (hs_preprocess_bwd_views): merged[v] is view v's blend_backward_rows output.
    Equal to render_backward over the views with accumulate=True after the first
    (GradientSet.add, rasterizer.py:100-105), the sum taken in view order."""
    scene = Scene.from_any(scene)
    cams = [CameraModel.from_any(c) for c in cams]
    if len(cams) != len(merged) or not cams:
        raise ValueError("one merged-row buffer per camera is required")
    if kernel not in ("half", "full"):
        raise ValueError("kernel must be 'half' or 'full'")
    for m in merged:
        if (tuple(m.shape) != (len(scene), MERGED_ROW_FLOATS) or m.dtype != torch.float32
                or m.device != scene.mu.device):
            raise MismatchedForward("merged rows do not match the scene")
    timer = timer or _NO_TIMER
    lib = _native.load()
    s = _stream()
    if grads is None:
        grads = DeviceGradientSet.empty_like_scene(scene)
    g = grads_struct(grads, 1 if accumulate else 0)
    _reduction_targets(g, reduce_ptrs)
    sc = scene_struct(scene)
    cs = (_native.HsCamera * len(cams))(*[camera_struct(c) for c in cams])
    rows = (ctypes.c_void_p * len(cams))(*[m.data_ptr() for m in merged])
    kcode = {"half": _native.HS_KERNEL_HALF, "full": _native.HS_KERNEL_FULL}[kernel]
    ranges = buckets if buckets is not None else [(0, len(scene))]
    with timer.span("preprocess_bwd"):
        for b, e in ranges:
            st = lib.hs_preprocess_bwd_views(ctypes.byref(sc), len(cams), cs, rows, kcode,
                                             ctypes.byref(g), b, e, s)
            _native.check(st, "hs_preprocess_bwd_views")
            if on_bucket is not None:
                on_bucket(b, e)
    return grads
