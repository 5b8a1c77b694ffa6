"""Multi-view data-parallel training step: views sharded over ranks, one
gradient all-reduce per step.

The reference renders one view per training iteration (trainer.py:396-401) and
has no distributed path; GradientSet.add (rasterizer.py:100-105) is the
accumulation rule.  Here each rank (one GPU, one process) holds a replica of
the Gaussians, renders its share of a batch of views, accumulates its
per-Gaussian gradients in one flat buffer, and the buffer is summed over ranks
with a single NCCL all-reduce over NVLink (gloo on CPU for tests).  The sum is
the batch gradient, Sum_v render_backward(view v).
"""

import contextlib
import os

import torch
import torch.distributed as dist


def shard_views(n_views, world, rank):
    """Contiguous block of view indices owned by `rank` (ceil(n/world) per rank)."""
    per = (n_views + world - 1) // world
    lo = min(rank * per, n_views)
    return list(range(lo, min(lo + per, n_views)))


class NcclComm:
    """An NCCL communicator of the library (hs_comm_*), one per process group: rank 0
    creates the unique id, the group broadcasts it, every rank joins on its current
    device.  hs_grad_allreduce then sums gradient ranges as single NCCL groups."""

    _cache = {}

    def __init__(self, group=None):
        import ctypes
        from . import _native
        lib = _native.load()
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        uid = torch.zeros(_native.HS_COMM_ID_BYTES, dtype=torch.uint8)
        if rank == 0:
            _native.check(lib.hs_comm_unique_id(ctypes.c_void_p(uid.data_ptr())),
                          "hs_comm_unique_id")
        on_gpu = dist.get_backend(group) == "nccl"
        buf = uid.cuda() if on_gpu else uid
        dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)
        uid = buf.cpu()
        self.handle = ctypes.c_void_p()
        _native.check(lib.hs_comm_init(ctypes.byref(self.handle), world, rank,
                                       ctypes.c_void_p(uid.data_ptr())), "hs_comm_init")
        self.world, self.rank = world, rank

    @classmethod
    def for_group(cls, group=None):
        key = id(group) if group is not None else None
        if key not in cls._cache:
            cls._cache[key] = cls(group)
        return cls._cache[key]

    def info(self):
        """(ranks, rank, NCCL version) as the communicator reports them."""
        import ctypes
        from . import _native
        w, r, v = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _native.check(_native.load().hs_comm_info(self.handle, ctypes.byref(w), ctypes.byref(r),
                                                  ctypes.byref(v)), "hs_comm_info")
        return w.value, r.value, v.value


class GradientAllReduce:
    """Sums a flat gradient buffer (+ int touch counts) over the default group.

    allreduce() sums everything after the last K7.  The bucketed form overlaps the
    exchange with K7: K7 runs over primitive buckets
    (`bucket_ranges`), start_range(b, e) issues the bucket's exchange right after
    its K7 launch on a side stream that waits for that launch, so it runs under the
    next bucket's K7, and finish() makes the compute stream wait for all of them.
    On CUDA tensors over NCCL each exchange is one grouped hs_grad_allreduce (every
    field slice and the touch counts of the range); with gloo (CPU tests) it is a
    public dist.all_reduce per slice."""

    def __init__(self, grads, group=None):
        if not hasattr(grads, "flat"):
            raise ValueError("gradients must be allocated with DeviceGradientSet.empty_flat")
        self.grads = grads
        self.group = group
        self._pending = []
        self._comm = None
        self._stream = None
        self._touch_done = False
        if self._active() and grads.flat.is_cuda and dist.get_backend(group) == "nccl":
            self._comm = NcclComm.for_group(group)
            self._stream = torch.cuda.Stream(device=grads.flat.device)

    @staticmethod
    def _active():
        return dist.is_available() and dist.is_initialized()

    def _native_range(self, b, e, stream):
        import ctypes
        from . import _native, device
        g = self.grads
        dtype = _native.HS_DTYPE_F64 if g.d_mu.dtype == torch.float64 else _native.HS_DTYPE_F32
        k = g.d_sh.shape[1]
        deg = {1: 0, 4: 1, 9: 2, 16: 3}[k]
        st = device.grads_struct(g, 0)
        _native.check(_native.load().hs_grad_allreduce(
            self._comm.handle, ctypes.byref(st), g.d_mu.shape[0], deg, dtype, b, e, 1,
            ctypes.c_void_p(stream.cuda_stream)), "hs_grad_allreduce")

    def allreduce(self):
        if not self._active():
            return self.grads
        if self._comm is not None:
            self._native_range(0, self.grads.d_mu.shape[0], torch.cuda.current_stream())
            return self.grads
        dist.all_reduce(self.grads.flat, op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(self.grads.touch_count, op=dist.ReduceOp.SUM, group=self.group)
        return self.grads

    @staticmethod
    def bucket_ranges(n, buckets=4, align=128):
        """[(begin, end)] covering n primitives; begins are multiples of `align`
        (K7's CTA size, hs_preprocess_bwd_range)."""
        per = -(-n // (buckets * align)) * align
        return [(b, min(b + per, n)) for b in range(0, n, per)] if n > 0 else []

    def slices(self, b, e):
        g = self.grads
        return [g.d_mu[b:e], g.d_log_scale[b:e], g.d_rotation[b:e], g.d_sh[b:e],
                g.d_normal[b:e], g.d_raw_opacity_a[b:e], g.d_raw_opacity_b[b:e],
                g.pos_grad_norm[b:e]]

    def start_range(self, b, e):
        if not self._active():
            return
        if self._comm is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._stream.wait_event(ev)
            self._native_range(b, e, self._stream)
            self._pending.append(True)
            return
        tensors = self.slices(b, e) + [self.grads.touch_count[b:e]]
        self._pending.extend(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group,
                                             async_op=True) for t in tensors)

    def finish(self):
        if not self._active():
            return self.grads
        if self._comm is not None:
            if self._pending:
                torch.cuda.current_stream().wait_stream(self._stream)
        else:
            for w in self._pending:
                w.wait()
        self._pending = []
        return self.grads


class FusedGradientReduce:
    """The gradient all-reduce fused into K7 (the multimem stretch).

    The flat gradient buffer (and the touch counts) live in torch symmetric memory,
    mapped by every rank of the node.  K7 adds its per-primitive results straight
    into the buffer's NVLS multicast address with `multimem.red.add`
    (hs_grads.accumulate = 3): the NVSwitch reduces every rank's contribution into
    every rank's copy as K7 produces it, so there is no separate collective and the
    reduction traffic overlaps the FP64 geometry backward tile by tile.

    Protocol per batch: begin() zeroes the local copy and barriers (nobody may add
    into a copy that is not zeroed yet), every view's K7 adds, end() barriers
    (after it every copy holds the global sum).  Without multicast support (a
    single GPU, no NVSwitch) the same protocol runs with device atomics into the
    local copy (accumulate = 2), which is exact for one rank; multi-rank callers
    should then use GradientAllReduce instead (`multicast` tells which).  Sums of
    more than two ranks' contributions are reduced in switch order, so the result
    is not bitwise reproducible run to run."""

    def __init__(self, scene, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        from . import device
        n, k, dev, dt = len(scene), scene.sh_coeffs.shape[1], scene.device, scene.dtype
        sizes = [3 * n, 3 * n, 4 * n, 3 * k * n, 3 * n, n, n, n]
        padded = [(sz + 3) // 4 * 4 for sz in sizes]
        self.flat = symm_mem.empty(sum(padded), dtype=dt, device=dev)
        self.touch = symm_mem.empty(n, dtype=torch.int32, device=dev)
        grp = group if group is not None else dist.group.WORLD
        self.h_flat = symm_mem.rendezvous(self.flat, grp)
        self.h_touch = symm_mem.rendezvous(self.touch, grp)
        parts = [p[:sz] for p, sz in zip(torch.split(self.flat, padded), sizes)]
        self.grads = device.DeviceGradientSet(
            d_mu=parts[0].view(n, 3), d_log_scale=parts[1].view(n, 3),
            d_rotation=parts[2].view(n, 4), d_sh=parts[3].view(n, k, 3),
            d_normal=parts[4].view(n, 3), d_raw_opacity_a=parts[5], d_raw_opacity_b=parts[6],
            pos_grad_norm=parts[7], touch_count=self.touch)
        self.grads.flat = self.flat
        mc_flat, mc_touch = self.h_flat.multicast_ptr, self.h_touch.multicast_ptr
        self.multicast = bool(mc_flat) and bool(mc_touch)

        def base(h, t, mc):
            # the multicast address of t: the buffer's multicast base + t's offset in it
            return mc + (t.data_ptr() - h.buffer_ptrs[h.rank]) if mc else t.data_ptr()

        fb = base(self.h_flat, self.flat, mc_flat if self.multicast else 0)
        self.ptrs = {name: fb + (getattr(self.grads, name).data_ptr() - self.flat.data_ptr())
                     for name in device.DeviceGradientSet.NAMES if name != "touch_count"}
        self.ptrs["touch_count"] = base(self.h_touch, self.touch,
                                        mc_touch if self.multicast else 0)
        self.ptrs["mode"] = 3 if self.multicast else 2

    def begin(self):
        self.flat.zero_()
        self.touch.zero_()
        self.h_flat.barrier(channel=0)

    def end(self):
        self.h_flat.barrier(channel=0)
        return self.grads


class ViewBatch:
    """The multi-view backward of a batch of views: per view K5, K6
    and the merged blend-gradient rows (device.blend_backward_rows) into a persistent
    per-view buffer, then ONE geometry backward over the scene for all of them
    (device.geometry_backward_views, hs_preprocess_bwd_views).  Against render_backward
    per view (K7 per view, accumulating) the scene is read once and the gradient
    buffer written once per batch instead of read-modify-written per view; the sum
    is the same, in the same order."""

    def __init__(self, scene, n_views, rast=None, shared_k1=True, streams=None):
        from . import device
        self.rast = rast if rast is not None else device.Rasterizer(scene.device)
        self.merged = [torch.empty((len(scene), device.MERGED_ROW_FLOATS),
                                   dtype=torch.float32, device=scene.device)
                       for _ in range(n_views)]
        # shared_k1: the views' K1 as one pass (device.prepare_views), each view in
        # its own workspace; else view by view through `rast`
        self.workspaces = ([device.Workspace(scene.device) for _ in range(n_views)]
                           if shared_k1 else [])
        # with own workspaces the views are independent after K1: each view's binning,
        # K5, K6 and K7a run on its own stream, so one view's kernels fill the tails
        # of the others' persistent blends (c4 331 -> 372, c2 1509 -> 1953 views/s
        # with a stream per view; 2 streams: 364 / 1808)
        if streams is None:  # HS_VIEW_STREAMS overrides one stream per view (<= 8)
            streams = int(os.environ.get("HS_VIEW_STREAMS", str(min(n_views, 8))))
        self.streams = ([torch.cuda.Stream(device=scene.device) for _ in range(streams)]
                        if shared_k1 and streams > 1 and torch.device(scene.device).type == "cuda"
                        else [])

    def run(self, scene, cams, d_colors, view_ids, grads, timer=None, reduce_ptrs=None,
            buckets=None, on_bucket=None):
        from . import device
        if len(view_ids) > len(self.merged):
            raise ValueError(f"{len(view_ids)} views for a batch of {len(self.merged)}")
        if self.workspaces:
            wss = self.workspaces[:len(view_ids)]
            frames = device.prepare_views(scene, [cams[v] for v in view_ids], self.rast.kernel,
                                          timer=timer, workspaces=wss,
                                          bin=not self.streams)
            main = torch.cuda.current_stream() if self.streams else None
            if main is not None:
                ready = torch.cuda.Event()
                ready.record(main)
                for st in self.streams:
                    st.wait_event(ready)
            for j, v in enumerate(view_ids):
                ctx = (torch.cuda.stream(self.streams[j % len(self.streams)]) if self.streams
                       else contextlib.nullcontext())
                with ctx:
                    frame = (device.bin_frame(frames[j], wss[j], timer) if self.streams
                             else frames[j])
                    r = device.render(scene, cams[v], self.rast.kernel, frame=frame,
                                      timer=timer, ws=wss[j])
                    device.blend_backward_rows(scene, cams[v], r, d_colors[v], self.merged[j],
                                               timer=timer)
            if main is not None:
                for st in self.streams:
                    main.wait_stream(st)
        else:
            for j, v in enumerate(view_ids):
                r = self.rast.render(scene, cams[v], timer=timer)
                device.blend_backward_rows(scene, cams[v], r, d_colors[v], self.merged[j],
                                           timer=timer)
        return device.geometry_backward_views(
            scene, [cams[v] for v in view_ids], self.merged[:len(view_ids)], grads=grads,
            kernel=self.rast.kernel, timer=timer, reduce_ptrs=reduce_ptrs, buckets=buckets,
            on_bucket=on_bucket)


def batch_gradients(scene, cams, d_colors, view_ids, out=None, rast=None, timer=None,
                    fused=None, batch=None):
    """Sum render_backward over this rank's views into `out` (flat buffer).

    With `batch` (a ViewBatch) the geometry backward of all the views runs as one
    pass over the scene.  Otherwise the first view overwrites and later ones
    accumulate inside the K7 kernel, so a batch costs no extra gradient-sized
    passes.  With `fused` (a FusedGradientReduce) every view's K7 adds into the
    shared buffer instead and the result is already summed over all ranks."""
    if fused is not None and batch is not None and view_ids:
        fused.begin()
        batch.run(scene, cams, d_colors, view_ids, fused.grads, timer=timer,
                  reduce_ptrs=fused.ptrs)
        return fused.end()
    if fused is not None:
        from . import device
        if rast is None:
            rast = device.Rasterizer(scene.device)
        fused.begin()
        for v in view_ids:
            r = rast.render(scene, cams[v], timer=timer)
            rast.render_backward(scene, cams[v], r, d_colors[v], grads=fused.grads, timer=timer,
                                 reduce_ptrs=fused.ptrs)
        return fused.end()
    from . import device
    if out is None:
        out = device.DeviceGradientSet.empty_flat(scene)
    if rast is None:
        rast = device.Rasterizer(scene.device)
    if not view_ids:
        out.flat.zero_()
        out.touch_count.zero_()
        return out
    if batch is not None:
        return batch.run(scene, cams, d_colors, view_ids, out, timer=timer)
    for j, v in enumerate(view_ids):
        r = rast.render(scene, cams[v], timer=timer)
        rast.render_backward(scene, cams[v], r, d_colors[v], grads=out, timer=timer,
                             accumulate=j > 0)
    return out


def multiview_step(scene, cams, d_colors, grads=None, rast=None, batch=None):
    """One data-parallel step: local views, then the all-reduce. Returns the batch gradient."""
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    views = shard_views(len(cams), world, rank)
    grads = batch_gradients(scene, cams, d_colors, views, grads, rast, batch=batch)
    GradientAllReduce(grads).allreduce()
    return grads
