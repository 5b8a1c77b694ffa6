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

import torch
import torch.distributed as dist


def shard_views(n_views, world, rank):
    """Contiguous block of view indices owned by `rank` (ceil(n/world) per rank)."""
    per = (n_views + world - 1) // world
    lo = min(rank * per, n_views)
    return list(range(lo, min(lo + per, n_views)))


class GradientAllReduce:
    """Sums a flat gradient buffer (+ int touch counts) over the default group."""

    def __init__(self, grads, group=None):
        if not hasattr(grads, "flat"):
            raise ValueError("gradients must be allocated with DeviceGradientSet.empty_flat")
        self.grads = grads
        self.group = group

    def allreduce(self):
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return self.grads
        dist.all_reduce(self.grads.flat, op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(self.grads.touch_count, op=dist.ReduceOp.SUM, group=self.group)
        return self.grads


def batch_gradients(scene, cams, d_colors, view_ids, out=None, rast=None, timer=None):
    """Sum render_backward over this rank's views into `out` (flat buffer).

    The first view overwrites, later ones accumulate inside the K7 kernel, so a
    batch costs no extra gradient-sized passes."""
    from . import device
    if out is None:
        out = device.DeviceGradientSet.empty_flat(scene)
    if rast is None:
        rast = device.Rasterizer(scene.device)
    if not view_ids:
        out.flat.zero_()
        out.touch_count.zero_()
    for j, v in enumerate(view_ids):
        r = rast.render(scene, cams[v], timer=timer)
        rast.render_backward(scene, cams[v], r, d_colors[v], grads=out, timer=timer,
                             accumulate=j > 0)
    return out


def multiview_step(scene, cams, d_colors, grads=None, rast=None):
    """One data-parallel step: local views, then the all-reduce. Returns the batch gradient."""
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    views = shard_views(len(cams), world, rank)
    grads = batch_gradients(scene, cams, d_colors, views, grads, rast)
    GradientAllReduce(grads).allreduce()
    return grads
