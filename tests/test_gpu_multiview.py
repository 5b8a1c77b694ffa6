"""The view-sharded training step across processes, on the one GPU
a gpurun box has: 2 ranks, each its own process driving cuda:0 through the
library, exchanging gradients over gloo on CUDA tensors (no kernel ever waits on
another rank, so sharing the GPU is safe).  The batch gradient every rank ends
with must equal the oracle's Sum_v render_backward(view v) over the whole batch,
summed in view order as GradientSet.add does (rasterizer.py:100-105)."""

import os

import numpy as np
import pytest

from parity import assert_grads

pytestmark = pytest.mark.gpu

N_VIEWS = 4
SCENE = dict(n=3000, sh=2, w=96, h=72, seed=31)
NAMES = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
         "d_raw_opacity_b", "pos_grad_norm", "touch_count")


def _scene_arrays():
    from paper_2406_02720_b200 import scenes
    return scenes.ball(SCENE["n"], SCENE["sh"], SCENE["w"], SCENE["h"], views=N_VIEWS,
                       seed=SCENE["seed"])


def _worker(rank, world, port, dtype_name, bucketed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_02720_b200 import device, multiview, scenes
        from paper_2406_02720_b200.geometry import CameraModel, Scene
        dtype = getattr(torch, dtype_name)
        sa = _scene_arrays()
        scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                      background_color=sa.background_color, device="cuda", dtype=dtype)
        cams = [CameraModel(**c) for c in sa.cameras]
        dcs = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=10 + i),
                               dtype=torch.float32, device="cuda") for i, c in enumerate(cams)]
        if bucketed == "views":
            # the multi-view backward (one K7 pass for the rank's views) in buckets,
            # each bucket's exchange issued right after its launch
            views = multiview.shard_views(len(cams), world, rank)
            grads = device.DeviceGradientSet.empty_flat(scene)
            red = multiview.GradientAllReduce(grads)
            batch = multiview.ViewBatch(scene, len(views))
            batch.run(scene, cams, dcs, views, grads,
                      buckets=multiview.GradientAllReduce.bucket_ranges(len(scene), buckets=3),
                      on_bucket=red.start_range)
            red.finish()
        elif bucketed:
            views = multiview.shard_views(len(cams), world, rank)
            grads = device.DeviceGradientSet.empty_flat(scene)
            red = multiview.GradientAllReduce(grads)
            rast = device.Rasterizer("cuda")
            buckets = multiview.GradientAllReduce.bucket_ranges(len(scene), buckets=3)
            for j, v in enumerate(views):
                out = rast.render(scene, cams[v])
                last = j == len(views) - 1
                rast.render_backward(scene, cams[v], out, dcs[v], grads=grads, accumulate=j > 0,
                                     buckets=buckets if last else None,
                                     on_bucket=red.start_range if last else None)
            red.finish()
        else:
            grads = multiview.multiview_step(scene, cams, dcs)
        torch.cuda.synchronize()
        q.put((rank, {name: getattr(grads, name).double().cpu().numpy() if name != "touch_count"
                      else getattr(grads, name).cpu().numpy() for name in NAMES}))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent instead of a queue timeout
        q.put((rank, repr(e)))


def _run(dtype_name, bucketed, port):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dtype_name, bucketed, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
    return res


def _oracle_batch():
    """Sum_v of the oracle's render_backward over the batch, in view order."""
    from oracle import oracle as O
    from paper_2406_02720_b200 import scenes
    from paper_2406_02720_b200.geometry import CameraModel
    s64 = _scene_arrays().as_float64()
    total = None
    for i, c in enumerate(s64.cameras):
        cam = CameraModel(**c)
        d_color = scenes.cotangent(cam.height, cam.width, seed=10 + i)
        d_color = d_color.astype(np.float32).astype(np.float64)  # what the GPU ranks consume
        out = O.render(s64, cam)
        g = O.render_backward(s64, cam, out, d_color)
        if total is None:
            total = {k: np.array(g[k], copy=True) for k in NAMES}
        else:
            for k in NAMES:
                total[k] += g[k]
    return total


@pytest.mark.parametrize("dtype_name,bucketed,port", [("float32", False, 29611),
                                                      ("float64", True, 29613),
                                                      ("float32", "views", 29615)])
def test_two_rank_batch_gradient_equals_oracle_sum(cuda, dtype_name, bucketed, port):
    res = _run(dtype_name, bucketed, port)
    ref = _oracle_batch()
    # both ranks hold the same sum, bit for bit
    for k in NAMES:
        assert np.array_equal(res[0][k], res[1][k]), k
    assert np.array_equal(res[0]["touch_count"], ref["touch_count"])
    assert_grads({k: res[0][k] for k in NAMES[:-1]}, {k: ref[k] for k in NAMES[:-1]},
                 groups=NAMES[:-1])
