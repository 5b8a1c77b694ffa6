"""Host-side logic that needs no GPU: cameras, scene validation, the backend
seam, the canonical generator, view sharding and the gloo all-reduce path."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_02720_b200 import backend, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene
from paper_2406_02720_b200.multiview import GradientAllReduce, shard_views


def test_camera_validation_mirrors_reference():
    with pytest.raises(ValueError):
        CameraModel(np.eye(3), 10, 10, 5, 5, 10, 10)
    bad = np.eye(4)
    bad[0, 0] = 2.0
    with pytest.raises(ValueError):
        CameraModel(bad, 10, 10, 5, 5, 10, 10)
    with pytest.raises(ValueError):
        CameraModel(np.eye(4), -1, 10, 5, 5, 10, 10)
    with pytest.raises(ValueError):
        CameraModel(np.eye(4), 10, 10, 50, 5, 10, 10)
    cam = CameraModel.look_at((3.0, -0.5, 0.0), (0, 0, 0), 64, 48, 50.0)
    np.testing.assert_allclose(cam.center, [3.0, -0.5, 0.0], atol=1e-12)
    r = cam.rotation
    np.testing.assert_allclose(r @ r.T, np.eye(3), atol=1e-12)


def test_look_at_matches_generator():
    w2c = scenes.look_at_matrix((1.0, 2.0, 3.0), (0.0, 0.0, 0.0))
    cam = CameraModel.look_at((1.0, 2.0, 3.0), (0.0, 0.0, 0.0), 32, 32, 30.0)
    assert np.array_equal(w2c, cam.world_to_cam)


def test_scene_validation_on_cpu():
    sa = scenes.frustum(50, 1, 32, 32, seed=1)
    fields = [getattr(sa, f) for f in sa.FIELDS]
    s = Scene(*fields, sh_degree=1, device="cpu")
    assert len(s) == 50 and s.dtype == torch.float32
    s64 = Scene(*[f.astype(np.float64) for f in fields], sh_degree=1, device="cpu")
    assert s64.dtype == torch.float64
    with pytest.raises(ValueError):
        Scene(*fields, sh_degree=2, device="cpu")
    bad = [f.copy() for f in fields]
    bad[4][3] = 0.0
    with pytest.raises(ValueError):
        Scene(*bad, sh_degree=1, device="cpu")
    with pytest.raises(ValueError):
        Scene(*fields, sh_degree=1, background_color=(2, 0, 0), device="cpu")


def test_autograd_front_end_checks_shapes_on_cpu():
    """torch_api builds its Scene unvalidated (no device sync), but the shape checks
    still run before anything reaches K1/K7: a shs tensor of the wrong degree or a
    field of the wrong length raises instead of reading out of bounds."""
    from paper_2406_02720_b200 import torch_api
    sa = scenes.frustum(20, 1, 32, 32, seed=1)
    t = {f: torch.from_numpy(getattr(sa, f)) for f in sa.FIELDS}
    settings = torch_api.HalfGaussianRasterizationSettings(
        image_height=32, image_width=32, world_to_cam=np.eye(4), fx=30.0, fy=30.0, cx=16.0,
        cy=16.0, sh_degree=2)
    with pytest.raises(ValueError, match="sh_coeffs"):
        torch_api.rasterize_half_gaussians(t["mu"], t["normal"], t["raw_opacity_a"],
                                           t["raw_opacity_b"], t["log_scale"], t["rotation"],
                                           t["sh_coeffs"], settings)
    settings.sh_degree = 1
    with pytest.raises(ValueError, match="opacity"):
        torch_api.rasterize_half_gaussians(t["mu"], t["normal"], t["raw_opacity_a"][:-1],
                                           t["raw_opacity_b"], t["log_scale"], t["rotation"],
                                           t["sh_coeffs"], settings)


def test_backend_seam():
    assert backend.available_backends() == ["cuda"]
    backend.set_backend("cuda")
    assert backend.backend_name() == "cuda"
    backend.set_backend(None)
    with pytest.raises(ValueError):
        backend.set_backend("cython")
    mod = backend.get_backend()
    assert hasattr(mod, "forward_tiles") and hasattr(mod, "backward_tiles")


def test_generator_reproduces_survey_counts():
    """c1 M=9,865, P=32,950 and c2 M=100,000, P=406,380."""
    from oracle import oracle as O

    class Cam:
        pass

    for name, m, p in (("c1", 9865, 32950), ("c2", 100_000, 406_380)):
        sa = scenes.make_config(name).as_float64()
        cam = Cam()
        for k, v in sa.cameras[0].items():
            setattr(cam, k, v)
        cam.near_clip = 0.01
        f = O.prepare(sa, cam)
        assert (f.valid.shape[0], f.pair_splat.shape[0]) == (m, p)


def test_generator_is_float32_exact():
    sa = scenes.frustum(100, 3, 64, 64, seed=2)
    for f in sa.FIELDS:
        a = getattr(sa, f)
        assert a.dtype == np.float32
        assert np.array_equal(a.astype(np.float64).astype(np.float32), a)


@pytest.mark.parametrize("n,world", [(8, 1), (8, 2), (8, 3), (8, 8), (3, 4)])
def test_shard_views_partition(n, world):
    got = [v for r in range(world) for v in shard_views(n, world, r)]
    assert got == list(range(n))


def _allreduce_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class G:
        pass

    g = G()
    n, k = 5, 4
    g.flat = torch.arange(n * (3 + 3 + 4 + 3 * k + 3 + 3), dtype=torch.float32) * (rank + 1)
    g.touch_count = torch.ones(n, dtype=torch.int32) * (rank + 1)
    GradientAllReduce(g).allreduce()
    q.put((rank, g.flat.numpy().copy(), g.touch_count.numpy().copy()))
    dist.destroy_process_group()


def test_gradient_allreduce_gloo_world2():
    """The multi-view exchange step on 2 CPU ranks: the batch gradient is the sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_allreduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    n, k = 5, 4
    base = np.arange(n * (3 + 3 + 4 + 3 * k + 3 + 3), dtype=np.float32)
    for _, flat, touch in res:
        np.testing.assert_array_equal(flat, base * 3)
        np.testing.assert_array_equal(touch, np.full(n, 3, np.int32))


def test_scene_io_header_errors(tmp_path):
    """scene_io header validation mirrors the reference's errors (scene_io.py:49-111);
    all raised on the host before any device work."""
    import pytest
    from paper_2406_02720_b200 import errors, scene_io

    def write(name, text, payload=b""):
        p = tmp_path / name
        p.write_bytes(text.encode("ascii") + payload)
        return str(p)

    with pytest.raises(errors.MalformedHeader):
        scene_io.load_scene(write("a.ply", "plx\n"))
    with pytest.raises(errors.MalformedHeader):
        scene_io.load_scene(write("b.ply", "ply\nformat ascii 1.0\nend_header\n"))
    with pytest.raises(errors.MalformedHeader):
        scene_io.load_scene(write("c.ply", "ply\nformat binary_little_endian 1.0\n"
                                           "element vertex 1\nproperty list uchar int f\n"
                                           "end_header\n"))
    with pytest.raises(errors.MissingProperty):
        scene_io.load_scene(write("d.ply", "ply\nformat binary_little_endian 1.0\n"
                                           "element vertex 1\nproperty double x\nend_header\n",
                                  b"\0" * 8))
    with pytest.raises(errors.TruncatedPayload):
        scene_io.load_scene(write("e.ply", "ply\nformat binary_little_endian 1.0\n"
                                           "element vertex 2\nproperty double x\nend_header\n",
                                  b"\0" * 8))
    with pytest.raises(ValueError):
        scene_io.import_3dgs(write("f.ply", "ply\n"), normal_init="bogus")
    # the reference's messages (scene_io.py:49-88), parsed before any device work
    for text, msg in [
            ("", "not a PLY file"),
            ("ply\n", "expected format binary_little_endian"),
            ("ply\nformat binary_little_endian 1.0\nelement face 2\nend_header\n",
             "unsupported element face"),
            ("ply\nformat binary_little_endian 1.0\nproperty half x\nend_header\n",
             "unsupported property type half"),
            ("ply\nformat binary_little_endian 1.0\nbogus line\nend_header\n",
             "unexpected header line 'bogus line'"),
            ("ply\nformat binary_little_endian 1.0\nproperty float x\nend_header\n",
             "missing vertex element"),
            ("ply\nformat binary_little_endian 1.0\nelement vertex 3\n", "unterminated header")]:
        with pytest.raises(errors.MalformedHeader, match=msg):
            scene_io.load_scene(write("g.ply", text))
    h = scene_io._parse_header(b"ply\nformat binary_little_endian 1.0\ncomment sh_degree 3\n"
                               b"comment background 0.1 0.2 0.3\n\nelement vertex 2\n"
                               b"property double x\nproperty float y\nend_header\nPAYLOAD")
    assert (h.count, h.props, h.stride) == (2, [("x", "double"), ("y", "float")], 12)
    assert h.comments == {"sh_degree": "3", "background": "0.1 0.2 0.3"}
    assert h.payload_offset == len(b"ply\nformat binary_little_endian 1.0\ncomment sh_degree 3\n"
                                   b"comment background 0.1 0.2 0.3\n\nelement vertex 2\n"
                                   b"property double x\nproperty float y\nend_header\n")
    assert scene_io._rest_names({"f_rest_1": 0, "f_rest_0": 0, "x": 0}) == ["f_rest_0",
                                                                            "f_rest_1"]
    with pytest.raises(errors.MissingProperty, match="not contiguous"):
        scene_io._rest_names({"f_rest_1": 0, "f_rest_2": 0})


def _bucketed_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_02720_b200.device import DeviceGradientSet

    class S:  # the attributes DeviceGradientSet.empty_flat reads
        pass

    n, k = 700, 9

    class Sc(S):
        sh_coeffs = torch.zeros((n, k, 3))
        device, dtype = torch.device("cpu"), torch.float32

        def __len__(self):
            return n

    g = DeviceGradientSet.empty_flat(Sc())
    torch.manual_seed(rank)
    for name in DeviceGradientSet.NAMES[:-1]:
        getattr(g, name).copy_(torch.randn(getattr(g, name).shape))
    g.touch_count.copy_(torch.randint(0, 3, (n,), dtype=torch.int32))
    want = [getattr(g, name).clone() for name in DeviceGradientSet.NAMES]
    for t in want:
        dist.all_reduce(t)
    red = GradientAllReduce(g)
    for b, e in GradientAllReduce.bucket_ranges(n, buckets=3):
        red.start_range(b, e)
    red.finish()
    ok = all(torch.equal(getattr(g, name), w) for name, w in zip(DeviceGradientSet.NAMES, want))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_bucketed_allreduce_gloo_world2():
    """The K7-bucketed exchange (start_range per primitive bucket, then finish) sums
    exactly what one all-reduce of every group sums, on 2 CPU ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_bucketed_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
