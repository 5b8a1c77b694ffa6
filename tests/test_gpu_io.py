"""Scene I/O (csrc/hs_io.cu + scene_io.py mirror) against the reference's
scene_io (tests/golden/io.npz, scene_io.py:136-269).

Contract: load_scene / import_3dgs give bit-identical parameter arrays;
save_scene writes a byte-identical file; export_3dgs is byte-identical except
the alpha-collapsed opacity, which may differ by one float32 ulp (CUDA vs numpy
log / exp)."""

import numpy as np
import pytest
import torch

import adam_cases as A
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _arrays(scene):
    n = len(scene)
    return np.concatenate([getattr(scene, f).cpu().numpy().astype(np.float64).reshape(n, -1)
                           for f in A.FIELDS], 1)


def _write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(np.asarray(data, dtype=np.uint8).tobytes())
    return str(p)


def _ref_scene(gold, dtype=torch.float64):
    from paper_2406_02720_b200.geometry import Scene
    f = A.split(gold["scene"], A.FIELDS, 3)
    return Scene(*(f[k] for k in A.FIELDS), sh_degree=3, background_color=(0.1, 0.25, 0.5),
                 device="cuda", dtype=dtype)


def test_load_and_save_native(cuda, tmp_path):
    from paper_2406_02720_b200 import scene_io
    gold = load_golden("io")
    sc = scene_io.load_scene(_write(tmp_path, "native.ply", gold["native_ply"]))
    assert np.array_equal(_arrays(sc), gold["scene"])
    assert sc.sh_degree == 3 and tuple(sc.background_color) == (0.1, 0.25, 0.5)
    out = tmp_path / "out.ply"
    scene_io.save_scene(_ref_scene(gold), str(out))
    assert out.read_bytes() == gold["native_ply"].tobytes()
    # float32 scenes round-trip through the double file exactly
    sc32 = _ref_scene(gold, torch.float32)
    scene_io.save_scene(sc32, str(out))
    back = scene_io.load_scene(str(out), dtype=torch.float32)
    for f in A.FIELDS:
        assert torch.equal(getattr(back, f), getattr(sc32, f)), f


def test_mixed_property_types(cuda, tmp_path):
    from paper_2406_02720_b200 import scene_io
    gold = load_golden("io")
    sc = scene_io.load_scene(_write(tmp_path, "mixed.ply", gold["mixed_ply"]))
    assert sc.sh_degree == 1
    assert np.array_equal(_arrays(sc), gold["mixed_scene"])


def test_export_and_import_3dgs(cuda, tmp_path):
    from paper_2406_02720_b200 import scene_io
    gold = load_golden("io")
    sc = _ref_scene(gold)
    for mode in ("mean", "first"):
        out = tmp_path / f"gs_{mode}.ply"
        scene_io.export_3dgs(sc, str(out), opacity=mode)
        got, ref = out.read_bytes(), gold[f"gs_{mode}_ply"].tobytes()
        hdr = ref.index(b"end_header\n") + len(b"end_header\n")
        assert got[:hdr] == ref[:hdr]
        g = np.frombuffer(got[hdr:], np.float32).reshape(45, -1)
        r = np.frombuffer(ref[hdr:], np.float32).reshape(45, -1)
        op = 9 + 45  # opacity column (after x..nz, f_dc, 45 f_rest)
        keep = [c for c in range(g.shape[1]) if c != op]
        assert np.array_equal(g[:, keep], r[:, keep]), mode
        ulps = np.abs(g[:, op].astype(np.float64) - r[:, op]) / np.spacing(np.abs(r[:, op]))
        assert ulps.max() <= 1, (mode, ulps.max())
    path = _write(tmp_path, "gs_mean.ply", gold["gs_mean_ply"])
    for init in ("zero_plus_jitter", "random_unit"):
        imp = scene_io.import_3dgs(path, normal_init=init, seed=5, background_color=(0.2,) * 3)
        assert np.array_equal(_arrays(imp), gold[f"import_{init}"]), init


def test_large_roundtrip(cuda, tmp_path):
    """1M primitives, SH degree 3: save -> load is exact (device pack/unpack)."""
    from paper_2406_02720_b200 import scene_io, scenes
    from paper_2406_02720_b200.geometry import Scene
    sa = scenes.make_config("c3")
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = tmp_path / "big.ply"
    scene_io.save_scene(sc, str(out))
    back = scene_io.load_scene(str(out), dtype=torch.float32)
    for f in A.FIELDS:
        assert torch.equal(getattr(back, f), getattr(sc, f)), f
