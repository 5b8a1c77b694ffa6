"""Scene I/O throughput at c3 size (1M half-Gaussians, SH3): device pack/unpack kernel
time (CUDA events) and end-to-end save/load through the drop-in scene_io API."""
import json
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02720_b200 import _native, device, scene_io, scenes  # noqa: E402
from paper_2406_02720_b200.geometry import Scene  # noqa: E402
import ctypes  # noqa: E402


def main():
    sa = scenes.make_config("c3")
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    lib = _native.load()
    row = lib.hs_ply_row_bytes(3, 0)
    buf = torch.empty(len(sc) * row, dtype=torch.uint8, device="cuda")
    st = device.scene_struct(sc)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        lib.hs_ply_pack(ctypes.byref(st), ctypes.c_void_p(buf.data_ptr()), 0, device._stream())
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        lib.hs_ply_pack(ctypes.byref(st), ctypes.c_void_p(buf.data_ptr()), 0, device._stream())
    ev[1].record()
    torch.cuda.synchronize()
    pack_ms = ev[0].elapsed_time(ev[1]) / 10
    scene_bytes = sum(getattr(sc, f).numel() for f in sc.FIELDS) * 4
    path = os.path.join(tempfile.mkdtemp(), "c3.ply")
    t0 = time.perf_counter()
    scene_io.save_scene(sc, path)
    save_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    back = scene_io.load_scene(path, dtype=torch.float32)
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t0
    ok = all(torch.equal(getattr(back, f), getattr(sc, f)) for f in sc.FIELDS)
    print(json.dumps({
        "n": len(sc), "file_bytes": os.path.getsize(path),
        "pack_kernel_ms": pack_ms,
        "pack_hbm_gbs": (scene_bytes + buf.numel()) / (pack_ms * 1e-3) / 1e9,
        "save_s": save_s, "load_s": load_s, "roundtrip_exact": ok}))


if __name__ == "__main__":
    main()
