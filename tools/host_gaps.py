"""Where does a step's wall time go?  Times one fwd+bwd step at c3 split by host
calls (perf_counter with device syncs) and reports GPU kernel time from events."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

sa = scenes.make_config("c3")
cam = CameraModel(**sa.cameras[0])
sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=3, background_color=sa.background_color,
           device="cuda", dtype=torch.float32)
dc = torch.as_tensor(scenes.cotangent(1080, 1920), dtype=torch.float32, device="cuda")
g = device.DeviceGradientSet.empty_flat(sc)
for _ in range(3):
    o = device.render(sc, cam); device.render_backward(sc, cam, o, dc, grads=g)
torch.cuda.synchronize()
for trial in range(3):
    t = {}
    t0 = time.perf_counter()
    fr = device.prepare(sc, cam); t["prepare(host, incl sync)"] = time.perf_counter() - t0
    t1 = time.perf_counter(); o = device.render(sc, cam, frame=fr); t["render launch"] = time.perf_counter() - t1
    t1 = time.perf_counter(); device.render_backward(sc, cam, o, dc, grads=g); t["bwd launch"] = time.perf_counter() - t1
    t1 = time.perf_counter(); torch.cuda.synchronize(); t["drain"] = time.perf_counter() - t1
    t["total"] = time.perf_counter() - t0
    print({k: "%.3f ms" % (v * 1e3) for k, v in t.items()})
# steady-state loop timing with events, no profiler, no nvidia-smi
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label in ("loop",):
    torch.cuda.synchronize(); s.record()
    for _ in range(20):
        o = device.render(sc, cam); device.render_backward(sc, cam, o, dc, grads=g)
    e.record(); torch.cuda.synchronize()
    print(label, "%.3f ms/step" % (s.elapsed_time(e) / 20))
# prepare internals
import ctypes
from paper_2406_02720_b200 import _native
lib = _native.load()
for trial in range(2):
    t0 = time.perf_counter(); f = device.DeviceFrame(sc, cam, "half"); a = time.perf_counter()
    st = lib.hs_preprocess_fwd(ctypes.byref(f.st), ctypes.byref(device.scene_struct(sc)),
                               ctypes.byref(device.camera_struct(cam)), device._ptr(f.radii), device._stream())
    b = time.perf_counter(); lib.hs_frame_read_num_pairs(ctypes.byref(f.st), device._stream()); c = time.perf_counter()
    f.alloc_binning(); d = time.perf_counter()
    lib.hs_bin_and_sort(ctypes.byref(f.st), device._stream()); e2 = time.perf_counter()
    torch.cuda.synchronize(); ff = time.perf_counter()
    print("frame init %.3f pre launch %.3f readP(sync) %.3f alloc_bin %.3f bin launch %.3f drain %.3f ms" % tuple(
        1e3 * x for x in (a - t0, b - a, c - b, d - c, e2 - d, ff - e2)))
