"""Host<->device copy rates on this box (pinned / pageable, both directions, and
concurrent), plus the host-side conversions the drop-in API may need."""
import time
import numpy as np
import torch


def bw(label, fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{label:44s} {dt * 1e3:8.2f} ms  {nbytes / dt / 1e9:7.1f} GB/s", flush=True)


n = 256 << 20
hp = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hp2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hq = torch.empty(n, dtype=torch.uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
bw("H2D pinned 256MB", lambda: d.copy_(hp, non_blocking=True), n)
bw("D2H pinned 256MB", lambda: hp.copy_(d, non_blocking=True), n)
bw("H2D pageable 256MB", lambda: d.copy_(hq), n)
bw("D2H pageable 256MB", lambda: hq.copy_(d), n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        d.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2):
        hp2.copy_(d2, non_blocking=True)
    s1.synchronize(); s2.synchronize()


bw("H2D + D2H concurrent 2x256MB", both, 2 * n)
a64 = np.random.default_rng(0).uniform(-1, 1, (1080, 1920, 3))
p32 = torch.empty(a64.shape, dtype=torch.float32, pin_memory=True)
bw("host f64->f32 into pinned (torch copy_)", lambda: p32.copy_(torch.from_numpy(a64)), a64.nbytes)
print("torch threads", torch.get_num_threads())
dd = torch.empty(a64.shape, dtype=torch.float64, device="cuda")
bw("H2D pageable f64 d_color 50MB", lambda: dd.copy_(torch.from_numpy(a64)), a64.nbytes)
bw("np.empty 260MB + touch", lambda: np.ones(65 << 20, np.float32), 260 << 20)
