import time, torch
nb = 252 * 1024 * 1024 // 4
dev = torch.empty(nb, dtype=torch.float32, device="cuda")
host = torch.empty(nb, dtype=torch.float32).pin_memory()
host.fill_(1.0)
def run(k, n=10, direction="h2d"):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = (nb + k - 1) // k
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                if direction == "h2d":
                    dev[i*chunk:(i+1)*chunk].copy_(host[i*chunk:(i+1)*chunk], non_blocking=True)
                else:
                    host[i*chunk:(i+1)*chunk].copy_(dev[i*chunk:(i+1)*chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{direction} {k} streams: {dt*1e3:.2f} ms  {nb*4/dt/1e9:.1f} GB/s")
for k in (1, 2, 4, 8):
    run(k)
for k in (1, 2, 4):
    run(k, direction="d2h")
# both directions at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dev2 = torch.empty_like(dev); host2 = torch.empty_like(host).pin_memory()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): dev.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2): host2.copy_(dev2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
print(f"duplex: {dt*1e3:.2f} ms for {2*nb*4/1e6:.0f} MB  {2*nb*4/dt/1e9:.1f} GB/s total")
