"""Device->host copy of ~10 GB into pinned memory: one stream vs two/four streams."""
import time
import torch
n = 10 * 2**30 // 8
dev = torch.empty(n, dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64).pin_memory()
def run(k):
    ss = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, s in enumerate(ss):
        a, b = n * i // k, n * (i + 1) // k
        with torch.cuda.stream(s):
            host[a:b].copy_(dev[a:b], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0
for k in (1, 2, 4, 1, 2):
    t = run(k)
    print(f"{k} streams: {1e3*t:.1f} ms  {n*8/t/1e9:.1f} GB/s", flush=True)
