"""Host->device upload probe (pageable vs registered vs threaded pageable)."""
import ctypes, threading, time
import numpy as np
import torch

torch.cuda.init()
N = 700 * 2**20
d = torch.empty(N, dtype=torch.uint8, device="cuda")
a = np.ones(N, np.uint8)
rt = torch.cuda.cudart()
lib = ctypes.CDLL("libcudart.so.12") if False else None


def pageable_threads(nt):
    chunk = N // nt
    streams = [torch.cuda.Stream() for _ in range(nt)]
    src = torch.from_numpy(a)

    def work(i):
        with torch.cuda.stream(streams[i]):
            d[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        streams[i].synchronize()

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(i,)) for i in range(nt)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for nt in (1, 2, 4, 8):
    best = min(pageable_threads(nt) for _ in range(3))
    print(f"pageable threads={nt}: {best*1e3:.1f} ms  {N/best/1e9:.1f} GB/s", flush=True)

for rep in range(2):
    t0 = time.perf_counter()
    rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms copy {1e3*(t2-t1):.1f} ms unregister {1e3*(t3-t2):.1f} ms", flush=True)
