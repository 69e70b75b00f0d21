"""Host->device copy paths for a 700 MB pageable array (the C4 link upload)."""
import time, threading
import numpy as np
import torch
n = 700 * 2**20
src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
st = torch.from_numpy(src)
print("pageable copy_       %.1f ms" % (1e3 * t(lambda: dev.copy_(st))))
pin = torch.empty(n, dtype=torch.uint8).pin_memory()
pn = pin.numpy()
print("pinned H2D           %.1f ms" % (1e3 * t(lambda: dev.copy_(pin, non_blocking=True))))
print("memcpy->pinned 1thr  %.1f ms" % (1e3 * t(lambda: np.copyto(pn, src))))
def par_copy(k):
    def run():
        th = []
        for i in range(k):
            a, b = n * i // k, n * (i + 1) // k
            th.append(threading.Thread(target=np.copyto, args=(pn[a:b], src[a:b])))
        for x in th: x.start()
        for x in th: x.join()
    return run
for k in (2, 4, 8, 16):
    print("memcpy->pinned %2dthr %.1f ms" % (k, 1e3 * t(par_copy(k))))
