import sys, time, os
sys.path.insert(0, '.')
import paper_1507_06565_b200 as pg
from paper_1507_06565_b200 import configs
w = configs.c4()
g = pg.voxelize_device(w.pack, w.dims, **w.voxelize_options())
for i in range(3):
    t0 = time.perf_counter()
    s = configs.make_simulation(w, g)
    s.synchronize()
    print("create", time.perf_counter() - t0, flush=True)
    t0 = time.perf_counter(); s.close(); print("close", time.perf_counter()-t0, flush=True)
