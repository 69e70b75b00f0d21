"""Breakdown of the e2e path on C4 (create / steps / get_pdfs / profile), both layouts."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1507_06565_b200 as pg
from paper_1507_06565_b200 import configs

w = configs.c4()
geom = w.geometry()
host = torch.empty(19 * geom.cells, dtype=torch.float64, pin_memory=True).numpy().reshape(19, *geom.dims[::-1])
for layout in sys.argv[1:] or ["compact", "dense"]:
    os.environ["PGPU_LAYOUT"] = layout
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim = configs.make_simulation(w, geom)
        t1 = time.perf_counter()
        sim.step(100)
        sim.synchronize() if hasattr(sim, "synchronize") else None
        t2 = time.perf_counter()
        sim.get_pdfs(host)
        t3 = time.perf_counter()
        prof = sim.planar_profile()
        t4 = time.perf_counter()
        prof = sim.planar_profile()
        t5 = time.perf_counter()
        print(f"{layout} rep{rep}: create {1e3*(t1-t0):.1f} ms  steps {1e3*(t2-t1):.1f}  get_pdfs {1e3*(t3-t2):.1f}  "
              f"profile {1e3*(t4-t3):.1f}  profile again {1e3*(t5-t4):.1f}", flush=True)
        del sim
