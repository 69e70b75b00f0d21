"""Check that the product voxelizer reproduces the REFERENCE voxelize() on the
full C4 geometry (512x256x512, 20,783 spheres): runs the reference (single
threaded, ~35-55 min) and stores the comparison in C4_voxelize_check.json."""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import RefLib  # noqa: E402
from paper_1507_06565_b200 import configs  # noqa: E402


def digest(g):
    h = hashlib.sha256()
    for a in (g.flags, np.asarray(g.porosity, np.float64), np.asarray(g.link_fluid_cell, np.int64),
              np.asarray(g.link_second_fluid, np.int64), np.asarray(g.link_direction, np.int32),
              np.asarray(g.link_q, np.float32)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


w = configs.c4()
t0 = time.time()
p = w.geometry()
tp = time.time() - t0
t0 = time.time()
r = RefLib().voxelize(w.pack.centers, w.pack.radii, w.pack.box, w.dims, (1, 1, 0), True, True)
tr = time.time() - t0
out = {"workload": w.name, "product_sha256": digest(p), "reference_sha256": digest(r),
       "identical": digest(p) == digest(r), "n_links": int(p.n_links),
       "q_fallback_count": [int(p.q_fallback_count), int(r.q_fallback_count)],
       "product_seconds_8_threads": tp, "reference_seconds_1_thread": tr}
(Path(__file__).resolve().parent / "C4_voxelize_check.json").write_text(json.dumps(out, indent=1))
print(out)
