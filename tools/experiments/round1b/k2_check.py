"""Experiment check used with the temporal-blocking prototype (tools/experiments/k2_plane_sync.cu wired in behind PGPU_K2=1; not in the product build): two-steps-per-launch vs the one-step sweep, bitwise."""
import os, sys, time, subprocess
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np

script = r'''
import sys, numpy as np, time
sys.path.insert(0, %r)
import paper_1507_06565_b200 as pg
from paper_1507_06565_b200 import configs
rng = np.random.default_rng(3)
dims = (96, 40, 48)
n = 40
c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n), rng.uniform(1, dims[2] - 1, n)]
r = rng.uniform(2.5, 6.0, n)
geom = pg.voxelize(pg.SpherePack(c, r, tuple(float(d) for d in dims)), dims, (True, True, False), True, True)
p = pg.relaxation_from_magic(0.1, 3.0 / 16.0)
p.body_force = (1e-6, 2e-7, 0.0)
sim = pg.Simulation.from_params(geom, p, pg.WallScheme.SBB)
sim.step(21)
np.save(sys.argv[1], sim.get_pdfs())
print("launches", sim.launch_count)
''' % str(ROOT)
out = {}
for k2 in ("0", "1"):
    env = dict(os.environ, PGPU_LAYOUT="compact", PGPU_K2=k2, PGPU_PERSISTENT="0")
    fn = f"/tmp/k2_{k2}.npy"
    res = subprocess.run([sys.executable, "-c", script, fn], env=env, capture_output=True, text=True)
    print(k2, res.stdout.strip(), res.stderr[-500:])
    out[k2] = np.load(fn)
print("bitwise equal:", np.array_equal(out["0"], out["1"]), "max diff", np.abs(out["0"] - out["1"]).max())
