import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1507_06565_b200 as pg
def geometry(dims, n, rmin, rmax, seed, periodic=(True, True, False), walls=True):
    rng = np.random.default_rng(seed)
    zlo, zhi = (1.0, dims[2] - 1.0) if walls else (0.0, float(dims[2]))
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n), rng.uniform(zlo, zhi, n)]
    r = rng.uniform(rmin, rmax, n)
    return pg.voxelize(pg.SpherePack(c, r, tuple(float(d) for d in dims)), dims, periodic, walls, walls)
for scheme in (0, 1):
  for dims in [(128, 32, 40), (64, 16, 12)]:
    g = geometry(dims, 20, 2.0, 5.0, 7)
    p = pg.relaxation_from_magic(0.08, 3.0/16.0); p.body_force = (2e-6, 1e-6, -5e-7)
    os.environ["PGPU_LAYOUT"] = "compact"
    os.environ["PGPU_SWEEP"] = "tb2"; a = pg.Simulation.from_params(g, p, pg.WallScheme(scheme))
    os.environ["PGPU_SWEEP"] = "cpipe"; b = pg.Simulation.from_params(g, p, pg.WallScheme(scheme))
    nx, ny, nz = dims
    m = g.flags.reshape(nz, ny, nx) == 0
    rng = np.random.default_rng(1); f0 = 1e-3*(2*rng.random((19, nz, ny, nx))-1); f0[:, ~m] = 0
    a.set_pdfs(f0); b.set_pdfs(f0)
    a.step(1); b.step(1)
    res = []
    for it in range(6):
        a.step(2); b.step(2)
        fa, fb = a.get_pdfs(), b.get_pdfs()
        d = fa[:, m] != fb[:, m]
        res.append(int(d.sum()))
        if d.any():
            bad = np.argwhere((fa != fb) & m[None])
            zs = sorted(set(bad[:, 1].tolist())); ys = sorted(set(bad[:, 2].tolist()))
            res.append(("z", zs[:10], "y", ys[:10], "dirs", sorted(set(bad[:,0].tolist()))))
            break
    print(scheme, dims, a.sweep_kernel, res, flush=True)
