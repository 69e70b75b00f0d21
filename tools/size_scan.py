"""Fluid MLUPS of the fluid-only K1 kernels over domain size and shape (one B200):
separates the small-domain losses (launch ramp / tail, L2 residency) from the
x-extent (units holding an x face take the wrap path).
    python tools/size_scan.py [units|cpipe ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_06565_b200 as pg  # noqa: E402

SHAPES = [(128, 64, 128), (512, 64, 32), (128, 128, 256), (512, 64, 128), (256, 128, 256),
          (128, 256, 512), (512, 128, 256)]


def geometry(dims, seed=3):
    rng = np.random.default_rng(seed)
    vol = dims[0] * dims[1] * (dims[2] // 2)
    n = int(0.55 * vol / (4.0 / 3.0 * np.pi * 6.0 ** 3))
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n), rng.uniform(1, dims[2] // 2, n)]
    pack = pg.SpherePack(c, np.full(n, 6.0), tuple(float(d) for d in dims))
    return pg.voxelize(pack, dims, (True, True, False), True, True)


def main():
    kernels = sys.argv[1:] or ["cpipe", "units"]
    os.environ["PGPU_LAYOUT"] = "compact"
    peak = 6558.7
    for dims in SHAPES:
        geom = geometry(dims)
        for scheme in (0, 1):
            for k in kernels:
                os.environ["PGPU_SWEEP"] = k
                p = pg.relaxation_from_magic(1.0 / 15.0, 3.0 / 16.0)
                p.body_force = (5e-7, 0.0, 0.0)
                sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
                sim.math_mode = pg.MathMode.FAST
                stream = torch.cuda.Stream()
                sim.set_stream(stream.cuda_stream)
                sim.step(20)
                sim.prepare()
                torch.cuda.synchronize()
                steps = max(32, int(2e9 / (304 * geom.fluid_cells)) // 16 * 16)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sim.step(steps)
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                gbs = 304 * geom.fluid_cells * steps / (ms * 1e-3) / 1e9
                print(dims, "cells", int(np.prod(dims)), "fluid", geom.fluid_cells, "links", geom.n_links,
                      "CLI" if scheme else "SBB", sim.sweep_kernel,
                      "us/step", round(1e3 * ms / steps, 1), "frac", round(gbs / peak, 3), flush=True)
                del sim


if __name__ == "__main__":
    main()
