"""Probe: lid set mid-run (SBB/CLI schemes, both layouts, both math modes) vs the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1507_06565_b200 as pg
from oracle.oracle import load_oracle
from test_gpu_fast import lid_bed, rel_err
from test_gpu_parity import fluid_mask
orc = load_oracle()
for layout in ("dense", "compact"):
    os.environ["PGPU_LAYOUT"] = layout
    for persistent in ("1", "0"):
        os.environ["PGPU_PERSISTENT"] = persistent
        for math in (0, 1):
            for scheme in (0, 1):
                for pre in (0, 7):
                    geom = lid_bed(pg)
                    p = pg.relaxation_from_magic(1.0 / 6.0, 3.0 / 16.0)
                    p.body_force = (1e-6, 0, 0)
                    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
                    sim.math_mode = math
                    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
                    sim.step(pre); o.step(pre)
                    sim.set_lid_velocity((0.01, 0.002, 0.0)); o.set_lid_velocity((0.01, 0.002, 0.0))
                    sim.step(30); o.step(30)
                    m = fluid_mask(geom)
                    print(layout, "pers" + persistent, "fast" if math else "exact", "scheme", scheme, "pre", pre,
                          f"{rel_err(sim.get_pdfs()[:, m], o.get_pdfs()[:, m]):.3e}", flush=True)
