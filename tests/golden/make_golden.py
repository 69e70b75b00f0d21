"""Generate the golden parity fixtures from the REFERENCE solver (oracle/_ref,
compiled from /root/reference's own sources).  Run in the build container:

    python tests/golden/make_golden.py C1 C2 C3 C5 [--threads 8]

For each BASELINE config it builds the geometry with the reference voxelizer
(same sphere list as paper_1507_06565_b200.configs), runs the reference
Simulation for the stated step count and stores, as JSON (floats as hex so
they round-trip exactly):
  * geometry: sha256 of flags / link arrays, counts, q fallbacks;
  * the fluid-cell populations f(N): sha256 of the bytes of f[:, fluid]
    (C order), per-direction sums, and 4096 seeded samples;
  * the velocity field: sha256 per component over fluid cells and samples;
  * the planar profile (u_superficial, u_intrinsic) and max_speed.
The GPU parity tests (tests/test_gpu_configs.py) compare against these without
needing /root/reference at run time.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import RefLib  # noqa: E402
from paper_1507_06565_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexs(a) -> list:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def geometry_record(g) -> dict:
    return {
        "dims": list(g.dims), "flags_sha256": sha(g.flags), "n_links": int(g.n_links),
        "fluid_cells": int(g.fluid_cells), "q_fallback_count": int(g.q_fallback_count),
        "links_sha256": sha(np.concatenate([
            np.ascontiguousarray(g.link_fluid_cell, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_second_fluid, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_direction, dtype=np.int32).view(np.uint8),
            np.ascontiguousarray(g.link_q, dtype=np.float32).view(np.uint8)])),
        "porosity_sha256": sha(np.asarray(g.porosity, dtype=np.float64)),
    }


def state_record(f: np.ndarray, fields, prof: dict, vmax: float, fluid: np.ndarray) -> dict:
    ff = f[:, fluid]  # (19, nfluid)
    rng = np.random.default_rng(12345)
    nfl = ff.shape[1]
    ks = rng.integers(0, 19, 4096)
    cs = rng.integers(0, nfl, 4096)
    fluid_idx = np.nonzero(fluid.ravel())[0]
    rec = {
        "pdf_sha256": sha(ff),
        "pdf_k_sums": hexs([math.fsum(ff[k]) for k in range(19)]),
        "pdf_absmax": float(np.abs(ff).max()).hex(),
        "sample_k": ks.tolist(), "sample_cell": fluid_idx[cs].tolist(),
        "sample_value": hexs(ff[ks, cs]),
    }
    names = ["drho", "ux", "uy", "uz"]
    for n, a in zip(names, fields):
        v = a[fluid]
        rec[f"{n}_sha256"] = sha(v)
        rec[f"{n}_sample"] = hexs(v[cs])
        rec[f"{n}_absmax"] = float(np.abs(v).max()).hex()
    rec["profile_z"] = hexs(prof["z"])
    rec["profile_u_superficial"] = hexs(prof["u_superficial"])
    rec["profile_u_intrinsic"] = hexs(prof["u_intrinsic"])
    rec["profile_u_max"] = float(prof["u_max"]).hex()
    rec["max_speed"] = float(vmax).hex()
    return rec


def make(name: str, threads: int, steps_override: int | None = None,
         product_geometry: bool = False) -> dict:
    ref = RefLib()
    ref.set_threads(threads)
    w = configs.ALL[name]()
    opt = dict(periodic=(True, True, False), wall_lo=True, wall_hi=True)
    t0 = time.time()
    if product_geometry:
        # C4: the reference voxelize() needs ~35-55 single-threaded minutes; the
        # product voxelizer is byte-identical (tests/test_voxelize.py, and for C4
        # itself tests/golden/verify_c4_voxelize.py -> C4_voxelize_check.json)
        g = w.geometry()
    elif w.pack is None:
        g = ref.make_box_geometry(w.dims, **opt)
    else:
        g = ref.voxelize(w.pack.centers, w.pack.radii, w.pack.box, w.dims, **opt)
    t_vox = time.time() - t0
    p = w.params()
    sim = ref.simulation(g, p.nu, p.omega_plus, p.omega_minus, p.lambda_magic, p.body_force,
                         int(w.scheme))
    gp = w.glbm_params()
    if gp is not None:
        sim.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, 0.0, True)
    steps = steps_override or w.steps
    t0 = time.time()
    sim.step(steps)
    t_run = time.time() - t0
    nx, ny, nz = w.dims
    fluid = (g.flags.reshape(nz, ny, nx) == 0)
    rec = {
        "config": name, "workload": w.name, "steps": steps, "scheme": w.scheme.name,
        "params": {"nu": p.nu, "omega_plus": p.omega_plus.hex(), "omega_minus": p.omega_minus.hex(),
                   "body_force": list(p.body_force)},
        "meta": {k: (v if isinstance(v, (int, float, str)) else str(v)) for k, v in w.meta.items()},
        "sphere_sha256": sha(np.c_[w.pack.centers, w.pack.radii]) if w.pack is not None else None,
        "geometry": geometry_record(g),
        "state": state_record(sim.get_pdfs(), sim.macroscopic_fields(), sim.planar_profile(),
                              sim.max_speed(), fluid),
        "reference_timing": {"voxelize_s": t_vox, "run_s": t_run, "threads": threads,
                             "fluid_mlups": float(g.fluid_cells) * steps / t_run / 1e6},
        "generator": "tests/golden/make_golden.py with oracle/_ref (reference sources, -O3 -fopenmp)",
        "geometry_source": "product voxelize (byte-identical)" if product_geometry
                           else "reference voxelize",
    }
    return rec


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--product-geometry", action="store_true")
    args = ap.parse_args()
    for name in args.configs:
        rec = make(name, args.threads, args.steps, args.product_geometry)
        suffix = "" if args.steps is None else f"_{args.steps}"
        (OUT / f"{name}{suffix}.json").write_text(json.dumps(rec, indent=1))
        print(name, rec["reference_timing"], flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
