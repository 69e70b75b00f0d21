"""ORACLE / TEST INFRASTRUCTURE ONLY: the BASELINE workloads built without the
product, for bench.py's reference arm (``--impl reference``).

Each workload follows the recipe of paper_1507_06565_b200/configs.py (same
seeds, generator parameters, physics), but the sphere list comes from the
oracle's harness generator (orc_generate_spheres), the geometry from the
oracle voxelizer (orc_voxelize_fast, byte-identical to the reference's
voxelize()), and the relaxation / GLBM parameters from the reference itself
(oracle/_ref).  The geometry is checked against the sha256 recorded in
tests/golden/<config>.json, which the reference's own voxelize() produced, so
the reference arm provably times the same input as the product arm.
tests/test_oracle.py checks these recipes against configs.py.
"""
from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

from .oracle import OracleLib, RefLib

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"
LAMBDA = 0.1875
SCHEME = {"SBB": 0, "CLI": 1}


@dataclass
class RefWorkload:
    name: str
    dims: tuple
    scheme: str
    nu: float
    g: tuple
    steps: int
    spheres: Optional[dict] = None  # orc_generate_spheres arguments
    glbm: bool = False
    meta: dict = field(default_factory=dict)


def _c4_spheres(nx_scale: int = 1) -> dict:
    nx, ny, nz = 512 * nx_scale, 256, 512
    return dict(mode=1, seed=4, box=(float(nx), float(ny), float(nz)), z_lo=1.0,
                z_hi=1.0 + 0.45 * (nz - 2), r_min=4.0, r_max=8.0,
                bed_volume=nx * ny * (0.45 * nz), target_porosity=0.5,
                max_attempts=50_000_000, capacity=4_000_000)


_C2_SPHERES = dict(mode=0, seed=2, box=(128.0, 64.0, 128.0), z_lo=1.0, z_hi=64.0, r_min=6.0,
                   r_max=6.0, bed_volume=128.0 * 64.0 * 64.0, target_porosity=0.60,
                   max_attempts=2_000_000, capacity=10_000)

WORKLOADS = {
    "C1": RefWorkload("C1_poiseuille_64x32x32_sbb", (64, 32, 32), "SBB", 0.1, (1e-6, 0.0, 0.0),
                      2000, meta=dict(tau=0.8)),
    "C2": RefWorkload("C2_bed_128x64x128_sbb", (128, 64, 128), "SBB", 0.2 / 3.0,
                      (5e-7, 0.0, 0.0), 5000, spheres=_C2_SPHERES,
                      meta=dict(tau=0.7, generator="RSA r=6 seed 2")),
    "C3": RefWorkload("C3_bed_128x64x128_cli", (128, 64, 128), "CLI", 0.2 / 3.0,
                      (5e-7, 0.0, 0.0), 5000, spheres=_C2_SPHERES,
                      meta=dict(tau=0.7, generator="RSA r=6 seed 2")),
    "C4": RefWorkload("C4_bed_512x256x512_cli", (512, 256, 512), "CLI", 0.2 / 3.0,
                      (1e-7, 0.0, 0.0), 1000, spheres=_c4_spheres(),
                      meta=dict(tau=0.7, generator="Boolean r~U[4,8] seed 4")),
    "C5": RefWorkload("C5_glbm_256x16x512", (256, 16, 512), "SBB", 1.0 / 6.0, (1e-6, 0.0, 0.0),
                      20000, glbm=True,
                      meta=dict(z_interface=256, transition=8, grain_diameter=10.0,
                                viscosity="Rescaled")),
}


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def geometry_hashes(g) -> dict:
    return {
        "flags_sha256": _sha(g.flags),
        "links_sha256": _sha(np.concatenate([
            np.ascontiguousarray(g.link_fluid_cell, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_second_fluid, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_direction, dtype=np.int32).view(np.uint8),
            np.ascontiguousarray(g.link_q, dtype=np.float32).view(np.uint8)])),
        "porosity_sha256": _sha(np.asarray(g.porosity, dtype=np.float64)),
    }


def build(key: str, orc: Optional[OracleLib] = None, check: bool = True):
    """(workload, geometry OGeom, meta) from oracle code only; raises if the
    geometry differs from the reference-made golden fixture."""
    orc = orc or OracleLib()
    w = WORKLOADS[key]
    meta = dict(w.meta)
    centers, radii = np.zeros((0, 3)), np.zeros(0)
    if w.spheres is not None:
        centers, radii, por = orc.generate_spheres(**w.spheres)
        meta["spheres"] = int(radii.size)
        meta["boolean_bed_porosity" if w.spheres["mode"] == 1 else "analytic_bed_porosity"] = por
    box = tuple(float(d) for d in w.dims)
    geom = orc.voxelize_fast(centers, radii, box, w.dims, (True, True, False), True, True)
    if check:
        path = GOLDEN / f"{key}.json"
        if path.exists():
            gold = json.loads(path.read_text())["geometry"]
            got = geometry_hashes(geom)
            for k, v in got.items():
                if gold.get(k) != v:
                    raise RuntimeError(f"{key}: oracle geometry {k} differs from the golden "
                                       f"fixture made by the reference voxelize()")
            meta["geometry_checked"] = f"sha256 == tests/golden/{key}.json (reference voxelize)"
    return w, geom, meta


def reference_simulation(ref: RefLib, w: RefWorkload, geom):
    """The reference's Simulation on the workload (oracle/_ref)."""
    wp, wm = ref.relaxation_from_magic(w.nu, LAMBDA)
    sim = ref.simulation(geom, w.nu, wp, wm, LAMBDA, w.g, SCHEME[w.scheme])
    if w.glbm:
        nz = w.dims[2]
        zc = np.arange(nz) + 0.5
        eps = np.where(zc >= 256.0, 1.0, np.where(zc <= 248.0, 0.5, 0.5 + 0.5 * (zc - 248.0) / 8.0))
        eps[0] = eps[-1] = 1.0
        K = ref.kozeny_carman(eps, 10.0)
        gwp, gwm = ref.make_glbm_params(eps, K, 0.0, w.nu, LAMBDA, 1)
        sim.set_porous(eps, K, gwp, gwm, 0.0, True)
    return sim
