"""The five BASELINE.json workloads, built through the product API.

Choices the BASELINE leaves open are fixed here and recorded in
each config's ``meta``:
  * periodic x/y, wall cell layers at z=0 and z=nz-1 (geometry.cpp:535-551);
  * nu = (tau - 1/2)/3 as a double literal, Lambda = 3/16, rho0 = 1, zero
    initial populations (= equilibrium at rest);
  * C2/C3: random sequential addition (no overlap, min-image in x/y) of r=6
    spheres with centres in [0,128)x[0,64)x[1,64], seed 2, until the analytic
    bed porosity 1 - sum V / (128*64*64) <= 0.60 or 2e6 attempts;
  * C4: the stated porosity 0.5 is below the RSA jamming limit, so the bed is
    a Boolean model (overlap allowed), radii U[4,8], centres z in
    [1, 1 + 0.45*510], seed 4, until exp(-sum V / V_bed) <= 0.5 with
    V_bed = 512*256*(0.45*512); tau = 0.7 (not given in BASELINE);
  * C5: eps(z_c = z + 1/2) = 1 above z_i = nz/2, 0.5 below z_i - 8, linear in
    between, wall planes 1; K = kozeny_carman(eps, 10); nu = 1/6; Rescaled
    viscosity; c_F = 0.
The sphere lists are synthetic (the reference ships no generator that reaches
these porosities); the same list feeds the reference voxelizer in the parity
tests, so parity does not depend on it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import porolb as P

LAMBDA = 0.1875


@dataclass
class Workload:
    name: str
    dims: tuple
    scheme: P.WallScheme
    nu: float
    g: tuple
    steps: int
    pack: Optional[P.SpherePack] = None
    glbm: Optional[dict] = None  # eps, K, mode
    meta: dict = field(default_factory=dict)

    def params(self) -> P.FluidParams:
        p = P.relaxation_from_magic(self.nu, LAMBDA)
        p.body_force = tuple(self.g)
        return p

    def voxelize_options(self) -> dict:
        return dict(periodic=(True, True, False), wall_z_lo=True, wall_z_hi=True)

    def geometry(self) -> P.VoxelGeometry:
        if self.pack is None:
            return P.make_box_geometry(self.dims, **self.voxelize_options())
        return P.voxelize(self.pack, self.dims, **self.voxelize_options())

    def geometry_slab(self, x0: int, x1: int) -> P.VoxelGeometry:
        pack = self.pack if self.pack is not None else P.SpherePack(
            np.zeros((0, 3)), np.zeros(0), tuple(float(d) for d in self.dims))
        return P.voxelize_slab(pack, self.dims, x0, x1, **self.voxelize_options())

    def glbm_params(self) -> Optional[P.GlbmPlaneParams]:
        if self.glbm is None:
            return None
        return P.make_glbm_params(self.glbm["eps"], self.glbm["K"], 0.0, self.nu, LAMBDA,
                                  P.GlbmViscosity.Rescaled)


def c1() -> Workload:
    return Workload("C1_poiseuille_64x32x32_sbb", (64, 32, 32), P.WallScheme.SBB, 0.1,
                    (1e-6, 0.0, 0.0), 2000, meta=dict(tau=0.8))


def _c2_pack() -> tuple:
    pack, por = P.generate_spheres(0, 2, (128.0, 64.0, 128.0), 1.0, 64.0, 6.0, 6.0,
                                   128.0 * 64.0 * 64.0, 0.60, 2_000_000, capacity=10_000)
    return pack, por


def c2() -> Workload:
    pack, por = _c2_pack()
    return Workload("C2_bed_128x64x128_sbb", (128, 64, 128), P.WallScheme.SBB, 0.2 / 3.0,
                    (5e-7, 0.0, 0.0), 5000, pack=pack,
                    meta=dict(tau=0.7, spheres=len(pack.radii), analytic_bed_porosity=por,
                              generator="RSA r=6 seed 2"))


def c3() -> Workload:
    w = c2()
    w.name = "C3_bed_128x64x128_cli"
    w.scheme = P.WallScheme.CLI
    return w


def c4(nx_scale: int = 1) -> Workload:
    """nx_scale > 1 replicates the bed statistics over an nx_scale-times wider
    box (weak scaling: 512*nx_scale x 256 x 512)."""
    nx, ny, nz = 512 * nx_scale, 256, 512
    zb = 0.45 * nz
    pack, por = P.generate_spheres(1, 4, (float(nx), float(ny), float(nz)), 1.0,
                                   1.0 + 0.45 * (nz - 2), 4.0, 8.0, nx * ny * zb, 0.5,
                                   50_000_000, capacity=4_000_000)
    return Workload(f"C4_bed_{nx}x{ny}x{nz}_cli", (nx, ny, nz), P.WallScheme.CLI, 0.2 / 3.0,
                    (1e-7, 0.0, 0.0), 1000, pack=pack,
                    meta=dict(tau=0.7, spheres=len(pack.radii), boolean_bed_porosity=por,
                              generator="Boolean r~U[4,8] seed 4"))


def c5_eps(nz: int = 512, z_i: float = 256.0, width: float = 8.0) -> np.ndarray:
    zc = np.arange(nz) + 0.5
    eps = np.where(zc >= z_i, 1.0, np.where(zc <= z_i - width, 0.5,
                                            0.5 + 0.5 * (zc - (z_i - width)) / width))
    eps[0] = 1.0
    eps[-1] = 1.0
    return eps


def c5() -> Workload:
    eps = c5_eps()
    K = P.kozeny_carman(eps, 10.0)
    return Workload("C5_glbm_256x16x512", (256, 16, 512), P.WallScheme.SBB, 1.0 / 6.0,
                    (1e-6, 0.0, 0.0), 20000, glbm=dict(eps=eps, K=K),
                    meta=dict(z_interface=256, transition=8, grain_diameter=10.0,
                              viscosity="Rescaled"))


ALL = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def make_simulation(w: Workload, geom: Optional[P.VoxelGeometry] = None,
                    device: int = 0) -> P.Simulation:
    geom = geom if geom is not None else w.geometry()
    sim = P.Simulation.from_params(geom, w.params(), w.scheme, device)
    gp = w.glbm_params()
    if gp is not None:
        sim.set_porous(gp)
    return sim
