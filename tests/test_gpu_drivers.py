"""The reference's driver-level known-answer tests for the homogenised (GLBM)
path, run on the B200 through run_to_steady and compared with the reference
solver's own run of the same setup (proj/tests/test_glbm.cpp:39-73;
proj/src/glbm.cpp:38-88 run_couette_porous, :113-144 run_glbm_channel)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["dense", "compact"], autouse=True)
def layout(request, monkeypatch):
    """Every test here runs on both PDF layouts (PGPU_LAYOUT is read at
    pgpu_create): the dense reference layout and the fluid-only one."""
    monkeypatch.setenv("PGPU_LAYOUT", request.param)
    return request.param


def channel_box(pg, nz):
    return pg.make_box_geometry((4, 4, nz), (True, True, False), True, True)


def test_glbm_channel_eps1_is_poiseuille(gpu, ref):
    """test_glbm.cpp:39-59 (run_glbm_channel with eps = 1, K = inf)."""
    pg = gpu
    H, g, nu = 16, 1e-8, 1.0 / 6.0
    geom = channel_box(pg, H + 2)
    eps = np.ones(H + 2)
    K = np.full(H + 2, np.inf)
    gp = pg.make_glbm_params(eps, K, 0.0, nu, 3.0 / 16.0, pg.GlbmViscosity.Rescaled)
    sim = pg.Simulation(geom, nu, 3.0 / 16.0, (g, 0, 0), pg.WallScheme.SBB)
    sim.set_porous(gp)
    st, prof = pg.run_to_steady(sim, 1e-12, 500, 300000)
    assert st.converged
    zz = prof.z - prof.z0
    exact = g / (2 * nu) * zz * (H - zz)
    assert np.all(np.abs(prof.u_superficial - exact) <= 1e-8 * np.abs(exact))
    wp, wm = ref.relaxation_from_magic(nu, 3.0 / 16.0)
    r = ref.simulation(geom, nu, wp, wm, 3.0 / 16.0, (g, 0, 0), 0)
    r.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, 0.0, True)
    rs = r.run_to_steady_state(1e-12, 500, 300000)
    assert (st.steps, st.residual) == (rs["steps"], rs["residual"])
    assert np.array_equal(prof.u_superficial, r.planar_profile()["u_superficial"])


def couette_semi_analytic(u0, H, eps, K, nu, nu_eff, y):
    """glbm.hpp:8-13 (two-domain Brinkman Couette profile)."""
    r = math.sqrt(nu * eps) / math.sqrt(nu_eff * K)
    a = 2.0 * u0 / (2.0 * r * K + eps * H)
    return np.where(y >= H / 2, r * K * a + eps * a * (y - H / 2),
                    r * K * a * np.exp(r * (y - H / 2)))


def test_half_porous_couette(gpu, ref):
    """test_glbm.cpp:61-73: GLBM + moving lid (velocity bounce-back) on a
    half-porous channel; B200 run bit-identical to the reference run and within
    2 % (L2) of the semi-analytic profile."""
    pg = gpu
    H, eps_p, darcy, J, re, nu, lam = 32, 0.4, 4.8e-4, 1.0, 0.1, 1.0 / 6.0, 3.0 / 16.0
    K = darcy * H * H
    u0 = re * nu / H
    nz = H + 2
    geom = channel_box(pg, nz)
    eps = np.ones(nz)
    perm = np.full(nz, np.inf)
    zc = np.arange(nz) + 0.5
    porous = (zc > 1.0) & (zc < 1.0 + H / 2.0)  # glbm.cpp:52-60
    eps[porous] = eps_p
    perm[porous] = K
    gp = pg.make_glbm_params(eps, perm, 0.0, nu, lam, pg.GlbmViscosity.ConstantRatio, J)
    sim = pg.Simulation(geom, nu, lam, (0, 0, 0), pg.WallScheme.SBB)
    sim.set_porous(gp)
    sim.set_lid_velocity((u0, 0.0, 0.0))
    st, prof = pg.run_to_steady(sim, 1e-11, 1000, 600000)
    assert st.converged
    wp, wm = ref.relaxation_from_magic(nu, lam)
    r = ref.simulation(geom, nu, wp, wm, lam, (0, 0, 0), 0)
    r.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, 0.0, True)
    r.set_lid_velocity((u0, 0.0, 0.0))
    rs = r.run_to_steady_state(1e-11, 1000, 600000)
    assert (st.steps, st.residual, st.converged) == (rs["steps"], rs["residual"], rs["converged"])
    rp = r.planar_profile()
    assert np.array_equal(prof.u_superficial, rp["u_superficial"])
    y = prof.z - 1.0
    ana = couette_semi_analytic(u0, H, eps_p, K, nu, J * nu, y)
    rel_l2 = math.sqrt(((prof.u_superficial - ana) ** 2).sum() / (ana ** 2).sum())
    assert rel_l2 < 0.02
