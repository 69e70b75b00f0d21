"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

The bar is BIT-EXACT equality of the fluid-cell populations, velocities and
profiles (the kernels use explicit round-to-nearest fp64 intrinsics in the
reference's operation order), which is stronger than the north star's
<= 1e-12 relative tolerance; where a test states a tolerance it is that
1e-12 bar.  Cases restate the reference's own known-answer tests
(proj/tests/test_simulation.cpp, test_boundary.cpp, acceptance_main.cpp).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["dense", "compact"], autouse=True)
def layout(request, monkeypatch):
    """Every test here runs on both PDF layouts (PGPU_LAYOUT is read at
    pgpu_create): the dense reference layout and the fluid-only one."""
    monkeypatch.setenv("PGPU_LAYOUT", request.param)
    return request.param

TOL = 1e-12  # north star: PDFs and velocities within 1e-12 relative


def fluid_mask(geom):
    nx, ny, nz = geom.dims
    return geom.flags.reshape(nz, ny, nx) == 0


def assert_bitwise(got, want, mask, what=""):
    a, b = got[..., mask] if got.ndim == 4 else got[mask], want[..., mask] if want.ndim == 4 else want[mask]
    if not np.array_equal(a, b):
        scale = max(np.abs(b).max(), 1e-300)
        raise AssertionError(f"{what}: not bit-identical, max rel diff {np.abs(a - b).max() / scale:.3e}")


def random_state(geom, seed, scale=1e-3):
    nx, ny, nz = geom.dims
    rng = np.random.default_rng(seed)
    f = scale * (2.0 * rng.random((19, nz, ny, nx)) - 1.0)
    f[:, ~fluid_mask(geom)] = 0.0
    return f


def pair(pg, orc, geom, nu=0.1, lam=3.0 / 16.0, g=(1e-6, 0.0, 0.0), scheme=0, rho0=1.0):
    p = pg.relaxation_from_magic(nu, lam)
    p.body_force = tuple(g)
    p.rho0 = rho0
    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme, rho0)
    return sim, o


def compare_all(sim, o, geom, what):
    m = fluid_mask(geom)
    assert_bitwise(sim.get_pdfs(), o.get_pdfs(), m, what + " pdfs")
    d, ux, uy, uz = sim.macroscopic_fields()
    od, oux, ouy, ouz = o.macroscopic_fields()
    for a, b, n in ((d, od, "drho"), (ux, oux, "ux"), (uy, ouy, "uy"), (uz, ouz, "uz")):
        assert_bitwise(a, b, m, f"{what} {n}")
    pa, pb = sim.planar_profile(), o.planar_profile()
    assert np.array_equal(pa.u_superficial, pb["u_superficial"]), what + " profile"
    assert np.array_equal(pa.u_intrinsic, pb["u_intrinsic"]), what + " profile intrinsic"
    assert np.array_equal(pa.z, pb["z"])
    assert pa.u_max == pb["u_max"]
    ms, oms = sim.max_speed(), o.max_speed()
    assert ms == oms or (np.isnan(ms) and np.isnan(oms)), (ms, oms)


def sphere_geometry(pg, dims=(40, 24, 32), n=9, seed=7, walls=True, periodic=(True, True, False)):
    rng = np.random.default_rng(seed)
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n),
              rng.uniform(1, dims[2] * 0.6, n)]
    r = rng.uniform(2.5, 5.5, n)
    pack = pg.SpherePack(c, r, tuple(float(d) for d in dims))
    return pg.voxelize(pack, dims, periodic, walls, walls)


# --- test_simulation.cpp:84-140: one full step vs collide + gather + bounce ----
def test_full_step_kat_4x4x6(gpu, orc):
    pg = gpu
    geom = pg.make_box_geometry((4, 4, 6), (True, True, False), True, True)
    sim, o = pair(pg, orc, geom, 0.1, 3.0 / 16.0, (1e-6, 2e-7, 0.0))
    f0 = random_state(geom, 23)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    sim.step(1)
    o.step(1)
    compare_all(sim, o, geom, "kat")
    # the reference test's own oracle: trt_collide per cell, push, SBB closure
    p = sim.params
    m = fluid_mask(geom)
    post = np.zeros_like(f0)
    for z, y, x in zip(*np.nonzero(m)):
        post[:, z, y, x] = pg.trt_collide(f0[:, z, y, x], p)
    exp = np.zeros_like(f0)
    E, OPP = pg.VELOCITIES, pg.OPPOSITE
    for z, y, x in zip(*np.nonzero(m)):
        for k in range(19):
            xn, yn, zn = (x + E[k, 0]) % 4, (y + E[k, 1]) % 4, z + E[k, 2]
            if 0 <= zn < 6 and m[zn, yn, xn]:
                exp[k, zn, yn, xn] = post[k, z, y, x]
            else:
                exp[OPP[k], z, y, x] = post[k, z, y, x]
    got = sim.get_pdfs()
    # doctest Approx(x).epsilon(1e-14): |a - b| <= 1e-14 * (1 + max(|a|, |b|))
    a, b = got[:, m], exp[:, m]
    assert np.all(np.abs(a - b) <= 1e-14 * (1.0 + np.maximum(np.abs(a), np.abs(b))))


@pytest.mark.parametrize("scheme", [0, 1])
def test_sphere_bed_random_state(gpu, orc, scheme):
    pg = gpu
    geom = sphere_geometry(pg)
    sim, o = pair(pg, orc, geom, 0.05, 3.0 / 16.0, (2e-6, -1e-6, 5e-7), scheme)
    f0 = random_state(geom, 11 + scheme)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    for n in (1, 3, 20):  # K0, K1 singles, then the graph path (>= 16)
        sim.step(n)
        o.step(n)
        compare_all(sim, o, geom, f"scheme{scheme} after {o.steps_done}")
    assert sim.steps_done == o.steps_done == 24
    if scheme == 1:
        assert sim.cli_fallback_count == int((geom.link_second_fluid < 0).sum())


def test_periodic_box_all_fluid(gpu, orc):
    pg = gpu
    geom = pg.make_box_geometry((8, 6, 5), (True, True, True))
    assert geom.n_links == 0
    sim, o = pair(pg, orc, geom, 1.0 / 6.0, 0.25, (1e-7, 0.0, 0.0))
    f0 = random_state(geom, 77, 1e-4)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    sim.step(5)
    o.step(5)
    compare_all(sim, o, geom, "periodic")


def test_rho0_not_one(gpu, orc):
    pg = gpu
    geom = sphere_geometry(pg, dims=(24, 16, 20), n=4, seed=3)
    for scheme in (0, 1):
        sim, o = pair(pg, orc, geom, 0.1, 3.0 / 16.0, (1e-6, 0, 0), scheme, rho0=1.3)
        f0 = random_state(geom, 5)
        sim.set_pdfs(f0)
        o.set_pdfs(f0)
        sim.step(18)
        o.step(18)
        compare_all(sim, o, geom, f"rho0 scheme{scheme}")


def test_moving_lid(gpu, orc):
    pg = gpu
    geom = pg.make_box_geometry((8, 8, 12), (True, True, False), True, True)
    sim, o = pair(pg, orc, geom, 1.0 / 6.0, 3.0 / 16.0, (0, 0, 0), 1)
    sim.set_lid_velocity((0.01, 0.002, 0.0))
    o.set_lid_velocity((0.01, 0.002, 0.0))
    sim.step(30)
    o.step(30)
    compare_all(sim, o, geom, "lid")


@pytest.mark.parametrize("scheme", [0, 1])
def test_lid_set_mid_run(gpu, orc, scheme):
    """simulation.cpp:104-112 between steps: step n's streaming and bounce-back
    already happened with the old wall velocity (the device materialises f(n)
    before switching).  Spheres touch the lid so CLI links turn moving."""
    pg = gpu
    dims = (24, 16, 20)
    c = np.array([[6.0, 5.0, 17.5], [15.0, 11.0, 18.2], [12.0, 8.0, 5.0]])
    pack = pg.SpherePack(c, np.array([2.6, 2.2, 3.5]), tuple(float(d) for d in dims))
    geom = pg.voxelize(pack, dims, (True, True, False), True, True)
    sim, o = pair(pg, orc, geom, 1.0 / 6.0, 3.0 / 16.0, (1e-6, 0, 0), scheme)
    sim.step(7)
    o.step(7)
    sim.set_lid_velocity((0.01, 0.002, 0.0))
    o.set_lid_velocity((0.01, 0.002, 0.0))
    sim.step(20)
    o.step(20)
    compare_all(sim, o, geom, "lid mid-run")
    sim.set_lid_velocity((-0.004, 0.0, 0.001))
    o.set_lid_velocity((-0.004, 0.0, 0.001))
    sim.step(17)
    o.step(17)
    compare_all(sim, o, geom, "lid changed")


@pytest.mark.parametrize("cf,eps_in_eq", [(0.0, True), (0.0, False), (0.3, True)])
def test_glbm(gpu, orc, cf, eps_in_eq):
    pg = gpu
    nz = 24
    geom = pg.make_box_geometry((8, 4, nz), (True, True, False), True, True)
    zc = np.arange(nz) + 0.5
    eps = np.where(zc >= 12, 1.0, np.where(zc <= 8, 0.5, 0.5 + 0.5 * (zc - 8) / 4))
    eps[0] = eps[-1] = 1.0
    K = pg.kozeny_carman(eps, 4.0)
    gp = pg.make_glbm_params(eps, K, cf, 1.0 / 6.0, 3.0 / 16.0, pg.GlbmViscosity.Rescaled)
    gp.eps_in_equilibrium = eps_in_eq
    sim, o = pair(pg, orc, geom, 1.0 / 6.0, 3.0 / 16.0, (1e-5, 0, 0), 0)
    sim.set_porous(gp)
    o.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, cf, eps_in_eq)
    f0 = random_state(geom, 9, 1e-4)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    sim.step(25)
    o.step(25)
    compare_all(sim, o, geom, f"glbm cf={cf}")


def test_glbm_free_is_core(gpu):
    """test_simulation.cpp:295-324: free GLBM parameters step bitwise like core."""
    pg = gpu
    geom = pg.make_box_geometry((6, 6, 6), (True, True, True))
    p = pg.relaxation_from_magic(1.0 / 6.0, 0.25)
    p.body_force = (1e-7, 0, 0)
    a = pg.Simulation.from_params(geom, p, pg.WallScheme.SBB)
    b = pg.Simulation.from_params(geom, p, pg.WallScheme.SBB)
    b.set_porous(pg.make_glbm_params(np.ones(6), np.full(6, np.inf), 0.0, p.nu, 0.25,
                                     pg.GlbmViscosity.Plain))
    f0 = random_state(geom, 77, 1e-4)
    a.set_pdfs(f0)
    b.set_pdfs(f0)
    a.step(5)
    b.step(5)
    assert np.array_equal(a.get_pdfs(), b.get_pdfs())


def test_state_machine_interleaving(gpu, orc):
    pg = gpu
    geom = sphere_geometry(pg, dims=(32, 16, 24), n=5, seed=4)
    sim, o = pair(pg, orc, geom, 0.08, 3.0 / 16.0, (3e-6, 0, 0), 1)
    sim.step(3)
    o.step(3)
    compare_all(sim, o, geom, "a")
    c = int(np.nonzero(geom.flags == 0)[0][100])
    newf = np.linspace(-1e-4, 1e-4, 19)
    sim.set_cell_populations(c, newf)
    f = o.get_pdfs()
    f.reshape(19, -1)[:, c] = newf
    o.set_pdfs(f)
    assert np.array_equal(sim.cell_populations(c), newf)
    sim.step(17)
    o.step(17)
    compare_all(sim, o, geom, "b")
    d, u = sim.macroscopic(c)
    od, ou = o.macroscopic_fields()[0].reshape(-1)[c], [x.reshape(-1)[c] for x in o.macroscopic_fields()[1:]]
    assert d == od and np.array_equal(u, np.array(ou))
    sim.initialize_equilibrium(0.01, (0.001, 0.0, -0.002))
    feq = pg.equilibrium(0.01, (0.001, 0.0, -0.002))
    f = o.get_pdfs()
    f[:, fluid_mask(geom)] = feq[:, None]
    o.set_pdfs(f)
    sim.step(2)
    o.step(2)
    compare_all(sim, o, geom, "c")


@pytest.mark.parametrize("persistent", ["1", "0"])
@pytest.mark.parametrize("scheme", [0, 1])
def test_multistep_paths_equal_single_steps(gpu, orc, monkeypatch, persistent, scheme, layout):
    """step(n) uses the persistent cooperative kernel (L2-resident domains) or
    CUDA graphs of K1 launches; both must equal n single steps and the oracle."""
    pg = gpu
    monkeypatch.setenv("PGPU_PERSISTENT", persistent)
    geom = sphere_geometry(pg, dims=(32, 16, 24), n=5, seed=8)
    p = pg.relaxation_from_magic(0.1, 3.0 / 16.0)
    p.body_force = (1e-6, 0, 0)
    a = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    b = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    a.step(51)
    for _ in range(51):
        b.step(1)
    assert np.array_equal(a.get_pdfs(), b.get_pdfs())
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
    o.step(51)
    fl = fluid_mask(geom)
    assert np.array_equal(a.get_pdfs()[:, fl], o.get_pdfs()[:, fl])
    if persistent == "1" and layout == "dense":
        assert a.launch_count < 10  # one cooperative launch for the 50 K1 steps


def test_nonfinite_guard(gpu):
    pg = gpu
    geom = pg.make_box_geometry((6, 6, 6), (True, True, True))
    sim = pg.Simulation(geom, 1.0 / 6.0, 3.0 / 16.0, (0, 0, 0), pg.WallScheme.SBB)
    f = np.zeros((19, 6, 6, 6))
    f[3, 2, 2, 2] = np.inf
    sim.set_pdfs(f)
    assert np.isnan(sim.max_speed())


def test_instability_guard_trips(gpu):
    """test_simulation.cpp:220-230."""
    pg = gpu
    geom = pg.make_box_geometry((6, 6, 6), (True, True, True))
    sim = pg.Simulation(geom, 1.0 / 6.0, 3.0 / 16.0, (0.05, 0, 0), pg.WallScheme.SBB)
    with pytest.raises(pg.NumericalInstability):
        pg.run_to_steady(sim, 1e-8, 200, 100000)


def test_run_to_steady_matches_reference(gpu, ref):
    pg = gpu
    geom = pg.make_box_geometry((4, 4, 18), (True, True, False), True, True)
    sim = pg.Simulation(geom, 1.0 / 6.0, 3.0 / 16.0, (1e-8, 0, 0), pg.WallScheme.SBB)
    st, prof = pg.run_to_steady(sim, 1e-12, 500, 20000)
    wp, wm = ref.relaxation_from_magic(1.0 / 6.0, 3.0 / 16.0)
    r = ref.simulation(geom, 1.0 / 6.0, wp, wm, 3.0 / 16.0, (1e-8, 0, 0), 0)
    rst = r.run_to_steady_state(1e-12, 500, 20000)
    assert st.steps == rst["steps"] and st.converged == rst["converged"]
    assert st.residual == rst["residual"]
    rp = r.planar_profile()
    assert np.array_equal(prof.u_superficial, rp["u_superficial"])
    # symmetric channel (test_simulation.cpp:198-218)
    n = prof.u_superficial.size
    np.testing.assert_allclose(prof.u_superficial, prof.u_superficial[::-1], rtol=1e-12)


def test_inconsistent_links_rejected(gpu):
    pg = gpu
    geom = pg.make_box_geometry((4, 4, 6), (True, True, False), True, True)
    bad = pg.VoxelGeometry(**{**geom.__dict__})
    bad.link_fluid_cell = geom.link_fluid_cell[1:]
    bad.link_second_fluid = geom.link_second_fluid[1:]
    bad.link_direction = geom.link_direction[1:]
    bad.link_q = geom.link_q[1:]
    bad.link_moving = geom.link_moving[1:]
    with pytest.raises(pg.ConfigError):
        pg.Simulation(bad, 0.1, 3.0 / 16.0, (0, 0, 0), pg.WallScheme.SBB)


@pytest.mark.parametrize("periodic", [(1, 1, 1), (1, 0, 1), (0, 1, 0)])
def test_free_stream_matches_reference(gpu, ref, periodic):
    """Free stream() (simulation.cpp:436-439) on a sphere bed with random
    populations in both buffers (slots the pass does not write keep `next`),
    and test_simulation.cpp:26-42's periodic advection."""
    pg = gpu
    rng = np.random.default_rng(3)
    flags = np.where(rng.random(16 * 12 * 20) < 0.2, 1, 0).astype(np.uint8)
    cur = rng.standard_normal((19, 16, 12, 20))
    nxt = rng.standard_normal((19, 16, 12, 20))
    a, b = cur.copy(), nxt.copy()
    pg.stream(a, b, flags, periodic)
    c, d = cur.copy(), nxt.copy()
    ref.stream(c, d, flags, periodic)
    assert np.array_equal(a, c) and np.array_equal(b, d)
    # periodic advection: a lone population moves one cell per call
    if all(periodic):
        box = pg.make_box_geometry((5, 4, 3), (True, True, True))
        f = np.zeros((19, 3, 4, 5))
        f[7, 1, 2, 4] = 1.0  # e_7 = (1, 1, 0)
        g = np.zeros_like(f)
        pg.stream(f, g, box.flags, (1, 1, 1))
        assert f[7, 1, 3, 0] == 1.0 and f.sum() == 1.0
