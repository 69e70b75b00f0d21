"""The units sweep (sweep_units.cu, pgpu_sweep_kernel UNITS: warps sweep runs of
up to 32 consecutive fluid slots instead of 32-cell chunks) bit for bit:
against the oracle in math mode EXACT (reference arithmetic) and against the
chunk sweep (k_sweep_cpipe) in math mode FAST, on the corner cases of its
addressing -- rows whose last chunk is partial (nx = 160, 36, 20), units that
hold both x faces, x-periodic wrap pulls, a fully periodic box, wall planes
whose units fill the link pool (5 links per cell; cells next to a wall and a
sphere end units early), CLI beds (units spanning three chunks), a moving lid (+inf records), the GLBM collision, and several
units-per-warp settings (pipeline lengths 1, 2, 3 and longer)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fluid_mask(geom):
    nx, ny, nz = geom.dims
    return geom.flags.reshape(nz, ny, nx) == 0


def geometry(pg, dims, n, rmin, rmax, seed, periodic=(True, True, False), walls=True):
    rng = np.random.default_rng(seed)
    zlo, zhi = (1.0, dims[2] - 1.0) if walls else (0.0, float(dims[2]))
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n), rng.uniform(zlo, zhi, n)]
    r = rng.uniform(rmin, rmax, n)
    pack = pg.SpherePack(c, r, tuple(float(d) for d in dims))
    return pg.voxelize(pack, dims, periodic, walls, walls)

CASES = {
    # name: dims, n spheres, r range, periodic, walls
    "nx160_partial_segment": ((160, 20, 24), 14, 2.0, 5.0, (True, True, False), True),
    "nx36_short_row": ((36, 18, 22), 6, 2.0, 4.0, (True, True, False), True),
    "nx20_one_chunk": ((20, 18, 22), 6, 2.0, 4.0, (True, True, False), True),
    "fully_periodic": ((64, 24, 28), 14, 2.0, 5.0, (True, True, True), False),
    "bed_128": ((128, 32, 40), 40, 3.0, 6.0, (True, True, False), True),
}


def _params(pg):
    p = pg.relaxation_from_magic(0.08, 3.0 / 16.0)
    p.body_force = (2e-6, 1e-6, -5e-7)
    return p


def _random_state(geom, seed):
    nx, ny, nz = geom.dims
    m = fluid_mask(geom)
    rng = np.random.default_rng(seed)
    f0 = 1e-3 * (2.0 * rng.random((19, nz, ny, nx)) - 1.0)
    f0[:, ~m] = 0.0
    return f0, m


def _units_sim(pg, monkeypatch, geom, p, scheme):
    monkeypatch.setenv("PGPU_LAYOUT", "compact")
    monkeypatch.setenv("PGPU_SWEEP", "units")
    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    assert sim.layout == "fluid-only"
    assert sim.sweep_kernel == "units", "the units sweep does not run for this simulation"
    return sim


@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("case", sorted(CASES))
def test_units_exact_vs_oracle(gpu, orc, monkeypatch, case, scheme):
    dims, n, rmin, rmax, per, walls = CASES[case]
    geom = geometry(gpu, dims, n, rmin, rmax, seed=len(case) + 3, periodic=per, walls=walls)
    assert geom.n_links > 0
    p = _params(gpu)
    sim = _units_sim(gpu, monkeypatch, geom, p, scheme)
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
    f0, m = _random_state(geom, 5)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    for k in (1, 2, 17, 20):  # 20: one graph replay of 16 K1 launches
        sim.step(k)
        o.step(k)
        got, want = sim.get_pdfs(), o.get_pdfs()
        assert np.array_equal(got[:, m], want[:, m]), f"pdfs differ after {k} more steps"
    d, ux, uy, uz = sim.macroscopic_fields()
    od, oux, ouy, ouz = o.macroscopic_fields()
    mf = m.reshape(-1)
    for a, b in ((d, od), (ux, oux), (uy, ouy), (uz, ouz)):
        assert np.array_equal(np.ravel(a)[mf], np.ravel(b)[mf])


def test_units_wall_planes_overflow_pool(gpu, orc, monkeypatch):
    """An all-fluid walled channel: every cell of the planes next to the walls
    has 5 links, 160 per full unit -- exactly the link pool (kUnitLinkCap)."""
    geom = gpu.make_box_geometry((128, 8, 12), (True, True, False), True, True)
    for scheme in (0, 1):
        p = _params(gpu)
        sim = _units_sim(gpu, monkeypatch, geom, p, scheme)
        o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
        f0, m = _random_state(geom, 9)
        sim.set_pdfs(f0)
        o.set_pdfs(f0)
        sim.step(7)
        o.step(7)
        assert np.array_equal(sim.get_pdfs()[:, m], o.get_pdfs()[:, m])


def test_units_moving_lid(gpu, orc, monkeypatch):
    dims = (128, 16, 20)
    geom = geometry(gpu, dims, 10, 2.0, 4.0, seed=21)
    p = _params(gpu)
    for scheme in (0, 1):
        sim = _units_sim(gpu, monkeypatch, geom, p, scheme)
        o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
        f0, m = _random_state(geom, 3)
        sim.set_pdfs(f0)
        o.set_pdfs(f0)
        sim.set_lid_velocity((0.01, -0.004, 0.0))
        o.set_lid_velocity((0.01, -0.004, 0.0))
        sim.step(19)
        o.step(19)
        assert np.array_equal(sim.get_pdfs()[:, m], o.get_pdfs()[:, m])


@pytest.mark.parametrize("scheme", [0, 1])
def test_units_fast_equals_cpipe_fast(gpu, monkeypatch, scheme):
    """Math mode FAST: the two K1 kernels share the collision, so they agree
    bit for bit (and FAST itself is checked against the reference in
    test_gpu_fast.py)."""
    dims = (128, 32, 40)
    geom = geometry(gpu, dims, 40, 3.0, 6.0, seed=4)
    p = _params(gpu)
    sim = _units_sim(gpu, monkeypatch, geom, p, scheme)
    sim.math_mode = gpu.MathMode.FAST
    monkeypatch.setenv("PGPU_SWEEP", "cpipe")
    ref = gpu.Simulation.from_params(geom, p, gpu.WallScheme(scheme))
    ref.math_mode = gpu.MathMode.FAST
    assert ref.sweep_kernel == "cpipe"
    f0, m = _random_state(geom, 7)
    sim.set_pdfs(f0)
    ref.set_pdfs(f0)
    sim.step(37)
    ref.step(37)
    assert np.array_equal(sim.get_pdfs()[:, m], ref.get_pdfs()[:, m])
    # switching the kernel mid-run keeps the trajectory
    sim.sweep_kernel = "cpipe"
    ref.sweep_kernel = "units"
    sim.step(5)
    ref.step(5)
    assert np.array_equal(sim.get_pdfs()[:, m], ref.get_pdfs()[:, m])


@pytest.mark.parametrize("upw,group", [(1, 1), (2, 1), (3, 2), (5, 3), (64, 1), (4, 8)])
def test_units_per_warp_settings(gpu, monkeypatch, upw, group):
    """Pipeline lengths: 1, 2, 3 units per warp (the prologue's partial cases),
    5 and 64 (steady state) and groups of blocks sharing a run of units -- all
    bit-identical to the chunk sweep."""
    dims = (96, 20, 26)
    geom = geometry(gpu, dims, 16, 2.0, 5.0, seed=11)
    p = _params(gpu)
    monkeypatch.setenv("PGPU_UPW", str(upw))
    monkeypatch.setenv("PGPU_UGROUP", str(group))
    sim = _units_sim(gpu, monkeypatch, geom, p, 1)
    monkeypatch.setenv("PGPU_SWEEP", "cpipe")
    ref = gpu.Simulation.from_params(geom, p, gpu.WallScheme(1))
    f0, m = _random_state(geom, 17)
    sim.set_pdfs(f0)
    ref.set_pdfs(f0)
    sim.step(19)
    ref.step(19)
    assert np.array_equal(sim.get_pdfs()[:, m], ref.get_pdfs()[:, m])
    sim.step(40)  # graph replays
    ref.step(40)
    assert np.array_equal(sim.get_pdfs()[:, m], ref.get_pdfs()[:, m])


def test_units_glbm_fluid_only(gpu, orc, monkeypatch):
    """The GLBM collision (per-plane coefficients by z) on the UNITS sweep."""
    dims = (128, 12, 24)
    geom = geometry(gpu, dims, 8, 2.0, 4.0, seed=33)
    p = _params(gpu)
    sim = _units_sim(gpu, monkeypatch, geom, p, 1)
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, 1)
    nz = dims[2]
    z = np.arange(nz)
    eps = np.where(z < nz // 2, 0.6, 1.0) - 0.01 * (z % 3)
    K = gpu.kozeny_carman(eps, 10.0)
    gp = gpu.make_glbm_params(eps, K, 0.3, p.nu, 3.0 / 16.0, gpu.GlbmViscosity.Rescaled)
    sim.set_porous(gp)
    o.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, 0.3, True)
    f0, m = _random_state(geom, 13)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    sim.step(21)
    o.step(21)
    assert np.array_equal(sim.get_pdfs()[:, m], o.get_pdfs()[:, m])


@pytest.mark.parametrize("nx,world", [(256, 2), (200, 2), (96, 3)])
@pytest.mark.parametrize("scheme", [0, 1])
def test_units_slab_interior(gpu, monkeypatch, nx, world, scheme):
    """x-slab split: the units cover the interior columns of each slab (the
    edge bands -- 32 columns, or the face columns of slabs narrower than 96 --
    stay on the chunk sweep, which alone reads ghosts and fills the send
    buffers).  Slabs of 128, 100 and 32 columns against the single domain on
    the chunk sweep, bit for bit."""
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import LocalTransport
    from test_gpu_dist import bed_workload
    monkeypatch.setenv("PGPU_LAYOUT", "compact")
    monkeypatch.setenv("PGPU_SWEEP", "units")
    w = bed_workload(gpu, scheme, nx=nx)
    lt = LocalTransport(w, world, device=0)
    assert all(r.sim.sweep_kernel == "units" for r in lt.ranks), "the slabs do not run the units sweep"
    lt.step(w.steps)
    monkeypatch.setenv("PGPU_SWEEP", "cpipe")
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    assert sim.sweep_kernel == "cpipe"
    sim.step(w.steps)
    fl = g.flags.reshape(w.dims[::-1]) == 0
    assert np.array_equal(lt.gather_pdfs()[:, fl], sim.get_pdfs()[:, fl])


@pytest.mark.parametrize("seed", range(12))
def test_units_random_domains(gpu, orc, monkeypatch, seed):
    """Random box sizes (x extents around the chunk and unit boundaries: 3..140),
    z periodic or walled, sphere packs and schemes: the units sweep
    against the oracle, bit for bit, over single steps and a graph replay."""
    rng = np.random.default_rng(1000 + seed)
    nx = int(rng.choice([3, 5, 31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 129, 140]))
    ny, nz = int(rng.integers(3, 14)), int(rng.integers(6, 18))
    pz = bool(rng.integers(2))  # x and y periodic as in every config; z periodic or walled
    walls = not pz
    per = (True, True, pz)
    n = int(rng.integers(1, 10))
    geom = geometry(gpu, (nx, ny, nz), n, 1.5, 4.0, seed=seed, periodic=per, walls=walls)
    scheme = int(rng.integers(2))
    p = _params(gpu)
    sim = _units_sim(gpu, monkeypatch, geom, p, scheme)
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
    f0, m = _random_state(geom, seed)
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    for k in (1, 2, 18):
        sim.step(k)
        o.step(k)
        assert np.array_equal(sim.get_pdfs()[:, m], o.get_pdfs()[:, m]), \
            f"dims {(nx, ny, nz)} periodic {per} walls {walls} scheme {scheme}: differ after {k} more steps"
