"""The x-slab (multi-GPU) kernels on ONE B200: P slabs of a domain run in one
process through dist.LocalTransport (edge part, device-copy halo exchange,
interior part -- sequentially, so no kernel waits on another).  The gathered
populations must equal the single-domain GPU run and the oracle bit for bit;
this exercises the ghost-column pulls, the 5-PDF send buffers, the
double-buffered ghosts and the CLI second-fluid-in-ghost case."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["dense", "compact"], autouse=True)
def layout(request, monkeypatch):
    """Every test here runs on both PDF layouts (PGPU_LAYOUT is read at
    pgpu_create): the dense reference layout and the fluid-only one."""
    monkeypatch.setenv("PGPU_LAYOUT", request.param)
    return request.param


def bed_workload(pg, scheme, nx=128, glbm=False):
    from paper_1507_06565_b200 import configs
    rng = np.random.default_rng(5)
    dims = (nx, 24, 32)
    n = 30
    c = np.c_[rng.uniform(0, nx, n), rng.uniform(0, 24, n), rng.uniform(1, 16, n)]
    r = rng.uniform(2.0, 5.0, n)
    pack = pg.SpherePack(c, r, (float(nx), 24.0, 32.0))
    w = configs.Workload("slab_test", dims, pg.WallScheme(scheme), 0.07, (3e-6, -1e-6, 2e-7), 23,
                         pack=pack)
    if glbm:
        eps = np.clip(np.linspace(0.45, 1.2, 32), 0.45, 1.0)
        eps[0] = eps[-1] = 1.0
        w.glbm = dict(eps=eps, K=pg.kozeny_carman(eps, 6.0))
        w.nu = 1.0 / 6.0
    return w


@pytest.mark.parametrize("nx,world", [(200, 2), (96, 2), (96, 3)])
@pytest.mark.parametrize("scheme", [0, 1])
def test_slabs_not_warp_multiples(gpu, nx, world, scheme):
    """Slab widths that are not multiples of 32 (100: 32-column per-cell edge
    bands + masked interior chunks; 48 and 32: face-column edge bands), the
    native local transport against the single domain, bit for bit, plus the
    global profile (metadata exact, values within 1e-12) and max speed."""
    pg = gpu
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import LocalTransport
    w = bed_workload(pg, scheme, nx=nx)
    lt = LocalTransport(w, world, device=0)
    lt.step(w.steps)
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    sim.step(w.steps)
    fl = g.flags.reshape(w.dims[::-1]) == 0
    assert np.array_equal(lt.gather_pdfs()[:, fl], sim.get_pdfs()[:, fl])
    a, b = lt.planar_profile(), sim.planar_profile()
    assert np.array_equal(a.z, b.z) and np.array_equal(a.epsilon, b.epsilon)
    assert (a.height, a.z0, a.nu, tuple(a.body_force), a.stream_axis) == \
        (b.height, b.z0, b.nu, tuple(b.body_force), b.stream_axis)
    assert np.abs(a.u_superficial - b.u_superficial).max() <= 1e-12 * abs(b.u_max)
    assert lt.max_speed() == sim.max_speed()


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("scheme", [0, 1])
def test_slabs_match_single_domain(gpu, orc, world, scheme):
    pg = gpu
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import LocalTransport
    w = bed_workload(pg, scheme)
    lt = LocalTransport(w, world, device=0)
    lt.step(w.steps)
    got = lt.gather_pdfs()
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    sim.step(w.steps)
    want = sim.get_pdfs()
    fl = g.flags.reshape(w.dims[::-1]) == 0
    assert np.array_equal(got[:, fl], want[:, fl])
    p = w.params()
    o = orc.simulation(g, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
    o.step(w.steps)
    assert np.array_equal(got[:, fl], o.get_pdfs()[:, fl])


def test_slabs_glbm(gpu):
    pg = gpu
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import LocalTransport
    w = bed_workload(pg, 0, glbm=True)
    w.pack = None  # homogenised channel
    lt = LocalTransport(w, 4, device=0)
    lt.step(17)
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    sim.step(17)
    fl = g.flags.reshape(w.dims[::-1]) == 0
    assert np.array_equal(lt.gather_pdfs()[:, fl], sim.get_pdfs()[:, fl])


@pytest.mark.parametrize("scheme", [0, 1])
def test_dist_transport_two_streams_single_rank(gpu, scheme):
    """SlabSimulation at world size 1: the native NCCL driver (edge part +
    exchange on the high-priority stream, interior on the simulation's stream,
    two-step CUDA-graph replays) with the periodic exchange going through
    ncclSend/ncclRecv to self: bit-identical to the single domain, also when
    observables and more steps interleave."""
    pg = gpu
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import SlabSimulation
    w = bed_workload(pg, scheme)
    ss = SlabSimulation(w, 0, 1, device=0)
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    fl = g.flags.reshape(w.dims[::-1]) == 0
    for n in (1, 9, 13):
        ss.step(n)
        sim.step(n)
        got = ss.sim.get_pdfs()
        assert np.array_equal(got[:, fl], sim.get_pdfs()[:, fl]), n
    assert ss.max_speed() == sim.max_speed()
    a, b = ss.planar_profile(), sim.planar_profile()
    assert (a.height, a.z0, a.nu, tuple(a.body_force)) == (b.height, b.z0, b.nu,
                                                           tuple(b.body_force))
    ss.close()


@pytest.mark.parametrize("scheme", [0, 1])
def test_slabs_moving_lid(gpu, scheme, layout):
    """Moving-wall links (lid into the top wall plane) across 2 and 4 slabs:
    the lid records (+inf) and, in the fluid-only layout, the static link
    descriptors are rebuilt per slab after set_lid_velocity; the edge and
    interior parts must reproduce the single-domain run bit for bit."""
    pg = gpu
    from paper_1507_06565_b200 import configs
    from paper_1507_06565_b200.dist import LocalTransport
    w = bed_workload(pg, scheme)
    lid = (3e-3, -1e-3, 0.0)
    g = w.geometry()
    sim = configs.make_simulation(w, g)
    sim.set_lid_velocity(lid)
    sim.step(15)
    want = sim.get_pdfs()
    fl = g.flags.reshape(w.dims[::-1]) == 0
    for world in (2, 4):
        lt = LocalTransport(w, world, device=0)
        for r in lt.ranks:
            r.sim.set_lid_velocity(lid)
        lt.step(15)
        assert np.array_equal(lt.gather_pdfs()[:, fl], want[:, fl]), world
