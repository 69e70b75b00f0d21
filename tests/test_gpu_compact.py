"""The fluid-only ("compact") PDF layout (sweep_compact.cu) on its corner
cases, bit for bit against the oracle: rows whose length is not a multiple of
the 32-cell chunk (the last chunk partial, or a single chunk holding both x
faces), a fully periodic box (source rows wrapping in z), and a link density
that overflows the per-warp CLI pool (the direct-load fallback).  The
SBB/CLI/lid/GLBM/slab paths in both layouts are covered by the `layout`
parametrisation of test_gpu_parity.py, test_gpu_dist.py and
test_gpu_drivers.py."""
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


def max_links_per_chunk_plane(geom):
    nx = geom.dims[0]
    cell = np.asarray(geom.link_fluid_cell)
    key = (cell // nx) * ((nx + 31) // 32) + (cell % nx) // 32
    return int(np.bincount(key).max()) if key.size else 0


def run_and_compare(pg, orc, geom, scheme, steps, seed=11):
    p = pg.relaxation_from_magic(0.08, 3.0 / 16.0)
    p.body_force = (2e-6, 1e-6, -5e-7)
    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
    nx, ny, nz = geom.dims
    m = fluid_mask(geom)
    rng = np.random.default_rng(seed)
    f0 = 1e-3 * (2.0 * rng.random((19, nz, ny, nx)) - 1.0)
    f0[:, ~m] = 0.0
    sim.set_pdfs(f0)
    o.set_pdfs(f0)
    for n in steps:  # observables between step batches exercise KP / K0 re-entry
        sim.step(n)
        o.step(n)
        got, want = sim.get_pdfs(), o.get_pdfs()
        assert np.array_equal(got[:, m], want[:, m]), f"pdfs differ after {n} steps"
    d, ux, uy, uz = sim.macroscopic_fields()
    od, oux, ouy, ouz = o.macroscopic_fields()
    mf = m.reshape(-1)
    for a, b in ((d, od), (ux, oux), (uy, ouy), (uz, ouz)):
        assert np.array_equal(np.ravel(a)[mf], np.ravel(b)[mf])
    return sim


CASES = {
    # name: dims, n spheres, r range, periodic, walls
    "nx45_partial_chunk": ((45, 20, 24), 10, 2.0, 4.5, (True, True, False), True),
    "nx20_one_chunk": ((20, 18, 22), 6, 2.0, 4.0, (True, True, False), True),
    "nx33_one_cell_chunk": ((33, 16, 20), 6, 2.0, 4.0, (True, True, False), True),
    "fully_periodic": ((64, 24, 28), 14, 2.0, 5.0, (True, True, True), False),
}


@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("case", sorted(CASES))
def test_compact_corner_cases(gpu, orc, monkeypatch, case, scheme):
    monkeypatch.setenv("PGPU_LAYOUT", "compact")
    dims, n, rmin, rmax, per, walls = CASES[case]
    geom = geometry(gpu, dims, n, rmin, rmax, seed=len(case), periodic=per, walls=walls)
    assert geom.n_links > 0
    run_and_compare(gpu, orc, geom, scheme, steps=(1, 2, 17))


@pytest.mark.parametrize("scheme", [0, 1])
def test_compact_link_pool_overflow(gpu, orc, monkeypatch, scheme):
    """Hundreds of small spheres: chunk-planes with more CLI links than the
    per-warp pool holds (96) close the rest with direct loads."""
    monkeypatch.setenv("PGPU_LAYOUT", "compact")
    geom = geometry(gpu, (64, 32, 32), 900, 0.6, 1.3, seed=3)
    assert max_links_per_chunk_plane(geom) > 96
    run_and_compare(gpu, orc, geom, scheme, steps=(1, 6))


def test_compact_equals_dense_larger_domain(gpu, monkeypatch):
    """A non-L2-resident domain (the default layout choice is compact): both
    layouts, graph-replayed multi-step runs, identical on every fluid slot."""
    geom = geometry(gpu, (96, 64, 48), 40, 2.5, 6.0, seed=21)
    p = gpu.relaxation_from_magic(0.1, 3.0 / 16.0)
    p.body_force = (1e-6, 0.0, 0.0)
    out = {}
    for layout in ("dense", "compact"):
        monkeypatch.setenv("PGPU_LAYOUT", layout)
        monkeypatch.setenv("PGPU_PERSISTENT", "0")
        sim = gpu.Simulation.from_params(geom, p, gpu.WallScheme.CLI)
        sim.step(40)
        out[layout] = sim.get_pdfs()
    m = fluid_mask(geom)
    assert np.array_equal(out["dense"][:, m], out["compact"][:, m])


def test_compact_plain_per_cell_sweep(gpu, orc, tmp_path):
    """PGPU_SWEEP=plain (read once at library load, hence a subprocess): the
    per-cell compact sweep -- the reference point of the pipelined kernel and
    the slab edge path for narrow bands -- against the oracle, SBB and CLI."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    script = f"""
import sys, numpy as np
sys.path.insert(0, {str(root)!r})
sys.path.insert(0, {str(Path(__file__).resolve().parent)!r})
import paper_1507_06565_b200 as pg
from test_gpu_compact import geometry
geom = geometry(pg, (45, 20, 24), 10, 2.0, 4.5, seed=5)
p = pg.relaxation_from_magic(0.08, 3.0 / 16.0)
p.body_force = (2e-6, 1e-6, -5e-7)
for scheme in (0, 1):
    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    sim.step(9)
    np.save({str(tmp_path)!r} + f"/plain_{{scheme}}.npy", sim.get_pdfs())
"""
    env = dict(os.environ, PGPU_SWEEP="plain", PGPU_LAYOUT="compact")
    res = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    geom = geometry(gpu, (45, 20, 24), 10, 2.0, 4.5, seed=5)
    m = fluid_mask(geom)
    p = gpu.relaxation_from_magic(0.08, 3.0 / 16.0)
    p.body_force = (2e-6, 1e-6, -5e-7)
    for scheme in (0, 1):
        o = orc.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.body_force, scheme)
        o.step(9)
        got = np.load(tmp_path / f"plain_{scheme}.npy")
        assert np.array_equal(got[:, m], o.get_pdfs()[:, m])


def test_fluid_only_footprint_has_no_dense_state(gpu, monkeypatch):
    """The fluid-only layout keeps no dense copy of the populations: the
    pre-collision state lives in the compact buffers and population I/O
    stages through the dead one (C4: 16.5 GB instead of 26.7 GB)."""
    pg = gpu
    monkeypatch.setenv("PGPU_LAYOUT", "compact")
    geom = geometry(pg, (96, 64, 80), 40, 3.0, 6.0, 5)
    sim = pg.Simulation(geom, 0.08, 3.0 / 16.0, (1e-6, 0, 0), pg.WallScheme.CLI)
    assert sim.layout == "fluid-only"
    fluid, cells, links = geom.fluid_cells, geom.cells, geom.n_links
    sweep = 2 * 19 * 8 * ((fluid + 31) // 32 * 32)
    b = sim.device_bytes
    assert sweep < b < sweep + 12 * cells + 20 * links + (1 << 20), (b, sweep)
    # observables and population I/O work without it (and leave it that way)
    sim.step(5)
    f = sim.get_pdfs()
    sim.set_pdfs(f)
    sim.step(3)
    sim.planar_profile()
    assert sim.device_bytes <= b


def test_more_than_113m_fluid_cells_stay_fluid_only(gpu, monkeypatch):
    """A 512x512x460 walled box (120 M fluid cells: 19 planes need unsigned
    32-bit slot offsets) runs in the fluid-only layout and steps bit for bit
    like the dense layout (profile, single-cell populations, max speed)."""
    pg = gpu
    geom = pg.make_box_geometry((512, 512, 460), (True, True, False), True, True)
    assert geom.fluid_cells > 113_000_000
    runs = {}
    for layout in ("compact", "dense"):
        monkeypatch.setenv("PGPU_LAYOUT", layout)
        sim = pg.Simulation(geom, 0.1, 3.0 / 16.0, (1e-6, 2e-7, 0), pg.WallScheme.SBB)
        assert sim.layout == ("fluid-only" if layout == "compact" else "dense")
        sim.step(6)
        cells = [512 * 512 * 1 + 7, 512 * 512 * 230 + 300 * 512 + 11, 512 * 512 * 458 + 511]
        runs[layout] = (sim.planar_profile().u_superficial, [sim.cell_populations(c) for c in cells],
                        sim.max_speed())
        del sim
    a, b = runs["compact"], runs["dense"]
    assert np.array_equal(a[0], b[0]) and a[2] == b[2]
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
