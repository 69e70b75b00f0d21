"""Device voxelizer against the host voxelizer, which
tests/test_voxelize.py pins byte-for-byte to the reference voxelize()."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def same(a, b):
    assert a.dims == b.dims
    assert a.flags.tobytes() == b.flags.tobytes()
    assert np.asarray(a.porosity).tobytes() == np.asarray(b.porosity).tobytes()
    assert a.fluid_cells == b.fluid_cells and a.q_fallback_count == b.q_fallback_count
    for f in ("link_fluid_cell", "link_second_fluid", "link_direction"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.link_q.tobytes() == b.link_q.tobytes()
    assert (a.wall_plane_lo, a.wall_plane_hi) == (b.wall_plane_lo, b.wall_plane_hi)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_beds(gpu, seed):
    pg = gpu
    rng = np.random.default_rng(seed)
    dims = (40, 28, 36)
    n = 25
    c = np.c_[rng.uniform(-3, 43, n), rng.uniform(-3, 31, n), rng.uniform(0, 30, n)]
    r = rng.uniform(1.5, 7.0, n)
    plate = [0.0, 2.7, -3.0][seed - 1]
    pack = pg.SpherePack(c, r, (40.0, 28.0, 36.0), plate)
    for per, walls, qmin in (((True, True, False), True, 0.05), ((True, True, True), False, 0.1)):
        same(pg.voxelize_device(pack, dims, per, walls, walls, qmin),
             pg.voxelize(pack, dims, per, walls, walls, qmin))


def test_box_and_open_face(gpu):
    pg = gpu
    empty = pg.SpherePack(np.zeros((0, 3)), np.zeros(0), (16.0, 8.0, 12.0))
    same(pg.voxelize_device(empty, (16, 8, 12), (True, True, False), True, True),
         pg.make_box_geometry((16, 8, 12), (True, True, False), True, True))
    with pytest.raises(pg.ConfigError):
        pg.voxelize_device(empty, (8, 8, 8), (True, True, False))


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_config_geometries(gpu, name):
    pg = gpu
    from paper_1507_06565_b200 import configs
    w = configs.ALL[name]()
    o = w.voxelize_options()
    same(pg.voxelize_device(w.pack, w.dims, **o), w.geometry())
