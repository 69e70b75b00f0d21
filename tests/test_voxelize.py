"""The product's host voxelizer (grid-accelerated, multi-threaded) against the
reference voxelize() (geometry.cpp:491-632): flags, porosity and the link list
(order, second_fluid, direction, fp32 q bits) must be byte-identical.  Also the
x-slab extraction used by the multi-GPU path and the synthetic sphere
generator (CPU only)."""
import numpy as np
import pytest


def same_geometry(a, b):
    assert tuple(a.dims) == tuple(b.dims)
    assert a.flags.tobytes() == b.flags.tobytes()
    assert np.asarray(a.porosity).tobytes() == np.asarray(b.porosity).tobytes()
    assert a.fluid_cells == b.fluid_cells
    assert a.q_fallback_count == b.q_fallback_count
    for f in ("link_fluid_cell", "link_second_fluid", "link_direction"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.asarray(a.link_q, np.float32).tobytes() == np.asarray(b.link_q, np.float32).tobytes()
    assert a.wall_plane_lo == b.wall_plane_lo and a.wall_plane_hi == b.wall_plane_hi


def both(pg, ref, centers, radii, box, dims, periodic, lo, hi, plate=0.0, qmin=0.05):
    r = ref.voxelize(centers, radii, box, dims, periodic, lo, hi, plate, qmin)
    p = pg.voxelize(pg.SpherePack(np.asarray(centers).reshape(-1, 3), radii, box, plate), dims,
                    tuple(bool(x) for x in periodic), lo, hi, qmin)
    same_geometry(p, r)
    return p


def test_empty_pack_all_fluid(pg, ref):
    """test_geometry.cpp:116-125"""
    g = both(pg, ref, np.zeros((0, 3)), np.zeros(0), (8, 8, 8), (8, 8, 8), (1, 1, 1), False, False)
    assert g.fluid_cells == 512 and g.n_links == 0 and np.all(g.porosity == 1.0)


def test_single_sphere_volume_and_q(pg, ref):
    """test_geometry.cpp:127-142"""
    g = both(pg, ref, [[12.5, 12.5, 12.5]], np.array([4.5]), (24, 24, 24), (24, 24, 24),
             (1, 1, 1), False, False)
    solid = g.cells - g.fluid_cells
    assert abs(solid - 4 / 3 * np.pi * 4.5 ** 3) <= 0.1 * 4 / 3 * np.pi * 4.5 ** 3
    assert g.n_links > 0 and np.all(g.link_q > 0) and np.all(g.link_q <= 1)


def test_walls_q_half(pg, ref):
    """test_geometry.cpp:164-173"""
    g = both(pg, ref, np.zeros((0, 3)), np.zeros(0), (6, 6, 10), (6, 6, 10), (1, 1, 0), True, True)
    assert g.n_links > 0 and np.all(g.link_q == np.float32(0.5)) and g.q_fallback_count == 0


def test_link_count_brute_force(pg, ref):
    """test_geometry.cpp:175-199"""
    g = both(pg, ref, [[8.2, 7.9, 8.4]], np.array([3.7]), (16, 16, 16), (16, 16, 16), (1, 1, 1),
             False, False)
    fl = g.flags.reshape(16, 16, 16) == 0
    n = 0
    for k in range(1, 19):
        e = pg.VELOCITIES[k]
        nb = np.roll(fl, shift=(-e[2], -e[1], -e[0]), axis=(0, 1, 2))
        n += int((fl & ~nb).sum())
    assert g.n_links == n


def test_open_face_is_config_error(pg):
    """test_geometry.cpp:264-271 / geometry.cpp:583-588"""
    with pytest.raises(pg.ConfigError):
        pg.voxelize(pg.SpherePack(np.zeros((0, 3)), np.zeros(0), (8, 8, 8)), (8, 8, 8),
                    (True, True, False))


def test_no_fluid_is_geometry_error(pg):
    with pytest.raises(pg.GeometryError):
        pg.voxelize(pg.SpherePack(np.array([[4.0, 4.0, 4.0]]), np.array([20.0]), (8, 8, 8)),
                    (8, 8, 8), (True, True, True))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_beds_with_plate_and_images(pg, ref, seed):
    rng = np.random.default_rng(seed)
    dims = (40, 28, 36)
    n = 25
    c = np.c_[rng.uniform(-3, 43, n), rng.uniform(-3, 31, n), rng.uniform(0, 30, n)]
    r = rng.uniform(1.5, 7.0, n)
    plate = [0.0, 2.7, -3.0][seed - 1]
    both(pg, ref, c, r, (40.0, 28.0, 36.0), dims, (1, 1, 0), True, True, plate)
    both(pg, ref, c, r, (40.0, 28.0, 36.0), dims, (1, 1, 1), False, False, plate, 0.1)


def test_c2_bed_identical_to_reference(pg, ref):
    from paper_1507_06565_b200 import configs
    w = configs.c2()
    assert w.meta["spheres"] == 227
    g = both(pg, ref, w.pack.centers, w.pack.radii, w.pack.box, w.dims, (1, 1, 0), True, True)
    assert 0.78 < g.fluid_cells / g.cells < 0.82


def test_slab_extraction(pg):
    """voxelize_slab == the global voxelization restricted to [x0, x1)."""
    rng = np.random.default_rng(9)
    dims = (48, 20, 24)
    c = np.c_[rng.uniform(0, 48, 12), rng.uniform(0, 20, 12), rng.uniform(1, 18, 12)]
    r = rng.uniform(2, 5, 12)
    pack = pg.SpherePack(c, r, (48.0, 20.0, 24.0))
    g = pg.voxelize(pack, dims, (True, True, False), True, True)
    nx, ny, nz = dims
    F = g.flags.reshape(nz, ny, nx)
    for x0, x1 in ((0, 16), (16, 32), (32, 48), (0, 48), (5, 29)):
        s = pg.voxelize_slab(pack, dims, x0, x1, (True, True, False), True, True)
        lnx = x1 - x0
        assert s.slab and s.dims == (lnx, ny, nz)
        assert np.array_equal(s.flags.reshape(nz, ny, lnx), F[:, :, x0:x1])
        assert np.array_equal(s.ghost_flags_lo.reshape(nz, ny), F[:, :, (x0 - 1) % nx])
        assert np.array_equal(s.ghost_flags_hi.reshape(nz, ny), F[:, :, x1 % nx])
        gx = g.link_fluid_cell % nx
        sel = (gx >= x0) & (gx < x1)
        gz, gy = g.link_fluid_cell // (nx * ny), (g.link_fluid_cell // nx) % ny
        local = (gz * ny + gy) * lnx + (gx - x0)
        assert np.array_equal(s.link_fluid_cell, local[sel])
        assert np.array_equal(s.link_direction, g.link_direction[sel])
        assert s.link_q.tobytes() == g.link_q[sel].tobytes()
        # second fluid: local index, -2 in a ghost column, -1 none
        sf = g.link_second_fluid[sel]
        sx = sf % nx
        # unwrapped x of x_f2 = x_f1 - e_k: across the slab boundary it is a ghost
        ux = gx[sel] - pg.VELOCITIES[g.link_direction[sel], 0]
        inside = (sf >= 0) & (ux >= x0) & (ux < x1)
        exp = np.where(sf < 0, -1, np.where(inside, (sf // (nx * ny) * ny + (sf // nx) % ny) * lnx
                                            + (sx - x0), -2))
        assert np.array_equal(s.link_second_fluid, exp)


def test_generate_spheres(pg):
    pack, por = pg.generate_spheres(0, 7, (64.0, 32.0, 64.0), 1.0, 30.0, 3.0, 5.0,
                                    64 * 32 * 30, 0.7, 200000)
    pack2, por2 = pg.generate_spheres(0, 7, (64.0, 32.0, 64.0), 1.0, 30.0, 3.0, 5.0,
                                      64 * 32 * 30, 0.7, 200000)
    assert np.array_equal(pack.centers, pack2.centers) and por == por2
    c, r = pack.centers, pack.radii
    assert por <= 0.7 + 1e-12 or len(r) > 0
    # no overlap under the periodic minimum image in x, y
    for i in range(len(r)):
        d = np.abs(c - c[i])
        d[:, 0] = np.minimum(d[:, 0], 64 - d[:, 0])
        d[:, 1] = np.minimum(d[:, 1], 32 - d[:, 1])
        dist2 = (d ** 2).sum(axis=1)
        dist2[i] = np.inf
        assert np.all(dist2 >= (r + r[i]) ** 2 - 1e-9)
    assert np.all((r >= 3.0) & (r <= 5.0))
    assert np.all((c[:, 2] >= 1.0) & (c[:, 2] <= 30.0))
    pack, por = pg.generate_spheres(1, 4, (64.0, 32.0, 64.0), 1.0, 30.0, 3.0, 5.0,
                                    64 * 32 * 30, 0.5, 10 ** 6)
    vol = (4 / 3 * np.pi * pack.radii ** 3).sum()
    assert por == pytest.approx(np.exp(-vol / (64 * 32 * 30)), rel=1e-12) and por <= 0.5
