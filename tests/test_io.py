"""File formats (proj/src/io.cpp) against the reference's own
io.cpp compiled into oracle/_ref: every writer byte-identical, every reader
returning the reference's values and raising its error types.

CPU tests exercise the host code in libporolb_cuda.so (no device needed); the
VTK writer reads the moments from the device, so its parity test is `gpu`.
"""
import struct

import numpy as np
import pytest


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def _random_doubles(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    vals = bits.view(np.float64)
    extra = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1 / 3, 1e-300, 5e-324, -5e-324, 1.7976931348623157e308,
                      np.inf, -np.inf, 123456789012345678.0, 1e16, 1e17, 9.999999999999999e22,
                      2.5, 0.5e-4, 1e-5, 123.0])
    nice = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)
    return np.concatenate([extra, vals, nice])


def test_format_double_matches_reference(pg, ref):
    for v in _random_doubles(20000, 1):
        a, b = pg.format_double(v), ref.format_double(v)
        assert a == b, (struct.pack("<d", v).hex(), a, b)
        if not np.isnan(v):
            assert a == "%.17g" % v or a in ("inf", "-inf")


def _profile(pg, n, seed, n_norm=None):
    rng = np.random.default_rng(seed)
    z = np.arange(n) + 0.5
    us = rng.standard_normal(n) * 1e-4
    ui = us / rng.uniform(0.3, 1.0, n)
    eps = rng.uniform(0.0, 1.0, n)
    un = us / np.abs(us).max()
    if n_norm is not None:
        un = un[:n_norm]
    return pg.ProfileData(z, us, ui, eps, un, float(np.abs(us).max()), 30.0, 1.0, 1 / 6,
                          (1e-6, -2.5e-9, 0.0), 0)


def _meta(p):
    return [p.u_max, p.height, p.z0, p.nu, *p.body_force, p.stream_axis]


@pytest.mark.parametrize("n,n_norm", [(37, None), (12, 5), (1, None), (9, 0)])
def test_profile_csv_write_identical_and_read_back(pg, ref, tmp_path, n, n_norm):
    p = _profile(pg, n, n, n_norm)
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    pg.write_profile_csv(ours, p)
    ref.write_profile_csv(theirs, p.z, p.u_superficial, p.u_intrinsic, p.epsilon,
                          p.u_normalized, _meta(p))
    assert _bytes(ours) == _bytes(theirs)
    q = pg.read_profile_csv(theirs)
    r = ref.read_profile_csv(theirs)
    for name in ("z", "u_superficial", "u_intrinsic", "epsilon", "u_normalized"):
        assert np.array_equal(getattr(q, name), r[name]), name
        want = getattr(p, name)
        if name == "u_normalized":  # missing entries are written as 0 (io.cpp:58)
            want = np.concatenate([want, np.zeros(n - want.size)])
        assert np.array_equal(getattr(q, name), want), name
    assert [q.u_max, q.height, q.z0, q.nu, *q.body_force, q.stream_axis] == list(r["meta"])


PROFILE_TEXTS = {
    "crlf_and_comments": "# nu = 0.25\r\n#no equals sign\n# g = 1 2 3\n\n# junk : 4\n"
                         "header,whatever\n1,2,3,4\r\n5,6,7,8,9\n10,11,12,13,\n",
    "extra_columns": "# stream_axis = 2\nz,a,b,c,d\n1,2,3,4,5,6,7\n",
    "trailing_garbage_numbers": "h\n1.5abc,2e3,  3,4\n",
    "no_header_comment_only": "# u_max = 7\n",
    "short_row": "z,a\n1,2,3\n",
    "only_header": "z,U\n\n",
    "bad_number": "z\nfoo,1,2,3\n",
}


@pytest.mark.parametrize("name", sorted(PROFILE_TEXTS))
def test_profile_csv_read_rules(pg, ref, tmp_path, name):
    path = tmp_path / "p.csv"
    path.write_bytes(PROFILE_TEXTS[name].encode())
    try:
        r = ref.read_profile_csv(path)
        ref_err = None
    except Exception as e:  # noqa: BLE001
        ref_err = e
    if ref_err is not None:
        with pytest.raises(Exception) as ei:
            pg.read_profile_csv(path)
        if getattr(ref_err, "code", None) == 1:
            assert isinstance(ei.value, pg.ConfigError)
            assert str(ei.value) == str(ref_err).split(": ", 1)[-1] or str(ref_err).endswith(str(ei.value))
        return
    q = pg.read_profile_csv(path)
    for k in ("z", "u_superficial", "u_intrinsic", "epsilon", "u_normalized"):
        assert np.array_equal(getattr(q, k), r[k]), k
    assert [q.u_max, q.height, q.z0, q.nu, *q.body_force, q.stream_axis] == list(r["meta"])


def test_profile_csv_missing_file(pg, tmp_path):
    with pytest.raises(pg.ConfigError, match="cannot open profile CSV"):
        pg.read_profile_csv(tmp_path / "absent.csv")


def test_comparison_csv_identical(pg, ref, tmp_path):
    rng = np.random.default_rng(3)
    a = _profile(pg, 50, 4)
    a.z = np.linspace(-2.0, 60.0, 50)
    zb = np.sort(rng.uniform(0.0, 50.0, 23))
    zb[5] = a.z[10]  # exact hit
    b = pg.ProfileData(zb, rng.standard_normal(23))
    pg.write_comparison_csv(tmp_path / "o.csv", a, "simulated", b, "analytic")
    ref.write_comparison_csv(tmp_path / "r.csv", a.z, a.u_superficial, "simulated", b.z,
                             b.u_superficial, "analytic")
    assert _bytes(tmp_path / "o.csv") == _bytes(tmp_path / "r.csv")
    with pytest.raises(pg.ConfigError, match="empty profile"):
        pg.write_comparison_csv(tmp_path / "e.csv", a, "a", pg.ProfileData(), "b")


def test_report_identical(pg, ref, tmp_path):
    entries = [("scenario", "dns"), ("nu", pg.format_double(1 / 6)), ("empty", ""),
               ("spaces in key", "a = b")]
    pg.write_report(tmp_path / "o.txt", entries)
    ref.write_report(tmp_path / "r.txt", entries)
    assert _bytes(tmp_path / "o.txt") == _bytes(tmp_path / "r.txt")
    pg.write_report(tmp_path / "o0.txt", [])
    assert _bytes(tmp_path / "o0.txt") == b""


def test_write_to_unwritable_path(pg, tmp_path):
    with pytest.raises(pg.ConfigError, match="cannot write file"):
        pg.write_report(tmp_path / "no_such_dir" / "r.txt", [("a", "b")])


def _pack(pg, n=40, seed=5, box=(64.0, 32.0, 48.0)):
    rng = np.random.default_rng(seed)
    c = np.c_[rng.uniform(0, box[0], n), rng.uniform(0, box[1], n), rng.uniform(2, box[2] * 0.6, n)]
    r = rng.uniform(2.0, 6.0, n)
    return pg.SpherePack(c, r, box, bottom_plate_z=-0.75, seed=2**63 + 12345)


def test_sphere_csv_identical_and_read_back(pg, ref, tmp_path):
    pack = _pack(pg)
    pg.write_sphere_csv(tmp_path / "o.csv", pack)
    ref.write_sphere_csv(tmp_path / "r.csv", pack.centers, pack.radii, pack.box,
                         pack.bottom_plate_z, pack.seed)
    assert _bytes(tmp_path / "o.csv") == _bytes(tmp_path / "r.csv")
    q = pg.read_sphere_csv(tmp_path / "r.csv")
    r = ref.read_sphere_csv(tmp_path / "r.csv")
    assert np.array_equal(q.centers, r["centers"]) and np.array_equal(q.radii, r["radii"])
    assert np.array_equal(q.centers, pack.centers) and np.array_equal(q.radii, pack.radii)
    assert q.box == r["box"] == pack.box
    assert q.bottom_plate_z == r["bottom_plate_z"] == pack.bottom_plate_z
    assert q.seed == r["seed"] == pack.seed
    assert q.achieved_height == r["achieved_height"]


@pytest.mark.parametrize("text,err", [
    ("x,y,z,r\n1,2,3,4\n", "missing the box header"),
    ("# box = 4 4 4\nx,y,z,r\n1,2,3\n", "rows need x,y,z,r"),
    ("# seed = 9 box = 8 8 8 plate_z = -1\nx\n1,1,1,0.5\n\n2,2,2,1.5\r\n", None),
    ("# box = 8 8 8\n", None),
])
def test_sphere_csv_read_rules(pg, ref, tmp_path, text, err):
    path = tmp_path / "s.csv"
    path.write_bytes(text.encode())
    if err:
        with pytest.raises(pg.ConfigError, match=err):
            pg.read_sphere_csv(path)
        with pytest.raises(Exception, match=err):
            ref.read_sphere_csv(path)
        return
    q, r = pg.read_sphere_csv(path), ref.read_sphere_csv(path)
    assert np.array_equal(q.centers.reshape(-1, 3), r["centers"].reshape(-1, 3))
    assert np.array_equal(q.radii, r["radii"])
    assert (q.box, q.bottom_plate_z, q.seed, q.achieved_height) == \
        (r["box"], r["bottom_plate_z"], r["seed"], r["achieved_height"])


def _geoms(pg):
    pack = _pack(pg, 30, 11, (48.0, 24.0, 40.0))
    yield "spheres_walls", pg.voxelize(pack, (48, 24, 40), (True, True, False), True, True)
    yield "spheres_periodic", pg.voxelize(pack, (48, 24, 40), (True, True, True))
    yield "box_periodic", pg.make_box_geometry((6, 5, 7), (True, True, True))
    yield "channel", pg.make_box_geometry((4, 4, 10), (True, True, False), True, True)


def _assert_same_geometry(a, b):
    assert tuple(a.dims) == tuple(b.dims)
    assert tuple(a.periodic) == tuple(b.periodic)
    assert np.array_equal(a.flags, b.flags)
    for k in ("link_fluid_cell", "link_second_fluid", "link_direction", "link_q", "link_moving",
              "porosity"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.fluid_cells == b.fluid_cells
    assert a.wall_plane_lo == b.wall_plane_lo and a.wall_plane_hi == b.wall_plane_hi


def test_voxel_file_identical_and_links_rebuilt(pg, ref, tmp_path):
    for name, g in _geoms(pg):
        ours, theirs = tmp_path / f"{name}_o.vox", tmp_path / f"{name}_r.vox"
        pg.write_voxel_file(ours, g)
        ref.write_voxel_file(theirs, g)
        assert _bytes(ours) == _bytes(theirs), name
        q = pg.read_voxel_file(theirs)
        r = ref.read_voxel_file(theirs)
        _assert_same_geometry(q, r)
        assert np.array_equal(q.flags, g.flags)
        assert np.all(q.link_q == np.float32(0.5)) and q.wall_plane_lo is None
        # same fluid->non-fluid directions as the voxelizer's links
        assert np.array_equal(q.link_fluid_cell, g.link_fluid_cell)
        assert np.array_equal(q.link_direction, g.link_direction)


def _vox_bytes(dims, periodic, flags):
    head = "porolb-voxel 1 %d %d %d %d %d %d\n" % (*dims, *[int(p) for p in periodic])
    return head.encode() + bytes(np.asarray(flags, dtype=np.uint8).tobytes())


@pytest.mark.parametrize("case", ["bad_magic", "bad_version", "truncated", "open_face",
                                  "no_fluid", "open_face_x", "walls_closed", "flag_seven"])
def test_voxel_file_read_rules(pg, ref, tmp_path, case):
    dims, per = (5, 4, 6), (True, True, False)
    flags = np.zeros(dims[::-1], dtype=np.uint8)
    flags[0] = flags[-1] = 2
    flags[2, 1, 2] = 1
    data = None
    err, kind = None, pg.ConfigError
    if case == "bad_magic":
        data, err = b"porolb-voxels 1 1 1 1 1 1 1\n\x00", "not a porolb voxel file"
    elif case == "bad_version":
        data, err = b"porolb-voxel 2 1 1 1 1 1 1\n\x00", "not a porolb voxel file"
    elif case == "truncated":
        data, err = _vox_bytes(dims, per, flags)[:-3], "truncated voxel data"
    elif case == "open_face":
        flags[-1] = 0
        err = "non-periodic open face"
    elif case == "open_face_x":
        per = (False, True, False)
        err = "non-periodic open face"
    elif case == "no_fluid":
        flags[:] = 1
        err, kind = "no fluid cells", pg.GeometryError
    elif case == "flag_seven":
        flags[3, 2, 1] = 7
    path = tmp_path / "g.vox"
    path.write_bytes(data if data is not None else _vox_bytes(dims, per, flags))
    if err:
        with pytest.raises(kind, match=err):
            pg.read_voxel_file(path)
        with pytest.raises(Exception, match=err):
            ref.read_voxel_file(path)
        return
    _assert_same_geometry(pg.read_voxel_file(path), ref.read_voxel_file(path))


def test_voxel_file_round_trip_feeds_simulation_geometry(pg, tmp_path):
    """write -> read keeps flags and periodicity; the rebuilt links close
    exactly the fluid->non-fluid directions (so pgpu_create accepts them)."""
    _, g = next(_geoms(pg))
    pg.write_voxel_file(tmp_path / "g.vox", g)
    h = pg.read_voxel_file(tmp_path / "g.vox")
    assert np.array_equal(h.flags, g.flags) and h.periodic == g.periodic
    assert h.n_links == g.n_links
    assert np.array_equal(h.porosity, g.porosity)


# ---- write_vtk (moments from the device) -------------------------------------------
def _sim_pair(pg, ref, geom, scheme, nu=0.1, g=(1e-5, 2e-6, -1e-6), glbm=False):
    p = pg.relaxation_from_magic(nu, 3.0 / 16.0)
    p.body_force = g
    sim = pg.Simulation.from_params(geom, p, pg.WallScheme(scheme))
    r = ref.simulation(geom, p.nu, p.omega_plus, p.omega_minus, p.lambda_magic, p.body_force,
                       scheme)
    if glbm:
        nz = geom.dims[2]
        eps = np.linspace(0.4, 1.0, nz)
        K = pg.kozeny_carman(eps, 8.0)
        gp = pg.make_glbm_params(eps, K, 0.0, nu, 3.0 / 16.0, pg.GlbmViscosity.Rescaled)
        sim.set_porous(gp)
        r.set_porous(gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus, gp.forchheimer_cf,
                     gp.eps_in_equilibrium)
    return sim, r


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cli_spheres", "sbb_spheres", "glbm_channel", "fresh"])
def test_write_vtk_identical(gpu, ref, tmp_path, case):
    pg = gpu
    if case == "glbm_channel":
        geom = pg.make_box_geometry((6, 5, 24), (True, True, False), True, True)
    else:
        _, geom = next(_geoms(pg))
    sim, r = _sim_pair(pg, ref, geom, 0 if case == "sbb_spheres" else 1,
                       glbm=case == "glbm_channel")
    steps = 0 if case == "fresh" else 57
    sim.step(steps)
    r.step(steps)
    sim_path, ref_path = tmp_path / "o.vtk", tmp_path / "r.vtk"
    pg.write_vtk(sim_path, sim)
    r.write_vtk(ref_path)
    a, b = _bytes(sim_path), _bytes(ref_path)
    assert len(a) == len(b) and a == b
    assert np.array_equal(sim.flags().reshape(-1), geom.flags)
