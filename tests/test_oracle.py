"""Pin the oracle (oracle/porolb_oracle.c) before trusting it (CPU only).

1. The reference's own known-answer tests, restated (proj/tests/test_lattice.cpp,
   test_boundary.cpp, test_simulation.cpp, acceptance_main.cpp criteria 3/11).
2. Bit-for-bit agreement with the reference compiled from its own sources
   (oracle/_ref) on randomised cells, links and whole multi-step runs.
3. Agreement with the committed golden fixture made by the reference at the
   BASELINE step count (tests/golden/C1.json).
"""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


def uniform01(rng):
    return rng.random()


def rand_pops(rng, scale=1e-3):
    return scale * (2.0 * rng.random(19) - 1.0)


# ---------------------------------------------------------------- lattice KATs
def test_d3q19_invariants(orc):
    """test_lattice.cpp:25-54"""
    e, w, opp = orc.tables()
    assert abs(w.sum() - 1.0) <= 1e-15
    assert np.all(w > 0)
    for i in range(3):
        assert abs((w * e[:, i]).sum()) < 1e-15
        for j in range(3):
            assert abs((w * e[:, i] * e[:, j]).sum() - (1 / 3 if i == j else 0)) <= 1e-15
    assert opp[0] == 0
    for k in range(19):
        assert opp[opp[k]] == k
        assert np.array_equal(e[opp[k]], -e[k])
    # pair order relied on by the collision (simulation.cpp:132-146)
    for p in range(9):
        assert opp[2 * p + 1] == 2 * p + 2


def test_equilibrium_kats(orc):
    """test_lattice.cpp:56-120"""
    e, w, _ = orc.tables()
    assert np.all(orc.equilibrium(0.0, (0, 0, 0)) == 0.0)
    np.testing.assert_allclose(orc.equilibrium(1.0, (0, 0, 0)), w, rtol=1e-15)
    u = np.array([0.01, 0.0, 0.0])
    feq = orc.equilibrium(0.0, u)
    for k in range(19):
        eu = e[k] @ u
        exp = w[k] * (3.0 * eu + 0.5 * 9.0 * eu * eu - 0.5 * 3.0 * (u @ u))
        assert feq[k] == pytest.approx(exp, rel=1e-14, abs=1e-14)
    d, mu = orc.moments(feq)
    assert abs(d) < 1e-16 and mu[0] == pytest.approx(0.01, rel=1e-14)
    d, mu = orc.moments(orc.equilibrium(0.5, (0.02, 0.0, -0.01)))
    assert d == pytest.approx(0.5, rel=1e-14)
    np.testing.assert_allclose(mu, [0.02, 0.0, -0.01], rtol=1e-14, atol=1e-17)
    wp, wm = orc.relaxation_from_magic(1 / 6, 3 / 16)
    f = orc.equilibrium(0.3, (0.02, -0.01, 0.015))
    out = orc.trt_collide(f, wp, wm, 1.0, (0, 0, 0))
    assert np.all(np.abs(out - f) <= 1e-14)


def test_trt_conservation(orc):
    """test_lattice.cpp:122-143 and acceptance criterion 11 (acceptance_main.cpp:500-529)."""
    e, _, _ = orc.tables()
    rng = np.random.default_rng(42)
    wp, wm = orc.relaxation_from_magic(0.02, 0.25)
    g = np.array([1e-6, -2e-6, 5e-7])
    for scale in (1e-3, 1e-2):
        for _ in range(2000):
            f = rand_pops(rng, scale)
            out = orc.trt_collide(f, wp, wm, 1.0, g)
            assert abs(out.sum() - f.sum()) <= 1e-14
            assert np.all(np.abs(e.T @ out - e.T @ f - g) <= 1e-14)


def test_trt_pairwise_oracle(orc):
    """test_lattice.cpp:145-175"""
    e, w, opp = orc.tables()
    rng = np.random.default_rng(5)
    f = rand_pops(rng)
    g = np.array([1e-6, 0, 0])
    d, u = orc.moments(f)
    feq = orc.equilibrium(d, u)
    exp = np.array([f[k] - 1.2 * (0.5 * (f[k] + f[opp[k]]) - 0.5 * (feq[k] + feq[opp[k]]))
                    - 1.0 * (0.5 * (f[k] - f[opp[k]]) - 0.5 * (feq[k] - feq[opp[k]]))
                    + 3.0 * w[k] * (e[k] @ g) for k in range(19)])
    np.testing.assert_allclose(orc.trt_collide(f, 1.2, 1.0, 1.0, g), exp, rtol=1e-14, atol=1e-18)


def test_relaxation_from_magic(orc):
    """test_lattice.cpp:177-211"""
    wp, wm = orc.relaxation_from_magic(1 / 6, 3 / 16)
    assert wp == pytest.approx(1.0, rel=1e-15) and wm == pytest.approx(1 / 0.875, rel=1e-14)
    wp, wm = orc.relaxation_from_magic(1 / 6, 0.25)
    assert wp == pytest.approx(1.0) and wm == pytest.approx(1.0)
    rng = np.random.default_rng(11)
    for _ in range(100):
        nu, lam = 0.01 + 0.5 * rng.random(), 0.05 + rng.random()
        wp, wm = orc.relaxation_from_magic(nu, lam)
        assert 0 < wp < 2 and 0 < wm < 2
        assert (1 / wp - 0.5) * (1 / wm - 0.5) == pytest.approx(lam, rel=1e-13)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        orc.relaxation_from_magic(-1.0, 0.25)
    with pytest.raises(OracleError):
        orc.relaxation_from_magic(0.1, -0.25)


def test_trt_nonfinite(orc):
    """test_lattice.cpp:213-219"""
    from oracle.oracle import OracleError
    f = np.zeros(19)
    f[3] = np.inf
    with pytest.raises(OracleError):
        orc.trt_collide(f, 1.0, 1.0, 1.0, (0, 0, 0))


def test_kozeny_carman(orc, ref):
    """test_glbm.cpp:98-108 value and the ε >= 0.999 -> infinity rule."""
    eps = np.array([0.4, 0.5, 0.9, 0.999, 1.0])
    K = orc.kozeny_carman(eps, 10.0)
    assert K[0] == pytest.approx(0.4 ** 3 * 100 / (180 * 0.36), rel=1e-15)
    assert np.isinf(K[3]) and np.isinf(K[4])
    assert np.array_equal(K, ref.kozeny_carman(eps, 10.0))


# ----------------------------------------------------- oracle vs the reference
def test_cell_ops_bitwise_vs_reference(orc, ref):
    rng = np.random.default_rng(1)
    for _ in range(500):
        nu, lam = 0.01 + 0.4 * rng.random(), 0.05 + rng.random()
        assert orc.relaxation_from_magic(nu, lam) == ref.relaxation_from_magic(nu, lam)
        wp, wm = orc.relaxation_from_magic(nu, lam)
        f = rand_pops(rng, 10 ** rng.uniform(-6, -1))
        g = rng.normal(size=3) * 1e-6
        rho0 = 1.0 if rng.random() < 0.5 else 0.5 + rng.random()
        assert np.array_equal(orc.trt_collide(f, wp, wm, rho0, g), ref.trt_collide(f, wp, wm, rho0, g))
        u = rng.normal(size=3) * 0.01
        assert np.array_equal(orc.equilibrium(0.1, u, rho0), ref.equilibrium(0.1, u, rho0))
    for mode in (0, 1, 2):
        eps = np.linspace(0.3, 1.0, 17)
        K = orc.kozeny_carman(eps, 7.0)
        a = orc.make_glbm_params(eps, 1 / 6, 3 / 16, mode, 0.7)
        b = ref.make_glbm_params(eps, K, 0.0, 1 / 6, 3 / 16, mode, 0.7)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_boundary_kats(ref):
    """test_boundary.cpp:49-120 and acceptance criterion 3 (acceptance_main.cpp:127-158)."""
    dims = (3, 3, 3)
    cells = 27
    idx = lambda x, y, z: (z * 3 + y) * 3 + x  # noqa: E731
    cur = np.zeros(19 * cells)
    cur[5 * cells + idx(1, 1, 1)] = 0.3
    assert ref.apply_link(0, dims, cur, idx(1, 1, 1), -1, 5, 0.5) == 0.3
    cur = np.zeros(19 * cells)
    f1, f2 = idx(1, 1, 1), idx(1, 1, 0)
    cur[5 * cells + f2], cur[6 * cells + f1], cur[5 * cells + f1] = 0.1, 0.2, 0.3
    assert ref.apply_link(1, dims, cur, f1, f2, 5, np.float32(0.25)) == pytest.approx(
        0.26666666666666666, rel=1e-12)
    rng = np.random.default_rng(1234)
    E = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
                  [1, 1, 0], [-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 0, 1], [-1, 0, -1],
                  [1, 0, -1], [-1, 0, 1], [0, 1, 1], [0, -1, -1], [0, 1, -1], [0, -1, 1]])
    for _ in range(1000):
        k = 1 + int(rng.integers(0, 18))
        kb = k + 1 if k % 2 else k - 1
        f2 = idx(*[(1 - E[k][i] + 3) % 3 for i in range(3)])
        v = rng.random(3)
        cur = np.zeros(19 * cells)
        cur[k * cells + f2], cur[kb * cells + f1], cur[k * cells + f1] = v
        a = ref.apply_link(1, dims, cur, f1, f2, k, np.float32(0.5))
        b = ref.apply_link(0, dims, cur, f1, f2, k, np.float32(0.5))
        assert a == b  # CLI(q=1/2) is bitwise SBB
    cur = np.zeros(19 * cells)
    cur[11 * cells + idx(1, 1, 2)] = 0.05
    got = ref.apply_link(2, dims, cur, idx(1, 1, 2), -1, 11, 0.5, (0.01, 0, 0))
    assert got == pytest.approx(0.05 - 2.0 * (1 / 36) * 3.0 * 0.01, rel=1e-15)


def sphere_geom(orc, dims, n, seed, walls=True, periodic=(1, 1, 0), plate=0.0):
    rng = np.random.default_rng(seed)
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n),
              rng.uniform(1, dims[2] * 0.7, n)]
    r = rng.uniform(2.0, 5.0, n)
    return orc.voxelize(c, r, dims, dims, periodic, walls, walls, plate), (c, r)


@pytest.mark.parametrize("scheme", [0, 1])
def test_multistep_bitwise_vs_reference(orc, ref, scheme):
    g, _ = sphere_geom(orc, (24, 16, 20), 6, 3)
    wp, wm = orc.relaxation_from_magic(0.07, 3 / 16)
    G = (2e-6, -3e-7, 1e-7)
    o = orc.simulation(g, 0.07, wp, wm, G, scheme)
    r = ref.simulation(g, 0.07, wp, wm, 3 / 16, G, scheme)
    rng = np.random.default_rng(8)
    f0 = 1e-4 * rng.normal(size=(19,) + tuple(g.dims[::-1]))
    f0[:, g.flags.reshape(g.dims[::-1]) != 0] = 0.0
    o.set_pdfs(f0)
    r.set_pdfs(f0)
    o.step(60)
    r.step(60)
    fl = g.flags.reshape(g.dims[::-1]) == 0
    assert np.array_equal(o.get_pdfs()[:, fl], r.get_pdfs()[:, fl])
    a, b = o.planar_profile(), r.planar_profile()
    for k in ("z", "u_superficial", "u_intrinsic", "epsilon", "u_normalized"):
        assert np.array_equal(a[k], b[k]), k
    assert o.max_speed() == r.max_speed()
    for x, y in zip(o.macroscopic_fields(), r.macroscopic_fields()):
        assert np.array_equal(x[fl], y[fl])


def test_glbm_and_lid_bitwise_vs_reference(orc, ref):
    nz = 20
    g = orc.voxelize(np.zeros((0, 3)), np.zeros(0), (8, 4, nz), (8, 4, nz), (1, 1, 0), True, True)
    eps = np.clip(np.linspace(0.4, 1.1, nz), 0, 1.0)
    K = orc.kozeny_carman(eps, 5.0)
    for cf, eq in ((0.0, True), (0.2, False)):
        wpz, wmz = orc.make_glbm_params(eps, 1 / 6, 3 / 16, 1)
        o = orc.simulation(g, 1 / 6, 1.0, 1 / 0.875, (1e-5, 0, 0), 0)
        r = ref.simulation(g, 1 / 6, 1.0, 1 / 0.875, 3 / 16, (1e-5, 0, 0), 0)
        o.set_porous(eps, K, wpz, wmz, cf, eq)
        r.set_porous(eps, K, wpz, wmz, cf, eq)
        o.step(40)
        r.step(40)
        fl = g.flags.reshape(g.dims[::-1]) == 0
        assert np.array_equal(o.get_pdfs()[:, fl], r.get_pdfs()[:, fl])
        assert np.array_equal(o.planar_profile()["u_superficial"], r.planar_profile()["u_superficial"])
    o = orc.simulation(g, 1 / 6, 1.0, 1 / 0.875, (0, 0, 0), 1)
    r = ref.simulation(g, 1 / 6, 1.0, 1 / 0.875, 3 / 16, (0, 0, 0), 1)
    o.set_lid_velocity((0.01, 0.0, 0.0))
    r.set_lid_velocity((0.01, 0.0, 0.0))
    o.step(30)
    r.step(30)
    assert np.array_equal(o.get_pdfs()[:, fl], r.get_pdfs()[:, fl])


def test_streaming_kats(orc):
    """test_simulation.cpp:26-82 on the oracle's push streaming (no links)."""
    e, _, _ = orc.tables()
    g = orc.voxelize(np.zeros((0, 3)), np.zeros(0), (5, 4, 3), (5, 4, 3), (1, 1, 1))
    o = orc.simulation(g, 0.1, 1.0, 1.0, (0, 0, 0), 0)
    # gather oracle on a random state: one push stream == f_k(x - e_k)
    rng = np.random.default_rng(17)
    f = rng.random((19, 3, 4, 5))
    import ctypes as C
    from oracle.oracle import _i3, _p
    nxt = np.zeros_like(f)
    o.o.lib.orc_stream_pass(_i3((5, 4, 3)), _i3((1, 1, 1)), _p(o.flags, C.c_uint8),
                            _p(np.ascontiguousarray(f), C.c_double), _p(nxt, C.c_double))
    for k in range(19):
        assert np.array_equal(nxt[k], np.roll(f[k], shift=(e[k][2], e[k][1], e[k][0]), axis=(0, 1, 2)))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_matches_golden_c1(orc, pg):
    """The C restatement reproduces the reference's own C1 run (2000 steps)
    bit for bit (fixture generated by tests/golden/make_golden.py)."""
    gold = json.loads((GOLDEN / "C1.json").read_text())
    from paper_1507_06565_b200 import configs
    w = configs.c1()
    g = orc.voxelize(np.zeros((0, 3)), np.zeros(0), w.dims, w.dims, (1, 1, 0), True, True)
    assert _sha(g.flags) == gold["geometry"]["flags_sha256"]
    p = w.params()
    o = orc.simulation(g, p.nu, p.omega_plus, p.omega_minus, p.body_force, 0)
    o.step(gold["steps"])
    fl = g.flags.reshape(w.dims[::-1]) == 0
    assert _sha(o.get_pdfs()[:, fl]) == gold["state"]["pdf_sha256"]
    prof = o.planar_profile()
    assert [float(v).hex() for v in prof["u_superficial"]] == gold["state"]["profile_u_superficial"]


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C5"])
def test_ref_workloads_match_configs(orc, pg, key):
    """oracle/ref_workloads.py (the reference arm's workloads, built without
    the product) restates configs.py: same recipe, same sphere list, and a
    geometry byte-identical to the reference-made golden fixture."""
    from oracle import ref_workloads
    from paper_1507_06565_b200 import configs
    w = configs.ALL[key]()
    rw, geom, meta = ref_workloads.build(key, orc)
    assert meta.pop("geometry_checked").startswith("sha256 == tests/golden")
    assert (rw.name, tuple(rw.dims), rw.scheme, rw.nu, tuple(rw.g), rw.steps) == \
        (w.name, tuple(w.dims), w.scheme.name, w.nu, tuple(w.g), w.steps)
    assert meta == w.meta
    assert rw.glbm == (w.glbm is not None)
    if w.pack is not None:
        c, r, _ = orc.generate_spheres(**rw.spheres)
        assert np.array_equal(c, w.pack.centers) and np.array_equal(r, w.pack.radii)
    g = w.geometry()
    assert np.array_equal(geom.flags, g.flags)
    for f in ("link_fluid_cell", "link_second_fluid", "link_direction", "link_q", "porosity"):
        assert np.array_equal(getattr(geom, f), getattr(g, f)), f


def test_c4_recipe_matches_configs(orc, pg):
    """C4's sphere list (Boolean model, 20 783 spheres) from the oracle
    generator equals the product harness one (geometry: checked against the
    golden hashes whenever the reference arm runs)."""
    from oracle import ref_workloads
    from paper_1507_06565_b200 import configs
    rw = ref_workloads.WORKLOADS["C4"]
    w = configs.c4()
    c, r, por = orc.generate_spheres(**rw.spheres)
    assert np.array_equal(c, w.pack.centers) and np.array_equal(r, w.pack.radii)
    assert por == w.meta["boolean_bed_porosity"]
    assert _sha(np.c_[c, r]) == json.loads((GOLDEN / "C4.json").read_text())["sphere_sha256"]
