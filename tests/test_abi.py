"""The C-ABI library (CPU side): it loads, exports every symbol the header
declares, its host functions are bit-identical to the reference, errors map
to the reference exception types, and there is no CPU fallback."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

HEADER = Path(__file__).resolve().parent.parent / "include" / "porolb_gpu.h"


def declared_symbols():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pgpu_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(pg):
    from paper_1507_06565_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 45
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert _lib.lib.pgpu_abi_version() == 1


def test_library_is_sm100a_only():
    """The product .so carries sm_100a SASS only (no PTX/JIT fallback)."""
    import subprocess
    so = Path(__file__).resolve().parent.parent / "paper_1507_06565_b200" / "libporolb_cuda.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))
    ptx = subprocess.run(["cuobjdump", "--list-ptx", str(so)], capture_output=True, text=True).stdout
    assert ptx.strip() == ""


def test_relaxation_bitwise_vs_reference(pg, ref):
    rng = np.random.default_rng(3)
    for _ in range(300):
        nu, lam = 0.005 + 0.6 * rng.random(), 0.02 + 2 * rng.random()
        try:
            want = ref.relaxation_from_magic(nu, lam)
        except Exception:
            with pytest.raises(pg.ConfigError):
                pg.relaxation_from_magic(nu, lam)
            continue
        p = pg.relaxation_from_magic(nu, lam)
        assert (p.omega_plus, p.omega_minus) == want
    with pytest.raises(pg.ConfigError):
        pg.relaxation_from_magic(-0.1, 0.25)
    with pytest.raises(pg.ConfigError):
        pg.relaxation_from_magic(0.1, 0.0)
    p = pg.relaxation_from_magic(0.1, 0.1875)
    assert p.omega_plus == 1.25 and p.omega_minus == 0.88888888888888884


def test_cell_functions_bitwise_vs_reference(pg, ref):
    rng = np.random.default_rng(4)
    for _ in range(300):
        f = 1e-3 * rng.normal(size=19)
        p = pg.relaxation_from_magic(0.02 + 0.3 * rng.random(), 3 / 16)
        p.body_force = tuple(rng.normal(size=3) * 1e-6)
        p.rho0 = 1.0 if rng.random() < 0.5 else 0.7 + rng.random()
        assert np.array_equal(pg.trt_collide(f, p),
                              ref.trt_collide(f, p.omega_plus, p.omega_minus, p.rho0, p.body_force))
        u = rng.normal(size=3) * 0.01
        assert np.array_equal(pg.equilibrium(0.2, u, p.rho0), ref.equilibrium(0.2, u, p.rho0))
    f = np.zeros(19)
    f[3] = np.inf
    with pytest.raises(pg.NumericalInstability):
        pg.trt_collide(f, pg.relaxation_from_magic(1 / 6, 0.25))


def test_glbm_host_functions(pg, ref, orc):
    eps = np.r_[np.linspace(0.35, 0.998, 30), [0.999, 1.0]]
    K = pg.kozeny_carman(eps, 10.0)
    assert np.array_equal(K, ref.kozeny_carman(eps, 10.0))
    for mode in (pg.GlbmViscosity.Plain, pg.GlbmViscosity.Rescaled, pg.GlbmViscosity.ConstantRatio):
        gp = pg.make_glbm_params(eps, K, 0.0, 1 / 6, 3 / 16, mode, 0.8)
        wp, wm = ref.make_glbm_params(eps, K, 0.0, 1 / 6, 3 / 16, int(mode), 0.8)
        assert np.array_equal(gp.omega_plus, wp) and np.array_equal(gp.omega_minus, wm)
    with pytest.raises(pg.ConfigError):
        pg.make_glbm_params([0.0, 0.5], [1.0, 1.0], 0.0, 1 / 6, 3 / 16, pg.GlbmViscosity.Plain)
    rng = np.random.default_rng(2)
    for _ in range(100):
        mom = rng.normal(size=3) * 1e-3
        e, k, cf = 0.3 + 0.7 * rng.random(), 10 ** rng.uniform(-4, 1), rng.choice([0.0, 0.1, 0.5])
        g = rng.normal(size=3) * 1e-6
        u, F = pg.glbm_force_and_velocity(mom, e, k, cf, g, 1 / 6)
        uo, Fo = orc.glbm_force_and_velocity(mom, e, k, cf, g, 1 / 6)
        assert np.array_equal(u, uo) and np.array_equal(F, Fo)
    # simulation.hpp:38-43 closed forms (test_simulation.cpp:232-260)
    u, F = pg.glbm_force_and_velocity((0.01, -0.002, 0.0), 1.0, np.inf, 0.0, (0, 0, 0), 1 / 6)
    assert u[0] == 0.01 and u[1] == -0.002 and F[0] == 0.0
    u, _ = pg.glbm_force_and_velocity((0.01, 0, 0), 0.5, 1e-3, 0.0, (1e-6, 0, 0), 1 / 6)
    assert u[0] == pytest.approx((0.01 + 0.25e-6) / (1 + 0.5 / 6 / 2e-3), rel=1e-15)


def test_no_cpu_fallback(pg):
    """Without a usable sm_100 device the product fails loudly."""
    if pg.device_count() > 0:
        pytest.skip("a GPU is visible")
    geom = pg.make_box_geometry((4, 4, 6), (True, True, False), True, True)
    with pytest.raises(pg.CudaError):
        pg.Simulation(geom, 0.1, 3 / 16, (0, 0, 0), pg.WallScheme.SBB)


def test_status_codes_and_last_error(pg):
    from paper_1507_06565_b200 import _lib
    out = _lib.FluidParams()
    assert _lib.lib.pgpu_relaxation_from_magic(-1.0, 0.25, C.byref(out)) == 1
    assert b"viscosity" in _lib.lib.pgpu_last_error()
    assert _lib.lib.pgpu_relaxation_from_magic(0.1, 0.25, None) == 5


def test_glbm_equilibrium_bitwise_vs_reference(pg, ref):
    """simulation.cpp:68-78 (bindings.cpp:92-97); ConfigError for eps <= 0."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        drho = 0.02 * rng.standard_normal()
        u = 0.05 * rng.standard_normal(3)
        eps = rng.uniform(0.05, 1.0)
        rho0 = rng.choice([1.0, 1.3])
        assert np.array_equal(pg.glbm_equilibrium(drho, u, eps, rho0),
                              ref.glbm_equilibrium(drho, u, eps, rho0))
    # eps = 1: the standard equilibrium (to rounding: the reference groups the
    # quadratic terms differently, simulation.cpp:76 vs lattice.cpp:84)
    u = (0.01, -0.002, 0.003)
    assert np.array_equal(pg.glbm_equilibrium(0.0, u, 1.0), ref.glbm_equilibrium(0.0, u, 1.0))
    np.testing.assert_allclose(pg.glbm_equilibrium(0.0, u, 1.0), ref.equilibrium(0.0, u, 1.0),
                               rtol=1e-14, atol=1e-20)
    for bad in (0.0, -0.5, float("nan")):
        with pytest.raises(pg.ConfigError):
            pg.glbm_equilibrium(0.0, u, bad)


def test_resolve_drive_vs_reference(pg, ref):
    """boundary.cpp:9-17 (dns.cpp:13 calls it)."""
    D = pg.DriveSpec
    spec = D(pg.DriveMode.BodyForce, (1e-6, 2e-7, -3e-8))
    assert pg.resolve_drive(spec) == ref.resolve_drive(0, (1e-6, 2e-7, -3e-8))
    for axis in (0, 1, 2):
        spec = D(pg.DriveMode.PressureGradientAsForce, (3e-5, 7e-6, 1e-6), stream_axis=axis,
                 channel_length=97.0)
        assert pg.resolve_drive(spec) == ref.resolve_drive(1, (3e-5, 7e-6, 1e-6), axis, 97.0)
    for length in (0.0, -1.0):
        with pytest.raises(pg.ConfigError, match="positive channel length"):
            pg.resolve_drive(D(pg.DriveMode.PressureGradientAsForce, (1e-5, 0, 0),
                               channel_length=length))
    with pytest.raises(pg.ConfigError):
        pg.resolve_drive(D(pg.DriveMode.PressureGradientAsForce, (1e-5, 0, 0), stream_axis=3,
                           channel_length=10.0))


def test_porosity_profile_vs_reference(pg, ref):
    """geometry.cpp:642-661 on a sphere bed (plate and walls included)."""
    rng = np.random.default_rng(4)
    dims = (30, 20, 26)
    c = np.c_[rng.uniform(0, 30, 7), rng.uniform(0, 20, 7), rng.uniform(2, 20, 7)]
    pack = pg.SpherePack(c, rng.uniform(2, 5, 7), (30.0, 20.0, 26.0), 3.2)
    g = pg.voxelize(pack, dims, (True, True, False), True, True)
    prof = pg.porosity_profile(g)
    z, eps = ref.porosity_profile(g)
    assert np.array_equal(prof.z, z) and np.array_equal(prof.epsilon, eps)
    assert not prof.u_superficial.any() and prof.u_normalized.size == dims[2]
    np.testing.assert_array_equal(prof.epsilon, g.porosity)  # voxelize's own porosity


def test_dns_driver_compiles_unchanged(pg):
    """the reference's dns.cpp make_simulation (with
    resolve_drive(cfg.drive)) compiles and links against the C++ mirror."""
    import subprocess
    root = Path(__file__).resolve().parent.parent
    res = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", f"-I{root / 'include'}",
                          str(root / "tests" / "cpp" / "dns_dropin.cpp")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
