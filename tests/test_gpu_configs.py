"""The five BASELINE configs at their stated step counts, on the B200 through
the C ABI, against golden fixtures made by the REFERENCE solver
(tests/golden/make_golden.py, oracle/_ref).  The fixture stores the sha256 of
the reference's fluid-cell populations f(N) and velocity components, so the
first assertion is bit-for-bit identity; samples, per-direction sums and the
u_x(z) profile are then checked against the north-star tolerance (1e-12
relative to the field's max) so that a failure is diagnosable."""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
TOL = 1e-12


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unhex(v):
    return np.array([float.fromhex(x) for x in v])


def geometry_hashes(g):
    return {
        "flags_sha256": sha(g.flags),
        "links_sha256": sha(np.concatenate([
            np.ascontiguousarray(g.link_fluid_cell, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_second_fluid, dtype=np.int64).view(np.uint8),
            np.ascontiguousarray(g.link_direction, dtype=np.int32).view(np.uint8),
            np.ascontiguousarray(g.link_q, dtype=np.float32).view(np.uint8)])),
        "porosity_sha256": sha(np.asarray(g.porosity, dtype=np.float64)),
    }


def run_config(name):
    path = GOLDEN / f"{name}.json"
    if not path.exists():
        pytest.skip(f"{path.name} not generated")
    gold = json.loads(path.read_text())
    import paper_1507_06565_b200 as pg
    from paper_1507_06565_b200 import configs
    w = configs.ALL[name]()
    if gold.get("sphere_sha256"):
        assert sha(np.c_[w.pack.centers, w.pack.radii]) == gold["sphere_sha256"]
    g = w.geometry()
    gh = geometry_hashes(g)
    for k, v in gh.items():
        assert v == gold["geometry"][k], f"geometry {k} differs from the reference voxelize()"
    assert g.n_links == gold["geometry"]["n_links"]
    assert g.q_fallback_count == gold["geometry"]["q_fallback_count"]
    sim = configs.make_simulation(w, g)
    sim.step(gold["steps"])
    assert sim.steps_done == gold["steps"]
    nx, ny, nz = w.dims
    fluid = g.flags.reshape(nz, ny, nx) == 0
    st = gold["state"]
    f = sim.get_pdfs()
    ff = f[:, fluid]
    del f
    # tolerance diagnostics first (so a mismatch reports its size)
    fmax = float.fromhex(st["pdf_absmax"])
    samp = ff[np.array(st["sample_k"]), np.searchsorted(np.nonzero(fluid.ravel())[0],
                                                        np.array(st["sample_cell"]))]
    err = np.abs(samp - unhex(st["sample_value"])).max() / fmax
    assert err <= TOL, f"sampled PDFs differ by {err:.3e} (relative to max)"
    sums = np.array([math.fsum(ff[k]) for k in range(19)])
    np.testing.assert_allclose(sums, unhex(st["pdf_k_sums"]), rtol=0,
                               atol=TOL * fmax * ff.shape[1])
    bitwise_pdfs = sha(ff) == st["pdf_sha256"]
    del ff
    d, ux, uy, uz = sim.macroscopic_fields()
    for n, a in (("drho", d), ("ux", ux), ("uy", uy), ("uz", uz)):
        v = a[fluid]
        vmax = max(float.fromhex(st[f"{n}_absmax"]), 1e-300)
        e = np.abs(v[np.searchsorted(np.nonzero(fluid.ravel())[0], np.array(st["sample_cell"]))]
                   - unhex(st[f"{n}_sample"])).max() / vmax
        assert e <= TOL, f"{n} differs by {e:.3e}"
        assert sha(v) == st[f"{n}_sha256"], f"{n} not bit-identical (within {e:.1e})"
    prof = sim.planar_profile()
    np.testing.assert_array_equal(prof.z, unhex(st["profile_z"]))
    us = unhex(st["profile_u_superficial"])
    assert np.abs(prof.u_superficial - us).max() <= TOL * np.abs(us).max()
    assert [float(x).hex() for x in prof.u_superficial] == st["profile_u_superficial"]
    assert [float(x).hex() for x in prof.u_intrinsic] == st["profile_u_intrinsic"]
    assert sim.max_speed() == float.fromhex(st["max_speed"])
    assert bitwise_pdfs, "PDFs within tolerance but not bit-identical"


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_config_matches_reference(gpu, name):
    run_config(name)


@pytest.mark.slow
def test_c4_matches_reference(gpu):
    run_config("C4")
