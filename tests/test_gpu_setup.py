"""pgpu_create's device-side link setup (csrc/setup.cu): the link list must
close exactly the fluid->non-fluid directions of the flag field
(geometry.cpp:574-591), CLI second_fluid must be x - e_k
(geometry.cpp:595-602), and any violation is a ConfigError, never a silent
misread.  Valid geometries are exercised by every parity test."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _geom(pg):
    rng = np.random.default_rng(5)
    dims = (24, 12, 16)
    c = np.c_[rng.uniform(0, 24, 5), rng.uniform(0, 12, 5), rng.uniform(2, 10, 5)]
    pack = pg.SpherePack(c, rng.uniform(2.0, 4.0, 5), (24.0, 12.0, 16.0))
    return pg.voxelize(pack, dims, (True, True, False), True, True)


def _copy(g, **over):
    import dataclasses

    fields = {f.name: getattr(g, f.name) for f in dataclasses.fields(g)}
    for k in ("link_fluid_cell", "link_second_fluid", "link_direction", "link_q", "link_moving"):
        fields[k] = np.array(fields[k], copy=True)
    fields.update(over)
    return type(g)(**fields)


def _create(pg, g, scheme=1):
    p = pg.relaxation_from_magic(0.1, 3.0 / 16.0)
    return pg.Simulation.from_params(g, p, pg.WallScheme(scheme))


def test_valid_geometry_counts(gpu):
    pg = gpu
    g = _geom(pg)
    sim = _create(pg, g)
    assert sim.fluid_cells == g.fluid_cells
    assert sim.cli_fallback_count == int((g.link_second_fluid == -1).sum())
    assert np.array_equal(sim.flags().reshape(-1), g.flags)


@pytest.mark.parametrize("case,msg", [
    ("missing", "do not match the fluid->non-fluid"),
    ("extra", "do not match the fluid->non-fluid"),
    ("duplicate", "duplicate boundary link"),
    ("direction", "direction must be in 1..18"),
    ("solid_cell", "non-fluid or out-of-range cell"),
    ("out_of_range", "non-fluid or out-of-range cell"),
    ("fluid_neighbour", "points to a fluid neighbour"),
    ("second_wrong", "second_fluid must be the cell"),
    ("second_not_fluid", "second_fluid is not a fluid cell"),
])
def test_invalid_links_raise(gpu, case, msg):
    pg = gpu
    g = _geom(pg)
    lf, ls, ld = g.link_fluid_cell, g.link_second_fluid, g.link_direction
    i = int(np.flatnonzero(ls >= 0)[3])
    if case == "missing":
        bad = _copy(g, link_fluid_cell=lf[1:], link_second_fluid=ls[1:], link_direction=ld[1:],
                    link_q=g.link_q[1:], link_moving=g.link_moving[1:])
    elif case == "extra":
        bad = _copy(g, link_fluid_cell=np.r_[lf, lf[:1]], link_second_fluid=np.r_[ls, ls[:1]],
                    link_direction=np.r_[ld, ld[:1]], link_q=np.r_[g.link_q, g.link_q[:1]],
                    link_moving=np.r_[g.link_moving, g.link_moving[:1]])
    else:
        bad = _copy(g)
        if case == "duplicate":
            bad.link_fluid_cell[i + 1] = lf[i]
            bad.link_direction[i + 1] = ld[i]
        elif case == "direction":
            bad.link_direction[i] = 19
        elif case == "solid_cell":
            bad.link_fluid_cell[i] = int(np.flatnonzero(g.flags != 0)[0])
        elif case == "out_of_range":
            bad.link_fluid_cell[i] = g.cells + 5
        elif case == "fluid_neighbour":
            # a direction of the same cell whose wall-side neighbour is fluid
            c = int(lf[i])
            used = set(int(d) for d in ld[lf == c])
            bad.link_direction[i] = next(k for k in range(1, 19) if k not in used)
        elif case == "second_wrong":
            bad.link_second_fluid[i] = ls[i] + 1 if g.flags[ls[i] + 1] == 0 else ls[i] - 1
        elif case == "second_not_fluid":
            j = int(np.flatnonzero(ls == -1)[0])
            bad.link_second_fluid[j] = 0
    with pytest.raises(pg.ConfigError, match=msg):
        _create(pg, bad)


def test_sbb_scheme_ignores_second_fluid(gpu):
    """SBB never reads second_fluid (boundary.cpp:19-25), so it is not validated."""
    pg = gpu
    g = _geom(pg)
    bad = _copy(g)
    bad.link_second_fluid[:] = -1
    sim = _create(pg, bad, scheme=0)
    ref = _create(pg, g, scheme=0)
    sim.step(7)
    ref.step(7)
    assert np.array_equal(sim.get_pdfs(), ref.get_pdfs())


def test_staged_upload_large_arrays(gpu):
    """Arrays of >= 32 MB go through the pinned-chunk uploader (staging.h):
    a 256x256x520 flag field (34 MB) and ~4.3 M links (> 32 MB per link
    array) must arrive intact -- the device-built cell words reproduce the
    flags byte for byte and the link list passes the exact validation."""
    pg = gpu
    rng = np.random.default_rng(11)
    dims = (256, 256, 520)
    n = 2600
    c = np.c_[rng.uniform(0, dims[0], n), rng.uniform(0, dims[1], n), rng.uniform(1, 519, n)]
    pack = pg.SpherePack(c, rng.uniform(3.0, 6.0, n), tuple(float(d) for d in dims))
    g = pg.voxelize(pack, dims, (True, True, False), True, True)
    assert g.flags.nbytes >= 32 << 20 and g.n_links * 8 >= 32 << 20
    sim = _create(pg, g)
    assert sim.fluid_cells == g.fluid_cells
    assert np.array_equal(sim.flags().reshape(-1), np.asarray(g.flags).reshape(-1))
