"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrappers of
  * oracle/liboracle.so          -- plain-C restatement of the reference hot path
                                    (oracle/porolb_oracle.c), and
  * oracle/_ref/libporolb_ref.so -- the reference itself, compiled from its own
                                    sources by oracle/Makefile (when present).
Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs
may import this module, and only as the checker or the timed CPU baseline;
the product (paper_1507_06565_b200) never does.

Geometries are exchanged as ``OGeom`` (plain numpy fields named like the
reference VoxelGeometry, geometry.hpp:62-73).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libporolb_ref.so"

i32, i64, u8, f32, f64 = C.c_int32, C.c_int64, C.c_uint8, C.c_float, C.c_double
P = C.POINTER
vp = C.c_void_p
Q = 19


def _p(a, t):
    return a.ctypes.data_as(P(t))


def _v3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def _i3(v):
    return (C.c_int * 3)(*[int(x) for x in v])


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


@dataclass
class OGeom:
    dims: tuple
    periodic: tuple
    flags: np.ndarray
    link_fluid_cell: np.ndarray
    link_second_fluid: np.ndarray
    link_direction: np.ndarray
    link_q: np.ndarray
    link_moving: np.ndarray
    porosity: np.ndarray
    fluid_cells: int
    q_fallback_count: int = 0
    wall_plane_lo: Optional[float] = None
    wall_plane_hi: Optional[float] = None

    @property
    def cells(self) -> int:
        return int(np.prod(self.dims))

    @property
    def n_links(self) -> int:
        return int(self.link_fluid_cell.size)


def _pack_arrays(centers, radii):
    c = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
    cols = [np.ascontiguousarray(c[:, i]) for i in range(3)]
    r = np.ascontiguousarray(radii, dtype=np.float64)
    return cols, r


# ============================================================================
# the reference, compiled from its own sources
# ============================================================================
class RefLib:
    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_sim_max_speed.restype = f64
        L.ref_sim_steps_done.restype = i64
        L.ref_geometry_free.argtypes = [vp]
        L.ref_sim_free.argtypes = [vp]
        L.ref_sim_step.argtypes = [vp, i64]
        L.ref_sim_max_speed.argtypes = [vp]
        L.ref_sim_steps_done.argtypes = [vp]
        L.ref_sim_cli_fallbacks.argtypes = [vp]
        L.ref_sim_get_pdfs.argtypes = [vp, P(f64)]
        L.ref_sim_set_pdfs.argtypes = [vp, P(f64)]
        L.ref_geometry_info.argtypes = [vp, P(i64), P(f64)]
        L.ref_geometry_copy.argtypes = [vp, P(u8), P(f64), P(i64), P(i64), P(i32), P(f32), P(u8)]
        L.ref_sim_macroscopic_fields.argtypes = [vp, P(f64), P(f64), P(f64), P(f64)]
        L.ref_sim_planar_profile.argtypes = [vp, C.c_int, P(C.c_int)] + [P(f64)] * 6
        L.ref_sim_set_porous.argtypes = [vp, C.c_int, P(f64), P(f64), P(f64), P(f64), f64,
                                         C.c_int]
        L.ref_sim_create.argtypes = [vp, f64, f64, f64, f64, f64, P(f64), C.c_int, P(vp)]
        L.ref_sim_set_body_force.argtypes = [vp, P(f64)]
        L.ref_sim_set_lid_velocity.argtypes = [vp, P(f64)]
        L.ref_sim_initialize_equilibrium.argtypes = [vp, f64, P(f64)]
        L.ref_sim_macroscopic.argtypes = [vp, i64, P(f64), P(f64)]
        L.ref_run_to_steady_state.argtypes = [vp, f64, C.c_int, i64, f64, P(f64)]
        L.ref_voxelize.argtypes = [i64, P(f64), P(f64), P(f64), P(f64), P(f64), f64, P(C.c_int),
                                   P(C.c_int), C.c_int, C.c_int, f64, P(vp)]
        L.ref_make_box_geometry.argtypes = [P(C.c_int), P(C.c_int), C.c_int, C.c_int, P(vp)]
        L.ref_geometry_from_arrays.argtypes = [P(C.c_int), P(C.c_int), P(u8), i64, P(i64), P(i64),
                                               P(i32), P(f32), P(u8), P(f64), i64, C.c_int, f64,
                                               C.c_int, f64, P(vp)]
        L.ref_relaxation_from_magic.argtypes = [f64, f64, P(f64), P(f64)]
        L.ref_equilibrium.argtypes = [f64, P(f64), f64, P(f64)]
        L.ref_trt_collide.argtypes = [P(f64), f64, f64, f64, P(f64), P(f64)]
        L.ref_apply_link.argtypes = [C.c_int, P(C.c_int), P(f64), i64, i64, C.c_int, f32, P(f64),
                                     f64, P(f64)]
        L.ref_kozeny_carman.argtypes = [C.c_int, P(f64), f64, f64, P(f64)]
        L.ref_make_glbm_params.argtypes = [C.c_int, P(f64), P(f64), f64, f64, f64, C.c_int, f64,
                                           P(f64), P(f64)]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_glbm_equilibrium.argtypes = [f64, P(f64), f64, f64, P(f64)]
        L.ref_resolve_drive.argtypes = [C.c_int, P(f64), C.c_int, f64, P(f64)]
        L.ref_stream.argtypes = [P(C.c_int), P(C.c_int), P(u8), P(f64), P(f64)]
        L.ref_porosity_profile.argtypes = [vp, P(f64), P(f64)]
        cs = C.c_char_p
        L.ref_format_double.argtypes = [f64, cs, C.c_int]
        L.ref_write_profile_csv.argtypes = [cs, C.c_int] + [P(f64)] * 4 + [C.c_int, P(f64), P(f64)]
        L.ref_read_profile_csv.argtypes = [cs, C.c_int, P(C.c_int)] + [P(f64)] * 6
        L.ref_write_comparison_csv.argtypes = [cs, C.c_int, P(f64), P(f64), cs, C.c_int, P(f64),
                                               P(f64), cs]
        L.ref_write_report.argtypes = [cs, C.c_int, P(cs), P(cs)]
        L.ref_write_vtk.argtypes = [cs, vp]
        L.ref_write_sphere_csv.argtypes = [cs, i64] + [P(f64)] * 5 + [f64, C.c_uint64]
        L.ref_read_sphere_csv.argtypes = [cs, i64, P(i64)] + [P(f64)] * 5 + [P(C.c_uint64)]
        L.ref_write_voxel_file.argtypes = [cs, vp]
        L.ref_read_voxel_file.argtypes = [cs, P(vp)]

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def set_threads(self, n: int) -> int:
        return int(self.lib.ref_set_threads(int(n)))

    # -- lattice ----------------------------------------------------------
    def relaxation_from_magic(self, nu, lam):
        wp, wm = C.c_double(), C.c_double()
        self._check(self.lib.ref_relaxation_from_magic(nu, lam, C.byref(wp), C.byref(wm)))
        return wp.value, wm.value

    def equilibrium(self, drho, u, rho0=1.0):
        out = np.zeros(Q)
        self._check(self.lib.ref_equilibrium(drho, _v3(u), rho0, _p(out, f64)))
        return out

    def trt_collide(self, f, wp, wm, rho0, g):
        fi = np.ascontiguousarray(f, dtype=np.float64)
        out = np.zeros(Q)
        self._check(self.lib.ref_trt_collide(_p(fi, f64), wp, wm, rho0, _v3(g), _p(out, f64)))
        return out

    def apply_link(self, kind, dims, cur, fluid_cell, second_fluid, direction, q, u_wall=(0, 0, 0),
                   rho0=1.0):
        c = np.ascontiguousarray(cur, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.ref_apply_link(kind, _i3(dims), _p(c, f64), fluid_cell, second_fluid,
                                            direction, q, _v3(u_wall), rho0, C.byref(out)))
        return out.value

    def glbm_equilibrium(self, drho, u, eps, rho0=1.0):
        out = np.zeros(Q)
        self._check(self.lib.ref_glbm_equilibrium(drho, _v3(u), eps, rho0, _p(out, f64)))
        return out

    def resolve_drive(self, mode, magnitude, stream_axis=0, channel_length=0.0):
        g = np.zeros(3)
        self._check(self.lib.ref_resolve_drive(int(mode), _v3(magnitude), int(stream_axis),
                                               float(channel_length), _p(g, f64)))
        return tuple(g)

    def stream(self, cur, nxt, flags, periodic):
        """free stream() in place on (19, nz, ny, nx) buffers (swap semantics)."""
        dims = cur.shape[1:][::-1]
        fl = np.ascontiguousarray(flags, dtype=np.uint8).reshape(-1)
        self._check(self.lib.ref_stream(_i3(dims), _i3(periodic), _p(fl, u8), _p(cur, f64),
                                        _p(nxt, f64)))

    def porosity_profile(self, geom):
        h = self.geometry_handle(geom)
        z, eps = np.zeros(geom.dims[2]), np.zeros(geom.dims[2])
        try:
            self._check(self.lib.ref_porosity_profile(h, _p(z, f64), _p(eps, f64)))
        finally:
            self.lib.ref_geometry_free(h)
        return z, eps

    def kozeny_carman(self, eps, d, threshold=0.999):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        K = np.zeros_like(e)
        self._check(self.lib.ref_kozeny_carman(e.size, _p(e, f64), d, threshold, _p(K, f64)))
        return K

    def make_glbm_params(self, eps, K, cf, nu, lam, mode, J=1.0):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        k = np.ascontiguousarray(K, dtype=np.float64)
        wp, wm = np.zeros_like(e), np.zeros_like(e)
        self._check(self.lib.ref_make_glbm_params(e.size, _p(e, f64), _p(k, f64), cf, nu, lam,
                                                  mode, J, _p(wp, f64), _p(wm, f64)))
        return wp, wm

    # -- geometry -----------------------------------------------------------
    def _read_geometry(self, h) -> OGeom:
        info = np.zeros(5, dtype=np.int64)
        planes = np.zeros(2)
        self.lib.ref_geometry_info(h, _p(info, i64), _p(planes, f64))
        return info, planes

    def _geom_from_handle(self, h, dims, periodic) -> OGeom:
        info, planes = self._read_geometry(h)
        n = int(info[0])
        cells = int(np.prod(dims))
        flags = np.zeros(cells, dtype=np.uint8)
        por = np.zeros(dims[2])
        lf = np.zeros(n, dtype=np.int64)
        ls = np.zeros(n, dtype=np.int64)
        ld = np.zeros(n, dtype=np.int32)
        lq = np.zeros(n, dtype=np.float32)
        lm = np.zeros(n, dtype=np.uint8)
        self.lib.ref_geometry_copy(h, _p(flags, u8), _p(por, f64), _p(lf, i64), _p(ls, i64),
                                   _p(ld, i32), _p(lq, f32), _p(lm, u8))
        return OGeom(tuple(dims), tuple(bool(p) for p in periodic), flags, lf, ls, ld, lq, lm,
                     por, int(info[1]), int(info[2]),
                     float(planes[0]) if info[3] else None, float(planes[1]) if info[4] else None)

    def voxelize(self, centers, radii, box, dims, periodic=(True, True, False), wall_lo=False,
                 wall_hi=False, plate_z=0.0, q_clamp_min=0.05) -> OGeom:
        cols, r = _pack_arrays(centers, radii)
        h = vp()
        self._check(self.lib.ref_voxelize(r.size, _p(cols[0], f64), _p(cols[1], f64),
                                          _p(cols[2], f64), _p(r, f64), _v3(box), plate_z,
                                          _i3(dims), _i3(periodic), int(wall_lo), int(wall_hi),
                                          q_clamp_min, C.byref(h)))
        try:
            return self._geom_from_handle(h, dims, periodic)
        finally:
            self.lib.ref_geometry_free(h)

    def make_box_geometry(self, dims, periodic=(True, True, False), wall_lo=False,
                          wall_hi=False) -> OGeom:
        h = vp()
        self._check(self.lib.ref_make_box_geometry(_i3(dims), _i3(periodic), int(wall_lo),
                                                   int(wall_hi), C.byref(h)))
        try:
            return self._geom_from_handle(h, dims, periodic)
        finally:
            self.lib.ref_geometry_free(h)

    def geometry_handle(self, g) -> vp:
        """VoxelGeometry owned by the reference library, built from arrays."""
        flags = np.ascontiguousarray(g.flags, dtype=np.uint8)
        lf = np.ascontiguousarray(g.link_fluid_cell, dtype=np.int64)
        ls = np.ascontiguousarray(g.link_second_fluid, dtype=np.int64)
        ld = np.ascontiguousarray(g.link_direction, dtype=np.int32)
        lq = np.ascontiguousarray(g.link_q, dtype=np.float32)
        lm = np.ascontiguousarray(g.link_moving, dtype=np.uint8)
        por = np.ascontiguousarray(g.porosity, dtype=np.float64)
        h = vp()
        self._check(self.lib.ref_geometry_from_arrays(
            _i3(g.dims), _i3(g.periodic), _p(flags, u8), lf.size, _p(lf, i64), _p(ls, i64),
            _p(ld, i32), _p(lq, f32), _p(lm, u8), _p(por, f64), int(g.fluid_cells),
            int(g.wall_plane_lo is not None), float(g.wall_plane_lo or 0.0),
            int(g.wall_plane_hi is not None), float(g.wall_plane_hi or 0.0), C.byref(h)))
        return h

    def simulation(self, geom, nu, wp, wm, lam, g, scheme, rho0=1.0) -> "RefSim":
        return RefSim(self, geom, nu, wp, wm, lam, g, scheme, rho0)

    # -- file formats (io.cpp) ---------------------------------------------------
    def format_double(self, v) -> str:
        buf = C.create_string_buffer(64)
        self._check(self.lib.ref_format_double(float(v), buf, 64))
        return buf.value.decode()

    def write_profile_csv(self, path, z, us, ui, eps, un, meta):
        cols = [np.ascontiguousarray(c, dtype=np.float64) for c in (z, us, ui, eps, un)]
        m = np.asarray(meta, dtype=np.float64)
        self._check(self.lib.ref_write_profile_csv(
            str(path).encode(), cols[0].size, *[_p(c, f64) for c in cols[:4]], cols[4].size,
            _p(cols[4], f64), _p(m, f64)))

    def read_profile_csv(self, path):
        counts = (C.c_int * 2)()
        meta = np.zeros(8)
        null = P(f64)()
        self._check(self.lib.ref_read_profile_csv(str(path).encode(), 0, counts, null, null, null,
                                                  null, null, _p(meta, f64)))
        n = counts[0]
        b = [np.zeros(max(n, 1)) for _ in range(5)]
        self._check(self.lib.ref_read_profile_csv(str(path).encode(), n, counts,
                                                  *[_p(x, f64) for x in b], _p(meta, f64)))
        return dict(z=b[0][:n], u_superficial=b[1][:n], u_intrinsic=b[2][:n], epsilon=b[3][:n],
                    u_normalized=b[4][:counts[1]], meta=meta)

    def write_comparison_csv(self, path, za, ua, name_a, zb, ub, name_b):
        a = [np.ascontiguousarray(c, dtype=np.float64) for c in (za, ua, zb, ub)]
        self._check(self.lib.ref_write_comparison_csv(
            str(path).encode(), a[0].size, _p(a[0], f64), _p(a[1], f64), name_a.encode(),
            a[2].size, _p(a[2], f64), _p(a[3], f64), name_b.encode()))

    def write_report(self, path, entries):
        n = len(entries)
        keys = (C.c_char_p * max(n, 1))(*[str(k).encode() for k, _ in entries])
        vals = (C.c_char_p * max(n, 1))(*[str(v).encode() for _, v in entries])
        self._check(self.lib.ref_write_report(str(path).encode(), n, keys, vals))

    def write_sphere_csv(self, path, centers, radii, box, plate_z=0.0, seed=0):
        cols, r = _pack_arrays(centers, radii)
        self._check(self.lib.ref_write_sphere_csv(
            str(path).encode(), r.size, _p(cols[0], f64), _p(cols[1], f64), _p(cols[2], f64),
            _p(r, f64), _v3(box), float(plate_z), int(seed)))

    def read_sphere_csv(self, path):
        n = C.c_int64()
        extra = np.zeros(5)
        seed = C.c_uint64()
        null = P(f64)()
        self._check(self.lib.ref_read_sphere_csv(str(path).encode(), 0, C.byref(n), null, null,
                                                 null, null, _p(extra, f64), C.byref(seed)))
        k = n.value
        b = [np.zeros(max(k, 1)) for _ in range(4)]
        self._check(self.lib.ref_read_sphere_csv(str(path).encode(), k, C.byref(n),
                                                 *[_p(x, f64) for x in b], _p(extra, f64),
                                                 C.byref(seed)))
        return dict(centers=np.stack([x[:k] for x in b[:3]], axis=1), radii=b[3][:k],
                    box=tuple(extra[:3]), bottom_plate_z=extra[3], achieved_height=extra[4],
                    seed=int(seed.value))

    def write_voxel_file(self, path, geom):
        h = self.geometry_handle(geom)
        try:
            self._check(self.lib.ref_write_voxel_file(str(path).encode(), h))
        finally:
            self.lib.ref_geometry_free(h)

    def read_voxel_file(self, path) -> OGeom:
        h = vp()
        self._check(self.lib.ref_read_voxel_file(str(path).encode(), C.byref(h)))
        try:
            with open(path, "rb") as f:  # dims/periodic from the header
                head = f.readline().split()
            dims = tuple(int(x) for x in head[2:5])
            periodic = tuple(int(x) != 0 for x in head[5:8])
            return self._geom_from_handle(h, dims, periodic)
        finally:
            self.lib.ref_geometry_free(h)


class RefSim:
    """porolb::Simulation from the reference sources (simulation.cpp:80-434)."""

    def __init__(self, ref: RefLib, geom, nu, wp, wm, lam, g, scheme, rho0=1.0):
        self.ref = ref
        self.dims = tuple(geom.dims)
        self.cells = int(np.prod(self.dims))
        self.flags = np.ascontiguousarray(geom.flags, dtype=np.uint8)
        gh = ref.geometry_handle(geom)
        self.h = vp()
        try:
            ref._check(ref.lib.ref_sim_create(gh, nu, wp, wm, lam, rho0, _v3(g), int(scheme),
                                              C.byref(self.h)))
        finally:
            ref.lib.ref_geometry_free(gh)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.ref.lib.ref_sim_free(self.h)
            self.h = vp()

    def step(self, n=1):
        self.ref._check(self.ref.lib.ref_sim_step(self.h, int(n)))

    @property
    def steps_done(self):
        return int(self.ref.lib.ref_sim_steps_done(self.h))

    @property
    def cli_fallback_count(self):
        return int(self.ref.lib.ref_sim_cli_fallbacks(self.h))

    def get_pdfs(self):
        out = np.empty((Q, self.dims[2], self.dims[1], self.dims[0]))
        self.ref.lib.ref_sim_get_pdfs(self.h, _p(out, f64))
        return out

    def set_pdfs(self, f):
        a = np.ascontiguousarray(f, dtype=np.float64)
        self.ref.lib.ref_sim_set_pdfs(self.h, _p(a, f64))

    def set_body_force(self, g):
        self.ref._check(self.ref.lib.ref_sim_set_body_force(self.h, _v3(g)))

    def set_lid_velocity(self, u):
        self.ref._check(self.ref.lib.ref_sim_set_lid_velocity(self.h, _v3(u)))

    def set_porous(self, eps, K, wp, wm, cf=0.0, eps_in_eq=True):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (eps, K, wp, wm)]
        self.ref._check(self.ref.lib.ref_sim_set_porous(self.h, arrs[0].size,
                                                        *[_p(a, f64) for a in arrs], cf,
                                                        int(eps_in_eq)))

    def initialize_equilibrium(self, drho, u):
        self.ref._check(self.ref.lib.ref_sim_initialize_equilibrium(self.h, drho, _v3(u)))

    def macroscopic(self, cell):
        d = C.c_double()
        u = np.zeros(3)
        self.ref._check(self.ref.lib.ref_sim_macroscopic(self.h, int(cell), C.byref(d),
                                                         _p(u, f64)))
        return d.value, u

    def macroscopic_fields(self):
        nx, ny, nz = self.dims
        outs = [np.zeros((nz, ny, nx)) for _ in range(4)]
        self.ref._check(self.ref.lib.ref_sim_macroscopic_fields(self.h,
                                                                *[_p(o, f64) for o in outs]))
        return tuple(outs)

    def planar_profile(self, axis=0):
        nz = self.dims[2]
        bufs = [np.zeros(nz) for _ in range(5)]
        meta = np.zeros(8)
        n = C.c_int()
        self.ref._check(self.ref.lib.ref_sim_planar_profile(self.h, axis, C.byref(n),
                                                            *[_p(b, f64) for b in bufs],
                                                            _p(meta, f64)))
        k = n.value
        return dict(z=bufs[0][:k], u_superficial=bufs[1][:k], u_intrinsic=bufs[2][:k],
                    epsilon=bufs[3][:k], u_normalized=bufs[4][:k], u_max=meta[0],
                    height=meta[1], z0=meta[2], nu=meta[3], body_force=tuple(meta[4:7]),
                    stream_axis=int(meta[7]))

    def max_speed(self):
        return float(self.ref.lib.ref_sim_max_speed(self.h))

    def write_vtk(self, path):
        self.ref._check(self.ref.lib.ref_write_vtk(str(path).encode(), self.h))

    def run_to_steady_state(self, tol=1e-8, check_interval=1000, max_steps=2000000,
                            max_speed=0.3 / 1.7320508075688772):
        st = np.zeros(6)
        self.ref._check(self.ref.lib.ref_run_to_steady_state(self.h, tol, check_interval,
                                                             max_steps, max_speed, _p(st, f64)))
        return dict(steps=int(st[0]), mlups=st[1], seconds=st[2], converged=bool(st[3]),
                    residual=st[4], cli_fallbacks=int(st[5]))


# ============================================================================
# the C restatement
# ============================================================================
class OracleLib:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_relaxation_from_magic.argtypes = [f64, f64, P(f64), P(f64)]
        L.orc_equilibrium.argtypes = [f64, P(f64), f64, P(f64)]
        L.orc_moments.argtypes = [P(f64), f64, P(f64), P(f64)]
        L.orc_trt_collide.argtypes = [P(f64), f64, f64, f64, P(f64), P(f64)]
        L.orc_collide_core.argtypes = [i64, P(u8), P(f64), f64, f64, f64, P(f64)]
        L.orc_collide_glbm.argtypes = [i64, i64, P(u8), P(f64), f64, f64, P(f64), P(f64), P(f64),
                                       P(f64), P(f64), f64, C.c_int]
        L.orc_stream_pass.argtypes = [P(C.c_int), P(C.c_int), P(u8), P(f64), P(f64)]
        L.orc_apply_links.argtypes = [i64, i64, P(i64), P(i64), P(i32), P(f32), P(u8), C.c_int,
                                      P(f64), f64, P(f64), P(f64)]
        L.orc_glbm_force_and_velocity.argtypes = [P(f64), f64, f64, f64, P(f64), f64, P(f64),
                                                  P(f64)]
        L.orc_glbm_equilibrium.argtypes = [f64, P(f64), f64, f64, P(f64)]
        L.orc_macroscopic.argtypes = [P(f64), i64, i64, f64, P(f64), f64, C.c_int, f64, f64, f64,
                                      P(f64), P(f64)]
        L.orc_glbm_all_free.argtypes = [C.c_int, P(f64), P(f64), f64]
        L.orc_planar_profile.argtypes = [P(C.c_int), P(u8), P(f64), P(f64), f64, P(f64), f64,
                                         P(f64), P(f64), f64, C.c_int, C.c_int, f64, C.c_int, f64,
                                         P(C.c_int), P(f64), P(f64), P(f64), P(f64), P(f64),
                                         P(f64)]
        L.orc_max_speed.restype = f64
        L.orc_max_speed.argtypes = [P(C.c_int), P(u8), P(f64), f64, P(f64), f64, P(f64), P(f64),
                                    f64]
        L.orc_kozeny_carman.argtypes = [C.c_int, P(f64), f64, f64, P(f64)]
        L.orc_make_glbm_params.argtypes = [C.c_int, P(f64), f64, f64, C.c_int, f64, P(f64), P(f64)]
        L.orc_voxelize.argtypes = [i64, P(f64), P(f64), P(f64), P(f64), P(f64), f64, P(C.c_int),
                                   P(C.c_int), C.c_int, C.c_int, f64, P(u8), P(f64), i64, P(i64),
                                   P(i64), P(i32), P(f32), P(u8), P(i64), P(i64), P(C.c_int)]
        L.orc_voxelize_fast.argtypes = L.orc_voxelize.argtypes
        L.orc_generate_spheres.argtypes = [C.c_int, C.c_uint64, P(f64), f64, f64, f64, f64, f64,
                                           f64, i64, i64, P(f64), P(f64), P(f64), P(f64), P(i64),
                                           P(f64)]
        L.orc_tables.argtypes = [P(C.c_int), P(f64), P(C.c_int)]

    def tables(self):
        e = np.zeros(Q * 3, dtype=np.int32)
        w = np.zeros(Q)
        o = np.zeros(Q, dtype=np.int32)
        self.lib.orc_tables(_p(e, C.c_int), _p(w, f64), _p(o, C.c_int))
        return e.reshape(Q, 3), w, o

    def relaxation_from_magic(self, nu, lam):
        wp, wm = C.c_double(), C.c_double()
        st = self.lib.orc_relaxation_from_magic(nu, lam, C.byref(wp), C.byref(wm))
        if st:
            raise OracleError(st, "relaxation rates")
        return wp.value, wm.value

    def equilibrium(self, drho, u, rho0=1.0):
        out = np.zeros(Q)
        self.lib.orc_equilibrium(drho, _v3(u), rho0, _p(out, f64))
        return out

    def moments(self, f, rho0=1.0):
        fi = np.ascontiguousarray(f, dtype=np.float64)
        d = C.c_double()
        u = np.zeros(3)
        self.lib.orc_moments(_p(fi, f64), rho0, C.byref(d), _p(u, f64))
        return d.value, u

    def trt_collide(self, f, wp, wm, rho0, g):
        fi = np.ascontiguousarray(f, dtype=np.float64)
        out = np.zeros(Q)
        st = self.lib.orc_trt_collide(_p(fi, f64), wp, wm, rho0, _v3(g), _p(out, f64))
        if st:
            raise OracleError(st, "non-finite population after collision")
        return out

    def glbm_force_and_velocity(self, mom, eps, K, cf, g, nu):
        u, F = np.zeros(3), np.zeros(3)
        st = self.lib.orc_glbm_force_and_velocity(_v3(mom), eps, K, cf, _v3(g), nu, _p(u, f64),
                                                  _p(F, f64))
        if st:
            raise OracleError(st)
        return u, F

    def kozeny_carman(self, eps, d, threshold=0.999):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        K = np.zeros_like(e)
        self.lib.orc_kozeny_carman(e.size, _p(e, f64), d, threshold, _p(K, f64))
        return K

    def make_glbm_params(self, eps, nu, lam, mode, J=1.0):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        wp, wm = np.zeros_like(e), np.zeros_like(e)
        st = self.lib.orc_make_glbm_params(e.size, _p(e, f64), nu, lam, mode, J, _p(wp, f64),
                                           _p(wm, f64))
        if st:
            raise OracleError(st)
        return wp, wm

    def voxelize(self, centers, radii, box, dims, periodic=(True, True, False), wall_lo=False,
                 wall_hi=False, plate_z=0.0, q_clamp_min=0.05, cap=None) -> OGeom:
        cols, r = _pack_arrays(centers, radii)
        cells = int(np.prod(dims))
        cap = cap if cap is not None else 18 * cells
        flags = np.zeros(cells, dtype=np.uint8)
        por = np.zeros(dims[2])
        lf = np.zeros(cap, dtype=np.int64)
        ls = np.zeros(cap, dtype=np.int64)
        ld = np.zeros(cap, dtype=np.int32)
        lq = np.zeros(cap, dtype=np.float32)
        lm = np.zeros(cap, dtype=np.uint8)
        nl, fl, qfb = C.c_int64(), C.c_int64(), C.c_int()
        st = self.lib.orc_voxelize(r.size, _p(cols[0], f64), _p(cols[1], f64), _p(cols[2], f64),
                                   _p(r, f64), _v3(box), plate_z, _i3(dims), _i3(periodic),
                                   int(wall_lo), int(wall_hi), q_clamp_min, _p(flags, u8),
                                   _p(por, f64), cap, _p(lf, i64), _p(ls, i64), _p(ld, i32),
                                   _p(lq, f32), _p(lm, u8), C.byref(nl), C.byref(fl),
                                   C.byref(qfb))
        if st:
            raise OracleError(st, "voxelize")
        n = nl.value
        return OGeom(tuple(dims), tuple(bool(p) for p in periodic), flags, lf[:n].copy(),
                     ls[:n].copy(), ld[:n].copy(), lq[:n].copy(), lm[:n].copy(), por, fl.value,
                     qfb.value, 1.0 if wall_lo else None,
                     float(dims[2] - 1) if wall_hi else None)

    def voxelize_fast(self, centers, radii, box, dims, periodic=(True, True, False),
                      wall_lo=False, wall_hi=False, plate_z=0.0, q_clamp_min=0.05) -> OGeom:
        """orc_voxelize_fast: grid-accelerated, OpenMP; byte-identical output."""
        cols, r = _pack_arrays(centers, radii)
        cells = int(np.prod(dims))
        flags = np.zeros(cells, dtype=np.uint8)
        por = np.zeros(dims[2])
        nl, fl, qfb = C.c_int64(), C.c_int64(), C.c_int()
        cap = 0
        for _ in range(2):  # first call sizes the link arrays (status 6)
            lf = np.zeros(cap, dtype=np.int64)
            ls = np.zeros(cap, dtype=np.int64)
            ld = np.zeros(cap, dtype=np.int32)
            lq = np.zeros(cap, dtype=np.float32)
            lm = np.zeros(cap, dtype=np.uint8)
            st = self.lib.orc_voxelize_fast(
                r.size, _p(cols[0], f64), _p(cols[1], f64), _p(cols[2], f64), _p(r, f64),
                _v3(box), plate_z, _i3(dims), _i3(periodic), int(wall_lo), int(wall_hi),
                q_clamp_min, _p(flags, u8), _p(por, f64), cap, _p(lf, i64), _p(ls, i64),
                _p(ld, i32), _p(lq, f32), _p(lm, u8), C.byref(nl), C.byref(fl), C.byref(qfb))
            if st == 6 and cap == 0:
                cap = nl.value
                continue
            break
        if st:
            raise OracleError(st, "voxelize_fast")
        n = nl.value
        return OGeom(tuple(dims), tuple(bool(p) for p in periodic), flags, lf[:n], ls[:n],
                     ld[:n], lq[:n], lm[:n], por, fl.value, qfb.value,
                     1.0 if wall_lo else None, float(dims[2] - 1) if wall_hi else None)

    def generate_spheres(self, mode, seed, box, z_lo, z_hi, r_min, r_max, bed_volume,
                         target_porosity, max_attempts, capacity):
        """Harness sphere generator (mode 0 RSA, 1 Boolean); returns
        (centers (n, 3), radii (n,), analytic porosity)."""
        cx, cy, cz, r = (np.zeros(capacity) for _ in range(4))
        n, por = C.c_int64(), C.c_double()
        st = self.lib.orc_generate_spheres(int(mode), int(seed), _v3(box), z_lo, z_hi, r_min,
                                           r_max, bed_volume, target_porosity, int(max_attempts),
                                           int(capacity), _p(cx, f64), _p(cy, f64), _p(cz, f64),
                                           _p(r, f64), C.byref(n), C.byref(por))
        if st:
            raise OracleError(st, "generate_spheres")
        k = n.value
        return np.c_[cx[:k], cy[:k], cz[:k]], r[:k].copy(), por.value

    def simulation(self, geom, nu, wp, wm, g, scheme, rho0=1.0) -> "OracleSim":
        return OracleSim(self, geom, nu, wp, wm, g, scheme, rho0)


class OracleSim:
    """Simulation restated in C (reference simulation.cpp:80-434) driven from Python."""

    def __init__(self, orc: OracleLib, geom, nu, wp, wm, g, scheme, rho0=1.0):
        self.o = orc
        self.dims = tuple(int(d) for d in geom.dims)
        self.periodic = tuple(int(bool(p)) for p in geom.periodic)
        self.cells = int(np.prod(self.dims))
        self.flags = np.ascontiguousarray(geom.flags, dtype=np.uint8)
        self.lf = np.ascontiguousarray(geom.link_fluid_cell, dtype=np.int64)
        self.ls = np.ascontiguousarray(geom.link_second_fluid, dtype=np.int64)
        self.ld = np.ascontiguousarray(geom.link_direction, dtype=np.int32)
        self.lq = np.ascontiguousarray(geom.link_q, dtype=np.float32)
        self.lm = np.ascontiguousarray(geom.link_moving, dtype=np.uint8).copy()
        self.porosity = np.ascontiguousarray(geom.porosity, dtype=np.float64)
        self.lo, self.hi = geom.wall_plane_lo, geom.wall_plane_hi
        self.nu, self.wp, self.wm, self.rho0 = nu, wp, wm, rho0
        self.g = np.array(g, dtype=np.float64)
        self.scheme = int(scheme)
        self.lid = np.zeros(3)
        self.cur = np.zeros((Q, self.dims[2], self.dims[1], self.dims[0]))
        self.nxt = np.zeros_like(self.cur)
        self.glbm = None
        self.steps_done = 0

    def set_porous(self, eps, K, wp, wm, cf=0.0, eps_in_eq=True):
        self.glbm = tuple(np.ascontiguousarray(a, dtype=np.float64) for a in (eps, K, wp, wm))
        self.cf, self.eps_in_eq = float(cf), int(eps_in_eq)

    def _glbm_active(self):
        if self.glbm is None:
            return False
        e, K = self.glbm[0], self.glbm[1]
        return not self.o.lib.orc_glbm_all_free(e.size, _p(e, f64), _p(K, f64), self.cf)

    def set_lid_velocity(self, u):  # simulation.cpp:104-112
        self.lid = np.array(u, dtype=np.float64)
        plane = self.dims[0] * self.dims[1]
        z = self.lf // plane
        ez = np.array([0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1])
        self.lm[(z + ez[self.ld]) == self.dims[2] - 1] = 1

    def step(self, n=1):  # simulation.cpp:344-352
        L = self.o.lib
        for _ in range(int(n)):
            if self._glbm_active():
                e, K, wp, wm = self.glbm
                L.orc_collide_glbm(self.cells, self.dims[0] * self.dims[1], _p(self.flags, u8),
                                   _p(self.cur, f64), self.rho0, self.nu, _v3(self.g),
                                   _p(e, f64), _p(K, f64), _p(wp, f64), _p(wm, f64), self.cf,
                                   self.eps_in_eq)
            else:
                L.orc_collide_core(self.cells, _p(self.flags, u8), _p(self.cur, f64), self.wp,
                                   self.wm, self.rho0, _v3(self.g))
            L.orc_stream_pass(_i3(self.dims), _i3(self.periodic), _p(self.flags, u8),
                              _p(self.cur, f64), _p(self.nxt, f64))
            L.orc_apply_links(self.cells, self.lf.size, _p(self.lf, i64), _p(self.ls, i64),
                              _p(self.ld, i32), _p(self.lq, f32), _p(self.lm, u8), self.scheme,
                              _v3(self.lid), self.rho0, _p(self.cur, f64), _p(self.nxt, f64))
            self.cur, self.nxt = self.nxt, self.cur
            self.steps_done += 1

    def get_pdfs(self):
        return self.cur.copy()

    def set_pdfs(self, f):
        self.cur[...] = np.asarray(f, dtype=np.float64).reshape(self.cur.shape)

    def _glbm_ptrs(self):
        if self._glbm_active():
            e, K = self.glbm[0], self.glbm[1]
            return _p(e, f64), _p(K, f64), self.cf
        return None, None, 0.0

    def macroscopic_fields(self):
        nx, ny, nz = self.dims
        d = np.zeros(self.cells)
        u = np.zeros((3, self.cells))
        active = self._glbm_active()
        plane = nx * ny
        tmp_u = np.zeros(3)
        tmp_d = C.c_double()
        for c in np.nonzero(self.flags == 0)[0]:
            z = int(c // plane)
            eps = self.glbm[0][z] if active else 1.0
            K = self.glbm[1][z] if active else 0.0
            self.o.lib.orc_macroscopic(_p(self.cur, f64), self.cells, int(c), self.rho0,
                                       _v3(self.g), self.nu, int(active), eps, K,
                                       getattr(self, "cf", 0.0), C.byref(tmp_d), _p(tmp_u, f64))
            d[c] = tmp_d.value
            u[:, c] = tmp_u
        shp = (nz, ny, nx)
        return d.reshape(shp), u[0].reshape(shp), u[1].reshape(shp), u[2].reshape(shp)

    def planar_profile(self, axis=0):
        nz = self.dims[2]
        bufs = [np.zeros(nz) for _ in range(5)]
        meta = np.zeros(3)
        n = C.c_int()
        e, K, cf = self._glbm_ptrs()
        st = self.o.lib.orc_planar_profile(
            _i3(self.dims), _p(self.flags, u8), _p(self.cur, f64), _p(self.porosity, f64),
            self.rho0, _v3(self.g), self.nu, e, K, cf, axis, int(self.lo is not None),
            float(self.lo or 0.0), int(self.hi is not None), float(self.hi or 0.0), C.byref(n),
            *[_p(b, f64) for b in bufs], _p(meta, f64))
        if st:
            raise OracleError(st, "planar_profile")
        k = n.value
        return dict(z=bufs[0][:k], u_superficial=bufs[1][:k], u_intrinsic=bufs[2][:k],
                    epsilon=bufs[3][:k], u_normalized=bufs[4][:k], u_max=meta[0],
                    height=meta[1], z0=meta[2])

    def max_speed(self):
        e, K, cf = self._glbm_ptrs()
        return float(self.o.lib.orc_max_speed(_i3(self.dims), _p(self.flags, u8),
                                               _p(self.cur, f64), self.rho0, _v3(self.g),
                                               self.nu, e, K, cf))


def load_ref() -> Optional[RefLib]:
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None


def load_oracle() -> OracleLib:
    return OracleLib()
