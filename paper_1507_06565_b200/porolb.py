"""Python mirror of the reference porolb API for the time-step path, over the
C ABI of libporolb_cuda.so (include/porolb_gpu.h).

Names, argument meaning and error behaviour follow the reference's pybind
module (proj/python/bindings.cpp:45-370) and C++ headers:
  Simulation(geometry, nu, lambda_magic, body_force, scheme)   bindings.cpp:228-243
  run_to_steady(sim, tolerance, check_interval, max_steps)     bindings.cpp:245-257
  voxelize / make_box_geometry                                 geometry.hpp:76-84
  relaxation_from_magic, equilibrium, trt_collide, moments     lattice.hpp:42-61
  kozeny_carman, make_glbm_params, glbm_force_and_velocity     glbm.hpp:44-46, simulation.hpp:31-43
Exceptions: ConfigError / NumericalInstability / GeometryError (errors.hpp:9-21).
Every compute call runs on the B200 through the C ABI; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib


class ConfigError(RuntimeError):
    pass


class NumericalInstability(RuntimeError):
    pass


class GeometryError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRORS = {1: ConfigError, 2: NumericalInstability, 3: GeometryError, 4: CudaError}


def _check(status: int) -> None:
    if status != 0:
        msg = lib.pgpu_last_error().decode(errors="replace")
        exc = _ERRORS.get(status)
        if exc is None:
            raise ValueError(msg)
        raise exc(msg)


def _p(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def _vec3(v) -> "C.Array":
    return (C.c_double * 3)(*[float(x) for x in v])


class WallScheme(enum.IntEnum):
    SBB = 0
    CLI = 1


class MathMode(enum.IntEnum):
    """pgpu_math_mode (include/porolb_gpu.h): EXACT is bit-identical to the
    reference; FAST is the FMA-contracted collision (<= 1e-12 vs the reference)."""
    EXACT = 0
    FAST = 1


# pgpu_sweep_kernel (include/porolb_gpu.h), by value
SWEEP_KERNELS = ("auto", "cpipe", "tma", "units")


class GlbmViscosity(enum.IntEnum):
    Plain = 0
    Rescaled = 1
    ConstantRatio = 2


Q = 19
# lattice.cpp:13-33
VELOCITIES = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1],
                       [0, 0, -1], [1, 1, 0], [-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 0, 1],
                       [-1, 0, -1], [1, 0, -1], [-1, 0, 1], [0, 1, 1], [0, -1, -1], [0, 1, -1],
                       [0, -1, 1]], dtype=np.int32)
OPPOSITE = np.array([0] + [k + 1 if k % 2 else k - 1 for k in range(1, Q)], dtype=np.int32)
WEIGHTS = np.array([1.0 / 3.0] + [1.0 / 18.0] * 6 + [1.0 / 36.0] * 12)


# ---------------------------------------------------------------------------
# lattice-level functions
# ---------------------------------------------------------------------------
@dataclass
class FluidParams:
    """lattice.hpp:32-39"""
    nu: float = 1.0 / 6.0
    omega_plus: float = 1.0
    omega_minus: float = 1.0
    lambda_magic: float = 3.0 / 16.0
    rho0: float = 1.0
    body_force: tuple = (0.0, 0.0, 0.0)

    def to_c(self) -> _lib.FluidParams:
        return _lib.FluidParams(self.nu, self.omega_plus, self.omega_minus, self.lambda_magic,
                                self.rho0, _vec3(self.body_force))

    @staticmethod
    def from_c(p: _lib.FluidParams) -> "FluidParams":
        return FluidParams(p.nu, p.omega_plus, p.omega_minus, p.lambda_magic, p.rho0,
                           tuple(p.body_force))


def relaxation_from_magic(nu: float, lambda_magic: float) -> FluidParams:
    out = _lib.FluidParams()
    _check(lib.pgpu_relaxation_from_magic(float(nu), float(lambda_magic), C.byref(out)))
    return FluidParams.from_c(out)


def equilibrium(delta_rho: float, u, rho0: float = 1.0) -> np.ndarray:
    out = np.zeros(Q)
    _check(lib.pgpu_equilibrium(float(delta_rho), _vec3(u), float(rho0), _p(out, C.c_double)))
    return out


def glbm_equilibrium(delta_rho: float, u, eps: float, rho0: float = 1.0) -> np.ndarray:
    """simulation.cpp:68-78 (bindings.cpp:92-97)."""
    out = np.zeros(Q)
    _check(lib.pgpu_glbm_equilibrium(float(delta_rho), _vec3(u), float(eps), float(rho0),
                                     _p(out, C.c_double)))
    return out


class DriveMode(enum.IntEnum):
    """boundary.hpp:24"""
    BodyForce = 0
    PressureGradientAsForce = 1


@dataclass
class DriveSpec:
    """boundary.hpp:28-34"""
    mode: DriveMode = DriveMode.BodyForce
    magnitude: tuple = (0.0, 0.0, 0.0)
    periodic_axes: tuple = (True, True, False)
    stream_axis: int = 0
    channel_length: float = 0.0


def resolve_drive(spec: DriveSpec) -> tuple:
    """boundary.cpp:9-17: the body force G for the collision."""
    c = _lib.DriveSpec(int(spec.mode), (C.c_double * 3)(*[float(v) for v in spec.magnitude]),
                       (C.c_uint8 * 3)(*[int(bool(v)) for v in spec.periodic_axes]),
                       int(spec.stream_axis), float(spec.channel_length))
    g = (C.c_double * 3)()
    _check(lib.pgpu_resolve_drive(C.byref(c), g))
    return tuple(g)


def trt_collide(f, params: FluidParams) -> np.ndarray:
    fi = np.ascontiguousarray(f, dtype=np.float64)
    if fi.size != Q:
        raise ValueError("expected 19 population values")
    out = np.zeros(Q)
    cp = params.to_c()
    _check(lib.pgpu_trt_collide(_p(fi, C.c_double), C.byref(cp), _p(out, C.c_double)))
    return out


def kozeny_carman(eps, grain_diameter: float, free_threshold: float = 0.999) -> np.ndarray:
    e = np.ascontiguousarray(eps, dtype=np.float64)
    K = np.zeros_like(e)
    _check(lib.pgpu_kozeny_carman(e.size, _p(e, C.c_double), float(grain_diameter),
                                  float(free_threshold), _p(K, C.c_double)))
    return K


@dataclass
class GlbmPlaneParams:
    """simulation.hpp:18-27"""
    eps: np.ndarray
    permeability: np.ndarray
    omega_plus: np.ndarray
    omega_minus: np.ndarray
    forchheimer_cf: float = 0.0
    eps_in_equilibrium: bool = True


def make_glbm_params(eps, permeability, c_F: float, nu: float, lambda_magic: float,
                     mode: GlbmViscosity, J: float = 1.0) -> GlbmPlaneParams:
    e = np.ascontiguousarray(eps, dtype=np.float64)
    K = np.ascontiguousarray(permeability, dtype=np.float64)
    if e.size != K.size:
        raise ConfigError("porosity and permeability profiles must have equal length")
    wp = np.zeros_like(e)
    wm = np.zeros_like(e)
    _check(lib.pgpu_make_glbm_params(e.size, _p(e, C.c_double), _p(K, C.c_double), float(c_F),
                                     float(nu), float(lambda_magic), int(mode), float(J),
                                     _p(wp, C.c_double), _p(wm, C.c_double)))
    return GlbmPlaneParams(e.copy(), K.copy(), wp, wm, float(c_F), True)


def glbm_force_and_velocity(momentum, eps: float, K: float, c_F: float, g, nu: float):
    u = np.zeros(3)
    F = np.zeros(3)
    _check(lib.pgpu_glbm_force_and_velocity(_vec3(momentum), float(eps), float(K), float(c_F),
                                            _vec3(g), float(nu), _p(u, C.c_double),
                                            _p(F, C.c_double)))
    return u, F


# ---------------------------------------------------------------------------
# geometry
# ---------------------------------------------------------------------------
@dataclass
class SpherePack:
    """geometry.hpp:25-32: centers (N,3), radii (N,), periodic box."""
    centers: np.ndarray
    radii: np.ndarray
    box: tuple
    bottom_plate_z: float = 0.0
    seed: int = 0
    achieved_height: float = 0.0  # max over spheres of z + r (read_sphere_csv)

    def to_c(self):
        c = np.ascontiguousarray(self.centers, dtype=np.float64).reshape(-1, 3)
        cols = [np.ascontiguousarray(c[:, i]) for i in range(3)]
        r = np.ascontiguousarray(self.radii, dtype=np.float64)
        keep = (cols, r)
        pk = _lib.SpherePackC(len(r), _p(cols[0], C.c_double), _p(cols[1], C.c_double),
                              _p(cols[2], C.c_double), _p(r, C.c_double),
                              (C.c_double * 3)(*self.box), float(self.bottom_plate_z))
        return pk, keep


@dataclass
class VoxelGeometry:
    """geometry.hpp:62-73 with the link list as structure-of-arrays."""
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
    # x-slab decomposition (multi-GPU)
    slab: bool = False
    x_offset: int = 0
    global_nx: int = 0
    ghost_flags_lo: Optional[np.ndarray] = None
    ghost_flags_hi: Optional[np.ndarray] = None

    @property
    def n_links(self) -> int:
        return int(self.link_fluid_cell.size)

    @property
    def cells(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def to_c(self):
        arrs = dict(
            flags=np.ascontiguousarray(self.flags, dtype=np.uint8),
            lf=np.ascontiguousarray(self.link_fluid_cell, dtype=np.int64),
            ls=np.ascontiguousarray(self.link_second_fluid, dtype=np.int64),
            ld=np.ascontiguousarray(self.link_direction, dtype=np.int32),
            lq=np.ascontiguousarray(self.link_q, dtype=np.float32),
            lm=np.ascontiguousarray(self.link_moving, dtype=np.uint8),
            por=np.ascontiguousarray(self.porosity, dtype=np.float64),
        )
        if arrs["flags"].size != self.cells:
            raise ConfigError("flags must have nx*ny*nz entries")
        if arrs["por"].size != self.dims[2]:
            raise ConfigError("porosity must have nz entries")
        g = _lib.Geometry()
        g.dims = (C.c_int32 * 3)(*self.dims)
        g.periodic = (C.c_uint8 * 3)(*[1 if p else 0 for p in self.periodic])
        g.flags = _p(arrs["flags"], C.c_uint8)
        g.n_links = arrs["lf"].size
        g.link_fluid_cell = _p(arrs["lf"], C.c_int64)
        g.link_second_fluid = _p(arrs["ls"], C.c_int64)
        g.link_direction = _p(arrs["ld"], C.c_int32)
        g.link_q = _p(arrs["lq"], C.c_float)
        g.link_moving = _p(arrs["lm"], C.c_uint8)
        g.porosity = _p(arrs["por"], C.c_double)
        g.fluid_cells = int(self.fluid_cells)
        g.has_wall_plane_lo = int(self.wall_plane_lo is not None)
        g.has_wall_plane_hi = int(self.wall_plane_hi is not None)
        g.wall_plane_lo = float(self.wall_plane_lo or 0.0)
        g.wall_plane_hi = float(self.wall_plane_hi or 0.0)
        g.slab = int(self.slab)
        g.x_offset = int(self.x_offset)
        g.global_nx = int(self.global_nx or self.dims[0])
        if self.slab:
            arrs["glo"] = np.ascontiguousarray(self.ghost_flags_lo, dtype=np.uint8)
            arrs["ghi"] = np.ascontiguousarray(self.ghost_flags_hi, dtype=np.uint8)
            g.ghost_flags_lo = _p(arrs["glo"], C.c_uint8)
            g.ghost_flags_hi = _p(arrs["ghi"], C.c_uint8)
        return g, arrs

    def flag(self, cell: int) -> int:
        return int(self.flags[cell])


def _geometry_from_handle(h: C.c_void_p) -> VoxelGeometry:
    v = _lib.Geometry()
    qfb = C.c_int32(0)
    try:
        _check(lib.pgpu_voxel_geometry_view(h, C.byref(v), C.byref(qfb)))
        dims = tuple(int(x) for x in v.dims)
        cells = dims[0] * dims[1] * dims[2]
        n = int(v.n_links)

        def arr(ptr, count, dtype):
            if count == 0:
                return np.zeros(0, dtype=dtype)
            return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)

        geom = VoxelGeometry(
            dims=dims, periodic=tuple(bool(x) for x in v.periodic),
            flags=arr(v.flags, cells, np.uint8),
            link_fluid_cell=arr(v.link_fluid_cell, n, np.int64),
            link_second_fluid=arr(v.link_second_fluid, n, np.int64),
            link_direction=arr(v.link_direction, n, np.int32),
            link_q=arr(v.link_q, n, np.float32),
            link_moving=arr(v.link_moving, n, np.uint8),
            porosity=arr(v.porosity, dims[2], np.float64),
            fluid_cells=int(v.fluid_cells), q_fallback_count=int(qfb.value),
            wall_plane_lo=float(v.wall_plane_lo) if v.has_wall_plane_lo else None,
            wall_plane_hi=float(v.wall_plane_hi) if v.has_wall_plane_hi else None,
            slab=bool(v.slab), x_offset=int(v.x_offset), global_nx=int(v.global_nx))
        if v.slab:
            geom.ghost_flags_lo = arr(v.ghost_flags_lo, dims[1] * dims[2], np.uint8)
            geom.ghost_flags_hi = arr(v.ghost_flags_hi, dims[1] * dims[2], np.uint8)
        return geom
    finally:
        lib.pgpu_voxel_geometry_free(h)


def _opts(periodic, wall_z_lo, wall_z_hi, q_clamp_min):
    return _lib.VoxelizeOptionsC((C.c_uint8 * 3)(*[1 if p else 0 for p in periodic]),
                                 1 if wall_z_lo else 0, 1 if wall_z_hi else 0, float(q_clamp_min))


def voxelize(pack: SpherePack, dims, periodic=(True, True, False), wall_z_lo: bool = False,
             wall_z_hi: bool = False, q_clamp_min: float = 0.05) -> VoxelGeometry:
    """geometry.cpp:491-632 (bit-exact; grid-accelerated, multi-threaded)."""
    pk, _keep = pack.to_c()
    d = (C.c_int32 * 3)(*dims)
    o = _opts(periodic, wall_z_lo, wall_z_hi, q_clamp_min)
    h = C.c_void_p()
    _check(lib.pgpu_voxelize(C.byref(pk), d, C.byref(o), C.byref(h)))
    return _geometry_from_handle(h)


def voxelize_device(pack: SpherePack, dims, periodic=(True, True, False), wall_z_lo: bool = False,
                    wall_z_hi: bool = False, q_clamp_min: float = 0.05,
                    device: int = 0) -> VoxelGeometry:
    """voxelize() computed by sm_100a kernels; byte-identical output."""
    pk, _keep = pack.to_c()
    d = (C.c_int32 * 3)(*dims)
    o = _opts(periodic, wall_z_lo, wall_z_hi, q_clamp_min)
    h = C.c_void_p()
    _check(lib.pgpu_voxelize_device(C.byref(pk), d, C.byref(o), int(device), C.byref(h)))
    return _geometry_from_handle(h)


def voxelize_slab(pack: SpherePack, dims, x0: int, x1: int, periodic=(True, True, False),
                  wall_z_lo: bool = False, wall_z_hi: bool = False,
                  q_clamp_min: float = 0.05) -> VoxelGeometry:
    """Columns [x0, x1) of voxelize(pack, dims, ...) plus ghost-column flags."""
    pk, _keep = pack.to_c()
    d = (C.c_int32 * 3)(*dims)
    o = _opts(periodic, wall_z_lo, wall_z_hi, q_clamp_min)
    h = C.c_void_p()
    _check(lib.pgpu_voxelize_slab(C.byref(pk), d, C.byref(o), int(x0), int(x1), C.byref(h)))
    return _geometry_from_handle(h)


def make_box_geometry(dims, periodic=(True, True, False), wall_z_lo: bool = False,
                      wall_z_hi: bool = False) -> VoxelGeometry:
    """geometry.cpp:634-640"""
    d = (C.c_int32 * 3)(*dims)
    o = _opts(periodic, wall_z_lo, wall_z_hi, 0.05)
    h = C.c_void_p()
    _check(lib.pgpu_make_box_geometry(d, C.byref(o), C.byref(h)))
    return _geometry_from_handle(h)


def generate_spheres(mode: int, seed: int, box, z_lo: float, z_hi: float, r_min: float,
                     r_max: float, bed_volume: float, target_porosity: float,
                     max_attempts: int, capacity: int = 2_000_000):
    """Seeded RSA (mode 0) or Boolean (mode 1) sphere lists; see porolb_gpu.h."""
    cx, cy, cz, r = (np.zeros(capacity) for _ in range(4))
    n = C.c_int64(0)
    por = C.c_double(0.0)
    _check(lib.pgpu_generate_spheres(int(mode), int(seed), (C.c_double * 3)(*box), float(z_lo),
                                     float(z_hi), float(r_min), float(r_max), float(bed_volume),
                                     float(target_porosity), int(max_attempts), int(capacity),
                                     _p(cx, C.c_double), _p(cy, C.c_double), _p(cz, C.c_double),
                                     _p(r, C.c_double), C.byref(n), C.byref(por)))
    k = n.value
    centers = np.stack([cx[:k], cy[:k], cz[:k]], axis=1)
    return SpherePack(centers, r[:k].copy(), tuple(box), 0.0, int(seed)), float(por.value)


# ---------------------------------------------------------------------------
# profiles / stats
# ---------------------------------------------------------------------------
@dataclass
class ProfileData:
    """profile.hpp:12-34"""
    z: np.ndarray = field(default_factory=lambda: np.zeros(0))
    u_superficial: np.ndarray = field(default_factory=lambda: np.zeros(0))
    u_intrinsic: np.ndarray = field(default_factory=lambda: np.zeros(0))
    epsilon: np.ndarray = field(default_factory=lambda: np.zeros(0))
    u_normalized: np.ndarray = field(default_factory=lambda: np.zeros(0))
    u_max: float = 0.0
    height: float = 0.0
    z0: float = 0.0
    nu: float = 0.0
    body_force: tuple = (0.0, 0.0, 0.0)
    stream_axis: int = 0

    def __len__(self) -> int:
        return int(self.z.size)


@dataclass
class RunStats:
    """simulation.hpp:125-132"""
    steps: int = 0
    mlups: float = 0.0
    seconds: float = 0.0
    converged: bool = False
    residual: float = 0.0
    cli_fallbacks: int = 0


def porosity_profile(geometry: "VoxelGeometry") -> ProfileData:
    """geometry.cpp:642-661: per-plane porosity from the flags, zero velocities."""
    g, keep = geometry.to_c()
    nz = int(geometry.dims[2])
    z, eps = np.zeros(nz), np.zeros(nz)
    _check(lib.pgpu_porosity_profile(C.byref(g), _p(z, C.c_double), _p(eps, C.c_double)))
    del keep
    return ProfileData(z=z, u_superficial=np.zeros(nz), u_intrinsic=np.zeros(nz), epsilon=eps,
                       u_normalized=np.zeros(nz))


def stream(cur: np.ndarray, nxt: np.ndarray, flags: np.ndarray, periodic, device: int = 0) -> None:
    """Free stream() (simulation.cpp:436-439) of a field given as its two
    population buffers (19, nz, ny, nx), in place: afterwards `cur` holds the
    streamed populations and `nxt` the previous ones (the buffer swap)."""
    if cur.shape != nxt.shape or cur.ndim != 4 or cur.shape[0] != Q:
        raise ConfigError("populations must be (19, nz, ny, nx) arrays of equal shape")
    for a in (cur, nxt):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ConfigError("populations must be C-contiguous float64")
    nz, ny, nx = cur.shape[1:]
    fl = np.ascontiguousarray(flags, dtype=np.uint8).reshape(-1)
    if fl.size != nx * ny * nz:
        raise ConfigError("flags do not match the field")
    dims = (C.c_int32 * 3)(nx, ny, nz)
    per = (C.c_uint8 * 3)(*[int(bool(p)) for p in periodic])
    _check(lib.pgpu_stream_field(dims, per, _p(fl, C.c_uint8), _p(cur, C.c_double),
                                 _p(nxt, C.c_double), int(device)))


def _profile(bufs, meta: _lib.ProfileMeta) -> ProfileData:
    n = int(meta.n_planes)
    z, us, ui, ep, un = (b[:n].copy() for b in bufs)
    return ProfileData(z, us, ui, ep, un, meta.u_max, meta.height, meta.z0, meta.nu,
                       tuple(meta.body_force), int(meta.stream_axis))


# ---------------------------------------------------------------------------
# the time stepper
# ---------------------------------------------------------------------------
class Simulation:
    """B200 drop-in for porolb::Simulation (simulation.hpp:53-111).

    ``Simulation(geometry, nu, lambda_magic, body_force, scheme)`` mirrors the
    pybind constructor (bindings.cpp:228-236); ``Simulation.from_params`` mirrors
    the C++ one (geometry, FluidParams, WallScheme).
    """

    def __init__(self, geometry: VoxelGeometry, nu: float, lambda_magic: float, body_force,
                 scheme: WallScheme = WallScheme.CLI, device: int = 0):
        params = relaxation_from_magic(nu, lambda_magic)
        params.body_force = tuple(float(x) for x in body_force)
        self._init(geometry, params, scheme, device)

    @classmethod
    def from_params(cls, geometry: VoxelGeometry, params: FluidParams,
                    scheme: WallScheme = WallScheme.CLI, device: int = 0) -> "Simulation":
        self = cls.__new__(cls)
        self._init(geometry, params, scheme, device)
        return self

    def _init(self, geometry, params, scheme, device):
        self._h = C.c_void_p()
        self.geometry_dims = tuple(int(x) for x in geometry.dims)
        self.nz = int(geometry.dims[2])
        self._glbm = None
        g, keep = geometry.to_c()
        cp = params.to_c()
        _check(lib.pgpu_create(C.byref(g), C.byref(cp), int(scheme), int(device),
                               C.byref(self._h)))
        del keep
        self.scheme = WallScheme(int(scheme))

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            lib.pgpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- parameters -------------------------------------------------------
    @property
    def params(self) -> FluidParams:
        p = _lib.FluidParams()
        _check(lib.pgpu_get_params(self._h, C.byref(p)))
        return FluidParams.from_c(p)

    def set_body_force(self, g) -> None:
        _check(lib.pgpu_set_body_force(self._h, _vec3(g)))

    @property
    def device_bytes(self) -> int:
        """Device memory held by the simulation (pgpu_device_bytes)."""
        n = C.c_int64()
        _check(lib.pgpu_device_bytes(self._h, C.byref(n)))
        return n.value

    @property
    def layout(self) -> str:
        """"dense", "fluid-only" or "dense-persistent" (pgpu_get_layout)."""
        m = C.c_int32()
        _check(lib.pgpu_get_layout(self._h, C.byref(m)))
        return ("dense", "fluid-only", "dense-persistent")[m.value]

    @property
    def math_mode(self) -> MathMode:
        m = C.c_int32()
        _check(lib.pgpu_get_math_mode(self._h, C.byref(m)))
        return MathMode(m.value)

    @math_mode.setter
    def math_mode(self, mode) -> None:
        _check(lib.pgpu_set_math_mode(self._h, int(mode)))

    @property
    def sweep_kernel(self) -> str:
        """Fluid-only K1 kernel: "auto", "cpipe", "tma" or "units" (pgpu_get_sweep_kernel)."""
        m = C.c_int32()
        _check(lib.pgpu_get_sweep_kernel(self._h, C.byref(m)))
        return SWEEP_KERNELS[m.value]

    @sweep_kernel.setter
    def sweep_kernel(self, kind: str) -> None:
        _check(lib.pgpu_set_sweep_kernel(self._h, SWEEP_KERNELS.index(kind)))

    def set_lid_velocity(self, u) -> None:
        _check(lib.pgpu_set_lid_velocity(self._h, _vec3(u)))

    def set_porous(self, glbm: GlbmPlaneParams) -> None:
        e = np.ascontiguousarray(glbm.eps, dtype=np.float64)
        K = np.ascontiguousarray(glbm.permeability, dtype=np.float64)
        wp = np.ascontiguousarray(glbm.omega_plus, dtype=np.float64)
        wm = np.ascontiguousarray(glbm.omega_minus, dtype=np.float64)
        n = e.size
        if not (K.size == wp.size == wm.size == n):
            raise ConfigError("GLBM plane parameters must cover every z-plane")
        _check(lib.pgpu_set_porous(self._h, n, _p(e, C.c_double), _p(K, C.c_double),
                                   _p(wp, C.c_double), _p(wm, C.c_double),
                                   float(glbm.forchheimer_cf), int(glbm.eps_in_equilibrium)))
        self._glbm = glbm

    @property
    def porous(self) -> bool:
        return self._glbm is not None

    def initialize_equilibrium(self, delta_rho: float, u) -> None:
        _check(lib.pgpu_initialize_equilibrium(self._h, float(delta_rho), _vec3(u)))

    # -- stepping ------------------------------------------------------------
    def step(self, n: int = 1) -> None:
        _check(lib.pgpu_step(self._h, int(n)))

    def prepare(self) -> None:
        """Instantiate the step's CUDA graphs now (pgpu_prepare): a later
        step() does not pay their capture.  No time step is taken."""
        _check(lib.pgpu_prepare(self._h))

    @property
    def steps_done(self) -> int:
        v = C.c_int64()
        _check(lib.pgpu_steps_done(self._h, C.byref(v)))
        return v.value

    @property
    def cli_fallback_count(self) -> int:
        v = C.c_int32()
        _check(lib.pgpu_cli_fallback_count(self._h, C.byref(v)))
        return v.value

    @property
    def fluid_cells(self) -> int:
        v = C.c_int64()
        _check(lib.pgpu_fluid_cells(self._h, C.byref(v)))
        return v.value

    @property
    def dims(self) -> tuple:
        return self.geometry_dims

    @property
    def cells(self) -> int:
        d = self.geometry_dims
        return d[0] * d[1] * d[2]

    def synchronize(self) -> None:
        _check(lib.pgpu_synchronize(self._h))

    def set_stream(self, stream_handle: int | None) -> None:
        _check(lib.pgpu_set_stream(self._h, C.c_void_p(stream_handle or 0)))

    @property
    def launch_count(self) -> int:
        v = C.c_int64()
        _check(lib.pgpu_launch_count(self._h, C.byref(v)))
        return v.value

    @property
    def algorithmic_bytes_per_step(self) -> float:
        v = C.c_double()
        _check(lib.pgpu_algorithmic_bytes_per_step(self._h, C.byref(v)))
        return v.value

    # -- state I/O -------------------------------------------------------------
    def get_pdfs(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """f(steps_done) in the reference layout, shape (19, nz, ny, nx)."""
        nx, ny, nz = self.geometry_dims
        if out is None:
            out = np.empty((Q, nz, ny, nx), dtype=np.float64)
        assert out.flags.c_contiguous and out.dtype == np.float64 and out.size == Q * self.cells
        _check(lib.pgpu_get_pdfs(self._h, _p(out, C.c_double)))
        return out

    def set_pdfs(self, f: np.ndarray) -> None:
        a = np.ascontiguousarray(f, dtype=np.float64)
        if a.size != Q * self.cells:
            raise ConfigError("expected 19*cells populations")
        _check(lib.pgpu_set_pdfs(self._h, _p(a, C.c_double)))

    def cell_populations(self, cell: int) -> np.ndarray:
        out = np.zeros(Q)
        _check(lib.pgpu_get_cell_populations(self._h, int(cell), _p(out, C.c_double)))
        return out

    def set_cell_populations(self, cell: int, f) -> None:
        a = np.ascontiguousarray(f, dtype=np.float64)
        if a.size != Q:
            raise ValueError("expected 19 population values")
        _check(lib.pgpu_set_cell_populations(self._h, int(cell), _p(a, C.c_double)))

    # -- observables -------------------------------------------------------------
    def macroscopic(self, cell: int):
        d = C.c_double()
        u = np.zeros(3)
        _check(lib.pgpu_macroscopic(self._h, int(cell), C.byref(d), _p(u, C.c_double)))
        return d.value, u

    def flags(self) -> np.ndarray:
        """The geometry's flag bytes (field.hpp:45), shaped (nz, ny, nx)."""
        nx, ny, nz = self.geometry_dims
        out = np.empty((nz, ny, nx), dtype=np.uint8)
        _check(lib.pgpu_get_flags(self._h, _p(out, C.c_uint8)))
        return out

    def macroscopic_fields(self, out=None):
        """(delta_rho, ux, uy, uz), each shaped (nz, ny, nx); 0 on non-fluid cells.
        `out`: four C-contiguous float64 arrays of that shape to fill (e.g. in
        pinned host memory), returned."""
        nx, ny, nz = self.geometry_dims
        if out is not None:
            outs = list(out)
            if len(outs) != 4 or any(o.dtype != np.float64 or o.size != nx * ny * nz
                                     or not o.flags.c_contiguous for o in outs):
                raise ValueError("out: four C-contiguous float64 arrays of nx*ny*nz cells")
        else:
            outs = [np.empty((nz, ny, nx)) for _ in range(4)]
        _check(lib.pgpu_macroscopic_fields(self._h, *[_p(o, C.c_double) for o in outs]))
        return tuple(outs)

    def planar_profile(self, stream_axis: int = 0) -> ProfileData:
        bufs = [np.zeros(self.nz) for _ in range(5)]
        meta = _lib.ProfileMeta()
        _check(lib.pgpu_planar_profile(self._h, int(stream_axis),
                                       *[_p(b, C.c_double) for b in bufs], C.byref(meta)))
        return _profile(bufs, meta)

    def plane_sums(self, stream_axis: int = 0) -> np.ndarray:
        out = np.zeros(self.nz)
        _check(lib.pgpu_plane_sums(self._h, int(stream_axis), _p(out, C.c_double)))
        return out

    def max_speed(self) -> float:
        v = C.c_double()
        _check(lib.pgpu_max_speed(self._h, C.byref(v)))
        return v.value

    def max_speed2(self):
        v = C.c_double()
        fin = C.c_int32()
        _check(lib.pgpu_max_speed2(self._h, C.byref(v), C.byref(fin)))
        return v.value, bool(fin.value)

    # -- multi-GPU halo -------------------------------------------------------
    @property
    def halo_elems(self) -> int:
        v = C.c_int64()
        _check(lib.pgpu_halo_elems(self._h, C.byref(v)))
        return v.value

    def set_halo_buffers(self, send_lo, send_hi, recv_lo0, recv_lo1, recv_hi0, recv_hi1) -> None:
        """Device buffers of halo_elems doubles each: raw pointers or CUDA tensors
        (kept alive by this object)."""
        bufs = (send_lo, send_hi, recv_lo0, recv_lo1, recv_hi0, recv_hi1)
        self._halo_keep = bufs
        ptrs = [b if isinstance(b, int) else b.data_ptr() for b in bufs]
        _check(lib.pgpu_set_halo_buffers(self._h, *[C.c_void_p(p) for p in ptrs]))

    @property
    def halo_parity(self) -> int:
        v = C.c_int32()
        _check(lib.pgpu_halo_parity(self._h, C.byref(v)))
        return v.value

    def step_part(self, part: int, stream_handle: Optional[int] = None) -> None:
        """Split step (slab mode); `stream_handle` (cudaStream_t as int) puts
        this part's kernels on another stream without re-binding the sim."""
        if stream_handle is None:
            _check(lib.pgpu_step_part(self._h, int(part)))
        else:
            _check(lib.pgpu_step_part_on(self._h, int(part), C.c_void_p(int(stream_handle))))

    def step_finish(self) -> None:
        _check(lib.pgpu_step_finish(self._h))


def run_to_steady(sim: Simulation, tolerance: float = 1e-8, check_interval: int = 1000,
                  max_steps: int = 2_000_000, max_speed: float = 0.3 / 1.7320508075688772):
    """bindings.cpp:245-257 / simulation.cpp:441-480 -> (RunStats, ProfileData)."""
    cfg = _lib.SteadyConfig(float(tolerance), int(check_interval), int(max_steps),
                            float(max_speed))
    st = _lib.RunStatsC()
    bufs = [np.zeros(sim.nz) for _ in range(5)]
    meta = _lib.ProfileMeta()
    _check(lib.pgpu_run_to_steady_state(sim._h, C.byref(cfg), C.byref(st),
                                        *[_p(b, C.c_double) for b in bufs], C.byref(meta)))
    stats = RunStats(int(st.steps), st.mlups, st.seconds, bool(st.converged), st.residual,
                     int(st.cli_fallbacks))
    return stats, _profile(bufs, meta)


def build_info() -> dict:
    """pgpu_build_info as a dict ({"kernel_hash": ...})."""
    buf = C.create_string_buffer(256)
    _check(lib.pgpu_build_info(buf, 256))
    return dict(kv.split("=", 1) for kv in buf.value.decode().split(";") if "=" in kv)


def device_count() -> int:
    return int(lib.pgpu_device_count())
