"""The reference's file formats (proj/include/porolb/io.hpp, proj/src/io.cpp),
served by libporolb_cuda.so's native writers/readers (csrc/io.cpp).

Same function names, arguments and error types as the reference module, so a
scenario driver (proj/src/scenarios.cpp:56-116,168-189) can switch by import:

    write_profile_csv(path, profile)          io.cpp:41-62
    read_profile_csv(path) -> ProfileData     io.cpp:64-97
    write_comparison_csv(path, a, na, b, nb)  io.cpp:99-110
    write_report(path, [(key, value), ...])   io.cpp:112-116
    write_vtk(path, sim)                      io.cpp:117-149 (moments from the device)
    write_sphere_csv(path, pack)              io.cpp:151-162
    read_sphere_csv(path) -> SpherePack       io.cpp:164-199
    write_voxel_file(path, geom)              io.cpp:201-208
    read_voxel_file(path) -> VoxelGeometry    io.cpp:210-278
    format_double(v) -> str                   io.cpp:11-15
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import lib
from .porolb import (ProfileData, Simulation, SpherePack, VoxelGeometry, _check,
                     _geometry_from_handle, _p)

_f64 = C.c_double


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _arr(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))


def format_double(v: float) -> str:
    buf = C.create_string_buffer(32)
    _check(lib.pgpu_format_double(float(v), buf, 32))
    return buf.value.decode()


def write_profile_csv(path, profile: ProfileData) -> None:
    cols = [_arr(profile.z), _arr(profile.u_superficial), _arr(profile.u_intrinsic),
            _arr(profile.epsilon)]
    n = cols[0].size
    if any(c.size != n for c in cols):
        raise ValueError("profile columns differ in length")
    un = _arr(profile.u_normalized)
    meta = _lib.ProfileMeta(n, profile.u_max, profile.height, profile.z0, profile.nu,
                            (_f64 * 3)(*profile.body_force), int(profile.stream_axis))
    _check(lib.pgpu_write_profile_csv(_path(path), C.byref(meta), *[_p(c, _f64) for c in cols],
                                      _p(un, _f64), int(un.size)))


def read_profile_csv(path) -> ProfileData:
    meta = _lib.ProfileMeta()
    nn = C.c_int32(0)
    null = C.POINTER(_f64)()
    _check(lib.pgpu_read_profile_csv(_path(path), 0, C.byref(meta), null, null, null, null, null,
                                     C.byref(nn)))
    n = int(meta.n_planes)
    bufs = [np.zeros(n) for _ in range(5)]
    _check(lib.pgpu_read_profile_csv(_path(path), n, C.byref(meta),
                                     *[_p(b, _f64) for b in bufs], C.byref(nn)))
    return ProfileData(bufs[0], bufs[1], bufs[2], bufs[3], bufs[4][:nn.value].copy(),
                       meta.u_max, meta.height, meta.z0, meta.nu, tuple(meta.body_force),
                       int(meta.stream_axis))


def write_comparison_csv(path, a: ProfileData, name_a: str, b: ProfileData, name_b: str) -> None:
    za, ua, zb, ub = _arr(a.z), _arr(a.u_superficial), _arr(b.z), _arr(b.u_superficial)
    _check(lib.pgpu_write_comparison_csv(_path(path), za.size, _p(za, _f64), _p(ua, _f64),
                                         name_a.encode(), zb.size, _p(zb, _f64), _p(ub, _f64),
                                         name_b.encode()))


def write_report(path, entries) -> None:
    entries = [(str(k), str(v)) for k, v in entries]
    keys = (C.c_char_p * max(1, len(entries)))(*[k.encode() for k, _ in entries])
    vals = (C.c_char_p * max(1, len(entries)))(*[v.encode() for _, v in entries])
    _check(lib.pgpu_write_report(_path(path), len(entries), keys, vals))


def write_vtk(path, sim: Simulation) -> None:
    _check(lib.pgpu_write_vtk(_path(path), sim._h))


def write_sphere_csv(path, pack: SpherePack) -> None:
    pk, keep = pack.to_c()
    _check(lib.pgpu_write_sphere_csv(_path(path), C.byref(pk), int(pack.seed)))
    del keep


def read_sphere_csv(path) -> SpherePack:
    n = C.c_int64(0)
    box = (_f64 * 3)()
    plate, top = _f64(0.0), _f64(0.0)
    seed = C.c_uint64(0)
    null = C.POINTER(_f64)()
    _check(lib.pgpu_read_sphere_csv(_path(path), 0, C.byref(n), null, null, null, null, box,
                                    C.byref(plate), C.byref(seed), C.byref(top)))
    cols = [np.zeros(n.value) for _ in range(4)]
    _check(lib.pgpu_read_sphere_csv(_path(path), n.value, C.byref(n),
                                    *[_p(c, _f64) for c in cols], box, C.byref(plate),
                                    C.byref(seed), C.byref(top)))
    return SpherePack(centers=np.stack(cols[:3], axis=1), radii=cols[3], box=tuple(box),
                      bottom_plate_z=plate.value, seed=int(seed.value),
                      achieved_height=top.value)


def write_voxel_file(path, geom: VoxelGeometry) -> None:
    g, keep = geom.to_c()
    _check(lib.pgpu_write_voxel_file(_path(path), C.byref(g)))
    del keep


def read_voxel_file(path) -> VoxelGeometry:
    h = C.c_void_p()
    _check(lib.pgpu_read_voxel_file(_path(path), C.byref(h)))
    return _geometry_from_handle(h)
