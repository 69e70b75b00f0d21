"""ctypes binding of libporolb_cuda.so (the C ABI declared in include/porolb_gpu.h).

The library is loaded from the package directory only; there is no fallback:
if it is missing the import fails loudly (run ``python -m
paper_1507_06565_b200.build``).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# PGPU_LIB selects an experiment build (paper_1507_06565_b200.build --variant=...).
LIB_PATH = Path(os.environ.get("PGPU_LIB") or Path(__file__).resolve().parent / "libporolb_cuda.so")

i32, i64, u8, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint8, C.c_uint64, C.c_float, C.c_double
P = C.POINTER
vp = C.c_void_p


class FluidParams(C.Structure):
    _fields_ = [("nu", f64), ("omega_plus", f64), ("omega_minus", f64), ("lambda_magic", f64),
                ("rho0", f64), ("body_force", f64 * 3)]


class Geometry(C.Structure):
    _fields_ = [("dims", i32 * 3), ("periodic", u8 * 3), ("flags", P(u8)), ("n_links", i64),
                ("link_fluid_cell", P(i64)), ("link_second_fluid", P(i64)),
                ("link_direction", P(i32)), ("link_q", P(f32)), ("link_moving", P(u8)),
                ("porosity", P(f64)), ("fluid_cells", i64), ("has_wall_plane_lo", i32),
                ("has_wall_plane_hi", i32), ("wall_plane_lo", f64), ("wall_plane_hi", f64),
                ("slab", i32), ("x_offset", i32), ("global_nx", i32),
                ("ghost_flags_lo", P(u8)), ("ghost_flags_hi", P(u8))]


class DriveSpec(C.Structure):
    _fields_ = [("mode", i32), ("magnitude", f64 * 3), ("periodic_axes", u8 * 3),
                ("stream_axis", i32), ("channel_length", f64)]


class SteadyConfig(C.Structure):
    _fields_ = [("tolerance", f64), ("check_interval", i32), ("max_steps", i64),
                ("max_speed", f64)]


class RunStatsC(C.Structure):
    _fields_ = [("steps", i64), ("mlups", f64), ("seconds", f64), ("converged", i32),
                ("residual", f64), ("cli_fallbacks", i32)]


class ProfileMeta(C.Structure):
    _fields_ = [("n_planes", i32), ("u_max", f64), ("height", f64), ("z0", f64), ("nu", f64),
                ("body_force", f64 * 3), ("stream_axis", i32)]


class SpherePackC(C.Structure):
    _fields_ = [("n_spheres", i64), ("cx", P(f64)), ("cy", P(f64)), ("cz", P(f64)),
                ("radius", P(f64)), ("box", f64 * 3), ("bottom_plate_z", f64)]


class VoxelizeOptionsC(C.Structure):
    _fields_ = [("periodic", u8 * 3), ("wall_z_lo", u8), ("wall_z_hi", u8),
                ("q_clamp_min", f64)]


# name -> (restype, argtypes); every entry point of include/porolb_gpu.h
SIGNATURES = {
    "pgpu_last_error": (C.c_char_p, []),
    "pgpu_abi_version": (C.c_int, []),
    "pgpu_build_info": (C.c_int, [C.c_char_p, i32]),
    "pgpu_device_count": (C.c_int, []),
    "pgpu_relaxation_from_magic": (C.c_int, [f64, f64, P(FluidParams)]),
    "pgpu_equilibrium": (C.c_int, [f64, P(f64), f64, P(f64)]),
    "pgpu_trt_collide": (C.c_int, [P(f64), P(FluidParams), P(f64)]),
    "pgpu_kozeny_carman": (C.c_int, [i32, P(f64), f64, f64, P(f64)]),
    "pgpu_make_glbm_params": (C.c_int, [i32, P(f64), P(f64), f64, f64, f64, i32, f64, P(f64),
                                        P(f64)]),
    "pgpu_glbm_force_and_velocity": (C.c_int, [P(f64), f64, f64, f64, P(f64), f64, P(f64),
                                               P(f64)]),
    "pgpu_voxelize": (C.c_int, [P(SpherePackC), P(i32), P(VoxelizeOptionsC), P(vp)]),
    "pgpu_voxelize_slab": (C.c_int, [P(SpherePackC), P(i32), P(VoxelizeOptionsC), i32, i32,
                                     P(vp)]),
    "pgpu_make_box_geometry": (C.c_int, [P(i32), P(VoxelizeOptionsC), P(vp)]),
    "pgpu_voxelize_device": (C.c_int, [P(SpherePackC), P(i32), P(VoxelizeOptionsC), i32, P(vp)]),
    "pgpu_voxel_geometry_view": (C.c_int, [vp, P(Geometry), P(i32)]),
    "pgpu_voxel_geometry_free": (None, [vp]),
    "pgpu_generate_spheres": (C.c_int, [i32, u64, P(f64), f64, f64, f64, f64, f64, f64, i64,
                                        i64, P(f64), P(f64), P(f64), P(f64), P(i64), P(f64)]),
    "pgpu_create": (C.c_int, [P(Geometry), P(FluidParams), i32, i32, P(vp)]),
    "pgpu_destroy": (C.c_int, [vp]),
    "pgpu_set_stream": (C.c_int, [vp, vp]),
    "pgpu_get_stream": (C.c_int, [vp, P(vp)]),
    "pgpu_synchronize": (C.c_int, [vp]),
    "pgpu_get_params": (C.c_int, [vp, P(FluidParams)]),
    "pgpu_set_math_mode": (C.c_int, [vp, i32]),
    "pgpu_set_sweep_kernel": (C.c_int, [vp, i32]),
    "pgpu_get_sweep_kernel": (C.c_int, [vp, P(i32)]),
    "pgpu_dist_nccl_unique_id": (C.c_int, [P(u8)]),
    "pgpu_dist_create_nccl": (C.c_int, [vp, P(u8), i32, i32, P(vp)]),
    "pgpu_dist_create_local": (C.c_int, [P(vp), i32, P(vp)]),
    "pgpu_dist_create_ipc": (C.c_int, [vp, i32, i32, P(vp)]),
    "pgpu_dist_ipc_blob_size": (C.c_int, [P(i64)]),
    "pgpu_dist_ipc_export": (C.c_int, [vp, vp]),
    "pgpu_dist_ipc_connect": (C.c_int, [vp, vp]),
    "pgpu_dist_set_graphs": (C.c_int, [vp, i32]),
    "pgpu_dist_step": (C.c_int, [vp, i64]),
    "pgpu_dist_synchronize": (C.c_int, [vp]),
    "pgpu_dist_plane_sums": (C.c_int, [vp, i32, P(f64)]),
    "pgpu_dist_max_speed2": (C.c_int, [vp, P(f64), P(i32)]),
    "pgpu_dist_planar_profile": (C.c_int, [vp, i32, P(f64), P(f64), P(f64), P(f64), P(f64),
                                           P(ProfileMeta)]),
    "pgpu_dist_destroy": (C.c_int, [vp]),
    "pgpu_glbm_equilibrium": (C.c_int, [f64, P(f64), f64, f64, P(f64)]),
    "pgpu_resolve_drive": (C.c_int, [P(DriveSpec), P(f64)]),
    "pgpu_porosity_profile": (C.c_int, [P(Geometry), P(f64), P(f64)]),
    "pgpu_stream_field": (C.c_int, [P(i32), P(u8), P(u8), P(f64), P(f64), i32]),
    "pgpu_get_layout": (C.c_int, [vp, P(i32)]),
    "pgpu_device_bytes": (C.c_int, [vp, P(i64)]),
    "pgpu_get_math_mode": (C.c_int, [vp, P(i32)]),
    "pgpu_set_body_force": (C.c_int, [vp, P(f64)]),
    "pgpu_set_lid_velocity": (C.c_int, [vp, P(f64)]),
    "pgpu_set_porous": (C.c_int, [vp, i32, P(f64), P(f64), P(f64), P(f64), f64, i32]),
    "pgpu_initialize_equilibrium": (C.c_int, [vp, f64, P(f64)]),
    "pgpu_step": (C.c_int, [vp, i64]),
    "pgpu_prepare": (C.c_int, [vp]),
    "pgpu_steps_done": (C.c_int, [vp, P(i64)]),
    "pgpu_cli_fallback_count": (C.c_int, [vp, P(i32)]),
    "pgpu_fluid_cells": (C.c_int, [vp, P(i64)]),
    "pgpu_dims": (C.c_int, [vp, P(i32)]),
    "pgpu_get_pdfs": (C.c_int, [vp, P(f64)]),
    "pgpu_set_pdfs": (C.c_int, [vp, P(f64)]),
    "pgpu_get_cell_populations": (C.c_int, [vp, i64, P(f64)]),
    "pgpu_set_cell_populations": (C.c_int, [vp, i64, P(f64)]),
    "pgpu_macroscopic": (C.c_int, [vp, i64, P(f64), P(f64)]),
    "pgpu_macroscopic_fields": (C.c_int, [vp, P(f64), P(f64), P(f64), P(f64)]),
    "pgpu_planar_profile": (C.c_int, [vp, i32, P(f64), P(f64), P(f64), P(f64), P(f64),
                                      P(ProfileMeta)]),
    "pgpu_plane_sums": (C.c_int, [vp, i32, P(f64)]),
    "pgpu_max_speed": (C.c_int, [vp, P(f64)]),
    "pgpu_max_speed2": (C.c_int, [vp, P(f64), P(i32)]),
    "pgpu_run_to_steady_state": (C.c_int, [vp, P(SteadyConfig), P(RunStatsC), P(f64), P(f64),
                                           P(f64), P(f64), P(f64), P(ProfileMeta)]),
    "pgpu_launch_count": (C.c_int, [vp, P(i64)]),
    "pgpu_algorithmic_bytes_per_step": (C.c_int, [vp, P(f64)]),
    "pgpu_halo_elems": (C.c_int, [vp, P(i64)]),
    "pgpu_set_halo_buffers": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "pgpu_halo_parity": (C.c_int, [vp, P(i32)]),
    "pgpu_step_part": (C.c_int, [vp, i32]),
    "pgpu_step_part_on": (C.c_int, [vp, i32, vp]),
    "pgpu_step_finish": (C.c_int, [vp]),
    "pgpu_get_flags": (C.c_int, [vp, P(u8)]),
    # file formats (io.hpp)
    "pgpu_format_double": (C.c_int, [f64, C.c_char_p, i32]),
    "pgpu_write_profile_csv": (C.c_int, [C.c_char_p, P(ProfileMeta), P(f64), P(f64), P(f64),
                                         P(f64), P(f64), i32]),
    "pgpu_read_profile_csv": (C.c_int, [C.c_char_p, i32, P(ProfileMeta), P(f64), P(f64), P(f64),
                                        P(f64), P(f64), P(i32)]),
    "pgpu_write_comparison_csv": (C.c_int, [C.c_char_p, i32, P(f64), P(f64), C.c_char_p, i32,
                                            P(f64), P(f64), C.c_char_p]),
    "pgpu_write_report": (C.c_int, [C.c_char_p, i32, P(C.c_char_p), P(C.c_char_p)]),
    "pgpu_write_vtk": (C.c_int, [C.c_char_p, vp]),
    "pgpu_write_sphere_csv": (C.c_int, [C.c_char_p, P(SpherePackC), u64]),
    "pgpu_read_sphere_csv": (C.c_int, [C.c_char_p, i64, P(i64), P(f64), P(f64), P(f64), P(f64),
                                       P(f64), P(f64), P(u64), P(f64)]),
    "pgpu_write_voxel_file": (C.c_int, [C.c_char_p, P(Geometry)]),
    "pgpu_read_voxel_file": (C.c_int, [C.c_char_p, P(vp)]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1507_06565_b200/build.py` "
            "(there is no CPU fallback for the B200 path)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
