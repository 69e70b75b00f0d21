"""B200-native (sm_100a) D3Q19 TRT time stepper for arXiv 1507.06565's pore-scale
lattice Boltzmann runs: a drop-in for the reference porolb Simulation path.

The compute lives in libporolb_cuda.so (CUDA kernels + C ABI,
include/porolb_gpu.h); this package is its Python mirror of the reference API.
"""
from .porolb import (  # noqa: F401
    OPPOSITE,
    Q,
    VELOCITIES,
    WEIGHTS,
    ConfigError,
    DriveMode,
    DriveSpec,
    CudaError,
    FluidParams,
    GeometryError,
    GlbmPlaneParams,
    GlbmViscosity,
    MathMode,
    NumericalInstability,
    ProfileData,
    RunStats,
    Simulation,
    SpherePack,
    VoxelGeometry,
    WallScheme,
    build_info,
    device_count,
    equilibrium,
    generate_spheres,
    glbm_equilibrium,
    glbm_force_and_velocity,
    kozeny_carman,
    make_box_geometry,
    make_glbm_params,
    porosity_profile,
    relaxation_from_magic,
    resolve_drive,
    run_to_steady,
    stream,
    trt_collide,
    voxelize,
    voxelize_device,
    voxelize_slab,
)

from .fileio import (  # noqa: F401,E402
    format_double,
    read_profile_csv,
    read_sphere_csv,
    read_voxel_file,
    write_comparison_csv,
    write_profile_csv,
    write_report,
    write_sphere_csv,
    write_voxel_file,
    write_vtk,
)

__version__ = "0.1.0"
