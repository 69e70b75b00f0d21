/*
 * porolb_gpu.h -- C ABI of libporolb_cuda.so, the B200 (sm_100a) drop-in for
 * the reference solver's time-step path (porolb::Simulation and its setup).
 *
 * Reference interfaces replaced (paths relative to the reference's proj/):
 *   pgpu_relaxation_from_magic   lattice.hpp:42-44,   lattice.cpp:58-75
 *   pgpu_voxelize / _slab / _device  geometry.hpp:76-81, geometry.cpp:491-632
 *   pgpu_make_box_geometry       geometry.hpp:83-84,  geometry.cpp:634-640
 *   pgpu_create                  simulation.hpp:55,   simulation.cpp:80-102
 *   pgpu_set_body_force          simulation.hpp:57
 *   pgpu_set_lid_velocity        simulation.hpp:60-61, simulation.cpp:104-112
 *   pgpu_set_porous              simulation.hpp:63-64, simulation.cpp:114-119
 *   pgpu_initialize_equilibrium  simulation.hpp:88-89, simulation.cpp:121-128
 *   pgpu_step                    simulation.hpp:67,   simulation.cpp:344-352
 *   pgpu_steps_done              simulation.hpp:68
 *   pgpu_get_pdfs / set_pdfs     simulation.hpp:71-72 (field().cur(k)), field.hpp:48-51
 *   pgpu_get/set_cell_populations field.hpp:53-60
 *   pgpu_macroscopic             simulation.hpp:76-78, simulation.cpp:354-369
 *   pgpu_macroscopic_fields      (bulk form of the above)
 *   pgpu_planar_profile          simulation.hpp:80-83, simulation.cpp:371-417, profile.cpp:10-19
 *   pgpu_max_speed               simulation.hpp:85-86, simulation.cpp:419-434
 *   pgpu_cli_fallback_count      simulation.hpp:73
 *   pgpu_fluid_cells             simulation.hpp:74
 *   pgpu_run_to_steady_state     simulation.hpp:134-138, simulation.cpp:441-480
 *   pgpu_kozeny_carman           glbm.hpp:40-46,      glbm.cpp:90-111
 *   pgpu_make_glbm_params        simulation.hpp:31-36, simulation.cpp:23-50
 *   pgpu_glbm_force_and_velocity simulation.hpp:38-43, simulation.cpp:52-66
 *   pgpu_equilibrium / trt_collide lattice.hpp:46-61, lattice.cpp:77-128
 *   pgpu_get_flags               field.hpp:45 (flags())
 *   pgpu_format_double           io.hpp:43,  io.cpp:11-15
 *   pgpu_write/read_profile_csv  io.hpp:14-18, io.cpp:41-97
 *   pgpu_write_comparison_csv    io.hpp:20-24, io.cpp:99-110 (interp_linear profile.cpp:21-29)
 *   pgpu_write_report            io.hpp:26-28, io.cpp:112-116
 *   pgpu_write_vtk               io.hpp:30-32, io.cpp:117-149
 *   pgpu_write/read_sphere_csv   io.hpp:34-36, io.cpp:151-199
 *   pgpu_write/read_voxel_file   io.hpp:38-41, io.cpp:201-278
 *
 * Conventions
 *  - Plain pointers and sizes only; every input array is COPIED by the callee,
 *    the caller keeps ownership (reference ctor deep-copies, simulation.cpp:80-91).
 *  - Layouts are the reference's: cell c = (z*ny + y)*nx + x (field.hpp:19-21),
 *    PDF slot f[k*cells + c] (field.hpp:36-37,48-51), fluctuation form.
 *  - Every call returns a status: PGPU_OK, or the code of the reference
 *    exception it replaces (errors.hpp:9-21); pgpu_last_error() holds the
 *    message (thread-local).  The C++ wrapper include/porolb_gpu/porolb_gpu.hpp
 *    rethrows the reference exception types.
 *  - A simulation handle is not thread-safe (same as the reference object).
 *  - There is no CPU fallback: without a usable sm_100 device pgpu_create
 *    fails with PGPU_ERR_CUDA.
 */
#ifndef POROLB_GPU_H
#define POROLB_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGPU_ABI_VERSION 1

enum pgpu_status {
  PGPU_OK = 0,
  PGPU_ERR_CONFIG = 1,      /* porolb::ConfigError */
  PGPU_ERR_INSTABILITY = 2, /* porolb::NumericalInstability */
  PGPU_ERR_GEOMETRY = 3,    /* porolb::GeometryError */
  PGPU_ERR_CUDA = 4,        /* device / driver failure (no reference analogue) */
  PGPU_ERR_INTERNAL = 5     /* invalid argument or other std::exception */
};

enum pgpu_wall_scheme { PGPU_SBB = 0, PGPU_CLI = 1 }; /* boundary.hpp:12 */
/* Arithmetic of the time step (no reference analogue: the reference has one).
 * EXACT: every fp64 operation in the reference's order, results bit-identical
 * to simulation.cpp.  FAST: the same TRT algebra FMA-contracted and
 * regrouped, with CLI links folded into the stored state;
 * agrees with the reference to <= 1e-12 relative (the north-star tolerance).
 * pgpu_create starts in EXACT unless the environment sets PGPU_MATH=fast. */
enum pgpu_math_mode { PGPU_MATH_EXACT = 0, PGPU_MATH_FAST = 1 };
enum pgpu_glbm_viscosity { PGPU_VISC_PLAIN = 0, PGPU_VISC_RESCALED = 1, PGPU_VISC_CONSTANT_RATIO = 2 };

typedef struct pgpu_sim pgpu_sim;
typedef struct pgpu_voxel_geometry pgpu_voxel_geometry;

/* FluidParams, lattice.hpp:32-39 */
typedef struct {
  double nu;
  double omega_plus;
  double omega_minus;
  double lambda_magic;
  double rho0;
  double body_force[3];
} pgpu_fluid_params;

/* VoxelGeometry (geometry.hpp:62-73) as plain arrays; BoundaryLink
 * (boundary.hpp:16-22) as structure-of-arrays.  n_links may be 0. */
typedef struct {
  int32_t dims[3];
  uint8_t periodic[3];
  const uint8_t* flags;          /* cells; 0 fluid, 1 solid, 2 wall */
  int64_t n_links;
  const int64_t* link_fluid_cell;
  const int64_t* link_second_fluid; /* -1 when none */
  const int32_t* link_direction;
  const float* link_q;
  const uint8_t* link_moving;    /* may be NULL: all false */
  const double* porosity;        /* nz entries */
  int64_t fluid_cells;
  int32_t has_wall_plane_lo, has_wall_plane_hi;
  double wall_plane_lo, wall_plane_hi;
  /* x-slab decomposition (multi-GPU).  When slab != 0 the
   * arrays above describe the local slab [x_offset, x_offset+dims[0]) of a
   * global domain of global_nx cells along x, and ghost_flags_lo/hi hold the
   * flags of the neighbouring columns x_offset-1 and x_offset+dims[0]
   * (ny*nz each, index z*ny+y).  link_second_fluid may be -2: the second
   * fluid cell lies in a ghost column.  periodic[0] is ignored. */
  int32_t slab;
  int32_t x_offset;
  int32_t global_nx;
  const uint8_t* ghost_flags_lo;
  const uint8_t* ghost_flags_hi;
} pgpu_geometry;

/* DriveMode / DriveSpec (boundary.hpp:24-34) */
enum pgpu_drive_mode { PGPU_DRIVE_BODY_FORCE = 0, PGPU_DRIVE_PRESSURE_GRADIENT_AS_FORCE = 1 };
typedef struct {
  int32_t mode;
  double magnitude[3];       /* body force, or Delta_p on the stream axis */
  uint8_t periodic_axes[3];
  int32_t stream_axis;
  double channel_length;     /* required for PGPU_DRIVE_PRESSURE_GRADIENT_AS_FORCE */
} pgpu_drive_spec;

/* SteadyConfig (simulation.hpp:118-123) */
typedef struct {
  double tolerance;
  int32_t check_interval;
  int64_t max_steps;
  double max_speed;
} pgpu_steady_config;

/* RunStats (simulation.hpp:125-132) */
typedef struct {
  int64_t steps;
  double mlups;
  double seconds;
  int32_t converged;
  double residual;
  int32_t cli_fallbacks;
} pgpu_run_stats;

/* ProfileData metadata (profile.hpp:12-34); the arrays are caller-provided
 * with capacity nz and n_planes entries are written. */
typedef struct {
  int32_t n_planes;
  double u_max, height, z0, nu;
  double body_force[3];
  int32_t stream_axis;
} pgpu_profile_meta;

/* Sphere list (geometry.hpp:14-32) for the voxelizer. */
typedef struct {
  int64_t n_spheres;
  const double* cx;
  const double* cy;
  const double* cz;
  const double* radius;
  double box[3];
  double bottom_plate_z;
} pgpu_sphere_pack;

/* VoxelizeOptions, geometry.hpp:51-57 */
typedef struct {
  uint8_t periodic[3];
  uint8_t wall_z_lo, wall_z_hi;
  double q_clamp_min;
} pgpu_voxelize_options;

/* ---- errors / library ---------------------------------------------------- */
const char* pgpu_last_error(void);
int pgpu_abi_version(void);
/* "kernel_hash=<16 hex>": identifies the sweep kernels' build (sources +
 * nvcc flags); profiles/ncu_traffic.json entries are keyed by it. */
int pgpu_build_info(char* buf, int32_t cap);
/* Number of visible CUDA devices (0 without a GPU; never fails). */
int pgpu_device_count(void);

/* ---- lattice-level host functions (bit-identical to the reference) -------- */
int pgpu_relaxation_from_magic(double nu, double lambda_magic, pgpu_fluid_params* out);
int pgpu_equilibrium(double delta_rho, const double u[3], double rho0, double out[19]);
int pgpu_trt_collide(const double f[19], const pgpu_fluid_params* p, double out[19]);
/* glbm_equilibrium (simulation.hpp:45-48, simulation.cpp:68-78): quadratic
 * terms scaled by 1/eps; ConfigError for eps <= 0. */
int pgpu_glbm_equilibrium(double delta_rho, const double u[3], double eps, double rho0,
                          double out[19]);
/* resolve_drive (boundary.hpp:24-38, boundary.cpp:9-17): the body force fed
 * to the collision for a body-force or pressure-gradient drive. */
int pgpu_resolve_drive(const pgpu_drive_spec* spec, double g_out[3]);
int pgpu_kozeny_carman(int32_t n, const double* eps, double grain_diameter,
                       double free_threshold, double* K_out);
int pgpu_make_glbm_params(int32_t n, const double* eps, const double* K, double c_F,
                          double nu, double lambda_magic, int32_t viscosity_mode, double J,
                          double* omega_plus_out, double* omega_minus_out);
int pgpu_glbm_force_and_velocity(const double momentum[3], double eps, double K, double c_F,
                                 const double g[3], double nu, double u_out[3],
                                 double force_out[3]);

/* ---- geometry (host, multi-threaded, bit-exact with voxelize) ------------ */
int pgpu_voxelize(const pgpu_sphere_pack* pack, const int32_t dims[3],
                  const pgpu_voxelize_options* opt, pgpu_voxel_geometry** out);
/* Local x-slab [x0, x1) of the global voxelization plus ghost-column flags. */
int pgpu_voxelize_slab(const pgpu_sphere_pack* pack, const int32_t dims[3],
                       const pgpu_voxelize_options* opt, int32_t x0, int32_t x1,
                       pgpu_voxel_geometry** out);
int pgpu_make_box_geometry(const int32_t dims[3], const pgpu_voxelize_options* opt,
                           pgpu_voxel_geometry** out);
/* porosity_profile (geometry.hpp:86-88, geometry.cpp:642-661): z[k] = k + 1/2,
 * eps[k] = fluid fraction of plane k (nz entries each). */
int pgpu_porosity_profile(const pgpu_geometry* geom, double* z, double* eps);
/* voxelize() on the GPU: byte-identical output, computed
 * by sm_100a kernels (flags, per-cell link counts, scan, links with q). */
int pgpu_voxelize_device(const pgpu_sphere_pack* pack, const int32_t dims[3],
                         const pgpu_voxelize_options* opt, int32_t device,
                         pgpu_voxel_geometry** out);
/* Fills a pgpu_geometry view whose arrays point into the handle (valid until
 * pgpu_voxel_geometry_free). */
int pgpu_voxel_geometry_view(const pgpu_voxel_geometry* g, pgpu_geometry* view,
                             int32_t* q_fallback_count);
void pgpu_voxel_geometry_free(pgpu_voxel_geometry* g);

/* Seeded synthetic sphere lists for the benchmark configurations (the
 * reference has no generator for them).  mode 0: random
 * sequential addition (no overlap, min-image in periodic x/y); mode 1:
 * Boolean model (overlap allowed).  Radii uniform in [r_min, r_max]; centres
 * uniform in [0,lx)x[0,ly)x[z_lo,z_hi].  Stops when the analytic bed porosity
 * (mode 0: 1 - sum V / V_bed; mode 1: exp(-sum V / V_bed)) reaches
 * target_porosity or after max_attempts draws.  Capacity-limited output. */
int pgpu_generate_spheres(int32_t mode, uint64_t seed, const double box[3], double z_lo,
                          double z_hi, double r_min, double r_max, double bed_volume,
                          double target_porosity, int64_t max_attempts, int64_t capacity,
                          double* cx, double* cy, double* cz, double* r, int64_t* n_out,
                          double* porosity_out);

/* ---- simulation ------------------------------------------------------------ */
int pgpu_create(const pgpu_geometry* geom, const pgpu_fluid_params* params, int32_t scheme,
                int32_t device, pgpu_sim** out);
int pgpu_destroy(pgpu_sim* sim);
/* Run all device work of this simulation on `stream` (a cudaStream_t); NULL
 * restores the simulation's own stream. */
int pgpu_set_stream(pgpu_sim* sim, void* stream);
int pgpu_get_stream(pgpu_sim* sim, void** stream);
int pgpu_synchronize(pgpu_sim* sim);

int pgpu_get_params(pgpu_sim* sim, pgpu_fluid_params* out);
int pgpu_set_math_mode(pgpu_sim* sim, int32_t mode);
/* PDF layout chosen at creation (PGPU_LAYOUT overrides). */
enum pgpu_layout { PGPU_LAYOUT_DENSE = 0, PGPU_LAYOUT_FLUID_ONLY = 1, PGPU_LAYOUT_DENSE_PERSISTENT = 2 };
int pgpu_get_layout(pgpu_sim* sim, int32_t* layout);
/* K1 kernel of the fluid-only layout (no reference analogue,
 * results are bit-identical): AUTO (the library's choice: UNITS wherever it
 * applies), CPIPE (per-thread asynchronous copies over 32-cell chunks,
 * k_sweep_cpipe), TMA (warp-specialised bulk-copy
 * pipeline, k_sweep_tma) or UNITS (k_sweep_units: warps sweep runs of 32
 * consecutive fluid slots, so no lane idles on a solid cell).
 * PGPU_SWEEP=cpipe|tma|units sets the default at creation. */
enum pgpu_sweep_kernel { PGPU_SWEEP_AUTO = 0, PGPU_SWEEP_CPIPE = 1, PGPU_SWEEP_TMA = 2,
                         PGPU_SWEEP_UNITS = 3 };
int pgpu_set_sweep_kernel(pgpu_sim* sim, int32_t kind);
/* Instantiate the step's CUDA graphs now (no time step is taken; no reference
 * analogue): a later step() does not pay their capture.  Optional. */
int pgpu_prepare(pgpu_sim* sim);
int pgpu_get_sweep_kernel(pgpu_sim* sim, int32_t* kind);
/* Device memory held by the simulation (PDF buffers, cell words, link data). */
int pgpu_device_bytes(pgpu_sim* sim, int64_t* bytes);
int pgpu_get_math_mode(pgpu_sim* sim, int32_t* mode);
int pgpu_set_body_force(pgpu_sim* sim, const double g[3]);
int pgpu_set_lid_velocity(pgpu_sim* sim, const double u[3]);
/* GlbmPlaneParams (simulation.hpp:18-27); n must equal nz. */
int pgpu_set_porous(pgpu_sim* sim, int32_t n, const double* eps, const double* K,
                    const double* omega_plus, const double* omega_minus, double c_F,
                    int32_t eps_in_equilibrium);
int pgpu_initialize_equilibrium(pgpu_sim* sim, double delta_rho, const double u[3]);

/* n time steps; asynchronous on the simulation's stream, ordered before any
 * later read. */
int pgpu_step(pgpu_sim* sim, int64_t n);
int pgpu_steps_done(pgpu_sim* sim, int64_t* out);
int pgpu_cli_fallback_count(pgpu_sim* sim, int32_t* out);
int pgpu_fluid_cells(pgpu_sim* sim, int64_t* out);
int pgpu_dims(pgpu_sim* sim, int32_t dims[3]);
/* The geometry's flag bytes (field.hpp:45 flags(); 0 fluid, 1 solid, 2 wall). */
int pgpu_get_flags(pgpu_sim* sim, uint8_t* out);

/* Pre-collision populations f(steps_done) in the reference layout
 * (19*cells doubles).  Only fluid-cell slots are defined on output. */
int pgpu_get_pdfs(pgpu_sim* sim, double* out);
int pgpu_set_pdfs(pgpu_sim* sim, const double* in);
int pgpu_get_cell_populations(pgpu_sim* sim, int64_t cell, double out[19]);
int pgpu_set_cell_populations(pgpu_sim* sim, int64_t cell, const double in[19]);

int pgpu_macroscopic(pgpu_sim* sim, int64_t cell, double* delta_rho, double u[3]);
/* Any output may be NULL; non-fluid cells are written as 0. */
int pgpu_macroscopic_fields(pgpu_sim* sim, double* delta_rho, double* ux, double* uy,
                            double* uz);
/* Arrays need nz capacity; meta->n_planes entries are written. */
int pgpu_planar_profile(pgpu_sim* sim, int32_t stream_axis, double* z, double* u_superficial,
                        double* u_intrinsic, double* epsilon, double* u_normalized,
                        pgpu_profile_meta* meta);
/* Per-plane sums of the stream-axis velocity over fluid cells, in the
 * reference's sequential cell order (building block for multi-GPU profiles). */
int pgpu_plane_sums(pgpu_sim* sim, int32_t stream_axis, double* sums_nz);
int pgpu_max_speed(pgpu_sim* sim, double* out);
/* Max of |u|^2 plus a finiteness flag (building block for multi-GPU guards). */
int pgpu_max_speed2(pgpu_sim* sim, double* vmax2, int32_t* finite);

int pgpu_run_to_steady_state(pgpu_sim* sim, const pgpu_steady_config* cfg,
                             pgpu_run_stats* stats, double* z, double* u_superficial,
                             double* u_intrinsic, double* epsilon, double* u_normalized,
                             pgpu_profile_meta* meta);

/* ---- instrumentation ------------------------------------------------------- */
/* Kernels launched by this simulation so far. */
int pgpu_launch_count(pgpu_sim* sim, int64_t* out);
/* Bytes per step the hot kernel must move by the 304 B/fluid-cell ledger. */
int pgpu_algorithmic_bytes_per_step(pgpu_sim* sim, double* out);

/* ---- multi-GPU halo (x-slab, 5 PDFs per face) ------------------------------ */
/* Element count of one face buffer: 5*ny*nz doubles. */
int pgpu_halo_elems(pgpu_sim* sim, int64_t* out);
/* Device buffers owned by the caller (e.g. torch tensors):
 *   send_lo: values leaving through x=0      (directions 2,8,10,12,14)
 *   send_hi: values leaving through x=nx-1   (directions 1,7,9,11,13)
 *   recv_lo[2], recv_hi[2]: ghost columns, double-buffered by step parity. */
int pgpu_set_halo_buffers(pgpu_sim* sim, double* send_lo, double* send_hi, double* recv_lo0,
                          double* recv_lo1, double* recv_hi0, double* recv_hi1);
/* Which recv parity the next kernel reads (the exchange must fill the other). */
int pgpu_halo_parity(pgpu_sim* sim, int32_t* parity);
/* Split step for overlap: part 0 = edge columns (fills send buffers),
 * part 1 = interior; pgpu_step_finish advances the step counter. */
int pgpu_step_part(pgpu_sim* sim, int32_t part);
/* Same, with the part's kernels on `stream` (a cudaStream_t; NULL = the
 * simulation's stream) so edge columns + exchange and the interior can run
 * on two streams; the caller orders them (dist.py DistTransport). */
int pgpu_step_part_on(pgpu_sim* sim, int32_t part, void* stream);
int pgpu_step_finish(pgpu_sim* sim);

/* ---- multi-GPU x-slab driver (dist.cpp) ----------------------
 * One handle drives the slabs of an x-slab decomposition: per step the edge
 * columns (high-priority stream) -> 5-PDF ghost exchange, concurrently with
 * the interior columns on the simulation's stream; the exchange is NCCL
 * (one rank per process; libnccl resolved at run time) or peer copies (all
 * slabs in this process).  Each simulation must come from a slab geometry
 * (pgpu_voxelize_slab) and must not have halo buffers of its own in use: the
 * driver owns them.  Observables are global (all ranks).  No reference
 * analogue (the reference is single-node OpenMP); the exchange rebuilds the
 * paper's communication-reducing ghost layer. */
typedef struct pgpu_dist pgpu_dist;
/* NCCL unique id (128 bytes): made by rank 0, distributed by the caller. */
int pgpu_dist_nccl_unique_id(uint8_t id[128]);
int pgpu_dist_create_nccl(pgpu_sim* sim, const uint8_t id[128], int32_t rank, int32_t world,
                          pgpu_dist** out);
/* sims[r] = slab r of `world` (any devices; same device is allowed). */
int pgpu_dist_create_local(pgpu_sim* const* sims, int32_t world, pgpu_dist** out);
/* IPC transport (one rank per process, all on one node): the edge-column
 * kernel stores its outgoing PDFs straight into the neighbours' ghost buffers
 * (CUDA IPC mappings over NVLink), ordered by interprocess events and a host
 * channel in POSIX shared memory.  Create on every rank, export this rank's
 * blob (pgpu_dist_ipc_blob_size bytes), all-gather the blobs in rank order by
 * any means (MPI, torch.distributed, files), then connect. */
int pgpu_dist_create_ipc(pgpu_sim* sim, int32_t rank, int32_t world, pgpu_dist** out);
int pgpu_dist_ipc_blob_size(int64_t* bytes);
int pgpu_dist_ipc_export(pgpu_dist* d, void* blob);
int pgpu_dist_ipc_connect(pgpu_dist* d, const void* blobs);
/* NCCL mode replays a CUDA graph of two steps (default on; PGPU_DIST_GRAPHS=0). */
int pgpu_dist_set_graphs(pgpu_dist* d, int32_t enable);
int pgpu_dist_step(pgpu_dist* d, int64_t n);
int pgpu_dist_synchronize(pgpu_dist* d);
int pgpu_dist_plane_sums(pgpu_dist* d, int32_t stream_axis, double* sums_nz);
int pgpu_dist_max_speed2(pgpu_dist* d, double* vmax2, int32_t* finite);
int pgpu_dist_planar_profile(pgpu_dist* d, int32_t stream_axis, double* z, double* u_superficial,
                             double* u_intrinsic, double* epsilon, double* u_normalized,
                             pgpu_profile_meta* meta);
int pgpu_dist_destroy(pgpu_dist* d);

/* Free stream() (simulation.hpp:113-116, simulation.cpp:436-439) of a field
 * given as host arrays (reference layout, 19*cells each): streaming over
 * fluid-fluid pairs with periodic wrap, then the buffer swap -- on return
 * `cur` holds the streamed populations and `next` the previous current ones.
 * Boundary links are not applied (as in the reference). */
int pgpu_stream_field(const int32_t dims[3], const uint8_t periodic[3], const uint8_t* flags,
                      double* cur, double* next, int32_t device);

/* ---- file formats (io.hpp; byte-identical to the reference's writers) ------ */
/* "%.17g" of v, NUL-terminated (cap >= 25 always suffices). */
int pgpu_format_double(double v, char* buf, int32_t cap);
/* Profile CSV: meta->n_planes rows; u_normalized may be shorter (n_norm
 * entries, missing ones print as 0 like io.cpp:58). */
int pgpu_write_profile_csv(const char* path, const pgpu_profile_meta* meta, const double* z,
                           const double* u_superficial, const double* u_intrinsic,
                           const double* epsilon, const double* u_normalized, int32_t n_norm);
/* Parses like io.cpp:64-97.  meta->n_planes = rows found, *n_norm = rows with
 * a fifth column; arrays are filled only when rows <= capacity (call with
 * capacity 0 to size them). */
int pgpu_read_profile_csv(const char* path, int32_t capacity, pgpu_profile_meta* meta, double* z,
                          double* u_superficial, double* u_intrinsic, double* epsilon,
                          double* u_normalized, int32_t* n_norm);
int pgpu_write_comparison_csv(const char* path, int32_t n_a, const double* z_a,
                              const double* u_a, const char* name_a, int32_t n_b,
                              const double* z_b, const double* u_b, const char* name_b);
int pgpu_write_report(const char* path, int32_t n, const char* const* keys,
                      const char* const* values);
/* Legacy VTK of the current state (flags, delta_rho, velocity); moments are
 * computed on the device, text is formatted on all host threads. */
int pgpu_write_vtk(const char* path, pgpu_sim* sim);
int pgpu_write_sphere_csv(const char* path, const pgpu_sphere_pack* pack, uint64_t seed);
/* Parses like io.cpp:164-199; same capacity convention as profiles. */
int pgpu_read_sphere_csv(const char* path, int64_t capacity, int64_t* n_spheres, double* cx,
                         double* cy, double* cz, double* radius, double box[3],
                         double* bottom_plate_z, uint64_t* seed, double* achieved_height);
int pgpu_write_voxel_file(const char* path, const pgpu_geometry* geom);
/* Flags from the file, links rebuilt with q = 1/2 (io.cpp:210-278). */
int pgpu_read_voxel_file(const char* path, pgpu_voxel_geometry** out);

#ifdef __cplusplus
}
#endif
#endif /* POROLB_GPU_H */
