// porolb_gpu.hpp -- header-only C++ mirror of the reference porolb API for the
// time-step path, implemented over the C ABI of libporolb_cuda.so
// (include/porolb_gpu.h).  A caller of porolb::Simulation (reference
// proj/include/porolb/simulation.hpp:53-111) switches by including this header
// and linking libporolb_cuda.so; names, argument meaning and the exception
// types (errors.hpp:9-21) are the reference's.
#pragma once

#include <array>
#include <cmath>
#include <limits>
#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <functional>
#include <vector>

#include "../porolb_gpu.h"

namespace porolb_gpu {

using Vec3 = std::array<double, 3>;  // lattice.hpp:10
inline constexpr int kQ = 19;

struct ConfigError : std::runtime_error {  // errors.hpp:9-12
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalInstability : std::runtime_error {  // errors.hpp:14-17
  explicit NumericalInstability(const std::string& m) : std::runtime_error(m) {}
};
struct GeometryError : std::runtime_error {  // errors.hpp:19-22
  explicit GeometryError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int status) {
  if (status == PGPU_OK) return;
  const std::string msg = pgpu_last_error();
  switch (status) {
    case PGPU_ERR_CONFIG: throw ConfigError(msg);
    case PGPU_ERR_INSTABILITY: throw NumericalInstability(msg);
    case PGPU_ERR_GEOMETRY: throw GeometryError(msg);
    case PGPU_ERR_CUDA: throw CudaError(msg);
    default: throw std::invalid_argument(msg);
  }
}

enum class WallScheme : std::uint8_t { SBB = PGPU_SBB, CLI = PGPU_CLI };  // boundary.hpp:12
enum class GlbmViscosity { Plain, Rescaled, ConstantRatio };               // simulation.hpp:29

struct FluidParams {  // lattice.hpp:32-39
  double nu = 1.0 / 6.0;
  double omega_plus = 1.0;
  double omega_minus = 1.0;
  double lambda_magic = 3.0 / 16.0;
  double rho0 = 1.0;
  Vec3 body_force{0.0, 0.0, 0.0};

  pgpu_fluid_params c() const {
    return pgpu_fluid_params{nu, omega_plus, omega_minus, lambda_magic, rho0,
                             {body_force[0], body_force[1], body_force[2]}};
  }
};

inline FluidParams relaxation_from_magic(double nu, double lambda_magic) {  // lattice.hpp:42-44
  pgpu_fluid_params p;
  check(pgpu_relaxation_from_magic(nu, lambda_magic, &p));
  FluidParams f;
  f.nu = p.nu;
  f.omega_plus = p.omega_plus;
  f.omega_minus = p.omega_minus;
  f.lambda_magic = p.lambda_magic;
  f.rho0 = p.rho0;
  return f;
}

struct Sphere {  // geometry.hpp:14-17
  Vec3 center{0.0, 0.0, 0.0};
  double radius = 0.0;
};
struct Box3 {
  double lx = 0.0, ly = 0.0, lz = 0.0;
};
struct SpherePack {  // geometry.hpp:25-32
  std::vector<Sphere> spheres;
  Box3 box;
  double bottom_plate_z = 0.0;
  std::uint64_t seed = 0;
  double achieved_height = 0.0;
};
struct Dims {
  int nx = 0, ny = 0, nz = 0;
  std::int64_t cells() const { return static_cast<std::int64_t>(nx) * ny * nz; }
  std::int64_t index(int x, int y, int z) const {
    return (static_cast<std::int64_t>(z) * ny + y) * nx + x;
  }
};
struct VoxelizeOptions {  // geometry.hpp:51-57
  std::array<bool, 3> periodic{true, true, false};
  bool wall_z_lo = false;
  bool wall_z_hi = false;
  double q_clamp_min = 0.05;
};

// VoxelGeometry (geometry.hpp:62-73): owns the voxelizer's arrays.
class VoxelGeometry {
 public:
  VoxelGeometry() = default;
  explicit VoxelGeometry(pgpu_voxel_geometry* h) : h_(h, pgpu_voxel_geometry_free) {
    check(pgpu_voxel_geometry_view(h, &view_, &q_fallback_count_));
  }
  const pgpu_geometry& c() const { return view_; }
  Dims dims() const { return Dims{view_.dims[0], view_.dims[1], view_.dims[2]}; }
  std::int64_t fluid_cells() const { return view_.fluid_cells; }
  std::int64_t n_links() const { return view_.n_links; }
  int q_fallback_count() const { return q_fallback_count_; }
  std::uint8_t flag(std::int64_t cell) const { return view_.flags[cell]; }
  double porosity(int z) const { return view_.porosity[z]; }

 private:
  std::shared_ptr<pgpu_voxel_geometry> h_;
  pgpu_geometry view_{};
  int q_fallback_count_ = 0;
};

namespace detail {
struct PackArrays {
  std::vector<double> x, y, z, r;
  pgpu_sphere_pack c{};
  explicit PackArrays(const SpherePack& p) {
    for (const Sphere& s : p.spheres) {
      x.push_back(s.center[0]);
      y.push_back(s.center[1]);
      z.push_back(s.center[2]);
      r.push_back(s.radius);
    }
    c.n_spheres = static_cast<std::int64_t>(p.spheres.size());
    c.cx = x.data();
    c.cy = y.data();
    c.cz = z.data();
    c.radius = r.data();
    c.box[0] = p.box.lx;
    c.box[1] = p.box.ly;
    c.box[2] = p.box.lz;
    c.bottom_plate_z = p.bottom_plate_z;
  }
};
inline pgpu_voxelize_options opts(const VoxelizeOptions& o) {
  pgpu_voxelize_options c{};
  for (int a = 0; a < 3; ++a) c.periodic[a] = o.periodic[a] ? 1 : 0;
  c.wall_z_lo = o.wall_z_lo ? 1 : 0;
  c.wall_z_hi = o.wall_z_hi ? 1 : 0;
  c.q_clamp_min = o.q_clamp_min;
  return c;
}
}  // namespace detail

inline VoxelGeometry voxelize(const SpherePack& pack, Dims dims, const VoxelizeOptions& opt) {
  detail::PackArrays pa(pack);
  const int32_t d[3] = {dims.nx, dims.ny, dims.nz};
  const pgpu_voxelize_options o = detail::opts(opt);
  pgpu_voxel_geometry* h = nullptr;
  check(pgpu_voxelize(&pa.c, d, &o, &h));
  return VoxelGeometry(h);
}

inline VoxelGeometry make_box_geometry(Dims dims, const VoxelizeOptions& opt) {
  const int32_t d[3] = {dims.nx, dims.ny, dims.nz};
  const pgpu_voxelize_options o = detail::opts(opt);
  pgpu_voxel_geometry* h = nullptr;
  check(pgpu_make_box_geometry(d, &o, &h));
  return VoxelGeometry(h);
}

// Local x-slab [x0, x1) of voxelize(pack, dims, opt) plus the ghost-column
// flags (multi-GPU runs, DistSimulation below); byte-identical to the
// corresponding columns of the single-domain geometry.
inline VoxelGeometry voxelize_slab(const SpherePack& pack, Dims dims, const VoxelizeOptions& opt,
                                   int x0, int x1) {
  detail::PackArrays pa(pack);
  const int32_t d[3] = {dims.nx, dims.ny, dims.nz};
  const pgpu_voxelize_options o = detail::opts(opt);
  pgpu_voxel_geometry* h = nullptr;
  check(pgpu_voxelize_slab(&pa.c, d, &o, x0, x1, &h));
  return VoxelGeometry(h);
}

// simulation.hpp:45-48: porosity-bearing equilibrium (quadratic terms / eps)
inline std::array<double, kQ> glbm_equilibrium(double delta_rho, const Vec3& u, double eps,
                                               double rho0 = 1.0) {
  std::array<double, kQ> f;
  check(pgpu_glbm_equilibrium(delta_rho, u.data(), eps, rho0, f.data()));
  return f;
}

using PeriodicAxes = std::array<bool, 3>;  // field.hpp:25

// DriveMode / DriveSpec / resolve_drive (boundary.hpp:24-38)
enum class DriveMode : std::uint8_t { BodyForce, PressureGradientAsForce };
struct DriveSpec {
  DriveMode mode = DriveMode::BodyForce;
  Vec3 magnitude{0.0, 0.0, 0.0};  // body force, or Delta_p on the stream axis
  PeriodicAxes periodic_axes{true, true, false};
  int stream_axis = 0;
  double channel_length = 0.0;  // required for PressureGradientAsForce
};
inline Vec3 resolve_drive(const DriveSpec& spec) {
  pgpu_drive_spec c{};
  c.mode = spec.mode == DriveMode::BodyForce ? PGPU_DRIVE_BODY_FORCE
                                             : PGPU_DRIVE_PRESSURE_GRADIENT_AS_FORCE;
  for (int i = 0; i < 3; ++i) {
    c.magnitude[i] = spec.magnitude[i];
    c.periodic_axes[i] = spec.periodic_axes[i] ? 1 : 0;
  }
  c.stream_axis = spec.stream_axis;
  c.channel_length = spec.channel_length;
  Vec3 g;
  check(pgpu_resolve_drive(&c, g.data()));
  return g;
}

// LatticeField (field.hpp:30-68) as host storage, for the free stream() below.
class LatticeField {
 public:
  LatticeField() = default;
  LatticeField(Dims dims, std::vector<std::uint8_t> flags)
      : dims_(dims), flags_(std::move(flags)),
        cur_(static_cast<std::size_t>(kQ * dims.cells()), 0.0),
        nxt_(static_cast<std::size_t>(kQ * dims.cells()), 0.0) {}
  const Dims& dims() const { return dims_; }
  std::int64_t cells() const { return dims_.cells(); }
  const std::vector<std::uint8_t>& flags() const { return flags_; }
  bool is_fluid(std::int64_t c) const { return flags_[static_cast<std::size_t>(c)] == 0; }
  double* cur(int k) { return cur_.data() + static_cast<std::size_t>(k) * cells(); }
  const double* cur(int k) const { return cur_.data() + static_cast<std::size_t>(k) * cells(); }
  double* next(int k) { return nxt_.data() + static_cast<std::size_t>(k) * cells(); }
  const double* next(int k) const { return nxt_.data() + static_cast<std::size_t>(k) * cells(); }
  void swap_buffers() { cur_.swap(nxt_); }

 private:
  Dims dims_;
  std::vector<std::uint8_t> flags_;
  std::vector<double> cur_, nxt_;
};

// simulation.hpp:113-116: streaming over fluid-fluid pairs + buffer swap, on
// the device (pgpu_stream_field; boundary links are not applied).
inline void stream(LatticeField& field, const PeriodicAxes& periodic, int device = 0) {
  const int32_t d[3] = {field.dims().nx, field.dims().ny, field.dims().nz};
  const uint8_t per[3] = {periodic[0], periodic[1], periodic[2]};
  check(pgpu_stream_field(d, per, field.flags().data(), field.cur(0), field.next(0), device));
}

struct GlbmPlaneParams {  // simulation.hpp:18-27
  std::vector<double> eps, permeability, omega_plus, omega_minus;
  double forchheimer_cf = 0.0;
  bool eps_in_equilibrium = true;
};

inline std::vector<double> kozeny_carman(const std::vector<double>& eps, double d,
                                         double free_threshold = 0.999) {
  std::vector<double> K(eps.size());
  check(pgpu_kozeny_carman(static_cast<int32_t>(eps.size()), eps.data(), d, free_threshold,
                           K.data()));
  return K;
}

inline GlbmPlaneParams make_glbm_params(const std::vector<double>& eps,
                                        const std::vector<double>& K, double c_F, double nu,
                                        double lambda, GlbmViscosity mode, double J = 1.0) {
  if (eps.size() != K.size())
    throw ConfigError("porosity and permeability profiles must have equal length");
  GlbmPlaneParams p{eps, K, std::vector<double>(eps.size()), std::vector<double>(eps.size()),
                    c_F, true};
  check(pgpu_make_glbm_params(static_cast<int32_t>(eps.size()), eps.data(), K.data(), c_F, nu,
                              lambda, static_cast<int32_t>(mode), J, p.omega_plus.data(),
                              p.omega_minus.data()));
  return p;
}

struct ProfileData {  // profile.hpp:12-34
  std::vector<double> z, u_superficial, u_intrinsic, epsilon, u_normalized;
  double u_max = 0.0, height = 0.0, z0 = 0.0, nu = 0.0;
  Vec3 body_force{0.0, 0.0, 0.0};
  int stream_axis = 0;
  std::size_t size() const { return z.size(); }
};

// geometry.hpp:86-88: per-plane porosity from the flags, zero velocity columns
inline ProfileData porosity_profile(const VoxelGeometry& geom) {
  const std::size_t nz = static_cast<std::size_t>(geom.dims().nz);
  ProfileData p;
  p.z.resize(nz);
  p.epsilon.resize(nz);
  p.u_superficial.assign(nz, 0.0);
  p.u_intrinsic.assign(nz, 0.0);
  p.u_normalized.assign(nz, 0.0);
  check(pgpu_porosity_profile(&geom.c(), p.z.data(), p.epsilon.data()));
  return p;
}

struct SteadyConfig {  // simulation.hpp:118-123
  double tolerance = 1e-8;
  int check_interval = 1000;
  long max_steps = 2000000;
  double max_speed = 0.3 / 1.7320508075688772;
};

struct RunStats {  // simulation.hpp:125-132
  long steps = 0;
  double mlups = 0.0;
  double seconds = 0.0;
  bool converged = false;
  double residual = 0.0;
  int cli_fallbacks = 0;
};

namespace detail {
inline ProfileData profile_from(std::vector<double> b[5], const pgpu_profile_meta& m) {
  ProfileData p;
  const std::size_t n = static_cast<std::size_t>(m.n_planes);
  for (auto* v : {&b[0], &b[1], &b[2], &b[3], &b[4]}) v->resize(n);
  p.z = b[0];
  p.u_superficial = b[1];
  p.u_intrinsic = b[2];
  p.epsilon = b[3];
  p.u_normalized = b[4];
  p.u_max = m.u_max;
  p.height = m.height;
  p.z0 = m.z0;
  p.nu = m.nu;
  p.body_force = {m.body_force[0], m.body_force[1], m.body_force[2]};
  p.stream_axis = m.stream_axis;
  return p;
}
}  // namespace detail

// porolb::Simulation on the B200 (simulation.hpp:53-111).
class Simulation {
 public:
  Simulation(const VoxelGeometry& geom, const FluidParams& params, WallScheme scheme,
             int device = 0)
      : dims_(geom.dims()) {
    const pgpu_fluid_params p = params.c();
    pgpu_sim* s = nullptr;
    check(pgpu_create(&geom.c(), &p, static_cast<int32_t>(scheme), device, &s));
    h_.reset(s);
  }

  void set_body_force(const Vec3& g) { check(pgpu_set_body_force(h(), g.data())); }
  FluidParams params() const {
    pgpu_fluid_params p;
    check(pgpu_get_params(h(), &p));
    FluidParams f;
    f.nu = p.nu;
    f.omega_plus = p.omega_plus;
    f.omega_minus = p.omega_minus;
    f.lambda_magic = p.lambda_magic;
    f.rho0 = p.rho0;
    f.body_force = {p.body_force[0], p.body_force[1], p.body_force[2]};
    return f;
  }
  void set_lid_velocity(const Vec3& u) { check(pgpu_set_lid_velocity(h(), u.data())); }
  void set_porous(const GlbmPlaneParams& g) {
    check(pgpu_set_porous(h(), static_cast<int32_t>(g.eps.size()), g.eps.data(),
                          g.permeability.data(), g.omega_plus.data(), g.omega_minus.data(),
                          g.forchheimer_cf, g.eps_in_equilibrium ? 1 : 0));
    porous_ = true;
  }
  bool porous() const { return porous_; }
  void step() { check(pgpu_step(h(), 1)); }
  void step(long n) { check(pgpu_step(h(), n)); }
  long steps_done() const {
    int64_t n;
    check(pgpu_steps_done(h(), &n));
    return static_cast<long>(n);
  }
  const Dims& dims() const { return dims_; }
  int cli_fallback_count() const {
    int32_t n;
    check(pgpu_cli_fallback_count(h(), &n));
    return n;
  }
  std::int64_t fluid_cells() const {
    int64_t n;
    check(pgpu_fluid_cells(h(), &n));
    return n;
  }
  void macroscopic(std::int64_t cell, double& delta_rho, Vec3& u) const {
    check(pgpu_macroscopic(h(), cell, &delta_rho, u.data()));
  }
  ProfileData planar_profile(int stream_axis = 0) const {
    std::vector<double> b[5];
    for (auto& v : b) v.resize(static_cast<std::size_t>(dims_.nz));
    pgpu_profile_meta m;
    check(pgpu_planar_profile(h(), stream_axis, b[0].data(), b[1].data(), b[2].data(),
                              b[3].data(), b[4].data(), &m));
    return detail::profile_from(b, m);
  }
  double max_speed() const {
    double v;
    check(pgpu_max_speed(h(), &v));
    return v;
  }
  void initialize_equilibrium(double delta_rho, const Vec3& u) {
    check(pgpu_initialize_equilibrium(h(), delta_rho, u.data()));
  }
  // field().cur(k) / cell_populations (field.hpp:48-60) as explicit copies
  std::vector<double> pdfs() const {
    std::vector<double> f(static_cast<std::size_t>(kQ * dims_.cells()));
    check(pgpu_get_pdfs(h(), f.data()));
    return f;
  }
  void set_pdfs(const std::vector<double>& f) { check(pgpu_set_pdfs(h(), f.data())); }
  std::array<double, kQ> cell_populations(std::int64_t cell) const {
    std::array<double, kQ> f;
    check(pgpu_get_cell_populations(h(), cell, f.data()));
    return f;
  }
  void set_cell_populations(std::int64_t cell, const std::array<double, kQ>& f) {
    check(pgpu_set_cell_populations(h(), cell, f.data()));
  }
  void synchronize() const { check(pgpu_synchronize(h())); }
  pgpu_sim* handle() const { return h(); }

 private:
  struct Del {
    void operator()(pgpu_sim* s) const { pgpu_destroy(s); }
  };
  pgpu_sim* h() const { return h_.get(); }
  std::unique_ptr<pgpu_sim, Del> h_;
  Dims dims_;
  bool porous_ = false;
};

// porolb::Simulation over P GPUs (x slabs, 5-PDF ghost exchange; dist.cpp).
// Local: every slab's Simulation lives in this process (devices may differ,
// exchange by peer copies).  NCCL: one slab per process; rank 0 makes the id
// with nccl_unique_id() and the caller distributes it (MPI, a file, ...).
class DistSimulation {
 public:
  explicit DistSimulation(const std::vector<Simulation*>& slabs) {
    std::vector<pgpu_sim*> h;
    for (Simulation* s : slabs) h.push_back(s->handle());
    pgpu_dist* d = nullptr;
    check(pgpu_dist_create_local(h.data(), static_cast<int32_t>(h.size()), &d));
    d_.reset(d);
    nz_ = slabs.front()->dims().nz;
  }
  DistSimulation(Simulation& slab, const std::array<std::uint8_t, 128>& nccl_id, int rank,
                 int world) {
    pgpu_dist* d = nullptr;
    check(pgpu_dist_create_nccl(slab.handle(), nccl_id.data(), rank, world, &d));
    d_.reset(d);
    nz_ = slab.dims().nz;
  }
  // IPC transport (one rank per process on one node): the edge kernel stores
  // into the neighbours' ghost buffers.  `allgather` receives this rank's
  // blob and returns all ranks' blobs in rank order (MPI_Allgather, a file
  // exchange, ...).
  using Allgather = std::function<std::vector<std::uint8_t>(const std::vector<std::uint8_t>&)>;
  static DistSimulation ipc(Simulation& slab, int rank, int world, const Allgather& allgather) {
    DistSimulation ds;
    pgpu_dist* d = nullptr;
    check(pgpu_dist_create_ipc(slab.handle(), rank, world, &d));
    ds.d_.reset(d);
    ds.nz_ = slab.dims().nz;
    int64_t n = 0;
    check(pgpu_dist_ipc_blob_size(&n));
    std::vector<std::uint8_t> blob(static_cast<std::size_t>(n));
    check(pgpu_dist_ipc_export(d, blob.data()));
    const std::vector<std::uint8_t> all = allgather(blob);
    if (all.size() != blob.size() * static_cast<std::size_t>(world))
      throw std::invalid_argument("allgather must return world blobs");
    check(pgpu_dist_ipc_connect(d, all.data()));
    return ds;
  }
  static std::array<std::uint8_t, 128> nccl_unique_id() {
    std::array<std::uint8_t, 128> id;
    check(pgpu_dist_nccl_unique_id(id.data()));
    return id;
  }
  void step(long n = 1) { check(pgpu_dist_step(d_.get(), n)); }
  void synchronize() const { check(pgpu_dist_synchronize(d_.get())); }
  // global observables (simulation.cpp:371-434 over all slabs)
  ProfileData planar_profile(int stream_axis = 0) const {
    std::vector<double> b[5];
    for (auto& v : b) v.resize(static_cast<std::size_t>(nz_));
    pgpu_profile_meta m;
    check(pgpu_dist_planar_profile(d_.get(), stream_axis, b[0].data(), b[1].data(), b[2].data(),
                                   b[3].data(), b[4].data(), &m));
    return detail::profile_from(b, m);
  }
  double max_speed() const {
    double v2;
    int32_t fin;
    check(pgpu_dist_max_speed2(d_.get(), &v2, &fin));
    return fin ? std::sqrt(v2) : std::numeric_limits<double>::quiet_NaN();
  }

 private:
  DistSimulation() = default;
  struct Del {
    void operator()(pgpu_dist* d) const { pgpu_dist_destroy(d); }
  };
  std::unique_ptr<pgpu_dist, Del> d_;
  int nz_ = 0;
};

// simulation.hpp:134-138
inline RunStats run_to_steady_state(Simulation& sim, const SteadyConfig& cfg,
                                    ProfileData* final_profile = nullptr) {
  pgpu_steady_config c{cfg.tolerance, cfg.check_interval, cfg.max_steps, cfg.max_speed};
  pgpu_run_stats s;
  std::vector<double> b[5];
  for (auto& v : b) v.resize(static_cast<std::size_t>(sim.dims().nz));
  pgpu_profile_meta m;
  check(pgpu_run_to_steady_state(sim.handle(), &c, &s, b[0].data(), b[1].data(), b[2].data(),
                                 b[3].data(), b[4].data(), &m));
  if (final_profile) *final_profile = detail::profile_from(b, m);
  RunStats r;
  r.steps = static_cast<long>(s.steps);
  r.mlups = s.mlups;
  r.seconds = s.seconds;
  r.converged = s.converged != 0;
  r.residual = s.residual;
  r.cli_fallbacks = s.cli_fallbacks;
  return r;
}

// ---- file formats (io.hpp:11-44), native writers in libporolb_cuda.so ----------
inline std::string format_double(double v) {  // io.cpp:11-15
  char buf[32];
  check(pgpu_format_double(v, buf, sizeof buf));
  return buf;
}

inline void write_profile_csv(const std::string& path, const ProfileData& p) {
  pgpu_profile_meta m{};
  m.n_planes = static_cast<int32_t>(p.z.size());
  m.u_max = p.u_max;
  m.height = p.height;
  m.z0 = p.z0;
  m.nu = p.nu;
  for (int a = 0; a < 3; ++a) m.body_force[a] = p.body_force[a];
  m.stream_axis = p.stream_axis;
  check(pgpu_write_profile_csv(path.c_str(), &m, p.z.data(), p.u_superficial.data(),
                               p.u_intrinsic.data(), p.epsilon.data(), p.u_normalized.data(),
                               static_cast<int32_t>(p.u_normalized.size())));
}

inline ProfileData read_profile_csv(const std::string& path) {
  pgpu_profile_meta m{};
  int32_t nn = 0;
  check(pgpu_read_profile_csv(path.c_str(), 0, &m, nullptr, nullptr, nullptr, nullptr, nullptr,
                              &nn));
  std::vector<double> b[5];
  for (auto& v : b) v.resize(static_cast<std::size_t>(m.n_planes));
  check(pgpu_read_profile_csv(path.c_str(), m.n_planes, &m, b[0].data(), b[1].data(),
                              b[2].data(), b[3].data(), b[4].data(), &nn));
  ProfileData p = detail::profile_from(b, m);
  p.u_normalized.resize(static_cast<std::size_t>(nn));
  return p;
}

inline void write_comparison_csv(const std::string& path, const ProfileData& a,
                                 const std::string& name_a, const ProfileData& b,
                                 const std::string& name_b) {
  check(pgpu_write_comparison_csv(path.c_str(), static_cast<int32_t>(a.z.size()), a.z.data(),
                                  a.u_superficial.data(), name_a.c_str(),
                                  static_cast<int32_t>(b.z.size()), b.z.data(),
                                  b.u_superficial.data(), name_b.c_str()));
}

inline void write_report(const std::string& path,
                         const std::vector<std::pair<std::string, std::string>>& entries) {
  std::vector<const char*> k, v;
  for (const auto& e : entries) {
    k.push_back(e.first.c_str());
    v.push_back(e.second.c_str());
  }
  check(pgpu_write_report(path.c_str(), static_cast<int32_t>(k.size()), k.data(), v.data()));
}

inline void write_vtk(const std::string& path, const Simulation& sim) {
  check(pgpu_write_vtk(path.c_str(), sim.handle()));
}

inline void write_sphere_csv(const std::string& path, const SpherePack& pack) {
  detail::PackArrays pa(pack);
  check(pgpu_write_sphere_csv(path.c_str(), &pa.c, pack.seed));
}

inline SpherePack read_sphere_csv(const std::string& path) {
  int64_t n = 0;
  SpherePack p;
  double box[3];
  check(pgpu_read_sphere_csv(path.c_str(), 0, &n, nullptr, nullptr, nullptr, nullptr, box,
                             &p.bottom_plate_z, &p.seed, &p.achieved_height));
  std::vector<double> c[4];
  for (auto& v : c) v.resize(static_cast<std::size_t>(n));
  check(pgpu_read_sphere_csv(path.c_str(), n, &n, c[0].data(), c[1].data(), c[2].data(),
                             c[3].data(), box, &p.bottom_plate_z, &p.seed, &p.achieved_height));
  p.box = {box[0], box[1], box[2]};
  for (int64_t i = 0; i < n; ++i) p.spheres.push_back({{c[0][i], c[1][i], c[2][i]}, c[3][i]});
  return p;
}

inline void write_voxel_file(const std::string& path, const VoxelGeometry& g) {
  check(pgpu_write_voxel_file(path.c_str(), &g.c()));
}

inline VoxelGeometry read_voxel_file(const std::string& path) {
  pgpu_voxel_geometry* h = nullptr;
  check(pgpu_read_voxel_file(path.c_str(), &h));
  return VoxelGeometry(h);
}

}  // namespace porolb_gpu
