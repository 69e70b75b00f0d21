// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference solver (porolb), compiled
// from the reference's own sources where they lie under /root/reference by
// oracle/Makefile into oracle/_ref/libporolb_ref.so (git-ignored).  Only
// tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs may load it, and only as the checker or the timed CPU baseline.
//
// Every entry point forwards to the reference public API:
//   relaxation_from_magic      proj/src/lattice.cpp:58-75
//   equilibrium / trt_collide  proj/src/lattice.cpp:77-128
//   voxelize / make_box        proj/src/geometry.cpp:491-640
//   Simulation                 proj/src/simulation.cpp:80-434
//   run_to_steady_state        proj/src/simulation.cpp:441-480
//   make_glbm_params           proj/src/simulation.cpp:23-50
//   kozeny_carman              proj/src/glbm.cpp:90-111
//   apply_sbb/cli/moving_wall  proj/src/boundary.cpp:19-41
//   file formats               proj/src/io.cpp:11-278
// Status codes: 0 ok, 1 ConfigError, 2 NumericalInstability, 3 GeometryError,
// 5 other std::exception.
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "porolb/boundary.hpp"
#include "porolb/errors.hpp"
#include "porolb/field.hpp"
#include "porolb/geometry.hpp"
#include "porolb/glbm.hpp"
#include "porolb/io.hpp"
#include "porolb/lattice.hpp"
#include "porolb/simulation.hpp"

using namespace porolb;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalInstability& e) {
    g_err = e.what();
    return 2;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

SpherePack make_pack(int64_t n, const double* cx, const double* cy, const double* cz,
                     const double* r, const double box[3], double plate_z) {
  SpherePack pack;
  pack.box = {box[0], box[1], box[2]};
  pack.bottom_plate_z = plate_z;
  pack.spheres.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    pack.spheres[i].center = {cx[i], cy[i], cz[i]};
    pack.spheres[i].radius = r[i];
  }
  return pack;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

int ref_relaxation_from_magic(double nu, double lam, double* wp, double* wm) {
  return guard([&] {
    const FluidParams p = relaxation_from_magic(nu, lam);
    *wp = p.omega_plus;
    *wm = p.omega_minus;
  });
}

int ref_equilibrium(double drho, const double u[3], double rho0, double out[19]) {
  return guard([&] {
    const Populations f = equilibrium(drho, {u[0], u[1], u[2]}, LatticeModel::d3q19(), rho0);
    std::memcpy(out, f.data(), sizeof(double) * kQ);
  });
}

int ref_trt_collide(const double f[19], double wp, double wm, double rho0, const double g[3],
                    double out[19]) {
  return guard([&] {
    FluidParams p;
    p.omega_plus = wp;
    p.omega_minus = wm;
    p.rho0 = rho0;
    p.body_force = {g[0], g[1], g[2]};
    Populations in;
    std::memcpy(in.data(), f, sizeof(double) * kQ);
    const Populations o = trt_collide(in, p, LatticeModel::d3q19());
    std::memcpy(out, o.data(), sizeof(double) * kQ);
  });
}

// kind: 0 sbb, 1 cli, 2 moving wall. Operates on a fresh field of `dims`
// whose cur buffer is given (19*cells); writes next slot value to *out.
int ref_apply_link(int kind, const int dims[3], const double* cur, int64_t fluid_cell,
                   int64_t second_fluid, int direction, float q, const double uw[3],
                   double rho0, double* out) {
  return guard([&] {
    const Dims d{dims[0], dims[1], dims[2]};
    LatticeField field(d, std::vector<std::uint8_t>(d.cells(), 0));
    for (int k = 0; k < kQ; ++k) std::memcpy(field.cur(k), cur + k * d.cells(), sizeof(double) * d.cells());
    BoundaryLink l;
    l.fluid_cell = fluid_cell;
    l.second_fluid = second_fluid;
    l.direction = direction;
    l.q = q;
    const LatticeModel& m = LatticeModel::d3q19();
    if (kind == 0) apply_sbb(l, field, m);
    else if (kind == 1) apply_cli(l, field, m);
    else apply_moving_wall(l, field, m, {uw[0], uw[1], uw[2]}, rho0);
    *out = field.next(m.opposite[direction])[fluid_cell];
  });
}

int ref_glbm_equilibrium(double drho, const double u[3], double eps, double rho0,
                         double out[19]) {
  return guard([&] {
    const Populations f = glbm_equilibrium(drho, {u[0], u[1], u[2]}, eps, LatticeModel::d3q19(), rho0);
    std::memcpy(out, f.data(), sizeof(double) * kQ);
  });
}

int ref_resolve_drive(int mode, const double mag[3], int stream_axis, double length,
                      double g[3]) {
  return guard([&] {
    DriveSpec spec;
    spec.mode = mode == 0 ? DriveMode::BodyForce : DriveMode::PressureGradientAsForce;
    spec.magnitude = {mag[0], mag[1], mag[2]};
    spec.stream_axis = stream_axis;
    spec.channel_length = length;
    const Vec3 r = resolve_drive(spec);
    for (int i = 0; i < 3; ++i) g[i] = r[i];
  });
}

// free stream() on a field built from the caller's buffers; returns the
// swapped buffers (cur = streamed, next = previous cur).
int ref_stream(const int dims[3], const int periodic[3], const uint8_t* flags, double* cur,
               double* next) {
  return guard([&] {
    const Dims d{dims[0], dims[1], dims[2]};
    LatticeField field(d, std::vector<std::uint8_t>(flags, flags + d.cells()));
    for (int k = 0; k < kQ; ++k) {
      std::memcpy(field.cur(k), cur + k * d.cells(), sizeof(double) * d.cells());
      std::memcpy(field.next(k), next + k * d.cells(), sizeof(double) * d.cells());
    }
    stream(field, {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0});
    for (int k = 0; k < kQ; ++k) {
      std::memcpy(cur + k * d.cells(), field.cur(k), sizeof(double) * d.cells());
      std::memcpy(next + k * d.cells(), field.next(k), sizeof(double) * d.cells());
    }
  });
}

// ---- geometry ----------------------------------------------------------------
int ref_porosity_profile(void* h, double* z, double* eps) {
  return guard([&] {
    const ProfileData p = porosity_profile(*static_cast<VoxelGeometry*>(h));
    for (size_t i = 0; i < p.z.size(); ++i) {
      z[i] = p.z[i];
      eps[i] = p.epsilon[i];
    }
  });
}

int ref_voxelize(int64_t n, const double* cx, const double* cy, const double* cz,
                 const double* r, const double box[3], double plate_z, const int dims[3],
                 const int periodic[3], int wall_lo, int wall_hi, double q_clamp_min,
                 void** out) {
  return guard([&] {
    VoxelizeOptions opt;
    opt.periodic = {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0};
    opt.wall_z_lo = wall_lo != 0;
    opt.wall_z_hi = wall_hi != 0;
    opt.q_clamp_min = q_clamp_min;
    const SpherePack pack = make_pack(n, cx, cy, cz, r, box, plate_z);
    *out = new VoxelGeometry(voxelize(pack, {dims[0], dims[1], dims[2]}, opt));
  });
}

int ref_make_box_geometry(const int dims[3], const int periodic[3], int wall_lo, int wall_hi,
                          void** out) {
  return guard([&] {
    VoxelizeOptions opt;
    opt.periodic = {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0};
    opt.wall_z_lo = wall_lo != 0;
    opt.wall_z_hi = wall_hi != 0;
    *out = new VoxelGeometry(make_box_geometry({dims[0], dims[1], dims[2]}, opt));
  });
}

void ref_geometry_free(void* g) { delete static_cast<VoxelGeometry*>(g); }

// info[0]=n_links info[1]=fluid_cells info[2]=q_fallback_count
// info[3]=has_lo info[4]=has_hi ; planes[0..1] = wall planes
void ref_geometry_info(void* h, int64_t info[5], double planes[2]) {
  const VoxelGeometry& g = *static_cast<VoxelGeometry*>(h);
  info[0] = static_cast<int64_t>(g.links.size());
  info[1] = g.fluid_cells;
  info[2] = g.q_fallback_count;
  info[3] = g.wall_plane_lo.has_value();
  info[4] = g.wall_plane_hi.has_value();
  planes[0] = g.wall_plane_lo.value_or(0.0);
  planes[1] = g.wall_plane_hi.value_or(0.0);
}

void ref_geometry_copy(void* h, uint8_t* flags, double* porosity, int64_t* fluid_cell,
                       int64_t* second_fluid, int32_t* direction, float* q, uint8_t* moving) {
  const VoxelGeometry& g = *static_cast<VoxelGeometry*>(h);
  if (flags) std::memcpy(flags, g.flags.data(), g.flags.size());
  if (porosity) std::memcpy(porosity, g.porosity.data(), sizeof(double) * g.porosity.size());
  for (size_t i = 0; i < g.links.size(); ++i) {
    const BoundaryLink& l = g.links[i];
    if (fluid_cell) fluid_cell[i] = l.fluid_cell;
    if (second_fluid) second_fluid[i] = l.second_fluid;
    if (direction) direction[i] = l.direction;
    if (q) q[i] = l.q;
    if (moving) moving[i] = l.moving ? 1 : 0;
  }
}

// Builds a VoxelGeometry from raw arrays (for hand-made geometries in tests).
int ref_geometry_from_arrays(const int dims[3], const int periodic[3], const uint8_t* flags,
                             int64_t n_links, const int64_t* fluid_cell,
                             const int64_t* second_fluid, const int32_t* direction,
                             const float* q, const uint8_t* moving, const double* porosity,
                             int64_t fluid_cells, int has_lo, double lo, int has_hi, double hi,
                             void** out) {
  return guard([&] {
    auto* g = new VoxelGeometry();
    g->dims = {dims[0], dims[1], dims[2]};
    g->periodic = {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0};
    g->flags.assign(flags, flags + g->dims.cells());
    g->links.resize(static_cast<size_t>(n_links));
    for (int64_t i = 0; i < n_links; ++i) {
      g->links[i].fluid_cell = fluid_cell[i];
      g->links[i].second_fluid = second_fluid[i];
      g->links[i].direction = direction[i];
      g->links[i].q = q[i];
      g->links[i].moving = moving[i] != 0;
    }
    g->porosity.assign(porosity, porosity + g->dims.nz);
    g->fluid_cells = fluid_cells;
    if (has_lo) g->wall_plane_lo = lo;
    if (has_hi) g->wall_plane_hi = hi;
    *out = g;
  });
}

// ---- simulation --------------------------------------------------------------
int ref_sim_create(void* geom, double nu, double wp, double wm, double lam, double rho0,
                   const double g[3], int scheme, void** out) {
  return guard([&] {
    FluidParams p;
    p.nu = nu;
    p.omega_plus = wp;
    p.omega_minus = wm;
    p.lambda_magic = lam;
    p.rho0 = rho0;
    p.body_force = {g[0], g[1], g[2]};
    *out = new Simulation(*static_cast<VoxelGeometry*>(geom), p,
                          scheme == 1 ? WallScheme::CLI : WallScheme::SBB);
  });
}

void ref_sim_free(void* s) { delete static_cast<Simulation*>(s); }

int ref_sim_set_body_force(void* s, const double g[3]) {
  return guard([&] { static_cast<Simulation*>(s)->set_body_force({g[0], g[1], g[2]}); });
}

int ref_sim_set_lid_velocity(void* s, const double u[3]) {
  return guard([&] { static_cast<Simulation*>(s)->set_lid_velocity({u[0], u[1], u[2]}); });
}

int ref_sim_set_porous(void* s, int n, const double* eps, const double* K, const double* wp,
                       const double* wm, double cf, int eps_in_eq) {
  return guard([&] {
    GlbmPlaneParams p;
    p.eps.assign(eps, eps + n);
    p.permeability.assign(K, K + n);
    p.omega_plus.assign(wp, wp + n);
    p.omega_minus.assign(wm, wm + n);
    p.forchheimer_cf = cf;
    p.eps_in_equilibrium = eps_in_eq != 0;
    static_cast<Simulation*>(s)->set_porous(std::move(p));
  });
}

int ref_sim_initialize_equilibrium(void* s, double drho, const double u[3]) {
  return guard([&] { static_cast<Simulation*>(s)->initialize_equilibrium(drho, {u[0], u[1], u[2]}); });
}

int ref_sim_step(void* s, int64_t n) {
  return guard([&] {
    Simulation* sim = static_cast<Simulation*>(s);
    for (int64_t i = 0; i < n; ++i) sim->step();
  });
}

int64_t ref_sim_steps_done(void* s) { return static_cast<Simulation*>(s)->steps_done(); }
int ref_sim_cli_fallbacks(void* s) { return static_cast<Simulation*>(s)->cli_fallback_count(); }

// Whole cur buffer (k-major SoA, 19*cells).
void ref_sim_get_pdfs(void* s, double* out) {
  const LatticeField& f = static_cast<Simulation*>(s)->field();
  std::memcpy(out, f.cur(0), sizeof(double) * kQ * f.cells());
}

void ref_sim_set_pdfs(void* s, const double* in) {
  LatticeField& f = static_cast<Simulation*>(s)->field();
  std::memcpy(f.cur(0), in, sizeof(double) * kQ * f.cells());
}

// Per-cell macroscopic of every fluid cell (non-fluid cells left untouched).
int ref_sim_macroscopic_fields(void* s, double* drho, double* ux, double* uy, double* uz) {
  return guard([&] {
    const Simulation* sim = static_cast<Simulation*>(s);
    const int64_t n = sim->field().cells();
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
      if (!sim->field().is_fluid(c)) continue;
      double d;
      Vec3 u;
      sim->macroscopic(c, d, u);
      drho[c] = d;
      ux[c] = u[0];
      uy[c] = u[1];
      uz[c] = u[2];
    }
  });
}

int ref_sim_macroscopic(void* s, int64_t cell, double* drho, double u[3]) {
  return guard([&] {
    Vec3 v;
    static_cast<Simulation*>(s)->macroscopic(cell, *drho, v);
    u[0] = v[0];
    u[1] = v[1];
    u[2] = v[2];
  });
}

// meta: [u_max, height, z0, nu, g0, g1, g2, stream_axis]; arrays sized nz.
int ref_sim_planar_profile(void* s, int axis, int* n_out, double* z, double* u_sup,
                           double* u_int, double* eps, double* u_norm, double meta[8]) {
  return guard([&] {
    const ProfileData p = static_cast<Simulation*>(s)->planar_profile(axis);
    *n_out = static_cast<int>(p.z.size());
    for (size_t i = 0; i < p.z.size(); ++i) {
      z[i] = p.z[i];
      u_sup[i] = p.u_superficial[i];
      u_int[i] = p.u_intrinsic[i];
      eps[i] = p.epsilon[i];
      u_norm[i] = p.u_normalized[i];
    }
    meta[0] = p.u_max;
    meta[1] = p.height;
    meta[2] = p.z0;
    meta[3] = p.nu;
    meta[4] = p.body_force[0];
    meta[5] = p.body_force[1];
    meta[6] = p.body_force[2];
    meta[7] = p.stream_axis;
  });
}

double ref_sim_max_speed(void* s) { return static_cast<Simulation*>(s)->max_speed(); }

// stats: [steps, mlups, seconds, converged, residual, cli_fallbacks]
int ref_run_to_steady_state(void* s, double tol, int check_interval, int64_t max_steps,
                            double max_speed, double stats[6]) {
  return guard([&] {
    SteadyConfig cfg;
    cfg.tolerance = tol;
    cfg.check_interval = check_interval;
    cfg.max_steps = max_steps;
    cfg.max_speed = max_speed;
    const RunStats r = run_to_steady_state(*static_cast<Simulation*>(s), cfg);
    stats[0] = static_cast<double>(r.steps);
    stats[1] = r.mlups;
    stats[2] = r.seconds;
    stats[3] = r.converged ? 1.0 : 0.0;
    stats[4] = r.residual;
    stats[5] = r.cli_fallbacks;
  });
}

// ---- GLBM parameters -----------------------------------------------------------
int ref_kozeny_carman(int n, const double* eps, double d, double threshold, double* K) {
  return guard([&] {
    const std::vector<double> v = kozeny_carman(std::vector<double>(eps, eps + n), d, threshold);
    std::memcpy(K, v.data(), sizeof(double) * v.size());
  });
}

// mode: 0 Plain, 1 Rescaled, 2 ConstantRatio
int ref_make_glbm_params(int n, const double* eps, const double* K, double cf, double nu,
                         double lam, int mode, double J, double* wp, double* wm) {
  return guard([&] {
    const GlbmPlaneParams p = make_glbm_params(
        std::vector<double>(eps, eps + n), std::vector<double>(K, K + n), cf, nu, lam,
        mode == 0 ? GlbmViscosity::Plain
                  : (mode == 1 ? GlbmViscosity::Rescaled : GlbmViscosity::ConstantRatio),
        J);
    std::memcpy(wp, p.omega_plus.data(), sizeof(double) * n);
    std::memcpy(wm, p.omega_minus.data(), sizeof(double) * n);
  });
}

// ---- file formats (io.cpp) ------------------------------------------------------
int ref_format_double(double v, char* buf, int cap) {
  return guard([&] {
    const std::string t = format_double(v);
    if (static_cast<int>(t.size()) + 1 > cap) throw std::runtime_error("buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}

namespace {
// meta: [u_max, height, z0, nu, g0, g1, g2, stream_axis]
ProfileData make_profile(int n, const double* z, const double* us, const double* ui,
                         const double* eps, int n_norm, const double* un, const double meta[8]) {
  ProfileData p;
  p.z.assign(z, z + n);
  p.u_superficial.assign(us, us + n);
  p.u_intrinsic.assign(ui, ui + n);
  p.epsilon.assign(eps, eps + n);
  if (n_norm > 0) p.u_normalized.assign(un, un + n_norm);
  p.u_max = meta[0];
  p.height = meta[1];
  p.z0 = meta[2];
  p.nu = meta[3];
  p.body_force = {meta[4], meta[5], meta[6]};
  p.stream_axis = static_cast<int>(meta[7]);
  return p;
}
}  // namespace

int ref_write_profile_csv(const char* path, int n, const double* z, const double* us,
                          const double* ui, const double* eps, int n_norm, const double* un,
                          const double meta[8]) {
  return guard([&] { write_profile_csv(path, make_profile(n, z, us, ui, eps, n_norm, un, meta)); });
}

// counts: [rows, n_norm]; arrays filled when rows <= cap
int ref_read_profile_csv(const char* path, int cap, int counts[2], double* z, double* us,
                         double* ui, double* eps, double* un, double meta[8]) {
  return guard([&] {
    const ProfileData p = read_profile_csv(path);
    counts[0] = static_cast<int>(p.z.size());
    counts[1] = static_cast<int>(p.u_normalized.size());
    meta[0] = p.u_max;
    meta[1] = p.height;
    meta[2] = p.z0;
    meta[3] = p.nu;
    meta[4] = p.body_force[0];
    meta[5] = p.body_force[1];
    meta[6] = p.body_force[2];
    meta[7] = p.stream_axis;
    if (counts[0] > cap) return;
    for (size_t i = 0; i < p.z.size(); ++i) {
      z[i] = p.z[i];
      us[i] = p.u_superficial[i];
      ui[i] = p.u_intrinsic[i];
      eps[i] = p.epsilon[i];
    }
    for (size_t i = 0; i < p.u_normalized.size(); ++i) un[i] = p.u_normalized[i];
  });
}

int ref_write_comparison_csv(const char* path, int na, const double* za, const double* ua,
                             const char* name_a, int nb, const double* zb, const double* ub,
                             const char* name_b) {
  return guard([&] {
    ProfileData a, b;
    a.z.assign(za, za + na);
    a.u_superficial.assign(ua, ua + na);
    b.z.assign(zb, zb + nb);
    b.u_superficial.assign(ub, ub + nb);
    write_comparison_csv(path, a, name_a, b, name_b);
  });
}

int ref_write_report(const char* path, int n, const char* const* keys,
                     const char* const* values) {
  return guard([&] {
    std::vector<std::pair<std::string, std::string>> e;
    for (int i = 0; i < n; ++i) e.emplace_back(keys[i], values[i]);
    write_report(path, e);
  });
}

int ref_write_vtk(const char* path, void* s) {
  return guard([&] { write_vtk(path, *static_cast<Simulation*>(s)); });
}

int ref_write_sphere_csv(const char* path, int64_t n, const double* cx, const double* cy,
                         const double* cz, const double* r, const double box[3], double plate_z,
                         uint64_t seed) {
  return guard([&] {
    SpherePack pack = make_pack(n, cx, cy, cz, r, box, plate_z);
    pack.seed = seed;
    write_sphere_csv(path, pack);
  });
}

// extra: [box0, box1, box2, plate_z, achieved_height]; arrays filled when n <= cap
int ref_read_sphere_csv(const char* path, int64_t cap, int64_t* n, double* cx, double* cy,
                        double* cz, double* r, double extra[5], uint64_t* seed) {
  return guard([&] {
    const SpherePack p = read_sphere_csv(path);
    *n = static_cast<int64_t>(p.spheres.size());
    extra[0] = p.box.lx;
    extra[1] = p.box.ly;
    extra[2] = p.box.lz;
    extra[3] = p.bottom_plate_z;
    extra[4] = p.achieved_height;
    *seed = p.seed;
    if (*n > cap) return;
    for (int64_t i = 0; i < *n; ++i) {
      cx[i] = p.spheres[i].center[0];
      cy[i] = p.spheres[i].center[1];
      cz[i] = p.spheres[i].center[2];
      r[i] = p.spheres[i].radius;
    }
  });
}

int ref_write_voxel_file(const char* path, void* g) {
  return guard([&] { write_voxel_file(path, *static_cast<VoxelGeometry*>(g)); });
}

int ref_read_voxel_file(const char* path, void** out) {
  return guard([&] { *out = new VoxelGeometry(read_voxel_file(path)); });
}

}  // extern "C"
