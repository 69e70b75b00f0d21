// Lattice-level host functions of the drop-in API.  Same formulas and
// operation order as the reference (cited per function); -ffp-contract=off.
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <sstream>

#include "host_common.h"

namespace pgpu {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

// lattice.cpp:58-75
void relaxation_from_magic(double nu, double lam, pgpu_fluid_params* p) {
  if (!(nu > 0.0)) throw ConfigError("viscosity must be positive");
  if (!(lam > 0.0)) throw ConfigError("magic parameter must be positive");
  p->nu = nu;
  p->lambda_magic = lam;
  p->rho0 = 1.0;
  p->body_force[0] = p->body_force[1] = p->body_force[2] = 0.0;
  p->omega_plus = 1.0 / (3.0 * nu + 0.5);
  p->omega_minus = 1.0 / (lam / (1.0 / p->omega_plus - 0.5) + 0.5);
  for (double w : {p->omega_plus, p->omega_minus}) {
    if (!(w > 0.0 && w < 2.0)) {
      std::ostringstream os;
      os << "relaxation rates out of (0,2): omega+=" << p->omega_plus
         << " omega-=" << p->omega_minus << " (nu=" << nu << ", lambda=" << lam << ")";
      throw ConfigError(os.str());
    }
  }
}

// lattice.cpp:77-86
void equilibrium(double drho, const double u[3], double rho0, double out[19]) {
  const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int k = 0; k < 19; ++k) {
    const double eu = kE[k][0] * u[0] + kE[k][1] * u[1] + kE[k][2] * u[2];
    out[k] = weight(k) * (drho + rho0 * (3.0 * eu + 4.5 * eu * eu - 1.5 * uu));
  }
}

// simulation.cpp:68-78 (glbm_equilibrium): quadratic terms scaled by 1/eps
void glbm_equilibrium(double drho, const double u[3], double eps, double rho0, double out[19]) {
  if (!(eps > 0.0)) throw ConfigError("porosity must be positive");
  const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];  // lattice.hpp:13 dot
  for (int k = 0; k < 19; ++k) {
    const double eu = kE[k][0] * u[0] + kE[k][1] * u[1] + kE[k][2] * u[2];
    out[k] = weight(k) * (drho + rho0 * (3.0 * eu + (4.5 * eu * eu - 1.5 * uu) / eps));
  }
}

// lattice.cpp:88-101
void moments(const double f[19], double rho0, double& drho, double u[3]) {
  drho = 0.0;
  u[0] = u[1] = u[2] = 0.0;
  for (int k = 0; k < 19; ++k) {
    drho += f[k];
    u[0] += kE[k][0] * f[k];
    u[1] += kE[k][1] * f[k];
    u[2] += kE[k][2] * f[k];
  }
  u[0] /= rho0;
  u[1] /= rho0;
  u[2] /= rho0;
}

// simulation.cpp:52-66
void glbm_force_and_velocity(const double mom[3], double eps, double K, double cf,
                             const double g[3], double nu, double u[3], double force[3]) {
  if (!(eps > 0.0)) throw ConfigError("porosity must be positive");
  double vhat[3];
  for (int i = 0; i < 3; ++i) vhat[i] = mom[i] + 0.5 * eps * g[i];
  const double c0 = 0.5 * (1.0 + eps * nu / (2.0 * K));
  const double c1 = 0.5 * eps * cf / std::sqrt(K);
  const double disc =
      c0 * c0 + c1 * std::sqrt(vhat[0] * vhat[0] + vhat[1] * vhat[1] + vhat[2] * vhat[2]);
  if (disc < 0.0) throw NumericalInstability("negative discriminant in drag velocity solve");
  const double denom = c0 + std::sqrt(disc);
  for (int i = 0; i < 3; ++i) u[i] = vhat[i] / denom;
  const double drag_lin = eps * nu / K;
  const double drag_quad =
      eps * cf / std::sqrt(K) * std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  for (int i = 0; i < 3; ++i) force[i] = -(drag_lin + drag_quad) * u[i] + eps * g[i];
}

}  // namespace pgpu

using namespace pgpu;

extern "C" {

const char* pgpu_last_error(void) { return g_last_error.c_str(); }
int pgpu_abi_version(void) { return PGPU_ABI_VERSION; }

#ifndef PGPU_KERNEL_HASH
#define PGPU_KERNEL_HASH "unknown"
#endif
// "kernel_hash=<16 hex>": sha256 of the sweep kernels' sources + nvcc flags
// (paper_1507_06565_b200/build.py kernel_hash); keys profiles/ncu_traffic.json.
int pgpu_build_info(char* buf, int32_t cap) {
  return guard([&] {
    if (!buf || cap <= 0) throw std::invalid_argument("null buffer");
    std::snprintf(buf, (size_t)cap, "kernel_hash=%s", PGPU_KERNEL_HASH);
  });
}

int pgpu_relaxation_from_magic(double nu, double lambda_magic, pgpu_fluid_params* out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output");
    relaxation_from_magic(nu, lambda_magic, out);
  });
}

int pgpu_equilibrium(double delta_rho, const double u[3], double rho0, double out[19]) {
  return guard([&] {
    if (!u || !out) throw std::invalid_argument("null pointer");
    equilibrium(delta_rho, u, rho0, out);
  });
}

// simulation.hpp:45-48, simulation.cpp:68-78
int pgpu_glbm_equilibrium(double delta_rho, const double u[3], double eps, double rho0,
                          double out[19]) {
  return guard([&] {
    if (!u || !out) throw std::invalid_argument("null pointer");
    glbm_equilibrium(delta_rho, u, eps, rho0, out);
  });
}

// boundary.hpp:24-38, boundary.cpp:9-17.  One tightening: a stream axis
// outside 0..2 (the reference would index past the vector) is a ConfigError.
int pgpu_resolve_drive(const pgpu_drive_spec* spec, double g_out[3]) {
  return guard([&] {
    if (!spec || !g_out) throw std::invalid_argument("null pointer");
    if (spec->mode == PGPU_DRIVE_BODY_FORCE) {
      for (int i = 0; i < 3; ++i) g_out[i] = spec->magnitude[i];
      return;
    }
    if (spec->mode != PGPU_DRIVE_PRESSURE_GRADIENT_AS_FORCE) throw ConfigError("unknown drive mode");
    if (!(spec->channel_length > 0.0))
      throw ConfigError("pressure drive requires a positive channel length");
    if (spec->stream_axis < 0 || spec->stream_axis > 2) throw ConfigError("stream axis must be 0, 1 or 2");
    double g[3] = {0.0, 0.0, 0.0};
    g[spec->stream_axis] = spec->magnitude[spec->stream_axis] / spec->channel_length;
    for (int i = 0; i < 3; ++i) g_out[i] = g[i];
  });
}

// geometry.hpp:86-88, geometry.cpp:642-661: per-plane porosity recounted from
// the flags (z at cell centres); the velocity columns of the reference's
// ProfileData are zero and are filled by the C++/Python mirrors.
int pgpu_porosity_profile(const pgpu_geometry* g, double* z_out, double* eps_out) {
  return guard([&] {
    if (!g || !g->flags || !z_out || !eps_out) throw std::invalid_argument("null pointer");
    const int nx = g->dims[0], ny = g->dims[1], nz = g->dims[2];
    if (nx <= 0 || ny <= 0 || nz <= 0) throw ConfigError("voxel dims must be positive");
    const int64_t plane = (int64_t)nx * ny;
    for (int z = 0; z < nz; ++z) {
      const uint8_t* f = g->flags + plane * z;
      int64_t fluid = 0;
      for (int64_t i = 0; i < plane; ++i) fluid += f[i] == 0;
      z_out[z] = z + 0.5;
      eps_out[z] = static_cast<double>(fluid) / (static_cast<double>(nx) * ny);
    }
  });
}

// lattice.cpp:103-128
int pgpu_trt_collide(const double f[19], const pgpu_fluid_params* p, double out[19]) {
  return guard([&] {
    if (!f || !p || !out) throw std::invalid_argument("null pointer");
    double drho, u[3], feq[19];
    moments(f, p->rho0, drho, u);
    equilibrium(drho, u, p->rho0, feq);
    double o[19];
    for (int k = 0; k < 19; ++k) {
      const int kb = opposite(k);
      const double fp = 0.5 * (f[k] + f[kb]);
      const double fm = 0.5 * (f[k] - f[kb]);
      const double ep = 0.5 * (feq[k] + feq[kb]);
      const double em = 0.5 * (feq[k] - feq[kb]);
      const double eg = kE[k][0] * p->body_force[0] + kE[k][1] * p->body_force[1] +
                        kE[k][2] * p->body_force[2];
      o[k] = f[k] - p->omega_plus * (fp - ep) - p->omega_minus * (fm - em) +
             3.0 * weight(k) * p->rho0 * eg;
    }
    for (double v : o)
      if (!std::isfinite(v)) throw NumericalInstability("non-finite population after collision");
    std::memcpy(out, o, sizeof(o));
  });
}

// glbm.cpp:90-111 (the optional calibration is not part of this path)
int pgpu_kozeny_carman(int32_t n, const double* eps, double grain_diameter,
                       double free_threshold, double* K_out) {
  return guard([&] {
    if (n < 0 || (n > 0 && (!eps || !K_out))) throw std::invalid_argument("bad arrays");
    const double factor = 1.0;
    for (int32_t i = 0; i < n; ++i) {
      const double e = eps[i];
      if (e >= free_threshold) {
        K_out[i] = std::numeric_limits<double>::infinity();
      } else {
        K_out[i] = factor * (e * e * e * grain_diameter * grain_diameter /
                             (180.0 * (1.0 - e) * (1.0 - e)));
      }
    }
  });
}

// simulation.cpp:23-50
int pgpu_make_glbm_params(int32_t n, const double* eps, const double* K, double c_F, double nu,
                          double lambda_magic, int32_t mode, double J, double* wp_out,
                          double* wm_out) {
  return guard([&] {
    (void)K;
    (void)c_F;
    if (n < 0 || (n > 0 && (!eps || !wp_out || !wm_out))) throw std::invalid_argument("bad arrays");
    for (int32_t i = 0; i < n; ++i) {
      if (!(eps[i] > 0.0 && eps[i] <= 1.0)) throw ConfigError("porosity must lie in (0, 1]");
      double nu_eff = nu;
      switch (mode) {
        case PGPU_VISC_PLAIN: break;
        case PGPU_VISC_RESCALED: nu_eff = nu / eps[i]; break;
        case PGPU_VISC_CONSTANT_RATIO: nu_eff = (eps[i] < 1.0) ? J * nu : nu; break;
        default: throw ConfigError("unknown GLBM viscosity mode");
      }
      pgpu_fluid_params fp;
      relaxation_from_magic(nu_eff, lambda_magic, &fp);
      wp_out[i] = fp.omega_plus;
      wm_out[i] = fp.omega_minus;
    }
  });
}

int pgpu_glbm_force_and_velocity(const double momentum[3], double eps, double K, double c_F,
                                 const double g[3], double nu, double u_out[3],
                                 double force_out[3]) {
  return guard([&] {
    if (!momentum || !g || !u_out || !force_out) throw std::invalid_argument("null pointer");
    glbm_force_and_velocity(momentum, eps, K, c_F, g, nu, u_out, force_out);
  });
}

}  // extern "C"
