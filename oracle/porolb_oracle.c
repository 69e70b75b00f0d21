/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Plain-C, single-threaded restatement of the reference porolb hot path
 * (D3Q19 TRT collide + push stream + SBB/CLI/moving-wall links, GLBM
 * collision, observables, voxelizer).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load oracle/liboracle.so, and only as
 * the checker.  Each function cites the reference file:line it restates
 * (paths relative to the reference's proj/ directory).  Floating-point
 * operation order follows the reference expression by expression; build with
 * -ffp-contract=off (oracle/Makefile) so no FMA is formed, which is what the
 * reference's own baseline x86-64 -O3 build produces.
 *
 * Parity pinning: tests/test_oracle.py checks this file bit-for-bit against
 * the reference compiled from its own sources (oracle/_ref) and against the
 * committed golden vectors in tests/golden/ (made by tests/golden/make_golden.py
 * from oracle/_ref).
 *
 * Layouts (reference proj/include/porolb/field.hpp:19-21,36-37,48-51):
 *   cell index c = (z*ny + y)*nx + x ; PDF slot f[k*cells + c]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define Q 19

/* lattice.cpp:13-33 -- D3Q19 velocity set, canonical order. */
const int ORC_E[Q][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                         {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                         {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                         {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
double ORC_W[Q];
int ORC_OPP[Q];
static int g_init = 0;

/* lattice.cpp:34-45 -- weights by speed order, opposite = index of -e. */
static void orc_init(void) {
  if (g_init) return;
  for (int k = 0; k < Q; ++k) {
    const int order = abs(ORC_E[k][0]) + abs(ORC_E[k][1]) + abs(ORC_E[k][2]);
    ORC_W[k] = (order == 0) ? 1.0 / 3.0 : (order == 1) ? 1.0 / 18.0 : 1.0 / 36.0;
  }
  for (int k = 0; k < Q; ++k)
    for (int j = 0; j < Q; ++j)
      if (ORC_E[j][0] == -ORC_E[k][0] && ORC_E[j][1] == -ORC_E[k][1] &&
          ORC_E[j][2] == -ORC_E[k][2]) {
        ORC_OPP[k] = j;
        break;
      }
  g_init = 1;
}

void orc_tables(int* e_out, double* w_out, int* opp_out) {
  orc_init();
  for (int k = 0; k < Q; ++k) {
    for (int i = 0; i < 3; ++i) e_out[3 * k + i] = ORC_E[k][i];
    w_out[k] = ORC_W[k];
    opp_out[k] = ORC_OPP[k];
  }
}

/* lattice.cpp:58-75 -- returns 1 (ConfigError) on invalid input/rates. */
int orc_relaxation_from_magic(double nu, double lam, double* wp, double* wm) {
  if (!(nu > 0.0)) return 1;
  if (!(lam > 0.0)) return 1;
  const double p = 1.0 / (3.0 * nu + 0.5);
  const double m = 1.0 / (lam / (1.0 / p - 0.5) + 0.5);
  *wp = p;
  *wm = m;
  if (!(p > 0.0 && p < 2.0)) return 1;
  if (!(m > 0.0 && m < 2.0)) return 1;
  return 0;
}

/* lattice.cpp:77-86 -- fluctuation-form equilibrium. */
void orc_equilibrium(double drho, const double u[3], double rho0, double out[Q]) {
  orc_init();
  const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int k = 0; k < Q; ++k) {
    const double eu = ORC_E[k][0] * u[0] + ORC_E[k][1] * u[1] + ORC_E[k][2] * u[2];
    out[k] = ORC_W[k] * (drho + rho0 * (3.0 * eu + 4.5 * eu * eu - 1.5 * uu));
  }
}

/* lattice.cpp:88-101 */
void orc_moments(const double f[Q], double rho0, double* drho, double u[3]) {
  orc_init();
  double d = 0.0, u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (int k = 0; k < Q; ++k) {
    d += f[k];
    u0 += ORC_E[k][0] * f[k];
    u1 += ORC_E[k][1] * f[k];
    u2 += ORC_E[k][2] * f[k];
  }
  *drho = d;
  u[0] = u0 / rho0;
  u[1] = u1 / rho0;
  u[2] = u2 / rho0;
}

/* lattice.cpp:103-128 -- per-cell TRT, returns 2 (NumericalInstability) on
 * non-finite output. */
int orc_trt_collide(const double f[Q], double wp, double wm, double rho0, const double g[3],
                    double out[Q]) {
  orc_init();
  double drho, u[3], feq[Q];
  orc_moments(f, rho0, &drho, u);
  orc_equilibrium(drho, u, rho0, feq);
  for (int k = 0; k < Q; ++k) {
    const int kb = ORC_OPP[k];
    const double fp = 0.5 * (f[k] + f[kb]);
    const double fm = 0.5 * (f[k] - f[kb]);
    const double ep = 0.5 * (feq[k] + feq[kb]);
    const double em = 0.5 * (feq[k] - feq[kb]);
    const double eg = ORC_E[k][0] * g[0] + ORC_E[k][1] * g[1] + ORC_E[k][2] * g[2];
    out[k] = f[k] - wp * (fp - ep) - wm * (fm - em) + 3.0 * ORC_W[k] * rho0 * eg;
  }
  for (int k = 0; k < Q; ++k)
    if (!isfinite(out[k])) return 2;
  return 0;
}

/* simulation.cpp:132-146 -- pair tables (k = 2p+1, kb = 2p+2). */
static double PX[9], PY[9], PZ[9], PW[9];
static void pair_init(void) {
  orc_init();
  for (int p = 0; p < 9; ++p) {
    const int k = 1 + 2 * p;
    PX[p] = ORC_E[k][0];
    PY[p] = ORC_E[k][1];
    PZ[p] = ORC_E[k][2];
    PW[p] = ORC_W[k];
  }
}

/* simulation.cpp:150-196 -- in-place TRT collide of every fluid cell. */
void orc_collide_core(int64_t cells, const uint8_t* flags, double* f, double wp, double wm,
                      double rho0, const double g[3]) {
  pair_init();
  for (int64_t c = 0; c < cells; ++c) {
    if (flags[c] != 0) continue;
    double fk[Q];
    for (int k = 0; k < Q; ++k) fk[k] = f[k * cells + c];
    double drho = fk[0];
    double vx = 0.0, vy = 0.0, vz = 0.0;
    for (int p = 0; p < 9; ++p) {
      const double a = fk[1 + 2 * p], b = fk[2 + 2 * p];
      drho += a + b;
      vx += PX[p] * (a - b);
      vy += PY[p] * (a - b);
      vz += PZ[p] * (a - b);
    }
    const double ux = vx / rho0, uy = vy / rho0, uz = vz / rho0;
    const double uu = ux * ux + uy * uy + uz * uz;
    const double feq0 = (1.0 / 3.0) * (drho - rho0 * 1.5 * uu);
    fk[0] -= wp * (fk[0] - feq0);
    for (int p = 0; p < 9; ++p) {
      const int k = 1 + 2 * p, kb = k + 1;
      const double eu = PX[p] * ux + PY[p] * uy + PZ[p] * uz;
      const double eg = PX[p] * g[0] + PY[p] * g[1] + PZ[p] * g[2];
      const double feq_p = PW[p] * (drho + rho0 * (4.5 * eu * eu - 1.5 * uu));
      const double feq_m = PW[p] * rho0 * 3.0 * eu;
      const double fp = 0.5 * (fk[k] + fk[kb]);
      const double fm = 0.5 * (fk[k] - fk[kb]);
      const double relax_p = wp * (fp - feq_p);
      const double relax_m = wm * (fm - feq_m);
      const double fpop = 3.0 * PW[p] * rho0 * eg;
      fk[k] += -relax_p - relax_m + fpop;
      fk[kb] += -relax_p + relax_m - fpop;
    }
    for (int k = 0; k < Q; ++k) f[k * cells + c] = fk[k];
  }
}

/* simulation.cpp:198-274 -- GLBM collision with per-plane eps, K, omega+-. */
void orc_collide_glbm(int64_t cells, int64_t plane, const uint8_t* flags, double* f,
                      double rho0, double nu, const double g[3], const double* eps_z,
                      const double* K_z, const double* wp_z, const double* wm_z, double cf,
                      int eps_in_eq) {
  pair_init();
  for (int64_t c = 0; c < cells; ++c) {
    if (flags[c] != 0) continue;
    const int z = (int)(c / plane);
    const double eps = eps_z[z];
    const double K = K_z[z];
    const double wp = wp_z[z];
    const double wm = wm_z[z];
    const double eq_eps = eps_in_eq ? eps : 1.0;
    double fk[Q];
    for (int k = 0; k < Q; ++k) fk[k] = f[k * cells + c];
    double drho = fk[0];
    double vx = 0.0, vy = 0.0, vz = 0.0;
    for (int p = 0; p < 9; ++p) {
      const double a = fk[1 + 2 * p], b = fk[2 + 2 * p];
      drho += a + b;
      vx += PX[p] * (a - b);
      vy += PY[p] * (a - b);
      vz += PZ[p] * (a - b);
    }
    const double vhx = vx / rho0 + 0.5 * eps * g[0];
    const double vhy = vy / rho0 + 0.5 * eps * g[1];
    const double vhz = vz / rho0 + 0.5 * eps * g[2];
    const double c0 = 0.5 * (1.0 + eps * nu / (2.0 * K));
    double denom;
    if (cf == 0.0) {
      denom = 2.0 * c0;
    } else {
      const double c1 = 0.5 * eps * cf / sqrt(K);
      const double vmag = sqrt(vhx * vhx + vhy * vhy + vhz * vhz);
      denom = c0 + sqrt(c0 * c0 + c1 * vmag);
    }
    const double ux = vhx / denom, uy = vhy / denom, uz = vhz / denom;
    const double umag = sqrt(ux * ux + uy * uy + uz * uz);
    const double drag = eps * nu / K + (cf != 0.0 ? eps * cf / sqrt(K) * umag : 0.0);
    const double Fx = -drag * ux + eps * g[0];
    const double Fy = -drag * uy + eps * g[1];
    const double Fz = -drag * uz + eps * g[2];
    const double uu = ux * ux + uy * uy + uz * uz;
    const double force_pref = (1.0 - 0.5 * wm) * 3.0 * rho0;
    const double feq0 = (1.0 / 3.0) * (drho - rho0 * 1.5 * uu / eq_eps);
    fk[0] -= wp * (fk[0] - feq0);
    for (int p = 0; p < 9; ++p) {
      const int k = 1 + 2 * p, kb = k + 1;
      const double eu = PX[p] * ux + PY[p] * uy + PZ[p] * uz;
      const double eF = PX[p] * Fx + PY[p] * Fy + PZ[p] * Fz;
      const double feq_p = PW[p] * (drho + rho0 * (4.5 * eu * eu - 1.5 * uu) / eq_eps);
      const double feq_m = PW[p] * rho0 * 3.0 * eu;
      const double fp = 0.5 * (fk[k] + fk[kb]);
      const double fm = 0.5 * (fk[k] - fk[kb]);
      const double relax_p = wp * (fp - feq_p);
      const double relax_m = wm * (fm - feq_m);
      const double fpop = force_pref * PW[p] * eF;
      fk[k] += -relax_p - relax_m + fpop;
      fk[kb] += -relax_p + relax_m - fpop;
    }
    for (int k = 0; k < Q; ++k) f[k * cells + c] = fk[k];
  }
}

/* simulation.cpp:278-321 -- push streaming, fluid -> fluid, periodic wrap. */
void orc_stream_pass(const int dims[3], const int periodic[3], const uint8_t* flags,
                     const double* cur, double* next) {
  orc_init();
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t cells = (int64_t)nx * ny * nz;
  for (int64_t c = 0; c < cells; ++c)
    if (flags[c] == 0) next[c] = cur[c];
  for (int k = 1; k < Q; ++k) {
    const int ex = ORC_E[k][0], ey = ORC_E[k][1], ez = ORC_E[k][2];
    const double* src = cur + (int64_t)k * cells;
    double* dst = next + (int64_t)k * cells;
    for (int z = 0; z < nz; ++z) {
      for (int y = 0; y < ny; ++y) {
        int zd = z + ez;
        if (zd < 0) zd = periodic[2] ? nz - 1 : -1;
        if (zd >= nz) zd = periodic[2] ? 0 : -1;
        int yd = y + ey;
        if (yd < 0) yd = periodic[1] ? ny - 1 : -1;
        if (yd >= ny) yd = periodic[1] ? 0 : -1;
        if (zd < 0 || yd < 0) continue;
        const int64_t row = ((int64_t)z * ny + y) * nx;
        const int64_t row_d = ((int64_t)zd * ny + yd) * nx;
        for (int x = 0; x < nx; ++x) {
          if (flags[row + x] != 0) continue;
          int xd = x + ex;
          if (xd < 0) xd = periodic[0] ? nx - 1 : -1;
          if (xd >= nx) xd = periodic[0] ? 0 : -1;
          if (xd < 0) continue;
          const int64_t d = row_d + xd;
          if (flags[d] == 0) dst[d] = src[row + x];
        }
      }
    }
  }
}

/* simulation.cpp:330-340 + boundary.cpp:19-41 -- link loop (scheme 1 = CLI). */
void orc_apply_links(int64_t cells, int64_t n_links, const int64_t* fluid_cell,
                     const int64_t* second_fluid, const int32_t* direction, const float* q,
                     const uint8_t* moving, int scheme, const double u_wall[3], double rho0,
                     const double* cur, double* next) {
  orc_init();
  for (int64_t i = 0; i < n_links; ++i) {
    const int k = direction[i];
    const int kb = ORC_OPP[k];
    const int64_t x = fluid_cell[i];
    if (moving && moving[i]) {
      /* boundary.cpp:34-41 ; m.inv_cs2 = 3.0 */
      const double eu =
          ORC_E[k][0] * u_wall[0] + ORC_E[k][1] * u_wall[1] + ORC_E[k][2] * u_wall[2];
      next[kb * cells + x] = cur[k * cells + x] - 2.0 * ORC_W[k] * rho0 * 3.0 * eu;
    } else if (scheme == 1 && second_fluid[i] >= 0) {
      /* boundary.cpp:24-32 */
      const double qq = q[i];
      const double c = (1.0 - 2.0 * qq) / (1.0 + 2.0 * qq);
      next[kb * cells + x] = c * cur[k * cells + second_fluid[i]] - c * cur[kb * cells + x] +
                             cur[k * cells + x];
    } else {
      /* boundary.cpp:19-22 */
      next[kb * cells + x] = cur[k * cells + x];
    }
  }
}

/* lattice.hpp:13-17 */
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* simulation.cpp:52-66 -- returns 1 ConfigError, 2 NumericalInstability. */
int orc_glbm_force_and_velocity(const double mom[3], double eps, double K, double cf,
                                const double g[3], double nu, double u[3], double force[3]) {
  if (!(eps > 0.0)) return 1;
  double vhat[3];
  for (int i = 0; i < 3; ++i) vhat[i] = mom[i] + 0.5 * eps * g[i];
  const double c0 = 0.5 * (1.0 + eps * nu / (2.0 * K));
  const double c1 = 0.5 * eps * cf / sqrt(K);
  const double disc = c0 * c0 + c1 * sqrt(dot3(vhat, vhat));
  if (disc < 0.0) return 2;
  const double denom = c0 + sqrt(disc);
  for (int i = 0; i < 3; ++i) u[i] = vhat[i] / denom;
  const double drag_lin = eps * nu / K;
  const double drag_quad = eps * cf / sqrt(K) * sqrt(dot3(u, u));
  for (int i = 0; i < 3; ++i) force[i] = -(drag_lin + drag_quad) * u[i] + eps * g[i];
  return 0;
}

/* simulation.cpp:68-78 */
int orc_glbm_equilibrium(double drho, const double u[3], double eps, double rho0,
                         double out[Q]) {
  orc_init();
  if (!(eps > 0.0)) return 1;
  const double uu = dot3(u, u);
  for (int k = 0; k < Q; ++k) {
    const double eu = ORC_E[k][0] * u[0] + ORC_E[k][1] * u[1] + ORC_E[k][2] * u[2];
    out[k] = ORC_W[k] * (drho + rho0 * (3.0 * eu + (4.5 * eu * eu - 1.5 * uu) / eps));
  }
  return 0;
}

/* simulation.cpp:354-369 -- macroscopic of one cell from the cur buffer.
 * glbm != 0 selects the porous branch (caller passes the plane's eps, K). */
int orc_macroscopic(const double* cur, int64_t cells, int64_t cell, double rho0,
                    const double g[3], double nu, int glbm, double eps, double K, double cf,
                    double* drho, double u[3]) {
  double fk[Q], v[3];
  for (int k = 0; k < Q; ++k) fk[k] = cur[k * cells + cell];
  orc_moments(fk, rho0, drho, v);
  if (glbm) {
    double force[3];
    return orc_glbm_force_and_velocity(v, eps, K, cf, g, nu, u, force);
  }
  for (int i = 0; i < 3; ++i) u[i] = v[i] + 0.5 * g[i] / rho0;
  return 0;
}

/* simulation.cpp:12-21 */
int orc_glbm_all_free(int n, const double* eps, const double* K, double cf) {
  if (cf != 0.0) return 0;
  for (int i = 0; i < n; ++i)
    if (eps[i] != 1.0) return 0;
  for (int i = 0; i < n; ++i)
    if (isfinite(K[i])) return 0;
  return 1;
}

/* simulation.cpp:371-417 + profile.cpp:10-19.  Arrays sized nz; returns the
 * number of planes in *n_out.  glbm arrays may be NULL (core mode).
 * meta: [u_max, height, z0]. */
int orc_planar_profile(const int dims[3], const uint8_t* flags, const double* cur,
                       const double* porosity, double rho0, const double g[3], double nu,
                       const double* eps_z, const double* K_z, double cf, int axis,
                       int has_lo, double lo, int has_hi, double hi, int* n_out, double* z_out,
                       double* u_sup, double* u_int, double* eps_out, double* u_norm,
                       double meta[3]) {
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t plane = (int64_t)nx * ny;
  const int64_t cells = plane * nz;
  int z_lo = nz, z_hi = -1;
  int64_t* count = (int64_t*)malloc(sizeof(int64_t) * (size_t)nz);
  for (int z = 0; z < nz; ++z) {
    count[z] = (int64_t)llround(porosity[z] * (double)nx * ny);
    if (count[z] > 0) {
      if (z < z_lo) z_lo = z;
      if (z > z_hi) z_hi = z;
    }
  }
  *n_out = 0;
  meta[0] = 0.0;
  if (has_lo && has_hi) {
    meta[2] = lo;
    meta[1] = hi - lo;
  } else {
    meta[2] = 0.0;
    meta[1] = nz;
  }
  if (z_hi < 0) {
    free(count);
    return 0;
  }
  const int glbm = eps_z != NULL && !orc_glbm_all_free(nz, eps_z, K_z, cf);
  for (int z = z_lo; z <= z_hi; ++z) {
    double sum = 0.0;
    for (int64_t c = plane * z; c < plane * (z + 1); ++c) {
      if (flags[c] != 0) continue;
      double drho, u[3];
      const int st = orc_macroscopic(cur, cells, c, rho0, g, nu, glbm, glbm ? eps_z[z] : 1.0,
                                     glbm ? K_z[z] : 0.0, cf, &drho, u);
      if (st) {
        free(count);
        return st;
      }
      sum += u[axis];
    }
    const int i = z - z_lo;
    z_out[i] = z + 0.5;
    u_sup[i] = sum / (double)plane;
    u_int[i] = count[z] > 0 ? sum / (double)count[z] : 0.0;
    eps_out[i] = porosity[z];
  }
  const int n = z_hi - z_lo + 1;
  *n_out = n;
  double umax = 0.0;
  for (int i = 0; i < n; ++i)
    if (fabs(u_sup[i]) > fabs(umax)) umax = u_sup[i];
  for (int i = 0; i < n; ++i) u_norm[i] = (umax != 0.0) ? u_sup[i] / umax : 0.0;
  meta[0] = umax;
  free(count);
  return 0;
}

/* simulation.cpp:419-434 -- NaN if any fluid cell is non-finite. */
double orc_max_speed(const int dims[3], const uint8_t* flags, const double* cur, double rho0,
                     const double g[3], double nu, const double* eps_z, const double* K_z,
                     double cf) {
  const int64_t plane = (int64_t)dims[0] * dims[1];
  const int64_t cells = plane * dims[2];
  const int glbm = eps_z != NULL && !orc_glbm_all_free(dims[2], eps_z, K_z, cf);
  double vmax2 = 0.0;
  int finite = 1;
  for (int64_t c = 0; c < cells; ++c) {
    if (flags[c] != 0) continue;
    const int z = (int)(c / plane);
    double drho, u[3];
    orc_macroscopic(cur, cells, c, rho0, g, nu, glbm, glbm ? eps_z[z] : 1.0,
                    glbm ? K_z[z] : 0.0, cf, &drho, u);
    const double m2 = dot3(u, u);
    finite = finite && isfinite(m2) && isfinite(drho);
    if (m2 > vmax2) vmax2 = m2;
  }
  if (!finite) return NAN;
  return sqrt(vmax2);
}

/* glbm.cpp:90-111 (calibration omitted: never used on the hot path). */
void orc_kozeny_carman(int n, const double* eps, double d, double threshold, double* K) {
  for (int i = 0; i < n; ++i) {
    const double e = eps[i];
    K[i] = (e >= threshold) ? INFINITY : 1.0 * (e * e * e * d * d / (180.0 * (1.0 - e) * (1.0 - e)));
  }
}

/* simulation.cpp:23-50 ; mode 0 Plain, 1 Rescaled, 2 ConstantRatio. */
int orc_make_glbm_params(int n, const double* eps, double nu, double lam, int mode, double J,
                         double* wp, double* wm) {
  for (int i = 0; i < n; ++i) {
    if (!(eps[i] > 0.0 && eps[i] <= 1.0)) return 1;
    double nu_eff = nu;
    if (mode == 1) nu_eff = nu / eps[i];
    if (mode == 2) nu_eff = (eps[i] < 1.0) ? J * nu : nu;
    const int st = orc_relaxation_from_magic(nu_eff, lam, &wp[i], &wm[i]);
    if (st) return st;
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Voxelizer: geometry.cpp:442-632.  Brute-force sphere scan exactly like the
 * reference (O(links x spheres)); small cases only.
 * Returns 0 ok, 1 ConfigError (open face), 3 GeometryError (no fluid),
 * 6 link capacity exceeded.
 * ------------------------------------------------------------------------- */
typedef struct {
  double c[3], r;
} osphere;

/* geometry.cpp:465-479 -- smallest t in (0, 1+1e-12] or -1 for none. */
static int ray_sphere(const double p[3], const int e[3], const osphere* s, double* t_out) {
  const double d[3] = {p[0] - s->c[0], p[1] - s->c[1], p[2] - s->c[2]};
  const double a = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
  const double b = 2.0 * (e[0] * d[0] + e[1] * d[1] + e[2] * d[2]);
  const double c = dot3(d, d) - s->r * s->r;
  const double disc = b * b - 4.0 * a * c;
  if (disc < 0.0) return 0;
  const double sq = sqrt(disc);
  const double ts[2] = {(-b - sq) / (2.0 * a), (-b + sq) / (2.0 * a)};
  int have = 0;
  double best = 0.0;
  for (int i = 0; i < 2; ++i) {
    const double t = ts[i];
    if (t > 0.0 && t <= 1.0 + 1e-12 && (!have || t < best)) {
      best = t;
      have = 1;
    }
  }
  *t_out = best;
  return have;
}

/* geometry.cpp:481-487 */
static int ray_plane_z(const double p[3], const int e[3], double plane_z, double* t_out) {
  if (e[2] == 0) return 0;
  const double t = (plane_z - p[2]) / e[2];
  if (t > 0.0 && t <= 1.0 + 1e-12) {
    *t_out = t;
    return 1;
  }
  return 0;
}

static int wrap_coord(int v, int n, int periodic) {
  if (v >= 0 && v < n) return v;
  if (!periodic) return -1;
  return (v % n + n) % n;
}

int orc_voxelize(int64_t n_sph, const double* cx, const double* cy, const double* cz,
                 const double* cr, const double box[3], double plate_z, const int dims[3],
                 const int periodic[3], int wall_lo, int wall_hi, double q_clamp_min,
                 uint8_t* flags, double* porosity, int64_t cap, int64_t* lf, int64_t* ls,
                 int32_t* ld, float* lq, uint8_t* lm, int64_t* n_links_out,
                 int64_t* fluid_out, int* q_fallback_out) {
  orc_init();
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (nx <= 0 || ny <= 0 || nz <= 0) return 1;
  const int64_t cells = (int64_t)nx * ny * nz;
  memset(flags, 0, (size_t)cells);
#define IDX(x, y, z) ((((int64_t)(z)) * ny + (y)) * nx + (x))

  /* geometry.cpp:442-462 effective_spheres */
  const int ixm = periodic[0] ? 1 : 0, iym = periodic[1] ? 1 : 0;
  osphere* sph = (osphere*)malloc(sizeof(osphere) * (size_t)(n_sph * 9 + 1));
  int64_t ns = 0;
  for (int64_t i = 0; i < n_sph; ++i)
    for (int ix = -ixm; ix <= ixm; ++ix)
      for (int iy = -iym; iy <= iym; ++iy) {
        osphere s;
        s.c[0] = cx[i] + ix * box[0];
        s.c[1] = cy[i] + iy * box[1];
        s.c[2] = cz[i];
        s.r = cr[i];
        if (s.c[0] + s.r < 0.0 || s.c[0] - s.r > nx || s.c[1] + s.r < 0.0 || s.c[1] - s.r > ny)
          continue;
        sph[ns++] = s;
      }

  /* geometry.cpp:501-510 plate */
  if (plate_z > 0.0) {
    const int k_max = (int)floor(plate_z - 0.5);
    for (int z = 0; z <= (k_max < nz - 1 ? k_max : nz - 1); ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) flags[IDX(x, y, z)] = 1;
  }
  /* geometry.cpp:512-533 sphere rasterization */
  for (int64_t i = 0; i < ns; ++i) {
    const osphere* s = &sph[i];
    int x0 = (int)floor(s->c[0] - s->r - 0.5); if (x0 < 0) x0 = 0;
    int x1 = (int)ceil(s->c[0] + s->r); if (x1 > nx - 1) x1 = nx - 1;
    int y0 = (int)floor(s->c[1] - s->r - 0.5); if (y0 < 0) y0 = 0;
    int y1 = (int)ceil(s->c[1] + s->r); if (y1 > ny - 1) y1 = ny - 1;
    int z0 = (int)floor(s->c[2] - s->r - 0.5); if (z0 < 0) z0 = 0;
    int z1 = (int)ceil(s->c[2] + s->r); if (z1 > nz - 1) z1 = nz - 1;
    const double r2 = s->r * s->r;
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const double dx = x + 0.5 - s->c[0];
          const double dy = y + 0.5 - s->c[1];
          const double dz = z + 0.5 - s->c[2];
          if (dx * dx + dy * dy + dz * dz < r2) flags[IDX(x, y, z)] = 1;
        }
  }
  /* geometry.cpp:535-551 wall layers */
  double planes[2];
  int nplanes = 0;
  if (wall_lo) {
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) flags[IDX(x, y, 0)] = 2;
    planes[nplanes++] = 1.0;
  }
  if (wall_hi) {
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) flags[IDX(x, y, nz - 1)] = 2;
    planes[nplanes++] = (double)(nz - 1);
  }
  /* geometry.cpp:553-565 porosity */
  int64_t fluid_total = 0;
  for (int z = 0; z < nz; ++z) {
    int64_t fl = 0;
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x)
        if (flags[IDX(x, y, z)] == 0) ++fl;
    porosity[z] = (double)fl / ((double)nx * ny);
    fluid_total += fl;
  }
  *fluid_out = fluid_total;
  *n_links_out = 0;
  *q_fallback_out = 0;
  if (fluid_total == 0) {
    free(sph);
    return 3;
  }
  /* geometry.cpp:567-631 links */
  int64_t nl = 0;
  int qfb = 0;
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const int64_t cell = IDX(x, y, z);
        if (flags[cell] != 0) continue;
        for (int k = 1; k < Q; ++k) {
          const int xn = wrap_coord(x + ORC_E[k][0], nx, periodic[0]);
          const int yn = wrap_coord(y + ORC_E[k][1], ny, periodic[1]);
          const int zn = wrap_coord(z + ORC_E[k][2], nz, periodic[2]);
          if (xn < 0 || yn < 0 || zn < 0) {
            free(sph);
            return 1;
          }
          if (flags[IDX(xn, yn, zn)] == 0) continue;
          if (nl >= cap) {
            free(sph);
            return 6;
          }
          const int kb = ORC_OPP[k];
          int64_t second = -1;
          const int xp = wrap_coord(x + ORC_E[kb][0], nx, periodic[0]);
          const int yp = wrap_coord(y + ORC_E[kb][1], ny, periodic[1]);
          const int zp = wrap_coord(z + ORC_E[kb][2], nz, periodic[2]);
          if (xp >= 0 && yp >= 0 && zp >= 0) {
            const int64_t pc = IDX(xp, yp, zp);
            if (flags[pc] == 0) second = pc;
          }
          const double pc3[3] = {x + 0.5, y + 0.5, z + 0.5};
          double q = INFINITY, t;
          for (int64_t i = 0; i < ns; ++i) {
            const osphere* s = &sph[i];
            if (pc3[0] < s->c[0] - s->r - 2.0 || pc3[0] > s->c[0] + s->r + 2.0 ||
                pc3[1] < s->c[1] - s->r - 2.0 || pc3[1] > s->c[1] + s->r + 2.0 ||
                pc3[2] < s->c[2] - s->r - 2.0 || pc3[2] > s->c[2] + s->r + 2.0)
              continue;
            if (ray_sphere(pc3, ORC_E[k], s, &t) && t < q) q = t;
          }
          if (plate_z > 0.0 && ray_plane_z(pc3, ORC_E[k], plate_z, &t) && t < q) q = t;
          for (int i = 0; i < nplanes; ++i)
            if (ray_plane_z(pc3, ORC_E[k], planes[i], &t) && t < q) q = t;
          if (!isfinite(q)) {
            q = 0.5;
            ++qfb;
          }
          /* std::clamp(q, q_clamp_min, 1.0) then cast to float (geometry.cpp:625) */
          const double qc = q < q_clamp_min ? q_clamp_min : (1.0 < q ? 1.0 : q);
          lf[nl] = cell;
          ls[nl] = second;
          ld[nl] = k;
          lq[nl] = (float)qc;
          lm[nl] = 0;
          ++nl;
        }
      }
#undef IDX
  *n_links_out = nl;
  *q_fallback_out = qfb;
  free(sph);
  return 0;
}

/* -------------------------------------------------------------------------
 * Harness sphere generator (the reference ships none that reaches the
 * BASELINE porosities): the same seeded recipe as the product's
 * synthetic generator (random sequential addition without overlap, mode 0,
 * or Boolean model, mode 1), restated here so that the reference arm of
 * bench.py builds its workload without the product.  Randomness follows the
 * reference convention: std::mt19937_64 + uniform01 = (rng() >> 11) * 2^-53
 * (geometry.cpp:19-21), four draws per attempt in the order x, y, z, r.
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_mt64;

static void mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(orc_mt64* s) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double mt64_u01(orc_mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* Returns 0 ok, 1 bad arguments, 6 capacity exceeded. */
int orc_generate_spheres(int mode, uint64_t seed, const double box[3], double z_lo, double z_hi,
                         double r_min, double r_max, double bed_volume, double target_porosity,
                         int64_t max_attempts, int64_t capacity, double* cx, double* cy,
                         double* cz, double* r, int64_t* n_out, double* porosity_out) {
  if (!(r_min > 0.0 && r_max >= r_min) || !(bed_volume > 0.0) || (mode != 0 && mode != 1))
    return 1;
  orc_mt64* rng = (orc_mt64*)malloc(sizeof(orc_mt64));
  mt64_seed(rng, seed);
  const double lx = box[0], ly = box[1], h = 2.0 * r_max;
  int gx = (int)floor(lx / h); if (gx < 1) gx = 1;
  int gy = (int)floor(ly / h); if (gy < 1) gy = 1;
  int gz = (int)ceil((z_hi - z_lo) / h) + 1; if (gz < 1) gz = 1;
  const double hx = lx / gx, hy = ly / gy;
  /* RSA neighbour grid: per-bin singly linked lists (head[bin], next[sphere]) */
  int32_t* head = NULL;
  int32_t* next = NULL;
  if (mode == 0) {
    head = (int32_t*)malloc(sizeof(int32_t) * (size_t)gx * gy * gz);
    for (int64_t i = 0; i < (int64_t)gx * gy * gz; ++i) head[i] = -1;
    next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(capacity > 0 ? capacity : 1));
  }
  int64_t n = 0;
  double vol = 0.0, poro = 1.0;
  int st = 0;
  const double kPi = 3.14159265358979323846;
  for (int64_t a = 0; a < max_attempts; ++a) {
    const double x = mt64_u01(rng) * lx;
    const double y = mt64_u01(rng) * ly;
    const double z = z_lo + mt64_u01(rng) * (z_hi - z_lo);
    const double rr = r_min + mt64_u01(rng) * (r_max - r_min);
    int bin = 0;
    if (mode == 0) {
      int ix = (int)floor(x / hx), iy = (int)floor(y / hy), iz = (int)floor((z - z_lo) / h);
      ix = ix < 0 ? 0 : (ix > gx - 1 ? gx - 1 : ix);
      iy = iy < 0 ? 0 : (iy > gy - 1 ? gy - 1 : iy);
      iz = iz < 0 ? 0 : (iz > gz - 1 ? gz - 1 : iz);
      int ok = 1;
      for (int dz = -1; dz <= 1 && ok; ++dz) {
        const int zz = iz + dz;
        if (zz < 0 || zz >= gz) continue;
        for (int dy = -1; dy <= 1 && ok; ++dy) {
          const int yy = ((iy + dy) % gy + gy) % gy;
          for (int dx = -1; dx <= 1 && ok; ++dx) {
            const int xx = ((ix + dx) % gx + gx) % gx;
            for (int32_t j = head[((int64_t)zz * gy + yy) * gx + xx]; j >= 0; j = next[j]) {
              double ddx = fabs(x - cx[j]), ddy = fabs(y - cy[j]);
              ddx = ddx < lx - ddx ? ddx : lx - ddx; /* minimum image */
              ddy = ddy < ly - ddy ? ddy : ly - ddy;
              const double ddz = z - cz[j], rs = rr + r[j];
              if (ddx * ddx + ddy * ddy + ddz * ddz < rs * rs) {
                ok = 0;
                break;
              }
            }
          }
        }
      }
      if (!ok) continue;
      bin = (iz * gy + iy) * gx + ix;
    }
    if (n >= capacity) {
      st = 6;
      break;
    }
    if (mode == 0) {
      next[n] = head[bin];
      head[bin] = (int32_t)n;
    }
    cx[n] = x;
    cy[n] = y;
    cz[n] = z;
    r[n] = rr;
    ++n;
    vol += 4.0 / 3.0 * kPi * rr * rr * rr;
    poro = (mode == 0) ? 1.0 - vol / bed_volume : exp(-vol / bed_volume);
    if (poro <= target_porosity) break;
  }
  free(head);
  free(next);
  free(rng);
  *n_out = n;
  *porosity_out = poro;
  return st;
}

/* -------------------------------------------------------------------------
 * orc_voxelize_fast: the same voxelizer (geometry.cpp:442-632), with the
 * link q search restricted to the sphere images binned in a uniform grid by
 * their +-(r+2) reject boxes, and planes processed on all OpenMP threads.
 * min() over the candidates is order-independent and the reject test is the
 * reference's own comparison, so the output equals orc_voxelize (and the
 * reference's) byte for byte (tests/test_oracle.py).  Needed for
 * the C4 workload (the brute-force scan takes about an hour there).
 * ------------------------------------------------------------------------- */
int orc_voxelize_fast(int64_t n_sph, const double* cx, const double* cy, const double* cz,
                      const double* cr, const double box[3], double plate_z, const int dims[3],
                      const int periodic[3], int wall_lo, int wall_hi, double q_clamp_min,
                      uint8_t* flags, double* porosity, int64_t cap, int64_t* lf, int64_t* ls,
                      int32_t* ld, float* lq, uint8_t* lm, int64_t* n_links_out,
                      int64_t* fluid_out, int* q_fallback_out) {
  orc_init();
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (nx <= 0 || ny <= 0 || nz <= 0) return 1;
  const int64_t cells = (int64_t)nx * ny * nz;
#define IDX(x, y, z) ((((int64_t)(z)) * ny + (y)) * nx + (x))
  const int ixm = periodic[0] ? 1 : 0, iym = periodic[1] ? 1 : 0;
  osphere* sph = (osphere*)malloc(sizeof(osphere) * (size_t)(n_sph * 9 + 1));
  int64_t ns = 0;
  for (int64_t i = 0; i < n_sph; ++i)
    for (int ix = -ixm; ix <= ixm; ++ix)
      for (int iy = -iym; iy <= iym; ++iy) {
        osphere s;
        s.c[0] = cx[i] + ix * box[0];
        s.c[1] = cy[i] + iy * box[1];
        s.c[2] = cz[i];
        s.r = cr[i];
        if (s.c[0] + s.r < 0.0 || s.c[0] - s.r > nx || s.c[1] + s.r < 0.0 || s.c[1] - s.r > ny)
          continue;
        sph[ns++] = s;
      }
  /* per-plane lists of the images whose rasterization box covers the plane */
  int64_t* zcount = (int64_t*)calloc((size_t)nz + 1, sizeof(int64_t));
  for (int64_t i = 0; i < ns; ++i) {
    int z0 = (int)floor(sph[i].c[2] - sph[i].r - 0.5); if (z0 < 0) z0 = 0;
    int z1 = (int)ceil(sph[i].c[2] + sph[i].r); if (z1 > nz - 1) z1 = nz - 1;
    for (int z = z0; z <= z1; ++z) ++zcount[z + 1];
  }
  for (int z = 0; z < nz; ++z) zcount[z + 1] += zcount[z];
  int64_t* zfill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nz + 1));
  memcpy(zfill, zcount, sizeof(int64_t) * (size_t)(nz + 1));
  int64_t* zlist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(zcount[nz] + 1));
  for (int64_t i = 0; i < ns; ++i) {
    int z0 = (int)floor(sph[i].c[2] - sph[i].r - 0.5); if (z0 < 0) z0 = 0;
    int z1 = (int)ceil(sph[i].c[2] + sph[i].r); if (z1 > nz - 1) z1 = nz - 1;
    for (int z = z0; z <= z1; ++z) zlist[zfill[z]++] = i;
  }
  const int kplate = plate_z > 0.0 ? (int)floor(plate_z - 0.5) : -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int z = 0; z < nz; ++z) {
    uint8_t* fz = flags + (int64_t)z * nx * ny;
    memset(fz, 0, (size_t)nx * ny);
    if (z <= kplate) memset(fz, 1, (size_t)nx * ny); /* geometry.cpp:501-510 */
    for (int64_t t = zcount[z]; t < zcount[z + 1]; ++t) { /* geometry.cpp:512-533 */
      const osphere* s = &sph[zlist[t]];
      int x0 = (int)floor(s->c[0] - s->r - 0.5); if (x0 < 0) x0 = 0;
      int x1 = (int)ceil(s->c[0] + s->r); if (x1 > nx - 1) x1 = nx - 1;
      int y0 = (int)floor(s->c[1] - s->r - 0.5); if (y0 < 0) y0 = 0;
      int y1 = (int)ceil(s->c[1] + s->r); if (y1 > ny - 1) y1 = ny - 1;
      const double r2 = s->r * s->r, dz = z + 0.5 - s->c[2];
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const double dx = x + 0.5 - s->c[0], dy = y + 0.5 - s->c[1];
          if (dx * dx + dy * dy + dz * dz < r2) fz[(int64_t)y * nx + x] = 1;
        }
    }
    if ((wall_lo && z == 0) || (wall_hi && z == nz - 1)) memset(fz, 2, (size_t)nx * ny);
  }
  free(zlist);
  free(zfill);
  free(zcount);
  double planes[2];
  int nplanes = 0;
  if (wall_lo) planes[nplanes++] = 1.0;
  if (wall_hi) planes[nplanes++] = (double)(nz - 1);
  int64_t fluid_total = 0;
  int64_t* plinks = (int64_t*)calloc((size_t)nz + 1, sizeof(int64_t));
  int open_face = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fluid_total) reduction(| : open_face)
  for (int z = 0; z < nz; ++z) { /* porosity (geometry.cpp:553-565) + link counts */
    int64_t fl = 0, nl = 0;
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        if (flags[IDX(x, y, z)] != 0) continue;
        ++fl;
        for (int k = 1; k < Q; ++k) {
          const int xn = wrap_coord(x + ORC_E[k][0], nx, periodic[0]);
          const int yn = wrap_coord(y + ORC_E[k][1], ny, periodic[1]);
          const int zn = wrap_coord(z + ORC_E[k][2], nz, periodic[2]);
          if (xn < 0 || yn < 0 || zn < 0) {
            open_face = 1;
            continue;
          }
          if (flags[IDX(xn, yn, zn)] != 0) ++nl;
        }
      }
    porosity[z] = (double)fl / ((double)nx * ny);
    fluid_total += fl;
    plinks[z + 1] = nl;
  }
  *fluid_out = fluid_total;
  *n_links_out = 0;
  *q_fallback_out = 0;
  if (fluid_total == 0 || open_face) {
    free(plinks);
    free(sph);
    return fluid_total == 0 ? 3 : 1;
  }
  for (int z = 0; z < nz; ++z) plinks[z + 1] += plinks[z];
  if (plinks[nz] > cap) { /* capacity: *n_links_out = the count needed */
    *n_links_out = plinks[nz];
    free(plinks);
    free(sph);
    return 6;
  }
  /* uniform grid of the images' reject boxes [c - r - 2, c + r + 2] */
  const int B = 8;
  const int gx = (nx + B - 1) / B, gy = (ny + B - 1) / B, gz = (nz + B - 1) / B;
  const int64_t nb = (int64_t)gx * gy * gz;
  int64_t* bcount = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* bfill = NULL;
    int64_t* blist = NULL;
    if (pass == 1) {
      for (int64_t b = 0; b < nb; ++b) bcount[b + 1] += bcount[b];
      bfill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb + 1));
      memcpy(bfill, bcount, sizeof(int64_t) * (size_t)(nb + 1));
      blist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(bcount[nb] + 1));
    }
    for (int64_t i = 0; i < ns; ++i) {
      const osphere* s = &sph[i];
      int lo[3], hi[3];
      const int n3[3] = {gx, gy, gz};
      int empty = 0;
      for (int a = 0; a < 3; ++a) {
        /* cell centres p with c - r - 2 <= p <= c + r + 2 (+1 cell of slack) */
        lo[a] = (int)floor((s->c[a] - s->r - 3.0) / B);
        hi[a] = (int)floor((s->c[a] + s->r + 3.0) / B);
        if (lo[a] < 0) lo[a] = 0;
        if (hi[a] > n3[a] - 1) hi[a] = n3[a] - 1;
        if (lo[a] > hi[a]) empty = 1;
      }
      if (empty) continue;
      for (int bz = lo[2]; bz <= hi[2]; ++bz)
        for (int by = lo[1]; by <= hi[1]; ++by)
          for (int bx = lo[0]; bx <= hi[0]; ++bx) {
            const int64_t b = ((int64_t)bz * gy + by) * gx + bx;
            if (pass == 0) ++bcount[b + 1];
            else blist[bfill[b]++] = i;
          }
    }
    if (pass == 1) {
      free(bfill);
      int qfb = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : qfb)
      for (int z = 0; z < nz; ++z) { /* links, geometry.cpp:567-631, (cell, k) order */
        int64_t nl = plinks[z];
        for (int y = 0; y < ny; ++y)
          for (int x = 0; x < nx; ++x) {
            const int64_t cell = IDX(x, y, z);
            if (flags[cell] != 0) continue;
            const int64_t b = ((int64_t)(z / B) * gy + y / B) * gx + x / B;
            for (int k = 1; k < Q; ++k) {
              const int xn = wrap_coord(x + ORC_E[k][0], nx, periodic[0]);
              const int yn = wrap_coord(y + ORC_E[k][1], ny, periodic[1]);
              const int zn = wrap_coord(z + ORC_E[k][2], nz, periodic[2]);
              if (flags[IDX(xn, yn, zn)] == 0) continue;
              const int kb = ORC_OPP[k];
              int64_t second = -1;
              const int xp = wrap_coord(x + ORC_E[kb][0], nx, periodic[0]);
              const int yp = wrap_coord(y + ORC_E[kb][1], ny, periodic[1]);
              const int zp = wrap_coord(z + ORC_E[kb][2], nz, periodic[2]);
              if (xp >= 0 && yp >= 0 && zp >= 0) {
                const int64_t pc = IDX(xp, yp, zp);
                if (flags[pc] == 0) second = pc;
              }
              const double pc3[3] = {x + 0.5, y + 0.5, z + 0.5};
              double q = INFINITY, t;
              for (int64_t u = bcount[b]; u < bcount[b + 1]; ++u) {
                const osphere* s = &sph[blist[u]];
                if (pc3[0] < s->c[0] - s->r - 2.0 || pc3[0] > s->c[0] + s->r + 2.0 ||
                    pc3[1] < s->c[1] - s->r - 2.0 || pc3[1] > s->c[1] + s->r + 2.0 ||
                    pc3[2] < s->c[2] - s->r - 2.0 || pc3[2] > s->c[2] + s->r + 2.0)
                  continue;
                if (ray_sphere(pc3, ORC_E[k], s, &t) && t < q) q = t;
              }
              if (plate_z > 0.0 && ray_plane_z(pc3, ORC_E[k], plate_z, &t) && t < q) q = t;
              for (int i = 0; i < nplanes; ++i)
                if (ray_plane_z(pc3, ORC_E[k], planes[i], &t) && t < q) q = t;
              if (!isfinite(q)) {
                q = 0.5;
                ++qfb;
              }
              const double qc = q < q_clamp_min ? q_clamp_min : (1.0 < q ? 1.0 : q);
              lf[nl] = cell;
              ls[nl] = second;
              ld[nl] = k;
              lq[nl] = (float)qc;
              lm[nl] = 0;
              ++nl;
            }
          }
      }
      *q_fallback_out = qfb;
      free(blist);
    }
  }
#undef IDX
  *n_links_out = plinks[nz];
  free(bcount);
  free(plinks);
  free(sph);
  return 0;
}
