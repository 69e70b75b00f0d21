// sm_100a kernels for the D3Q19 TRT time step (reference: proj/src/simulation.cpp).
//
// Storage: fp64 structure-of-arrays, two grids (A/B), direction plane k at
// element offset k*ks, cell c = (z*ny + y)*nx + x (reference field.hpp:19-21).
// The device keeps the POST-collision state g = C(f) and applies the
// reference's push streaming + link bounce-back in PULL form inside the next
// sweep:
//   K1  k_sweep<OP_STREAM_COLLIDE> : g' = C(P(g))   the hot kernel
//   K0  k_collide_inplace          : g  = C(f)      first step from a pre-collision state
//   KP  k_sweep<OP_STREAM_ONLY>    : f  = P(g)      materialise f(n) for observables
// Every floating-point operation uses the explicit round-to-nearest
// intrinsics (__dadd_rn, __dmul_rn, ...) in the reference's expression order,
// so no FMA is ever contracted and the result is bit-identical to the
// reference CPU solver (x86-64 baseline, which has no FMA).
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"
#include "kparams.h"

namespace pgpu {

#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DSQRT(a) __dsqrt_rn(a)

// D3Q19 in the reference order (lattice.cpp:13-33).
__device__ constexpr int EX[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
__device__ constexpr int EY[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
__device__ constexpr int EZ[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
__host__ __device__ constexpr int opp(int k) { return k == 0 ? 0 : ((k & 1) ? k + 1 : k - 1); }
// Halo slot of a direction with e_x = +1 (1,7,9,11,13) or e_x = -1 (2,8,10,12,14).
__host__ __device__ constexpr int halo_slot(int k) {
  return (k <= 2) ? 0 : (k - 7) / 2 + 1;
}
// Pair weights (k = 2p+1): p = 0..2 axis (1/18), p = 3..8 diagonal (1/36).
__device__ __forceinline__ constexpr double pair_w(int p) { return p < 3 ? 1.0 / 18.0 : 1.0 / 36.0; }

enum SweepOp { OP_STREAM_COLLIDE = 0, OP_STREAM_ONLY = 1 };
enum SweepPart { PART_ALL = 0, PART_EDGES = 1, PART_INTERIOR = 2 };

// ---------------------------------------------------------------------------
// Collision: simulation.cpp:150-196 (core) and :198-274 (GLBM), literal order.
// ---------------------------------------------------------------------------
template <bool RHO1>
__device__ __forceinline__ void collide_core(double (&fk)[19], const KParams& p) {
  const double wp = p.wp, wm = p.wm, rho0 = p.rho0;
  double drho = fk[0];
  double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const double a = fk[1 + 2 * q], b = fk[2 + 2 * q];
    drho = DADD(drho, DADD(a, b));
    const double d = DSUB(a, b);
    vx = DADD(vx, DMUL((double)EX[1 + 2 * q], d));
    vy = DADD(vy, DMUL((double)EY[1 + 2 * q], d));
    vz = DADD(vz, DMUL((double)EZ[1 + 2 * q], d));
  }
  const double ux = RHO1 ? vx : DDIV(vx, rho0);
  const double uy = RHO1 ? vy : DDIV(vy, rho0);
  const double uz = RHO1 ? vz : DDIV(vz, rho0);
  const double uu = DADD(DADD(DMUL(ux, ux), DMUL(uy, uy)), DMUL(uz, uz));
  const double uu15 = DMUL(1.5, uu);
  const double feq0 = DMUL(1.0 / 3.0, DSUB(drho, RHO1 ? uu15 : DMUL(DMUL(rho0, 1.5), uu)));
  fk[0] = DSUB(fk[0], DMUL(wp, DSUB(fk[0], feq0)));
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int k = 1 + 2 * q, kb = k + 1;
    const double eu = DADD(DADD(DMUL((double)EX[k], ux), DMUL((double)EY[k], uy)),
                           DMUL((double)EZ[k], uz));
    double t = DSUB(DMUL(DMUL(4.5, eu), eu), uu15);
    if (!RHO1) t = DMUL(rho0, t);
    const double feq_p = DMUL(pair_w(q), DADD(drho, t));
    const double feq_m = DMUL(p.wr3[q], eu);
    const double fp = DMUL(0.5, DADD(fk[k], fk[kb]));
    const double fm = DMUL(0.5, DSUB(fk[k], fk[kb]));
    const double relax_p = DMUL(wp, DSUB(fp, feq_p));
    const double relax_m = DMUL(wm, DSUB(fm, feq_m));
    const double fpop = p.fpop[q];
    fk[k] = DADD(fk[k], DADD(DSUB(-relax_p, relax_m), fpop));
    fk[kb] = DADD(fk[kb], DSUB(DADD(-relax_p, relax_m), fpop));
  }
}

template <bool RHO1>
__device__ __forceinline__ void collide_glbm(double (&fk)[19], const KParams& p, int z) {
  const PlaneCoef& pc = p.planes[z];
  const double rho0 = p.rho0;
  const double wp = pc.wp, wm = pc.wm, eq_eps = pc.eq_eps;
  double drho = fk[0];
  double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const double a = fk[1 + 2 * q], b = fk[2 + 2 * q];
    drho = DADD(drho, DADD(a, b));
    const double d = DSUB(a, b);
    vx = DADD(vx, DMUL((double)EX[1 + 2 * q], d));
    vy = DADD(vy, DMUL((double)EY[1 + 2 * q], d));
    vz = DADD(vz, DMUL((double)EZ[1 + 2 * q], d));
  }
  const double vhx = DADD(RHO1 ? vx : DDIV(vx, rho0), pc.half_eps_g[0]);
  const double vhy = DADD(RHO1 ? vy : DDIV(vy, rho0), pc.half_eps_g[1]);
  const double vhz = DADD(RHO1 ? vz : DDIV(vz, rho0), pc.half_eps_g[2]);
  double denom;
  if (p.cf == 0.0) {
    denom = pc.denom_lin;
  } else {
    const double vmag = DSQRT(DADD(DADD(DMUL(vhx, vhx), DMUL(vhy, vhy)), DMUL(vhz, vhz)));
    denom = DADD(pc.c0, DSQRT(DADD(DMUL(pc.c0, pc.c0), DMUL(pc.c1, vmag))));
  }
  const double ux = DDIV(vhx, denom), uy = DDIV(vhy, denom), uz = DDIV(vhz, denom);
  double drag;
  if (p.cf != 0.0) {
    const double umag = DSQRT(DADD(DADD(DMUL(ux, ux), DMUL(uy, uy)), DMUL(uz, uz)));
    drag = DADD(pc.drag_lin, DMUL(pc.drag_q, umag));
  } else {
    drag = pc.drag_lin0;
  }
  const double Fx = DADD(DMUL(-drag, ux), pc.eps_g[0]);
  const double Fy = DADD(DMUL(-drag, uy), pc.eps_g[1]);
  const double Fz = DADD(DMUL(-drag, uz), pc.eps_g[2]);
  const double uu = DADD(DADD(DMUL(ux, ux), DMUL(uy, uy)), DMUL(uz, uz));
  const double uu15 = DMUL(1.5, uu);
  const double feq0 = DMUL(
      1.0 / 3.0, DSUB(drho, DDIV(RHO1 ? uu15 : DMUL(DMUL(rho0, 1.5), uu), eq_eps)));
  fk[0] = DSUB(fk[0], DMUL(wp, DSUB(fk[0], feq0)));
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int k = 1 + 2 * q, kb = k + 1;
    const double eu = DADD(DADD(DMUL((double)EX[k], ux), DMUL((double)EY[k], uy)),
                           DMUL((double)EZ[k], uz));
    const double eF = DADD(DADD(DMUL((double)EX[k], Fx), DMUL((double)EY[k], Fy)),
                           DMUL((double)EZ[k], Fz));
    double t = DSUB(DMUL(DMUL(4.5, eu), eu), uu15);
    if (!RHO1) t = DMUL(rho0, t);
    const double feq_p = DMUL(pair_w(q), DADD(drho, DDIV(t, eq_eps)));
    const double feq_m = DMUL(p.wr3[q], eu);
    const double fp = DMUL(0.5, DADD(fk[k], fk[kb]));
    const double fm = DMUL(0.5, DSUB(fk[k], fk[kb]));
    const double relax_p = DMUL(wp, DSUB(fp, feq_p));
    const double relax_m = DMUL(wm, DSUB(fm, feq_m));
    const double fpop = DMUL(DMUL(pc.force_pref, pair_w(q)), eF);
    fk[k] = DADD(fk[k], DADD(DSUB(-relax_p, relax_m), fpop));
    fk[kb] = DADD(fk[kb], DSUB(DADD(-relax_p, relax_m), fpop));
  }
}

// ---------------------------------------------------------------------------
// Pull-form streaming + bounce-back: for fluid x and direction
// j with fluid upstream s = x - e_j:  f_j(x) = g_j(s).  Otherwise the link
// (x, k = opp j) closes it (boundary.cpp:19-41 written for the receiving slot):
//   SBB    f_j(x) = g_k(x)
//   CLI    f_j(x) = c*g_k(x - e_k) - c*g_j(x) + g_k(x),  c = (1-2q)/(1+2q)
//   moving f_j(x) = g_k(x) - 2 w_k rho0 3 (e_k . u_w)
// and g_k(x - e_k) is exactly the pull value of direction k at x.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

template <int J, bool SLAB>
__device__ __forceinline__ double pull(const double* __restrict__ src, int x, int y, int z,
                                       const KParams& p) {
  constexpr int ex = EX[J], ey = EY[J], ez = EZ[J];
  int ys = y - ey, zs = z - ez;
  if (ey == 1 && y == 0) ys = p.ny - 1;
  if (ey == -1 && y == p.ny - 1) ys = 0;
  if (ez == 1 && z == 0) zs = p.nz - 1;
  if (ez == -1 && z == p.nz - 1) zs = 0;
  int xs = x - ex;
  const double* plane = src + (int64_t)J * p.ks;
  if (ex == 1) {
    if (x == 0) {
      if (SLAB) return ldg(p.ghost_lo + (int64_t)halo_slot(J) * p.ny * p.nz + zs * p.ny + ys);
      xs = p.nx - 1;
    }
  } else if (ex == -1) {
    if (x == p.nx - 1) {
      if (SLAB) return ldg(p.ghost_hi + (int64_t)halo_slot(J) * p.ny * p.nz + zs * p.ny + ys);
      xs = 0;
    }
  }
  return ldg(plane + ((int64_t)zs * p.ny + ys) * p.nx + xs);
}

template <int J, bool SLAB>
__device__ __forceinline__ void pull_all(double (&f)[19], const double* __restrict__ src, int x,
                                         int y, int z, const KParams& p, uint32_t w) {
  if constexpr (J < 19) {
    if (J == 0 || !((w >> J) & 1u)) f[J] = pull<J, SLAB>(src, x, y, z, p);
    pull_all<J + 1, SLAB>(f, src, x, y, z, p, w);
  }
}

template <int J, bool SLAB>
__device__ __forceinline__ void pull_all_fast(double (&f)[19], const double* __restrict__ src,
                                              int x, int y, int z, const KParams& p) {
  if constexpr (J < 19) {
    f[J] = pull<J, SLAB>(src, x, y, z, p);
    pull_all_fast<J + 1, SLAB>(f, src, x, y, z, p);
  }
}

template <int J, bool RECORDS>
__device__ __forceinline__ void bounce_all(double (&f)[19], const double* __restrict__ src,
                                           int64_t c, const KParams& p, uint32_t w, int32_t base) {
  if constexpr (J < 19) {
    if ((w >> J) & 1u) {
      constexpr int K = opp(J);
      const double gk = ldg(src + (int64_t)K * p.ks + c);  // g_k(x)
      double v = gk;                                        // SBB, boundary.cpp:19-22
      if (RECORDS) {
        const int32_t r = base + __popc(w & ((1u << J) - 1u) & ~1u);
        const LinkRec rec = p.links[r];
        if (rec.kind == kLinkCLI) {  // boundary.cpp:24-32
          const double q = (double)rec.q;
          const double cc = DDIV(DSUB(1.0, DMUL(2.0, q)), DADD(1.0, DMUL(2.0, q)));
          const double gj = ldg(src + (int64_t)J * p.ks + c);  // g_kb(x_f1)
          v = DADD(DSUB(DMUL(cc, f[K]), DMUL(cc, gj)), gk);
        } else if (rec.kind == kLinkMoving) {  // boundary.cpp:34-41
          v = DSUB(gk, p.mw[K]);
        }
      }
      f[J] = v;
    }
    bounce_all<J + 1, RECORDS>(f, src, c, p, w, base);
  }
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__device__ __forceinline__ void sweep_cell(const KParams& p, const double* __restrict__ src,
                                           double* __restrict__ dst, int x, int y, int z) {
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = __ldg(p.cellword + c);
  if (w & 1u) return;  // solid / wall: never read, never written
  double f[19];
  if (w == 0u) {
    pull_all_fast<0, SLAB>(f, src, x, y, z, p);
  } else {
    pull_all<0, SLAB>(f, src, x, y, z, p, w);
    const int32_t base = RECORDS ? __ldg(p.link_base + c) : 0;
    bounce_all<1, RECORDS>(f, src, c, p, w, base);
  }
  if (OP == OP_STREAM_COLLIDE) {
    if (GLBM)
      collide_glbm<RHO1>(f, p, z);
    else
      collide_core<RHO1>(f, p);
  }
#pragma unroll
  for (int j = 0; j < 19; ++j) __stcs(dst + (int64_t)j * p.ks + c, f[j]);
  if (SLAB && OP == OP_STREAM_COLLIDE) {
    const int64_t hp = (int64_t)p.ny * p.nz;
    const int64_t h = (int64_t)z * p.ny + y;
    if (x == 0) {
      p.send_lo[0 * hp + h] = f[2];
      p.send_lo[1 * hp + h] = f[8];
      p.send_lo[2 * hp + h] = f[10];
      p.send_lo[3 * hp + h] = f[12];
      p.send_lo[4 * hp + h] = f[14];
    }
    if (x == p.nx - 1) {
      p.send_hi[0 * hp + h] = f[1];
      p.send_hi[1 * hp + h] = f[7];
      p.send_hi[2 * hp + h] = f[9];
      p.send_hi[3 * hp + h] = f[11];
      p.send_hi[4 * hp + h] = f[13];
    }
  }
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_sweep(const KParams p, const double* __restrict__ src,
                                               double* __restrict__ dst, int part) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  if (part == PART_INTERIOR && (x == 0 || x == p.nx - 1)) return;
  sweep_cell<RHO1, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z);
}

// Edge columns x = 0 and x = nx-1 only (slab overlap path).
template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_sweep_edges(const KParams p,
                                                     const double* __restrict__ src,
                                                     double* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t hp = (int64_t)p.ny * p.nz;
  if (t >= 2 * hp) return;
  const int side = (int)(t / hp);
  const int64_t h = t - side * hp;
  const int z = (int)(h / p.ny), y = (int)(h - (int64_t)z * p.ny);
  const int x = side ? p.nx - 1 : 0;
  if (side == 1 && p.nx == 1) return;
  sweep_cell<RHO1, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z);
}

// K0: collide every fluid cell in place (first step from a pre-collision state).
template <bool RHO1, bool GLBM, bool SLAB>
__global__ void __launch_bounds__(128) k_collide_inplace(const KParams p, double* buf) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  if (__ldg(p.cellword + c) & 1u) return;
  double f[19];
#pragma unroll
  for (int j = 0; j < 19; ++j) f[j] = buf[(int64_t)j * p.ks + c];
  if (GLBM)
    collide_glbm<RHO1>(f, p, z);
  else
    collide_core<RHO1>(f, p);
#pragma unroll
  for (int j = 0; j < 19; ++j) buf[(int64_t)j * p.ks + c] = f[j];
  if (SLAB) {
    const int64_t hp = (int64_t)p.ny * p.nz;
    const int64_t h = (int64_t)z * p.ny + y;
    if (x == 0) {
      p.send_lo[0 * hp + h] = f[2];
      p.send_lo[1 * hp + h] = f[8];
      p.send_lo[2 * hp + h] = f[10];
      p.send_lo[3 * hp + h] = f[12];
      p.send_lo[4 * hp + h] = f[14];
    }
    if (x == p.nx - 1) {
      p.send_hi[0 * hp + h] = f[1];
      p.send_hi[1 * hp + h] = f[7];
      p.send_hi[2 * hp + h] = f[9];
      p.send_hi[3 * hp + h] = f[11];
      p.send_hi[4 * hp + h] = f[13];
    }
  }
}

// ---------------------------------------------------------------------------
// Observables from a pre-collision state f (simulation.cpp:354-434).
// ---------------------------------------------------------------------------
// moments(): lattice.cpp:88-101, literal order over k = 0..18.
template <bool GLBM>
__device__ __forceinline__ bool macro_cell(const KParams& p, const double* __restrict__ f,
                                           int64_t c, int z, double& drho, double (&u)[3]) {
  double d = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
  for (int k = 0; k < 19; ++k) {
    const double fk = f[(int64_t)k * p.ks + c];
    d = DADD(d, fk);
    v0 = DADD(v0, DMUL((double)EX[k], fk));
    v1 = DADD(v1, DMUL((double)EY[k], fk));
    v2 = DADD(v2, DMUL((double)EZ[k], fk));
  }
  v0 = DDIV(v0, p.rho0);
  v1 = DDIV(v1, p.rho0);
  v2 = DDIV(v2, p.rho0);
  drho = d;
  if (!GLBM) {  // simulation.cpp:367
    u[0] = DADD(v0, p.hg[0]);
    u[1] = DADD(v1, p.hg[1]);
    u[2] = DADD(v2, p.hg[2]);
    return true;
  }
  // glbm_force_and_velocity, simulation.cpp:52-66
  const PlaneCoef& pc = p.planes[z];
  const double vh0 = DADD(v0, pc.half_eps_g[0]);
  const double vh1 = DADD(v1, pc.half_eps_g[1]);
  const double vh2 = DADD(v2, pc.half_eps_g[2]);
  const double nrm = DSQRT(DADD(DADD(DMUL(vh0, vh0), DMUL(vh1, vh1)), DMUL(vh2, vh2)));
  const double disc = DADD(DMUL(pc.c0, pc.c0), DMUL(pc.c1, nrm));
  const double denom = DADD(pc.c0, DSQRT(disc));
  u[0] = DDIV(vh0, denom);
  u[1] = DDIV(vh1, denom);
  u[2] = DDIV(vh2, denom);
  return !(disc < 0.0);
}

template <bool GLBM>
__global__ void k_macro_fields(const KParams p, const double* __restrict__ f, double* drho,
                               double* ux, double* uy, double* uz, int* err) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  if (__ldg(p.cellword + c) & 1u) {
    if (drho) drho[c] = 0.0;
    if (ux) ux[c] = 0.0;
    if (uy) uy[c] = 0.0;
    if (uz) uz[c] = 0.0;
    return;
  }
  double d, u[3];
  if (!macro_cell<GLBM>(p, f, c, z, d, u)) atomicOr(err, 1);
  if (drho) drho[c] = d;
  if (ux) ux[c] = u[0];
  if (uy) uy[c] = u[1];
  if (uz) uz[c] = u[2];
}

// Sequential per-plane sum in ascending cell order (simulation.cpp:400-407),
// one thread per plane so the rounding sequence is the reference's.
__global__ void k_plane_sums(const uint32_t* __restrict__ cellword,
                             const double* __restrict__ u, int64_t plane, int nz,
                             double* sums) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= nz) return;
  double s = 0.0;
  const int64_t c0 = plane * z;
  for (int64_t i = 0; i < plane; ++i) {
    if (__ldg(cellword + c0 + i) & 1u) continue;
    s = DADD(s, __ldg(u + c0 + i));
  }
  sums[z] = s;
}

// max |u|^2 and finiteness over fluid cells (simulation.cpp:419-434).
template <bool GLBM>
__global__ void k_max_speed2(const KParams p, const double* __restrict__ f,
                             unsigned long long* vmax2_bits, int* nonfinite, int* err) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  double m2 = 0.0;
  bool bad = false;
  if (x < p.nx) {
    const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
    if (!(__ldg(p.cellword + c) & 1u)) {
      double d, u[3];
      if (!macro_cell<GLBM>(p, f, c, z, d, u)) atomicOr(err, 1);
      m2 = DADD(DADD(DMUL(u[0], u[0]), DMUL(u[1], u[1])), DMUL(u[2], u[2]));
      bad = !(isfinite(m2) && isfinite(d));
      if (!(m2 > 0.0)) m2 = 0.0;  // std::max(vmax2, m2) ignores NaN and keeps 0
    }
  }
  // warp reduce (m2 >= 0 so the IEEE bit pattern orders like an unsigned int)
  unsigned long long bits = (unsigned long long)__double_as_longlong(m2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = other > bits ? other : bits;
  }
  const unsigned anybad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(vmax2_bits, bits);
    if (anybad) atomicOr(nonfinite, 1);
  }
}

__global__ void k_fill_equilibrium(const uint32_t* __restrict__ cellword, int64_t cells,
                                   int64_t ks, double* f, const double* feq /*19*/) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  if (cellword[c] & 1u) return;
#pragma unroll
  for (int k = 0; k < 19; ++k) f[(int64_t)k * ks + c] = feq[k];
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
namespace {
constexpr int kBX = 128;
dim3 cell_grid(const KParams& p) { return dim3((p.nx + kBX - 1) / kBX, p.ny, p.nz); }
dim3 cell_block(const KParams& p) { return dim3(p.nx < kBX ? ((p.nx + 31) / 32) * 32 : kBX); }
dim3 cell_grid2(const KParams& p) {
  const int bx = cell_block(p).x;
  return dim3((p.nx + bx - 1) / bx, p.ny, p.nz);
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
void launch_sweep_t(const KParams& p, const double* src, double* dst, int part,
                    cudaStream_t s) {
  if (part == PART_EDGES) {
    const int64_t n = 2 * (int64_t)p.ny * p.nz;
    k_sweep_edges<RHO1, GLBM, RECORDS, SLAB, OP>
        <<<(unsigned)((n + kBX - 1) / kBX), kBX, 0, s>>>(p, src, dst);
  } else {
    k_sweep<RHO1, GLBM, RECORDS, SLAB, OP><<<cell_grid2(p), cell_block(p), 0, s>>>(p, src, dst,
                                                                                  part);
  }
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB>
void dispatch_op(int op, const KParams& p, const double* src, double* dst, int part,
                 cudaStream_t s) {
  if (op == OP_STREAM_COLLIDE)
    launch_sweep_t<RHO1, GLBM, RECORDS, SLAB, OP_STREAM_COLLIDE>(p, src, dst, part, s);
  else
    launch_sweep_t<RHO1, GLBM, RECORDS, SLAB, OP_STREAM_ONLY>(p, src, dst, part, s);
}
template <bool RHO1, bool GLBM, bool RECORDS>
void dispatch_slab(bool slab, int op, const KParams& p, const double* src, double* dst,
                   int part, cudaStream_t s) {
  if (slab)
    dispatch_op<RHO1, GLBM, RECORDS, true>(op, p, src, dst, part, s);
  else
    dispatch_op<RHO1, GLBM, RECORDS, false>(op, p, src, dst, part, s);
}
template <bool RHO1, bool GLBM>
void dispatch_rec(bool rec, bool slab, int op, const KParams& p, const double* src,
                  double* dst, int part, cudaStream_t s) {
  if (rec)
    dispatch_slab<RHO1, GLBM, true>(slab, op, p, src, dst, part, s);
  else
    dispatch_slab<RHO1, GLBM, false>(slab, op, p, src, dst, part, s);
}
}  // namespace

void launch_sweep(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  const bool rho1 = p.rho0 == 1.0;
  if (rho1) {
    if (cfg.glbm)
      dispatch_rec<true, true>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
    else
      dispatch_rec<true, false>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
  } else {
    if (cfg.glbm)
      dispatch_rec<false, true>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
    else
      dispatch_rec<false, false>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
  }
}

void launch_collide_inplace(bool glbm, bool slab, const KParams& p, double* buf,
                            cudaStream_t s) {
  const dim3 g = cell_grid2(p), b = cell_block(p);
  const bool rho1 = p.rho0 == 1.0;
#define PGPU_K0(R, G, S) k_collide_inplace<R, G, S><<<g, b, 0, s>>>(p, buf)
  if (rho1) {
    if (glbm) { if (slab) PGPU_K0(true, true, true); else PGPU_K0(true, true, false); }
    else { if (slab) PGPU_K0(true, false, true); else PGPU_K0(true, false, false); }
  } else {
    if (glbm) { if (slab) PGPU_K0(false, true, true); else PGPU_K0(false, true, false); }
    else { if (slab) PGPU_K0(false, false, true); else PGPU_K0(false, false, false); }
  }
#undef PGPU_K0
}

void launch_macro_fields(bool glbm, const KParams& p, const double* f, double* drho,
                         double* ux, double* uy, double* uz, int* err, cudaStream_t s) {
  if (glbm)
    k_macro_fields<true><<<cell_grid2(p), cell_block(p), 0, s>>>(p, f, drho, ux, uy, uz, err);
  else
    k_macro_fields<false><<<cell_grid2(p), cell_block(p), 0, s>>>(p, f, drho, ux, uy, uz, err);
}

void launch_plane_sums(const KParams& p, const double* u, double* sums, cudaStream_t s) {
  const int64_t plane = (int64_t)p.nx * p.ny;
  k_plane_sums<<<(p.nz + 31) / 32, 32, 0, s>>>(p.cellword, u, plane, p.nz, sums);
}

void launch_max_speed2(bool glbm, const KParams& p, const double* f,
                       unsigned long long* vmax2_bits, int* nonfinite, int* err,
                       cudaStream_t s) {
  if (glbm)
    k_max_speed2<true><<<cell_grid2(p), cell_block(p), 0, s>>>(p, f, vmax2_bits, nonfinite, err);
  else
    k_max_speed2<false><<<cell_grid2(p), cell_block(p), 0, s>>>(p, f, vmax2_bits, nonfinite,
                                                                err);
}

void launch_fill_equilibrium(const KParams& p, int64_t cells, double* f, const double* feq,
                             cudaStream_t s) {
  k_fill_equilibrium<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(p.cellword, cells, p.ks, f,
                                                                     feq);
}

}  // namespace pgpu
