// Device-side D3Q19 lattice constants and the TRT / GLBM collisions shared by
// the sweep kernels (kernels.cu: dense layout, sweep_compact.cu: fluid-only
// layout).  Reference: proj/src/lattice.cpp:11-56, proj/src/simulation.cpp:150-274.
// Every floating-point operation uses the explicit round-to-nearest
// intrinsics in the reference's expression order (no FMA contraction).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

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

// x-slab split: the edge part sweeps a band of columns at each x face
// (x < w or x >= nx - w; it alone reads ghosts and fills the send buffers),
// the interior part the rest.  Slabs of >= 96 columns use warp-aligned bands
// of 32 (coalesced edge rows); narrower slabs (64 columns = C4 strong scaling
// at 8 GPUs) use the single face columns, so the interior part -- which the
// halo exchange overlaps -- is not empty (the edge part then reads one slot
// per row and 32-byte sector, but for only 2 of the slab's columns).
__host__ __device__ __forceinline__ int edge_band(int nx) { return nx >= 96 ? 32 : 1; }
__device__ __forceinline__ bool in_edge_band(int x, int nx) {
  const int w = edge_band(nx);
  return x < w || x >= nx - w;
}

// Fluid-only layout: slot of fluid cell (x, y, z) from its row chunk entry.
__device__ __forceinline__ int64_t compact_slot(const KParams& p, int x, int y, int z) {
  const ChunkEnt e = p.ctab[((int64_t)z * p.ny + y) * p.nchunk + (x >> 5)];
  return (int64_t)e.rank + __popc(e.mask & ((1u << (x & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// Collision: simulation.cpp:150-196 (core) and :198-274 (GLBM), literal order.
// ---------------------------------------------------------------------------
// Multiply-add of a lattice-constant coefficient e in {-1, 0, 1}: acc + e*v.
// The reference multiplies literally (its pair table is a runtime array);
// with e = 0 the term e*v is a signed zero and acc + (+-0) == acc whenever acc
// is not -0.  In the rho0 == 1 core path every accumulator starts at +0 and a
// round-to-nearest sum is -0 only if both addends are -0, so acc is never -0
// and dropping the zero terms is bit-identical for every finite state (a
// non-finite population makes the cell non-finite either way).  e = +-1 terms
// are exact (x*1 = x, x*-1 = -x, a + -b == a - b).
// (e is a compile-time constant after unrolling; the branches fold away.)
__device__ __forceinline__ double macc(int e, double acc, double v) {
  if (e == 0) return acc;
  if (e == 1) return DADD(acc, v);
  return DSUB(acc, v);
}
// First term of a dot product e.u started from a literal (+0 + e*v).
__device__ __forceinline__ double mfirst(int e, double v) {
  if (e == 0) return 0.0;
  if (e == 1) return DADD(0.0, v);
  return DSUB(0.0, v);
}

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
    if (RHO1) {
      vx = macc(EX[1 + 2 * q], vx, d);
      vy = macc(EY[1 + 2 * q], vy, d);
      vz = macc(EZ[1 + 2 * q], vz, d);
    } else {
      vx = DADD(vx, DMUL((double)EX[1 + 2 * q], d));
      vy = DADD(vy, DMUL((double)EY[1 + 2 * q], d));
      vz = DADD(vz, DMUL((double)EZ[1 + 2 * q], d));
    }
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
    double eu;
    if (RHO1) {
      // ((ex*ux + ey*uy) + ez*uz) with the zero terms dropped (see macc)
      eu = macc(EZ[k], macc(EY[k], mfirst(EX[k], ux), uy), uz);
    } else {
      eu = DADD(DADD(DMUL((double)EX[k], ux), DMUL((double)EY[k], uy)), DMUL((double)EZ[k], uz));
    }
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
  double ux, uy, uz;
  if (p.cf == 0.0 && pc.denom_mode == 0) {  // denom == 1: identity (free planes)
    ux = vhx;
    uy = vhy;
    uz = vhz;
  } else if (p.cf == 0.0 && pc.denom_mode == 1) {  // power of two: exact reciprocal
    ux = DMUL(vhx, pc.inv_denom);
    uy = DMUL(vhy, pc.inv_denom);
    uz = DMUL(vhz, pc.inv_denom);
  } else {
    ux = DDIV(vhx, denom);
    uy = DDIV(vhy, denom);
    uz = DDIV(vhz, denom);
  }
  // x / eq_eps with the same shortcuts (plane-uniform branch)
  auto div_eps = [&](double v) {
    return pc.eq_mode == 0 ? v : (pc.eq_mode == 1 ? DMUL(v, pc.inv_eq_eps) : DDIV(v, eq_eps));
  };
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
  const double feq0 =
      DMUL(1.0 / 3.0, DSUB(drho, div_eps(RHO1 ? uu15 : DMUL(DMUL(rho0, 1.5), uu))));
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
    const double feq_p = DMUL(pair_w(q), DADD(drho, div_eps(t)));
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
// Math mode PGPU_MATH_FAST: the same TRT algebra regrouped and FMA-contracted
// (kparams.h FastCoef).  Half the fp64 instructions of the literal-order
// collision; agrees with it to rounding, not bit for bit.
// ---------------------------------------------------------------------------
// e.u for pair q (direction k = 2q+1) with the compile-time lattice vector.
__device__ __forceinline__ double fast_eu(int q, double ux, double uy, double uz) {
  const int k = 1 + 2 * q;
  double r = 0.0;
  bool first = true;
  auto acc = [&](int e, double v) {
    if (e == 0) return;
    if (first) r = e > 0 ? v : -v;
    else r = e > 0 ? r + v : r - v;
    first = false;
  };
  acc(EX[k], ux);
  acc(EY[k], uy);
  acc(EZ[k], uz);
  return r;
}

// In place: f[k] <- a + b, f[kb] <- a - b for every pair; returns drho and
// the momentum (reference moments, simulation.cpp:166-174, reassociated).
__device__ __forceinline__ void fast_moments(double (&f)[19], double& drho, double& vx, double& vy,
                                             double& vz) {
  double s[9], d[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    s[q] = f[1 + 2 * q] + f[2 + 2 * q];
    d[q] = f[1 + 2 * q] - f[2 + 2 * q];
    f[1 + 2 * q] = s[q];
    f[2 + 2 * q] = d[q];
  }
  // pairwise sums (shorter dependency chains than the reference's serial sum)
  drho = ((f[0] + s[0]) + (s[1] + s[2])) + ((s[3] + s[4]) + (s[5] + s[6])) + (s[7] + s[8]);
  // pairs: 0 (1,0,0) 1 (0,1,0) 2 (0,0,1) 3 (1,1,0) 4 (1,-1,0) 5 (1,0,1) 6 (1,0,-1)
  //        7 (0,1,1) 8 (0,1,-1)
  vx = (d[0] + d[3]) + (d[4] + d[5]) + d[6];
  vy = (d[1] + d[3]) - (d[4] - d[7]) + d[8];
  vz = (d[2] + d[5]) - (d[6] - d[7]) - d[8];
}

// Pair updates from s/d in f: a' = P + M, b' = P - M.
__device__ __forceinline__ void fast_pairs(double (&f)[19], const FastCoef& c, double B0,
                                           double B1, double ux, double uy, double uz,
                                           const double (&fpop)[9]) {
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int cl = q < 3 ? 0 : 1;
    const double eu = fast_eu(q, ux, uy, uz);
    const double P = fma(c.hp, f[1 + 2 * q], fma(c.C[cl], eu * eu, cl ? B1 : B0));
    const double M = fma(c.hm, f[2 + 2 * q], fma(c.D[cl], eu, fpop[q]));
    f[1 + 2 * q] = P + M;
    f[2 + 2 * q] = P - M;
  }
}

__device__ __forceinline__ void collide_core_fast(double (&f)[19], const KParams& p) {
  const FastCoef& c = p.fc;
  double drho, vx, vy, vz;
  fast_moments(f, drho, vx, vy, vz);
  const double ux = vx * c.inv_rho0, uy = vy * c.inv_rho0, uz = vz * c.inv_rho0;
  const double uu = fma(uz, uz, fma(uy, uy, ux * ux));
  f[0] = fma(c.w0, f[0], fma(c.a0, drho, c.b0 * uu));
  const double B0 = fma(c.kw1[0], drho, c.kw2[0] * uu);
  const double B1 = fma(c.kw1[1], drho, c.kw2[1] * uu);
  fast_pairs(f, c, B0, B1, ux, uy, uz, p.fpop);
}

// GLBM (simulation.cpp:198-274) in the same regrouped form; the per-plane
// constants (incl. 1/eq_eps and the plane's omegas) are in pc.fc.
__device__ __forceinline__ void collide_glbm_fast(double (&f)[19], const KParams& p, int z) {
  const PlaneCoef& pc = p.planes[z];
  const FastCoef& c = pc.fc;
  double drho, vx, vy, vz;
  fast_moments(f, drho, vx, vy, vz);
  const double vhx = fma(vx, c.inv_rho0, pc.half_eps_g[0]);
  const double vhy = fma(vy, c.inv_rho0, pc.half_eps_g[1]);
  const double vhz = fma(vz, c.inv_rho0, pc.half_eps_g[2]);
  double inv, drag;
  if (p.cf == 0.0) {
    inv = pc.f_inv_denom;
  } else {
    const double vmag = sqrt(fma(vhz, vhz, fma(vhy, vhy, vhx * vhx)));
    inv = 1.0 / (pc.c0 + sqrt(fma(pc.c1, vmag, pc.c0 * pc.c0)));
  }
  const double ux = vhx * inv, uy = vhy * inv, uz = vhz * inv;
  const double uu = fma(uz, uz, fma(uy, uy, ux * ux));
  if (p.cf != 0.0)
    drag = fma(pc.drag_q, sqrt(uu), pc.drag_lin);
  else
    drag = pc.drag_lin0;
  const double Fx = fma(-drag, ux, pc.eps_g[0]);
  const double Fy = fma(-drag, uy, pc.eps_g[1]);
  const double Fz = fma(-drag, uz, pc.eps_g[2]);
  f[0] = fma(c.w0, f[0], fma(c.a0, drho, c.b0 * uu));
  const double B0 = fma(c.kw1[0], drho, c.kw2[0] * uu);
  const double B1 = fma(c.kw1[1], drho, c.kw2[1] * uu);
  double fpop[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) fpop[q] = c.fw[q < 3 ? 0 : 1] * fast_eu(q, Fx, Fy, Fz);
  fast_pairs(f, c, B0, B1, ux, uy, uz, fpop);
}

// Collision mode (template parameter CM of the sweep kernels):
//   0 literal order, general rho0   1 literal order, rho0 == 1   2 fast (any rho0)
//   3 fast + folded CLI links (fluid-only layout, kparams.h KParams::fold)
enum CollideMode { CM_EXACT = 0, CM_EXACT_RHO1 = 1, CM_FAST = 2, CM_FAST_FOLD = 3 };
__host__ __device__ __forceinline__ int collide_mode(const KParams& p) {
  return p.fast ? (p.fold ? CM_FAST_FOLD : CM_FAST) : (p.rho0 == 1.0 ? CM_EXACT_RHO1 : CM_EXACT);
}
template <int CM, bool GLBM>
__device__ __forceinline__ void collide(double (&f)[19], const KParams& p, int z) {
  if constexpr (CM >= CM_FAST) {
    if constexpr (GLBM) collide_glbm_fast(f, p, z);
    else collide_core_fast(f, p);
  } else {
    if constexpr (GLBM) collide_glbm<CM == CM_EXACT_RHO1>(f, p, z);
    else collide_core<CM == CM_EXACT_RHO1>(f, p);
  }
}

}  // namespace pgpu
