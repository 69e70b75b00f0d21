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

// x-slab split: the edge part sweeps one warp-aligned band of columns at each
// x face (x < w or x >= nx - w; it alone reads ghosts and fills the send
// buffers), the interior part the rest.  Bands of 32 keep the edge rows
// coalesced, so the edge part streams like the interior instead of touching
// one 8-byte slot per DRAM line.
__host__ __device__ __forceinline__ int edge_band(int nx) { return nx < 64 ? (nx + 1) / 2 : 32; }
__device__ __forceinline__ bool in_edge_band(int x, int nx) {
  const int w = edge_band(nx);
  return x < w || x >= nx - w;
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

}  // namespace pgpu
