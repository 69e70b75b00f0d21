// Plain structs shared by the host runtime (sim.cpp) and the sm_100a kernels
// (kernels.cu).  No torch types anywhere.
#pragma once
#include <cstdint>

namespace pgpu {

constexpr int kQ = 19;

// Per-link record, stored in (cell, incoming direction j) order so that the
// kernel finds the record of bounce direction j of cell c at
//   link_base[c] + popcount(cellword[c] & ((1u << j) - 1) & ~1u).
enum LinkKind : uint32_t { kLinkSBB = 0, kLinkCLI = 1, kLinkMoving = 2 };
struct LinkRec {
  float q;        // fp32 wall distance exactly as stored by voxelize (geometry.cpp:625)
  uint32_t kind;  // LinkKind
};

// GLBM per-plane coefficients (simulation.cpp:213-253), evaluated on the host
// with the reference's operation order so the kernel reproduces it bit for bit.
struct PlaneCoef {
  double eps, K, wp, wm, eq_eps;
  double half_eps_g[3];  // 0.5 * eps * g[i]            (:233-235)
  double eps_g[3];       // eps * g[i]                  (:248-250)
  double c0;             // 0.5 * (1.0 + eps*nu/(2.0*K)) (:236)
  double denom_lin;      // 2.0 * c0                    (:239)
  double c1;             // 0.5 * eps * cf / sqrt(K)    (:241)
  double drag_lin;       // eps * nu / K                (:247, first term)
  double drag_lin0;      // drag_lin + 0.0              (:247 with cf == 0)
  double drag_q;         // eps * cf / sqrt(K)          (:247, second term)
  double force_pref;     // (1.0 - 0.5*wm) * 3.0 * rho0 (:253)
};

// Everything a sweep kernel needs, passed by value.
struct KParams {
  int32_t nx, ny, nz;
  int32_t px, py, pz;  // periodic flags (x ignored in slab mode)
  int64_t ks;          // element stride between the 19 direction planes
  const uint32_t* cellword;  // bit0: not fluid; bit j (1..18): f_j comes from a link
  const int32_t* link_base;  // per-cell first record (only with records)
  const LinkRec* links;
  double wp, wm, rho0, nu, cf;
  double fpop[9];   // core force term ((3*w)*rho0)*eg per pair (simulation.cpp:190)
  double wr3[9];    // (w*rho0)*3 per pair                      (simulation.cpp:185)
  double mw[19];    // moving-wall term 2*w*rho0*3*(e.u_w) per link direction (boundary.cpp:38-40)
  double hg[3];     // 0.5*g[i]/rho0  (simulation.cpp:367)
  double g[3];
  const PlaneCoef* planes;  // GLBM only
  // x-slab halo (slab mode only)
  const double* ghost_lo;  // [5][ny*nz] g of directions 1,7,9,11,13 at x=-1
  const double* ghost_hi;  // [5][ny*nz] g of directions 2,8,10,12,14 at x=nx
  double* send_lo;         // [5][ny*nz] our g of directions 2,8,10,12,14 at x=0
  double* send_hi;         // [5][ny*nz] our g of directions 1,7,9,11,13 at x=nx-1
};

}  // namespace pgpu
