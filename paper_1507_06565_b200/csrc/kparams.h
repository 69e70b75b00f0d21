// Plain structs shared by the host runtime (sim.cpp) and the sm_100a kernels
// (kernels.cu).  No torch types anywhere.
#pragma once
#include <cstdint>

namespace pgpu {

constexpr int kQ = 19;

// Per-link record, one double in (cell, incoming direction j) order so that
// the kernel finds the record of bounce direction j of cell c at
//   cell.base + popcount(cell.w & ((1u << j) - 1) & kBounceMask).
// CLI links store c = (1-2q)/(1+2q) computed on the host exactly like
// boundary.cpp:27-28 (q the fp32 value of geometry.cpp:625); SBB links store
// a quiet NaN, moving-wall links +infinity.
enum LinkKind : uint32_t { kLinkSBB = 0, kLinkCLI = 1, kLinkMoving = 2 };
typedef double LinkRec;

// Per-cell word: bit 0 = not fluid; bits 1..18 = f_j comes from a link;
// bit 19 = non-fluid cell that shares a 32-byte sector with a fluid cell
// (written with zeros so no sector is ever partially written); bits 24..31 =
// the reference flag byte of a non-fluid cell (write_vtk, pgpu_get_flags).
constexpr uint32_t kNonFluid = 1u;
constexpr uint32_t kBounceMask = 0x7FFFEu;
constexpr uint32_t kFillSector = 1u << 19;
constexpr int kFlagShift = 24;
// Fluid-only ("compact") PDF layout: the fluid cells are numbered in the
// reference's linear cell order (z, y, x).  Per 32-cell chunk of a row
// (row = z*ny + y, chunk = x >> 5): the slot of its first fluid cell and the
// fluid mask, so slot(x) = rank + popc(mask & ((1 << (x & 31)) - 1)).
struct alignas(8) ChunkEnt {
  uint32_t rank;
  uint32_t mask;
};

// Units sweep (sweep_units.cu): a unit is a run of <= 32 consecutive fluid
// slots of one row whose cells lie in <= 3 consecutive chunks and hold at most
// kUnitLinkCap link records together (the warp closes them from a fixed pool
// in shared memory), so a warp that sweeps a unit has no lane on a solid
// cell.  Units are numbered in slot order.
//   yz   = y | z << 16
//   info = n (bits 0..5) | holds x = 0 (bit 6) | holds x = nx-1 (bit 7)
//          | first chunk c0 (bits 8..19) | link records (bits 20..31)
#ifndef PGPU_UNITS_LCAP
#define PGPU_UNITS_LCAP 160  // a full unit next to a wall: 32 cells x 5 links
#endif
constexpr int kUnitLinkCap = PGPU_UNITS_LCAP;
struct alignas(16) UnitRec {
  uint32_t s0;     // first fluid slot
  uint32_t lbase;  // first link record (the unit's records are contiguous)
  uint32_t yz;
  uint32_t info;
};
// Per fluid slot (units sweep): the cell word's bits 0..18 | position relative
// to the unit's first chunk, (chunk - c0) * 32 + (x & 31), in bits 19..25 |
// x == 0 (bit 26) | x == nx-1 (bit 27).
constexpr int kSlotRelShift = 19;
constexpr uint32_t kSlotX0 = 1u << 26;
constexpr uint32_t kSlotXN = 1u << 27;

struct alignas(8) CellWord {
  uint32_t w;
  int32_t base;  // first link record of the cell
};

// Constants of the contracted ("fast") TRT collision, math mode
// PGPU_MATH_FAST (lattice.cuh collide_core_fast / collide_glbm_fast).  The
// reference's per-pair update (simulation.cpp:180-193)
//   a' = a - wp(s/2 - feq+) - wm(d/2 - feq-) + fpop,  b' = b - wp(...) + wm(...) - fpop
// with s = a + b, d = a - b is regrouped as a' = P + M, b' = P - M where
//   P = hp*s + (kw1*drho + kw2*uu) + C*eu^2,   M = hm*d + D*eu + fpop
// (per weight class: 0 = axis pairs w = 1/18, 1 = diagonal pairs w = 1/36),
// and the rest population as f0' = w0*f0 + a0*drho + b0*uu.  Same algebra,
// FMA-contracted and reassociated: agrees with the reference to rounding
// (<= 1e-12 relative is the north-star tolerance; tests/test_gpu_fast.py).
struct FastCoef {
  double hp, hm;           // (1 - wp)/2, (1 - wm)/2
  double w0, a0, b0;       // 1 - wp, wp/3, -wp*rho0*1.5/3 (/eq_eps for GLBM)
  double kw1[2], kw2[2];   // wp*w, -1.5*wp*w*rho0 (/eq_eps)
  double C[2], D[2];       // 4.5*wp*w*rho0 (/eq_eps), 3*wm*w*rho0
  double fw[2];            // GLBM: force_pref * w
  double inv_rho0;
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
  // Division shortcuts that are bit-identical to the division: mode 0 divisor
  // is 1 (identity), mode 1 divisor is a power of two (multiply by its exact
  // reciprocal), mode 2 general (divide).
  int32_t eq_mode, denom_mode;
  double inv_eq_eps, inv_denom;
  FastCoef fc;         // math mode PGPU_MATH_FAST
  double f_inv_denom;  // 1 / denom_lin (fast mode, c_F == 0)
};

// Everything a sweep kernel needs, passed by value.
struct KParams {
  int32_t nx, ny, nz;
  int32_t px, py, pz;  // periodic flags (x ignored in slab mode)
  int64_t ks;          // element stride between the 19 direction planes of the sweep buffers
  int64_t ksd;         // plane stride of the dense (observable) layout, cells rounded to 32
  const ChunkEnt* ctab;  // compact layout: [rows][nchunk] chunk entries (null: dense layout)
  uint32_t poff[19];     // compact layout: j * ks; slot offsets are 32-bit unsigned
                         // (19 * ks < 2^32, i.e. up to 226 M fluid cells per GPU)
  const uint32_t* cellw;     // per-cell word (kNonFluid / bounce bits / kFillSector)
  const int32_t* cellbase;   // per-cell first link record (per-cell kernels)
  const int32_t* chunkbase;  // first link record of each 32-cell chunk of a row
  int32_t nchunk;            // chunks per row = ceil(nx / 32)
  const LinkRec* links;
  const uint16_t* linkdesc;  // per record: owner lane (x & 31) | j << 5 (compact CLI sweep)
  int64_t nrec;              // link records (bounds checks of debug builds)
  int32_t fill_sectors;      // write zeros into fill-flagged non-fluid cells
  double wp, wm, rho0, nu, cf;
  // Math mode PGPU_MATH_FAST: contracted collision (FastCoef) and, in the
  // fluid-only layout with link records, folded CLI links: the otherwise
  // unread slot k = opp(j) of a cell with a CLI link in direction j stores
  // h = g_k(x) - c*g_j(x) instead of g_k(x), so the closure is
  // f_j = c*g_k(x - e_k) + h and needs no g_j(x) load (records: SBB = 0).
  int32_t fast;
  int32_t fold;    // fast mode, fluid-only layout, records present: links folded
  int32_t moving;  // some link is a moving wall (records hold +inf for it)
  int32_t sweep;   // fluid-only K1 kernel: pgpu_sweep_kernel (0 auto, 1 cpipe, 2 tma, 3 units)
  // units sweep (sweep_units.cu; built when it is selected)
  const UnitRec* units;
  const uint32_t* slotw;   // per fluid slot
  const uint16_t* udesc;   // per link record: owner lane in its unit | j << 5
  int64_t nunits;
  // x-slab split with 32-column edge bands: the units of the two bands (the
  // edge part); `units` then covers the interior columns
  const UnitRec* units_edge;
  int64_t nunits_edge;
  uint32_t* tickets;  // TMA sweep: [0] next work item, [1] finished blocks (zero between launches)
  int32_t stream_stores;  // sweeps store the new state evict-first (domains far larger than L2)
  FastCoef fc;
  double fpop[9];   // core force term ((3*w)*rho0)*eg per pair (simulation.cpp:190)
  double wr3[9];    // (w*rho0)*3 per pair                      (simulation.cpp:185)
  double mw[19];    // moving-wall term 2*w*rho0*3*(e.u_w) per link direction (boundary.cpp:38-40)
  double hg[3];     // 0.5*g[i]/rho0  (simulation.cpp:367)
  double g[3];
  const PlaneCoef* planes;  // GLBM only
  // x-slab halo (slab mode only)
  // element offsets relative to the cell index c, valid for cells off every
  // periodic wrap face: pull source of direction j (j*ks - e_j . strides),
  // bounce source g_opp(j)(x) (opp(j)*ks), and the plane stride j*ks
  int64_t pull_off[19];
  int64_t bounce_delta[19];  // bounce source offset - pull_off
  int64_t plane_off[19];
  const double* ghost_lo;  // [5][ny*nz] g of directions 1,7,9,11,13 at x=-1
  const double* ghost_hi;  // [5][ny*nz] g of directions 2,8,10,12,14 at x=nx
  double* send_lo;         // [5][ny*nz] our g of directions 2,8,10,12,14 at x=0
  double* send_hi;         // [5][ny*nz] our g of directions 1,7,9,11,13 at x=nx-1
};

}  // namespace pgpu
