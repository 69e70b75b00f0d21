// K1 over the fluid-only layout by units of fluid slots (sm_100a).
//
// Same step as sweep_compact.cu's k_sweep_cpipe -- g' = C(P(g)), P the pull
// form of the reference's push streaming + link bounce-back
// (simulation.cpp:278-342, boundary.cpp:19-41), C the TRT / GLBM collision
// (simulation.cpp:150-274) -- with the lanes mapped to FLUID SLOTS instead of
// x positions.  k_sweep_cpipe gives every lane one cell of a 32-cell chunk, so
// inside a sphere packing (porosity 0.5) half of each warp's lanes sit on
// solid cells while the warp still issues every instruction: per fluid cell
// the bed costs twice the instructions of the free flow, and ncu shows the
// sweep issue-bound there.  Here a warp sweeps a *unit*: a run of up to 32
// consecutive fluid slots of one row (kparams.h UnitRec, built once by
// setup.cu's k_units; the cells of a unit lie in at most 3 consecutive
// chunks).  Every lane of a full unit updates a fluid cell, its 19 stores are
// one contiguous 256-byte run per direction, and the instruction count per
// fluid cell no longer depends on the porosity.
//
// Addresses: a lane's cell sits at bit b of chunk c0 + k of its row (the
// per-slot word holds k and b); with the chunk entry {rank, mask} of source
// row r at chunk c0 + k,  q_r = rank + popc(mask & ((1 << b) - 1))  is the slot
// of the fluid cell at or after this x in that row, and the pull source is
// q_r (e_x = 0), q_r - 1 (e_x = +1) or q_r + bit(mask, b) (e_x = -1), exactly
// as in k_sweep_cpipe.  The 27 chunk entries of a unit (9 source rows x 3
// chunks) and the 5 + 5 x-wrap partners are loaded by one lane each.
//
// Schedule: units are numbered in slot order (z, y, x); a block owns a run of
// 4 * upw consecutive units, dealt round-robin to its 4 warps, and each warp
// sweeps its upw units one after the other with a four-level per-warp pipeline of 8-byte / 4-byte cp.async copies -- while
// unit i is collided and stored, the populations (and link records, g_j(x))
// of unit i+1, the slot words / chunk entries / link descriptors of unit i+2
// and the unit record of i+3 are in flight.  Warps never synchronise with
// each other.
//
// The arithmetic per cell is the sweep_compact.cu one (collide<CM, GLBM>, the
// link closures in the reference order), so the results are bit-identical to
// k_sweep_cpipe in EXACT and FAST (tests/test_gpu_units.py).  It sweeps the
// whole domain or, in the x-slab split, the interior columns and the two
// 32-column edge bands in separate launches over their own unit lists (the
// EDGE instantiation reads ghost columns and fills the send buffers); KP,
// folded links and the face columns of slabs narrower than 96 stay on
// sweep_compact.cu's kernels (same state layout, so the kernels mix freely).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "kparams.h"
#include "lattice.cuh"

namespace pgpu {
namespace {

#ifndef PGPU_UNITS_MINB
#define PGPU_UNITS_MINB 4
#endif
#ifndef PGPU_BOUNDS
#define PGPU_BOUNDS 0
#endif
#ifndef PGPU_STCS
#define PGPU_STCS 1
#endif
#ifndef PGPU_UNITS_WARPS
#define PGPU_UNITS_WARPS 4
#endif
constexpr int kUW = PGPU_UNITS_WARPS;    // warps per block (independent)
constexpr int kULCap = kUnitLinkCap;     // a unit holds at most this many link records (kparams.h)

__device__ __forceinline__ uint32_t usmem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ucpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(usmem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void ucpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(usmem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void ucpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(usmem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void ucommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void uwait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void updl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void updl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void ubounds(bool ok) {
  if (PGPU_BOUNDS && !ok) __trap();
}

// Source rows exactly as in sweep_compact.cu: row r holds the directions with
// (e_y, e_z) = (urow_ey(r), urow_ez(r)).
//   r0 (0,0): 0 1 2   r1 (1,0): 3 7 10   r2 (-1,0): 4 8 9   r3 (0,1): 5 11 14
//   r4 (0,-1): 6 12 13   r5 (1,1): 15   r6 (-1,-1): 16   r7 (1,-1): 17   r8 (-1,1): 18
__host__ __device__ constexpr int urow_ey(int r) {
  return (r == 1 || r == 5 || r == 7) ? 1 : ((r == 2 || r == 6 || r == 8) ? -1 : 0);
}
__host__ __device__ constexpr int urow_ez(int r) {
  return (r == 3 || r == 5 || r == 8) ? 1 : ((r == 4 || r == 6 || r == 7) ? -1 : 0);
}
__host__ __device__ constexpr int urow_of(int j) {
  return j <= 2 ? 0
         : (j == 3 || j == 7 || j == 10) ? 1
         : (j == 4 || j == 8 || j == 9)  ? 2
         : (j == 5 || j == 11 || j == 14) ? 3
         : (j == 6 || j == 12 || j == 13) ? 4
                                          : j - 10;
}
constexpr uint32_t upack(int v0, int v1, int v2, int v3, int v4, int v5, int v6, int v7, int v8) {
  return (uint32_t)(v0 + 1) | (uint32_t)(v1 + 1) << 2 | (uint32_t)(v2 + 1) << 4 |
         (uint32_t)(v3 + 1) << 6 | (uint32_t)(v4 + 1) << 8 | (uint32_t)(v5 + 1) << 10 |
         (uint32_t)(v6 + 1) << 12 | (uint32_t)(v7 + 1) << 14 | (uint32_t)(v8 + 1) << 16;
}
constexpr uint32_t kURowEY = upack(urow_ey(0), urow_ey(1), urow_ey(2), urow_ey(3), urow_ey(4),
                                   urow_ey(5), urow_ey(6), urow_ey(7), urow_ey(8));
constexpr uint32_t kURowEZ = upack(urow_ez(0), urow_ez(1), urow_ez(2), urow_ez(3), urow_ez(4),
                                   urow_ez(5), urow_ez(6), urow_ez(7), urow_ez(8));
__device__ __forceinline__ int urt_ey(int r) { return (int)((kURowEY >> (2 * r)) & 3u) - 1; }
__device__ __forceinline__ int urt_ez(int r) { return (int)((kURowEZ >> (2 * r)) & 3u) - 1; }

__device__ __forceinline__ bool uwrap(int& v, int n, int periodic) {
  if (v >= 0 && v < n) return true;
  if (!periodic) return false;
  v = v < 0 ? v + n : v - n;
  return true;
}

// Chunk entries of a unit: ent[3 * r + k] = source row r, chunk c0 + k;
// ent[27 + r] = chunk nchunk-1 of source row r (the x = 0 cell's pulls with
// e_x = +1, rows 0..4); ent[32 + r] = chunk 0 of source row r (x = nx-1).
template <bool RECORDS>
struct alignas(16) UMeta {
  uint32_t sw[32];
  ChunkEnt ent[40];
  uint16_t ldesc[RECORDS ? kULCap + 8 : 8];
};
template <bool RECORDS>
struct alignas(16) UWarp {
  double stage[19][32];
  double pool[RECORDS ? 2 * kULCap : 2];  // per link: record, g_j(x)
  UMeta<RECORDS> meta[3];
  UnitRec rec[8];
};

// Closure of one link in the stage (boundary.cpp:24-41 in pull form): slot j
// of the owner holds g_k(x), slot k its pull value.
__device__ __forceinline__ void uclose_link(double* stage, int owner, int j, double rec, double gj,
                                            const KParams& p) {
  if (rec == rec) {
    const int k = (j & 1) ? j + 1 : j - 1;
    double* sj = stage + j * 32 + owner;
    const double gk = *sj;
    if (!isinf(rec))
      *sj = DADD(DSUB(DMUL(rec, stage[k * 32 + owner]), DMUL(rec, gj)), gk);
    else
      *sj = DSUB(gk, p.mw[k]);
  }  // NaN: simple bounce-back, slot j already holds g_k(x)
}

// EDGE: the launch sweeps the edge bands of an x-slab (units_edge): cells in
// the face columns pull their e_x = +-1 sources from the ghost columns and
// store their 5 outgoing populations into the send buffers (write_sends of
// sweep_compact.cu); everything else is the same kernel.
template <int CM, bool GLBM, bool RECORDS, bool EDGE>
__global__ void __launch_bounds__(kUW * 32, PGPU_UNITS_MINB)
    k_sweep_units(const KParams p, const UnitRec* __restrict__ units, int64_t nunits,
                  const double* __restrict__ src, double* __restrict__ dst, int upw, int group,
                  int rev) {
  extern __shared__ __align__(16) unsigned char usmem_raw[];
  updl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  UWarp<RECORDS>& S = reinterpret_cast<UWarp<RECORDS>*>(usmem_raw)[warp];
  // `group` consecutive blocks share a run of group * kUW * upw units, dealt
  // round-robin to their warps: at every pipeline step the warps of a block
  // (and, roughly, of the group) work on adjacent units -- per direction one
  // contiguous stretch of memory, and the sectors two units share hit L1.
  // (A dynamic schedule -- one resident wave of warps drawing units from a
  // global counter -- measured the same or worse on C2/C3 and was removed.)
  // block order (the hardware dispatches blockIdx.x ascending): 0 ascending in
  // z, 1 descending (consecutive SBB sweeps alternate: each starts on the
  // planes the last one wrote, still in L2), 2 two-ended (even blocks from the
  // bottom, odd blocks from the top: link-heavy bed units and free-flow units
  // are in flight together instead of one after the other)
  // 3: two-ended outward (mode 2 backwards: from the middle to both ends).
  int64_t blk = blockIdx.x;
  if (rev == 1 || rev == 3) blk = (int64_t)gridDim.x - 1 - blk;
  if (rev >= 2) blk = (blk & 1) ? (int64_t)gridDim.x - 1 - (blk >> 1) : (blk >> 1);
  const int stride = group * kUW;
  // first unit of the block and its pipeline length: block-uniform by
  // construction (blockIdx and kernel parameters only), so the compiler keeps
  // the loop control and the memory descriptors in uniform registers.  Only
  // the last block's warps 1..3 may run one unit past the end: the unit array
  // ends with zero records (n = 0: nothing to load, collide or store).
  const int64_t first = (blk / group) * ((int64_t)stride * upw) + (blk % group) * kUW;
  const int nu = (int)min((int64_t)upw, (nunits - first + stride - 1) / stride);
  const UnitRec* const U = units + first + warp;
  // the chunk entry this lane loads for every unit: lanes 0..26 source row
  // lane / 3, chunk c0 + lane % 3; lanes 27..31 the x = nx-1 partner of rows 0..4
  const int er = lane < 27 ? lane / 3 : lane - 27;
  const int ek = lane < 27 ? lane - 3 * er : 0;
  const int eey = urt_ey(er), eez = urt_ez(er);
  const uint32_t xn_below = (1u << ((p.nx - 1) & 31)) - 1u;

  auto rec_load = [&](int i) {
    if (lane == 0) ucpa16(&S.rec[i & 7], U + (int64_t)i * stride);
  };

  // slot words, chunk entries and link descriptors of unit i (its record has landed)
  auto meta_load = [&](int i) {
    const UnitRec R = S.rec[i & 7];
    UMeta<RECORDS>& M = S.meta[i % 3];
    const int n = R.info & 63, c0 = (R.info >> 8) & 0xFFF;
    const int y = R.yz & 0xFFFF, z = R.yz >> 16;
    if (lane < n) {
      ubounds((int64_t)R.s0 + lane < p.ks);
      ucpa4(&M.sw[lane], p.slotw + R.s0 + lane);
    }
    {
      int ys = y - eey, zs = z - eez;
      const bool oky = uwrap(ys, p.ny, p.py), okz = uwrap(zs, p.nz, p.pz);
      const ChunkEnt* row = p.ctab + ((int64_t)zs * p.ny + ys) * p.nchunk;
      bool ok = oky && okz;
      int c;
      if (lane < 27) {
        c = c0 + ek;
        ok = ok && c < p.nchunk;
      } else {
        c = p.nchunk - 1;
        ok = ok && !EDGE && (R.info & 64u);
      }
      if (ok)
        ucpa8(&M.ent[lane], row + c);
      else
        M.ent[lane] = ChunkEnt{0u, 0u};
    }
    if (!EDGE && (R.info & 128u) && lane < 5) {  // warp-uniform: the unit holds x = nx-1 (pulls from x = 0)
      int ys = y - urt_ey(lane), zs = z - urt_ez(lane);
      const bool oky = uwrap(ys, p.ny, p.py), okz = uwrap(zs, p.nz, p.pz);
      if (oky && okz)
        ucpa8(&M.ent[32 + lane], p.ctab + ((int64_t)zs * p.ny + ys) * p.nchunk);
      else
        M.ent[32 + lane] = ChunkEnt{0u, 0u};
    }
    if (RECORDS) {
      const int nl = min((int)(R.info >> 20), kULCap);
      if (nl) {  // 4-byte pairs from the even record at or below the unit's first
        const uint32_t a0 = R.lbase & ~1u;
        const int npairs = (int)(R.lbase + nl - a0 + 1) >> 1;
        for (int t = lane; t < npairs; t += 32) ucpa4(&M.ldesc[2 * t], p.udesc + a0 + 2 * t);
      }
    }
  };

  // populations and link extras of unit i into the stage / pool (its meta has landed)
  auto issue = [&](int i) {
    const UnitRec R = S.rec[i & 7];
    const UMeta<RECORDS>& M = S.meta[i % 3];
    const int n = R.info & 63;
    if (lane < n) {
      const uint32_t sw = M.sw[lane];
      const int rel = (sw >> kSlotRelShift) & 127;
      const int b = rel & 31;
      const uint32_t below = (1u << b) - 1u;
      const ChunkEnt* E = M.ent + (rel >> 5);
      int q[9];
      uint32_t bits = 0;  // bit r: source row r has a fluid cell at this x (rows 0..4)
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const ChunkEnt e = E[3 * r];
        q[r] = (int)e.rank + __popc(e.mask & below);
        if (r < 5) bits |= ((e.mask >> b) & 1u) << r;
      }
      const uint32_t fc = R.s0 + lane;
      ubounds((uint32_t)q[0] == fc);
      double* const st = &S.stage[0][lane];
      // slot of the e_x = +1 / -1 source per row (rows 0..4 hold those
      // directions).  A cell on an x face pulls from the periodic partner
      // column instead: its slots replace the values (selects, no divergent
      // path; x faces that are not periodic carry bounce bits, so the values
      // go unused there).
      int qp[5], qn[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        qp[r] = q[r] - 1;
        qn[r] = q[r] + (int)((bits >> r) & 1u);
      }
      if (!EDGE && (R.info & 64u)) {  // warp-uniform: the unit holds x = 0
        const bool me = sw & kSlotX0;
#pragma unroll
        for (int r = 0; r < 5; ++r) {
          const ChunkEnt e = M.ent[27 + r];
          const int v = (int)e.rank + __popc(e.mask & xn_below);
          if (me) qp[r] = v;
        }
      }
      if (!EDGE && (R.info & 128u)) {  // ... x = nx-1
        const bool me = sw & kSlotXN;
#pragma unroll
        for (int r = 0; r < 5; ++r) {
          const int v = (int)M.ent[32 + r].rank;
          if (me) qn[r] = v;
        }
      }
      // slab edge bands: ghost-column element of the source row per row 0..4
      int64_t hrow[5];
      const bool face = EDGE && (sw & (kSlotX0 | kSlotXN));
      if (EDGE && (R.info & 192u)) {  // warp-uniform: the unit holds a face column
        const int y = R.yz & 0xFFFF, z = R.yz >> 16;
#pragma unroll
        for (int r = 0; r < 5; ++r) {
          int ys = y - urow_ey(r), zs = z - urow_ez(r);
          uwrap(ys, p.ny, p.py);  // rows off a non-periodic axis carry bounce bits: unused
          uwrap(zs, p.nz, p.pz);
          hrow[r] = (int64_t)zs * p.ny + ys;
        }
      }
#pragma unroll
      for (int j = 0; j < 19; ++j) {
        uint32_t idx;  // unsigned: 19 * ks may exceed 2^31
        if (j == 0) {
          idx = fc;
        } else if ((sw >> j) & 1u) {
          idx = fc + p.poff[opp(j)];  // bounce: g_k(x)
        } else {
          const int r = urow_of(j);
          idx = (EX[j] == 0 ? q[r] : (EX[j] == 1 ? qp[r] : qn[r])) + p.poff[j];
        }
        const double* a = src + idx;
        if (EDGE && EX[j] != 0 && face && !((sw >> j) & 1u)) {
          const int64_t hp = (int64_t)p.ny * p.nz;
          if (EX[j] == 1 && (sw & kSlotX0)) a = p.ghost_lo + halo_slot(j) * hp + hrow[urow_of(j)];
          if (EX[j] == -1 && (sw & kSlotXN)) a = p.ghost_hi + halo_slot(j) * hp + hrow[urow_of(j)];
        } else {
          ubounds(idx < 19ull * p.ks);
        }
        ucpa8(st + j * 32, a);
      }
    }
    if (RECORDS) {
      const int nl = min((int)(R.info >> 20), kULCap);
      if (nl) {
        const uint16_t* ld = M.ldesc + (R.lbase & 1u);
        for (int e = lane; e < nl; e += 32) {
          const int d = ld[e];
          ubounds((int64_t)R.lbase + e < p.nrec);
          ucpa8(S.pool + 2 * e, p.links + R.lbase + e);
          ucpa8(S.pool + 2 * e + 1, src + (uint32_t)(R.s0 + (d & 31) + p.poff[d >> 5]));
        }
      }
    }
  };

  // prologue: three dependent levels of static data, then the first populations
  rec_load(0);
  if (nu > 1) rec_load(1);
  if (nu > 2) rec_load(2);
  ucommit();
  uwait_all();
  __syncwarp();
  meta_load(0);
  if (nu > 1) meta_load(1);
  if (nu > 3) rec_load(3);
  ucommit();
  uwait_all();
  __syncwarp();
  updl_wait();  // everything above is static; populations come from the previous sweep
  issue(0);
  ucommit();

  for (int i = 0; i < nu; ++i) {
    uwait_all();
    __syncwarp();
    const UnitRec R = S.rec[i & 7];
    const UMeta<RECORDS>& M = S.meta[i % 3];
    const int n = R.info & 63;
    const bool fluid = lane < n;
    const uint32_t fc = R.s0 + lane;
    if (RECORDS) {
      const int nl = (int)(R.info >> 20);
      if (nl) {  // warp-uniform
        double* const stage = &S.stage[0][0];
        const int ncoop = min(nl, kULCap);
        const uint16_t* ld = M.ldesc + (R.lbase & 1u);
        // two links per lane and round, all shared-memory reads before the
        // arithmetic (the closures of different links are independent: a
        // link whose opposite direction is cut as well has no second fluid
        // cell, so its record is SBB or moving and reads only its own slot)
        for (int e0 = lane; e0 < ncoop; e0 += 64) {
          const int e1 = e0 + 32;
          const bool two = e1 < ncoop;
          const int d0 = ld[e0], d1 = two ? ld[e1] : 0;
          const double r0 = S.pool[2 * e0], g0 = S.pool[2 * e0 + 1];
          const double r1 = two ? S.pool[2 * e1] : nan(""), g1 = two ? S.pool[2 * e1 + 1] : 0.0;
          const int j0 = d0 >> 5, o0 = d0 & 31, j1 = d1 >> 5, o1 = d1 & 31;
          const int k0 = (j0 & 1) ? j0 + 1 : j0 - 1, k1 = (j1 & 1) ? j1 + 1 : j1 - 1;
          double* const s0 = stage + j0 * 32 + o0;
          double* const s1 = stage + j1 * 32 + o1;
          const double gk0 = *s0, pk0 = stage[k0 * 32 + o0];
          double gk1 = 0.0, pk1 = 0.0;
          if (two) {
            gk1 = *s1;
            pk1 = stage[k1 * 32 + o1];
          }
          if (r0 == r0) *s0 = isinf(r0) ? DSUB(gk0, p.mw[k0]) : DADD(DSUB(DMUL(r0, pk0), DMUL(r0, g0)), gk0);
          if (r1 == r1) *s1 = isinf(r1) ? DSUB(gk1, p.mw[k1]) : DADD(DSUB(DMUL(r1, pk1), DMUL(r1, g1)), gk1);
        }
        __syncwarp();
      }
    }
    double f[19];
    if (fluid) {
#pragma unroll
      for (int j = 0; j < 19; ++j) f[j] = S.stage[j][lane];
    }
    __syncwarp();  // stage and pool consumed: refill them with unit i+1
    if (i + 1 < nu) issue(i + 1);
    if (i + 2 < nu) meta_load(i + 2);
    if (i + 4 < nu) rec_load(i + 4);
    ucommit();
    if (fluid) {
      collide<CM, GLBM>(f, p, (int)(R.yz >> 16));
      // one 64-bit base per cell, the plane offset added per direction; the
      // store kind is chosen once (inside the unrolled loop the compiler
      // predicates both stores: 2 x 19 more instructions per unit)
      double* const d0 = dst + fc;
      if (PGPU_STCS && p.stream_stores) {
#pragma unroll
        for (int j = 0; j < 19; ++j) __stcs(d0 + p.poff[j], f[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 19; ++j) d0[p.poff[j]] = f[j];
      }
      if (EDGE) {  // the 5 populations leaving through each face (sweep_compact.cu write_sends)
        const uint32_t sw = M.sw[lane];
        if (sw & (kSlotX0 | kSlotXN)) {
          const int64_t hp = (int64_t)p.ny * p.nz;
          const int64_t h = (int64_t)(R.yz >> 16) * p.ny + (R.yz & 0xFFFF);
          if (sw & kSlotX0) {
            p.send_lo[0 * hp + h] = f[2];
            p.send_lo[1 * hp + h] = f[8];
            p.send_lo[2 * hp + h] = f[10];
            p.send_lo[3 * hp + h] = f[12];
            p.send_lo[4 * hp + h] = f[14];
          }
          if (sw & kSlotXN) {
            p.send_hi[0 * hp + h] = f[1];
            p.send_hi[1 * hp + h] = f[7];
            p.send_hi[2 * hp + h] = f[9];
            p.send_hi[3 * hp + h] = f[11];
            p.send_hi[4 * hp + h] = f[13];
          }
        }
      }
    }
  }
  uwait_all();
}

int units_upw(const KParams& p) {
  const char* e = std::getenv("PGPU_UPW");  // experiments and tests (read per launch / graph capture)
  const int env = e ? std::atoi(e) : 0;
  if (env > 0) return env;
  (void)p;
  return 4;  // measured on C2/C3/C4 (tools/gpu_units_ab.sh): shorter runs pay the prologue, longer lose balance
}

template <int CM, bool GLBM, bool RECORDS, bool EDGE>
bool units_launch(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  const UnitRec* const units = EDGE ? p.units_edge : p.units;
  const int64_t nunits = EDGE ? p.nunits_edge : p.nunits;
  constexpr int smem = (int)sizeof(UWarp<RECORDS>) * kUW;
  static bool attr = [] {
    cudaFuncSetAttribute(k_sweep_units<CM, GLBM, RECORDS, EDGE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  static const bool pdl_env = [] {
    const char* e = std::getenv("PGPU_PDL");
    return !(e && e[0] == '0');
  }();
  const int upw = units_upw(p);
  // Block order, alternating between consecutive sweeps so that each starts on
  // the planes the last one wrote (still in L2).  States far above L2 (C4):
  // ascending / descending.  Smaller ones (C2, C3; KParams::stream_stores is
  // that size test): two-ended inward / outward -- the link-heavy bed units
  // and the free-flow units are then in flight together instead of one after
  // the other (C3 0.68 -> 0.72; on C4 the two fronts cost 2 %).
  // PGPU_UORDER=ab (two digits: even / odd sweeps) overrides, for experiments.
  const char* oe = std::getenv("PGPU_UORDER");
  int order = p.stream_stores ? (cfg.odd ? 1 : 0) : (cfg.odd ? 3 : 2);
  if (oe && oe[0] && oe[1]) order = (cfg.odd ? oe[1] : oe[0]) - '0';
  const char* ge = std::getenv("PGPU_UGROUP");
  const int group = std::max(1, ge ? std::atoi(ge) : 1);
  const int64_t per_group = (int64_t)group * kUW * upw;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)((nunits + per_group - 1) / per_group * group));
  lc.blockDim = dim3(kUW * 32);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_env && !cfg.slab ? 1 : 0;
  return cudaLaunchKernelEx(&lc, k_sweep_units<CM, GLBM, RECORDS, EDGE>, p, units, nunits, src, dst,
                            upw, group, order) == cudaSuccess;
}

template <int CM, bool EDGE>
bool units_cm_e(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                cudaStream_t s) {
  if (cfg.glbm)
    return cfg.records ? units_launch<CM, true, true, EDGE>(cfg, p, src, dst, s)
                       : units_launch<CM, true, false, EDGE>(cfg, p, src, dst, s);
  return cfg.records ? units_launch<CM, false, true, EDGE>(cfg, p, src, dst, s)
                     : units_launch<CM, false, false, EDGE>(cfg, p, src, dst, s);
}
template <int CM>
bool units_cm(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
              cudaStream_t s) {
  return cfg.part == PART_EDGES ? units_cm_e<CM, true>(cfg, p, src, dst, s)
                                : units_cm_e<CM, false>(cfg, p, src, dst, s);
}

}  // namespace

int sweep_edge_band(int nx) { return edge_band(nx); }

bool units_sweep_supported(const SweepConfig& cfg, const KParams& p) {
  // slab split: `units` covers the interior columns, `units_edge` the two
  // 32-column edge bands when the slab has them (sim_impl.h ensure_units)
  const bool edges = cfg.slab && cfg.part == PART_EDGES && p.units_edge && p.nunits_edge > 0;
  return p.ctab && p.units && p.slotw && p.nunits > 0 &&
         (edges || cfg.part == (cfg.slab ? PART_INTERIOR : PART_ALL)) && cfg.op == OP_STREAM_COLLIDE && collide_mode(p) != CM_FAST_FOLD &&
         (p.udesc || !cfg.records) && p.nchunk <= 4096 && p.ny <= 65535 && p.nz <= 65535;
}

bool launch_sweep_units(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                        cudaStream_t s) {
  switch (collide_mode(p)) {
    case CM_FAST: return units_cm<CM_FAST>(cfg, p, src, dst, s);
    case CM_EXACT_RHO1: return units_cm<CM_EXACT_RHO1>(cfg, p, src, dst, s);
    case CM_EXACT: return units_cm<CM_EXACT>(cfg, p, src, dst, s);
    default: return false;
  }
}

}  // namespace pgpu
