// sm_100a sweeps over the fluid-only ("compact") PDF layout.
//
// Layout: the fluid cells are numbered in the reference's linear cell order
// (z, y, x) (field.hpp:19-21 restricted to fluid cells); direction plane j of
// a sweep buffer holds g_j of fluid cell n at element j*ks + n.  Per 32-cell
// chunk of a row a ChunkEnt {rank, mask} gives
//     slot(x) = rank + popc(mask & ((1 << (x & 31)) - 1)).
// Solid and wall cells occupy no storage, so a sweep moves exactly the 304 B
// per fluid cell of the algorithm (no 32-byte sectors shared with solid cells,
// no sector-completion writes).  The observable ("pre-collision") state stays
// in the reference's dense layout in a separate buffer (plane stride ksd):
//   K0  k_collide_to_compact : g = C(f)   dense f -> compact g (first step)
//   K1  k_sweep_cpipe        : g' = C(P(g))  compact -> compact (the hot kernel)
//   KP  k_sweep_cpipe<KP>    : f = P(g)   compact -> dense (observables)
// with P the pull form of the reference's push streaming + link bounce-back
// (simulation.cpp:278-342, boundary.cpp:19-41), exactly as in
// kernels.cu.
//
// K1 keeps the structure of kernels.cu's k_sweep_pipe (per-thread cp.async
// pipeline, pooled link closures) with fluid-only addressing: one chunk entry
// per source row and plane gives every pull slot with a popcount, and the
// CLI link lists come from static per-record descriptors (see
// k_sweep_cpipe).  A TMA variant (one cp.async.bulk per direction run and
// warp) moved the same bytes but was instruction-bound (3.35 G instructions
// per C4 launch vs 2.16 G, 7.1 ms); it is kept in tools/experiments/, and the
// measured configuration choices are in profiles/r01b_compact_k1_ncu_summary.md.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "kparams.h"
#include "lattice.cuh"

namespace pgpu {
bool g_plain_sweep();  // kernels.cu: PGPU_SWEEP=plain
namespace {

// ---------------------------------------------------------------------------
// Small PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cpa4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// Programmatic dependent launch (no-ops without the launch attribute): let the
// next sweep's blocks start, and wait for the previous grid's results.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Compact index helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t fidx(const KParams& p, int x, int y, int z) {
  return compact_slot(p, x, y, z);
}

// Source rows: row r holds the directions with (e_y, e_z) = (row_ey(r), row_ez(r)); their
// pull sources lie in row (y - e_y, z - e_z).
//   r0 (0,0): 0 1 2   r1 (1,0): 3 7 10   r2 (-1,0): 4 8 9   r3 (0,1): 5 11 14
//   r4 (0,-1): 6 12 13   r5 (1,1): 15   r6 (-1,-1): 16   r7 (1,-1): 17   r8 (-1,1): 18
__host__ __device__ constexpr int row_ey(int r) {
  return (r == 1 || r == 5 || r == 7) ? 1 : ((r == 2 || r == 6 || r == 8) ? -1 : 0);
}
__host__ __device__ constexpr int row_ez(int r) {
  return (r == 3 || r == 5 || r == 8) ? 1 : ((r == 4 || r == 6 || r == 7) ? -1 : 0);
}
__host__ __device__ constexpr int row_of(int j) {
  return j <= 2 ? 0
         : (j == 3 || j == 7 || j == 10) ? 1
         : (j == 4 || j == 8 || j == 9)  ? 2
         : (j == 5 || j == 11 || j == 14) ? 3
         : (j == 6 || j == 12 || j == 13) ? 4
                                          : j - 10;  // 15..18 -> 5..8
}

// x-slab split: each edge band (edge_band() = 32 columns) is exactly the first
// / last 32-cell chunk of a row.
__host__ __device__ __forceinline__ bool edge_chunks(const KParams& p) {
  return p.nx % 32 == 0 && edge_band(p.nx) == 32;
}

// Periodic wrap of a row coordinate; false if it leaves a non-periodic axis.
__device__ __forceinline__ bool wrap_coord(int& v, int n, int periodic) {
  if (v >= 0 && v < n) return true;
  if (!periodic) return false;
  v = v < 0 ? v + n : v - n;
  return true;
}

// ---------------------------------------------------------------------------
// Per-cell compact sweep (edge bands of the slab split, PGPU_SWEEP=plain, and
// the reference point for the pipelined kernel): same arithmetic as kernels.cu's
// sweep_cell, addresses through the chunk table.
// ---------------------------------------------------------------------------
template <int J, bool SLAB>
__device__ __forceinline__ const double* cpull_addr(const double* __restrict__ src, int x, int y,
                                                    int z, int64_t fc, const KParams& p,
                                                    uint32_t w) {
  constexpr int ex = EX[J], ey = EY[J], ez = EZ[J];
  if (J == 0) return src + fc;
  if ((w >> J) & 1u) return src + (int64_t)opp(J) * p.ks + fc;  // bounce: g_k(x)
  int ys = y - ey, zs = z - ez;
  if (ey == 1 && y == 0) ys = p.ny - 1;
  if (ey == -1 && y == p.ny - 1) ys = 0;
  if (ez == 1 && z == 0) zs = p.nz - 1;
  if (ez == -1 && z == p.nz - 1) zs = 0;
  int xs = x - ex;
  if (ex == 1 && x == 0) {
    if (SLAB) return p.ghost_lo + (int64_t)halo_slot(J) * p.ny * p.nz + zs * p.ny + ys;
    xs = p.nx - 1;
  }
  if (ex == -1 && x == p.nx - 1) {
    if (SLAB) return p.ghost_hi + (int64_t)halo_slot(J) * p.ny * p.nz + zs * p.ny + ys;
    xs = 0;
  }
  return src + (int64_t)J * p.ks + fidx(p, xs, ys, zs);
}

template <int J, bool SLAB>
__device__ __forceinline__ void cload_all(double (&f)[19], const double* __restrict__ src, int x,
                                          int y, int z, int64_t fc, const KParams& p,
                                          uint32_t w) {
  if constexpr (J < 19) {
    f[J] = __ldg(cpull_addr<J, SLAB>(src, x, y, z, fc, p, w));
    cload_all<J + 1, SLAB>(f, src, x, y, z, fc, p, w);
  }
}

// CLI / moving-wall closures; f[J] already holds g_k(x) (boundary.cpp:24-41).
template <int J>
__device__ __forceinline__ void clinks_all(double (&f)[19], const double* __restrict__ src,
                                           int64_t fc, const KParams& p, uint32_t w,
                                           int32_t base) {
  if constexpr (J < 19) {
    if ((w >> J) & 1u) {
      constexpr int K = opp(J);
      const int32_t r = base + __popc(w & ((1u << J) - 1u) & kBounceMask);
      const double rec = __ldg(p.links + r);
      const double gj = __ldg(src + (int64_t)J * p.ks + fc);
      if (rec == rec) {
        if (!isinf(rec))
          f[J] = DADD(DSUB(DMUL(rec, f[K]), DMUL(rec, gj)), f[J]);
        else
          f[J] = DSUB(f[J], p.mw[K]);
      }
    }
    clinks_all<J + 1>(f, src, fc, p, w, base);
  }
}

// Math mode fast, fluid-only layout with records: folded CLI links (kparams.h
// KParams::fast).  f[J] holds h (slot k = opp J of the cell); CLI records
// close f_J = c*g_k(x - e_k) + h; moving walls (+inf, only when p.moving)
// keep h = g_k(x) unfolded and subtract the wall term exactly like
// boundary.cpp:34-41; SBB records are 0 (nothing to do).  f[K] of a CLI link
// is a pull value (x - e_k is fluid), never the target of another closure.
__device__ __forceinline__ void close_fold(double& fj, double fk, double rec, const KParams& p,
                                           int k) {
  if (rec != 0.0) fj = (p.moving && isinf(rec)) ? DSUB(fj, p.mw[k]) : fma(rec, fk, fj);
}
template <int J>
__device__ __forceinline__ void clinks_fold_all(double (&f)[19], const KParams& p, uint32_t w,
                                                int32_t base) {
  if constexpr (J < 19) {
    if ((w >> J) & 1u) {
      const int32_t r = base + __popc(w & ((1u << J) - 1u) & kBounceMask);
      close_fold(f[J], f[opp(J)], __ldg(p.links + r), p, opp(J));
    }
    clinks_fold_all<J + 1>(f, p, w, base);
  }
}
// Epilogue of a folded sweep: for each link of the cell (bounce bits `bm`, its
// records rec(0), rec(1), ... in (cell, j) order) store h = g_k - c*g_j in
// slot k = opp(j) of the new post-collision state.  Both links of a pair read
// the un-folded values.
template <class Rec>
__device__ __forceinline__ void fold_epilogue(double (&f)[19], uint32_t bm, const KParams& p,
                                              Rec&& rec) {
  int r = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int k = 1 + 2 * q, kb = k + 1;
    const double gk = f[k], gkb = f[kb];
    if ((bm >> k) & 1u) {  // link closing f_k: its h lives in slot kb
      const double c = rec(r++);
      if (!(p.moving && isinf(c))) f[kb] = fma(-c, gk, gkb);
    }
    if ((bm >> kb) & 1u) {
      const double c = rec(r++);
      if (!(p.moving && isinf(c))) f[k] = fma(-c, gkb, gk);
    }
  }
}

// The same for a warp of the pipelined sweep whose chunk-plane records all sit
// in the shared-memory pool (no moving walls): `um` = the warp's union of
// bounce bits (uniform), so directions no lane links are skipped without
// divergence; the rest is predicated (pool reads past the lane's own records
// land in the pool and are unused).
__device__ __forceinline__ void fold_epilogue_pool(double (&f)[19], uint32_t bm, uint32_t um,
                                                   const double* pool, int r) {
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int k = 1 + 2 * q, kb = k + 1;
    const double gk = f[k], gkb = f[kb];
    if ((um >> k) & 1u) {
      const bool b = (bm >> k) & 1u;
      const double c = pool[r];
      if (b) f[kb] = fma(-c, gk, gkb);
      r += b;
    }
    if ((um >> kb) & 1u) {
      const bool b = (bm >> kb) & 1u;
      const double c = pool[r];
      if (b) f[k] = fma(-c, gkb, gk);
      r += b;
    }
  }
}

template <bool SLAB>
__device__ __forceinline__ void write_sends(const KParams& p, int x, int y, int z,
                                            const double (&f)[19]) {
  if (!SLAB) return;
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

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__device__ __forceinline__ void csweep_cell(const KParams& p, const double* __restrict__ src,
                                            double* __restrict__ dst, int x, int y, int z) {
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = __ldg(p.cellw + c);
  if (w & kNonFluid) return;
  const int64_t fc = fidx(p, x, y, z);
  constexpr bool FOLD = RECORDS && CM == CM_FAST_FOLD;
  double f[19];
  cload_all<0, SLAB>(f, src, x, y, z, fc, p, w);
  const int32_t base = (RECORDS && (w & kBounceMask)) ? __ldg(p.cellbase + c) : 0;
  if (RECORDS && (w & kBounceMask)) {
    if (FOLD) clinks_fold_all<1>(f, p, w, base);
    else clinks_all<1>(f, src, fc, p, w, base);
  }
  if (OP == OP_STREAM_COLLIDE) {
    collide<CM, GLBM>(f, p, z);
    if (FOLD && (w & kBounceMask))
      fold_epilogue(f, w & kBounceMask, p, [&](int i) { return __ldg(p.links + base + i); });
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcs(dst + (int64_t)j * p.ks + fc, f[j]);
    write_sends<SLAB>(p, x, y, z, f);
  } else {  // KP: f(n) into the other compact buffer
#pragma unroll
    for (int j = 0; j < 19; ++j) dst[(int64_t)j * p.ks + fc] = f[j];
  }
}

// One thread per cell of the box (part ALL / INTERIOR) ...
template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_csweep_cells(const KParams p,
                                                      const double* __restrict__ src,
                                                      double* __restrict__ dst, int part) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= p.nx) return;
  if (part == PART_INTERIOR && in_edge_band(x, p.nx)) return;
  csweep_cell<CM, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, blockIdx.y, blockIdx.z);
}
// ... or of the two x edge bands (slab split; threads walk the band's
// (y, column) pairs, grid (2, ceil(ny * band / 128), nz)).
template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_csweep_edges(const KParams p,
                                                      const double* __restrict__ src,
                                                      double* __restrict__ dst) {
  const int w = edge_band(p.nx);
  const int t = blockIdx.y * blockDim.x + threadIdx.x;
  const int xx = t % w, y = t / w;
  const int z = blockIdx.z;
  if (y >= p.ny) return;
  const int x = blockIdx.x ? p.nx - w + xx : xx;
  if (blockIdx.x && x < w) return;
  csweep_cell<CM, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z);
}

// K0: pre-collision f(n) -> post-collision g(n) in place on the compact
// buffer (simulation.cpp:150-274).
template <int CM, bool GLBM, bool SLAB, bool FOLD>
__global__ void __launch_bounds__(128) k_collide_compact(const KParams p, double* buf) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = __ldg(p.cellw + c);
  if (w & kNonFluid) return;
  const int64_t fc = fidx(p, x, y, z);
  double f[19];
#pragma unroll
  for (int j = 0; j < 19; ++j) f[j] = buf[(int64_t)j * p.ks + fc];
  collide<CM, GLBM>(f, p, z);
  if (FOLD && (w & kBounceMask)) {
    const int32_t base = __ldg(p.cellbase + c);
    fold_epilogue(f, w & kBounceMask, p, [&](int i) { return __ldg(p.links + base + i); });
  }
#pragma unroll
  for (int j = 0; j < 19; ++j) buf[(int64_t)j * p.ks + fc] = f[j];
  write_sends<SLAB>(p, x, y, z, f);
}

// Reference-layout staging of a z-range [z0, z0 + nzc) for population I/O:
// expand (compact -> dense, zeros in non-fluid cells) or pack (dense ->
// compact).  `dense` holds 19 planes of nzc * nx * ny cells.
template <bool EXPAND>
__global__ void k_compact_io(const KParams p, double* __restrict__ f, double* __restrict__ dense,
                             int z0, int nzc) {
  const int64_t chunk = (int64_t)nzc * p.ny * p.nx;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= chunk) return;
  const int x = (int)(i % p.nx), y = (int)((i / p.nx) % p.ny), z = z0 + (int)(i / ((int64_t)p.nx * p.ny));
  const bool fluid = !(__ldg(p.cellw + ((int64_t)z * p.ny + y) * p.nx + x) & kNonFluid);
  const int64_t fc = fluid ? fidx(p, x, y, z) : 0;
#pragma unroll
  for (int j = 0; j < 19; ++j) {
    if (EXPAND)
      dense[(int64_t)j * chunk + i] = fluid ? f[(int64_t)j * p.ks + fc] : 0.0;
    else if (fluid)
      f[(int64_t)j * p.ks + fc] = dense[(int64_t)j * chunk + i];
  }
}

__global__ void k_fill_compact(const KParams p, int64_t nfluid, double* __restrict__ f,
                               const double* __restrict__ feq) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nfluid) return;
#pragma unroll
  for (int j = 0; j < 19; ++j) f[(int64_t)j * p.ks + i] = feq[j];
}

// Order of the z-blocks (the hardware dispatches blockIdx.z in increasing
// order).  bit 0: descending, so consecutive sweeps alternate and each starts
// on the planes the previous one wrote last (still in L2); bit 1: the two
// boundary z-blocks first -- they hold the planes next to the walls (5 links
// per cell), the slowest blocks, which must not end up in the tail wave.
__device__ __forceinline__ int zblock_of(int pos, int zg, int mode) {
  const bool rev = mode & 1;
  if (!(mode & 2) || zg < 3) return rev ? zg - 1 - pos : pos;
  if (!rev) return pos == 0 ? zg - 1 : pos - 1;  // zg-1, 0, 1, ..., zg-2
  return pos == 0 ? 0 : zg - pos;                // 0, zg-1, zg-2, ..., 1
}

// Warp-exclusive prefix sum of n; the warp total in *total.
__device__ __forceinline__ int warp_scan_excl(int n, int lane, int* total) {
  int v = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  *total = __shfl_sync(0xffffffffu, v, 31);
  return v - n;
}

// Pull source of direction j for the lane at x = 0 (e_x = +1) or x = nx-1
// (e_x = -1): the periodic partner cell x = nx-1 / 0 of the source row (its
// chunk entry `pe`), or the slab ghost column.  The source is fluid.
template <bool SLAB>
__device__ __forceinline__ const double* wrap_src(const KParams& p, const double* src,
                                                  ChunkEnt pe, int j, int x, int y, int z) {
  int ys = y - EY[j], zs = z - EZ[j];
  if (ys < 0) ys += p.ny;
  if (ys >= p.ny) ys -= p.ny;
  if (zs < 0) zs += p.nz;
  if (zs >= p.nz) zs -= p.nz;
  const bool plus = EX[j] == 1;
  if (SLAB)
    return (plus ? p.ghost_lo : p.ghost_hi) + (int64_t)halo_slot(j) * p.ny * p.nz +
           (int64_t)zs * p.ny + ys;
  const int64_t idx =
      plus ? (int64_t)pe.rank + __popc(pe.mask & ((1u << ((p.nx - 1) & 31)) - 1u)) : (int64_t)pe.rank;
  return src + (int64_t)j * p.ks + idx;
}

// ---------------------------------------------------------------------------
// K1 / KP: asynchronous-copy pipeline over the compact layout.
//
// A block owns a 128-cell x segment of one row (4 warps = 4 chunks) and
// marches through `zper` z-planes.  While plane z is collided, each thread's
// 19 loads for plane z+1 are in flight as 8-byte cp.async copies into its own
// shared-memory slots, and the cell words and chunk entries of plane z+3 are
// on their way (a 3-slot ring).  The pull source of direction j lies in
// source row r = row_of(j); with the row's chunk entry {rank, mask},
//     q_r = rank + popc(mask & lanemask_lt)
// is the slot of the fluid cell at (or after) this x in that row, and the
// source slot is q_r (e_x = 0), q_r - 1 (e_x = +1) or q_r + bit(mask, lane)
// (e_x = -1) -- exact because a pulled source is always fluid.  Bounce
// directions load g_k(x) from the cell's own slot instead (f_j = g_k(x) for
// SBB).  CLI / moving-wall links: a chunk-plane's links are the records
// [chunkbase, next chunkbase); their descriptors (owner lane | j << 5, built
// once at setup) ride in the meta ring, the 32 lanes copy each link's record
// and g_j(x) into a per-warp pool with the plane's populations, and close the
// links cooperatively in shared memory before the collision.  Addresses are
// unsigned 32-bit slot offsets from the buffer base (plane j at p.poff[j]); only lanes
// on the periodic x faces take the general path (partner chunk / slab ghosts).
// ---------------------------------------------------------------------------
#ifndef PGPU_CW
#define PGPU_CW 4
#endif
constexpr int kCW = PGPU_CW;      // warps (= chunks) per block
constexpr int kCBXp = kCW * 32;   // cells per block
#ifndef PGPU_CLI_STAGES
#define PGPU_CLI_STAGES 1
#endif
#ifndef PGPU_CLI_MINB
#define PGPU_CLI_MINB 4
#endif
#ifndef PGPU_SBB_MINB
#define PGPU_SBB_MINB 4
#endif
#ifndef PGPU_SBB_STAGES
#define PGPU_SBB_STAGES 1
#endif
__host__ __device__ constexpr int cp_stages(bool records) {
  return records ? PGPU_CLI_STAGES : PGPU_SBB_STAGES;
}
__host__ __device__ constexpr int cp_minb(bool records) {
  return records ? PGPU_CLI_MINB : PGPU_SBB_MINB;
}
#ifndef PGPU_SMEM_PAD
#define PGPU_SMEM_PAD 0
#endif
#ifndef PGPU_BOUNDS
#define PGPU_BOUNDS 0  // debug builds: trap on any out-of-range slot / record / ghost address
#endif
#ifndef PGPU_STCS
#define PGPU_STCS 1  // streaming (evict-first) stores of the new state
#endif
// CLane.w bit of a fluid cell that the launch's part does not sweep
constexpr uint32_t kInactive = 1u << 20;
#ifndef PGPU_CPOOL
#define PGPU_CPOOL 192
#endif
constexpr int kCPool = PGPU_CPOOL;    // per-warp, per-stage extras (record + g_j(x) per link)
constexpr int kCLinkCap = kCPool / 2;

// Packed row tables (2 bits per row, value + 1).
constexpr uint32_t pack_rows(int v0, int v1, int v2, int v3, int v4, int v5, int v6, int v7, int v8) {
  return (uint32_t)(v0 + 1) | (uint32_t)(v1 + 1) << 2 | (uint32_t)(v2 + 1) << 4 |
         (uint32_t)(v3 + 1) << 6 | (uint32_t)(v4 + 1) << 8 | (uint32_t)(v5 + 1) << 10 |
         (uint32_t)(v6 + 1) << 12 | (uint32_t)(v7 + 1) << 14 | (uint32_t)(v8 + 1) << 16;
}
constexpr uint32_t kRowEYp = pack_rows(row_ey(0), row_ey(1), row_ey(2), row_ey(3), row_ey(4),
                                       row_ey(5), row_ey(6), row_ey(7), row_ey(8));
constexpr uint32_t kRowEZp = pack_rows(row_ez(0), row_ez(1), row_ez(2), row_ez(3), row_ez(4),
                                       row_ez(5), row_ez(6), row_ez(7), row_ez(8));
__device__ __forceinline__ int rt_row_ey(int r) { return (int)((kRowEYp >> (2 * r)) & 3u) - 1; }
__device__ __forceinline__ int rt_row_ez(int r) { return (int)((kRowEZp >> (2 * r)) & 3u) - 1; }

__device__ __forceinline__ int opp_rt(int j) { return (j & 1) ? j + 1 : j - 1; }
__device__ __forceinline__ void bounds_ok(bool ok) {
  if (PGPU_BOUNDS && !ok) __trap();
}
// slot `idx` lies in direction plane `plane` of a compact buffer
__device__ __forceinline__ bool in_plane(const KParams& p, uint32_t idx, int plane) {
  return idx >= p.poff[plane] && (int64_t)idx < (int64_t)p.poff[plane] + p.ks;
}
// address lies in a sweep buffer or a ghost column buffer
__device__ __forceinline__ bool in_src(const KParams& p, const double* src, const double* a) {
  const int64_t hp = 5 * (int64_t)p.ny * p.nz;
  return (a >= src && a < src + 19 * p.ks) ||
         (p.ghost_lo && a >= p.ghost_lo && a < p.ghost_lo + hp) ||
         (p.ghost_hi && a >= p.ghost_hi && a < p.ghost_hi + hp);
}

struct CLinkDesc {
  int32_t rec;  // index into p.links
  int32_t oj;   // owner thread << 8 | j
};
struct CLane {
  uint32_t w;  // cell word of the plane (| kInactive: a fluid cell this part skips)
  int32_t fc;  // compact slot of the cell
};
struct alignas(16) CMeta {  // one plane, loaded two planes ahead of its issue
  uint32_t cw[kCBXp];
  ChunkEnt ent[kCW][16];  // per warp: 0..8 source rows, 9..13 x-wrap partners of rows 0..4,
                          // 14.rank / 15.rank = first link record of the chunk / the next one
  uint16_t ldesc[kCW][kCLinkCap + 2];  // the chunk's link descriptors (one-stage CLI sweeps)
};
// FOLD (folded CLI links, math mode fast): the pool holds only the records,
// for two planes (by z parity): the epilogue of plane z reads them after the
// stage has been refilled with plane z+1.
template <bool RECORDS, bool FOLD>
struct alignas(16) CSmem {
  static constexpr int S = cp_stages(RECORDS);
  static constexpr int PW = FOLD ? 2 * kCLinkCap : (RECORDS ? kCPool + kCLinkCap : 1);
  double main[S][19][kCBXp];
  double pool[S][kCW][PW];
  CLane lane[S][kCBXp];
  int32_t cbase[S][kCW];
  CMeta meta[3];
};

__device__ __forceinline__ void cpublish_links(CLinkDesc* desc, uint32_t w, int32_t base, int off,
                                               int tx) {
  uint32_t m = w & kBounceMask;
  int i = 0;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    const int e = off + i;
    if (e < kCLinkCap) desc[e] = CLinkDesc{base + i, (tx << 8) | j};
    ++i;
  }
}

// Closure of one link in the stage (boundary.cpp:24-41 in pull form): slot j
// of the owner holds g_k(x), slot k its pull value.
__device__ __forceinline__ void cclose_link(double* stage, int owner, int j, double rec, double gj,
                                            const KParams& p) {
  if (rec == rec) {
    const int k = (j & 1) ? j + 1 : j - 1;
    double* sj = stage + j * kCBXp + owner;
    const double gk = *sj;
    if (!isinf(rec))
      *sj = DADD(DSUB(DMUL(rec, stage[k * kCBXp + owner]), DMUL(rec, gj)), gk);
    else
      *sj = DSUB(gk, p.mw[k]);
  }  // NaN: simple bounce-back, slot j already holds g_k(x)
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(kCBXp, cp_minb(RECORDS))
    k_sweep_cpipe(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                  int part, int zper, int zrev) {
  constexpr bool FOLD = RECORDS && CM == CM_FAST_FOLD;
  using Sm = CSmem<RECORDS, FOLD>;
  constexpr int kS = Sm::S;
  static_assert(!FOLD || kS == 1, "folded links: one-stage pipeline");
  // one-stage CLI sweeps take each chunk-plane's link list from the static
  // per-record descriptors (p.linkdesc); two-stage ones build it per plane
  constexpr bool kStaticDesc = RECORDS && kS == 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  // with programmatic dependent launch the next sweep's blocks may be
  // scheduled now: their static meta loads overlap this grid's tail
  pdl_trigger();
  const int tx = threadIdx.x, lane = tx & 31, warp = tx >> 5;
  // warps are independent: a block covers 4 chunks of one row, or (edge part,
  // x-slab split) the first and last chunk of two rows
  const bool edges = part == PART_EDGES;
  // interior part with whole-chunk edge bands: warps walk the (row, interior
  // chunk) pairs linearly, so no warp slot is spent on an edge chunk
  const bool ilin = part == PART_INTERIOR && edge_chunks(p);
  int xc, y;
  if (edges) {
    xc = (warp & 1) ? p.nchunk - 1 : 0;
    y = blockIdx.y * (kCW / 2) + (warp >> 1);
  } else if (ilin) {
    const int ni = p.nchunk - 2, wl = blockIdx.x * kCW + warp;
    y = wl / ni;
    xc = 1 + wl % ni;
  } else {
    xc = blockIdx.x * kCW + warp;
    y = blockIdx.y;
  }
  const int x = xc * 32 + lane;
  const int z0 = zblock_of(blockIdx.z, gridDim.z, zrev) * zper;
  const int z1 = min(z0 + zper, p.nz);
  const bool wok = xc < p.nchunk && y < p.ny;
  const bool valid = wok && x < p.nx;
  const bool active = valid && (part == PART_ALL || (in_edge_band(x, p.nx) == edges));
  if (!__any_sync(0xffffffffu, active)) return;  // whole warp (no block-level sync below)
  const uint32_t ltl = (1u << lane) - 1u;
  // per-lane parts of the meta addresses that do not change along z: the
  // in-plane offset of this lane's chunk entry (lanes 0..8 source rows,
  // 9..13 x-wrap partners, 14 the chunk's link base), -1: nothing to load
  int eoff = -1;
  if (lane < 16 && wok) {
    if (lane < 14) {
      const int r = lane < 9 ? lane : lane - 9;
      int ys = y - rt_row_ey(r);
      const bool wrapchunk = xc == 0 || xc == p.nchunk - 1;
      if (wrap_coord(ys, p.ny, p.py) && (lane < 9 || (!SLAB && wrapchunk)))
        eoff = ys * p.nchunk + (lane < 9 ? xc : (xc == 0 ? p.nchunk - 1 : 0));
    } else if (RECORDS) {
      eoff = y * p.nchunk + xc;  // lane 14: this chunk's link base (lane 15: the next one)
    }
  }

  auto meta_load = [&](int z, int m) {
    CMeta& M = S.meta[m];
    if (valid)
      cpa4(&M.cw[tx], p.cellw + ((int64_t)z * p.ny + y) * p.nx + x);
    else
      M.cw[tx] = kNonFluid;
    if (lane < 16) {
      const int64_t plane = (int64_t)p.ny * p.nchunk;
      if (lane < 14) {
        int zs = z - rt_row_ez(lane < 9 ? lane : lane - 9);
        const bool ok = wrap_coord(zs, p.nz, p.pz) && eoff >= 0;
        if (ok)
          cpa8(&M.ent[warp][lane], p.ctab + zs * plane + eoff);
        else
          M.ent[warp][lane] = ChunkEnt{0u, 0u};
      } else if (eoff >= 0) {  // chunk bases are contiguous; a sentinel follows the last
        cpa4(&M.ent[warp][lane].rank, p.chunkbase + z * plane + eoff + (lane - 14));
      }
    }
  };

  // issue plane z (meta slot m) into stage s; returns the warp's link count
  // what: 1 the populations, 2 the link extras (records, g_j(x)), 3 both
  auto issue = [&](int z, int s, int m, int what = 3) -> int {
    const CMeta& M = S.meta[m];
    const uint32_t cw = M.cw[tx];
    const bool fl = !(cw & kNonFluid);
    const ChunkEnt* E = M.ent[warp];
    if (what & 1) {
    int q[9];
    uint32_t bits = 0;  // bit r: the source row r has a fluid cell at this x (rows 0..4)
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const ChunkEnt e = E[r];
      q[r] = (int)e.rank + __popc(e.mask & ltl);
      if (r < 5) bits |= ((e.mask >> lane) & 1u) << r;
    }
    const int fc = q[0];
    S.lane[s][tx] = CLane{active ? cw : (cw | kInactive), fc};
    if (lane == 0 && RECORDS) S.cbase[s][warp] = (int32_t)E[14].rank;
    if (fl && active) {
      double* const st = &S.main[s][0][tx];
      if (!(x == 0 || x == p.nx - 1)) {
#pragma unroll
        for (int j = 0; j < 19; ++j) {
          uint32_t idx;  // unsigned: 19 * ks may exceed 2^31
          if (j == 0) {
            idx = fc;
          } else if ((cw >> j) & 1u) {
            idx = fc + p.poff[opp(j)];  // bounce: g_k(x)
          } else {
            const int r = row_of(j);
            idx = q[r] + p.poff[j];
            if (EX[j] == 1) idx -= 1;
            if (EX[j] == -1) idx += (bits >> r) & 1u;
          }
          bounds_ok(in_plane(p, idx, ((cw >> j) & 1u) ? opp(j) : j));
          cpa8(st + j * kCBXp, src + (uint32_t)idx);
        }
      } else {  // periodic x face / slab edge column: partner chunk or ghost
#pragma unroll
        for (int j = 0; j < 19; ++j) {
          const double* a;
          if (j == 0) {
            a = src + (uint32_t)fc;
          } else if ((cw >> j) & 1u) {
            a = src + (uint32_t)(fc + p.poff[opp(j)]);
          } else if ((EX[j] == 1 && x == 0) || (EX[j] == -1 && x == p.nx - 1)) {
            a = wrap_src<SLAB>(p, src, E[9 + row_of(j)], j, x, y, z);
          } else {
            const int r = row_of(j);
            uint32_t idx = q[r] + p.poff[j];
            if (EX[j] == 1) idx -= 1;
            if (EX[j] == -1) idx += (bits >> r) & 1u;
            a = src + (uint32_t)idx;
          }
          bounds_ok(in_src(p, src, a));
          cpa8(st + j * kCBXp, a);
        }
      }
    }
    }  // what & 1
    int total = 0;
    if (!(what & 2)) return total;
    if (RECORDS && kStaticDesc) {
      // the chunk-plane's links are records [cb, cbn) with their (lane, j)
      // descriptors already in the meta slot: no prefix sum, no publish loop
      const int32_t cb = (int32_t)E[14].rank;
      total = (int32_t)E[15].rank - cb;
      if (FOLD && total) {  // records only, contiguous: no descriptors needed here
        double* pool = S.pool[s][warp] + (z & 1) * kCLinkCap;
        const int nl = min(total, kCLinkCap);
        for (int e = lane; e < nl; e += 32) {
          bounds_ok(cb + e < p.nrec);
          cpa8(pool + e, p.links + cb + e);
        }
      } else if (total) {
        double* pool = S.pool[s][warp];
        const uint16_t* ld = M.ldesc[warp] + (cb & 1);
        const int nl = min(total, kCLinkCap);
        __syncwarp();  // every lane's S.lane entry of plane z is written
        for (int e = lane; e < nl; e += 32) {
          const int d = ld[e];
          const int j = d >> 5, fco = S.lane[s][(tx & ~31) | (d & 31)].fc;
          bounds_ok(cb + e < p.nrec && in_plane(p, fco + p.poff[j], j));
          cpa8(pool + 2 * e, p.links + cb + e);
          cpa8(pool + 2 * e + 1, src + (uint32_t)(fco + p.poff[j]));
        }
      }
    } else if (RECORDS) {
      const int n = fl ? __popc(cw & kBounceMask) : 0;  // every cell of the chunk keeps its records
      const int off = warp_scan_excl(n, lane, &total);
      if (total) {
        double* pool = S.pool[s][warp];
        CLinkDesc* desc = reinterpret_cast<CLinkDesc*>(pool + kCPool);
        if (n) cpublish_links(desc, cw, (int32_t)E[14].rank + off, off, tx);
        __syncwarp();
        const int nl = min(total, kCLinkCap);
        for (int e = lane; e < nl; e += 32) {
          const CLinkDesc d = desc[e];
          const int j = d.oj & 31;
          bounds_ok(d.rec >= 0 && d.rec < p.nrec && in_plane(p, S.lane[s][d.oj >> 8].fc + p.poff[j], j));
          cpa8(pool + 2 * e, p.links + d.rec);
          cpa8(pool + 2 * e + 1, src + (uint32_t)(S.lane[s][d.oj >> 8].fc + p.poff[j]));
        }
      }
    }
    return total;
  };

  // link descriptors of plane z (meta slot m; its chunk bases have landed) as
  // 4-byte pairs from the even record at or below the chunk's first
  auto desc_load = [&](int m) {
    CMeta& M = S.meta[m];
    const int32_t cb = (int32_t)M.ent[warp][14].rank;
    const int n = min((int32_t)M.ent[warp][15].rank - cb, kCLinkCap);
    const int a0 = cb & ~1, npairs = (cb + n - a0 + 1) >> 1;
    for (int t = lane; t < npairs; t += 32) cpa4(&M.ldesc[warp][2 * t], p.linkdesc + a0 + 2 * t);
  };

  // prologue: meta of planes z0, z0+1; issue z0; meta of z0+2
  meta_load(z0, 0);
  if (z0 + 1 < z1) meta_load(z0 + 1, 1);
  cpa_commit();
  cpa_wait_all();
  __syncwarp();
  int cnt_cur;
  if (kStaticDesc) {
    // the descriptors (addressed by the chunk bases just landed) and the first
    // plane's populations go in flight together; the link extras follow once
    // the descriptors have landed
    desc_load(0);
    if (z0 + 1 < z1) desc_load(1);
    cpa_commit();
    pdl_wait();  // everything before read static data; populations come from the previous sweep
    issue(z0, 0, 0, 1);
    cpa_commit();
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // the descriptors (not the populations)
    __syncwarp();
    cnt_cur = issue(z0, 0, 0, 2);
  } else {
    pdl_wait();
    cnt_cur = issue(z0, 0, 0);
  }
  __syncwarp();
  if (z0 + 2 < z1) meta_load(z0 + 2, 2);
  cpa_commit();
  int ms = 0;  // meta slot of plane z
  for (int i = 0, z = z0; z < z1; ++i, ++z) {
    const int s = kS == 2 ? (i & 1) : 0;
    const int m1 = ms == 2 ? 0 : ms + 1;
    int cnt_next = 0;
    if (kS == 2) {
      if (z + 1 < z1) {
        cnt_next = issue(z + 1, s ^ 1, m1);
        __syncwarp();
        if (z + 3 < z1) meta_load(z + 3, ms);
      }
      cpa_commit();
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // plane z landed (this lane)
    } else {
      cpa_wait_all();
    }
    __syncwarp();  // ... and every lane's copies
    if (kStaticDesc && z + 2 < z1) desc_load(ms == 0 ? 2 : ms - 1);  // plane z+2's chunk bases landed
    const CLane li = S.lane[s][tx];
    // folded links: this lane's first record in the chunk-plane's list and the
    // list base (the epilogue runs after the stage is refilled with plane z+1)
    int foff = 0;
    int32_t fcb = 0;
    uint32_t fum = 0;  // the warp's union of bounce bits
    if (FOLD && cnt_cur) {  // warp-uniform
      int tot;
      const uint32_t lbm = (li.w & kNonFluid) ? 0u : (li.w & kBounceMask);
      foff = warp_scan_excl(__popc(lbm), lane, &tot);
      fum = __reduce_or_sync(0xffffffffu, lbm);
      fcb = S.cbase[s][warp];
    }
    const double* const fpool = S.pool[0][warp] + (z & 1) * kCLinkCap;
    if (FOLD && cnt_cur) {  // folded closures of plane z: f_j = c * (pull of k) + h
      double* const stage = &S.main[s][0][0];
      const int ncoop = min(cnt_cur, kCLinkCap);
      const uint16_t* ld = S.meta[ms].ldesc[warp] + (fcb & 1);
      for (int e = lane; e < ncoop; e += 32) {
        const int d = ld[e];
        const int owner = (tx & ~31) | (d & 31), j = d >> 5, k = opp_rt(j);
        close_fold(stage[j * kCBXp + owner], stage[k * kCBXp + owner], fpool[e], p, k);
      }
      if (cnt_cur > kCLinkCap && !(li.w & kNonFluid)) {  // pool overflow: own links past the cap
        uint32_t mm = li.w & kBounceMask;
        int i = foff;
        while (mm) {
          const int j = __ffs(mm) - 1;
          mm &= mm - 1;
          if (i >= kCLinkCap) {
            const int k = opp_rt(j);
            close_fold(stage[j * kCBXp + tx], stage[k * kCBXp + tx], __ldg(p.links + fcb + i), p, k);
          }
          ++i;
        }
      }
      __syncwarp();
    } else if (RECORDS && cnt_cur) {  // link closures of plane z (one-stage sweeps)
      double* const stage = &S.main[s][0][0];
      const double* pool = S.pool[s][warp];
      const int ncoop = min(cnt_cur, kCLinkCap);
      if (kStaticDesc) {
        const uint16_t* ld = S.meta[ms].ldesc[warp] + (S.cbase[s][warp] & 1);
        for (int e = lane; e < ncoop; e += 32) {
          const int d = ld[e];
          cclose_link(stage, (tx & ~31) | (d & 31), d >> 5, pool[2 * e], pool[2 * e + 1], p);
        }
      } else {
        const CLinkDesc* desc = reinterpret_cast<const CLinkDesc*>(pool + kCPool);
        for (int e = lane; e < ncoop; e += 32) {
          const CLinkDesc d = desc[e];
          cclose_link(stage, d.oj >> 8, d.oj & 31, pool[2 * e], pool[2 * e + 1], p);
        }
      }
      if (cnt_cur > kCLinkCap) {  // warp-uniform: pool overflow, each lane closes the rest itself
        const uint32_t w = li.w;
        const bool lf = !(w & kNonFluid);  // lanes past the row hold kNonFluid
        int tot;
        const int off = warp_scan_excl(lf ? __popc(w & kBounceMask) : 0, lane, &tot);
        uint32_t mm = lf ? (w & kBounceMask) : 0u;
        int k = 0;
        while (mm) {
          const int j = __ffs(mm) - 1;
          mm &= mm - 1;
          if (off + k >= kCLinkCap)
            cclose_link(stage, tx, j, __ldg(p.links + S.cbase[s][warp] + off + k),
                        __ldg(src + (uint32_t)(li.fc + p.poff[j])), p);
          ++k;
        }
      }
      __syncwarp();
    }
    const bool fluid = !(li.w & (kNonFluid | kInactive));
    double f[19];
    if (fluid) {
#pragma unroll
      for (int j = 0; j < 19; ++j) f[j] = S.main[s][j][tx];
    }
    if (kS == 1) {  // stage consumed: refill it with plane z+1
      __syncwarp();
      if (z + 1 < z1) {
        cnt_next = issue(z + 1, 0, m1);
        __syncwarp();
        if (z + 3 < z1) meta_load(z + 3, ms);
      }
      cpa_commit();
    }
    if (fluid) {
      if (OP == OP_STREAM_COLLIDE) {
        collide<CM, GLBM>(f, p, z);
        if (FOLD && cnt_cur) {
          if (cnt_cur <= kCLinkCap && !p.moving)
            fold_epilogue_pool(f, li.w & kBounceMask, fum, fpool, foff);
          else
            fold_epilogue(f, li.w & kBounceMask, p, [&](int i) {
              const int r = foff + i;
              return r < kCLinkCap ? fpool[r] : __ldg(p.links + fcb + r);
            });
        }
#pragma unroll
        for (int j = 0; j < 19; ++j) {
          bounds_ok(in_plane(p, li.fc + p.poff[j], j));
          if (PGPU_STCS && p.stream_stores)
            __stcs(dst + (uint32_t)(li.fc + p.poff[j]), f[j]);
          else
            dst[(uint32_t)(li.fc + p.poff[j])] = f[j];
        }
        write_sends<SLAB>(p, x, y, z, f);
      } else {  // KP: f(n) into the other compact buffer
#pragma unroll
        for (int j = 0; j < 19; ++j) dst[(uint32_t)(li.fc + p.poff[j])] = f[j];
      }
    }
    cnt_cur = cnt_next;
    ms = m1;
  }
  cpa_wait_all();
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
constexpr int kCBX = 128;
dim3 ccell_block(const KParams& p) { return dim3(p.nx < kCBX ? ((p.nx + 31) / 32) * 32 : kCBX); }
dim3 ccell_grid(const KParams& p) {
  const int bx = ccell_block(p).x;
  return dim3((p.nx + bx - 1) / bx, p.ny, p.nz);
}

int cpipe_zper(const KParams& p) {
  return zper_for((int64_t)((p.nchunk + kCW - 1) / kCW) * p.ny, p.nz);
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
void launch_compact_t(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                      cudaStream_t s) {
  // the pipelined kernel sweeps the slab edge bands when each band is one chunk
  if (cfg.part == PART_EDGES && (!edge_chunks(p) || g_plain_sweep())) {
    k_csweep_edges<CM, GLBM, RECORDS, SLAB, OP>
        <<<dim3(2, (p.ny * edge_band(p.nx) + 127) / 128, p.nz), 128, 0, s>>>(p, src, dst);
  } else if (g_plain_sweep()) {
    k_csweep_cells<CM, GLBM, RECORDS, SLAB, OP><<<ccell_grid(p), ccell_block(p), 0, s>>>(
        p, src, dst, cfg.part);
  } else {
    const int zper = cpipe_zper(p);
    const int zg = (p.nz + zper - 1) / zper;
    dim3 grid((p.nchunk + kCW - 1) / kCW, p.ny, zg);
    if (cfg.part == PART_EDGES) grid = dim3(1, (p.ny + kCW / 2 - 1) / (kCW / 2), zg);
    if (cfg.part == PART_INTERIOR && edge_chunks(p))
      grid = dim3((unsigned)(((int64_t)p.ny * (p.nchunk - 2) + kCW - 1) / kCW), 1, zg);
    if (grid.x == 0) return;
    constexpr int smem = (int)sizeof(CSmem<RECORDS, RECORDS && CM == CM_FAST_FOLD>) + PGPU_SMEM_PAD;  // pad: L1-capacity experiment
    static bool attr = [] {
      cudaFuncSetAttribute(k_sweep_cpipe<CM, GLBM, RECORDS, SLAB, OP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return true;
    }();
    (void)attr;
    // whole-domain sweeps launch as programmatic dependents of the previous
    // kernel (PGPU_PDL=0: off): their prologue overlaps its tail
    static const bool pdl_env = [] {
      const char* e = std::getenv("PGPU_PDL");
      return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kCBXp);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = (pdl_env && !SLAB && cfg.part == PART_ALL && OP == OP_STREAM_COLLIDE) ? 1 : 0;
    // CLI sweeps: the wall-adjacent planes' blocks (5 links per cell) first
    // (C3 +1.5 %; SBB sweeps gain nothing there and keep the plain order)
    static const int heavy_first = [] {
      const char* e = std::getenv("PGPU_HEAVYFIRST");
      return e ? (e[0] == '0' ? 0 : 2) : (RECORDS ? 2 : 0);
    }();
    cudaLaunchKernelEx(&lc, k_sweep_cpipe<CM, GLBM, RECORDS, SLAB, OP>, p, src, dst, cfg.part, zper,
                       (cfg.zrev ? 1 : 0) | heavy_first);
  }
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB>
void cdispatch_op(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  if (cfg.op == OP_STREAM_COLLIDE)
    launch_compact_t<CM, GLBM, RECORDS, SLAB, OP_STREAM_COLLIDE>(cfg, p, src, dst, s);
  else  // KP has no collision: one instantiation per records/slab (and link folding)
    launch_compact_t<(CM == CM_FAST_FOLD && RECORDS) ? CM_FAST_FOLD : CM_EXACT_RHO1, false, RECORDS, SLAB,
                     OP_STREAM_ONLY>(cfg, p, src, dst, s);
}
template <int CM, bool GLBM>
void cdispatch(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
               cudaStream_t s) {
  if (cfg.records) {
    if (cfg.slab) cdispatch_op<CM, GLBM, true, true>(cfg, p, src, dst, s);
    else cdispatch_op<CM, GLBM, true, false>(cfg, p, src, dst, s);
  } else {
    if (cfg.slab) cdispatch_op<CM, GLBM, false, true>(cfg, p, src, dst, s);
    else cdispatch_op<CM, GLBM, false, false>(cfg, p, src, dst, s);
  }
}
template <int CM>
void cdispatch_cm(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  if (cfg.glbm) cdispatch<CM, true>(cfg, p, src, dst, s);
  else cdispatch<CM, false>(cfg, p, src, dst, s);
}

template <int CM, bool FOLD>
void collide_compact_cm(bool glbm, bool slab, const KParams& p, double* buf, cudaStream_t s) {
  const dim3 g = ccell_grid(p), b = ccell_block(p);
  if (glbm) {
    if (slab) k_collide_compact<CM, true, true, FOLD><<<g, b, 0, s>>>(p, buf);
    else k_collide_compact<CM, true, false, FOLD><<<g, b, 0, s>>>(p, buf);
  } else {
    if (slab) k_collide_compact<CM, false, true, FOLD><<<g, b, 0, s>>>(p, buf);
    else k_collide_compact<CM, false, false, FOLD><<<g, b, 0, s>>>(p, buf);
  }
}

}  // namespace

void launch_sweep_compact(const SweepConfig& cfg, const KParams& p, const double* src,
                          double* dst, cudaStream_t s) {
  if (p.sweep == 2 && tma_sweep_supported(cfg, p) && launch_sweep_tma(cfg, p, src, dst, s)) return;
  if ((p.sweep == 3 || p.sweep == 0) && units_sweep_supported(cfg, p) &&
      launch_sweep_units(cfg, p, src, dst, s))
    return;
  switch (collide_mode(p)) {
    case CM_FAST: cdispatch_cm<CM_FAST>(cfg, p, src, dst, s); break;
    case CM_FAST_FOLD: cdispatch_cm<CM_FAST_FOLD>(cfg, p, src, dst, s); break;
    case CM_EXACT_RHO1: cdispatch_cm<CM_EXACT_RHO1>(cfg, p, src, dst, s); break;
    default: cdispatch_cm<CM_EXACT>(cfg, p, src, dst, s);
  }
}

void launch_collide_compact(bool glbm, bool slab, bool records, const KParams& p, double* buf,
                            cudaStream_t s) {
  switch (collide_mode(p)) {
    case CM_FAST: collide_compact_cm<CM_FAST, false>(glbm, slab, p, buf, s); break;
    case CM_FAST_FOLD:
      if (records) collide_compact_cm<CM_FAST_FOLD, true>(glbm, slab, p, buf, s);
      else collide_compact_cm<CM_FAST, false>(glbm, slab, p, buf, s);
      break;
    case CM_EXACT_RHO1: collide_compact_cm<CM_EXACT_RHO1, false>(glbm, slab, p, buf, s); break;
    default: collide_compact_cm<CM_EXACT, false>(glbm, slab, p, buf, s);
  }
}

void launch_compact_io(bool expand, const KParams& p, double* f, double* dense, int z0, int nzc,
                       cudaStream_t s) {
  const int64_t n = (int64_t)nzc * p.ny * p.nx;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (expand) k_compact_io<true><<<blocks, 256, 0, s>>>(p, f, dense, z0, nzc);
  else k_compact_io<false><<<blocks, 256, 0, s>>>(p, f, dense, z0, nzc);
}

void launch_fill_compact(const KParams& p, int64_t nfluid, double* f, const double* feq,
                         cudaStream_t s) {
  if (nfluid == 0) return;
  k_fill_compact<<<(unsigned)((nfluid + 255) / 256), 256, 0, s>>>(p, nfluid, f, feq);
}

// z-planes per block: long marching columns (the per-block prologue is paid
// once per column), but >= ~6.5 waves of blocks over 148 SMs x 4 resident
// blocks, so the last wave -- the launch's tail -- is a small part of it.
// Measured on one B200 (per_config): C2 zper 2/3/4 = 0.757/0.744/0.729, C5
// (dense) 2/4/6 = 0.843/0.852/0.834, C4 4/8 = 0.786/0.799 (capped at 8).
int zper_for(int64_t cols, int nz) {
  if (const char* e = std::getenv("PGPU_ZPER")) return std::max(1, std::min(atoi(e), nz));
  static const int64_t waves2 = [] {  // twice the target wave count
    const char* e = std::getenv("PGPU_ZWAVES2");
    return (int64_t)(e ? std::max(1, atoi(e)) : 13);
  }();
  const int zper = (int)std::min<int64_t>(8, std::max<int64_t>(1, 2 * cols * nz / (148 * 4 * waves2)));
  return std::min(zper, nz);
}
}  // namespace pgpu
