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
//   K1  k_sweep_bulk         : g' = C(P(g))  compact -> compact (the hot kernel)
//   KP  k_sweep_bulk<KP>     : f = P(g)   compact -> dense (observables)
// with P the pull form of the reference's push streaming + link bounce-back
// (simulation.cpp:278-342, boundary.cpp:19-41), exactly as in
// kernels.cu.
//
// K1 is warp-centric.  A warp owns one 32-cell chunk of a row and marches
// through z-planes.  For the chunk, the pull sources of each direction j lie
// in ONE of 9 neighbouring rows (source row (y - e_jy, z - e_jz)) and, for the
// fluid sources, form a contiguous run of compact slots: cells x0-1 .. x0+32
// of that row.  So the warp fetches each direction with one bulk copy
// (cp.async.bulk, TMA engine, completion on a per-stage mbarrier) of at most
// 36 doubles into shared memory, one plane ahead, and every lane finds its
// value at
//     q_r = (rank_r - lo_r) + popc(mask_r & lanemask_lt)
// (ex = 0: q_r, ex = +1: q_r - 1, ex = -1: q_r + bit(mask_r, lane); the
// source is fluid whenever it is pulled, which is what makes the +-1 exact
// even across chunk boundaries).  What does not come from a run -- bounce
// sources g_k(x), CLI records and g_j(x), the periodic x wrap, slab ghosts --
// goes through a per-warp list of 8-byte asynchronous copies issued
// round-robin by the 32 lanes.  No per-lane address arithmetic for the 19
// regular pulls, no in-flight bytes in registers.
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
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Bulk global -> shared copy (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Compact index helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t fidx(const KParams& p, int x, int y, int z) {
  const ChunkEnt e = p.ctab[((int64_t)z * p.ny + y) * p.nchunk + (x >> 5)];
  return (int64_t)e.rank + __popc(e.mask & ((1u << (x & 31)) - 1u));
}

// Directions with e_x = +1 / -1 (their x = 0 / x = nx-1 pulls wrap).
constexpr uint32_t kExPlus = (1u << 1) | (1u << 7) | (1u << 9) | (1u << 11) | (1u << 13);
constexpr uint32_t kExMinus = (1u << 2) | (1u << 8) | (1u << 10) | (1u << 12) | (1u << 14);

// Source rows: row r holds the directions with (e_y, e_z) = kRowE[r]; their
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
__host__ __device__ constexpr int row_ndirs(int r) { return r < 5 ? 3 : 1; }
__host__ __device__ constexpr int row_dir(int r, int i) {
  return r == 0 ? i
         : r == 1 ? (i == 0 ? 3 : (i == 1 ? 7 : 10))
         : r == 2 ? (i == 0 ? 4 : (i == 1 ? 8 : 9))
         : r == 3 ? (i == 0 ? 5 : (i == 1 ? 11 : 14))
         : r == 4 ? (i == 0 ? 6 : (i == 1 ? 12 : 13))
                  : r + 10;
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
// the reference point for the bulk kernel): same arithmetic as kernels.cu's
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

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__device__ __forceinline__ void csweep_cell(const KParams& p, const double* __restrict__ src,
                                            double* __restrict__ dst, int x, int y, int z) {
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = __ldg(p.cellw + c);
  if (w & kNonFluid) return;
  const int64_t fc = fidx(p, x, y, z);
  double f[19];
  cload_all<0, SLAB>(f, src, x, y, z, fc, p, w);
  if (RECORDS && (w & kBounceMask)) clinks_all<1>(f, src, fc, p, w, __ldg(p.cellbase + c));
  if (OP == OP_STREAM_COLLIDE) {
    if (GLBM)
      collide_glbm<RHO1>(f, p, z);
    else
      collide_core<RHO1>(f, p);
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcs(dst + (int64_t)j * p.ks + fc, f[j]);
    write_sends<SLAB>(p, x, y, z, f);
  } else {  // KP: dense observable buffer
#pragma unroll
    for (int j = 0; j < 19; ++j) dst[(int64_t)j * p.ksd + c] = f[j];
  }
}

// One thread per cell of the box (part ALL / INTERIOR) ...
template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_csweep_cells(const KParams p,
                                                      const double* __restrict__ src,
                                                      double* __restrict__ dst, int part) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= p.nx) return;
  if (part == PART_INTERIOR && in_edge_band(x, p.nx)) return;
  csweep_cell<RHO1, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, blockIdx.y, blockIdx.z);
}
// ... or of the two x edge bands (slab split; grid (2, ceil(ny/4), nz)).
template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_csweep_edges(const KParams p,
                                                      const double* __restrict__ src,
                                                      double* __restrict__ dst) {
  const int w = edge_band(p.nx);
  const int xx = threadIdx.x & 31;
  const int y = blockIdx.y * 4 + (threadIdx.x >> 5);
  const int z = blockIdx.z;
  if (xx >= w || y >= p.ny) return;
  const int x = blockIdx.x ? p.nx - w + xx : xx;
  if (blockIdx.x && x < w) return;
  csweep_cell<RHO1, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z);
}

// K0: dense pre-collision f -> compact post-collision g (simulation.cpp:150-274).
template <bool RHO1, bool GLBM, bool SLAB>
__global__ void __launch_bounds__(128) k_collide_to_compact(const KParams p,
                                                            const double* __restrict__ f0,
                                                            double* __restrict__ dst) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  if (__ldg(p.cellw + c) & kNonFluid) return;
  double f[19];
#pragma unroll
  for (int j = 0; j < 19; ++j) f[j] = __ldg(f0 + (int64_t)j * p.ksd + c);
  if (GLBM)
    collide_glbm<RHO1>(f, p, z);
  else
    collide_core<RHO1>(f, p);
  const int64_t fc = fidx(p, x, y, z);
#pragma unroll
  for (int j = 0; j < 19; ++j) dst[(int64_t)j * p.ks + fc] = f[j];
  write_sends<SLAB>(p, x, y, z, f);
}

// ---------------------------------------------------------------------------
// K1 / KP bulk sweep
// ---------------------------------------------------------------------------
constexpr int kBW = 4;     // warps (chunks) per block
constexpr int kSpan = 36;  // doubles per direction and stage: cells x0-1..x0+32 + alignment
__host__ __device__ constexpr int bulk_pool(bool records) { return records ? 96 : 64; }
#ifndef PGPU_BULK_MINB
#define PGPU_BULK_MINB 4
#endif

struct RowInfo {
  int32_t rel;    // stage slot of the chunk's first cell (rank - lo)
  uint32_t mask;  // fluid mask of the source row's chunk
};
struct LaneInfo {
  uint32_t w;     // bounce bits, or kNonFluid for lanes that skip the plane
  uint16_t ext;   // first extras slot of the lane
  uint16_t rec;   // link records of the warp's lanes before this one
};
template <int P>
struct alignas(16) WarpStage {
  double main[19][kSpan];
  double pool[P];  // extras: 8-byte copies (first the source addresses, then the values)
  RowInfo rows[9];
  ChunkEnt part[5];  // x-wrap partner chunk of rows 0..4
  int32_t rank00;    // compact slot of the chunk's first cell (own row)
  int32_t recbase;   // first link record of the chunk
  int32_t pad[2];
  LaneInfo lane[32];
};
struct alignas(16) WarpMeta {  // cell words and chunk entries of one plane, loaded ahead
  uint32_t cw[32];
  ChunkEnt ent[16];  // 0..8 source rows, 9..13 x-wrap partners of rows 0..4, 14.rank = chunk base
};
template <int P>
struct alignas(16) WarpSmem {
  WarpStage<P> st[2];
  WarpMeta meta[2];
  uint64_t bar[2];
};
template <bool RECORDS>
constexpr int bulk_smem() {
  return kBW * (int)sizeof(WarpSmem<bulk_pool(RECORDS)>);
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

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(kBW * 32, PGPU_BULK_MINB)
    k_sweep_bulk(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                 int part, int zper) {
  constexpr int P = bulk_pool(RECORDS);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem<P>& S = reinterpret_cast<WarpSmem<P>*>(smem_raw)[warp];
  const int xc = blockIdx.x * kBW + warp;
  if (xc >= p.nchunk) return;  // whole warp; no block-level synchronisation below
  const int y = blockIdx.y;
  const int z0 = blockIdx.z * zper, z1 = min(z0 + zper, p.nz);
  const int x0 = xc << 5, x = x0 + lane;
  const bool valid = x < p.nx;
  const bool active = valid && !(part == PART_INTERIOR && in_edge_band(x, p.nx));
  if (!__any_sync(0xffffffffu, active)) return;
  const uint32_t ltl = (1u << lane) - 1u;
  const bool wrapchunk = (xc == 0 || xc == p.nchunk - 1);

  if (lane == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_fence_init();
  }
  __syncwarp();

  // cell words and source-row chunk entries of plane z into meta slot m
  auto meta_load = [&](int z, int m) {
    WarpMeta& M = S.meta[m];
    const int64_t row = (int64_t)z * p.ny + y;
    if (valid)
      cpa4(&M.cw[lane], p.cellw + row * p.nx + x);
    else
      M.cw[lane] = kNonFluid;
    if (lane < 14) {
      const int r = lane < 9 ? lane : lane - 9;
      int ys = y - row_ey(r), zs = z - row_ez(r);
      const bool ok = wrap_coord(ys, p.ny, p.py) & wrap_coord(zs, p.nz, p.pz);
      const int cx = lane < 9 ? xc : (xc == 0 ? p.nchunk - 1 : 0);
      if (ok && (lane < 9 || (!SLAB && wrapchunk)))
        cpa8(&M.ent[lane], p.ctab + ((int64_t)zs * p.ny + ys) * p.nchunk + cx);
      else
        M.ent[lane] = ChunkEnt{0u, 0u};
    } else if (lane == 14 && RECORDS) {
      cpa4(&M.ent[14].rank, p.chunkbase + row * p.nchunk + xc);
    }
  };

  // plane z (meta slot m) into stage s: bulk copies of the 19 source runs,
  // extras list, per-lane info
  auto issue = [&](int z, int s, int m) {
    WarpStage<P>& T = S.st[s];
    const WarpMeta& M = S.meta[m];
    uint32_t bytes = 0;
    int lo = 0, nel = 0;
    if (lane < 9) {
      const ChunkEnt e = M.ent[lane];
      int first = (int)e.rank - (x0 > 0 ? 1 : 0);
      if (first < 0) first = 0;
      const int last = (int)e.rank + __popc(e.mask) + (x0 + 32 < p.nx ? 1 : 0);
      lo = first & ~1;
      nel = ((last + 1) & ~1) - lo;
      T.rows[lane] = RowInfo{(int)e.rank - lo, e.mask};
      bytes = (uint32_t)nel * 8u * (lane < 5 ? 3u : 1u);
    } else if (lane < 14) {
      T.part[lane - 9] = M.ent[lane];
    } else if (lane == 14) {
      T.rank00 = (int32_t)M.ent[0].rank;
      T.recbase = RECORDS ? (int32_t)M.ent[14].rank : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    // extras: bounce sources (+ CLI record and g_j(x)), x-wrap / ghost pulls
    const uint32_t cw = M.cw[lane];
    const bool fl = !(cw & kNonFluid);  // lanes past the row hold kNonFluid
    const uint32_t bb = fl ? (cw & kBounceMask) : 0u;
    uint32_t wr = 0;
    if (fl && active) {
      if (x == 0) wr |= kExPlus & ~bb;
      if (x == p.nx - 1) wr |= kExMinus & ~bb;
    }
    const int nb = __popc(bb);
    const int ne = (fl && active) ? nb * (RECORDS ? 3 : 1) + __popc(wr) : 0;
    int tot;
    const int pre = warp_scan_excl(nb | (ne << 16), lane, &tot);
    const int orec = pre & 0xFFFF, oext = pre >> 16, text = tot >> 16;
    T.lane[lane] = LaneInfo{(fl && active) ? bb : kNonFluid, (uint16_t)oext, (uint16_t)orec};
    if (ne) {
      const ChunkEnt e0 = M.ent[0];
      const int64_t fc = (int64_t)e0.rank + __popc(e0.mask & ltl);
      const int32_t rb = RECORDS ? (int32_t)M.ent[14].rank + orec : 0;
      int slot = oext, ib = 0;
      auto put = [&](const void* a) {
        if (slot < P) T.pool[slot] = __longlong_as_double((long long)(uintptr_t)a);
        ++slot;
      };
      uint32_t mm = bb | wr;
      while (mm) {
        const int j = __ffs(mm) - 1;
        mm &= mm - 1;
        if ((bb >> j) & 1u) {
          put(src + (int64_t)opp(j) * p.ks + fc);  // g_k(x)
          if (RECORDS) {
            put(p.links + rb + ib);               // record
            put(src + (int64_t)j * p.ks + fc);    // g_j(x)
          }
          ++ib;
        } else {
          put(wrap_src<SLAB>(p, src, M.ent[9 + row_of(j)], j, x, y, z));
        }
      }
    }
    __syncwarp();
    const int nis = min(text, P);
    for (int e = lane; e < nis; e += 32) {
      const double* a = reinterpret_cast<const double*>(
          (uintptr_t)__double_as_longlong(T.pool[e]));
      cpa8(&T.pool[e], a);
    }
    if (lane == 0) mbar_arrive_expect_tx(&S.bar[s], bytes);
    __syncwarp();
    if (lane < 9 && nel > 0) {
      fence_proxy_async();
      const uint32_t nb8 = (uint32_t)nel * 8u;
      const double* base = src + lo;
      if (lane < 5) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int j = row_dir(lane, i);
          bulk_g2s(&T.main[j][0], base + (int64_t)j * p.ks, nb8, &S.bar[s]);
        }
      } else {
        const int j = lane + 10;
        bulk_g2s(&T.main[j][0], base + (int64_t)j * p.ks, nb8, &S.bar[s]);
      }
    }
  };

  // prologue: meta of the first two planes, issue of the first
  meta_load(z0, 0);
  if (z0 + 1 < z1) meta_load(z0 + 1, 1);
  cpa_commit();
  cpa_wait_all();
  __syncwarp();
  issue(z0, 0, 0);
  __syncwarp();
  if (z0 + 2 < z1) meta_load(z0 + 2, 0);
  cpa_commit();

  uint32_t phase = 0;
  for (int i = 0, z = z0; z < z1; ++i, ++z) {
    const int s = i & 1;
    cpa_wait_all();  // extras of plane z, meta of plane z+1 (this lane's copies)
    __syncwarp();    // ... and every other lane's
    if (z + 1 < z1) {
      issue(z + 1, s ^ 1, (i + 1) & 1);
      __syncwarp();  // meta slot (i+1)&1 consumed
      if (z + 3 < z1) meta_load(z + 3, (i + 1) & 1);
    }
    cpa_commit();
    mbar_wait(&S.bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;

    const WarpStage<P>& T = S.st[s];
    const LaneInfo li = T.lane[lane];
    if (!(li.w & kNonFluid)) {
      double f[19];
      int q[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const RowInfo ri = T.rows[r];
        q[r] = ri.rel + __popc(ri.mask & ltl);
      }
      const uint32_t own1 = 1u << lane;
#pragma unroll
      for (int j = 0; j < 19; ++j) {
        const int r = row_of(j);
        int sl = q[r];
        if (EX[j] == 1) sl -= 1;
        if (EX[j] == -1) sl += (T.rows[r].mask & own1) ? 1 : 0;
        f[j] = T.main[j][sl];
      }
      const uint32_t bb = li.w & kBounceMask;
      uint32_t wr = 0;
      if (x == 0) wr |= kExPlus & ~bb;
      if (x == p.nx - 1) wr |= kExMinus & ~bb;
      const int64_t fc = (int64_t)T.rank00 + __popc(T.rows[0].mask & ltl);
      if (bb | wr) {
        int pos = li.ext;
#pragma unroll
        for (int j = 1; j < 19; ++j) {
          if ((bb >> j) & 1u) {
            f[j] = pos < P ? T.pool[pos] : __ldg(src + (int64_t)opp(j) * p.ks + fc);
            pos += RECORDS ? 3 : 1;
          } else if ((wr >> j) & 1u) {
            f[j] = pos < P ? T.pool[pos]
                           : __ldg(wrap_src<SLAB>(p, src, T.part[row_of(j)], j, x, y, z));
            pos += 1;
          }
        }
        if (RECORDS && bb) {
          pos = li.ext;
          int ib = 0;
#pragma unroll
          for (int j = 1; j < 19; ++j) {
            if ((bb >> j) & 1u) {
              const int K = opp(j);
              const double rec =
                  pos + 1 < P ? T.pool[pos + 1] : __ldg(p.links + T.recbase + li.rec + ib);
              const double gj = pos + 2 < P ? T.pool[pos + 2] : __ldg(src + (int64_t)j * p.ks + fc);
              if (rec == rec) {  // CLI (boundary.cpp:24-32) or moving wall (:34-41)
                if (!isinf(rec))
                  f[j] = DADD(DSUB(DMUL(rec, f[K]), DMUL(rec, gj)), f[j]);
                else
                  f[j] = DSUB(f[j], p.mw[K]);
              }  // NaN: simple bounce-back
              pos += 3;
              ++ib;
            } else if ((wr >> j) & 1u) {
              pos += 1;
            }
          }
        }
      }
      if (OP == OP_STREAM_COLLIDE) {
        if (GLBM)
          collide_glbm<RHO1>(f, p, z);
        else
          collide_core<RHO1>(f, p);
        double* const d = dst + fc;
#pragma unroll
        for (int j = 0; j < 19; ++j) __stcs(d + (int64_t)j * p.ks, f[j]);
        write_sends<SLAB>(p, x, y, z, f);
      } else {  // KP into the dense observable buffer
        double* const d = dst + ((int64_t)z * p.ny + y) * p.nx + x;
#pragma unroll
        for (int j = 0; j < 19; ++j) d[(int64_t)j * p.ksd] = f[j];
      }
    }
  }
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

// z-planes per warp: long marching columns, but >= ~4 waves of blocks over
// 148 SMs x 4 resident blocks.
int bulk_zper(const KParams& p) {
  if (const char* e = std::getenv("PGPU_ZPER")) return std::max(1, std::min(atoi(e), p.nz));
  const int64_t cols = (int64_t)((p.nchunk + kBW - 1) / kBW) * p.ny;
  const int zper = (int)std::min<int64_t>(8, std::max<int64_t>(1, cols * p.nz / (148 * 4 * 4)));
  return std::min(zper, p.nz);
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB, int OP>
void launch_compact_t(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                      cudaStream_t s) {
  if (cfg.part == PART_EDGES) {
    k_csweep_edges<RHO1, GLBM, RECORDS, SLAB, OP>
        <<<dim3(2, (p.ny + 3) / 4, p.nz), 128, 0, s>>>(p, src, dst);
  } else if (g_plain_sweep()) {
    k_csweep_cells<RHO1, GLBM, RECORDS, SLAB, OP><<<ccell_grid(p), ccell_block(p), 0, s>>>(
        p, src, dst, cfg.part);
  } else {
    const int zper = bulk_zper(p);
    const dim3 grid((p.nchunk + kBW - 1) / kBW, p.ny, (p.nz + zper - 1) / zper);
    constexpr int smem = bulk_smem<RECORDS>();
    static bool attr = [] {
      cudaFuncSetAttribute(k_sweep_bulk<RHO1, GLBM, RECORDS, SLAB, OP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return true;
    }();
    (void)attr;
    k_sweep_bulk<RHO1, GLBM, RECORDS, SLAB, OP><<<grid, kBW * 32, smem, s>>>(p, src, dst,
                                                                           cfg.part, zper);
  }
}

template <bool RHO1, bool GLBM, bool RECORDS, bool SLAB>
void cdispatch_op(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  if (cfg.op == OP_STREAM_COLLIDE)
    launch_compact_t<RHO1, GLBM, RECORDS, SLAB, OP_STREAM_COLLIDE>(cfg, p, src, dst, s);
  else  // KP has no collision: one instantiation per records/slab
    launch_compact_t<true, false, RECORDS, SLAB, OP_STREAM_ONLY>(cfg, p, src, dst, s);
}
template <bool RHO1, bool GLBM>
void cdispatch(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
               cudaStream_t s) {
  if (cfg.records) {
    if (cfg.slab) cdispatch_op<RHO1, GLBM, true, true>(cfg, p, src, dst, s);
    else cdispatch_op<RHO1, GLBM, true, false>(cfg, p, src, dst, s);
  } else {
    if (cfg.slab) cdispatch_op<RHO1, GLBM, false, true>(cfg, p, src, dst, s);
    else cdispatch_op<RHO1, GLBM, false, false>(cfg, p, src, dst, s);
  }
}

}  // namespace

void launch_sweep_compact(const SweepConfig& cfg, const KParams& p, const double* src,
                          double* dst, cudaStream_t s) {
  const bool rho1 = p.rho0 == 1.0;
  if (rho1) {
    if (cfg.glbm) cdispatch<true, true>(cfg, p, src, dst, s);
    else cdispatch<true, false>(cfg, p, src, dst, s);
  } else {
    if (cfg.glbm) cdispatch<false, true>(cfg, p, src, dst, s);
    else cdispatch<false, false>(cfg, p, src, dst, s);
  }
}

void launch_collide_to_compact(bool glbm, bool slab, const KParams& p, const double* dense,
                               double* dst, cudaStream_t s) {
  const dim3 g = ccell_grid(p), b = ccell_block(p);
  const bool rho1 = p.rho0 == 1.0;
#define PGPU_K0C(R, G, S) k_collide_to_compact<R, G, S><<<g, b, 0, s>>>(p, dense, dst)
  if (rho1) {
    if (glbm) { if (slab) PGPU_K0C(true, true, true); else PGPU_K0C(true, true, false); }
    else { if (slab) PGPU_K0C(true, false, true); else PGPU_K0C(true, false, false); }
  } else {
    if (glbm) { if (slab) PGPU_K0C(false, true, true); else PGPU_K0C(false, true, false); }
    else { if (slab) PGPU_K0C(false, false, true); else PGPU_K0C(false, false, false); }
  }
#undef PGPU_K0C
}

}  // namespace pgpu
