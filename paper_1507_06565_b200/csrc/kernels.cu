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
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "kparams.h"
#include "lattice.cuh"

namespace pgpu {
namespace cg = cooperative_groups;


// ---------------------------------------------------------------------------
// Pull-form streaming + bounce-back: for fluid x and direction
// j with fluid upstream s = x - e_j:  f_j(x) = g_j(s).  Otherwise the link
// (x, k = opp j) closes it (boundary.cpp:19-41 written for the receiving slot):
//   SBB    f_j(x) = g_k(x)
//   CLI    f_j(x) = c*g_k(x - e_k) - c*g_j(x) + g_k(x),  c = (1-2q)/(1+2q)
//   moving f_j(x) = g_k(x) - 2 w_k rho0 3 (e_k . u_w)
// g_k(x - e_k) is exactly the pull value of direction k at x, and g_k(x) of
// a bounce direction is read by nobody else, so every post-collision value is
// read exactly once per sweep: one load per direction, its address selected by
// the cell's bounce bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
// L2-coherent load for state written earlier in the same (persistent) kernel.
template <bool COHERENT>
__device__ __forceinline__ double ldstate(const double* p) {
  if constexpr (COHERENT) return __ldcg(p);
  else return __ldg(p);
}

template <int J, bool SLAB>
__device__ __forceinline__ const double* pull_addr(const double* __restrict__ src, int x, int y,
                                                   int z, int64_t c, const KParams& p,
                                                   uint32_t w) {
  constexpr int ex = EX[J], ey = EY[J], ez = EZ[J];
  if (J != 0 && ((w >> J) & 1u)) return src + (int64_t)opp(J) * p.ks + c;  // bounce: g_k(x)
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
  return src + (int64_t)J * p.ks + ((int64_t)zs * p.ny + ys) * p.nx + xs;
}

template <int J, bool SLAB, bool COHERENT = false>
__device__ __forceinline__ void load_all(double (&f)[19], const double* __restrict__ src, int x,
                                         int y, int z, int64_t c, const KParams& p, uint32_t w) {
  if constexpr (J < 19) {
    f[J] = ldstate<COHERENT>(pull_addr<J, SLAB>(src, x, y, z, c, p, w));
    load_all<J + 1, SLAB, COHERENT>(f, src, x, y, z, c, p, w);
  }
}

// Second phase for CLI / moving-wall links: f[J] already holds g_k(x).
template <int J, bool COHERENT = false>
__device__ __forceinline__ void links_all(double (&f)[19], const double* __restrict__ src,
                                          int64_t c, const KParams& p, uint32_t w, int32_t base) {
  if constexpr (J < 19) {
    if ((w >> J) & 1u) {
      constexpr int K = opp(J);
      const int32_t r = base + __popc(w & ((1u << J) - 1u) & kBounceMask);
      const double rec = __ldg(p.links + r);
      const double gj = ldstate<COHERENT>(src + (int64_t)J * p.ks + c);  // g_kb(x_f1), boundary.cpp:29-31
      if (rec == rec) {
        if (!isinf(rec)) {  // CLI, boundary.cpp:24-32: ((c*a) - (c*b)) + d
          f[J] = DADD(DSUB(DMUL(rec, f[K]), DMUL(rec, gj)), f[J]);
        } else {  // moving wall, boundary.cpp:34-41
          f[J] = DSUB(f[J], p.mw[K]);
        }
      }  // NaN: simple bounce-back, f[J] = g_k(x) already
    }
    links_all<J + 1, COHERENT>(f, src, c, p, w, base);
  }
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP, bool COHERENT = false>
__device__ __forceinline__ void sweep_cell(const KParams& p, const double* __restrict__ src,
                                           double* __restrict__ dst, int x, int y, int z,
                                           CellWord cw) {
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = cw.w;
  if (w & kNonFluid) {  // solid / wall: never read; optionally completes a sector
    if (w & kFillSector) {
#pragma unroll
      for (int j = 0; j < 19; ++j) __stcs(dst + (int64_t)j * p.ks + c, 0.0);
    }
    return;
  }
  double f[19];
  load_all<0, SLAB, COHERENT>(f, src, x, y, z, c, p, w);
  if (RECORDS && (w & kBounceMask)) links_all<1, COHERENT>(f, src, c, p, w, cw.base);
  if (OP == OP_STREAM_COLLIDE) collide<CM, GLBM>(f, p, z);
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

// Cell word and the cell's first link record (per-cell kernels).
__device__ __forceinline__ CellWord ld_cw(const KParams& p, int64_t c) {
  return CellWord{__ldg(p.cellw + c), __ldg(p.cellbase + c)};
}

// Each block sweeps kZPer consecutive z-planes of one (x-segment, y) column;
// the next cell word is prefetched while the current cell is processed.
constexpr int kZPer = 4;
#ifndef PGPU_SWEEP_MINB
#define PGPU_SWEEP_MINB 5
#endif

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128, PGPU_SWEEP_MINB) k_sweep(const KParams p, const double* __restrict__ src,
                                               double* __restrict__ dst, int part) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int z0 = blockIdx.z * kZPer;
  if (x >= p.nx) return;
  if (part == PART_INTERIOR && in_edge_band(x, p.nx)) return;
  const int z1 = min(z0 + kZPer, p.nz);
  CellWord next = ld_cw(p, ((int64_t)z0 * p.ny + y) * p.nx + x);
  for (int z = z0; z < z1; ++z) {
    const CellWord cw = next;
    if (z + 1 < z1) next = ld_cw(p, ((int64_t)(z + 1) * p.ny + y) * p.nx + x);
    sweep_cell<CM, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z, cw);
  }
}

// Asynchronous-copy pipeline helpers (k_sweep_pipe).
constexpr int kPipeBX = 128;
// Pipeline depth per variant (measured on C4, round 1): SBB sweeps keep two
// shared-memory stages at 4 blocks/SM; sweeps with link records (CLI /
// moving walls) use one stage (the landed plane is moved to registers and the
// stage refilled) at 5 blocks/SM, which leaves L1 room for the pooled extras.
#ifndef PGPU_DENSE_SBB_STAGES
#define PGPU_DENSE_SBB_STAGES 2
#endif
#ifndef PGPU_DENSE_SBB_MINB
#define PGPU_DENSE_SBB_MINB 4
#endif
__host__ __device__ constexpr int pipe_stages(bool records) {
  return records ? 1 : PGPU_DENSE_SBB_STAGES;
}
__host__ __device__ constexpr int pipe_minb(bool records) { return records ? 5 : PGPU_DENSE_SBB_MINB; }
#ifndef PGPU_POOL
#define PGPU_POOL 192
#endif
#ifndef PGPU_CW_EARLY
#define PGPU_CW_EARLY 0
#endif
#ifndef PGPU_CW_LATE2
#define PGPU_CW_LATE2 0
#endif
constexpr int kPool = PGPU_POOL;  // per-warp, per-stage slots for CLI / moving-wall extras
constexpr int kLinkCap = kPool / 2;  // link entries per warp and stage (2 pool slots each)
// per stage: 19 population slots per thread + per warp (pool + descriptors)
__host__ __device__ constexpr int pipe_smem(bool records) {
  return pipe_stages(records) *
         (19 * kPipeBX + (records ? (kPipeBX / 32) * (kPool + kLinkCap) : 0)) *
         (int)sizeof(double);
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int J, bool SLAB>
__device__ __forceinline__ void issue_all(double* stage, const double* __restrict__ src, int x,
                                          int y, int z, int64_t c, const KParams& p,
                                          uint32_t w) {
  if constexpr (J < 19) {
    cp_async8(stage + J * kPipeBX, pull_addr<J, SLAB>(src, x, y, z, c, p, w));
    issue_all<J + 1, SLAB>(stage, src, x, y, z, c, p, w);
  }
}

// Cells off every periodic wrap face: source = cell + constant offset, the
// offset picked by the bounce bit (host-precomputed, KParams).
template <int J>
__device__ __forceinline__ void issue_fast(double* stage, const double* cellp,
                                           const KParams& p, uint32_t w) {
  if constexpr (J < 19) {
    const double* a = cellp + p.pull_off[J];
#ifndef PGPU_EXPERIMENT_NOBOUNCE  // traffic-attribution experiment only (wrong results)
    if (J != 0 && ((w >> J) & 1u)) a += p.bounce_delta[J];
#endif
    cp_async8(stage + J * kPipeBX, a);
    issue_fast<J + 1>(stage, cellp, p, w);
  }
}

// Warp-exclusive prefix sum of n; returns the warp total in *total.
__device__ __forceinline__ int warp_excl_scan(int n, int lane, int* total) {
  int v = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  *total = __shfl_sync(0xffffffffu, v, 31);
  return v - n;
}

// Special registers read through volatile asm: values recomputed at their use
// instead of being kept live (and spilled) across the z loop.
__device__ __forceinline__ int v_tid_x() {
  int r;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ int v_ctaid_x() {
  int r;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ int v_ctaid_y() {
  int r;
  asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(r));
  return r;
}
__device__ __forceinline__ int v_ctaid_z() {
  int r;
  asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(r));
  return r;
}

// Warp-cooperative link handling.  A warp's bounce links of one plane form a
// list (entry e = owner lane's i-th bounce direction, ordered by a warp
// prefix sum).  Owners publish a descriptor per entry {record index,
// owner thread << 8 | j}; then all 32 lanes issue the record / g_j(x) copies
// and later apply the closures round-robin over the list, so a warp iterates
// ceil(links / 32) times instead of as often as its busiest lane.
struct LinkDesc {
  int32_t rec;  // index into p.links
  int32_t oj;   // owner thread << 8 | j
};

__device__ __forceinline__ void publish_links(LinkDesc* desc, uint32_t w, int32_t base, int off,
                                              int tx) {
  uint32_t m = w & kBounceMask;
  int i = 0;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    const int e = off + i;
    if (e < kLinkCap) desc[e] = LinkDesc{base + i, (tx << 8) | j};
    ++i;
  }
}

__device__ __forceinline__ void issue_links(double* pool, const LinkDesc* desc, int n, int lane,
                                            const double* __restrict__ src, int64_t row_cell0,
                                            const KParams& p) {
  for (int e = lane; e < n; e += 32) {
    const LinkDesc d = desc[e];
    const int j = d.oj & 31;
    cp_async8(pool + 2 * e, p.links + d.rec);
    cp_async8(pool + 2 * e + 1, src + row_cell0 + (d.oj >> 8) + (int64_t)j * p.ks);
  }
}

// Closure of one entry (boundary.cpp:24-41 in pull form, same arithmetic as
// links_all): slot j of the owner holds g_k(x), slot k the pull value.
__device__ __forceinline__ void close_link(double* stage_base, int owner, int j, double rec,
                                           double gj, const KParams& p) {
  if (rec == rec) {
    const int k = (j & 1) ? j + 1 : j - 1;
    double* sj = stage_base + j * kPipeBX + owner;
    const double gk = *sj;
    if (!isinf(rec))
      *sj = DADD(DSUB(DMUL(rec, stage_base[k * kPipeBX + owner]), DMUL(rec, gj)), gk);
    else
      *sj = DSUB(gk, p.mw[k]);
  }
}

// ---------------------------------------------------------------------------
// K1 main sweep: asynchronous-copy pipeline.  A block owns a 128-cell x
// segment of one (y) row and marches through `zper` consecutive z-planes.
// While plane z is collided from shared memory, each thread's loads for plane
// z+1 are already in flight as cp.async (LDGSTS) copies into the other stage:
// the 19 population loads (predicated per cell, address selected by the
// bounce bit exactly as in sweep_cell) and, for cells with CLI / moving-wall
// links, the link records and g_j(x) into a per-warp pool allocated by a warp
// prefix sum (cells that overflow it load those directly).  In-flight bytes
// therefore cost no registers.  Non-fluid cells that share a 32-byte sector
// with fluid cells write zeros so no DRAM sector is ever partially written.
// ---------------------------------------------------------------------------
template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(kPipeBX, pipe_minb(RECORDS))
    k_sweep_pipe(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                 int part, int zper) {
  extern __shared__ double smem[];
  // programmatic dependent launch (no-op without the attribute): the next
  // sweep's blocks may start during this grid's tail
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  constexpr int kStages = pipe_stages(RECORDS);
  const int tx = threadIdx.x;
  const int lane = tx & 31, warp = tx >> 5;
  const int x = blockIdx.x * kPipeBX + tx;
  const int y = blockIdx.y;
  const int z0 = blockIdx.z * zper;
  const int z1 = min(z0 + zper, p.nz);
  // valid: a cell of the row (its links stay in the warp's link list so record
  // indices follow from the chunk base); active: the cell is swept by this part.
  const bool valid = x < p.nx;
  const bool active = valid && !(part == PART_INTERIOR && in_edge_band(x, p.nx));
  const int xx = valid ? x : 0;
  double* const main0 = smem + tx;
  constexpr int kMainStride = 19 * kPipeBX;
  constexpr int kWarpExtra = kPool + kLinkCap;              // doubles per warp per stage
  constexpr int kExtraStride = (kPipeBX / 32) * kWarpExtra;  // per stage
  double* const pool0 = smem + kStages * kMainStride + warp * kWarpExtra;
  LinkDesc* const desc0 = reinterpret_cast<LinkDesc*>(pool0 + kPool);
  auto cidx = [&](int z) { return ((int64_t)z * p.ny + y) * p.nx + xx; };
  const CellWord kSkip{kNonFluid, 0};
  // 4-byte cell word + the warp's chunk base (uniform address: one transaction)
  const int chunk = (blockIdx.x * kPipeBX + warp * 32) >> 5;
  auto ld_w = [&](int z) {
    return CellWord{__ldg(p.cellw + cidx(z)),
                    RECORDS ? __ldg(p.chunkbase + ((int64_t)z * p.ny + y) * p.nchunk + chunk)
                            : 0};
  };
  // word of plane z+2: two-stage sweeps load it unconditionally (clamped
  // plane; masked where used), one-stage sweeps select (measured per variant)
  auto next_w = [&](int z2) {
    if (pipe_stages(RECORDS) == 2) return ld_w(min(z2, p.nz - 1));
    return (valid && z2 < min((v_ctaid_z() + 1) * zper, p.nz)) ? ld_w(z2) : CellWord{kNonFluid, 0};
  };

  // issue plane z into stage s; returns the warp's link count for plane z.
  // z-plane range end and the wrap-free predicate are recomputed where used
  auto z_end = [&]() { return min((v_ctaid_z() + 1) * zper, p.nz); };
  auto off_wrap = [&](int z) {
    const int xv = v_ctaid_x() * kPipeBX + v_tid_x(), yv = v_ctaid_y();
    return xv > 0 && xv < p.nx - 1 && yv > 0 && yv < p.ny - 1 && z > 0 && z < p.nz - 1;
  };
  auto issue = [&](int z, int s, CellWord cw) -> int {
    const bool fluid = !(cw.w & kNonFluid);
    if (fluid && active) {
      if (off_wrap(z))
        issue_fast<0>(main0 + s * kMainStride, src + cidx(z), p, cw.w);
      else
        issue_all<0, SLAB>(main0 + s * kMainStride, src, xx, y, z, cidx(z), p, cw.w);
    }
    int total = 0;
    if (RECORDS) {
      const int n = fluid ? __popc(cw.w & kBounceMask) : 0;
      const int off = warp_excl_scan(n, lane, &total);
      if (total) {
        LinkDesc* desc = reinterpret_cast<LinkDesc*>(pool0 + s * kExtraStride + kPool);
        if (n) publish_links(desc, cw.w, cw.base + off, off, tx);
        __syncwarp();
        issue_links(pool0 + s * kExtraStride, desc, min(total, kLinkCap), lane, src,
                    cidx(z) - xx + blockIdx.x * kPipeBX, p);
      }
    }
    return total;
  };

  // Peeled pipeline: iteration z issues plane z+1 and computes plane z
  // (z = z0-1 only issues), so the issue code exists once.  With two stages
  // plane z+1 is issued before waiting for plane z; with one stage plane z is
  // first moved to registers and the stage refilled with plane z+1.  issue()
  // runs at a convergence point (it contains a warp scan).
  // The word of plane z+2 is loaded after plane z's collision where the
  // collision's register demand would otherwise spill it right after its load
  // (one-stage sweeps at 96 registers, GLBM sweeps); measured per variant.
  constexpr bool kLateW = kStages == 1 ? !PGPU_CW_EARLY : (GLBM || PGPU_CW_LATE2);
  // Words are loaded unconditionally (clamped plane, x = 0 for lanes past the
  // row) and masked where used, so no select waits on a load in flight.
  CellWord cw_cur = kSkip;
  CellWord cw_next = ld_w(z0);
  // static data only so far; the populations come from the previous sweep
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  int off_cur = 0;
  int s = kStages == 2 ? 1 : 0;
  for (int z = z0 - 1; z < z_end(); ++z) {
    int off_next = 0;
    CellWord cw_nn = kSkip;
    if (kStages == 2) {
      if (z + 1 < z_end()) off_next = issue(z + 1, s ^ 1, valid ? cw_next : kSkip);
      cp_async_commit();
      if (!kLateW) cw_nn = next_w(z + 2);
      cp_async_wait<1>();  // this thread's copies for plane z have landed
    } else {
      cp_async_wait<0>();  // plane z landed (the only group in flight)
    }
    const uint32_t w = active ? cw_cur.w : kNonFluid;
    const bool fluid = !(w & kNonFluid);
    const int64_t c = cidx(z);
    double f[19];
    if (RECORDS && off_cur) {  // off_cur: this warp's link count for plane z
      __syncwarp();            // every lane's copies of plane z have landed
      double* stage_base = smem + s * kMainStride + warp * 32;
      const double* pool = pool0 + s * kExtraStride;
      const LinkDesc* desc = reinterpret_cast<const LinkDesc*>(pool + kPool);
      const int ncoop = min(off_cur, kLinkCap);
      for (int e = lane; e < ncoop; e += 32) {
        const LinkDesc d = desc[e];
        close_link(stage_base - warp * 32, d.oj >> 8, d.oj & 31, pool[2 * e], pool[2 * e + 1], p);
      }
      if (off_cur > kLinkCap) {  // warp-uniform: the pool overflowed for plane z
        // each lane closes its own entries past the cap with direct loads
        int tot;
        const bool lf = valid && !(cw_cur.w & kNonFluid);  // same counting as issue()
        const int off = warp_excl_scan(lf ? __popc(cw_cur.w & kBounceMask) : 0, lane, &tot);
        uint32_t m = fluid ? (w & kBounceMask) : 0u;
        int i = 0;
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          if (off + i >= kLinkCap)
            close_link(smem + s * kMainStride, tx, j, __ldg(p.links + cw_cur.base + off + i),
                       ldg(src + (int64_t)j * p.ks + c), p);
          ++i;
        }
      }
      __syncwarp();  // closures of other lanes' cells are visible
    }
    if (fluid) {
      const double* st = main0 + s * kMainStride;
#pragma unroll
      for (int j = 0; j < 19; ++j) f[j] = st[j * kPipeBX];
    }
    if (kStages == 1) {  // stage consumed: refill it with plane z+1
      if (z + 1 < z_end()) off_next = issue(z + 1, 0, valid ? cw_next : kSkip);
      cp_async_commit();
      // plane z+2's word: loaded after the collision so it does not occupy
      // registers across it (at 96 registers it would be spilled right after
      // its load, which exposes the load latency)
      if (PGPU_CW_EARLY) cw_nn = next_w(z + 2);
    }
    bool got_nn = false;
    if (w & kFillSector) {
      double* const dc = dst + c;
#pragma unroll
      for (int j = 0; j < 19; ++j) __stcs(dc + p.plane_off[j], 0.0);
    } else if (fluid) {
      if (OP == OP_STREAM_COLLIDE) collide<CM, GLBM>(f, p, z);
      if (kLateW) {
        cw_nn = next_w(z + 2);
        got_nn = true;
      }
      double* const dc = dst + c;
#pragma unroll
      for (int j = 0; j < 19; ++j) __stcs(dc + p.plane_off[j], f[j]);
      if (SLAB && OP == OP_STREAM_COLLIDE) {
        const int64_t hp = (int64_t)p.ny * p.nz;
        const int64_t h = (int64_t)z * p.ny + y;
        if (xx == 0) {
          p.send_lo[0 * hp + h] = f[2];
          p.send_lo[1 * hp + h] = f[8];
          p.send_lo[2 * hp + h] = f[10];
          p.send_lo[3 * hp + h] = f[12];
          p.send_lo[4 * hp + h] = f[14];
        }
        if (xx == p.nx - 1) {
          p.send_hi[0 * hp + h] = f[1];
          p.send_hi[1 * hp + h] = f[7];
          p.send_hi[2 * hp + h] = f[9];
          p.send_hi[3 * hp + h] = f[11];
          p.send_hi[4 * hp + h] = f[13];
        }
      }
    }
    if (kLateW && !got_nn)
      cw_nn = next_w(z + 2);
    cw_cur = cw_next;
    cw_next = cw_nn;
    off_cur = off_next;
    if (kStages == 2) s ^= 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Persistent sweep for L2-resident domains (e.g. C1, 20 MB of state): ONE
// cooperative launch runs `nsteps` K1 sweeps, ping-ponging the two buffers,
// with a grid-wide barrier between steps instead of a kernel boundary.  The
// evolving state is read with L2-coherent loads (written by other blocks in
// the same launch); the grid barrier orders the steps.
// ---------------------------------------------------------------------------
template <int CM, bool GLBM, bool RECORDS>
__global__ void __launch_bounds__(128) k_sweep_persistent(const KParams p, double* a, double* b,
                                                          int64_t nsteps) {
  cg::grid_group grid = cg::this_grid();
  const int64_t cells = (int64_t)p.nx * p.ny * p.nz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = 0; s < nsteps; ++s) {
    const double* src = (s & 1) ? b : a;
    double* dst = (s & 1) ? a : b;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += stride) {
      const int x = (int)(c % p.nx);
      const int64_t r = c / p.nx;
      const int y = (int)(r % p.ny), z = (int)(r / p.ny);
      sweep_cell<CM, GLBM, RECORDS, false, OP_STREAM_COLLIDE, true>(p, src, dst, x, y, z,
                                                                      ld_cw(p, c));
    }
    grid.sync();
  }
}

// Edge columns x = 0 and x = nx-1 only (slab overlap path).
template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
__global__ void __launch_bounds__(128) k_sweep_edges(const KParams p,
                                                     const double* __restrict__ src,
                                                     double* __restrict__ dst) {
  // grid (2 faces, ceil(ny * band / 128), nz); threads walk (y, column) pairs
  const int w = edge_band(p.nx);
  const int t = blockIdx.y * blockDim.x + threadIdx.x;
  const int xx = t % w, y = t / w;
  const int z = blockIdx.z;
  if (y >= p.ny) return;
  const int x = blockIdx.x ? p.nx - w + xx : xx;
  if (blockIdx.x && x < w) return;  // the bands overlap when nx < 2w
  const CellWord cw = ld_cw(p, ((int64_t)z * p.ny + y) * p.nx + x);
  sweep_cell<CM, GLBM, RECORDS, SLAB, OP>(p, src, dst, x, y, z, cw);
}

// K0: collide every fluid cell in place (first step from a pre-collision state).
template <int CM, bool GLBM, bool SLAB>
__global__ void __launch_bounds__(128) k_collide_inplace(const KParams p, double* buf) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  if (p.cellw[c] & kNonFluid) return;
  double f[19];
#pragma unroll
  for (int j = 0; j < 19; ++j) f[j] = buf[(int64_t)j * p.ks + c];
  collide<CM, GLBM>(f, p, z);
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
// moments(): lattice.cpp:88-101, literal order over k = 0..18.  `slot` and
// `stride`: the cell's element and the plane stride of the state's layout
// (dense: cell index / ksd; fluid-only: compact slot / ks).
template <bool GLBM>
__device__ __forceinline__ bool macro_cell(const KParams& p, const double* __restrict__ f,
                                           int64_t slot, int64_t stride, int z, double& drho,
                                           double (&u)[3]) {
  double d = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
  for (int k = 0; k < 19; ++k) {
    const double fk = f[(int64_t)k * stride + slot];
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

template <bool GLBM, bool COMPACT>
__global__ void k_macro_fields(const KParams p, const double* __restrict__ f, double* drho,
                               double* ux, double* uy, double* uz, int* err) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= p.nx) return;
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  if (p.cellw[c] & kNonFluid) {
    if (drho) drho[c] = 0.0;
    if (ux) ux[c] = 0.0;
    if (uy) uy[c] = 0.0;
    if (uz) uz[c] = 0.0;
    return;
  }
  double d, u[3];
  const int64_t slot = COMPACT ? compact_slot(p, x, y, z) : c;
  if (!macro_cell<GLBM>(p, f, slot, COMPACT ? p.ks : p.ksd, z, d, u)) atomicOr(err, 1);
  if (drho) drho[c] = d;
  if (ux) ux[c] = u[0];
  if (uy) uy[c] = u[1];
  if (uz) uz[c] = u[2];
}

// Sequential per-plane sum in ascending cell order (simulation.cpp:400-407):
// one block per plane; thread 0 adds the plane's values in cell order (the
// reference's rounding sequence) from shared-memory tiles that the other
// warps stream in ahead of it.  Non-fluid cells hold +0.0 (k_macro_fields),
// and s + (+0.0) == s exactly because a round-to-nearest sum that starts at
// +0.0 is never -0.0, so adding every cell equals adding the fluid cells.
constexpr int kSumTile = 2048;
__global__ void __launch_bounds__(256) k_plane_sums(const double* __restrict__ u, int64_t plane,
                                                    double* sums) {
  __shared__ double buf[2][kSumTile];
  const int z = blockIdx.x;
  const double* src = u + plane * z;
  const int64_t ntiles = (plane + kSumTile - 1) / kSumTile;
  auto load = [&](int64_t t, int first, int stride) {
    const int64_t base = t * kSumTile;
    double* b = buf[t & 1];
    for (int i = first; i < kSumTile; i += stride)
      b[i] = base + i < plane ? __ldg(src + base + i) : 0.0;
  };
  load(0, threadIdx.x, blockDim.x);
  __syncthreads();
  double s = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    if (threadIdx.x >= 32) {
      if (t + 1 < ntiles) load(t + 1, threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x == 0) {
      const double* b = buf[t & 1];
      const int n = (int)min((int64_t)kSumTile, plane - t * kSumTile);
      for (int i = 0; i < n; ++i) s = DADD(s, b[i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[z] = s;
}

// max |u|^2 and finiteness over fluid cells (simulation.cpp:419-434).
template <bool GLBM, bool COMPACT>
__global__ void k_max_speed2(const KParams p, const double* __restrict__ f,
                             unsigned long long* vmax2_bits, int* nonfinite, int* err) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  double m2 = 0.0;
  bool bad = false;
  if (x < p.nx) {
    const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
    if (!(p.cellw[c] & kNonFluid)) {
      double d, u[3];
      const int64_t slot = COMPACT ? compact_slot(p, x, y, z) : c;
      if (!macro_cell<GLBM>(p, f, slot, COMPACT ? p.ks : p.ksd, z, d, u)) atomicOr(err, 1);
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

// Free stream() (simulation.cpp:278-321 stream_pass + swap, 436-439) in pull
// form: fluid d gets cur_k(d - e_k) when that (wrapped) source is fluid; other
// slots keep `next` (the reference writes only fluid-fluid pairs).
__global__ void k_stream_field(const uint8_t* __restrict__ flags, int nx, int ny, int nz, int px,
                               int py, int pz, const double* __restrict__ cur,
                               double* __restrict__ next, int64_t cells) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells || flags[c] != 0) return;
  const int x = (int)(c % nx), y = (int)((c / nx) % ny), z = (int)(c / ((int64_t)nx * ny));
  next[c] = cur[c];
#pragma unroll
  for (int k = 1; k < 19; ++k) {
    int xs = x - EX[k], ys = y - EY[k], zs = z - EZ[k];
    if (xs < 0) xs = px ? nx - 1 : -1;
    if (xs >= nx) xs = px ? 0 : -1;
    if (ys < 0) ys = py ? ny - 1 : -1;
    if (ys >= ny) ys = py ? 0 : -1;
    if (zs < 0) zs = pz ? nz - 1 : -1;
    if (zs >= nz) zs = pz ? 0 : -1;
    if (xs < 0 || ys < 0 || zs < 0) continue;
    const int64_t s = ((int64_t)zs * ny + ys) * nx + xs;
    if (flags[s] == 0) next[(int64_t)k * cells + c] = cur[(int64_t)k * cells + s];
  }
}

void launch_stream_field(const uint8_t* flags, const int dims[3], const int per[3],
                         const double* cur, double* next, cudaStream_t s) {
  const int64_t cells = (int64_t)dims[0] * dims[1] * dims[2];
  k_stream_field<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(
      flags, dims[0], dims[1], dims[2], per[0], per[1], per[2], cur, next, cells);
}

__global__ void k_fill_equilibrium(const uint32_t* __restrict__ cw, int64_t cells,
                                   int64_t ks, double* f, const double* feq /*19*/) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  if (cw[c] & kNonFluid) return;
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
// z-planes per block: long marching columns, but at least ~6.5 waves of
// blocks over 148 SMs x 4 resident blocks (zper_for, sweep_compact.cu).
int pipe_zper(const KParams& p) {
  return zper_for((int64_t)((p.nx + kPipeBX - 1) / kPipeBX) * p.ny, p.nz);
}
// PGPU_SWEEP=pipe (default) | plain: the async-copy pipeline, or the plain
// one-cell-per-thread sweep kept as the round-1 reference point.
int g_sweep_mode = [] {
  const char* e = std::getenv("PGPU_SWEEP");
  return (e && e[0] == 'p' && e[1] == 'l') ? 2 : 1;
}();
}  // namespace
bool g_plain_sweep() { return g_sweep_mode == 2; }
namespace {
dim3 sweep_grid(const KParams& p) {
  const int bx = cell_block(p).x;
  return dim3((p.nx + bx - 1) / bx, p.ny, (p.nz + kZPer - 1) / kZPer);
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB, int OP>
void launch_sweep_t(const KParams& p, const double* src, double* dst, int part,
                    cudaStream_t s) {
  if (part == PART_EDGES) {
    k_sweep_edges<CM, GLBM, RECORDS, SLAB, OP>
        <<<dim3(2, (p.ny * edge_band(p.nx) + 127) / 128, p.nz), 128, 0, s>>>(p, src, dst);
  } else if (g_sweep_mode <= 1) {
    const int zper = pipe_zper(p);
    const dim3 grid((p.nx + kPipeBX - 1) / kPipeBX, p.ny, (p.nz + zper - 1) / zper);
    static bool attr = [] {
      cudaFuncSetAttribute(k_sweep_pipe<CM, GLBM, RECORDS, SLAB, OP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, pipe_smem(RECORDS));
      if (const char* e = std::getenv("PGPU_CARVEOUT"))  // experiment knob (percent)
        cudaFuncSetAttribute(k_sweep_pipe<CM, GLBM, RECORDS, SLAB, OP>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
      return true;
    }();
    (void)attr;
    static const bool pdl_env = [] {
      const char* e = std::getenv("PGPU_PDL");
      return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kPipeBX);
    lc.dynamicSmemBytes = pipe_smem(RECORDS);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = (pdl_env && !SLAB && part == PART_ALL && OP == OP_STREAM_COLLIDE) ? 1 : 0;
    cudaLaunchKernelEx(&lc, k_sweep_pipe<CM, GLBM, RECORDS, SLAB, OP>, p, src, dst, part, zper);
  } else {
    k_sweep<CM, GLBM, RECORDS, SLAB, OP><<<sweep_grid(p), cell_block(p), 0, s>>>(p, src, dst,
                                                                                  part);
  }
}

template <int CM, bool GLBM, bool RECORDS, bool SLAB>
void dispatch_op(int op, const KParams& p, const double* src, double* dst, int part,
                 cudaStream_t s) {
  if (op == OP_STREAM_COLLIDE)
    launch_sweep_t<CM, GLBM, RECORDS, SLAB, OP_STREAM_COLLIDE>(p, src, dst, part, s);
  else
    launch_sweep_t<CM, GLBM, RECORDS, SLAB, OP_STREAM_ONLY>(p, src, dst, part, s);
}
template <int CM, bool GLBM, bool RECORDS>
void dispatch_slab(bool slab, int op, const KParams& p, const double* src, double* dst,
                   int part, cudaStream_t s) {
  if (slab)
    dispatch_op<CM, GLBM, RECORDS, true>(op, p, src, dst, part, s);
  else
    dispatch_op<CM, GLBM, RECORDS, false>(op, p, src, dst, part, s);
}
template <int CM, bool GLBM>
void dispatch_rec(bool rec, bool slab, int op, const KParams& p, const double* src,
                  double* dst, int part, cudaStream_t s) {
  if (rec)
    dispatch_slab<CM, GLBM, true>(slab, op, p, src, dst, part, s);
  else
    dispatch_slab<CM, GLBM, false>(slab, op, p, src, dst, part, s);
}
}  // namespace

void launch_sweep(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s) {
  if (p.ctab) {  // fluid-only layout (sweep_compact.cu)
    launch_sweep_compact(cfg, p, src, dst, s);
    return;
  }
  switch (collide_mode(p)) {
    case CM_FAST:
    case CM_FAST_FOLD:  // (folding is a fluid-only-layout feature)
      if (cfg.glbm) dispatch_rec<CM_FAST, true>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
      else dispatch_rec<CM_FAST, false>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
      break;
    case CM_EXACT_RHO1:
      if (cfg.glbm) dispatch_rec<CM_EXACT_RHO1, true>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
      else dispatch_rec<CM_EXACT_RHO1, false>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
      break;
    default:
      if (cfg.glbm) dispatch_rec<CM_EXACT, true>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
      else dispatch_rec<CM_EXACT, false>(cfg.records, cfg.slab, cfg.op, p, src, dst, cfg.part, s);
  }
}

template <int CM, bool GLBM, bool RECORDS>
int64_t persistent_t(const KParams& p, double* a, double* b, int64_t nsteps, cudaStream_t s) {
  auto kern = k_sweep_persistent<CM, GLBM, RECORDS>;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  const int64_t cells = (int64_t)p.nx * p.ny * p.nz;
  const int64_t want = (cells + 127) / 128;
  const int blocks = (int)std::min<int64_t>(want, (int64_t)sms * per_sm);
  if (blocks < 1) return -1;
  KParams pp = p;
  void* args[] = {(void*)&pp, (void*)&a, (void*)&b, (void*)&nsteps};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(blocks), dim3(128), args, 0, s) ==
                 cudaSuccess
             ? 0
             : -1;
}

template <int CM>
int64_t persistent_cm(const SweepConfig& cfg, const KParams& p, double* a, double* b,
                      int64_t nsteps, cudaStream_t s) {
  if (cfg.glbm) return cfg.records ? persistent_t<CM, true, true>(p, a, b, nsteps, s)
                                   : persistent_t<CM, true, false>(p, a, b, nsteps, s);
  return cfg.records ? persistent_t<CM, false, true>(p, a, b, nsteps, s)
                     : persistent_t<CM, false, false>(p, a, b, nsteps, s);
}

int launch_sweep_persistent(const SweepConfig& cfg, const KParams& p, double* a, double* b,
                            int64_t nsteps, cudaStream_t s) {
  switch (collide_mode(p)) {
    case CM_FAST:
    case CM_FAST_FOLD: return (int)persistent_cm<CM_FAST>(cfg, p, a, b, nsteps, s);
    case CM_EXACT_RHO1: return (int)persistent_cm<CM_EXACT_RHO1>(cfg, p, a, b, nsteps, s);
    default: return (int)persistent_cm<CM_EXACT>(cfg, p, a, b, nsteps, s);
  }
}

template <int CM>
void collide_inplace_cm(bool glbm, bool slab, const KParams& p, double* buf, cudaStream_t s) {
  const dim3 g = cell_grid2(p), b = cell_block(p);
  if (glbm) {
    if (slab) k_collide_inplace<CM, true, true><<<g, b, 0, s>>>(p, buf);
    else k_collide_inplace<CM, true, false><<<g, b, 0, s>>>(p, buf);
  } else {
    if (slab) k_collide_inplace<CM, false, true><<<g, b, 0, s>>>(p, buf);
    else k_collide_inplace<CM, false, false><<<g, b, 0, s>>>(p, buf);
  }
}

void launch_collide_inplace(bool glbm, bool slab, const KParams& p, double* buf,
                            cudaStream_t s) {
  switch (collide_mode(p)) {
    case CM_FAST:
    case CM_FAST_FOLD: collide_inplace_cm<CM_FAST>(glbm, slab, p, buf, s); break;
    case CM_EXACT_RHO1: collide_inplace_cm<CM_EXACT_RHO1>(glbm, slab, p, buf, s); break;
    default: collide_inplace_cm<CM_EXACT>(glbm, slab, p, buf, s);
  }
}

void launch_macro_fields(bool glbm, const KParams& p, const double* f, double* drho,
                         double* ux, double* uy, double* uz, int* err, cudaStream_t s) {
  const dim3 g = cell_grid2(p), b = cell_block(p);
  if (p.ctab) {
    if (glbm) k_macro_fields<true, true><<<g, b, 0, s>>>(p, f, drho, ux, uy, uz, err);
    else k_macro_fields<false, true><<<g, b, 0, s>>>(p, f, drho, ux, uy, uz, err);
  } else {
    if (glbm) k_macro_fields<true, false><<<g, b, 0, s>>>(p, f, drho, ux, uy, uz, err);
    else k_macro_fields<false, false><<<g, b, 0, s>>>(p, f, drho, ux, uy, uz, err);
  }
}

void launch_plane_sums(const KParams& p, const double* u, double* sums, cudaStream_t s) {
  const int64_t plane = (int64_t)p.nx * p.ny;
  k_plane_sums<<<p.nz, 256, 0, s>>>(u, plane, sums);
}

void launch_max_speed2(bool glbm, const KParams& p, const double* f,
                       unsigned long long* vmax2_bits, int* nonfinite, int* err,
                       cudaStream_t s) {
  const dim3 g = cell_grid2(p), b = cell_block(p);
  if (p.ctab) {
    if (glbm) k_max_speed2<true, true><<<g, b, 0, s>>>(p, f, vmax2_bits, nonfinite, err);
    else k_max_speed2<false, true><<<g, b, 0, s>>>(p, f, vmax2_bits, nonfinite, err);
  } else {
    if (glbm) k_max_speed2<true, false><<<g, b, 0, s>>>(p, f, vmax2_bits, nonfinite, err);
    else k_max_speed2<false, false><<<g, b, 0, s>>>(p, f, vmax2_bits, nonfinite, err);
  }
}

void launch_fill_equilibrium(const KParams& p, int64_t cells, double* f, const double* feq,
                             cudaStream_t s) {
  k_fill_equilibrium<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(p.cellw, cells, p.ksd, f,
                                                                     feq);
}

// Load the observable kernels' code once per process (CUDA loads modules
// lazily at first launch, ~10 ms on the first observable otherwise).
void preload_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_macro_fields<true, false>);
  cudaFuncGetAttributes(&a, k_macro_fields<false, false>);
  cudaFuncGetAttributes(&a, k_macro_fields<true, true>);
  cudaFuncGetAttributes(&a, k_macro_fields<false, true>);
  cudaFuncGetAttributes(&a, k_plane_sums);
  cudaFuncGetAttributes(&a, k_max_speed2<true, false>);
  cudaFuncGetAttributes(&a, k_max_speed2<false, false>);
  cudaFuncGetAttributes(&a, k_max_speed2<true, true>);
  cudaFuncGetAttributes(&a, k_max_speed2<false, true>);
  cudaFuncGetAttributes(&a, k_fill_equilibrium);
  cudaGetLastError();
}

}  // namespace pgpu
