// K1 over the fluid-only layout as a warp-specialised TMA pipeline (sm_100a).
//
// Same step as sweep_compact.cu's k_sweep_cpipe -- g' = C(P(g)), P the pull
// form of the reference's push streaming + link bounce-back
// (simulation.cpp:278-342, boundary.cpp:19-41), C the TRT / GLBM collision
// (simulation.cpp:150-274) -- with a different memory schedule:
//
// * Work item = one row segment of kTWB = 32*kTNC cells (kTNC chunks) at one
//   z, numbered (z, y, segment) with the segment fastest.  A persistent grid
//   (2 blocks per SM) draws the items in increasing order from a global
//   counter, so the whole GPU works on a narrow band of neighbouring rows at
//   any moment: the sectors shared by the runs of neighbouring segments and
//   the re-read link sources stay in L2 (a static round-robin deal let the
//   blocks drift apart and cost 1.6 GB of extra DRAM reads per C4 step).
// * Fluid-only slots are numbered in the reference's cell order, so the pull
//   sources of direction j for a segment are ONE contiguous slot run of the
//   source row (y - e_jy, z - e_jz): the fluid cells with x in
//   [x0 - e_jx, x0 + kTWB - e_jx).  Producer warps copy the 19 runs of an
//   item, its cell words, CLI records and link descriptors with
//   `cp.async.bulk` (TMA engine: straight into shared memory, no L1, no
//   registers) into a stage of a kTS-deep ring, completion on the stage's
//   mbarrier; the bytes in flight per SM are ~(kTS - 1) stages x 2 blocks
//   (~120 KB) instead of one plane of per-thread copies.
// * The link sources (bounce source g_k(x), CLI g_j(x)) and the x-wrap pulls
//   are single slots: once an item's descriptors have landed, its producer
//   issues them as 8-byte cp.async copies tracked by a second mbarrier
//   (cp.async.mbarrier.arrive.noinc), one own item later.
// * kTNC consumer warps (one chunk each) wait for both barriers, close the
//   CLI / moving-wall links cooperatively in shared memory (one lane per link,
//   the reference's arithmetic), take their 19 pulls with a popcount per
//   source row, release the stage, and collide / store while it is refilled.
//
// Arithmetic per cell is the sweep_compact.cu / kernels.cu one (collide<CM,
// GLBM>, the link closures in the reference order), so the results are
// bit-identical to k_sweep_cpipe in every math mode it supports (EXACT and
// FAST; folded links stay on k_sweep_cpipe).  tests/test_gpu_tma.py.
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

#ifndef PGPU_TMA_NC
#define PGPU_TMA_NC 4
#endif
#ifndef PGPU_TMA_STAGES
#define PGPU_TMA_STAGES 4
#endif
#ifndef PGPU_TMA_LC
#define PGPU_TMA_LC 192
#endif
#ifndef PGPU_TMA_MINB
#define PGPU_TMA_MINB 2
#endif
#ifndef PGPU_TMA_PROD
#define PGPU_TMA_PROD 2
#endif
#ifndef PGPU_TMA_BATCH
#define PGPU_TMA_BATCH 1
#endif
constexpr int kTNC = PGPU_TMA_NC;       // consumer warps = chunks per item
constexpr int kTS = PGPU_TMA_STAGES;    // stages of the ring
constexpr int kTLC = PGPU_TMA_LC;       // links per item staged in shared memory
constexpr int kTWB = 32 * kTNC;         // cells per item
constexpr int kTSpan = kTWB + 4;        // slots per direction run (+1 cell each side, alignment)
constexpr int kTM = 4;                  // chunk-entry ring per producer (own items u .. u+3)
constexpr int kTP = PGPU_TMA_PROD;      // producer warps (items dealt round-robin)
constexpr uint32_t kTB = PGPU_TMA_BATCH; // work items per counter draw
constexpr int kTThreads = 32 * (kTNC + kTP + 1);  // producers, the link warp, consumers
constexpr int kTEnt = 9 * (kTNC + 2);   // chunk entries per item: 9 source rows x chunks c0-1 .. c0+kTNC

__device__ __forceinline__ uint32_t tsmem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tcpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tsmem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void tcpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(tsmem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void tcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void twait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tsmem(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tsmem(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tsmem(b)),
               "r"(bytes)
               : "memory");
}
// every earlier cp.async of this thread completes -> one arrival (pre-counted)
__device__ __forceinline__ void mbar_cpasync_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(tsmem(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(tsmem(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          tsmem(dst)),
      "l"(src), "r"(bytes), "r"(tsmem(b))
      : "memory");
}

// Source rows (as sweep_compact.cu): row r holds the directions with
// (e_y, e_z) = (trow_ey(r), trow_ez(r)).
//   r0 (0,0): 0 1 2   r1 (1,0): 3 7 10   r2 (-1,0): 4 8 9   r3 (0,1): 5 11 14
//   r4 (0,-1): 6 12 13   r5 (1,1): 15   r6 (-1,-1): 16   r7 (1,-1): 17   r8 (-1,1): 18
__host__ __device__ constexpr int trow_ey(int r) {
  return (r == 1 || r == 5 || r == 7) ? 1 : ((r == 2 || r == 6 || r == 8) ? -1 : 0);
}
__host__ __device__ constexpr int trow_ez(int r) {
  return (r == 3 || r == 5 || r == 8) ? 1 : ((r == 4 || r == 6 || r == 7) ? -1 : 0);
}
__host__ __device__ constexpr int trow_of(int j) {
  return j <= 2 ? 0
         : (j == 3 || j == 7 || j == 10) ? 1
         : (j == 4 || j == 8 || j == 9)  ? 2
         : (j == 5 || j == 11 || j == 14) ? 3
         : (j == 6 || j == 12 || j == 13) ? 4
                                          : j - 10;
}
// runtime lookups (4-bit / 2-bit packed tables)
__host__ __device__ constexpr uint64_t pack_trow(int q) {
  return q == 15 ? 0ull : ((uint64_t)trow_of(q) << (4 * q)) | pack_trow(q + 1);
}
__host__ __device__ constexpr int tex(int q) {
  return (q == 1 || q == 7 || q == 9 || q == 11 || q == 13) ? 1
         : (q == 2 || q == 8 || q == 10 || q == 12 || q == 14) ? -1 : 0;
}
__host__ __device__ constexpr uint64_t pack_tex(int q) {
  return q == 19 ? 0ull : ((uint64_t)(tex(q) + 1) << (2 * q)) | pack_tex(q + 1);
}
constexpr uint64_t kTRow = pack_trow(0);
constexpr uint64_t kTEx = pack_tex(0);
__device__ __forceinline__ int rt_trow(int j) {  // rows 5..8 hold j = 15..18 alone
  return j >= 15 ? j - 10 : (int)((kTRow >> (4 * j)) & 15u);
}
__device__ __forceinline__ int rt_ex(int j) { return (int)((kTEx >> (2 * j)) & 3u) - 1; }
__device__ __forceinline__ int rt_opp(int j) { return (j & 1) ? j + 1 : j - 1; }
__device__ __forceinline__ bool twrap(int& v, int n, int periodic) {
  if (v >= 0 && v < n) return true;
  if (!periodic) return false;
  v = v < 0 ? v + n : v - n;
  return true;
}
// x-wrap directions of the source rows 0..4: e_x = +1 (lane at x = 0) and
// e_x = -1 (lane at x = nx - 1)
__host__ __device__ constexpr int wrap_plus(int r) {
  return r == 0 ? 1 : r == 1 ? 7 : r == 2 ? 9 : r == 3 ? 11 : 13;
}
__host__ __device__ constexpr int wrap_minus(int r) {
  return r == 0 ? 2 : r == 1 ? 10 : r == 2 ? 8 : r == 3 ? 14 : 12;
}

struct alignas(16) TStage {
  double pop[19][kTSpan];    // direction runs: slot base_r + i of source row r at pop[j][i]
  double gk[kTLC];           // per link: g_k(x) (bounce source), then the closed value
  double gj[kTLC];           // per link: g_j(x) (CLI)
  double rec[kTLC + 2];      // link records from the even record at or below the first
  double wrap[10];           // x-wrap pulls of the lanes at x = 0 (0..4) / x = nx-1 (5..9)
  uint32_t cw[kTWB];         // cell words
  uint16_t desc[kTLC + 16];  // per link: owner lane | j << 5, from the record at or below the
                             // first that is a multiple of 8 (16-byte bulk copy)
  uint2 rowinfo[9][kTNC];    // per source row and chunk: {rank - base_r, fluid mask}
  uint32_t own_rank[kTNC];   // compact slot of each chunk's first fluid cell
  int32_t lofs[kTNC + 1];    // first link of each chunk in the item's list; [kTNC] = count
  uint32_t wsrc[10];         // x-wrap pull sources (element offsets into src), ~0u: none
  int32_t cb_lo;             // first link record of the item
  int32_t recoff;            // cb_lo & 1
  int32_t descoff;           // cb_lo & 7
  int32_t x0, z;             // the item's first cell and plane
  uint32_t item;             // work item, kTDone: its producer has no more items
};
// bulk-copy destinations are 16-byte aligned
static_assert(offsetof(TStage, pop) % 16 == 0 && (kTSpan * 8) % 16 == 0, "runs");
static_assert(offsetof(TStage, rec) % 16 == 0 && offsetof(TStage, cw) % 16 == 0 &&
                  offsetof(TStage, desc) % 16 == 0,
              "bulk destinations");
struct alignas(16) TMeta {
  uint2 ent[9][kTNC + 2];  // chunk entries c0-1 .. c0+kTNC of the 9 source rows (zero: absent)
  uint2 part[10];          // x-wrap partners of rows 0..4: last chunk (0..4), chunk 0 (5..9)
  int32_t cbase[kTNC + 1]; // link record bases of chunks c0 .. c0+kTNC
  uint32_t item;           // work item (kTDone: none)
  int32_t c0, y, z, row;   // its decoded coordinates
};
constexpr uint32_t kTDone = 0xffffffffu;
struct alignas(128) TSmem {
  TStage st[kTS];
  TMeta meta[kTP][kTM];
  uint64_t full[kTS];   // bulk bytes of the stage (and the producer's header stores)
  uint64_t xfull[kTS];  // link-source copies of the stage (32 link-warp lanes)
  uint64_t hdr[kTS];    // the stage header is written (the link warp starts on it)
  uint64_t empty[kTS];  // kTNC consumer warps released the stage
};

struct TItem {
  int c0, x0, y, z, row;  // row = z * ny + y
};
// n / d for n < 2^31 from a double reciprocal (exact after one correction)
struct TDiv {
  uint32_t d;
  double inv;
};
__device__ __forceinline__ uint32_t tdiv(uint32_t n, TDiv v) {
  uint32_t q = (uint32_t)((double)n * v.inv);
  if (q * v.d > n) --q;
  if ((q + 1) * v.d <= n) ++q;
  return q;
}
__device__ __forceinline__ TItem titem(uint32_t t, TDiv nseg, TDiv ny) {
  TItem it;
  const uint32_t row = tdiv(t, nseg);
  it.c0 = (int)(t - row * nseg.d) * kTNC;
  it.x0 = it.c0 * 32;
  it.row = (int)row;
  it.z = (int)tdiv(row, ny);
  it.y = (int)(row - (uint32_t)it.z * ny.d);
  return it;
}
// source-row offsets as packed 2-bit tables (value + 1)
__device__ __forceinline__ int rt_row_ey(int r) {
  constexpr uint32_t t = (trow_ey(0) + 1) | (trow_ey(1) + 1) << 2 | (trow_ey(2) + 1) << 4 |
                         (trow_ey(3) + 1) << 6 | (trow_ey(4) + 1) << 8 | (trow_ey(5) + 1) << 10 |
                         (trow_ey(6) + 1) << 12 | (trow_ey(7) + 1) << 14 | (trow_ey(8) + 1) << 16;
  return (int)((t >> (2 * r)) & 3u) - 1;
}
__device__ __forceinline__ int rt_row_ez(int r) {
  constexpr uint32_t t = (trow_ez(0) + 1) | (trow_ez(1) + 1) << 2 | (trow_ez(2) + 1) << 4 |
                         (trow_ez(3) + 1) << 6 | (trow_ez(4) + 1) << 8 | (trow_ez(5) + 1) << 10 |
                         (trow_ez(6) + 1) << 12 | (trow_ez(7) + 1) << 14 | (trow_ez(8) + 1) << 16;
  return (int)((t >> (2 * r)) & 3u) - 1;
}
__device__ __forceinline__ void bulk_g2s_u(uint32_t dst, const void* src, uint32_t bytes,
                                           uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

template <int CM, bool GLBM, bool RECORDS>
__global__ void __launch_bounds__(kTThreads, GLBM ? 1 : PGPU_TMA_MINB)
    k_sweep_tma(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                uint32_t nitems, TDiv nseg, TDiv nyd) {
  static_assert(kTS % kTP == 0, "each stage belongs to one producer");
  extern __shared__ __align__(128) unsigned char tsm_raw[];
  TSmem& S = *reinterpret_cast<TSmem*>(tsm_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTS; ++s) {
      mbar_init(&S.full[s], 1);  // the producer's expect_tx arrival; the bulk bytes complete it
      mbar_init(&S.xfull[s], 32);
      mbar_init(&S.hdr[s], 1);
      mbar_init(&S.empty[s], kTNC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint32_t ks = (uint32_t)p.ks;
  const bool links = p.linkdesc != nullptr;

  if (warp < kTP) {
    // ------------------------------------------------------------------ producers
    // Producer warp `warp` fills stages k = warp, warp + kTP, ... of the block;
    // its own item u = k / kTP indexes its private ring of chunk entries.
    TMeta* const MR = S.meta[warp];
    // chunk entries, x-wrap partners and record bases of item t -> ring slot m
    auto meta_issue = [&](uint32_t t, int m) {
      TMeta& M = MR[m];
      if (lane == 0) M.item = t;
      if (t == kTDone) return;
      const TItem it = titem(t, nseg, nyd);
      if (lane == 0) {
        M.c0 = it.c0;
        M.y = it.y;
        M.z = it.z;
        M.row = it.row;
      }
      int srow = -1;  // lanes 0..8: source row r = lane (z * ny + y), -1 absent
      if (lane < 9) {
        int ys = it.y - rt_row_ey(lane), zs = it.z - rt_row_ez(lane);
        if (twrap(ys, p.ny, p.py) && twrap(zs, p.nz, p.pz)) srow = zs * p.ny + ys;
      }
      for (int i0 = 0; i0 < kTEnt + 32; i0 += 32) {  // uniform trip count (shuffles)
        const int i = i0 + lane;
        if (i < kTEnt) {
          const int r = i / (kTNC + 2), cc = i - r * (kTNC + 2);
          const int sr = __shfl_sync(0xffffffffu, srow, r);
          const int ch = it.c0 - 1 + cc;
          if (sr >= 0 && ch >= 0 && ch < p.nchunk)
            tcpa8(&M.ent[r][cc], p.ctab + (size_t)sr * p.nchunk + ch);
          else
            M.ent[r][cc] = make_uint2(0u, 0u);
        } else {
          const int w = i - kTEnt;  // 0..9 partners, 10..10+kTNC record bases
          const int sr = __shfl_sync(0xffffffffu, srow, w < 10 ? w % 5 : 0);
          if (w < 10) {
            const bool need = p.px && (w < 5 ? it.c0 == 0 : it.c0 + kTNC >= p.nchunk);
            if (need && sr >= 0)
              tcpa8(&M.part[w], p.ctab + (size_t)sr * p.nchunk + (w < 5 ? p.nchunk - 1 : 0));
            else
              M.part[w] = make_uint2(0u, 0u);
          } else if (w <= 10 + kTNC) {
            const int ch = min(it.c0 + w - 10, p.nchunk);  // may be the next row's chunk 0
            tcpa4(&M.cbase[w - 10], p.chunkbase + (size_t)it.row * p.nchunk + ch);
          }
        }
      }
    };
    // Work items come from the global counter in increasing order; a draw is
    // issued one iteration before its value is used (the atomic's latency is
    // hidden), and once the counter has passed nitems every later draw is done.
    // A draw takes kTB consecutive items (neighbouring segments); the next
    // draw is issued when a batch is started, so its latency hides behind the
    // batch.
    bool out = false;
    uint32_t pend = 0;  // lane 0: the next batch's counter value, in flight
    uint32_t cur = 0, left = 0;
    auto draw_issue = [&]() {
      if (lane == 0) pend = atomicAdd(p.tickets, 1u);
    };
    auto draw_take = [&]() -> uint32_t {
      if (out) return kTDone;
      if (left == 0) {
        cur = __shfl_sync(0xffffffffu, pend, 0) * kTB;
        left = kTB;
        if (cur >= nitems) {
          out = true;
          return kTDone;
        }
        draw_issue();
      }
      const uint32_t t = cur++;
      --left;
      if (t >= nitems) {
        out = true;
        return kTDone;
      }
      return t;
    };
    // prologue: the first kTM - 1 own items and their entries
    draw_issue();
    for (int u = 0; u + 1 < kTM; ++u) {
      meta_issue(draw_take(), u);
      tcommit();
    }
    for (uint32_t u = 0;; ++u) {
      const uint32_t k = u * kTP + warp;
      const int s = (int)(k % kTS), m = (int)(u % kTM);
      if (k >= kTS) mbar_wait(&S.empty[s], ((k / kTS) - 1) & 1u);
      twait_group<kTM - 2>();  // own item u's entries (kTM - 1 groups ago) landed
      __syncwarp();
      TStage& T = S.st[s];
      const TMeta& M = MR[m];
      const uint32_t t = M.item;
      if (t == kTDone) {  // publish the end of this producer's items
        if (lane == 0) {
          T.item = kTDone;
          mbar_arrive(&S.hdr[s]);
          mbar_arrive_tx(&S.full[s], 0u);
        }
        break;
      }
      TItem it;
      it.c0 = M.c0;
      it.x0 = it.c0 * 32;
      it.y = M.y;
      it.z = M.z;
      it.row = M.row;
      // per source row (lanes 0..8): the run base and its ends for e_x = +1, 0, -1
      uint32_t base = 0, ep = 0, e0 = 0, em = 0;
      if (lane < 9) {
        auto rank_at = [&](int X) -> uint32_t {
          if (X >= p.nx) {
            const uint2 e = M.ent[lane][p.nchunk - it.c0];  // last chunk of the row
            return e.x + __popc(e.y);
          }
          const uint2 e = M.ent[lane][(X >> 5) - it.c0 + 1];
          return e.x + __popc(e.y & ((1u << (X & 31)) - 1u));
        };
        base = rank_at(max(it.x0 - 1, 0)) & ~1u;
        ep = max(rank_at(min(it.x0 + kTWB - 1, p.nx)), base);
        e0 = max(rank_at(min(it.x0 + kTWB, p.nx)), base);
        em = max(rank_at(min(it.x0 + kTWB + 1, p.nx)), base);
      }
      // stage header
      for (int i0 = 0; i0 < 9 * kTNC; i0 += 32) {  // uniform trip count: every lane shuffles
        const int i = i0 + lane;
        const int r = min(i / kTNC, 8), cc = i % kTNC;
        const uint32_t br = __shfl_sync(0xffffffffu, base, r);
        if (i < 9 * kTNC) {
          const uint2 e = M.ent[r][cc + 1];
          T.rowinfo[r][cc] = make_uint2(e.x - br, it.c0 + cc < p.nchunk ? e.y : 0u);
        }
      }
      const int32_t cb_lo = M.cbase[0];
      const int nl = links ? min(M.cbase[kTNC] - cb_lo, kTLC) : 0;
      if (lane < kTNC) T.own_rank[lane] = M.ent[0][lane + 1].x;
      if (lane <= kTNC) T.lofs[lane] = links ? M.cbase[lane] - cb_lo : 0;
      if (lane == 0) {
        T.cb_lo = cb_lo;
        T.recoff = cb_lo & 1;
        T.descoff = cb_lo & 1;
        T.x0 = it.x0;
        T.z = it.z;
        T.item = t;
      }
      // x-wrap pull sources (periodic x): the lane at x = 0 takes its e_x = +1
      // directions from x = nx - 1 of the source rows, the lane at x = nx - 1
      // its e_x = -1 ones from x = 0
      if (lane < 10) {
        const int r = lane % 5;
        const bool lo = lane < 5;
        uint32_t w = ~0u;
        if (p.px && (lo ? it.c0 == 0 : it.c0 + kTNC >= p.nchunk)) {
          const uint2 e = M.part[lane];
          const int xs = lo ? p.nx - 1 : 0;
          if ((e.y >> (xs & 31)) & 1u)
            w = (uint32_t)(lo ? wrap_plus(r) : wrap_minus(r)) * ks + e.x +
                __popc(e.y & ((1u << (xs & 31)) - 1u));
        }
        T.wsrc[lane] = w;
      }
      __syncwarp();  // the header is complete: the link warp may start on the item
      if (lane == 0) mbar_arrive(&S.hdr[s]);
      // bulk copies: lanes 0..18 the direction runs, 19 the cell words, 20 the
      // records
      uint32_t bytes = 0, bdst = 0;
      const void* bsrc = nullptr;
      {
        const int j = lane < 19 ? lane : 0;
        const int r = rt_trow(j), ex = rt_ex(j);
        const uint32_t br = __shfl_sync(0xffffffffu, base, r);
        const uint32_t a = __shfl_sync(0xffffffffu, ep, r);
        const uint32_t b = __shfl_sync(0xffffffffu, e0, r);
        const uint32_t c = __shfl_sync(0xffffffffu, em, r);
        if (lane < 19) {
          const uint32_t end = ex > 0 ? a : (ex == 0 ? b : c);
          bytes = (((end + 1u) & ~1u) - br) * 8u;
          bsrc = src + ((uint32_t)j * ks + br);
          bdst = tsmem(&T.pop[j][0]);
        } else if (lane == 19) {
          bytes = (uint32_t)min(kTWB, p.nx - it.x0) * 4u;
          bsrc = p.cellw + (size_t)it.row * p.nx + it.x0;
          bdst = tsmem(&T.cw[0]);
        } else if (lane == 20 && RECORDS && nl > 0) {
          const int a0 = cb_lo & ~1;
          bytes = (uint32_t)(((cb_lo + nl - a0) + 1) & ~1) * 8u;
          bsrc = p.links + a0;
          bdst = tsmem(&T.rec[0]);
        }
      }
      uint32_t total = bytes;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      const uint32_t fbar = tsmem(&S.full[s]);
      __syncwarp();  // every lane's header stores precede the release below
      if (lane == 0) mbar_arrive_tx(&S.full[s], total);
      if (bytes) bulk_g2s_u(bdst, bsrc, bytes, fbar);
      // look-ahead: the entries of own item u + kTM - 1, the next draw
      meta_issue(draw_take(), (int)((u + kTM - 1) % kTM));
      tcommit();
      __syncwarp();
    }
    twait_group<0>();
  } else if (warp == kTP) {
    // ------------------------------------------------------------------- link warp
    // As soon as a stage's header is written (while its bulk copies fly), load
    // the item's link descriptors, then copy its link sources: g_k(x) and, for
    // CLI, g_j(x) per link, and the x-wrap pulls -- in parallel with the bulk
    // data instead of after it.
    uint32_t fin = 0;
    for (uint32_t k = 0; fin != (1u << kTP) - 1u; ++k) {
      if ((fin >> (k % kTP)) & 1u) continue;
      const int s = (int)(k % kTS);
      mbar_wait(&S.hdr[s], (k / kTS) & 1u);
      TStage& T = S.st[s];
      if (T.item == kTDone) {
        fin |= 1u << (k % kTP);
        continue;
      }
      const int nl = min(T.lofs[kTNC], kTLC);
      if (nl > 0) {
        const int32_t cb = T.cb_lo;
        const int a0 = cb & ~1, npairs = (cb + nl - a0 + 1) >> 1;
        for (int i = lane; i < npairs; i += 32) tcpa4(&T.desc[2 * i], p.linkdesc + a0 + 2 * i);
        tcommit();
        twait_group<0>();
        __syncwarp();
        int32_t lb[kTNC - 1];
#pragma unroll
        for (int q = 0; q < kTNC - 1; ++q) lb[q] = T.lofs[q + 1];
        const uint16_t* dd = T.desc + T.descoff;
        for (int e = lane; e < nl; e += 32) {
          const uint32_t d = dd[e];
          int c = 0;
#pragma unroll
          for (int q = 0; q < kTNC - 1; ++q) c += e >= lb[q];
          const int owner = d & 31, j = d >> 5;
          const uint32_t fc = T.own_rank[c] + __popc(T.rowinfo[0][c].y & ((1u << owner) - 1u));
          tcpa8(&T.gk[e], src + ((uint32_t)rt_opp(j) * ks + fc));
          if (RECORDS) tcpa8(&T.gj[e], src + ((uint32_t)j * ks + fc));
        }
      }
      if (lane < 10 && T.wsrc[lane] != ~0u) tcpa8(&T.wrap[lane], src + T.wsrc[lane]);
      mbar_cpasync_arrive(&S.xfull[s]);
    }
    twait_group<0>();
  } else {
    // ---------------------------------------------------------------- consumers
    // Consumer warp c owns chunk c of every item.
    const int c = warp - kTP - 1;
    const int tc = c * 32 + lane;
    const uint32_t ltl = (1u << lane) - 1u;
    uint32_t fin = 0;  // bit q: producer q has published the end of its items
    for (uint32_t k = 0; fin != (1u << kTP) - 1u; ++k) {
      if ((fin >> (k % kTP)) & 1u) continue;
      const int s = (int)(k % kTS);
      const uint32_t par = (k / kTS) & 1u;
      mbar_wait(&S.full[s], par);
      TStage& T = S.st[s];
      if (T.item == kTDone) {
        fin |= 1u << (k % kTP);
        continue;
      }
      mbar_wait(&S.xfull[s], par);
      const int x0 = T.x0, x = x0 + tc;
      const uint32_t cw = T.cw[tc];
      const bool fl = x < p.nx && !(cw & kNonFluid);
      if (!__any_sync(0xffffffffu, fl)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        continue;
      }
      const int z = T.z;
      int q[9];
      uint32_t bits = 0;  // bit r: the source row r has a fluid cell at this x (rows 0..4)
      uint32_t m0 = 0;
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const uint2 ri = T.rowinfo[r][c];
        q[r] = (int)ri.x + __popc(ri.y & ltl);
        if (r < 5) bits |= ((ri.y >> lane) & 1u) << r;
        if (r == 0) m0 = ri.y;
      }
      const uint32_t fc = T.own_rank[c] + __popc(m0 & ltl);
      double f[19];
      if (fl) {  // lanes past the row hold no valid run index
#pragma unroll
        for (int j = 0; j < 19; ++j) {
          const int r = trow_of(j);
          int idx = q[r];
          if (EX[j] == 1) idx -= 1;
          if (EX[j] == -1) idx += (bits >> r) & 1u;
          f[j] = T.pop[j][idx];
        }
      }
      if (p.px && (x == 0 || x == p.nx - 1)) {
#pragma unroll
        for (int r = 0; r < 5; ++r) {
          if (x == 0) f[wrap_plus(r)] = T.wrap[r];
          if (x == p.nx - 1) f[wrap_minus(r)] = T.wrap[5 + r];
        }
      }
      const int32_t l0 = T.lofs[c], l1 = T.lofs[c + 1];
      if (l1 > l0) {  // warp-uniform: this chunk has links
        if (RECORDS) {  // cooperative closures (boundary.cpp:24-41 in pull form)
          const int le = min(l1, kTLC);
          const uint16_t* dd = T.desc + T.descoff;
          for (int e = l0 + lane; e < le; e += 32) {
            const double rec = T.rec[T.recoff + e];
            if (rec == rec) {  // NaN: simple bounce-back, gk stays
              const uint32_t d = dd[e];
              const int owner = d & 31, j = d >> 5, kk = rt_opp(j);
              double v;
              if (!isinf(rec)) {
                // f_k(owner): its pull of direction k = opp(j) (x - e_k is fluid)
                const int r = rt_trow(kk), exk = rt_ex(kk);
                const int xo = x0 + c * 32 + owner;
                double fk;
                if (p.px && ((exk == 1 && xo == 0) || (exk == -1 && xo == p.nx - 1))) {
                  fk = T.wrap[(exk == 1 ? 0 : 5) + r];
                } else {
                  const uint2 ri = T.rowinfo[r][c];
                  int idx = (int)ri.x + __popc(ri.y & ((1u << owner) - 1u));
                  if (exk == 1) idx -= 1;
                  if (exk == -1) idx += (ri.y >> owner) & 1u;
                  fk = T.pop[kk][idx];
                }
                v = DADD(DSUB(DMUL(rec, fk), DMUL(rec, T.gj[e])), T.gk[e]);
              } else {
                v = DSUB(T.gk[e], p.mw[kk]);
              }
              T.gk[e] = v;
            }
          }
          __syncwarp();
        }
        const uint32_t bb = fl ? (cw & kBounceMask) : 0u;
        const uint32_t um = __reduce_or_sync(0xffffffffu, bb);
        int n = __popc(bb);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, n, o);
          if (lane >= o) n += t;
        }
        int pos = l0 + n - __popc(bb);
        const int32_t cb_lo = T.cb_lo;
        if (l1 <= kTLC) {
#pragma unroll
          for (int j = 1; j < 19; ++j) {
            if ((um >> j) & 1u) {
              if ((bb >> j) & 1u) f[j] = T.gk[pos];
              pos += (bb >> j) & 1u;
            }
          }
        } else {  // more links than the stage holds: the overflow closes from global memory
#pragma unroll
          for (int j = 1; j < 19; ++j) {
            if ((um >> j) & 1u) {
              if ((bb >> j) & 1u) {
                if (pos < kTLC) {
                  f[j] = T.gk[pos];
                } else {
                  const int kk = opp(j);
                  const double gk = __ldg(src + ((uint32_t)kk * ks + fc));
                  double v = gk;
                  if (RECORDS) {
                    const double rec = __ldg(p.links + cb_lo + pos);
                    if (rec == rec) {
                      if (!isinf(rec))
                        v = DADD(DSUB(DMUL(rec, f[kk]),
                                      DMUL(rec, __ldg(src + ((uint32_t)j * ks + fc)))),
                                 gk);
                      else
                        v = DSUB(gk, p.mw[kk]);
                    }
                  }
                  f[j] = v;
                }
              }
              pos += (bb >> j) & 1u;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);  // stage s consumed: the producer may refill it
      if (fl) {
        collide<CM, GLBM>(f, p, z);
#pragma unroll
        for (int j = 0; j < 19; ++j) __stcs(dst + (fc + p.poff[j]), f[j]);
      }
    }
  }

  // the last block to finish resets the work counter for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.tickets + 1, 1u) == gridDim.x - 1) {
      atomicExch(p.tickets, 0u);
      atomicExch(p.tickets + 1, 0u);
    }
  }
}

template <int CM, bool GLBM, bool RECORDS>
bool launch_tma_t(const KParams& p, const double* src, double* dst, cudaStream_t s) {
  const int nseg = (p.nchunk + kTNC - 1) / kTNC;
  const int64_t nitems = (int64_t)nseg * p.ny * p.nz;
  if (nitems == 0) return true;
  if (nitems > 0x7fffffff) return false;
  constexpr int smem = (int)sizeof(TSmem);
  static int grid_per_sm = [] {
    cudaFuncSetAttribute(k_sweep_tma<CM, GLBM, RECORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep_tma<CM, GLBM, RECORDS>, kTThreads, smem);
    return nb;
  }();
  if (grid_per_sm <= 0) return false;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::min<int64_t>(nitems, (int64_t)sms * grid_per_sm);
  const TDiv dseg{(uint32_t)nseg, 1.0 / nseg}, dny{(uint32_t)p.ny, 1.0 / p.ny};
  k_sweep_tma<CM, GLBM, RECORDS><<<(unsigned)g, kTThreads, smem, s>>>(p, src, dst, (uint32_t)nitems,
                                                                       dseg, dny);
  return true;
}

template <int CM>
bool tma_cm(bool glbm, bool records, const KParams& p, const double* src, double* dst,
            cudaStream_t s) {
  if (glbm)
    return records ? launch_tma_t<CM, true, true>(p, src, dst, s)
                   : launch_tma_t<CM, true, false>(p, src, dst, s);
  return records ? launch_tma_t<CM, false, true>(p, src, dst, s)
                 : launch_tma_t<CM, false, false>(p, src, dst, s);
}

}  // namespace

bool tma_sweep_supported(const SweepConfig& cfg, const KParams& p) {
  return p.ctab && !cfg.slab && cfg.part == PART_ALL && cfg.op == OP_STREAM_COLLIDE &&
         collide_mode(p) != CM_FAST_FOLD && p.nx % 4 == 0 && (p.linkdesc || !cfg.records);
}

bool launch_sweep_tma(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                      cudaStream_t s) {
  switch (collide_mode(p)) {
    case CM_FAST: return tma_cm<CM_FAST>(cfg.glbm, cfg.records, p, src, dst, s);
    case CM_EXACT_RHO1: return tma_cm<CM_EXACT_RHO1>(cfg.glbm, cfg.records, p, src, dst, s);
    case CM_EXACT: return tma_cm<CM_EXACT>(cfg.glbm, cfg.records, p, src, dst, s);
    default: return false;
  }
}

}  // namespace pgpu
