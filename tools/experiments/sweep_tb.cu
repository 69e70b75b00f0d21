// Two time steps per launch over the fluid-only layout (temporal blocking).
//
//   g(n+1) = C(P(g(n)))   step A: src (HBM) -> an L2-resident ring of planes
//   g(n+2) = C(P(g(n+1))) step B: ring -> dst (HBM)
//
// with the arithmetic of the one-step sweeps (pull form of the reference's
// push streaming + link bounce-back, simulation.cpp:278-342 and
// boundary.cpp:19-41; collide<CM, GLBM>, simulation.cpp:150-274), so every
// population is bit-identical to two one-step sweeps.  HBM sees the 152 B per
// cell that step A reads and the 152 B that step B writes: 152 B per cell
// update instead of 304.
//
// Schedule: a cooperative grid in which every warp owns one chunk column
// (row, 32-cell chunk) of a y-band and walks the phases A(0), A(1), A(2),
// B(0), A(3), B(1), ... with the one-step sweep's asynchronous-copy pipeline
// (meta three phases ahead, populations one phase ahead).  Warps synchronise
// only with their 3x3 neighbour columns through per-column progress
// counters: step B of plane z waits until the neighbours have finished step A
// of plane z+1; step A of plane z (ring slot z mod 5) waits until they have
// finished step B of plane z-4, the last reader of the slot's previous
// occupant.  The ring (5 planes of a band's step-A rows) stays in L2; step A
// also covers the band's two neighbouring rows (halo), computed by both
// bands.  z must not be periodic (the wavefront starts at z = 0).
//
// Status: selectable (pgpu_sweep_kernel TB2), bit-identical, and SLOWER than
// the one-step sweep (C4: 6.7 k vs 17 k fluid MLUPS).  Two
// findings: (1) the ring is rewritten during the launch and L1 is not
// coherent -- step-B reads through cp.async.ca saw stale L1 lines of a slot's
// previous occupant even after a GPU-scope fence (wrong results on the second
// band), so they are synchronous L2 loads (__ldcg) here; (2) the neighbour
// waits couple the warps into a lockstep wavefront whose per-phase latency,
// not HBM, bounds it.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "kparams.h"
#include "lattice.cuh"

namespace cg = cooperative_groups;

namespace pgpu {
namespace {

#ifndef PGPU_TB_SYNCRING
#define PGPU_TB_SYNCRING 1  // step-B ring reads as L2 loads (cp.async.ca would see stale L1 lines: see below)
#endif
constexpr int kTbW = 4;                 // warps per block
constexpr int kTbBX = 32 * kTbW;
constexpr int kTbSlots = 5;             // ring planes (step-A planes z-1 .. z+2 live + slack)
constexpr int kTbPool = 192;            // per-warp link extras (record + g_j(x) per link)
constexpr int kTbLinkCap = kTbPool / 2;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t tsm(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp8(void* d, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tsm(d)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp4(void* d, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(tsm(d)), "l"(g) : "memory");
}
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpwait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// source rows (as sweep_compact.cu): row r holds the directions with
// (e_y, e_z) = (row r)
__host__ __device__ constexpr int tw_row_of(int j) {
  return j <= 2 ? 0
         : (j == 3 || j == 7 || j == 10) ? 1
         : (j == 4 || j == 8 || j == 9)  ? 2
         : (j == 5 || j == 11 || j == 14) ? 3
         : (j == 6 || j == 12 || j == 13) ? 4
                                          : j - 10;
}
__device__ __forceinline__ int tw_row_ey(int r) {
  constexpr uint32_t t = (0 + 1) | (1 + 1) << 2 | (-1 + 1) << 4 | (0 + 1) << 6 | (0 + 1) << 8 |
                         (1 + 1) << 10 | (-1 + 1) << 12 | (1 + 1) << 14 | (-1 + 1) << 16;
  return (int)((t >> (2 * r)) & 3u) - 1;
}
__device__ __forceinline__ int tw_row_ez(int r) {
  constexpr uint32_t t = (0 + 1) | (0 + 1) << 2 | (0 + 1) << 4 | (1 + 1) << 6 | (-1 + 1) << 8 |
                         (1 + 1) << 10 | (-1 + 1) << 12 | (-1 + 1) << 14 | (1 + 1) << 16;
  return (int)((t >> (2 * r)) & 3u) - 1;
}

struct TbBand {
  int y0, y1;            // step-B rows [y0, y1)
  int ya0, nar;          // step-A rows ya0 .. ya0 + nar - 1 (wrapping)
  const int32_t* delta;  // [nz][nar]: ring row base - rank of the row's first fluid cell
};
struct TbParams {
  double* ring;
  int64_t cap;           // ring slots per plane slot
  int nband;
  TbBand band[8];
  uint32_t* prog;        // per band: [2][max columns] step A / step B planes done per column
  int maxcols;
  uint32_t poffr[19];    // j * ring direction stride (5 * cap)
};

struct alignas(16) TwMeta {  // one phase of one warp
  uint32_t cw[32];
  ChunkEnt ent[16];  // 0..8 source rows, 9..13 x-wrap partners of rows 0..4, 14/15 .rank link bases
  int32_t roff[10];  // ring offsets of the source rows (step B) and [9] of the own row
  int32_t z, kind;   // plane; kind 0 step A, 1 step B, -1 no phase
  uint16_t ldesc[kTbLinkCap + 2];
};
struct alignas(16) TwWarp {
  double main[19][32];
  double pool[kTbPool];
  uint32_t lw[32];     // cell word of the staged phase (| kNonFluid: skip)
  int32_t lfc[32];     // own slot of the staged phase in its source array
  int32_t cbase, z, kind, pad;
  TwMeta meta[3];
};

// warp `gw` of the grid: its column (A row index yl, chunk xc) in the band;
// phases: A(0), A(1), A(2), then (B(i), A(i+3)) pairs, then the last B's
__device__ __forceinline__ void tw_phase(int k, bool hasB, int nz, int& kind, int& z) {
  if (!hasB) {
    kind = k < nz ? 0 : -1;
    z = k;
    return;
  }
  if (k < 3) {
    kind = 0;
    z = k;
    return;
  }
  const int j = k - 3;
  if (j < 2 * (nz - 3)) {
    kind = (j & 1) ? 0 : 1;
    z = (j & 1) ? j / 2 + 3 : j / 2;
    return;
  }
  z = nz - 3 + (j - 2 * (nz - 3));
  kind = z < nz ? 1 : -1;
}

template <int CM, bool GLBM, bool RECORDS>
__global__ void __launch_bounds__(kTbBX, 4)
    k_sweep_tb2(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                const TbParams tp) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char tw_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TwWarp& S = reinterpret_cast<TwWarp*>(tw_raw)[warp];
  const int gw = blockIdx.x * kTbW + warp;
  const uint32_t ltl = (1u << lane) - 1u;
  const int nz = p.nz, nch = p.nchunk;
  const int64_t rs = 5 * tp.cap;
  for (int b = 0; b < tp.nband; ++b) {
    const TbBand& B = tp.band[b];
    const int ncol = B.nar * nch;
    uint32_t* progA = tp.prog + (size_t)b * 2 * tp.maxcols;
    uint32_t* progB = progA + tp.maxcols;
    if (gw < ncol) {
      const int yl = gw / nch, xc = gw - yl * nch;
      int y = B.ya0 + yl;
      if (y < 0) y += p.ny;
      if (y >= p.ny) y -= p.ny;
      const bool hasB = yl >= B.y0 - B.ya0 && yl < B.y0 - B.ya0 + (B.y1 - B.y0);
      const int x = xc * 32 + lane;
      const bool valid = x < p.nx;
      // the 9 neighbour columns (yl-1..yl+1, xc-1..xc+1; x periodic): lane n < 9
      int ncolidx = -1;
      bool nbB = false;  // the neighbour column has step-B rows
      if (lane < 9) {
        const int dy = lane / 3 - 1, dx = lane % 3 - 1;
        const int ny_ = yl + dy;
        int nx_ = xc + dx;
        if (nx_ < 0) nx_ = p.px ? nx_ + nch : -1;
        if (nx_ >= nch) nx_ = p.px ? nx_ - nch : -1;
        if (ny_ >= 0 && ny_ < B.nar && nx_ >= 0) {
          ncolidx = ny_ * nch + nx_;
          nbB = ny_ >= B.y0 - B.ya0 && ny_ < B.y0 - B.ya0 + (B.y1 - B.y0);
        }
      }
      // wait until every neighbour column has finished `need` planes of step A (B)
      auto wait_nb = [&](uint32_t* prog, int need, bool stepB) {
        if (lane < 9 && ncolidx >= 0 && (!stepB || nbB)) {
          const long long t0 = clock64();
          while ((int)ld_acquire(prog + ncolidx) < need) {
            __nanosleep(64);
            if (clock64() - t0 > 20000000000ll) __trap();
          }
        }
        // the ring is rewritten during the launch and L1 is not coherent: a
        // GPU-scope fence after the acquire invalidates this SM's L1 (CCTL.IVALL)
        // before the step-B copies (cp.async.ca) read the neighbours' planes
        if (!stepB && lane == 0) __threadfence();
        __syncwarp();
      };
      // per-lane chunk-entry offsets of this column that do not change with z
      int eoff = -1, rowl = -1;  // rowl: band row index of the lane's source row
      if (lane < 16) {
        if (lane < 14) {
          const int r = lane < 9 ? lane : lane - 9;
          int ys = y - tw_row_ey(r);
          bool ok = true;
          if (ys < 0 || ys >= p.ny) {
            if (p.py) ys = ys < 0 ? ys + p.ny : ys - p.ny;
            else ok = false;
          }
          const bool wrapchunk = xc == 0 || xc == nch - 1;
          if (ok && (lane < 9 || wrapchunk)) {
            eoff = ys * nch + (lane < 9 ? xc : (xc == 0 ? nch - 1 : 0));
            int l = ys - B.ya0;
            if (l < 0) l += p.ny;
            if (l >= p.ny) l -= p.ny;
            rowl = l;
          }
        } else if (RECORDS) {
          eoff = y * nch + xc;
        }
      }
      const int ownl = yl;
      auto meta_load = [&](int k, int m) {
        TwMeta& M = S.meta[m];
        int kind, z;
        tw_phase(k, hasB, nz, kind, z);
        if (lane == 0) {
          M.kind = kind;
          M.z = z;
        }
        if (kind < 0) return;
        if (valid)
          cp4(&M.cw[lane], p.cellw + ((int64_t)z * p.ny + y) * p.nx + x);
        else
          M.cw[lane] = kNonFluid;
        const int64_t plane = (int64_t)p.ny * nch;
        if (lane < 14) {
          const int zs = z - tw_row_ez(lane < 9 ? lane : lane - 9);
          const bool ok = zs >= 0 && zs < nz && eoff >= 0;
          if (ok) {
            cp8(&M.ent[lane], p.ctab + zs * plane + eoff);
            if (lane < 9) M.roff[lane] = (zs % kTbSlots) * (int32_t)tp.cap + B.delta[(int64_t)zs * B.nar + rowl];
          } else {
            M.ent[lane] = ChunkEnt{0u, 0u};
            if (lane < 9) M.roff[lane] = 0;
          }
        } else if (lane < 16) {
          if (eoff >= 0) cp4(&M.ent[lane].rank, p.chunkbase + z * plane + eoff + (lane - 14));
          else M.ent[lane] = ChunkEnt{0u, 0u};
        } else if (lane == 16) {
          M.roff[9] = (z % kTbSlots) * (int32_t)tp.cap + B.delta[(int64_t)z * B.nar + ownl];
        }
      };
      auto desc_load = [&](int m) {
        TwMeta& M = S.meta[m];
        if (M.kind < 0) return;
        const int32_t cb = (int32_t)M.ent[14].rank;
        const int n = min((int32_t)M.ent[15].rank - cb, kTbLinkCap);
        const int a0 = cb & ~1, npairs = (cb + n - a0 + 1) >> 1;
        for (int t = lane; t < npairs; t += 32) cp4(&M.ldesc[2 * t], p.linkdesc + a0 + 2 * t);
      };
      // stage the populations (and link extras) of the phase in meta slot m;
      // step B: after every neighbour finished the step-A planes it reads
      auto issue = [&](int m) -> int {
        const TwMeta& M = S.meta[m];
        const int kind = M.kind, z = M.z;
        if (lane == 0) {
          S.kind = kind;
          S.z = z;
        }
        if (kind < 0) {
          S.lw[lane] = kNonFluid;
          return 0;
        }
        if (kind == 1) wait_nb(progA, min(z + 2, nz), false);
        const bool ring = kind == 1;
        const double* base = ring ? tp.ring : src;
        const uint32_t cw = M.cw[lane];
        const bool fl = !(cw & kNonFluid);
        int q[9];
        uint32_t bits = 0;
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          const ChunkEnt e = M.ent[r];
          q[r] = (int)e.rank + __popc(e.mask & ltl) + (ring ? M.roff[r] : 0);
          if (r < 5) bits |= ((e.mask >> lane) & 1u) << r;
        }
        const int own_g = (int)M.ent[0].rank + __popc(M.ent[0].mask & ltl);
        const int fc = ring ? own_g + M.roff[9] : own_g;
        S.lw[lane] = cw;
        S.lfc[lane] = fc;
        if (lane == 0 && RECORDS) S.cbase = (int32_t)M.ent[14].rank;
        if (fl) {
          double* const st = &S.main[0][lane];
#pragma unroll
          for (int j = 0; j < 19; ++j) {
            const uint32_t pj = ring ? tp.poffr[j] : p.poff[j];
            uint32_t idx;
            if (j == 0) {
              idx = fc;
            } else if ((cw >> j) & 1u) {
              idx = fc + (ring ? tp.poffr[opp(j)] : p.poff[opp(j)]);
            } else if ((EX[j] == 1 && x == 0) || (EX[j] == -1 && x == p.nx - 1)) {
              // x-wrap: the partner chunk of the source row (same row and plane)
              const int r = tw_row_of(j);
              const ChunkEnt pe = M.ent[9 + r];
              const int xs = EX[j] == 1 ? p.nx - 1 : 0;
              idx = pe.rank + __popc(pe.mask & ((1u << (xs & 31)) - 1u)) + (ring ? M.roff[r] : 0) + pj;
            } else {
              const int r = tw_row_of(j);
              idx = q[r] + pj;
              if (EX[j] == 1) idx -= 1;
              if (EX[j] == -1) idx += (bits >> r) & 1u;
            }
            if (PGPU_TB_SYNCRING && ring) st[j * 32] = __ldcg(base + idx);
            else cp8(st + j * 32, base + idx);
          }
        }
        int total = 0;
        if (RECORDS) {
          const int32_t cb = (int32_t)M.ent[14].rank;
          total = (int32_t)M.ent[15].rank - cb;
          if (total) {
            const uint16_t* ld = M.ldesc + (cb & 1);
            const int nl = min(total, kTbLinkCap);
            __syncwarp();
            for (int e = lane; e < nl; e += 32) {
              const int d = ld[e];
              const int j = d >> 5, fco = S.lfc[d & 31];
              cp8(S.pool + 2 * e, p.links + cb + e);
              const double* ga = base + (uint32_t)(fco + (ring ? tp.poffr[j] : p.poff[j]));
              if (PGPU_TB_SYNCRING && ring) S.pool[2 * e + 1] = __ldcg(ga);
              else cp8(S.pool + 2 * e + 1, ga);
            }
          }
        }
        return total;
      };

      // prologue (cpipe's): meta of phases 0, 1; descriptors; issue 0; meta of 2
      meta_load(0, 0);
      meta_load(1, 1);
      cpcommit();
      cpwait0();
      __syncwarp();
      if (RECORDS) {
        desc_load(0);
        desc_load(1);
        cpcommit();
        cpwait0();
        __syncwarp();
      }
      int cnt_cur = issue(0);
      __syncwarp();
      meta_load(2, 2);
      cpcommit();
      int ms = 0;
      for (int k = 0;; ++k) {
        const int m1 = ms == 2 ? 0 : ms + 1;
        cpwait0();
        __syncwarp();
        if (RECORDS) desc_load(ms == 0 ? 2 : ms - 1);  // phase k+2's chunk bases landed
        const int kind = S.kind, z = S.z;
        if (kind < 0) break;
        if (RECORDS && cnt_cur) {  // cooperative link closures (boundary.cpp:24-41 in pull form)
          const bool ring = kind == 1;
          const uint16_t* ld = S.meta[ms].ldesc + (S.cbase & 1);
          const int ncoop = min(cnt_cur, kTbLinkCap);
          for (int e = lane; e < ncoop; e += 32) {
            const int d = ld[e];
            const int owner = d & 31, j = d >> 5, kk = (j & 1) ? j + 1 : j - 1;
            const double rec = S.pool[2 * e];
            if (rec == rec) {
              double* sj = &S.main[j][owner];
              if (!isinf(rec))
                *sj = DADD(DSUB(DMUL(rec, S.main[kk][owner]), DMUL(rec, S.pool[2 * e + 1])), *sj);
              else
                *sj = DSUB(*sj, p.mw[kk]);
            }
          }
          if (cnt_cur > kTbLinkCap) {  // past the pool: each lane closes its own remaining links
            const uint32_t w = S.lw[lane];
            const bool lf = !(w & kNonFluid);
            int n = lf ? __popc(w & kBounceMask) : 0, tot = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, tot, o);
              if (lane >= o) tot += t;
            }
            const int off = tot - n;
            uint32_t mm = lf ? (w & kBounceMask) : 0u;
            int c = 0;
            while (mm) {
              const int j = __ffs(mm) - 1;
              mm &= mm - 1;
              if (off + c >= kTbLinkCap) {
                const double rec2 = __ldg(p.links + S.cbase + off + c);
                if (rec2 == rec2) {
                  const int kk = (j & 1) ? j + 1 : j - 1;
                  double* sj = &S.main[j][lane];
                  const double* gb = (ring ? (const double*)tp.ring : src) +
                                     (uint32_t)(S.lfc[lane] + (ring ? tp.poffr[j] : p.poff[j]));
                  const double gj = ring ? __ldcg(gb) : __ldg(gb);
                  if (!isinf(rec2))
                    *sj = DADD(DSUB(DMUL(rec2, S.main[kk][lane]), DMUL(rec2, gj)), *sj);
                  else
                    *sj = DSUB(*sj, p.mw[kk]);
                }
              }
              ++c;
            }
          }
          __syncwarp();
        }
        const uint32_t w = S.lw[lane];
        const int fc = S.lfc[lane];
        const bool fluid = !(w & kNonFluid);
        double f[19];
        if (fluid) {
#pragma unroll
          for (int j = 0; j < 19; ++j) f[j] = S.main[j][lane];
        }
        const int own_ring = kind == 0 ? 0 : 0;
        (void)own_ring;
        int32_t roff_own = S.meta[ms].roff[9];
        int own_g = fc - (kind == 1 ? roff_own : 0);
        __syncwarp();
        cnt_cur = issue(m1);  // refill the stage with phase k+1
        __syncwarp();
        meta_load(k + 3, ms);
        cpcommit();
        if (fluid) collide<CM, GLBM>(f, p, z);
        if (kind == 0) {
          // step A into ring slot z % 5, once every neighbour has finished the
          // step-B planes that read its previous occupant
          wait_nb(progB, z - 3, true);
          if (fluid) {
#pragma unroll
            for (int j = 0; j < 19; ++j) __stcg(tp.ring + (uint32_t)(own_g + roff_own + tp.poffr[j]), f[j]);
          }
          __threadfence();
          __syncwarp();
          if (lane == 0) st_release(progA + gw, (uint32_t)(z + 1));
        } else {
          if (fluid) {
#pragma unroll
            for (int j = 0; j < 19; ++j) __stcs(dst + (uint32_t)(own_g + p.poff[j]), f[j]);
          }
          __syncwarp();
          if (lane == 0) st_release(progB + gw, (uint32_t)(z + 1));
        }
        ms = m1;
      }
      cpwait0();
    }
    grid.sync();  // the next band reuses the ring and the progress counters' slots
  }
}

// ring row bases of one band: delta[z][yl] = (fluid cells of the band's
// rows before yl in plane z) - (rank of row yl's first fluid cell)
__global__ void k_tb_delta(const KParams p, int ya0, int nar, int32_t* delta) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= p.nz) return;
  int32_t acc = 0;
  for (int yl = 0; yl < nar; ++yl) {
    int y = ya0 + yl;
    if (y < 0) y += p.ny;
    if (y >= p.ny) y -= p.ny;
    const ChunkEnt* row = p.ctab + ((int64_t)z * p.ny + y) * p.nchunk;
    delta[(int64_t)z * nar + yl] = acc - (int32_t)row[0].rank;
    const ChunkEnt last = row[p.nchunk - 1];
    acc += (int32_t)(last.rank + __popc(last.mask) - row[0].rank);
  }
}

constexpr int kTwSmem = kTbW * (int)sizeof(TwWarp);

template <int CM, bool GLBM, bool RECORDS>
int tb_capacity() {  // co-resident blocks of the cooperative launch
  static int g = [] {
    cudaFuncSetAttribute(k_sweep_tb2<CM, GLBM, RECORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTwSmem);
    int nb = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep_tb2<CM, GLBM, RECORDS>, kTbBX, kTwSmem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return nb * sms;
  }();
  return g;
}

template <int CM, bool GLBM, bool RECORDS>
cudaError_t launch_tb_t(const KParams& p, const double* src, double* dst, const TbParams& tp,
                        cudaStream_t s) {
  const int cap = tb_capacity<CM, GLBM, RECORDS>();
  const int blocks = (tp.maxcols + kTbW - 1) / kTbW;
  if (blocks > cap) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {(void*)&p, (void*)&src, (void*)&dst, (void*)&tp};
  return cudaLaunchCooperativeKernel((const void*)k_sweep_tb2<CM, GLBM, RECORDS>, dim3(blocks),
                                     dim3(kTbBX), args, kTwSmem, s);
}

template <int CM>
cudaError_t tb_dispatch(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                        const TbParams& tp, cudaStream_t s) {
  if (cfg.glbm)
    return cfg.records ? launch_tb_t<CM, true, true>(p, src, dst, tp, s)
                       : launch_tb_t<CM, true, false>(p, src, dst, tp, s);
  return cfg.records ? launch_tb_t<CM, false, true>(p, src, dst, tp, s)
                     : launch_tb_t<CM, false, false>(p, src, dst, tp, s);
}

}  // namespace

// Device buffers of the two-step sweep (owned by the simulation).
struct TbState {
  double* ring = nullptr;
  int64_t cap = 0;
  int32_t* delta = nullptr;
  uint32_t* prog = nullptr;
  size_t prog_bytes = 0;
  TbParams tp{};
  ~TbState() {
    cudaFree(ring);
    cudaFree(delta);
    cudaFree(prog);
  }
};

TbState* tb_create(const KParams& p, cudaStream_t s) {
  // y-bands: every step-A column of a band gets its own warp of the
  // cooperative grid (148 SMs x 16 warps), and the ring (5 planes of a band's
  // step-A rows) stays inside L2
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int warps = sms * 4 * kTbW;
  int nband = 2;
  while (nband < 8 && ((int64_t)(p.ny / nband + 3) * p.nchunk > warps)) ++nband;
  if (const char* e = std::getenv("PGPU_TB_BANDS")) nband = std::max(1, std::min(8, atoi(e)));
  if (p.py && nband < 2) nband = 2;  // a periodic band needs distinct halo rows
  nband = std::min(nband, p.ny);
  TbState* st = new TbState();
  TbParams& tp = st->tp;
  tp.nband = nband;
  int maxnar = 0;
  for (int b = 0; b < nband; ++b) {
    TbBand& B = tp.band[b];
    B.y0 = (int)((int64_t)p.ny * b / nband);
    B.y1 = (int)((int64_t)p.ny * (b + 1) / nband);
    if (p.py) {
      B.ya0 = B.y0 - 1;
      B.nar = B.y1 - B.y0 + 2;
    } else {
      B.ya0 = std::max(B.y0 - 1, 0);
      B.nar = std::min(B.y1 + 1, p.ny) - B.ya0;
    }
    maxnar = std::max(maxnar, B.nar);
  }
  tp.maxcols = maxnar * p.nchunk;
  st->cap = ((int64_t)maxnar * p.nx + 31) / 32 * 32;
  for (int j = 0; j < 19; ++j) tp.poffr[j] = (uint32_t)(j * kTbSlots * st->cap);
  int64_t dtotal = 0;
  for (int b = 0; b < nband; ++b) dtotal += (int64_t)p.nz * tp.band[b].nar;
  st->prog_bytes = sizeof(uint32_t) * 2 * (size_t)nband * tp.maxcols;
  bool ok = 19 * kTbSlots * st->cap < (int64_t)UINT32_MAX &&
            cudaMalloc(&st->ring, sizeof(double) * 19 * kTbSlots * (size_t)st->cap) == cudaSuccess &&
            cudaMalloc(&st->delta, sizeof(int32_t) * (size_t)dtotal) == cudaSuccess &&
            cudaMalloc(&st->prog, st->prog_bytes) == cudaSuccess;
  if (!ok) {
    delete st;
    cudaGetLastError();
    return nullptr;
  }
  int64_t off = 0;
  for (int b = 0; b < nband; ++b) {
    TbBand& B = tp.band[b];
    B.delta = st->delta + off;
    k_tb_delta<<<(p.nz + 127) / 128, 128, 0, s>>>(p, B.ya0, B.nar, st->delta + off);
    off += (int64_t)p.nz * B.nar;
  }
  tp.ring = st->ring;
  tp.cap = st->cap;
  tp.prog = st->prog;
  return st;
}

void tb_destroy(TbState* st) { delete st; }

int64_t tb_device_bytes(const TbState* st) {
  if (!st) return 0;
  int64_t d = 0;
  for (int b = 0; b < st->tp.nband; ++b) d += st->tp.band[b].nar;
  return 19 * kTbSlots * st->cap * 8 + (int64_t)st->prog_bytes + d * 4;
}

bool tb_supported(const SweepConfig& cfg, const KParams& p) {
  return p.ctab && !cfg.slab && cfg.part == PART_ALL && cfg.op == OP_STREAM_COLLIDE && !p.pz &&
         collide_mode(p) != CM_FAST_FOLD && p.nz >= 4 && (p.linkdesc || !cfg.records);
}

// g(n+2) = C(P(C(P(g(n))))) from src into dst; false: not launchable here
bool launch_sweep_tb2(const SweepConfig& cfg, const KParams& p, TbState* st, const double* src,
                      double* dst, cudaStream_t s) {
  if (!st) return false;
  TbParams tp = st->tp;
  if (cudaMemsetAsync(st->prog, 0, st->prog_bytes, s) != cudaSuccess) return false;
  cudaError_t e;
  switch (collide_mode(p)) {
    case CM_FAST: e = tb_dispatch<CM_FAST>(cfg, p, src, dst, tp, s); break;
    case CM_EXACT_RHO1: e = tb_dispatch<CM_EXACT_RHO1>(cfg, p, src, dst, tp, s); break;
    case CM_EXACT: e = tb_dispatch<CM_EXACT>(cfg, p, src, dst, tp, s); break;
    default: return false;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

}  // namespace pgpu
