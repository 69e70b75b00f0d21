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
// Schedule: a cooperative grid sweeps a wavefront along z.  In round t every
// block computes step A on plane t and then step B on plane t-2 (which needs
// the step-A planes t-3 .. t-1).  Per-plane completion counters order the
// grid: step B of plane t-2 waits until every block has finished step A of
// plane t-1, and step A of plane t (which reuses ring slot t mod 4) waits until
// every block has finished step B of plane t-3.  Both waits have a round of
// slack.  To keep the ring in L2 (4 planes) the domain is processed in y-bands;
// step A also covers the band's two neighbouring rows (halo), computed by
// both bands (bit-identical either way).  z must not be periodic (the
// wavefront starts at z = 0).
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

constexpr int kTbBX = 128;  // cells per block-column (one row segment)

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// every block: wait until *ctr >= target (one thread spins; bounded: a lost
// signal traps instead of hanging the device)
__device__ __forceinline__ void tb_wait(const uint32_t* ctr, uint32_t target) {
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    while (ld_acquire(ctr) < target) {
      __nanosleep(100);
      if (clock64() - t0 > 20000000000ll) __trap();
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void tb_signal(uint32_t* ctr) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(ctr, 1u);
}

template <bool RING>
__device__ __forceinline__ double tb_ld(const double* a) {
  if (RING) return __ldcg(a);  // written by this launch: coherent (L2) loads
  return __ldg(a);
}

// Pull source addresses of one fluid cell.  Step A reads src (the compact
// state, plane j at j * ks); step B reads the ring: direction plane j at
// j * RS, plane slot z & 3 at (z & 3) * cap, row ys of the band at its
// fluid-slot rank + delta[z][row of the band].
struct TbRing {
  double* base;
  int64_t cap, rs;      // slots per ring plane slot, per direction (4 * cap)
  const int32_t* delta;  // [nz][nar]: ring row base - row start rank
  int ya0, nar;          // first ring row (may be -1: wraps), rows
};

// ring index of the cell whose compact slot (global rank) is s, in row y, plane z
__device__ __forceinline__ int64_t tb_ring_index(const KParams& p, const TbRing& R, int64_t s, int y,
                                                 int z) {
  int yl = y - R.ya0;
  if (yl < 0) yl += p.ny;
  if (yl >= p.ny) yl -= p.ny;
  return (int64_t)(z & 3) * R.cap + s + R.delta[(int64_t)z * R.nar + yl];
}
template <bool RING>
__device__ __forceinline__ int64_t tb_slot(const KParams& p, const TbRing& R, int x, int y, int z) {
  const int64_t s = compact_slot(p, x, y, z);
  return RING ? tb_ring_index(p, R, s, y, z) : s;
}

template <int J, bool RING>
__device__ __forceinline__ void tb_load_all(double (&f)[19], const KParams& p, const TbRing& R,
                                            const double* __restrict__ src, int x, int y, int z,
                                            int64_t own, uint32_t w) {
  if constexpr (J < 19) {
    const int64_t stride = RING ? R.rs : p.ks;
    const double* base = RING ? R.base : src;
    constexpr int ex = EX[J], ey = EY[J], ez = EZ[J];
    int64_t a;
    if (J == 0) {
      a = own;
    } else if ((w >> J) & 1u) {
      a = (int64_t)opp(J) * stride + own;  // bounce: g_k(x)
    } else {
      int xs = x - ex, ys = y - ey;
      const int zs = z - ez;  // z is not periodic; a pulled source is fluid, so in range
      if (xs < 0) xs += p.nx;
      if (xs >= p.nx) xs -= p.nx;
      if (ys < 0) ys += p.ny;
      if (ys >= p.ny) ys -= p.ny;
      a = (int64_t)J * stride + tb_slot<RING>(p, R, xs, ys, zs);
    }
    f[J] = tb_ld<RING>(base + a);
    tb_load_all<J + 1, RING>(f, p, R, src, x, y, z, own, w);
  }
}

// CLI / moving-wall closures (boundary.cpp:24-41 in pull form); f[J] holds g_k(x)
template <int J, bool RING>
__device__ __forceinline__ void tb_links_all(double (&f)[19], const KParams& p, const TbRing& R,
                                             const double* __restrict__ src, int64_t own,
                                             uint32_t w, int32_t base) {
  if constexpr (J < 19) {
    if ((w >> J) & 1u) {
      constexpr int K = opp(J);
      const int32_t r = base + __popc(w & ((1u << J) - 1u) & kBounceMask);
      const double rec = __ldg(p.links + r);
      if (rec == rec) {
        if (!isinf(rec)) {
          const double gj = tb_ld<RING>((RING ? R.base : src) + (int64_t)J * (RING ? R.rs : p.ks) + own);
          f[J] = DADD(DSUB(DMUL(rec, f[K]), DMUL(rec, gj)), f[J]);
        } else {
          f[J] = DSUB(f[J], p.mw[K]);
        }
      }
    }
    tb_links_all<J + 1, RING>(f, p, R, src, own, w, base);
  }
}

// One cell of step A (RING = false: src -> ring) or B (true: ring -> dst).
template <int CM, bool GLBM, bool RECORDS, bool RING>
__device__ __forceinline__ void tb_cell(const KParams& p, const TbRing& R,
                                        const double* __restrict__ src, double* __restrict__ dst,
                                        int x, int y, int z) {
  const int64_t c = ((int64_t)z * p.ny + y) * p.nx + x;
  const uint32_t w = __ldg(p.cellw + c);
  if (w & kNonFluid) return;
  const int64_t g = compact_slot(p, x, y, z);  // the cell's slot in src / dst
  const int64_t ring_own = tb_ring_index(p, R, g, y, z);
  const int64_t own_src = RING ? ring_own : g;  // where this cell's own populations are read
  double f[19];
  tb_load_all<0, RING>(f, p, R, src, x, y, z, own_src, w);
  if (RECORDS && (w & kBounceMask)) tb_links_all<1, RING>(f, p, R, src, own_src, w, __ldg(p.cellbase + c));
  collide<CM, GLBM>(f, p, z);
  if (!RING) {  // step A: into the ring
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcg(R.base + (int64_t)j * R.rs + ring_own, f[j]);
  } else {  // step B: the new state, streamed to HBM
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcs(dst + (int64_t)j * p.ks + g, f[j]);
  }
}

struct TbBand {
  int y0, y1;            // step-B rows [y0, y1)
  int ya0, nar;          // step-A rows ya0 .. ya0 + nar - 1 (wrapping)
  const int32_t* delta;  // [nz][nar]
};
struct TbParams {
  double* ring;
  int64_t cap;
  int nband;
  TbBand band[8];
  uint32_t* ctr;  // [nband][2][nz] completion counters (zero at launch)
  int nseg;
};

template <int CM, bool GLBM, bool RECORDS>
__global__ void __launch_bounds__(kTbBX, 4)
    k_sweep_tb2(const KParams p, const double* __restrict__ src, double* __restrict__ dst,
                const TbParams tp) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, nz = p.nz, nseg = tp.nseg;
  for (int b = 0; b < tp.nband; ++b) {
    const TbBand& B = tp.band[b];
    const TbRing R{tp.ring, tp.cap, 4 * tp.cap, B.delta, B.ya0, B.nar};
    const uint32_t numA = (uint32_t)(B.nar * nseg), numB = (uint32_t)((B.y1 - B.y0) * nseg);
    uint32_t* doneA = tp.ctr + (size_t)b * 2 * nz;
    uint32_t* doneB = doneA + nz;
    for (int t = 0; t < nz + 2; ++t) {
      if (t < nz) {
        if (t >= 3) tb_wait(&doneB[t - 3], numB);  // ring slot t & 3 is free again
        for (uint32_t col = blockIdx.x; col < numA; col += G) {
          const int yl = (int)(col / nseg), xb = (int)(col % nseg);
          int y = B.ya0 + yl;
          if (y < 0) y += p.ny;
          if (y >= p.ny) y -= p.ny;
          const int x = xb * kTbBX + threadIdx.x;
          if (x < p.nx) tb_cell<CM, GLBM, RECORDS, false>(p, R, src, dst, x, y, t);
          tb_signal(&doneA[t]);
        }
      }
      if (t >= 2) {
        const int zb = t - 2;
        tb_wait(&doneA[min(zb + 1, nz - 1)], numA);  // step-A planes zb-1 .. zb+1 everywhere
        for (uint32_t col = blockIdx.x; col < numB; col += G) {
          const int yl = (int)(col / nseg), xb = (int)(col % nseg);
          const int y = B.y0 + yl;
          const int x = xb * kTbBX + threadIdx.x;
          if (x < p.nx) tb_cell<CM, GLBM, RECORDS, true>(p, R, src, dst, x, y, zb);
          tb_signal(&doneB[zb]);
        }
      }
    }
    grid.sync();  // the next band reuses the ring
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

template <int CM, bool GLBM, bool RECORDS>
cudaError_t launch_tb_t(const KParams& p, const double* src, double* dst, const TbParams& tp,
                        int grid, cudaStream_t s) {
  void* args[] = {(void*)&p, (void*)&src, (void*)&dst, (void*)&tp};
  return cudaLaunchCooperativeKernel((const void*)k_sweep_tb2<CM, GLBM, RECORDS>, dim3(grid),
                                     dim3(kTbBX), args, 0, s);
}

template <int CM, bool GLBM, bool RECORDS>
int tb_grid() {
  static int g = [] {
    int nb = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep_tb2<CM, GLBM, RECORDS>, kTbBX, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return nb * sms;
  }();
  return g;
}

template <int CM>
cudaError_t tb_dispatch(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                        const TbParams& tp, cudaStream_t s) {
  if (cfg.glbm)
    return cfg.records ? launch_tb_t<CM, true, true>(p, src, dst, tp, tb_grid<CM, true, true>(), s)
                       : launch_tb_t<CM, true, false>(p, src, dst, tp, tb_grid<CM, true, false>(), s);
  return cfg.records ? launch_tb_t<CM, false, true>(p, src, dst, tp, tb_grid<CM, false, true>(), s)
                     : launch_tb_t<CM, false, false>(p, src, dst, tp, tb_grid<CM, false, false>(), s);
}

}  // namespace

// Device buffers of the two-step sweep (owned by the simulation).
struct TbState {
  double* ring = nullptr;
  int64_t cap = 0;
  int32_t* delta = nullptr;
  uint32_t* ctr = nullptr;
  TbParams tp{};
  ~TbState() {
    cudaFree(ring);
    cudaFree(delta);
    cudaFree(ctr);
  }
};

TbState* tb_create(const KParams& p, cudaStream_t s) {
  // bands of at most `rows` rows: the ring (4 planes of a band's step-A rows)
  // stays well inside L2
  const int nseg = (p.nchunk * 32 + kTbBX - 1) / kTbBX;
  int nband = 2;
  if (const char* e = std::getenv("PGPU_TB_BANDS")) nband = std::max(1, std::min(8, atoi(e)));
  if (p.py && nband < 2) nband = 2;  // a periodic band needs distinct halo rows
  nband = std::min(nband, p.ny);
  TbState* st = new TbState();
  TbParams& tp = st->tp;
  tp.nseg = nseg;
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
  st->cap = ((int64_t)maxnar * p.nx + 31) / 32 * 32;
  int64_t dtotal = 0;
  for (int b = 0; b < nband; ++b) dtotal += (int64_t)p.nz * tp.band[b].nar;
  bool ok = cudaMalloc(&st->ring, sizeof(double) * 19 * 4 * (size_t)st->cap) == cudaSuccess &&
            cudaMalloc(&st->delta, sizeof(int32_t) * (size_t)dtotal) == cudaSuccess &&
            cudaMalloc(&st->ctr, sizeof(uint32_t) * 2 * (size_t)nband * p.nz) == cudaSuccess;
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
  tp.ctr = st->ctr;
  return st;
}

void tb_destroy(TbState* st) { delete st; }

int64_t tb_device_bytes(const TbState* st) {
  if (!st) return 0;
  int64_t d = 0;
  for (int b = 0; b < st->tp.nband; ++b) d += st->tp.band[b].nar;
  return 19 * 4 * st->cap * 8 + 2 * (int64_t)st->tp.nband * 4 + d * 4;
}

bool tb_supported(const SweepConfig& cfg, const KParams& p) {
  return p.ctab && !cfg.slab && cfg.part == PART_ALL && cfg.op == OP_STREAM_COLLIDE && !p.pz &&
         collide_mode(p) != CM_FAST_FOLD && p.nz >= 4;
}

// g(n+2) = C(P(C(P(g(n))))) from src into dst; false: not launchable here
bool launch_sweep_tb2(const SweepConfig& cfg, const KParams& p, TbState* st, const double* src,
                      double* dst, cudaStream_t s) {
  if (!st) return false;
  TbParams tp = st->tp;
  if (cudaMemsetAsync(st->ctr, 0, sizeof(uint32_t) * 2 * (size_t)tp.nband * p.nz, s) != cudaSuccess)
    return false;
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
