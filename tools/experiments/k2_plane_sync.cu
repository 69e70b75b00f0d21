// EXPERIMENT (not built; measured once and kept for the next round): two
// time steps per launch over the fluid-only layout -- temporal blocking
// through an L2-resident ring.  It was wired into pgpu_sim::step() behind
// PGPU_K2=1 (ring of 4 planes, per-plane first rank `pbase`, in-place
// update) and reproduced two K1 steps bit for bit (96x40x48 sphere bed, SBB,
// 21 steps), but ran C4 SBB at 4.6 k MLUPS against 18.4 k for the one-step
// sweep: with a grid barrier per plane round (514 per launch) and
// synchronous per-item loads (chunk entries, then populations) every round
// exposes two memory latencies and the barrier (~43 us per round).  A viable
// version needs neighbour-progress flags instead of grid barriers and the
// cp.async z-march pipeline of k_sweep_cpipe within each warp.
//
// One cooperative launch.  In round r every warp sweeps
//   phase A: plane r   of step n   (buffer f   -> ring slot r mod 4)
//   phase B: plane r-2 of step n+1 (ring       -> buffer f, in place)
// then a grid barrier.  Phase B of round r writes plane r-2 of f while phase A
// of later rounds reads planes >= r-1, so the update is in place.  Ring plane
// z holds the fluid cells of plane z at (z mod 4) * cap + (rank - pbase[z]).
// Per-cell arithmetic is the K1 arithmetic (collide_core, pull form), so the
// result is bit-identical to two K1 sweeps.  Scope of the experiment: core
// collision, no link records (SBB walls), no slab, non-periodic z, x wrap
// through the chunk table.  Each warp handles one 32-cell chunk of a row per
// item with direct (register) loads; no intra-warp pipeline.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.h"
#include "kparams.h"
#include "lattice.cuh"

namespace pgpu {
namespace {
namespace cg = cooperative_groups;

constexpr int kRing = 4;
#ifndef PGPU_K2_MINB
#define PGPU_K2_MINB 3
#endif

__device__ __forceinline__ int row_ey2(int r) {
  return (r == 1 || r == 5 || r == 7) ? 1 : ((r == 2 || r == 6 || r == 8) ? -1 : 0);
}
__device__ __forceinline__ int row_ez2(int r) {
  return (r == 3 || r == 5 || r == 8) ? 1 : ((r == 4 || r == 6 || r == 7) ? -1 : 0);
}
__host__ __device__ constexpr int row_of2(int j) {
  return j <= 2 ? 0
         : (j == 3 || j == 7 || j == 10) ? 1
         : (j == 4 || j == 8 || j == 9)  ? 2
         : (j == 5 || j == 11 || j == 14) ? 3
         : (j == 6 || j == 12 || j == 13) ? 4
                                          : j - 10;
}

struct K2Args {
  double* f;            // sweep buffer (in place)
  double* ring;         // [19][kRing * cap]
  const int32_t* pbase; // first fluid rank of each plane (nz + 1)
  int32_t cap;          // fluid cells per ring plane (max over planes)
};

// slot offset of a compact rank of plane zs in the buffer being read
template <bool FROM_RING>
__device__ __forceinline__ int64_t src_slot(const K2Args& a, int64_t rank, int zs) {
  if (!FROM_RING) return rank;
  return (int64_t)(zs & (kRing - 1)) * a.cap + (rank - a.pbase[zs]);
}

template <bool RHO1, bool FROM_RING>
__device__ __forceinline__ void k2_item(const KParams& p, const K2Args& a, int z, int y, int xc,
                                        int lane) {
  const int x = xc * 32 + lane;
  const bool valid = x < p.nx;
  const int64_t row = (int64_t)z * p.ny + y;
  const ChunkEnt e0 = p.ctab[row * p.nchunk + xc];
  const uint32_t ltl = (1u << lane) - 1u;
  const bool fluid = valid && ((e0.mask >> lane) & 1u);
  // entries of the 9 source rows (uniform loads)
  int q[9];
  uint32_t bits = 0;
  int zsr[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    int ys = y - row_ey2(r), zs = z - row_ez2(r);
    if (ys < 0) ys += p.ny;
    if (ys >= p.ny) ys -= p.ny;
    zs = min(max(zs, 0), p.nz - 1);  // non-periodic z: out-of-range rows are never pulled
    zsr[r] = zs;
    const ChunkEnt e = p.ctab[((int64_t)zs * p.ny + ys) * p.nchunk + xc];
    q[r] = (int)e.rank + __popc(e.mask & ltl);
    if (r < 5) bits |= ((e.mask >> lane) & 1u) << r;
  }
  if (!fluid) return;
  const uint32_t w = __ldg(p.cellw + row * p.nx + x);
  const double* src = FROM_RING ? a.ring : a.f;
  const int64_t ps = FROM_RING ? (int64_t)kRing * a.cap : p.ks;  // plane stride
  const int64_t fc = q[0];
  const int64_t own = src_slot<FROM_RING>(a, fc, z);
  double f[19];
#pragma unroll
  for (int j = 0; j < 19; ++j) {
    int64_t slot;
    if (j == 0) {
      slot = own;
    } else if ((w >> j) & 1u) {
      f[j] = __ldcg(src + (int64_t)opp(j) * ps + own);  // bounce: g_k(x)
      continue;
    } else {
      const int r = row_of2(j);
      int64_t rk;
      if ((EX[j] == 1 && x == 0) || (EX[j] == -1 && x == p.nx - 1)) {  // periodic x partner
        int ys = y - EY[j], zs = z - EZ[j];
        if (ys < 0) ys += p.ny;
        if (ys >= p.ny) ys -= p.ny;
        const int xs = EX[j] == 1 ? p.nx - 1 : 0;
        const ChunkEnt pe = p.ctab[((int64_t)zs * p.ny + ys) * p.nchunk + (xs >> 5)];
        rk = (int64_t)pe.rank + __popc(pe.mask & ((1u << (xs & 31)) - 1u));
      } else {
        rk = q[r];
        if (EX[j] == 1) rk -= 1;
        if (EX[j] == -1) rk += (bits >> r) & 1u;
      }
      slot = src_slot<FROM_RING>(a, rk, zsr[r]);
    }
    f[j] = __ldcg(src + (int64_t)j * ps + slot);
  }
  collide_core<RHO1>(f, p);
  if (!FROM_RING) {  // phase A: into the ring
    double* d = a.ring + src_slot<true>(a, fc, z);
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcg(d + (int64_t)j * kRing * a.cap, f[j]);
  } else {  // phase B: into the buffer, in place
    double* d = a.f + fc;
#pragma unroll
    for (int j = 0; j < 19; ++j) __stcs(d + (int64_t)j * p.ks, f[j]);
  }
}

template <bool RHO1>
__global__ void __launch_bounds__(128, PGPU_K2_MINB) k_sweep_k2(const KParams p, const K2Args a) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ni = (int64_t)p.ny * p.nchunk;
  for (int r = 0; r < p.nz + 2; ++r) {
    if (r < p.nz)
      for (int64_t i = gw; i < ni; i += W)
        k2_item<RHO1, false>(p, a, r, (int)(i / p.nchunk), (int)(i % p.nchunk), lane);
    if (r >= 2)
      for (int64_t i = gw; i < ni; i += W)
        k2_item<RHO1, true>(p, a, r - 2, (int)(i / p.nchunk), (int)(i % p.nchunk), lane);
    grid.sync();
  }
}

}  // namespace

// Returns 0 on launch, -1 if not launchable (caller falls back to K1 steps).
int launch_sweep_k2(const KParams& p, double* f, double* ring, const int32_t* pbase, int32_t cap,
                    cudaStream_t s) {
  auto kern = p.rho0 == 1.0 ? k_sweep_k2<true> : k_sweep_k2<false>;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  if (per_sm < 1) return -1;
  K2Args a{f, ring, pbase, cap};
  KParams pp = p;
  void* args[] = {(void*)&pp, (void*)&a};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(sms * per_sm), dim3(128), args, 0, s) ==
                 cudaSuccess
             ? 0
             : -1;
}

}  // namespace pgpu
