// Device-side construction of the sweep's link structures (pgpu_create,
// simulation.cpp:80-102): from the caller's flag field and link list, uploaded
// once, sm_100a kernels build
//   * the per-cell words (bit0 non-fluid + flag byte, bits 1..18 "f_j comes
//     from a link", bit19 sector fill) -- the fluid->non-fluid test of
//     geometry.cpp:574-591 in pull form, with the periodic / open / ghost-column
//     rules of the host voxelizer;
//   * the per-cell and per-32-cell-chunk record bases (exclusive scan);
//   * one record per link (CLI coefficient c = (1-2q)/(1+2q) from the fp32 q,
//     boundary.cpp:27-28, NaN = SBB, +inf = moving wall) after validating that
//     the links close exactly the fluid->non-fluid directions.
// Replaces a multi-threaded host pass plus the upload of its results: the
// host only moves the caller's arrays (flags 1 B/cell, links 25 B/link).
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "kparams.h"
#include "setup.h"

namespace pgpu {
namespace {

__constant__ int8_t cE[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},   {0, -1, 0},
                                 {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                                 {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                                 {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};

__device__ __forceinline__ int dopp(int k) { return k == 0 ? 0 : ((k & 1) ? k + 1 : k - 1); }

__device__ __forceinline__ int dwrap(int v, int n, bool periodic) {
  if (v >= 0 && v < n) return v;
  if (!periodic) return -1;
  return (v % n + n) % n;
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                                                 cudaGetErrorString(e));
}

// One thread per cell; grid (x blocks, y, z).
__global__ void k_cellwords(const uint8_t* __restrict__ flags, const uint8_t* __restrict__ glo,
                            const uint8_t* __restrict__ ghi, int nx, int ny, int nz, bool px,
                            bool py, bool pz, bool slab, uint32_t* __restrict__ cellw,
                            int32_t* __restrict__ count) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= nx) return;
  const int64_t c = ((int64_t)z * ny + y) * nx + x;
  const uint8_t own = flags[c];
  if (own != 0) {
    cellw[c] = kNonFluid | ((uint32_t)own << kFlagShift);
    count[c] = 0;
    return;
  }
  uint32_t w = 0;
#pragma unroll
  for (int j = 1; j < 19; ++j) {
    const int ys = dwrap(y - cE[j][1], ny, py);
    const int zs = dwrap(z - cE[j][2], nz, pz);
    bool nonfluid;
    if (ys < 0 || zs < 0) {
      nonfluid = true;
    } else {
      const int xr = x - cE[j][0];
      if (slab && xr < 0) {
        nonfluid = glo[(int64_t)zs * ny + ys] != 0;
      } else if (slab && xr >= nx) {
        nonfluid = ghi[(int64_t)zs * ny + ys] != 0;
      } else {
        const int xs = slab ? xr : dwrap(xr, nx, px);
        nonfluid = xs < 0 || flags[((int64_t)zs * ny + ys) * nx + xs] != 0;
      }
    }
    if (nonfluid) w |= 1u << j;
  }
  cellw[c] = w;
  count[c] = __popc(w & kBounceMask);
}

// Non-fluid cells sharing an aligned 4-cell (32-byte) group with a fluid cell.
__global__ void k_fill_sectors(uint32_t* __restrict__ cellw, int64_t cells) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c0 = g * 4;
  if (c0 >= cells) return;
  const int64_t c1 = c0 + 4 < cells ? c0 + 4 : cells;
  bool anyfluid = false;
  for (int64_t c = c0; c < c1; ++c) anyfluid |= !(cellw[c] & kNonFluid);
  if (!anyfluid) return;
  for (int64_t c = c0; c < c1; ++c)
    if (cellw[c] & kNonFluid) cellw[c] |= kFillSector;
}

// chunkbase[rows * nchunk] is a sentinel = the link total, so a chunk's link
// count is chunkbase[i + 1] - chunkbase[i].
__global__ void k_chunkbase(const int32_t* __restrict__ base, int32_t* __restrict__ chunkbase,
                            int nx, int64_t rows, int nchunk, const int64_t* __restrict__ total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == rows * nchunk) chunkbase[i] = (int32_t)*total;
  if (i >= rows * nchunk) return;
  const int64_t r = i / nchunk;
  const int ch = (int)(i - r * nchunk);
  chunkbase[i] = base[r * nx + ch * 32];
}

struct ToI64 {
  __host__ __device__ int64_t operator()(int32_t v) const { return v; }
};

// One thread per input link (validation as pgpu_create's contract, records).
__global__ void k_links(LinkSetupArgs a, uint32_t* __restrict__ seen,
                        unsigned long long* __restrict__ err,
                        unsigned long long* __restrict__ fallbacks, int* __restrict__ moving_any) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool fb = false, mv = false;
  int code = 0;
  if (i < a.n_links) {
    const int64_t c = a.link_cell[i];
    const int k = a.link_dir[i];
    if (c < 0 || c >= a.cells || (a.cellw[c] & kNonFluid)) {
      code = kSetupErrCell;
    } else if (k < 1 || k > 18) {
      code = kSetupErrDir;
    } else {
      const int j = dopp(k);
      const uint32_t w = a.cellw[c];
      if (!((w >> j) & 1u)) {
        code = kSetupErrFluidNeighbour;
      } else {
        const int64_t r = (int64_t)a.cellbase[c] + __popc(w & ((1u << j) - 1u) & kBounceMask);
        const uint32_t bit = 1u << (r & 31);
        if (atomicOr(&seen[r >> 5], bit) & bit) {
          code = kSetupErrDuplicate;
        } else {
          const int64_t sf = a.link_second[i];
          mv = a.link_moving && a.link_moving[i];
          fb = a.cli && sf == -1;  // simulation.cpp:97-101
          double rec = __longlong_as_double(0x7FF8000000000000ll);  // SBB
          if (mv) {
            rec = __longlong_as_double(0x7FF0000000000000ll);  // +inf
          } else if (a.cli && sf != -1) {
            if ((w >> k) & 1u) {
              code = kSetupErrSecondNotFluid;
            } else {
              const int nx = a.nx, ny = a.ny, nz = a.nz;
              const int x = (int)(c % nx), y = (int)((c / nx) % ny),
                        z = (int)(c / ((int64_t)nx * ny));
              const int xr = x - cE[k][0];
              const int ys = dwrap(y - cE[k][1], ny, a.py);
              const int zs = dwrap(z - cE[k][2], nz, a.pz);
              bool ok;
              if (a.slab && (xr < 0 || xr >= nx)) {
                ok = sf == -2;
              } else {
                const int xs = a.slab ? xr : dwrap(xr, nx, a.px);
                ok = sf == ((int64_t)zs * ny + ys) * nx + xs;
              }
              if (!ok) code = kSetupErrSecondCell;
              // boundary.cpp:27-28 from the fp32 q, round-to-nearest each op
              const double q = (double)a.link_q[i];
              rec = __ddiv_rn(__dsub_rn(1.0, __dmul_rn(2.0, q)), __dadd_rn(1.0, __dmul_rn(2.0, q)));
            }
          }
          if (a.recs) a.recs[r] = rec;
        }
      }
    }
  }
  if (code) atomicMin(err, ((unsigned long long)i << 8) | (unsigned long long)code);
  const unsigned m = __activemask();
  const unsigned bf = __ballot_sync(m, fb), bm = __ballot_sync(m, mv);
  if ((threadIdx.x & 31) == (__ffs(m) - 1)) {
    if (bf) atomicAdd(fallbacks, (unsigned long long)__popc(bf));
    if (bm) atomicOr(moving_any, 1);
  }
}

__global__ void k_fill_nan(double* __restrict__ recs, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) recs[i] = __longlong_as_double(0x7FF8000000000000ll);
}

// Records of the folded-link sweeps (math mode fast): SBB (NaN) -> 0.
__global__ void k_fold_records(const double* __restrict__ recs, double* __restrict__ out,
                               int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double r = recs[i];
    out[i] = r == r ? r : 0.0;
  }
}

// simulation.cpp:104-112: links whose wall neighbour lies in plane nz-1 move.
__global__ void k_mark_lid(const uint32_t* __restrict__ cellw, const int32_t* __restrict__ base,
                           double* __restrict__ recs, int nx, int ny, int nz,
                           int* __restrict__ any) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= nx) return;
  const int64_t c = ((int64_t)z * ny + y) * nx + x;
  const uint32_t w = cellw[c];
  if ((w & kNonFluid) || !(w & kBounceMask)) return;
  int64_t r = base[c];
  bool hit = false;
  for (int j = 1; j < 19; ++j) {
    if (!((w >> j) & 1u)) continue;
    if (z + cE[dopp(j)][2] == nz - 1) {
      recs[r] = __longlong_as_double(0x7FF0000000000000ll);
      hit = true;
    }
    ++r;
  }
  if (hit) atomicOr(any, 1);
}

// Fluid-only layout: per 32-cell chunk of a row its fluid mask and count (one
// warp per chunk), then {rank, mask} after an exclusive scan of the counts.
__global__ void k_chunk_fluid(const uint32_t* __restrict__ cellw, int nx, int64_t nchunks,
                              int nchunk, uint32_t* __restrict__ mask, int32_t* __restrict__ cnt) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= nchunks) return;  // warp-uniform
  const int64_t row = gw / nchunk;
  const int x = (int)(gw - row * nchunk) * 32 + lane;
  const bool fluid = x < nx && !(cellw[row * nx + x] & kNonFluid);
  const unsigned m = __ballot_sync(0xffffffffu, fluid);
  if (lane == 0) {
    mask[gw] = m;
    cnt[gw] = __popc(m);
  }
}
__global__ void k_pack_ctab(const uint32_t* __restrict__ mask, const int32_t* __restrict__ rank,
                            ChunkEnt* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = ChunkEnt{(uint32_t)rank[i], mask[i]};
}

// Per link record: the owner's lane in its 32-cell chunk and the incoming
// direction j, (x & 31) | j << 5 -- the compact CLI sweep's link list of a
// chunk-plane is then a contiguous run of this array (no per-plane prefix
// sum and publish in the kernel).  One thread per cell, links in (cell, j)
// order exactly like the records.
__global__ void k_linkdesc(const uint32_t* __restrict__ cellw, const int32_t* __restrict__ cellbase,
                           int nx, int64_t cells, uint16_t* __restrict__ desc) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const uint32_t w = cellw[c];
  if (w & kNonFluid) return;
  uint32_t m = w & kBounceMask;
  int32_t r = cellbase[c];
  const uint16_t lane = (uint16_t)((c % nx) & 31);
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    desc[r++] = (uint16_t)(lane | (j << 5));
  }
}

// Units of one row per thread (greedy: up to 32 fluid cells from at most 3
// consecutive chunks).  FILL = false counts them; FILL = true writes the unit
// records, the per-slot words and the per-record descriptors.
template <bool FILL>
__global__ void k_units(const ChunkEnt* __restrict__ ctab, const uint32_t* __restrict__ cellw,
                        const int32_t* __restrict__ cellbase, int nx, int ny, int64_t rows,
                        int nchunk, int xlo, int xhi, bool outside,
                        const int32_t* __restrict__ ubase, int32_t* __restrict__ cnt,
                        UnitRec* __restrict__ units, uint32_t* __restrict__ slotw,
                        uint16_t* __restrict__ udesc) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const uint32_t y = (uint32_t)(row % ny), z = (uint32_t)(row / ny);
  const int64_t u0 = FILL ? ubase[row] : 0;
  int nu = 0, n = 0, c0 = 0, nl = 0;
  uint32_t s0 = 0, lbase = 0, wrap = 0;
  auto close = [&] {
    if (FILL)
      units[u0 + nu] = UnitRec{s0, lbase, y | z << 16,
                               (uint32_t)n | wrap << 6 | (uint32_t)c0 << 8 | (uint32_t)nl << 20};
    ++nu;
    n = 0;
  };
  for (int c = 0; c < nchunk; ++c) {
    const ChunkEnt e = ctab[row * nchunk + c];
    // cells of [xlo, xhi) only, or the cells outside it (slab split: interior
    // columns and edge bands are swept by separate launches)
    uint32_t rm = 0xffffffffu;
    const int lo = xlo - 32 * c, hi = xhi - 32 * c;
    if (lo > 0) rm &= lo >= 32 ? 0u : ~((1u << lo) - 1u);
    if (hi < 32) rm &= hi <= 0 ? 0u : ((1u << hi) - 1u);
    uint32_t m = e.mask & (outside ? ~rm : rm);
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t slot = e.rank + __popc(e.mask & ((1u << b) - 1u));
      if (n && slot != s0 + (uint32_t)n) close();  // a unit is a run of consecutive slots
      const int x = c * 32 + b;
      const int64_t cell = row * nx + x;
      const uint32_t w = cellw[cell];
      const int wl = __popc(w & kBounceMask);
      if (n && (n == 32 || c - c0 >= 3 || nl + wl > kUnitLinkCap)) close();
      if (!n) {
        c0 = c;
        s0 = slot;
        nl = 0;
        wrap = 0;
        if (FILL) lbase = (uint32_t)cellbase[cell];
      }
      if (FILL) {
        const uint32_t fx = (x == 0 ? kSlotX0 : 0u) | (x == nx - 1 ? kSlotXN : 0u);
        slotw[slot] = (w & 0x7FFFFu) | (uint32_t)((c - c0) * 32 + b) << kSlotRelShift | fx;
        wrap |= (x == 0 ? 1u : 0u) | (x == nx - 1 ? 2u : 0u);
        uint32_t mm = w & kBounceMask;
        int32_t r = cellbase[cell];
        while (mm) {
          const int j = __ffs(mm) - 1;
          mm &= mm - 1;
          if (udesc) udesc[r] = (uint16_t)(n | (j << 5));
          ++r;
        }
      }
      nl += wl;
      ++n;
    }
  }
  if (n) close();
  if (!FILL) cnt[row] = nu;
}

__global__ void k_unpack_flags(const uint32_t* __restrict__ cellw, uint8_t* __restrict__ out,
                               int64_t cells) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < cells) out[c] = (uint8_t)(cellw[c] >> kFlagShift);
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void setup_cellwords(const CellSetupArgs& a, cudaStream_t s) {
  const dim3 blk(128), grid((a.nx + 127) / 128, a.ny, a.nz);
  k_cellwords<<<grid, blk, 0, s>>>(a.flags, a.ghost_lo, a.ghost_hi, a.nx, a.ny, a.nz, a.px, a.py,
                                   a.pz, a.slab, a.cellw, a.count);
  ck(cudaGetLastError(), "k_cellwords");
  const int64_t cells = (int64_t)a.nx * a.ny * a.nz;
  if (a.fill_sectors) {
    k_fill_sectors<<<blocks((cells + 3) / 4, 256), 256, 0, s>>>(a.cellw, cells);
    ck(cudaGetLastError(), "k_fill_sectors");
  }
}

int64_t setup_bases(const int32_t* count, int32_t* base, int32_t* chunkbase, int nx, int64_t rows,
                    int nchunk, void* scratch, size_t scratch_bytes, int64_t* d_total,
                    cudaStream_t s) {
  const int64_t cells = (int64_t)nx * rows;
  cub::TransformInputIterator<int64_t, ToI64, const int32_t*> wide(count, ToI64());
  size_t need_r = 0, need_s = 0;
  ck(cub::DeviceReduce::Sum(nullptr, need_r, wide, d_total, cells, s), "reduce size");
  ck(cub::DeviceScan::ExclusiveSum(nullptr, need_s, count, base, cells, s), "scan size");
  if (need_r > scratch_bytes || need_s > scratch_bytes) return -1;
  ck(cub::DeviceReduce::Sum(scratch, scratch_bytes, wide, d_total, cells, s), "reduce");
  int64_t total = 0;
  ck(cudaMemcpyAsync(&total, d_total, sizeof(total), cudaMemcpyDeviceToHost, s), "total");
  ck(cudaStreamSynchronize(s), "total sync");
  if (total > INT32_MAX) return total;  // caller rejects; the scan would overflow
  ck(cub::DeviceScan::ExclusiveSum(scratch, scratch_bytes, count, base, cells, s), "scan");
  k_chunkbase<<<blocks(rows * nchunk + 1, 256), 256, 0, s>>>(base, chunkbase, nx, rows, nchunk,
                                                               d_total);
  ck(cudaGetLastError(), "k_chunkbase");
  return total;
}

size_t setup_scratch_bytes(int64_t cells) {
  cub::TransformInputIterator<int64_t, ToI64, const int32_t*> wide(nullptr, ToI64());
  size_t need_r = 0, need_s = 0;
  cub::DeviceReduce::Sum(nullptr, need_r, wide, (int64_t*)nullptr, cells);
  cub::DeviceScan::ExclusiveSum(nullptr, need_s, (const int32_t*)nullptr, (int32_t*)nullptr, cells);
  return need_r > need_s ? need_r : need_s;
}

void setup_links(const LinkSetupArgs& a, uint32_t* seen_bits, unsigned long long* d_err,
                 unsigned long long* d_fallbacks, int* d_moving, cudaStream_t s) {
  if (a.n_links == 0) return;
  k_links<<<blocks(a.n_links, 256), 256, 0, s>>>(a, seen_bits, d_err, d_fallbacks, d_moving);
  ck(cudaGetLastError(), "k_links");
}

void fill_records_nan(double* recs, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  k_fill_nan<<<blocks(n, 256), 256, 0, s>>>(recs, n);
  ck(cudaGetLastError(), "k_fill_nan");
}

void fold_records(const double* recs, double* out, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  k_fold_records<<<blocks(n, 256), 256, 0, s>>>(recs, out, n);
  ck(cudaGetLastError(), "k_fold_records");
}

void mark_lid_links(const uint32_t* cellw, const int32_t* base, double* recs, int nx, int ny,
                    int nz, int* d_any, cudaStream_t s) {
  const dim3 blk(128), grid((nx + 127) / 128, ny, nz);
  k_mark_lid<<<grid, blk, 0, s>>>(cellw, base, recs, nx, ny, nz, d_any);
  ck(cudaGetLastError(), "k_mark_lid");
}

int64_t build_ctab(const uint32_t* cellw, int nx, int64_t rows, int nchunk, ChunkEnt* ctab,
                   cudaStream_t s) {
  const int64_t n = rows * nchunk;
  uint32_t* mask = nullptr;
  int32_t *cnt = nullptr, *rank = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  ck(cudaMalloc(&mask, sizeof(uint32_t) * n), "ctab alloc");
  ck(cudaMalloc(&cnt, sizeof(int32_t) * n), "ctab alloc");
  ck(cudaMalloc(&rank, sizeof(int32_t) * n), "ctab alloc");
  k_chunk_fluid<<<blocks(n * 32, 256), 256, 0, s>>>(cellw, nx, n, nchunk, mask, cnt);
  ck(cudaGetLastError(), "k_chunk_fluid");
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rank, n, s), "ctab scan size");
  ck(cudaMalloc(&tmp, tb), "ctab alloc");
  ck(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rank, n, s), "ctab scan");
  k_pack_ctab<<<blocks(n, 256), 256, 0, s>>>(mask, rank, ctab, n);
  ck(cudaGetLastError(), "k_pack_ctab");
  int32_t last[2] = {0, 0};
  ck(cudaMemcpyAsync(&last[0], rank + n - 1, 4, cudaMemcpyDeviceToHost, s), "ctab total");
  ck(cudaMemcpyAsync(&last[1], cnt + n - 1, 4, cudaMemcpyDeviceToHost, s), "ctab total");
  ck(cudaStreamSynchronize(s), "ctab sync");
  cudaFree(mask);
  cudaFree(cnt);
  cudaFree(rank);
  cudaFree(tmp);
  return (int64_t)last[0] + last[1];
}

int64_t build_units(const ChunkEnt* ctab, const uint32_t* cellw, const int32_t* cellbase, int nx,
                    int ny, int64_t rows, int nchunk, int xlo, int xhi, bool outside,
                    UnitRec** units_out, uint32_t* slotw, uint16_t* udesc, cudaStream_t s) {
  int32_t *cnt = nullptr, *ubase = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  ck(cudaMalloc(&cnt, sizeof(int32_t) * rows), "units alloc");
  ck(cudaMalloc(&ubase, sizeof(int32_t) * rows), "units alloc");
  k_units<false><<<blocks(rows, 128), 128, 0, s>>>(ctab, cellw, cellbase, nx, ny, rows, nchunk,
                                                    xlo, xhi, outside, nullptr, cnt, nullptr, nullptr, nullptr);
  ck(cudaGetLastError(), "k_units count");
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, ubase, rows, s), "units scan size");
  ck(cudaMalloc(&tmp, tb), "units alloc");
  ck(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, ubase, rows, s), "units scan");
  int32_t last[2] = {0, 0};
  ck(cudaMemcpyAsync(&last[0], ubase + rows - 1, 4, cudaMemcpyDeviceToHost, s), "units total");
  ck(cudaMemcpyAsync(&last[1], cnt + rows - 1, 4, cudaMemcpyDeviceToHost, s), "units total");
  ck(cudaStreamSynchronize(s), "units sync");
  const int64_t nunits = (int64_t)last[0] + last[1];
  UnitRec* units = nullptr;
  ck(cudaMalloc(&units, sizeof(UnitRec) * (nunits + 4)), "units alloc");
  ck(cudaMemsetAsync(units, 0, sizeof(UnitRec) * (nunits + 4), s), "units clear");
  k_units<true><<<blocks(rows, 128), 128, 0, s>>>(ctab, cellw, cellbase, nx, ny, rows, nchunk,
                                                   xlo, xhi, outside, ubase, nullptr, units, slotw, udesc);
  ck(cudaGetLastError(), "k_units fill");
  ck(cudaStreamSynchronize(s), "units sync");
  cudaFree(cnt);
  cudaFree(ubase);
  cudaFree(tmp);
  *units_out = units;
  return nunits;
}

void build_linkdesc(const uint32_t* cellw, const int32_t* cellbase, int nx, int64_t cells,
                    uint16_t* desc, cudaStream_t s) {
  k_linkdesc<<<blocks(cells, 256), 256, 0, s>>>(cellw, cellbase, nx, cells, desc);
  ck(cudaGetLastError(), "k_linkdesc");
}

void unpack_flags(const uint32_t* cellw, uint8_t* out, int64_t cells, cudaStream_t s) {
  k_unpack_flags<<<blocks(cells, 256), 256, 0, s>>>(cellw, out, cells);
  ck(cudaGetLastError(), "k_unpack_flags");
}

}  // namespace pgpu
