// Device-side construction of the link structures (setup.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "kparams.h"

namespace pgpu {

// Validation failures of the caller's link list (pgpu_create contract).
enum SetupError : int {
  kSetupOk = 0,
  kSetupErrCell = 1,            // link on a non-fluid or out-of-range cell
  kSetupErrDir = 2,             // direction outside 1..18
  kSetupErrFluidNeighbour = 3,  // the wall side x + e_k is fluid
  kSetupErrDuplicate = 4,
  kSetupErrSecondNotFluid = 5,  // CLI second_fluid given where x - e_k is not fluid
  kSetupErrSecondCell = 6,      // CLI second_fluid is not the cell x - e_k
};

struct CellSetupArgs {
  const uint8_t* flags;     // device, cells bytes
  const uint8_t* ghost_lo;  // device, ny*nz (slab only)
  const uint8_t* ghost_hi;
  int nx, ny, nz;
  bool px, py, pz, slab, fill_sectors;
  uint32_t* cellw;  // out
  int32_t* count;   // out: links per cell
};

struct LinkSetupArgs {
  int64_t n_links, cells;
  int nx, ny, nz;
  bool px, py, pz, slab, cli;
  const int64_t* link_cell;  // device copies of the caller's SoA
  const int64_t* link_second;
  const int32_t* link_dir;
  const float* link_q;
  const uint8_t* link_moving;  // may be null
  const uint32_t* cellw;
  const int32_t* cellbase;
  double* recs;  // null: validate only
};

void setup_cellwords(const CellSetupArgs& a, cudaStream_t s);
size_t setup_scratch_bytes(int64_t cells);
// Per-cell exclusive bases + per-chunk bases (+ one sentinel = the total: the
// chunk base array has rows * nchunk + 1 entries); returns the link total (host
// value; > INT32_MAX means the bases were not written), -1 if scratch is short.
int64_t setup_bases(const int32_t* count, int32_t* base, int32_t* chunkbase, int nx, int64_t rows,
                    int nchunk, void* scratch, size_t scratch_bytes, int64_t* d_total,
                    cudaStream_t s);
void setup_links(const LinkSetupArgs& a, uint32_t* seen_bits, unsigned long long* d_err,
                 unsigned long long* d_fallbacks, int* d_moving, cudaStream_t s);
void fill_records_nan(double* recs, int64_t n, cudaStream_t s);
// Records of the folded-link sweeps (math mode fast): NaN (SBB) -> 0.
void fold_records(const double* recs, double* out, int64_t n, cudaStream_t s);
void mark_lid_links(const uint32_t* cellw, const int32_t* base, double* recs, int nx, int ny,
                    int nz, int* d_any, cudaStream_t s);
// Fluid-only layout chunk table [rows][nchunk] {rank, mask}; returns the fluid count.
int64_t build_ctab(const uint32_t* cellw, int nx, int64_t rows, int nchunk, ChunkEnt* ctab,
                   cudaStream_t s);
// Per link record (x & 31) | j << 5 in record order (compact CLI sweep).
void build_linkdesc(const uint32_t* cellw, const int32_t* cellbase, int nx, int64_t cells,
                    uint16_t* desc, cudaStream_t s);
// Units of the units sweep (kparams.h UnitRec) with their per-slot words and
// per-record descriptors (udesc may be null: no links) over the cells with x in
// [xlo, xhi) (slab split: the interior columns) or, with `outside`, over the
// other cells (the two edge bands); *units_out is cudaMalloc'ed here (+ 4 zero
// records).  Returns the unit count.
int64_t build_units(const ChunkEnt* ctab, const uint32_t* cellw, const int32_t* cellbase, int nx,
                    int ny, int64_t rows, int nchunk, int xlo, int xhi, bool outside,
                    UnitRec** units_out, uint32_t* slotw, uint16_t* udesc, cudaStream_t s);
void unpack_flags(const uint32_t* cellw, uint8_t* out, int64_t cells, cudaStream_t s);

}  // namespace pgpu
