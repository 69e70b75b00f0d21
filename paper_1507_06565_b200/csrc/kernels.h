// Host-callable launchers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "kparams.h"

namespace pgpu {

struct SweepConfig {
  int op = 0;        // 0: stream+collide (K1), 1: stream only (KP)
  int part = 0;      // 0: all cells, 1: edge columns only, 2: interior only
  bool glbm = false;
  bool records = false;
  bool slab = false;
  // visit the z-blocks in descending order: consecutive sweeps alternate, so
  // each starts on the planes the previous one wrote last (still in L2)
  bool zrev = false;
  // the sweep reads buffer 1 (every second sweep of a run): the units sweep
  // alternates its block order on it
  bool odd = false;
};

// Dense layout (kernels.cu) or, when p.ctab is set, the fluid-only layout
// (sweep_compact.cu); op 1 (KP) writes f(n) into the other buffer of the
// same layout.
void launch_sweep(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                  cudaStream_t s);
void launch_sweep_compact(const SweepConfig& cfg, const KParams& p, const double* src,
                          double* dst, cudaStream_t s);
// K1 of the fluid-only layout as a warp-specialised TMA pipeline (sweep_tma.cu):
// whole-domain stream+collide, no slab, no folded links, nx % 4 == 0.
bool tma_sweep_supported(const SweepConfig& cfg, const KParams& p);
bool launch_sweep_tma(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                      cudaStream_t s);
// K1 of the fluid-only layout by units of 32 consecutive fluid slots
// (sweep_units.cu): stream+collide of the whole domain or, in the x-slab
// split, of the interior columns [sweep_edge_band(nx), nx - sweep_edge_band(nx))
// (KParams::units then covers those columns only) and of the 32-column edge
// bands (KParams::units_edge); no folded links; needs KParams::units / slotw
// (/ udesc with records).
int sweep_edge_band(int nx);
bool units_sweep_supported(const SweepConfig& cfg, const KParams& p);
bool launch_sweep_units(const SweepConfig& cfg, const KParams& p, const double* src, double* dst,
                        cudaStream_t s);
// K0 of the fluid-only layout: pre-collision f(n) -> post-collision g(n) in
// place (with records in math mode fast + PGPU_FOLD: folded CLI slots).
void launch_collide_compact(bool glbm, bool slab, bool records, const KParams& p, double* buf,
                            cudaStream_t s);
// Population I/O of the fluid-only layout through a reference-layout staging
// buffer of the planes [z0, z0 + nzc): expand (compact -> dense) or pack.
void launch_compact_io(bool expand, const KParams& p, double* f, double* dense, int z0, int nzc,
                       cudaStream_t s);
// initialize_equilibrium in the fluid-only layout (every fluid slot = feq)
void launch_fill_compact(const KParams& p, int64_t nfluid, double* f, const double* feq,
                         cudaStream_t s);
// One cooperative launch running nsteps K1 sweeps (a -> b -> a ...); returns 0
// on success, -1 if the cooperative launch is not possible.
// z-planes per block of the marching sweeps (cols = blocks per z-plane)
int zper_for(int64_t cols, int nz);
int launch_sweep_persistent(const SweepConfig& cfg, const KParams& p, double* a, double* b,
                            int64_t nsteps, cudaStream_t s);
void launch_collide_inplace(bool glbm, bool slab, const KParams& p, double* buf,
                            cudaStream_t s);
void launch_macro_fields(bool glbm, const KParams& p, const double* f, double* drho,
                         double* ux, double* uy, double* uz, int* err, cudaStream_t s);
void launch_plane_sums(const KParams& p, const double* u, double* sums, cudaStream_t s);
void launch_max_speed2(bool glbm, const KParams& p, const double* f,
                       unsigned long long* vmax2_bits, int* nonfinite, int* err,
                       cudaStream_t s);
void preload_kernels();
// free stream() over a reference-layout field (plane stride = cells)
void launch_stream_field(const uint8_t* flags, const int dims[3], const int per[3],
                         const double* cur, double* next, cudaStream_t s);
void launch_fill_equilibrium(const KParams& p, int64_t cells, double* f, const double* feq,
                             cudaStream_t s);

}  // namespace pgpu
