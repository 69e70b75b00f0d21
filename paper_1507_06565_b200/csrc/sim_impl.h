// Internal: the simulation handle behind the C ABI (sim.cpp) and the x-slab
// multi-GPU driver (dist.cpp).  Not part of the public interface.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "host_common.h"
#include "kernels.h"
#include "kparams.h"
#include "setup.h"
#include <nvtx3/nvToolsExt.h>  // header-only; no cost without a profiler attached

namespace pgpu {
// NVTX range for the host-side issue of a phase (K0, K1 parts, KP, halo
// exchange): visible in nsys / ncu --nvtx timelines next to the kernels.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};
}  // namespace pgpu

namespace pgpu {
void moments(const double f[19], double rho0, double& drho, double u[3]);
void equilibrium(double drho, const double u[3], double rho0, double out[19]);
void glbm_force_and_velocity(const double mom[3], double eps, double K, double cf,
                             const double g[3], double nu, double u[3], double force[3]);
}  // namespace pgpu

using namespace pgpu;

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e__ = (call);                                                         \
    if (e__ != cudaSuccess) {                                                         \
      std::ostringstream os__;                                                        \
      os__ << #call << " failed: " << cudaGetErrorString(e__) << " (" << __FILE__ << ":" \
           << __LINE__ << ")";                                                        \
      throw CudaError(os__.str());                                                    \
    }                                                                                 \
  } while (0)

namespace pgpu {
bool g_plain_sweep();  // kernels.cu: PGPU_SWEEP=plain selected
}

struct pgpu_sim {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int nx = 0, ny = 0, nz = 0;
  bool per[3] = {true, true, false};
  bool slab = false;
  int x_offset = 0, global_nx = 0;
  int64_t cells = 0, ks = 0;
  pgpu_fluid_params params{};
  int scheme = PGPU_SBB;
  std::vector<double> porosity;
  std::vector<int64_t> plane_fluid_count;
  bool has_lo = false, has_hi = false;
  double lo = 0.0, hi = 0.0;
  int64_t fluid_cells = 0;
  int32_t cli_fallbacks = 0;
  // link structures live on the device only (setup.cu builds them)
  int64_t n_links = 0;
  bool any_moving = false;
  double lid[3] = {0.0, 0.0, 0.0};
  // GLBM (set_porous)
  bool porous = false, glbm_active = false;
  std::vector<double> eps, K, gwp, gwm;
  double cf = 0.0;
  bool eps_in_eq = true;
  // device memory: f[0]/f[1] hold the pre-collision state f(n) (in f[cur],
  // "pre") or the post-collision state g(n-1) ("post"), in the dense layout
  // (plane stride ks) or the fluid-only one (plane stride kp.ks); population
  // I/O of the fluid-only layout stages through the dead buffer.
  double* f[2] = {nullptr, nullptr};
  bool compact = false;
  int64_t nfluid_slots = 0;  // fluid-only layout: fluid cells (slots 0..n-1 of every plane)
  ChunkEnt* d_ctab = nullptr;
  double* d_scratch = nullptr;  // compact layout: observable scratch when f[1-cur] is too small
  int64_t scratch_n = 0;
  uint32_t* d_cellw = nullptr;
  int32_t* d_cellbase = nullptr;
  int32_t* d_chunkbase = nullptr;
  LinkRec* d_recs = nullptr;
  // math mode PGPU_MATH_FAST: contracted collision; in the fluid-only layout
  // CLI links are folded (kparams.h KParams::fast) and read d_recs_fold
  // (the records with SBB = 0)
  bool fast = false;
  LinkRec* d_recs_fold = nullptr;
  uint16_t* d_linkdesc = nullptr;  // per record: owner lane | j << 5 (compact CLI sweep)
  PlaneCoef* d_planes = nullptr;
  double* d_feq = nullptr;
  int* d_flags = nullptr;  // [0] err, [1] nonfinite
  unsigned long long* d_vmax = nullptr;
  double* d_sums = nullptr;
  UnitRec* d_units = nullptr;     // units sweep (built when it is selected)
  UnitRec* d_units_edge = nullptr;  // slab split: units of the edge bands
  int64_t n_units_edge = 0;
  uint32_t* d_slotw = nullptr;
  uint16_t* d_udesc = nullptr;
  int64_t n_units = 0;
  uint32_t* d_tickets = nullptr;  // TMA sweep work counter (KParams::tickets)
  // state
  int cur = 0;
  bool post = false;
  int64_t steps = 0;
  int64_t launches = 0;
  // halo (slab mode)
  double* send_lo = nullptr;
  double* send_hi = nullptr;
  double* recv_lo[2] = {nullptr, nullptr};
  double* recv_hi[2] = {nullptr, nullptr};
  int ghost_cur = 0;
  int pending = 0;  // 0 none, 1 K0 issued, 2 K1 parts issued
  // CUDA graphs of kGraphSteps K1 launches (one per starting buffer)
  static constexpr int kGraphSteps = 16;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  bool persistent = false;  // L2-resident domain: cooperative multi-step sweep
  // alternate the z order of consecutive SBB sweeps (PGPU_ZREV=0: off); CLI
  // sweeps keep the bed's link-heavy z-blocks first instead (less tail)
  bool zrev_on = true;
  cudaStream_t graph_stream = nullptr;
  KParams kp{};

  ~pgpu_sim() {
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    cudaSetDevice(device);
    for (double* p : f) cudaFree(p);
    cudaFree(d_ctab);
    cudaFree(d_scratch);
    cudaFree(d_cellw);
    cudaFree(d_cellbase);
    cudaFree(d_chunkbase);
    cudaFree(d_recs);
    cudaFree(d_recs_fold);
    cudaFree(d_linkdesc);
    cudaFree(d_planes);
    cudaFree(d_feq);
    cudaFree(d_flags);
    cudaFree(d_vmax);
    cudaFree(d_sums);
    cudaFree(d_units);
    cudaFree(d_units_edge);
    cudaFree(d_slotw);
    cudaFree(d_udesc);
    cudaFree(d_tickets);
    if (own_stream) cudaStreamDestroy(own_stream);
  }

  void drop_graphs() {
    for (auto& g : graph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
  }

  int plane_of(int64_t c) const { return static_cast<int>(c / ((int64_t)nx * ny)); }

  // ---- derived constants (host, reference operation order) ----------------
  void refresh_params() {
    const double* g = params.body_force;
    const double rho0 = params.rho0;
    kp.wp = params.omega_plus;
    kp.wm = params.omega_minus;
    kp.rho0 = rho0;
    kp.nu = params.nu;
    kp.cf = cf;
    for (int q = 0; q < 9; ++q) {
      const int k = 1 + 2 * q;
      const double w = weight(k);
      // simulation.cpp:183,185,190
      const double eg = static_cast<double>(kE[k][0]) * g[0] +
                        static_cast<double>(kE[k][1]) * g[1] +
                        static_cast<double>(kE[k][2]) * g[2];
      kp.fpop[q] = 3.0 * w * rho0 * eg;
      kp.wr3[q] = w * rho0 * 3.0;
    }
    for (int k = 0; k < 19; ++k) {
      // boundary.cpp:38-40 with m.inv_cs2 = 3.0
      const double eu = kE[k][0] * lid[0] + kE[k][1] * lid[1] + kE[k][2] * lid[2];
      kp.mw[k] = 2.0 * weight(k) * rho0 * 3.0 * eu;
    }
    for (int i = 0; i < 3; ++i) {
      kp.hg[i] = 0.5 * g[i] / rho0;  // simulation.cpp:367
      kp.g[i] = g[i];
    }
    kp.fast = fast ? 1 : 0;
    fill_fast(kp.fc, params.omega_plus, params.omega_minus, rho0, 1.0, 0.0);
    if (porous) upload_planes();
    update_links();
    drop_graphs();
  }

  // FastCoef (kparams.h) of a TRT collision with omegas wp/wm; inv_eq =
  // 1/eq_eps of the GLBM equilibrium (1 for the core collision)
  static void fill_fast(FastCoef& c, double wp, double wm, double rho0, double inv_eq,
                        double force_pref) {
    c.hp = 0.5 * (1.0 - wp);
    c.hm = 0.5 * (1.0 - wm);
    c.w0 = 1.0 - wp;
    c.a0 = wp / 3.0;
    c.b0 = -0.5 * wp * rho0 * inv_eq;
    for (int cl = 0; cl < 2; ++cl) {
      const double w = cl == 0 ? 1.0 / 18.0 : 1.0 / 36.0;
      c.kw1[cl] = wp * w;
      c.kw2[cl] = -1.5 * wp * w * rho0 * inv_eq;
      c.C[cl] = 4.5 * wp * w * rho0 * inv_eq;
      c.D[cl] = 3.0 * wm * w * rho0;
      c.fw[cl] = force_pref * w;
    }
    c.inv_rho0 = 1.0 / rho0;
  }

  // PGPU_FOLD=1: fold CLI links in fast mode (measured slower on C4/C3, off by default)
  bool fold_enabled = false;
  bool fold_links() const { return fast && fold_enabled && compact && d_recs != nullptr; }
  // Link records the kernels read: the folded-link sweeps take SBB = 0.
  void update_links() {
    kp.moving = any_moving ? 1 : 0;
    kp.fold = fold_links() ? 1 : 0;
    if (fold_links()) {
      if (!d_recs_fold) CK(cudaMalloc(&d_recs_fold, sizeof(LinkRec) * n_links));
      fold_records(d_recs, d_recs_fold, n_links, stream);
      CK(cudaGetLastError());
      kp.links = d_recs_fold;
    } else {
      kp.links = d_recs;
    }
  }

  void upload_planes() {
    const double* g = params.body_force;
    const double rho0 = params.rho0, nu = params.nu;
    std::vector<PlaneCoef> pc(nz);
    for (int z = 0; z < nz; ++z) {
      PlaneCoef& c = pc[z];
      const double e = eps[z], k = K[z];
      c.eps = e;
      c.K = k;
      c.wp = gwp[z];
      c.wm = gwm[z];
      c.eq_eps = eps_in_eq ? e : 1.0;  // simulation.cpp:218
      for (int i = 0; i < 3; ++i) {
        c.half_eps_g[i] = 0.5 * e * g[i];  // :233-235
        c.eps_g[i] = e * g[i];             // :248-250
      }
      c.c0 = 0.5 * (1.0 + e * nu / (2.0 * k));  // :236
      c.denom_lin = 2.0 * c.c0;                 // :239
      c.c1 = 0.5 * e * cf / std::sqrt(k);       // :241 and simulation.cpp:58
      c.drag_lin = e * nu / k;                  // :247
      c.drag_lin0 = c.drag_lin + 0.0;           // :247 with c_F == 0
      c.drag_q = e * cf / std::sqrt(k);         // :247
      c.force_pref = (1.0 - 0.5 * c.wm) * 3.0 * rho0;  // :253
      // x / d == x * (1/d) exactly when d is a power of two (1/d is exact)
      auto mode_of = [](double d, double& inv) {
        inv = 1.0;
        if (d == 1.0) return 0;
        int ex = 0;
        if (std::isfinite(d) && d > 0.0 && std::frexp(d, &ex) == 0.5 &&
            std::isfinite(1.0 / d) && 1.0 / d != 0.0) {
          inv = 1.0 / d;
          return 1;
        }
        return 2;
      };
      c.eq_mode = mode_of(c.eq_eps, c.inv_eq_eps);
      c.denom_mode = mode_of(c.denom_lin, c.inv_denom);
      fill_fast(c.fc, c.wp, c.wm, rho0, 1.0 / c.eq_eps, c.force_pref);
      c.f_inv_denom = 1.0 / c.denom_lin;
    }
    if (!d_planes) CK(cudaMalloc(&d_planes, sizeof(PlaneCoef) * nz));
    CK(cudaMemcpyAsync(d_planes, pc.data(), sizeof(PlaneCoef) * nz, cudaMemcpyHostToDevice,
                       stream));
    CK(cudaStreamSynchronize(stream));
    kp.planes = d_planes;
  }

  bool records_needed() const { return scheme == PGPU_CLI || any_moving; }

  // Records are built by pgpu_create when the scheme is CLI or a link moves;
  // a later set_lid_velocity on an SBB simulation starts from all-SBB (NaN).
  void ensure_records() {
    if (d_recs || n_links == 0) return;
    CK(cudaMalloc(&d_recs, sizeof(LinkRec) * (n_links + 2)));  // + 2: even-rounded bulk copies
    fill_records_nan(d_recs, n_links, stream);
    ensure_linkdesc();
    update_links();
    kp.nrec = n_links;
    drop_graphs();
  }

  // per-record link descriptors for the compact sweeps (+ 16: pair / 16-byte bulk copies)
  void ensure_linkdesc() {
    if (d_linkdesc || n_links == 0) return;
    CK(cudaMalloc(&d_linkdesc, sizeof(uint16_t) * (n_links + 16)));
    CK(cudaMemsetAsync(d_linkdesc, 0, sizeof(uint16_t) * (n_links + 16), stream));
    build_linkdesc(d_cellw, d_cellbase, nx, cells, d_linkdesc, stream);
    kp.linkdesc = d_linkdesc;
  }

  // static data of the units sweep (fluid-only layout): unit records, per-slot
  // words, per-record descriptors
  void ensure_units() {
    if (d_units || !compact || !d_ctab) return;
    CK(cudaMalloc(&d_slotw, sizeof(uint32_t) * (kp.ks + 32)));
    if (n_links > 0) {
      CK(cudaMalloc(&d_udesc, sizeof(uint16_t) * (n_links + 16)));
      CK(cudaMemsetAsync(d_udesc, 0, sizeof(uint16_t) * (n_links + 16), stream));
    }
    const int eb = slab ? sweep_edge_band(nx) : 0;  // slab split: interior columns only
    n_units = build_units(d_ctab, d_cellw, d_cellbase, nx, ny, (int64_t)ny * nz, kp.nchunk, eb, nx - eb,
                          false, &d_units, d_slotw, d_udesc, stream);
    if (slab && eb == 32 && nx % 32 == 0) {  // whole-chunk edge bands: the edge part on units too
      n_units_edge = build_units(d_ctab, d_cellw, d_cellbase, nx, ny, (int64_t)ny * nz, kp.nchunk, eb,
                                 nx - eb, true, &d_units_edge, d_slotw, d_udesc, stream);
      kp.units_edge = d_units_edge;
      kp.nunits_edge = n_units_edge;
    }
    kp.units = d_units;
    kp.slotw = d_slotw;
    kp.udesc = d_udesc;
    kp.nunits = n_units;
  }

  // the K1 kernel the whole-domain step runs (pgpu_sweep_kernel; AUTO for the
  // dense layout, which has one)
  int resolved_sweep() const {
    if (!compact) return PGPU_SWEEP_AUTO;
    if (kp.sweep == PGPU_SWEEP_TMA && tma_sweep_supported(sweep_cfg(0, 0), kp)) return PGPU_SWEEP_TMA;
    if ((kp.sweep == PGPU_SWEEP_UNITS || kp.sweep == PGPU_SWEEP_AUTO) &&
        units_sweep_supported(sweep_cfg(0, slab ? 2 : 0), kp))
      return PGPU_SWEEP_UNITS;
    return PGPU_SWEEP_CPIPE;
  }

  SweepConfig sweep_cfg(int op, int part) const {
    SweepConfig c;
    c.op = op;
    c.part = part;
    c.glbm = glbm_active;
    c.records = records_needed() && n_links > 0;
    c.slab = slab;
    return c;
  }

  void set_ghost_ptrs() {
    if (!slab) return;
    kp.ghost_lo = recv_lo[ghost_cur];
    kp.ghost_hi = recv_hi[ghost_cur];
    kp.send_lo = send_lo;
    kp.send_hi = send_hi;
  }

  void check_launch() { CK(cudaGetLastError()); }

  // device memory held by this simulation (its resident allocations)
  int64_t device_bytes() const {
    const int64_t rows = (int64_t)ny * nz, nch = kp.nchunk;
    int64_t b = 2 * 19 * (int64_t)sizeof(double) * kp.ks;  // the two PDF buffers
    b += cells * (int64_t)(sizeof(uint32_t) + sizeof(int32_t));  // cell words + record bases
    b += (rows * nch + 1) * (int64_t)sizeof(int32_t);             // chunk record bases
    if (d_ctab) b += rows * nch * (int64_t)sizeof(ChunkEnt);
    if (d_recs) b += (n_links + 2) * (int64_t)sizeof(LinkRec);
    if (d_recs_fold) b += n_links * (int64_t)sizeof(LinkRec);
    if (d_linkdesc) b += (n_links + 16) * (int64_t)sizeof(uint16_t);
    if (d_units) b += (n_units + 4) * (int64_t)sizeof(UnitRec) + (kp.ks + 32) * (int64_t)sizeof(uint32_t);
    if (d_units_edge) b += (n_units_edge + 4) * (int64_t)sizeof(UnitRec);
    if (d_udesc) b += (n_links + 16) * (int64_t)sizeof(uint16_t);
    if (d_planes) b += nz * (int64_t)sizeof(PlaneCoef);
    if (d_scratch) b += scratch_n * (int64_t)sizeof(double);
    b += (19 + 2 + 1 + nz) * 8;  // feq, flags, vmax, plane sums
    return b;
  }

  // buffer holding the pre-collision state (valid when !post), in the
  // simulation's layout (fluid-only: compact slots, plane stride kp.ks)
  double* pre_buf() const { return f[cur]; }
  // fluid-only layout: compact slot of a cell (-1: not fluid)
  int64_t compact_slot_of(int64_t cell) {
    const int x = (int)(cell % nx), y = (int)((cell / nx) % ny), z = (int)(cell / ((int64_t)nx * ny));
    ChunkEnt e;
    CK(cudaMemcpy(&e, d_ctab + ((int64_t)z * ny + y) * kp.nchunk + (x >> 5), sizeof(e),
                  cudaMemcpyDeviceToHost));
    if (!((e.mask >> (x & 31)) & 1u)) return -1;
    return (int64_t)e.rank + __builtin_popcount(e.mask & ((1u << (x & 31)) - 1u));
  }
  // fluid-only layout: planes per staging chunk of the population I/O (the
  // dead sweep buffer, 19 * kp.ks doubles, holds 19 dense planes of them)
  int io_planes() const {
    const int64_t plane = (int64_t)nx * ny;
    return (int)std::max<int64_t>(1, std::min<int64_t>(nz, kp.ks / plane));
  }
  // n doubles of device scratch that do not alias the pre-collision state
  double* scratch(int64_t n) {
    if (19 * kp.ks >= n) return f[1 - cur];  // dead in the pre state
    if (scratch_n < n) {
      cudaFree(d_scratch);
      d_scratch = nullptr;
      scratch_n = 0;
      CK(cudaMalloc(&d_scratch, sizeof(double) * n));
      scratch_n = n;
    }
    return d_scratch;
  }

  // ---- state transitions -----------------------------------------------------
  void k0() {
    Nvtx r("K0 collide");
    set_ghost_ptrs();
    if (compact)
      launch_collide_compact(glbm_active, slab, sweep_cfg(0, 0).records, kp, f[cur], stream);
    else
      launch_collide_inplace(glbm_active, slab, kp, f[cur], stream);
    check_launch();
    ++launches;
  }
  void k1(int part) {
    Nvtx r(part == 0 ? "K1 sweep" : (part == 1 ? "K1 edge columns" : "K1 interior columns"));
    set_ghost_ptrs();
    SweepConfig c = sweep_cfg(0, part);
    c.zrev = zrev_on && !c.records && cur == 1;
    c.odd = zrev_on && cur == 1;
    launch_sweep(c, kp, f[cur], f[1 - cur], stream);
    check_launch();
    ++launches;
  }
  void ensure_pre() {
    // every observable and population access goes through here: in the middle
    // of a split step (slab mode) no buffer holds a consistent f(n)
    if (slab && pending) throw ConfigError("observable requested in the middle of a split step");
    if (!post) return;
    Nvtx r("KP materialise f(n)");
    set_ghost_ptrs();
    launch_sweep(sweep_cfg(1, 0), kp, f[cur], f[1 - cur], stream);
    check_launch();
    ++launches;
    cur = 1 - cur;
    post = false;
  }

  void build_graph(int start) {
    // kGraphSteps ping-pong K1 launches; ends on the starting buffer.
    cudaStream_t cs = stream;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int c = start;
    for (int i = 0; i < kGraphSteps; ++i) {
      SweepConfig sc = sweep_cfg(0, 0);
      sc.zrev = zrev_on && !sc.records && c == 1;
      sc.odd = zrev_on && c == 1;
      launch_sweep(sc, kp, f[c], f[1 - c], cs);
      c = 1 - c;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (e != cudaSuccess) throw CudaError(std::string("graph capture failed: ") + cudaGetErrorString(e));
    CK(cudaGraphInstantiate(&graph[start], g, 0));
    cudaGraphDestroy(g);
    graph_stream = cs;
  }

  void prepare() {
    if (slab || persistent) return;
    if (graph_stream != stream) drop_graphs();
    for (int c = 0; c < 2; ++c)
      if (!graph[c]) build_graph(c);
  }

  void step(int64_t n) {
    if (slab) throw ConfigError("slab simulations step through pgpu_step_part + halo exchange");
    for (int64_t i = 0; i < n;) {
      if (!post) {
        k0();
        post = true;
        ++steps;
        ++i;
        continue;
      }
      if (persistent && n - i >= 2) {
        // L2-resident domain: one cooperative launch for all remaining steps
        const int64_t m = n - i;
        if (launch_sweep_persistent(sweep_cfg(0, 0), kp, f[cur], f[1 - cur], m, stream) == 0) {
          check_launch();
          ++launches;
          if (m & 1) cur = 1 - cur;
          steps += m;
          i += m;
          continue;
        }
        cudaGetLastError();
        persistent = false;  // not launchable here: fall back to graphs
      }
      if (n - i >= kGraphSteps) {
        if (graph_stream != stream) drop_graphs();
        if (!graph[cur]) build_graph(cur);
        CK(cudaGraphLaunch(graph[cur], stream));
        launches += kGraphSteps;
        steps += kGraphSteps;
        i += kGraphSteps;
        continue;
      }
      k1(0);
      cur = 1 - cur;
      ++steps;
      ++i;
    }
  }

  // ---- observables -------------------------------------------------------------
  void sync() { CK(cudaStreamSynchronize(stream)); }

  void reset_flags() { CK(cudaMemsetAsync(d_flags, 0, sizeof(int) * 2, stream)); }

  void check_err_flag() {
    int h[2];
    CK(cudaMemcpyAsync(h, d_flags, sizeof(h), cudaMemcpyDeviceToHost, stream));
    sync();
    if (h[0]) throw NumericalInstability("negative discriminant in drag velocity solve");
  }

  void plane_sums(int axis, std::vector<double>& sums) {
    if (axis < 0 || axis > 2) throw ConfigError("stream axis must be 0, 1 or 2");
    ensure_pre();
    reset_flags();
    double* u = scratch(ks);  // dead in the pre state
    launch_macro_fields(glbm_active, kp, pre_buf(), nullptr, axis == 0 ? u : nullptr,
                        axis == 1 ? u : nullptr, axis == 2 ? u : nullptr, d_flags, stream);
    check_launch();
    launch_plane_sums(kp, u, d_sums, stream);
    check_launch();
    launches += 2;
    sums.resize(nz);
    CK(cudaMemcpyAsync(sums.data(), d_sums, sizeof(double) * nz, cudaMemcpyDeviceToHost, stream));
    check_err_flag();
  }

  // simulation.cpp:371-417 + profile.cpp:10-19
  void planar_profile(int axis, double* z_out, double* u_sup, double* u_int, double* eps_out,
                      double* u_norm, pgpu_profile_meta* meta) {
    int z_lo = nz, z_hi = -1;
    for (int z = 0; z < nz; ++z)
      if (plane_fluid_count[z] > 0) {
        z_lo = std::min(z_lo, z);
        z_hi = std::max(z_hi, z);
      }
    meta->n_planes = 0;
    meta->u_max = 0.0;
    meta->stream_axis = axis;
    meta->nu = params.nu;
    for (int i = 0; i < 3; ++i) meta->body_force[i] = params.body_force[i];
    if (has_lo && has_hi) {
      meta->z0 = lo;
      meta->height = hi - lo;
    } else {
      meta->z0 = 0.0;
      meta->height = nz;
    }
    if (z_hi < 0) return;
    std::vector<double> sums;
    plane_sums(axis, sums);
    const int64_t plane = (int64_t)nx * ny;
    for (int z = z_lo; z <= z_hi; ++z) {
      const int i = z - z_lo;
      z_out[i] = z + 0.5;
      u_sup[i] = sums[z] / static_cast<double>(plane);
      u_int[i] = plane_fluid_count[z] > 0 ? sums[z] / static_cast<double>(plane_fluid_count[z]) : 0.0;
      eps_out[i] = porosity[z];
    }
    const int n = z_hi - z_lo + 1;
    meta->n_planes = n;
    double u_max = 0.0;
    for (int i = 0; i < n; ++i)
      if (std::abs(u_sup[i]) > std::abs(u_max)) u_max = u_sup[i];
    for (int i = 0; i < n; ++i) u_norm[i] = (u_max != 0.0) ? u_sup[i] / u_max : 0.0;
    meta->u_max = u_max;
  }

  void max_speed2(double& vmax2, bool& finite) {
    ensure_pre();
    reset_flags();
    CK(cudaMemsetAsync(d_vmax, 0, sizeof(unsigned long long), stream));
    launch_max_speed2(glbm_active, kp, pre_buf(), d_vmax, d_flags + 1, d_flags, stream);
    check_launch();
    ++launches;
    unsigned long long bits = 0;
    CK(cudaMemcpyAsync(&bits, d_vmax, sizeof(bits), cudaMemcpyDeviceToHost, stream));
    int h[2];
    CK(cudaMemcpyAsync(h, d_flags, sizeof(h), cudaMemcpyDeviceToHost, stream));
    sync();
    if (h[0]) throw NumericalInstability("negative discriminant in drag velocity solve");
    std::memcpy(&vmax2, &bits, sizeof(double));
    finite = h[1] == 0;
  }

  double max_speed() {
    double v2;
    bool fin;
    max_speed2(v2, fin);
    if (!fin) return std::numeric_limits<double>::quiet_NaN();
    return std::sqrt(v2);
  }

  void get_cell(int64_t cell, double out[19]) {
    if (cell < 0 || cell >= cells) throw ConfigError("cell index out of range");
    ensure_pre();
    int64_t slot = cell, stride = ks;
    if (compact) {
      sync();
      slot = compact_slot_of(cell);
      stride = kp.ks;
      if (slot < 0) {  // non-fluid cells hold no populations in this layout
        for (int k = 0; k < 19; ++k) out[k] = 0.0;
        return;
      }
    }
    CK(cudaMemcpy2DAsync(out, sizeof(double), pre_buf() + slot, stride * sizeof(double),
                         sizeof(double), 19, cudaMemcpyDeviceToHost, stream));
    sync();
  }

  // simulation.cpp:354-369
  void macroscopic(int64_t cell, double& drho, double u[3]) {
    double fk[19], v[3];
    get_cell(cell, fk);
    moments(fk, params.rho0, drho, v);
    if (glbm_active) {
      const int z = plane_of(cell);
      double force[3];
      glbm_force_and_velocity(v, eps[z], K[z], cf, params.body_force, params.nu, u, force);
    } else {
      for (int i = 0; i < 3; ++i) u[i] = v[i] + 0.5 * params.body_force[i] / params.rho0;
    }
  }
};

