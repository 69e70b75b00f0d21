// C-ABI runtime of the B200 time stepper: the drop-in for porolb::Simulation
// (reference proj/include/porolb/simulation.hpp:53-111, proj/src/simulation.cpp).
//
// State machine.  The reference keeps pre-collision f(n) in
// `cur` and runs collide -> push-stream -> links per step().  The device keeps
// either
//   pre : buffer[cur] holds f(n)            (after construction / set / materialise)
//   post: buffer[cur] holds g(n-1) = C(f(n-1)), and f(n) = P(g(n-1))
// step() from pre runs K0 (collide in place) and becomes post; step() from
// post runs K1 (fused pull-stream + bounce + collide) into the other buffer.
// Every observable first materialises f(n) = P(g) with KP (pre again), so
// reads always see exactly the reference's f(steps_done).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <sstream>
#include <vector>

#include "host_common.h"
#include "kernels.h"
#include "kparams.h"
#include "setup.h"
#include "staging.h"

#include "sim_impl.h"

namespace {

// Device temporary freed at scope exit.
struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <class T>
void upload(DevBuf& b, const T* host, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  CK(cudaMalloc(&b.p, sizeof(T) * n));
  CK(StagedUpload::get().h2d(b.p, host, sizeof(T) * n, st));
}

const char* setup_error_text(int code) {
  switch (code) {
    case kSetupErrCell: return "boundary link on a non-fluid or out-of-range cell";
    case kSetupErrDir: return "boundary link direction must be in 1..18";
    case kSetupErrFluidNeighbour: return "boundary link points to a fluid neighbour";
    case kSetupErrDuplicate: return "duplicate boundary link";
    case kSetupErrSecondNotFluid: return "CLI second_fluid is not a fluid cell";
    case kSetupErrSecondCell: return "CLI second_fluid must be the cell x_f1 - e_k";
    default: return "invalid boundary link";
  }
}

// Builds cell words, record bases and link records on the device from the
// caller's flags and link list (setup.cu).  Only the caller's arrays cross
// PCIe: flags 1 B/cell (+ ghost columns), links 25 B/link.
template <class Lap>
void device_setup(pgpu_sim* s, const pgpu_geometry* g, bool fill_sectors, Lap&& lap) {
  const cudaStream_t st = s->stream;
  const int64_t cells = s->cells, rows = (int64_t)s->ny * s->nz;
  const int nchunk = (s->nx + 31) / 32;
  const int64_t L = g->n_links;
  DevBuf flags, glo, ghi, count, scratch, total, lf, ls, ld, lq, lm, seen, res;
  upload(flags, g->flags, cells, st);
  if (s->slab) {
    upload(glo, g->ghost_flags_lo, rows, st);
    upload(ghi, g->ghost_flags_hi, rows, st);
  }
  lap("upload flags");
  upload(lf, g->link_fluid_cell, L, st);
  lap("upload link cells");
  upload(ls, g->link_second_fluid, L, st);
  upload(ld, g->link_direction, L, st);
  upload(lq, g->link_q, L, st);
  if (g->link_moving) upload(lm, g->link_moving, L, st);
  lap("upload other link arrays");

  CK(cudaMalloc(&s->d_cellw, sizeof(uint32_t) * cells));
  CK(cudaMalloc(&s->d_cellbase, sizeof(int32_t) * cells));
  CK(cudaMalloc(&s->d_chunkbase, sizeof(int32_t) * (rows * nchunk + 1)));
  CK(cudaMalloc(&count.p, sizeof(int32_t) * cells));
  CellSetupArgs ca;
  ca.flags = flags.as<uint8_t>();
  ca.ghost_lo = glo.as<uint8_t>();
  ca.ghost_hi = ghi.as<uint8_t>();
  ca.nx = s->nx;
  ca.ny = s->ny;
  ca.nz = s->nz;
  ca.px = s->per[0];
  ca.py = s->per[1];
  ca.pz = s->per[2];
  ca.slab = s->slab;
  ca.fill_sectors = fill_sectors;
  ca.cellw = s->d_cellw;
  ca.count = count.as<int32_t>();
  setup_cellwords(ca, st);
  const size_t sb = setup_scratch_bytes(cells);
  CK(cudaMalloc(&scratch.p, sb));
  CK(cudaMalloc(&total.p, sizeof(int64_t)));
  const int64_t tot = setup_bases(count.as<int32_t>(), s->d_cellbase, s->d_chunkbase, s->nx, rows,
                                  nchunk, scratch.p, sb, total.as<int64_t>(), st);
  if (tot < 0) throw CudaError("setup: scan scratch too small");
  if (tot > std::numeric_limits<int32_t>::max()) throw ConfigError("too many boundary links");
  if (L != tot) {
    std::ostringstream os;
    os << "boundary links (" << L << ") do not match the fluid->non-fluid lattice "
       << "directions of the flag field (" << tot << "); links must close exactly those directions";
    throw ConfigError(os.str());
  }
  s->n_links = tot;
  s->kp.nchunk = nchunk;
  lap("cell words+bases");

  // records: CLI coefficients / SBB / moving wall; validation in the same pass
  const bool cli = s->scheme == PGPU_CLI;
  if (L > 0 && (cli || g->link_moving)) CK(cudaMalloc(&s->d_recs, sizeof(LinkRec) * (L + 2)));
  const int64_t words = (L + 31) / 32;
  if (words) {
    CK(cudaMalloc(&seen.p, sizeof(uint32_t) * words));
    CK(cudaMemsetAsync(seen.p, 0, sizeof(uint32_t) * words, st));
  }
  struct Res {
    unsigned long long err, fallbacks;
    int moving;
  } host_res{~0ull, 0ull, 0};
  CK(cudaMalloc(&res.p, sizeof(Res)));
  CK(cudaMemcpyAsync(res.p, &host_res, sizeof(Res), cudaMemcpyHostToDevice, st));
  LinkSetupArgs la;
  la.n_links = L;
  la.cells = cells;
  la.nx = s->nx;
  la.ny = s->ny;
  la.nz = s->nz;
  la.px = s->per[0];
  la.py = s->per[1];
  la.pz = s->per[2];
  la.slab = s->slab;
  la.cli = cli;
  la.link_cell = lf.as<int64_t>();
  la.link_second = ls.as<int64_t>();
  la.link_dir = ld.as<int32_t>();
  la.link_q = lq.as<float>();
  la.link_moving = lm.as<uint8_t>();
  la.cellw = s->d_cellw;
  la.cellbase = s->d_cellbase;
  la.recs = s->d_recs;
  Res* dr = res.as<Res>();
  setup_links(la, seen.as<uint32_t>(), &dr->err, &dr->fallbacks, &dr->moving, st);
  CK(cudaMemcpyAsync(&host_res, res.p, sizeof(Res), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (host_res.err != ~0ull) throw ConfigError(setup_error_text((int)(host_res.err & 0xFF)));
  s->cli_fallbacks = cli ? (int32_t)host_res.fallbacks : 0;
  s->any_moving = host_res.moving != 0;
  if (s->d_recs && !s->records_needed()) {
    CK(cudaFree(s->d_recs));
    s->d_recs = nullptr;
  }
  s->kp.links = s->d_recs;
  s->kp.nrec = s->d_recs ? L : 0;
  if (s->d_recs) s->ensure_linkdesc();
  lap("link records");
}

}  // namespace

extern "C" {

// simulation.hpp:113-116, simulation.cpp:436-439: streaming of a field's
// current buffer into the next one, then the swap.  The field is the caller's
// host arrays (reference layout); on return `cur` holds the streamed state
// (the reference's field.cur() after the swap) and `next` the previous one.
int pgpu_stream_field(const int32_t dims[3], const uint8_t periodic[3], const uint8_t* flags,
                      double* cur, double* next, int32_t device) {
  return guard([&] {
    if (!dims || !periodic || !flags || !cur || !next) throw std::invalid_argument("null pointer");
    if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0) throw ConfigError("voxel dims must be positive");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device available: the B200 path has no CPU fallback");
    }
    if (device < 0 || device >= ndev) throw CudaError("device index out of range");
    CK(cudaSetDevice(device));
    const int64_t cells = (int64_t)dims[0] * dims[1] * dims[2];
    const size_t bytes = sizeof(double) * 19 * (size_t)cells;
    DevBuf df, dc, dn;
    CK(cudaMalloc(&df.p, (size_t)cells));
    CK(cudaMalloc(&dc.p, bytes));
    CK(cudaMalloc(&dn.p, bytes));
    CK(cudaMemcpy(df.p, flags, (size_t)cells, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc.p, cur, bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dn.p, next, bytes, cudaMemcpyHostToDevice));
    const int d[3] = {dims[0], dims[1], dims[2]};
    const int per[3] = {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0};
    launch_stream_field(df.as<uint8_t>(), d, per, dc.as<double>(), dn.as<double>(), 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(next, dc.p, bytes, cudaMemcpyDeviceToHost));  // swap: old cur
    CK(cudaMemcpy(cur, dn.p, bytes, cudaMemcpyDeviceToHost));   // streamed
  });
}

int pgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pgpu_create(const pgpu_geometry* g, const pgpu_fluid_params* params, int32_t scheme,
                int32_t device, pgpu_sim** out) {
  return guard([&] {
    if (!g || !params || !out) throw std::invalid_argument("null pointer");
    *out = nullptr;
    if (g->dims[0] <= 0 || g->dims[1] <= 0 || g->dims[2] <= 0) throw ConfigError("voxel dims must be positive");
    if (!g->flags || !g->porosity) throw std::invalid_argument("geometry needs flags and porosity");
    if (g->n_links < 0 || (g->n_links > 0 && (!g->link_fluid_cell || !g->link_second_fluid ||
                                              !g->link_direction || !g->link_q)))
      throw std::invalid_argument("bad link arrays");
    if (scheme != PGPU_SBB && scheme != PGPU_CLI) throw ConfigError("unknown wall scheme");
    if (g->slab && (!g->ghost_flags_lo || !g->ghost_flags_hi)) throw ConfigError("slab geometry needs ghost flags");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device available: the B200 path has no CPU fallback");
    }
    if (device < 0 || device >= ndev) throw CudaError("device index out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      std::ostringstream os;
      os << "device " << device << " is sm_" << prop.major << prop.minor
         << "; this library is built for sm_100a (B200) only";
      throw CudaError(os.str());
    }
    std::unique_ptr<pgpu_sim> s(new pgpu_sim());
    s->device = device;
    CK(cudaSetDevice(device));
    static std::once_flag preload;
    std::call_once(preload, preload_kernels);
    // L2 fetch granularity hint (bytes): the sweep's loads are 8-byte-per-cell
    // and sector-sparse next to solid cells (experiment knob PGPU_L2_FETCH).
    if (const char* e = std::getenv("PGPU_L2_FETCH")) {
      CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)std::atoi(e)));
    }
    CK(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking));
    s->stream = s->own_stream;
    s->nx = g->dims[0];
    s->ny = g->dims[1];
    s->nz = g->dims[2];
    for (int a = 0; a < 3; ++a) s->per[a] = g->periodic[a] != 0;
    s->slab = g->slab != 0;
    s->x_offset = g->x_offset;
    s->global_nx = g->slab ? g->global_nx : g->dims[0];
    s->cells = (int64_t)s->nx * s->ny * s->nz;
    if (s->cells > (int64_t)std::numeric_limits<int32_t>::max()) throw ConfigError("domain too large for one device");
    s->ks = (s->cells + 31) / 32 * 32;
    s->params = *params;
    s->scheme = scheme;
    s->porosity.assign(g->porosity, g->porosity + s->nz);
    s->plane_fluid_count.assign(s->nz, 0);
    for (int z = 0; z < s->nz; ++z)  // simulation.cpp:93-96
      s->plane_fluid_count[z] = static_cast<int64_t>(
          std::llround(s->porosity[z] * static_cast<double>(s->nx) * s->ny));
    s->has_lo = g->has_wall_plane_lo != 0;
    s->has_hi = g->has_wall_plane_hi != 0;
    s->lo = g->wall_plane_lo;
    s->hi = g->wall_plane_hi;
    s->fluid_cells = g->fluid_cells;
    const bool trace = std::getenv("PGPU_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!trace) return;
      const auto t1 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[pgpu] create %-22s %8.1f ms\n", what,
                   std::chrono::duration<double, std::milli>(t1 - t0).count());
      t0 = t1;
    };
    if (const char* e = std::getenv("PGPU_MATH")) s->fast = e[0] == 'f';
    if (const char* e = std::getenv("PGPU_FOLD")) s->fold_enabled = e[0] == '1';
    const char* fill_env = std::getenv("PGPU_FILL_SECTORS");
    device_setup(s.get(), g, !(fill_env && fill_env[0] == '0'), lap);

    {  // two PDF grids well inside the 126 MB L2 -> persistent multi-step sweeps
      const char* e = std::getenv("PGPU_PERSISTENT");
      const double state_bytes = 2.0 * 19.0 * 8.0 * (double)s->ks;
      s->persistent = !s->slab && (e ? e[0] == '1' : state_bytes <= 48e6);
    }
    // Layout: fluid-only for every domain that is not L2-resident (those run
    // the persistent dense sweep).  With the units sweep it is the faster
    // layout even for a walled channel without solids inside (C5: 0.92 against
    // 0.84 of the dense sweep); the dense layout remains for PGPU_LAYOUT=dense
    // and for more than 226 M fluid cells.  PGPU_LAYOUT=dense|compact overrides.
    int64_t sweep_ks = s->ks;
    {
      const char* e = std::getenv("PGPU_LAYOUT");
      const bool want = e ? e[0] == 'c' : !s->persistent;
      if (want) {
        const int64_t rows = (int64_t)s->ny * s->nz;
        CK(cudaMalloc(&s->d_ctab, sizeof(ChunkEnt) * rows * s->kp.nchunk));
        const int64_t nf = build_ctab(s->d_cellw, s->nx, rows, s->kp.nchunk, s->d_ctab, s->stream);
        const int64_t ksc = std::max<int64_t>(32, (nf + 31) / 32 * 32);
        // unsigned 32-bit slot offsets must reach all 19 planes (226 M fluid cells)
        s->compact = 19 * ksc <= (int64_t)std::numeric_limits<uint32_t>::max();
        if (s->compact) {
          sweep_ks = ksc;
          s->nfluid_slots = nf;
          s->persistent = false;
        } else {
          CK(cudaFree(s->d_ctab));
          s->d_ctab = nullptr;
        }
      }
    }
    // device buffers: two PDF grids, zero-filled like the reference
    const size_t fbytes = sizeof(double) * 19 * (size_t)sweep_ks;
    for (int b = 0; b < 2; ++b) {
      CK(cudaMalloc(&s->f[b], fbytes));
      CK(cudaMemsetAsync(s->f[b], 0, fbytes, s->stream));
    }
    CK(cudaMalloc(&s->d_feq, sizeof(double) * 19));
    CK(cudaMalloc(&s->d_flags, sizeof(int) * 2));
    CK(cudaMalloc(&s->d_vmax, sizeof(unsigned long long)));
    CK(cudaMalloc(&s->d_sums, sizeof(double) * s->nz));
    CK(cudaMalloc(&s->d_tickets, sizeof(uint32_t) * 2));
    CK(cudaMemsetAsync(s->d_tickets, 0, sizeof(uint32_t) * 2, s->stream));
    KParams& kp = s->kp;
    kp.nx = s->nx;
    kp.ny = s->ny;
    kp.nz = s->nz;
    kp.px = s->per[0];
    kp.py = s->per[1];
    kp.pz = s->per[2];
    kp.ks = sweep_ks;
    kp.ksd = s->ks;
    kp.ctab = s->d_ctab;
    for (int j = 0; j < 19; ++j) kp.poff[j] = s->compact ? (uint32_t)(j * sweep_ks) : 0u;
    for (int j = 0; j < 19; ++j) {
      const int64_t d = kE[j][0] + (int64_t)kE[j][1] * s->nx + (int64_t)kE[j][2] * s->nx * s->ny;
      kp.pull_off[j] = (int64_t)j * s->ks - d;
      kp.bounce_delta[j] = (int64_t)opposite(j) * s->ks - kp.pull_off[j];
      kp.plane_off[j] = (int64_t)j * s->ks;
    }
    kp.cellw = s->d_cellw;
    kp.cellbase = s->d_cellbase;
    kp.chunkbase = s->d_chunkbase;
    // fluid-only K1 kernel (PGPU_SWEEP=tma|cpipe overrides the default); the
    // TMA sweep addresses the link sources of every scheme through the
    // per-record descriptors
    if (s->compact) s->ensure_linkdesc();
    kp.tickets = s->d_tickets;
    // evict-first stores only where the state dwarfs L2 (C4); smaller domains
    // keep the new state in L2 for the next sweep (read first, zrev order)
    {
      const char* e = std::getenv("PGPU_STREAM_STORES");
      const double buf_bytes = 19.0 * 8.0 * (double)sweep_ks;
      kp.stream_stores = e ? (e[0] == '1') : (buf_bytes > 4.0 * 126e6);
      const char* z = std::getenv("PGPU_ZREV");
      s->zrev_on = !(z && z[0] == '0');
    }
    if (const char* e = std::getenv("PGPU_SWEEP"))
      kp.sweep = e[0] == 'u' ? PGPU_SWEEP_UNITS
                 : e[0] == 't' ? PGPU_SWEEP_TMA : (e[0] == 'c' ? PGPU_SWEEP_CPIPE : PGPU_SWEEP_AUTO);
    // AUTO: the fluid-only layout runs the units sweep
    if (kp.sweep == PGPU_SWEEP_UNITS || (kp.sweep == PGPU_SWEEP_AUTO && s->compact)) s->ensure_units();
    lap("alloc pdfs");
    s->refresh_params();
    CK(cudaStreamSynchronize(s->stream));
    lap("params+sync");
    *out = s.release();
  });
}

int pgpu_destroy(pgpu_sim* sim) {
  return guard([&] { delete sim; });
}

#define SIM_CHECK() \
  if (!sim) throw std::invalid_argument("null simulation handle"); \
  CK(cudaSetDevice(sim->device))

int pgpu_set_stream(pgpu_sim* sim, void* stream) {
  return guard([&] {
    SIM_CHECK();
    CK(cudaStreamSynchronize(sim->stream));
    sim->stream = stream ? static_cast<cudaStream_t>(stream) : sim->own_stream;
    sim->drop_graphs();
  });
}

int pgpu_get_stream(pgpu_sim* sim, void** stream) {
  return guard([&] {
    SIM_CHECK();
    *stream = sim->stream;
  });
}

int pgpu_synchronize(pgpu_sim* sim) {
  return guard([&] {
    SIM_CHECK();
    sim->sync();
  });
}

int pgpu_get_params(pgpu_sim* sim, pgpu_fluid_params* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->params;
  });
}

// Math mode (not in the reference: the reference has one arithmetic):
// PGPU_MATH_EXACT reproduces the reference bit for bit, PGPU_MATH_FAST is the
// contracted collision with folded CLI links (<= 1e-12 relative).  A switch
// mid-run materialises f(n) first when the stored state's meaning changes.
int pgpu_set_math_mode(pgpu_sim* sim, int32_t mode) {
  return guard([&] {
    SIM_CHECK();
    if (mode != PGPU_MATH_EXACT && mode != PGPU_MATH_FAST) throw ConfigError("unknown math mode");
    const bool want = mode == PGPU_MATH_FAST;
    if (want == sim->fast) return;
    if (sim->slab && sim->pending) throw ConfigError("split step in progress");
    if (sim->post && sim->compact && sim->d_recs) sim->ensure_pre();  // folded <-> plain slots
    sim->sync();
    sim->fast = want;
    sim->refresh_params();
    sim->sync();
  });
}

// K1 kernel of the fluid-only layout (not in the reference: a schedule choice,
// results are bit-identical between them).
int pgpu_set_sweep_kernel(pgpu_sim* sim, int32_t kind) {
  return guard([&] {
    SIM_CHECK();
    if (kind != PGPU_SWEEP_AUTO && kind != PGPU_SWEEP_CPIPE && kind != PGPU_SWEEP_TMA &&
        kind != PGPU_SWEEP_UNITS)
      throw ConfigError("unknown sweep kernel");
    if (kind == sim->kp.sweep) return;
    sim->sync();
    sim->kp.sweep = kind;
    if (kind == PGPU_SWEEP_UNITS) sim->ensure_units();
    sim->drop_graphs();  // graphs hold the kernel parameters by value
  });
}

int pgpu_get_sweep_kernel(pgpu_sim* sim, int32_t* kind) {
  return guard([&] {
    SIM_CHECK();
    *kind = sim->resolved_sweep();
  });
}

int pgpu_device_bytes(pgpu_sim* sim, int64_t* bytes) {
  return guard([&] {
    SIM_CHECK();
    *bytes = sim->device_bytes();
  });
}

int pgpu_get_layout(pgpu_sim* sim, int32_t* layout) {
  return guard([&] {
    SIM_CHECK();
    *layout = sim->compact ? PGPU_LAYOUT_FLUID_ONLY
                           : (sim->persistent ? PGPU_LAYOUT_DENSE_PERSISTENT : PGPU_LAYOUT_DENSE);
  });
}

int pgpu_get_math_mode(pgpu_sim* sim, int32_t* mode) {
  return guard([&] {
    SIM_CHECK();
    *mode = sim->fast ? PGPU_MATH_FAST : PGPU_MATH_EXACT;
  });
}

int pgpu_set_body_force(pgpu_sim* sim, const double g[3]) {
  return guard([&] {
    SIM_CHECK();
    sim->sync();
    for (int i = 0; i < 3; ++i) sim->params.body_force[i] = g[i];
    sim->refresh_params();
  });
}

// simulation.cpp:104-112
int pgpu_set_lid_velocity(pgpu_sim* sim, const double u[3]) {
  return guard([&] {
    SIM_CHECK();
    sim->sync();
    for (int i = 0; i < 3; ++i) sim->lid[i] = u[i];
    // The stored post-collision state g(n-1) still owes the pull
    // f(n) = P(g(n-1)) with the OLD wall velocity (the reference streamed and
    // bounced step n before this call, simulation.cpp:325-342): materialise
    // f(n) first, the next step re-collides from it.  (Also required by the
    // folded CLI slots of math mode fast.)
    if (sim->post) sim->ensure_pre();
    sim->ensure_records();  // SBB scheme: all-SBB records first
    if (sim->d_recs) {
      DevBuf any;
      CK(cudaMalloc(&any.p, sizeof(int)));
      CK(cudaMemsetAsync(any.p, 0, sizeof(int), sim->stream));
      mark_lid_links(sim->d_cellw, sim->d_cellbase, sim->d_recs, sim->nx, sim->ny, sim->nz,
                     any.as<int>(), sim->stream);
      int hit = 0;
      CK(cudaMemcpyAsync(&hit, any.p, sizeof(int), cudaMemcpyDeviceToHost, sim->stream));
      CK(cudaStreamSynchronize(sim->stream));
      if (hit) sim->any_moving = true;
    }
    sim->refresh_params();
  });
}

// simulation.cpp:114-119 (+ all_free, :12-21)
int pgpu_set_porous(pgpu_sim* sim, int32_t n, const double* eps, const double* K,
                    const double* wp, const double* wm, double c_F, int32_t eps_in_eq) {
  return guard([&] {
    SIM_CHECK();
    if (n != sim->nz) throw ConfigError("GLBM plane parameters must cover every z-plane");
    if (!eps || !K || !wp || !wm) throw std::invalid_argument("null array");
    sim->sync();
    sim->porous = true;
    sim->eps.assign(eps, eps + n);
    sim->K.assign(K, K + n);
    sim->gwp.assign(wp, wp + n);
    sim->gwm.assign(wm, wm + n);
    sim->cf = c_F;
    sim->eps_in_eq = eps_in_eq != 0;
    bool free = c_F == 0.0;
    for (double e : sim->eps)
      if (e != 1.0) free = false;
    for (double k : sim->K)
      if (std::isfinite(k)) free = false;
    sim->glbm_active = !free;
    sim->refresh_params();
  });
}

// simulation.cpp:121-128
int pgpu_initialize_equilibrium(pgpu_sim* sim, double delta_rho, const double u[3]) {
  return guard([&] {
    SIM_CHECK();
    if (sim->slab && sim->pending) throw ConfigError("split step in progress");
    double feq[19];
    equilibrium(delta_rho, u, sim->params.rho0, feq);
    if (sim->post) {  // the dead buffer becomes the pre-collision state
      sim->cur = 1 - sim->cur;
      sim->post = false;
    }
    CK(cudaMemcpyAsync(sim->d_feq, feq, sizeof(feq), cudaMemcpyHostToDevice, sim->stream));
    if (sim->compact)
      launch_fill_compact(sim->kp, sim->nfluid_slots, sim->pre_buf(), sim->d_feq, sim->stream);
    else
      launch_fill_equilibrium(sim->kp, sim->cells, sim->pre_buf(), sim->d_feq, sim->stream);
    sim->check_launch();
    ++sim->launches;
    sim->sync();
  });
}

int pgpu_step(pgpu_sim* sim, int64_t n) {
  return guard([&] {
    SIM_CHECK();
    if (n < 0) throw ConfigError("step count must be non-negative");
    sim->step(n);
  });
}

// Instantiate the multi-step CUDA graphs of both buffer parities now (no
// time step is taken), so a timed step() does not pay their capture.
int pgpu_prepare(pgpu_sim* sim) {
  return guard([&] {
    SIM_CHECK();
    sim->prepare();
  });
}

int pgpu_steps_done(pgpu_sim* sim, int64_t* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->steps;
  });
}

int pgpu_cli_fallback_count(pgpu_sim* sim, int32_t* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->scheme == PGPU_CLI ? sim->cli_fallbacks : 0;
  });
}

int pgpu_fluid_cells(pgpu_sim* sim, int64_t* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->fluid_cells;
  });
}

int pgpu_get_flags(pgpu_sim* sim, uint8_t* out) {
  return guard([&] {
    SIM_CHECK();
    if (!out) throw std::invalid_argument("null output");
    DevBuf tmp;
    CK(cudaMalloc(&tmp.p, sim->cells));
    unpack_flags(sim->d_cellw, tmp.as<uint8_t>(), sim->cells, sim->stream);
    CK(cudaMemcpyAsync(out, tmp.p, sim->cells, cudaMemcpyDeviceToHost, sim->stream));
    CK(cudaStreamSynchronize(sim->stream));
  });
}

int pgpu_dims(pgpu_sim* sim, int32_t dims[3]) {
  return guard([&] {
    SIM_CHECK();
    dims[0] = sim->nx;
    dims[1] = sim->ny;
    dims[2] = sim->nz;
  });
}

int pgpu_get_pdfs(pgpu_sim* sim, double* out) {
  return guard([&] {
    SIM_CHECK();
    if (!out) throw std::invalid_argument("null output");
    sim->ensure_pre();
    if (!sim->compact) {
      CK(cudaMemcpy2DAsync(out, sim->cells * sizeof(double), sim->pre_buf(),
                           sim->ks * sizeof(double), sim->cells * sizeof(double), 19,
                           cudaMemcpyDeviceToHost, sim->stream));
    } else {  // expand z-chunks into the dead sweep buffer, then copy each out
      Nvtx r("get_pdfs expand");
      const int64_t plane = (int64_t)sim->nx * sim->ny;
      double* stage = sim->f[1 - sim->cur];
      for (int z0 = 0; z0 < sim->nz; z0 += sim->io_planes()) {
        const int nzc = std::min(sim->io_planes(), sim->nz - z0);
        if (z0) CK(cudaStreamSynchronize(sim->stream));  // staging reused
        launch_compact_io(true, sim->kp, sim->pre_buf(), stage, z0, nzc, sim->stream);
        sim->check_launch();
        ++sim->launches;
        const size_t w = sizeof(double) * (size_t)(nzc * plane);
        CK(cudaMemcpy2DAsync(out + z0 * plane, sim->cells * sizeof(double), stage, w, w, 19,
                             cudaMemcpyDeviceToHost, sim->stream));
      }
    }
    sim->sync();
  });
}

int pgpu_set_pdfs(pgpu_sim* sim, const double* in) {
  return guard([&] {
    SIM_CHECK();
    if (!in) throw std::invalid_argument("null input");
    if (sim->slab && sim->pending) throw ConfigError("split step in progress");
    sim->sync();
    if (sim->post) sim->cur = 1 - sim->cur;
    sim->post = false;
    if (!sim->compact) {
      CK(cudaMemcpy2DAsync(sim->pre_buf(), sim->ks * sizeof(double), in,
                           sim->cells * sizeof(double), sim->cells * sizeof(double), 19,
                           cudaMemcpyHostToDevice, sim->stream));
    } else {  // z-chunks through the dead sweep buffer, packed into fluid slots
      const int64_t plane = (int64_t)sim->nx * sim->ny;
      double* stage = sim->f[1 - sim->cur];
      for (int z0 = 0; z0 < sim->nz; z0 += sim->io_planes()) {
        const int nzc = std::min(sim->io_planes(), sim->nz - z0);
        const size_t w = sizeof(double) * (size_t)(nzc * plane);
        CK(cudaMemcpy2DAsync(stage, w, in + z0 * plane, sim->cells * sizeof(double), w, 19,
                             cudaMemcpyHostToDevice, sim->stream));
        launch_compact_io(false, sim->kp, sim->pre_buf(), stage, z0, nzc, sim->stream);
        sim->check_launch();
        ++sim->launches;
      }
    }
    sim->sync();
  });
}

int pgpu_get_cell_populations(pgpu_sim* sim, int64_t cell, double out[19]) {
  return guard([&] {
    SIM_CHECK();
    sim->get_cell(cell, out);
  });
}

int pgpu_set_cell_populations(pgpu_sim* sim, int64_t cell, const double in[19]) {
  return guard([&] {
    SIM_CHECK();
    if (cell < 0 || cell >= sim->cells) throw ConfigError("cell index out of range");
    sim->ensure_pre();
    int64_t slot = cell, stride = sim->ks;
    if (sim->compact) {
      sim->sync();
      slot = sim->compact_slot_of(cell);
      stride = sim->kp.ks;
      if (slot < 0) return;  // non-fluid cells hold no populations in this layout
    }
    CK(cudaMemcpy2DAsync(sim->pre_buf() + slot, stride * sizeof(double), in, sizeof(double),
                         sizeof(double), 19, cudaMemcpyHostToDevice, sim->stream));
    sim->sync();
  });
}

int pgpu_macroscopic(pgpu_sim* sim, int64_t cell, double* delta_rho, double u[3]) {
  return guard([&] {
    SIM_CHECK();
    sim->macroscopic(cell, *delta_rho, u);
  });
}

int pgpu_macroscopic_fields(pgpu_sim* sim, double* drho, double* ux, double* uy, double* uz) {
  return guard([&] {
    SIM_CHECK();
    sim->ensure_pre();
    sim->reset_flags();
    double* scratch = sim->scratch(4 * sim->ks);
    double* outs[4] = {drho, ux, uy, uz};
    double* dev[4];
    for (int i = 0; i < 4; ++i) dev[i] = outs[i] ? scratch + (int64_t)i * sim->ks : nullptr;
    launch_macro_fields(sim->glbm_active, sim->kp, sim->pre_buf(), dev[0], dev[1], dev[2],
                        dev[3], sim->d_flags, sim->stream);
    sim->check_launch();
    ++sim->launches;
    for (int i = 0; i < 4; ++i)
      if (outs[i])
        CK(cudaMemcpyAsync(outs[i], dev[i], sizeof(double) * sim->cells, cudaMemcpyDeviceToHost,
                           sim->stream));
    sim->check_err_flag();
  });
}

int pgpu_planar_profile(pgpu_sim* sim, int32_t axis, double* z, double* u_sup, double* u_int,
                        double* eps, double* u_norm, pgpu_profile_meta* meta) {
  return guard([&] {
    SIM_CHECK();
    if (!z || !u_sup || !u_int || !eps || !u_norm || !meta) throw std::invalid_argument("null output");
    sim->planar_profile(axis, z, u_sup, u_int, eps, u_norm, meta);
  });
}

int pgpu_plane_sums(pgpu_sim* sim, int32_t axis, double* sums_nz) {
  return guard([&] {
    SIM_CHECK();
    std::vector<double> s;
    sim->plane_sums(axis, s);
    std::memcpy(sums_nz, s.data(), sizeof(double) * s.size());
  });
}

int pgpu_max_speed(pgpu_sim* sim, double* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->max_speed();
  });
}

int pgpu_max_speed2(pgpu_sim* sim, double* vmax2, int32_t* finite) {
  return guard([&] {
    SIM_CHECK();
    bool fin;
    sim->max_speed2(*vmax2, fin);
    *finite = fin ? 1 : 0;
  });
}

// simulation.cpp:441-480
int pgpu_run_to_steady_state(pgpu_sim* sim, const pgpu_steady_config* cfg,
                             pgpu_run_stats* stats, double* z, double* u_sup, double* u_int,
                             double* eps, double* u_norm, pgpu_profile_meta* meta) {
  return guard([&] {
    SIM_CHECK();
    if (!cfg || !stats) throw std::invalid_argument("null pointer");
    const int nz = sim->nz;
    std::vector<double> pz(nz), ps(nz), pi(nz), pe(nz), pn(nz);
    std::vector<double> cz(nz), cs(nz), ci(nz), ce(nz), cn(nz);
    pgpu_profile_meta pm{}, cm{};
    *stats = pgpu_run_stats{};
    stats->cli_fallbacks = sim->scheme == PGPU_CLI ? sim->cli_fallbacks : 0;
    sim->planar_profile(0, pz.data(), ps.data(), pi.data(), pe.data(), pn.data(), &pm);
    const auto t0 = std::chrono::steady_clock::now();
    int64_t done = 0;
    while (done < cfg->max_steps) {
      const int64_t burst = std::min<int64_t>(cfg->check_interval, cfg->max_steps - done);
      sim->step(burst);
      done += burst;
      const double vmax = sim->max_speed();
      if (!std::isfinite(vmax) || vmax > cfg->max_speed) {
        std::ostringstream os;
        os << "instability after " << done << " steps: max |u| = " << vmax;
        throw NumericalInstability(os.str());
      }
      sim->planar_profile(0, cz.data(), cs.data(), ci.data(), ce.data(), cn.data(), &cm);
      double diff = 0.0, scale = 0.0;
      for (int i = 0; i < cm.n_planes; ++i) {
        diff = std::max(diff, std::abs(cs[i] - ps[i]));
        scale = std::max(scale, std::abs(cs[i]));
      }
      stats->residual = scale > 0.0 ? diff / scale : diff;
      std::swap(pz, cz);
      std::swap(ps, cs);
      std::swap(pi, ci);
      std::swap(pe, ce);
      std::swap(pn, cn);
      pm = cm;
      if (stats->residual < cfg->tolerance) {
        stats->converged = 1;
        break;
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    stats->steps = done;
    stats->seconds = std::chrono::duration<double>(t1 - t0).count();
    stats->mlups = stats->seconds > 0.0
                       ? static_cast<double>(sim->cells) * done / stats->seconds / 1e6
                       : 0.0;
    if (meta) {
      *meta = pm;
      for (int i = 0; i < pm.n_planes; ++i) {
        if (z) z[i] = pz[i];
        if (u_sup) u_sup[i] = ps[i];
        if (u_int) u_int[i] = pi[i];
        if (eps) eps[i] = pe[i];
        if (u_norm) u_norm[i] = pn[i];
      }
    }
  });
}

int pgpu_launch_count(pgpu_sim* sim, int64_t* out) {
  return guard([&] {
    SIM_CHECK();
    *out = sim->launches;
  });
}

int pgpu_algorithmic_bytes_per_step(pgpu_sim* sim, double* out) {
  return guard([&] {
    SIM_CHECK();
    *out = 304.0 * static_cast<double>(sim->fluid_cells);
  });
}

// ---- multi-GPU halo ---------------------------------------------------------
int pgpu_halo_elems(pgpu_sim* sim, int64_t* out) {
  return guard([&] {
    SIM_CHECK();
    *out = 5 * (int64_t)sim->ny * sim->nz;
  });
}

int pgpu_set_halo_buffers(pgpu_sim* sim, double* send_lo, double* send_hi, double* recv_lo0,
                          double* recv_lo1, double* recv_hi0, double* recv_hi1) {
  return guard([&] {
    SIM_CHECK();
    if (!sim->slab) throw ConfigError("halo buffers need a slab geometry");
    if (!send_lo || !send_hi || !recv_lo0 || !recv_lo1 || !recv_hi0 || !recv_hi1)
      throw std::invalid_argument("null halo buffer");
    sim->send_lo = send_lo;
    sim->send_hi = send_hi;
    sim->recv_lo[0] = recv_lo0;
    sim->recv_lo[1] = recv_lo1;
    sim->recv_hi[0] = recv_hi0;
    sim->recv_hi[1] = recv_hi1;
  });
}

int pgpu_halo_parity(pgpu_sim* sim, int32_t* parity) {
  return guard([&] {
    SIM_CHECK();
    *parity = 1 - sim->ghost_cur;
  });
}

int pgpu_step_part_on(pgpu_sim* sim, int32_t part, void* stream) {
  return guard([&] {
    SIM_CHECK();
    if (!sim->slab) throw ConfigError("split steps need a slab geometry");
    if (!sim->send_lo) throw ConfigError("halo buffers not set");
    // the part's kernels go to `stream` (null: the simulation's stream)
    const cudaStream_t keep = sim->stream;
    if (stream) sim->stream = static_cast<cudaStream_t>(stream);
    struct Restore {
      pgpu_sim* s;
      cudaStream_t st;
      ~Restore() { s->stream = st; }
    } restore{sim, keep};
    if (part == 0) {
      if (sim->pending) throw ConfigError("previous split step not finished");
      if (!sim->post) {
        sim->k0();  // collide-only, fills the send buffers; no ghost reads
        sim->pending = 1;
      } else {
        sim->k1(1);  // edge columns: read ghosts, fill send buffers
        sim->pending = 2;
      }
    } else if (part == 1) {
      if (!sim->pending) throw ConfigError("step part 0 must come first");
      if (sim->pending == 2) sim->k1(2);  // interior columns
    } else {
      throw ConfigError("part must be 0 or 1");
    }
  });
}

int pgpu_step_part(pgpu_sim* sim, int32_t part) { return pgpu_step_part_on(sim, part, nullptr); }

int pgpu_step_finish(pgpu_sim* sim) {
  return guard([&] {
    SIM_CHECK();
    if (!sim->pending) throw ConfigError("no split step in progress");
    if (sim->pending == 1)
      sim->post = true;
    else
      sim->cur = 1 - sim->cur;
    sim->pending = 0;
    sim->ghost_cur = 1 - sim->ghost_cur;
    ++sim->steps;
  });
}

}  // extern "C"
