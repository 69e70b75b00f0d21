// Multi-GPU host path in C++ (include/porolb_gpu/porolb_gpu.hpp DistSimulation
// over csrc/dist.cpp): a sphere bed split into x slabs, stepped through
//   * the local transport (all slabs in this process, peer copies), and
//   * NCCL at world size 1 (one slab = the whole domain, periodic
//     self-exchange through ncclSend/ncclRecv, CUDA-graph replay),
// each compared bit for bit with the single-domain Simulation, plus the
// global profile and max speed.  Prints one JSON line.
//   dist_demo [nx ny nz slabs steps]      (default 256 64 96 2 23)
//   dist_demo ipc [nx ny nz steps]        the IPC transport at world size 2:
//       two processes (fork before any CUDA call, blobs all-gathered through
//       pipes) whose edge kernels store into each other's ghost buffers; each
//       compares its slab with its own single-domain run.
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "porolb_gpu/porolb_gpu.hpp"

namespace pl = porolb_gpu;

// seeded overlapping spheres in the lower half (64-bit LCG)
static pl::SpherePack make_pack(int nx, int ny, int nz) {
  pl::SpherePack pack;
  pack.box = {double(nx), double(ny), double(nz)};
  unsigned long long s = 12345;
  auto u01 = [&] {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return double(s >> 11) * 0x1.0p-53;
  };
  const int nsph = nx * ny * nz / 4000;
  for (int i = 0; i < nsph; ++i)
    pack.spheres.push_back({{u01() * nx, u01() * ny, 1.0 + u01() * 0.45 * (nz - 2)},
                            4.0 + 4.0 * u01()});
  return pack;
}

// world-2 IPC run of one rank; returns true if its slab, the global profile
// and the max speed match its own single-domain run
static bool ipc_rank(int rank, int rfd, int wfd, int nx, int ny, int nz, long steps) {
  const pl::SpherePack pack = make_pack(nx, ny, nz);
  pl::VoxelizeOptions opt;
  opt.wall_z_lo = opt.wall_z_hi = true;
  pl::FluidParams p = pl::relaxation_from_magic(0.2 / 3.0, 3.0 / 16.0);
  p.body_force = {1e-6, 0.0, 0.0};
  const pl::Dims d{nx, ny, nz};
  pl::Simulation single(pl::voxelize(pack, d, opt), p, pl::WallScheme::CLI);
  single.step(steps);
  const std::vector<double> want = single.pdfs();
  const pl::VoxelGeometry full = pl::voxelize(pack, d, opt);
  const int x0 = rank * nx / 2, x1 = (rank + 1) * nx / 2;
  pl::Simulation slab(pl::voxelize_slab(pack, d, opt, x0, x1), p, pl::WallScheme::CLI);
  auto allgather = [&](const std::vector<std::uint8_t>& mine) {
    std::vector<std::uint8_t> other(mine.size());
    if (write(wfd, mine.data(), mine.size()) != (ssize_t)mine.size()) throw std::runtime_error("pipe write");
    size_t got = 0;
    while (got < other.size()) {
      const ssize_t n = read(rfd, other.data() + got, other.size() - got);
      if (n <= 0) throw std::runtime_error("pipe read");
      got += (size_t)n;
    }
    std::vector<std::uint8_t> all;
    const auto& b0 = rank == 0 ? mine : other;
    const auto& b1 = rank == 0 ? other : mine;
    all.insert(all.end(), b0.begin(), b0.end());
    all.insert(all.end(), b1.begin(), b1.end());
    return all;
  };
  pl::DistSimulation dist = pl::DistSimulation::ipc(slab, rank, 2, allgather);
  dist.step(steps / 2);
  const pl::ProfileData prof_mid = dist.planar_profile();  // observables in the middle
  (void)prof_mid;
  dist.step(steps - steps / 2);
  const std::vector<double> got = slab.pdfs();
  const int w = x1 - x0;
  const long cells = long(nx) * ny * nz, lc = long(w) * ny * nz;
  bool ok = true;
  for (int k = 0; k < 19 && ok; ++k)
    for (long yz = 0; yz < long(ny) * nz && ok; ++yz)
      for (int x = 0; x < w; ++x) {
        const long c = yz * nx + x0 + x;
        if (full.flag(c) != 0) continue;
        if (std::memcmp(&got[k * lc + yz * w + x], &want[k * cells + c], sizeof(double))) {
          ok = false;
          break;
        }
      }
  const pl::ProfileData a = dist.planar_profile(), b = single.planar_profile();
  ok = ok && a.size() == b.size();
  for (std::size_t i = 0; ok && i < a.size(); ++i)
    ok = std::abs(a.u_superficial[i] - b.u_superficial[i]) <= 1e-12 * std::abs(b.u_max);
  ok = ok && dist.max_speed() == single.max_speed();
  return ok;
}

static int ipc_main(int argc, char** argv) {
  const int nx = argc > 2 ? std::atoi(argv[2]) : 128;
  const int ny = argc > 3 ? std::atoi(argv[3]) : 32;
  const int nz = argc > 4 ? std::atoi(argv[4]) : 48;
  const long steps = argc > 5 ? std::atol(argv[5]) : 15;
  int p01[2], p10[2];
  if (pipe(p01) || pipe(p10)) return 2;
  const pid_t child = fork();  // before any CUDA call in either process
  if (child < 0) return 2;
  if (child == 0) {
    bool ok = false;
    try {
      ok = ipc_rank(1, p01[0], p10[1], nx, ny, nz, steps);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "rank 1: %s\n", e.what());
    }
    _exit(ok ? 0 : 1);
  }
  bool ok0 = false;
  std::string err;
  try {
    ok0 = ipc_rank(0, p10[0], p01[1], nx, ny, nz, steps);
  } catch (const std::exception& e) {
    err = e.what();
  }
  int st = 0;
  waitpid(child, &st, 0);
  const bool ok1 = WIFEXITED(st) && WEXITSTATUS(st) == 0;
  std::printf("{\"ipc_world\": 2, \"dims\": [%d, %d, %d], \"steps\": %ld, \"rank0_ok\": %s, "
              "\"rank1_ok\": %s, \"error\": \"%s\"}\n",
              nx, ny, nz, steps, ok0 ? "true" : "false", ok1 ? "true" : "false", err.c_str());
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "ipc") == 0) return ipc_main(argc, argv);
  const int nx = argc > 1 ? std::atoi(argv[1]) : 256;
  const int ny = argc > 2 ? std::atoi(argv[2]) : 64;
  const int nz = argc > 3 ? std::atoi(argv[3]) : 96;
  const int P = argc > 4 ? std::atoi(argv[4]) : 2;
  const long steps = argc > 5 ? std::atol(argv[5]) : 23;
  // seeded overlapping spheres in the lower half (64-bit LCG)
  const pl::SpherePack pack = make_pack(nx, ny, nz);
  pl::VoxelizeOptions opt;
  opt.wall_z_lo = opt.wall_z_hi = true;
  pl::FluidParams p = pl::relaxation_from_magic(0.2 / 3.0, 3.0 / 16.0);
  p.body_force = {1e-6, 0.0, 0.0};
  const pl::Dims d{nx, ny, nz};

  pl::Simulation single(pl::voxelize(pack, d, opt), p, pl::WallScheme::CLI);
  single.step(steps);
  const std::vector<double> want = single.pdfs();
  const pl::ProfileData want_prof = single.planar_profile();
  const double want_vmax = single.max_speed();
  const pl::VoxelGeometry full = pl::voxelize(pack, d, opt);

  // slab r's populations against the single domain's columns [x0, x1)
  auto same = [&](const std::vector<double>& got, int x0, int x1) {
    const int w = x1 - x0;
    const long cells = long(nx) * ny * nz, lc = long(w) * ny * nz;
    for (int k = 0; k < 19; ++k)
      for (long yz = 0; yz < long(ny) * nz; ++yz)
        for (int x = 0; x < w; ++x) {
          const long c = yz * nx + x0 + x;
          if (full.flag(c) != 0) continue;  // fluid cells are defined
          if (std::memcmp(&got[k * lc + yz * w + x], &want[k * cells + c], sizeof(double)))
            return false;
        }
    return true;
  };
  auto prof_close = [&](const pl::ProfileData& a) {
    if (a.size() != want_prof.size() || a.height != want_prof.height || a.nu != want_prof.nu)
      return false;
    for (std::size_t i = 0; i < a.size(); ++i)
      if (std::abs(a.u_superficial[i] - want_prof.u_superficial[i]) >
          1e-12 * std::abs(want_prof.u_max))
        return false;
    return true;
  };

  // (a) local transport: P slabs in this process
  bool local_ok = true, local_prof = false;
  double local_vmax = 0.0;
  {
    std::vector<pl::Simulation> slabs;
    slabs.reserve(P);
    for (int r = 0; r < P; ++r)
      slabs.emplace_back(pl::voxelize_slab(pack, d, opt, r * nx / P, (r + 1) * nx / P), p,
                         pl::WallScheme::CLI);
    std::vector<pl::Simulation*> ptrs;
    for (auto& sl : slabs) ptrs.push_back(&sl);
    pl::DistSimulation dist(ptrs);
    dist.step(steps / 2);
    dist.step(steps - steps / 2);
    for (int r = 0; r < P; ++r) local_ok = local_ok && same(slabs[r].pdfs(), r * nx / P, (r + 1) * nx / P);
    local_prof = prof_close(dist.planar_profile());
    local_vmax = dist.max_speed();
  }
  // (b) NCCL at world size 1: periodic self-exchange, graph replay
  bool nccl_ok = false, nccl_prof = false;
  double nccl_vmax = 0.0;
  std::string nccl_err;
  try {
    pl::Simulation slab(pl::voxelize_slab(pack, d, opt, 0, nx), p, pl::WallScheme::CLI);
    pl::DistSimulation dist(slab, pl::DistSimulation::nccl_unique_id(), 0, 1);
    dist.step(1);      // K0 from the initial state (eager)
    dist.step(steps - 1);  // graph replays of two steps (+ one eager step when odd)
    nccl_ok = same(slab.pdfs(), 0, nx);
    nccl_prof = prof_close(dist.planar_profile());
    nccl_vmax = dist.max_speed();
  } catch (const std::exception& e) {
    nccl_err = e.what();
  }
  std::printf("{\"dims\": [%d, %d, %d], \"slabs\": %d, \"steps\": %ld, \"local_bitwise\": %s, "
              "\"local_profile\": %s, \"local_vmax_equal\": %s, \"nccl_bitwise\": %s, "
              "\"nccl_profile\": %s, \"nccl_vmax_equal\": %s, \"nccl_error\": \"%s\"}\n",
              nx, ny, nz, P, steps, local_ok ? "true" : "false", local_prof ? "true" : "false",
              local_vmax == want_vmax ? "true" : "false", nccl_ok ? "true" : "false",
              nccl_prof ? "true" : "false", nccl_vmax == want_vmax ? "true" : "false",
              nccl_err.c_str());
  return 0;
}
