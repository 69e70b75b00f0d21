// Multi-GPU host path in C++ (include/porolb_gpu/porolb_gpu.hpp DistSimulation
// over csrc/dist.cpp): a sphere bed split into x slabs, stepped through
//   * the local transport (all slabs in this process, peer copies), and
//   * NCCL at world size 1 (one slab = the whole domain, periodic
//     self-exchange through ncclSend/ncclRecv, CUDA-graph replay),
// each compared bit for bit with the single-domain Simulation, plus the
// global profile and max speed.  Prints one JSON line.
//   dist_demo [nx ny nz slabs steps]      (default 256 64 96 2 23)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "porolb_gpu/porolb_gpu.hpp"

namespace pl = porolb_gpu;

int main(int argc, char** argv) {
  const int nx = argc > 1 ? std::atoi(argv[1]) : 256;
  const int ny = argc > 2 ? std::atoi(argv[2]) : 64;
  const int nz = argc > 3 ? std::atoi(argv[3]) : 96;
  const int P = argc > 4 ? std::atoi(argv[4]) : 2;
  const long steps = argc > 5 ? std::atol(argv[5]) : 23;
  // seeded overlapping spheres in the lower half (64-bit LCG)
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
