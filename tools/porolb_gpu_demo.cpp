// C++ drop-in demo: the reference's own callers, rewritten against
// include/porolb_gpu/porolb_gpu.hpp (the only change a reference user makes is
// the namespace and the link line).  Mirrors
//   * acceptance criterion 1, Poiseuille exactness at Lambda = 3/16
//     (proj/tests/acceptance/acceptance_main.cpp:59-75);
//   * run_bench / time_scheme, SBB vs CLI on the 128^3 sphere-in-box bench
//     geometry (proj/src/bench.cpp:17-66; acceptance criterion 10).
// Prints one JSON object.  Build: python paper_1507_06565_b200/build.py --all
#include <chrono>
#include <cmath>
#include <cstdio>
#include <string>

#include "porolb_gpu/porolb_gpu.hpp"

using namespace porolb_gpu;

namespace {

// acceptance_main.cpp:39-56 channel_config + :59-75 criterion 1
double poiseuille_max_rel_err(bool& converged) {
  const int H = 32;
  const double nu = 1.0 / 6.0, g = 1e-8;
  VoxelizeOptions opt;
  opt.periodic = {true, true, false};
  opt.wall_z_lo = opt.wall_z_hi = true;
  const VoxelGeometry geom = make_box_geometry({4, 4, H + 2}, opt);
  FluidParams p = relaxation_from_magic(nu, 3.0 / 16.0);
  p.body_force = {g, 0.0, 0.0};
  Simulation sim(geom, p, WallScheme::SBB);
  SteadyConfig cfg;
  cfg.tolerance = 1e-13;
  cfg.check_interval = 500;
  cfg.max_steps = 500000;
  ProfileData prof;
  const RunStats st = run_to_steady_state(sim, cfg, &prof);
  converged = st.converged;
  double max_rel = 0.0;
  for (std::size_t i = 0; i < prof.z.size(); ++i) {
    const double zz = prof.z[i] - prof.z0;
    const double exact = g / (2.0 * nu) * zz * (H - zz);
    max_rel = std::max(max_rel, std::abs(prof.u_superficial[i] - exact) / exact);
  }
  return max_rel;
}

// bench.cpp:17-46 time_scheme
double time_scheme(const VoxelGeometry& geom, WallScheme scheme, int warmup, int steps) {
  FluidParams p = relaxation_from_magic(1.0 / 6.0, 3.0 / 16.0);
  p.body_force = {1e-6, 0.0, 0.0};
  Simulation sim(geom, p, scheme);
  sim.step(warmup);
  sim.synchronize();
  const auto t0 = std::chrono::steady_clock::now();
  sim.step(steps);
  sim.synchronize();
  const auto t1 = std::chrono::steady_clock::now();
  const double s = std::chrono::duration<double>(t1 - t0).count();
  return static_cast<double>(geom.dims().cells()) * steps / s / 1e6;  // bench.cpp:38
}

}  // namespace

int main() {
  try {
    bool conv = false;
    const double err = poiseuille_max_rel_err(conv);
    // bench.cpp:50-66: sphere of diameter 76 centred in a periodic 128^3 box
    const int n = 128;
    SpherePack pack;
    pack.box = {double(n), double(n), double(n)};
    pack.spheres.push_back({{n / 2.0, n / 2.0, n / 2.0}, 76.0 / 2.0});
    VoxelizeOptions opt;
    opt.periodic = {true, true, true};
    const VoxelGeometry geom = voxelize(pack, {n, n, n}, opt);
    const double sbb = time_scheme(geom, WallScheme::SBB, 20, 2000);
    const double cli = time_scheme(geom, WallScheme::CLI, 20, 2000);
    std::printf(
        "{\"poiseuille_max_rel_err\": %.3e, \"poiseuille_converged\": %s, "
        "\"bench_cells\": %lld, \"bench_fluid_fraction\": %.4f, \"sbb_mlups\": %.1f, "
        "\"cli_mlups\": %.1f, \"cli_over_sbb\": %.3f}\n",
        err, conv ? "true" : "false", static_cast<long long>(geom.dims().cells()),
        double(geom.fluid_cells()) / geom.dims().cells(), sbb, cli, cli / sbb);
    return (err <= 1e-8 && conv && cli / sbb >= 0.75) ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
