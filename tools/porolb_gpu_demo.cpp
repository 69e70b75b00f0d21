// C++ drop-in demo: the reference's own callers, rewritten against
// include/porolb_gpu/porolb_gpu.hpp (the only change a reference user makes is
// the namespace and the link line).  Mirrors
//   * acceptance criterion 1, Poiseuille exactness at Lambda = 3/16
//     (proj/tests/acceptance/acceptance_main.cpp:59-75);
//   * run_bench / time_scheme, SBB vs CLI on the 128^3 sphere-in-box bench
//     geometry (proj/src/bench.cpp:17-66; acceptance criterion 10);
//   * the scenario outputs (scenarios.cpp:92-116): profile CSV, sphere CSV and
//     voxel file written and read back through the io.hpp mirror.
// Prints one JSON object.  Build: python paper_1507_06565_b200/build.py --all
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "porolb_gpu/porolb_gpu.hpp"

using namespace porolb_gpu;

namespace {

// acceptance_main.cpp:39-56 channel_config + :59-75 criterion 1
double poiseuille_max_rel_err(bool& converged, ProfileData& prof) {
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

// scenarios.cpp:71,92,169: the files a scenario run leaves behind, read back.
bool io_round_trip(const ProfileData& prof, const SpherePack& pack, const VoxelGeometry& geom) {
  const std::string dir = std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp";
  const std::string pc = dir + "/porolb_gpu_demo_profile.csv";
  const std::string sc = dir + "/porolb_gpu_demo_pack.csv";
  const std::string vx = dir + "/porolb_gpu_demo_geometry.vox";
  write_profile_csv(pc, prof);
  write_sphere_csv(sc, pack);
  write_voxel_file(vx, geom);
  const ProfileData p2 = read_profile_csv(pc);
  const SpherePack s2 = read_sphere_csv(sc);
  const VoxelGeometry g2 = read_voxel_file(vx);
  bool ok = p2.z == prof.z && p2.u_superficial == prof.u_superficial && p2.nu == prof.nu;
  ok = ok && s2.spheres.size() == pack.spheres.size() &&
       s2.spheres[0].radius == pack.spheres[0].radius && s2.box.lx == pack.box.lx;
  ok = ok && g2.dims().cells() == geom.dims().cells() && g2.n_links() == geom.n_links() &&
       g2.fluid_cells() == geom.fluid_cells();
  for (std::int64_t c = 0; ok && c < geom.dims().cells(); ++c) ok = g2.flag(c) == geom.flag(c);
  std::remove(pc.c_str());
  std::remove(sc.c_str());
  std::remove(vx.c_str());
  return ok;
}

}  // namespace

int main() {
  try {
    bool conv = false;
    ProfileData prof;
    const double err = poiseuille_max_rel_err(conv, prof);
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
    const bool io_ok = io_round_trip(prof, pack, geom);
    std::printf(
        "{\"poiseuille_max_rel_err\": %.3e, \"poiseuille_converged\": %s, "
        "\"bench_cells\": %lld, \"bench_fluid_fraction\": %.4f, \"sbb_mlups\": %.1f, "
        "\"cli_mlups\": %.1f, \"cli_over_sbb\": %.3f, \"io_round_trip\": %s}\n",
        err, conv ? "true" : "false", static_cast<long long>(geom.dims().cells()),
        double(geom.fluid_cells()) / geom.dims().cells(), sbb, cli, cli / sbb,
        io_ok ? "true" : "false");
    return (err <= 1e-8 && conv && cli / sbb >= 0.75 && io_ok) ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
