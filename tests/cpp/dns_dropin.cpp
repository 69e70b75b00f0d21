// The reference's pore-scale driver (proj/src/dns.cpp:11-22, proj/include/
// porolb/dns.hpp:13-27) compiled against the B200 mirror with only the
// namespace changed: make_simulation() keeps `resolve_drive(cfg.drive)`.
// tests/test_abi.py compiles this file (no GPU needed); tests/test_gpu_cpp_demo.py
// also runs it.
#include <cstdio>
#include <utility>

#include "porolb_gpu/porolb_gpu.hpp"

namespace porolb = porolb_gpu;

namespace dns {
using namespace porolb;

struct RunConfig {  // dns.hpp:13-20
  VoxelGeometry geometry;
  double nu = 1.0 / 6.0;
  double lambda = 3.0 / 16.0;
  WallScheme scheme = WallScheme::CLI;
  DriveSpec drive;
  SteadyConfig steady;
};

struct DnsResult {  // dns.hpp:22-26
  Simulation sim;
  ProfileData profile;
  RunStats stats;
};

Simulation make_simulation(const RunConfig& cfg) {  // dns.cpp:11-15, unchanged
  FluidParams params = relaxation_from_magic(cfg.nu, cfg.lambda);
  params.body_force = resolve_drive(cfg.drive);
  return Simulation(cfg.geometry, params, cfg.scheme);
}

DnsResult run_to_steady(const RunConfig& cfg) {  // dns.cpp:17-22, unchanged
  Simulation sim = make_simulation(cfg);
  ProfileData profile;
  RunStats stats = run_to_steady_state(sim, cfg.steady, &profile);
  return DnsResult{std::move(sim), std::move(profile), stats};
}
}  // namespace dns

int main() {
  using namespace porolb;
  dns::RunConfig cfg;
  VoxelizeOptions opt;
  opt.wall_z_lo = opt.wall_z_hi = true;
  cfg.geometry = make_box_geometry({4, 4, 18}, opt);
  cfg.scheme = WallScheme::SBB;
  cfg.drive.mode = DriveMode::PressureGradientAsForce;  // Delta_p over the channel length
  cfg.drive.magnitude = {4e-8, 0.0, 0.0};
  cfg.drive.channel_length = 4.0;
  cfg.steady.tolerance = 1e-10;
  cfg.steady.check_interval = 500;
  cfg.steady.max_steps = 20000;
  dns::DnsResult r = dns::run_to_steady(cfg);
  const ProfileData eps = porosity_profile(cfg.geometry);
  std::printf("steps=%ld converged=%d g=%.17g u_max=%.17g eps_wall=%.17g eps_mid=%.17g\n",
              r.stats.steps, r.stats.converged ? 1 : 0, r.sim.params().body_force[0],
              r.profile.u_max, eps.epsilon[0], eps.epsilon[9]);
  return 0;
}
