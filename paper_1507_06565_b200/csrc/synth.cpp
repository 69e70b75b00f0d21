// Seeded synthetic sphere lists for the benchmark configurations.  The
// reference ships only a drop-and-roll packer (geometry.cpp:86-437) that
// cannot reach the configs' porosities, so configs 2-4 are fed
// by this generator; the same sphere list is handed to both the reference
// voxelizer and ours, so parity is unaffected.  Randomness follows the
// reference's convention: std::mt19937_64 + uniform01 = (rng() >> 11) * 2^-53
// (geometry.cpp:19-21), four draws per attempt in the order x, y, z, r.
#include <cmath>
#include <random>
#include <vector>

#include "host_common.h"

namespace pgpu {
namespace {
inline double uniform01(std::mt19937_64& rng) {
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}
constexpr double kPi = 3.14159265358979323846;
}  // namespace
}  // namespace pgpu

using namespace pgpu;

extern "C" int pgpu_generate_spheres(int32_t mode, uint64_t seed, const double box[3],
                                     double z_lo, double z_hi, double r_min, double r_max,
                                     double bed_volume, double target_porosity,
                                     int64_t max_attempts, int64_t capacity, double* cx,
                                     double* cy, double* cz, double* r, int64_t* n_out,
                                     double* porosity_out) {
  return guard([&] {
    if (!box || !n_out || !porosity_out || (capacity > 0 && (!cx || !cy || !cz || !r)))
      throw std::invalid_argument("null pointer");
    if (!(r_min > 0.0 && r_max >= r_min)) throw ConfigError("radii must satisfy 0 < r_min <= r_max");
    if (!(bed_volume > 0.0)) throw ConfigError("bed volume must be positive");
    if (mode != 0 && mode != 1) throw ConfigError("mode must be 0 (RSA) or 1 (Boolean)");
    std::mt19937_64 rng(seed);
    const double lx = box[0], ly = box[1];
    // neighbour grid for the RSA overlap test (x, y periodic; z open)
    const double h = 2.0 * r_max;
    const int gx = std::max(1, (int)std::floor(lx / h));
    const int gy = std::max(1, (int)std::floor(ly / h));
    const int gz = std::max(1, (int)std::ceil((z_hi - z_lo) / h) + 1);
    const double hx = lx / gx, hy = ly / gy;
    std::vector<std::vector<int32_t>> cells((size_t)gx * gy * gz);
    auto cell_of = [&](double x, double y, double z, int& ix, int& iy, int& iz) {
      ix = std::min(gx - 1, std::max(0, (int)std::floor(x / hx)));
      iy = std::min(gy - 1, std::max(0, (int)std::floor(y / hy)));
      iz = std::min(gz - 1, std::max(0, (int)std::floor((z - z_lo) / h)));
    };
    int64_t n = 0;
    double vol = 0.0;
    double poro = 1.0;
    for (int64_t a = 0; a < max_attempts; ++a) {
      const double x = uniform01(rng) * lx;
      const double y = uniform01(rng) * ly;
      const double z = z_lo + uniform01(rng) * (z_hi - z_lo);
      const double rr = r_min + uniform01(rng) * (r_max - r_min);
      if (mode == 0) {
        int ix, iy, iz;
        cell_of(x, y, z, ix, iy, iz);
        bool ok = true;
        for (int dz = -1; dz <= 1 && ok; ++dz) {
          const int zz = iz + dz;
          if (zz < 0 || zz >= gz) continue;
          for (int dy = -1; dy <= 1 && ok; ++dy) {
            const int yy = ((iy + dy) % gy + gy) % gy;
            for (int dx = -1; dx <= 1 && ok; ++dx) {
              const int xx = ((ix + dx) % gx + gx) % gx;
              for (int32_t j : cells[((size_t)zz * gy + yy) * gx + xx]) {
                double ddx = std::fabs(x - cx[j]);
                double ddy = std::fabs(y - cy[j]);
                ddx = std::min(ddx, lx - ddx);  // minimum image
                ddy = std::min(ddy, ly - ddy);
                const double ddz = z - cz[j];
                const double rs = rr + r[j];
                if (ddx * ddx + ddy * ddy + ddz * ddz < rs * rs) {
                  ok = false;
                  break;
                }
              }
            }
          }
        }
        if (!ok) continue;
        if (n >= capacity) throw ConfigError("sphere capacity exceeded");
        cells[((size_t)iz * gy + iy) * gx + ix].push_back((int32_t)n);
      } else if (n >= capacity) {
        throw ConfigError("sphere capacity exceeded");
      }
      cx[n] = x;
      cy[n] = y;
      cz[n] = z;
      r[n] = rr;
      ++n;
      vol += 4.0 / 3.0 * kPi * rr * rr * rr;
      poro = (mode == 0) ? 1.0 - vol / bed_volume : std::exp(-vol / bed_volume);
      if (poro <= target_porosity) break;
    }
    *n_out = n;
    *porosity_out = poro;
  });
}
