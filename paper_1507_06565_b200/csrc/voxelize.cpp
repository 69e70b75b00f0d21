// Host voxelizer, bit-exact with the reference voxelize() (geometry.cpp:491-632)
// but O(links x spheres-near-link) instead of O(links x all spheres): sphere
// images are binned into a uniform grid over their reject boxes, and every
// image that the reference's "cheap reject" (geometry.cpp:607-611) would keep
// is in the bin of the link's cell centre, so the min over hits (order
// independent) sees the same candidate set.  The arithmetic of every test is
// the reference's own expression order (-ffp-contract=off).  Flags and links
// are built in parallel over z-planes and concatenated in (cell, k) order.
//
// Slab mode produces the columns [x0, x1) of the global voxelization with
// local cell indices, plus the flags of the two neighbouring ghost columns.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <sstream>
#include <vector>

#include "host_common.h"
#include "voxel_geometry.h"


namespace pgpu {
namespace {

struct Sph {
  double c[3];
  double r;
};

// geometry.cpp:442-462
std::vector<Sph> effective_spheres(const pgpu_sphere_pack& pack, const uint8_t periodic[3],
                                   const int32_t dims[3]) {
  std::vector<Sph> out;
  const int ix_max = periodic[0] ? 1 : 0;
  const int iy_max = periodic[1] ? 1 : 0;
  for (int64_t i = 0; i < pack.n_spheres; ++i) {
    for (int ix = -ix_max; ix <= ix_max; ++ix) {
      for (int iy = -iy_max; iy <= iy_max; ++iy) {
        Sph img{{pack.cx[i], pack.cy[i], pack.cz[i]}, pack.radius[i]};
        img.c[0] += ix * pack.box[0];
        img.c[1] += iy * pack.box[1];
        if (img.c[0] + img.r < 0.0 || img.c[0] - img.r > dims[0] || img.c[1] + img.r < 0.0 ||
            img.c[1] - img.r > dims[1]) {
          continue;
        }
        out.push_back(img);
      }
    }
  }
  return out;
}

// geometry.cpp:465-479
inline bool ray_sphere(const double p[3], const int e[3], const Sph& s, double& t_out) {
  const double d[3] = {p[0] - s.c[0], p[1] - s.c[1], p[2] - s.c[2]};
  const double a = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
  const double b = 2.0 * (e[0] * d[0] + e[1] * d[1] + e[2] * d[2]);
  const double c = (d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) - s.r * s.r;
  const double disc = b * b - 4.0 * a * c;
  if (disc < 0.0) return false;
  const double sq = std::sqrt(disc);
  bool have = false;
  double best = 0.0;
  for (double t : {(-b - sq) / (2.0 * a), (-b + sq) / (2.0 * a)}) {
    if (t > 0.0 && t <= 1.0 + 1e-12 && (!have || t < best)) {
      best = t;
      have = true;
    }
  }
  t_out = best;
  return have;
}

// geometry.cpp:481-487
inline bool ray_plane_z(const double p[3], const int e[3], double plane_z, double& t_out) {
  if (e[2] == 0) return false;
  const double t = (plane_z - p[2]) / e[2];
  if (t > 0.0 && t <= 1.0 + 1e-12) {
    t_out = t;
    return true;
  }
  return false;
}

inline int wrap_coord(int v, int n, bool periodic) {
  if (v >= 0 && v < n) return v;
  if (!periodic) return -1;
  return (v % n + n) % n;
}

// Uniform grid of sphere images keyed by their reject boxes.
struct SphereGrid {
  double h = 8.0;
  int gx = 1, gy = 1, gz = 1;
  std::vector<int64_t> start;
  std::vector<int32_t> items;
  void build(const std::vector<Sph>& s, const int32_t dims[3]) {
    double rmax = 0.0;
    for (const Sph& x : s) rmax = std::max(rmax, x.r);
    h = std::max(4.0, rmax + 2.0);
    gx = std::max(1, (int)std::ceil(dims[0] / h));
    gy = std::max(1, (int)std::ceil(dims[1] / h));
    gz = std::max(1, (int)std::ceil(dims[2] / h));
    const int64_t ncell = (int64_t)gx * gy * gz;
    std::vector<int64_t> count(ncell + 1, 0);
    auto range = [&](const Sph& x, int a, int n, int& lo, int& hi) {
      // identical bounds to the reject test geometry.cpp:607-611
      const double L = x.c[a] - x.r - 2.0, U = x.c[a] + x.r + 2.0;
      lo = (int)std::floor(L / h);
      hi = (int)std::floor(U / h);
      lo = std::max(lo, 0);
      hi = std::min(hi, n - 1);
    };
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {
        start.assign(ncell + 1, 0);
        for (int64_t i = 0; i < ncell; ++i) start[i + 1] = start[i] + count[i];
        items.assign(start[ncell], 0);
        std::fill(count.begin(), count.end(), 0);
      }
      for (size_t i = 0; i < s.size(); ++i) {
        int x0, x1, y0, y1, z0, z1;
        range(s[i], 0, gx, x0, x1);
        range(s[i], 1, gy, y0, y1);
        range(s[i], 2, gz, z0, z1);
        for (int z = z0; z <= z1; ++z)
          for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
              const int64_t g = ((int64_t)z * gy + y) * gx + x;
              if (pass == 0)
                ++count[g];
              else
                items[start[g] + count[g]++] = (int32_t)i;
            }
      }
    }
  }
  // Bin of a point inside the domain.
  int64_t bin(const double p[3]) const {
    int x = std::min(gx - 1, std::max(0, (int)std::floor(p[0] / h)));
    int y = std::min(gy - 1, std::max(0, (int)std::floor(p[1] / h)));
    int z = std::min(gz - 1, std::max(0, (int)std::floor(p[2] / h)));
    return ((int64_t)z * gy + y) * gx + x;
  }
};

}  // namespace

VoxHostGrid build_vox_host_grid(const pgpu_sphere_pack& pack, const uint8_t periodic[3],
                                const int32_t dims[3]) {
  VoxHostGrid out;
  const std::vector<Sph> s = effective_spheres(pack, periodic, dims);
  SphereGrid grid;
  grid.build(s, dims);
  out.spheres.resize(s.size());
  for (size_t i = 0; i < s.size(); ++i)
    out.spheres[i] = VoxSph{{s[i].c[0], s[i].c[1], s[i].c[2]}, s[i].r};
  out.h = grid.h;
  out.gx = grid.gx;
  out.gy = grid.gy;
  out.gz = grid.gz;
  out.start = grid.start;
  out.items = grid.items;
  return out;
}

namespace {

// Core: voxelize the global domain restricted to global columns [x0, x1).
// When slab, ghost columns x0-1 and x1 (periodic wrap along x) are also
// rasterised and links refer to local indices.
std::unique_ptr<pgpu_voxel_geometry> voxelize_impl(const pgpu_sphere_pack& pack,
                                                   const int32_t dims[3],
                                                   const pgpu_voxelize_options& opt, int x0,
                                                   int x1, bool slab) {
  if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0) throw ConfigError("voxel dims must be positive");
  if (pack.n_spheres < 0 || (pack.n_spheres > 0 && (!pack.cx || !pack.cy || !pack.cz || !pack.radius)))
    throw std::invalid_argument("bad sphere arrays");
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (slab) {
    if (!(0 <= x0 && x0 < x1 && x1 <= nx)) throw ConfigError("slab range must satisfy 0 <= x0 < x1 <= nx");
    if (!opt.periodic[0]) throw ConfigError("x-slab decomposition needs a periodic x axis");
  } else {
    x0 = 0;
    x1 = nx;
  }
  const int lnx = x1 - x0;
  // window columns: w = 0..wn-1 map to global column gcol(w)
  const int wpad = slab ? 1 : 0;
  const int wn = lnx + 2 * wpad;
  std::vector<int> gcol(wn);
  for (int w = 0; w < wn; ++w) gcol[w] = ((x0 - wpad + w) % nx + nx) % nx;
  std::vector<int> wcol_of(nx, -1);  // global column -> window column (core columns only)
  for (int w = wpad; w < wpad + lnx; ++w) wcol_of[gcol[w]] = w;

  const bool per[3] = {opt.periodic[0] != 0, opt.periodic[1] != 0, opt.periodic[2] != 0};
  const std::vector<Sph> spheres = effective_spheres(pack, opt.periodic, dims);

  // window flags, index (z*ny + y)*wn + w
  std::vector<uint8_t> wf((size_t)wn * ny * nz, 0);
  auto WIDX = [&](int w, int y, int z) { return ((int64_t)z * ny + y) * wn + w; };

  // geometry.cpp:501-510 plate
  if (pack.bottom_plate_z > 0.0) {
    const int k_max = (int)std::floor(pack.bottom_plate_z - 0.5);
    for (int z = 0; z <= std::min(k_max, nz - 1); ++z)
      for (int y = 0; y < ny; ++y)
        for (int w = 0; w < wn; ++w) wf[WIDX(w, y, z)] = 1;
  }
  // geometry.cpp:512-533 sphere rasterisation, parallel over z bands
  parallel_for(nz, [&](int64_t za, int64_t zb, int) {
    for (const Sph& s : spheres) {
      const int bx0 = std::max(0, (int)std::floor(s.c[0] - s.r - 0.5));
      const int bx1 = std::min(nx - 1, (int)std::ceil(s.c[0] + s.r));
      const int by0 = std::max(0, (int)std::floor(s.c[1] - s.r - 0.5));
      const int by1 = std::min(ny - 1, (int)std::ceil(s.c[1] + s.r));
      const int bz0 = std::max(0, (int)std::floor(s.c[2] - s.r - 0.5));
      const int bz1 = std::min(nz - 1, (int)std::ceil(s.c[2] + s.r));
      const int z0 = std::max<int>(bz0, (int)za), z1 = std::min<int>(bz1, (int)zb - 1);
      if (z0 > z1 || bx0 > bx1) continue;
      const double r2 = s.r * s.r;
      for (int w = 0; w < wn; ++w) {
        const int x = gcol[w];
        if (x < bx0 || x > bx1) continue;
        for (int z = z0; z <= z1; ++z)
          for (int y = by0; y <= by1; ++y) {
            const double dx = x + 0.5 - s.c[0];
            const double dy = y + 0.5 - s.c[1];
            const double dz = z + 0.5 - s.c[2];
            if (dx * dx + dy * dy + dz * dz < r2) wf[WIDX(w, y, z)] = 1;
          }
      }
    }
  });
  // geometry.cpp:535-551 wall layers
  std::vector<double> wall_planes;
  auto g = std::make_unique<pgpu_voxel_geometry>();
  if (opt.wall_z_lo) {
    for (int y = 0; y < ny; ++y)
      for (int w = 0; w < wn; ++w) wf[WIDX(w, y, 0)] = 2;
    wall_planes.push_back(1.0);
    g->has_lo = 1;
    g->lo = 1.0;
  }
  if (opt.wall_z_hi) {
    for (int y = 0; y < ny; ++y)
      for (int w = 0; w < wn; ++w) wf[WIDX(w, y, nz - 1)] = 2;
    wall_planes.push_back(static_cast<double>(nz - 1));
    g->has_hi = 1;
    g->hi = static_cast<double>(nz - 1);
  }

  g->dims[0] = lnx;
  g->dims[1] = ny;
  g->dims[2] = nz;
  for (int a = 0; a < 3; ++a) g->periodic[a] = opt.periodic[a] ? 1 : 0;
  g->slab = slab ? 1 : 0;
  g->x_offset = x0;
  g->global_nx = nx;
  const int64_t lcells = (int64_t)lnx * ny * nz;
  g->flags.resize(lcells);
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      std::memcpy(&g->flags[((int64_t)z * ny + y) * lnx], &wf[WIDX(wpad, y, z)], lnx);
  if (slab) {
    g->ghost_lo.resize((size_t)ny * nz);
    g->ghost_hi.resize((size_t)ny * nz);
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y) {
        g->ghost_lo[(size_t)z * ny + y] = wf[WIDX(0, y, z)];
        g->ghost_hi[(size_t)z * ny + y] = wf[WIDX(wn - 1, y, z)];
      }
  }

  // geometry.cpp:553-565 porosity per plane (over the local columns)
  g->porosity.assign(nz, 0.0);
  g->fluid_cells = 0;
  for (int z = 0; z < nz; ++z) {
    int64_t fluid = 0;
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < lnx; ++x)
        if (g->flags[((int64_t)z * ny + y) * lnx + x] == 0) ++fluid;
    g->porosity[z] = static_cast<double>(fluid) / (static_cast<double>(lnx) * ny);
    g->fluid_cells += fluid;
  }
  if (g->fluid_cells == 0 && !slab) throw GeometryError("geometry has no fluid cells");

  // geometry.cpp:567-631 links, parallel over z-planes, concatenated in order
  SphereGrid grid;
  grid.build(spheres, dims);
  const int nthreads = hw_threads();
  std::vector<std::vector<int64_t>> tlf(nthreads), tls(nthreads);
  std::vector<std::vector<int32_t>> tld(nthreads);
  std::vector<std::vector<float>> tlq(nthreads);
  std::vector<int> tqfb(nthreads, 0);
  std::vector<std::string> terr(nthreads);
  std::vector<int64_t> first_bad(nthreads, std::numeric_limits<int64_t>::max());
  // chunk boundaries must be identical for reassembly: use explicit chunking
  std::vector<int64_t> zchunk(nthreads + 1);
  for (int i = 0; i <= nthreads; ++i) zchunk[i] = (int64_t)nz * i / nthreads;
  std::vector<std::thread> th;
  for (int tid = 0; tid < nthreads; ++tid) {
    th.emplace_back([&, tid] {
      auto& lf = tlf[tid];
      auto& ls = tls[tid];
      auto& ld = tld[tid];
      auto& lq = tlq[tid];
      for (int z = (int)zchunk[tid]; z < (int)zchunk[tid + 1]; ++z) {
        for (int y = 0; y < ny; ++y) {
          for (int lx = 0; lx < lnx; ++lx) {
            const int w = lx + wpad;
            const int x = gcol[w];
            if (wf[WIDX(w, y, z)] != 0) continue;
            const int64_t cell = ((int64_t)z * ny + y) * lnx + lx;
            for (int k = 1; k < 19; ++k) {
              const int xn = wrap_coord(x + kE[k][0], nx, per[0]);
              const int yn = wrap_coord(y + kE[k][1], ny, per[1]);
              const int zn = wrap_coord(z + kE[k][2], nz, per[2]);
              if (xn < 0 || yn < 0 || zn < 0) {
                if (cell < first_bad[tid]) {
                  first_bad[tid] = cell;
                  std::ostringstream os;
                  os << "fluid cell (" << x << "," << y << "," << z
                     << ") touches a non-periodic open face; add a wall layer or periodic axis";
                  terr[tid] = os.str();
                }
                continue;
              }
              const int wn_col = slab ? w + kE[k][0] : xn;  // window column of the neighbour
              if (wf[WIDX(wn_col, yn, zn)] == 0) continue;
              const int kb = opposite(k);
              int64_t second = -1;
              const int xp = wrap_coord(x + kE[kb][0], nx, per[0]);
              const int yp = wrap_coord(y + kE[kb][1], ny, per[1]);
              const int zp = wrap_coord(z + kE[kb][2], nz, per[2]);
              if (xp >= 0 && yp >= 0 && zp >= 0) {
                const int wp_col = slab ? w + kE[kb][0] : xp;
                if (wf[WIDX(wp_col, yp, zp)] == 0) {
                  if (!slab)
                    second = ((int64_t)zp * ny + yp) * nx + xp;
                  else if (wp_col == 0 || wp_col == wn - 1)
                    second = -2;  // ghost column
                  else
                    second = ((int64_t)zp * ny + yp) * lnx + (wp_col - wpad);
                }
              }
              const double pc[3] = {x + 0.5, y + 0.5, z + 0.5};
              double q = std::numeric_limits<double>::infinity();
              const int64_t b = grid.bin(pc);
              for (int64_t it = grid.start[b]; it < grid.start[b + 1]; ++it) {
                const Sph& s = spheres[grid.items[it]];
                if (pc[0] < s.c[0] - s.r - 2.0 || pc[0] > s.c[0] + s.r + 2.0 ||
                    pc[1] < s.c[1] - s.r - 2.0 || pc[1] > s.c[1] + s.r + 2.0 ||
                    pc[2] < s.c[2] - s.r - 2.0 || pc[2] > s.c[2] + s.r + 2.0) {
                  continue;
                }
                double t;
                if (ray_sphere(pc, kE[k], s, t)) q = std::min(q, t);
              }
              double t;
              if (pack.bottom_plate_z > 0.0 && ray_plane_z(pc, kE[k], pack.bottom_plate_z, t))
                q = std::min(q, t);
              for (double plane : wall_planes)
                if (ray_plane_z(pc, kE[k], plane, t)) q = std::min(q, t);
              if (!std::isfinite(q)) {
                q = 0.5;
                ++tqfb[tid];
              }
              lf.push_back(cell);
              ls.push_back(second);
              ld.push_back(k);
              lq.push_back(static_cast<float>(std::clamp(q, opt.q_clamp_min, 1.0)));
            }
          }
        }
      }
    });
  }
  for (auto& t : th) t.join();
  // the reference throws at the first offending cell in scan order
  int64_t bad = std::numeric_limits<int64_t>::max();
  std::string msg;
  for (int i = 0; i < nthreads; ++i)
    if (first_bad[i] < bad) {
      bad = first_bad[i];
      msg = terr[i];
    }
  if (!msg.empty()) throw ConfigError(msg);
  size_t total = 0;
  for (int i = 0; i < nthreads; ++i) total += tlf[i].size();
  g->lf.reserve(total);
  g->ls.reserve(total);
  g->ld.reserve(total);
  g->lq.reserve(total);
  for (int i = 0; i < nthreads; ++i) {
    g->lf.insert(g->lf.end(), tlf[i].begin(), tlf[i].end());
    g->ls.insert(g->ls.end(), tls[i].begin(), tls[i].end());
    g->ld.insert(g->ld.end(), tld[i].begin(), tld[i].end());
    g->lq.insert(g->lq.end(), tlq[i].begin(), tlq[i].end());
    g->q_fallback_count += tqfb[i];
  }
  g->lm.assign(total, 0);
  return g;
}

}  // namespace
}  // namespace pgpu

using namespace pgpu;

extern "C" {

int pgpu_voxelize(const pgpu_sphere_pack* pack, const int32_t dims[3],
                  const pgpu_voxelize_options* opt, pgpu_voxel_geometry** out) {
  return guard([&] {
    if (!pack || !dims || !opt || !out) throw std::invalid_argument("null pointer");
    *out = voxelize_impl(*pack, dims, *opt, 0, dims[0], false).release();
  });
}

int pgpu_voxelize_slab(const pgpu_sphere_pack* pack, const int32_t dims[3],
                       const pgpu_voxelize_options* opt, int32_t x0, int32_t x1,
                       pgpu_voxel_geometry** out) {
  return guard([&] {
    if (!pack || !dims || !opt || !out) throw std::invalid_argument("null pointer");
    *out = voxelize_impl(*pack, dims, *opt, x0, x1, true).release();
  });
}

// geometry.cpp:634-640
int pgpu_make_box_geometry(const int32_t dims[3], const pgpu_voxelize_options* opt,
                           pgpu_voxel_geometry** out) {
  return guard([&] {
    if (!dims || !opt || !out) throw std::invalid_argument("null pointer");
    pgpu_sphere_pack empty{};
    empty.n_spheres = 0;
    empty.box[0] = dims[0];
    empty.box[1] = dims[1];
    empty.box[2] = dims[2];
    empty.bottom_plate_z = 0.0;
    *out = voxelize_impl(empty, dims, *opt, 0, dims[0], false).release();
  });
}

int pgpu_voxel_geometry_view(const pgpu_voxel_geometry* g, pgpu_geometry* v,
                             int32_t* q_fallback_count) {
  return guard([&] {
    if (!g || !v) throw std::invalid_argument("null pointer");
    std::memset(v, 0, sizeof(*v));
    for (int a = 0; a < 3; ++a) {
      v->dims[a] = g->dims[a];
      v->periodic[a] = g->periodic[a];
    }
    v->flags = g->flags.data();
    v->n_links = (int64_t)g->lf.size();
    v->link_fluid_cell = g->lf.data();
    v->link_second_fluid = g->ls.data();
    v->link_direction = g->ld.data();
    v->link_q = g->lq.data();
    v->link_moving = g->lm.data();
    v->porosity = g->porosity.data();
    v->fluid_cells = g->fluid_cells;
    v->has_wall_plane_lo = g->has_lo;
    v->has_wall_plane_hi = g->has_hi;
    v->wall_plane_lo = g->lo;
    v->wall_plane_hi = g->hi;
    v->slab = g->slab;
    v->x_offset = g->x_offset;
    v->global_nx = g->global_nx;
    v->ghost_flags_lo = g->slab ? g->ghost_lo.data() : nullptr;
    v->ghost_flags_hi = g->slab ? g->ghost_hi.data() : nullptr;
    if (q_fallback_count) *q_fallback_count = g->q_fallback_count;
  });
}

void pgpu_voxel_geometry_free(pgpu_voxel_geometry* g) { delete g; }

}  // extern "C"
