// The reference's file formats (io.hpp:11-44, io.cpp) as
// native host code over the C ABI: byte-identical output, the same parse rules
// and the same exception types (ConfigError / GeometryError -> status codes).
//
// Where the reference is slow, the B200 build is not a transliteration:
//   * write_vtk pulls the moments from the device in one pass
//     (pgpu_macroscopic_fields) and formats rows on every host thread into
//     ordered blocks, with a writer thread streaming the previous round to the
//     file (the reference formats one value at a time through an ofstream,
//     io.cpp:117-149);
//   * read_voxel_file rebuilds the q = 1/2 link list plane-parallel and
//     concatenates the per-thread lists in the reference's (cell, k) order
//     (io.cpp:236-276).
// Numbers are printed as "%.17g" (io.cpp:11-15) through std::to_chars with
// chars_format::general and precision 17, which the standard specifies as
// printf's %.*g in the C locale; tests/test_io.py checks the bytes against
// the reference build.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "host_common.h"
#include "voxel_geometry.h"

namespace pgpu {
namespace {

constexpr int kDoubleChars = 32;  // "%.17g" needs at most 24

inline char* put_double(char* p, char* end, double v) {
  return std::to_chars(p, end, v, std::chars_format::general, 17).ptr;
}

inline char* put_int(char* p, char* end, int64_t v) { return std::to_chars(p, end, v).ptr; }

std::string fmt(double v) {
  char b[kDoubleChars];
  return std::string(b, put_double(b, b + sizeof b, v));
}

// Rethrows a failed C-ABI call with its own type and message.
void check_status(int st) {
  if (st == PGPU_OK) return;
  const std::string m = pgpu_last_error();
  switch (st) {
    case PGPU_ERR_CONFIG: throw ConfigError(m);
    case PGPU_ERR_INSTABILITY: throw NumericalInstability(m);
    case PGPU_ERR_GEOMETRY: throw GeometryError(m);
    case PGPU_ERR_CUDA: throw CudaError(m);
    default: throw std::runtime_error(m);
  }
}

// Binary output stream (io.cpp:19-23 opens with std::ios::binary).
class OutFile {
 public:
  explicit OutFile(const std::string& path) : path_(path) {
    f_ = std::fopen(path.c_str(), "wb");
    if (!f_) throw ConfigError("cannot write file: " + path);
  }
  ~OutFile() {
    if (f_) std::fclose(f_);
  }
  OutFile(const OutFile&) = delete;
  OutFile& operator=(const OutFile&) = delete;
  void put(const char* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f_) != n) throw ConfigError("write failed: " + path_);
  }
  void put(const std::string& s) { put(s.data(), s.size()); }
  void close() {
    const int rc = std::fclose(f_);
    f_ = nullptr;
    if (rc != 0) throw ConfigError("write failed: " + path_);
  }

 private:
  std::string path_;
  FILE* f_ = nullptr;
};

// Formats rows [0, n) on all host threads and appends them to `out` in order.
// `row(i, p)` writes row i (at most max_row bytes) at p and returns its end.
// Rounds of blocks are double-buffered: one writer thread streams round r
// while the workers format round r + 1.
template <class Row>
void write_rows(OutFile& out, int64_t n, int max_row, const Row& row) {
  if (n <= 0) return;
  const int nt = hw_threads();
  const int64_t block = int64_t(1) << 14;
  const int64_t nblocks = (n + block - 1) / block;
  const int64_t per_round = std::min<int64_t>(nblocks, 2 * int64_t(nt));
  struct Slot {
    std::unique_ptr<char[]> buf;
    size_t used = 0;
  };
  std::vector<Slot> slots[2];
  for (auto& set : slots) {
    set.resize(per_round);
    for (auto& s : set) s.buf.reset(new char[block * max_row]);
  }
  std::thread writer;
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{writer};
  std::exception_ptr write_error;
  int side = 0;
  for (int64_t b0 = 0; b0 < nblocks; b0 += per_round, side ^= 1) {
    const int64_t nb = std::min(per_round, nblocks - b0);
    Slot* const set = slots[side].data();
    parallel_for(nb, [&](int64_t a, int64_t e, int) {
      for (int64_t bi = a; bi < e; ++bi) {
        const int64_t r0 = (b0 + bi) * block, r1 = std::min(n, r0 + block);
        char* p = set[bi].buf.get();
        for (int64_t r = r0; r < r1; ++r) p = row(r, p);
        set[bi].used = static_cast<size_t>(p - set[bi].buf.get());
      }
    });
    if (writer.joinable()) writer.join();
    if (write_error) std::rethrow_exception(write_error);
    writer = std::thread([&out, set, nb, &write_error] {
      try {
        for (int64_t bi = 0; bi < nb; ++bi) out.put(set[bi].buf.get(), set[bi].used);
      } catch (...) {
        write_error = std::current_exception();
      }
    });
  }
  writer.join();
  if (write_error) std::rethrow_exception(write_error);
}

// io.cpp:25-39: split on ',', carriage returns dropped.
std::vector<std::string> split_fields(const std::string& line) {
  std::vector<std::string> out(1);
  for (char ch : line) {
    if (ch == ',')
      out.emplace_back();
    else if (ch != '\r')
      out.back().push_back(ch);
  }
  return out;
}

// profile.cpp:21-29: piecewise linear with clamped ends.
double interp_clamped(const double* zs, const double* vs, int64_t n, double x) {
  if (n <= 0) throw ConfigError("interpolation over an empty profile");
  if (x <= zs[0]) return vs[0];
  if (x >= zs[n - 1]) return vs[n - 1];
  const int64_t i = std::upper_bound(zs, zs + n, x) - zs;
  const double t = (x - zs[i - 1]) / (zs[i] - zs[i - 1]);
  return vs[i - 1] + t * (vs[i] - vs[i - 1]);
}

inline int wrap_or_open(int v, int n, bool periodic) {  // io.cpp:238-242
  if (v >= 0 && v < n) return v;
  if (!periodic) return -1;
  return (v % n + n) % n;
}

}  // namespace
}  // namespace pgpu

using namespace pgpu;

extern "C" {

int pgpu_format_double(double v, char* buf, int32_t cap) {
  return guard([&] {
    if (!buf || cap <= 0) throw std::invalid_argument("null output");
    const std::string s = fmt(v);
    if (static_cast<int32_t>(s.size()) + 1 > cap) throw ConfigError("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// io.cpp:41-62
int pgpu_write_profile_csv(const char* path, const pgpu_profile_meta* m, const double* z,
                           const double* u_sup, const double* u_int, const double* eps,
                           const double* u_norm, int32_t n_norm) {
  return guard([&] {
    if (!path || !m) throw std::invalid_argument("null argument");
    const int64_t n = m->n_planes;
    if (n > 0 && (!z || !u_sup || !u_int || !eps)) throw std::invalid_argument("null profile");
    std::string s;
    s += "# nu = " + fmt(m->nu) + "\n";
    s += "# g = " + fmt(m->body_force[0]) + " " + fmt(m->body_force[1]) + " " +
         fmt(m->body_force[2]) + "\n";
    s += "# stream_axis = " + std::to_string(m->stream_axis) + "\n";
    s += "# height = " + fmt(m->height) + "\n";
    s += "# z0 = " + fmt(m->z0) + "\n";
    s += "# u_max = " + fmt(m->u_max) + "\n";
    s += "z,U_superficial,U_intrinsic,epsilon,U_normalized\n";
    for (int64_t i = 0; i < n; ++i) {
      s += fmt(z[i]) + "," + fmt(u_sup[i]) + "," + fmt(u_int[i]) + "," + fmt(eps[i]) + "," +
           fmt(i < n_norm && u_norm ? u_norm[i] : 0.0) + "\n";
    }
    OutFile out(path);
    out.put(s);
    out.close();
  });
}

// io.cpp:64-97.  Rows beyond `capacity` are counted, not stored: call with
// capacity 0 to size the arrays (meta->n_planes = rows found).
int pgpu_read_profile_csv(const char* path, int32_t capacity, pgpu_profile_meta* m, double* z,
                          double* u_sup, double* u_int, double* eps, double* u_norm,
                          int32_t* n_norm) {
  return guard([&] {
    if (!path || !m) throw std::invalid_argument("null argument");
    std::ifstream in(path);
    if (!in) throw ConfigError(std::string("cannot open profile CSV: ") + path);
    pgpu_profile_meta meta{};
    std::vector<double> col[5];
    std::string line;
    bool header = false;
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      if (line[0] == '#') {
        std::istringstream is(line.substr(1));
        std::string key, eq;
        is >> key >> eq;
        if (eq != "=") continue;
        if (key == "nu") is >> meta.nu;
        if (key == "g") is >> meta.body_force[0] >> meta.body_force[1] >> meta.body_force[2];
        if (key == "stream_axis") is >> meta.stream_axis;
        if (key == "height") is >> meta.height;
        if (key == "z0") is >> meta.z0;
        if (key == "u_max") is >> meta.u_max;
        continue;
      }
      if (!header) {
        header = true;
        continue;
      }
      const std::vector<std::string> f = split_fields(line);
      if (f.size() < 4) throw ConfigError(std::string(path) + ": malformed CSV row: " + line);
      for (int c = 0; c < 4; ++c) col[c].push_back(std::stod(f[c]));
      if (f.size() >= 5) col[4].push_back(std::stod(f[4]));
    }
    if (col[0].empty()) throw ConfigError(std::string(path) + ": profile CSV has no data rows");
    meta.n_planes = static_cast<int32_t>(col[0].size());
    *m = meta;
    if (n_norm) *n_norm = static_cast<int32_t>(col[4].size());
    if (meta.n_planes > capacity) return;
    double* dst[5] = {z, u_sup, u_int, eps, u_norm};
    for (int c = 0; c < 5; ++c)
      if (dst[c] && !col[c].empty()) std::memcpy(dst[c], col[c].data(), col[c].size() * sizeof(double));
  });
}

// io.cpp:99-110
int pgpu_write_comparison_csv(const char* path, int32_t n_a, const double* z_a,
                              const double* u_a, const char* name_a, int32_t n_b,
                              const double* z_b, const double* u_b, const char* name_b) {
  return guard([&] {
    if (!path || !name_a || !name_b) throw std::invalid_argument("null argument");
    OutFile out(path);
    std::string s = std::string("z,") + name_a + "," + name_b + "\n";
    for (int32_t i = 0; i < n_a; ++i) {
      const double vb = interp_clamped(z_b, u_b, n_b, z_a[i]);
      s += fmt(z_a[i]) + "," + fmt(u_a[i]) + "," + fmt(vb) + "\n";
    }
    out.put(s);
    out.close();
  });
}

// io.cpp:112-116
int pgpu_write_report(const char* path, int32_t n, const char* const* keys,
                      const char* const* values) {
  return guard([&] {
    if (!path || (n > 0 && (!keys || !values))) throw std::invalid_argument("null argument");
    OutFile out(path);
    std::string s;
    for (int32_t i = 0; i < n; ++i) s += std::string(keys[i]) + " = " + values[i] + "\n";
    out.put(s);
    out.close();
  });
}

// io.cpp:117-149.  The moments come from one device pass; a slab simulation
// writes its own block with local dimensions.
int pgpu_write_vtk(const char* path, pgpu_sim* sim) {
  return guard([&] {
    if (!path || !sim) throw std::invalid_argument("null argument");
    int32_t d[3];
    check_status(pgpu_dims(sim, d));
    const int64_t cells = int64_t(d[0]) * d[1] * d[2];
    std::unique_ptr<uint8_t[]> flags(new uint8_t[cells]);
    std::unique_ptr<double[]> mom(new double[4 * cells]);
    double* drho = mom.get();
    double* ux = drho + cells;
    double* uy = ux + cells;
    double* uz = uy + cells;
    check_status(pgpu_get_flags(sim, flags.get()));
    check_status(pgpu_macroscopic_fields(sim, drho, ux, uy, uz));

    OutFile out(path);
    std::string h = "# vtk DataFile Version 3.0\nporolb field\nASCII\nDATASET STRUCTURED_POINTS\n";
    h += "DIMENSIONS " + std::to_string(d[0]) + " " + std::to_string(d[1]) + " " +
         std::to_string(d[2]) + "\n";
    h += "ORIGIN 0.5 0.5 0.5\nSPACING 1 1 1\nPOINT_DATA " + std::to_string(cells) + "\n";
    h += "SCALARS flags unsigned_char 1\nLOOKUP_TABLE default\n";
    out.put(h);
    const uint8_t* fl = flags.get();
    write_rows(out, cells, 4, [fl](int64_t c, char* p) {
      p = put_int(p, p + 3, fl[c]);
      *p++ = '\n';
      return p;
    });
    out.put("SCALARS delta_rho double 1\nLOOKUP_TABLE default\n");
    write_rows(out, cells, kDoubleChars, [drho](int64_t c, char* p) {
      p = put_double(p, p + kDoubleChars - 1, drho[c]);
      *p++ = '\n';
      return p;
    });
    out.put("VECTORS velocity double\n");
    write_rows(out, cells, 3 * kDoubleChars, [ux, uy, uz](int64_t c, char* p) {
      char* const e = p + 3 * kDoubleChars;
      p = put_double(p, e, ux[c]);
      *p++ = ' ';
      p = put_double(p, e, uy[c]);
      *p++ = ' ';
      p = put_double(p, e, uz[c]);
      *p++ = '\n';
      return p;
    });
    out.close();
  });
}

// io.cpp:151-162
int pgpu_write_sphere_csv(const char* path, const pgpu_sphere_pack* pack, uint64_t seed) {
  return guard([&] {
    if (!path || !pack) throw std::invalid_argument("null argument");
    std::string s = "# box = " + fmt(pack->box[0]) + " " + fmt(pack->box[1]) + " " +
                    fmt(pack->box[2]) + " plate_z = " + fmt(pack->bottom_plate_z) +
                    " seed = " + std::to_string(seed) + "\n";
    s += "x,y,z,r\n";
    for (int64_t i = 0; i < pack->n_spheres; ++i) {
      s += fmt(pack->cx[i]) + "," + fmt(pack->cy[i]) + "," + fmt(pack->cz[i]) + "," +
           fmt(pack->radius[i]) + "\n";
    }
    OutFile out(path);
    out.put(s);
    out.close();
  });
}

// io.cpp:164-199.  As with profiles, capacity 0 sizes the arrays.
int pgpu_read_sphere_csv(const char* path, int64_t capacity, int64_t* n_spheres, double* cx,
                         double* cy, double* cz, double* radius, double box[3],
                         double* bottom_plate_z, uint64_t* seed, double* achieved_height) {
  return guard([&] {
    if (!path || !n_spheres) throw std::invalid_argument("null argument");
    std::ifstream in(path);
    if (!in) throw ConfigError(std::string("cannot open sphere CSV: ") + path);
    double bx[3] = {0.0, 0.0, 0.0}, plate = 0.0, top = 0.0;
    uint64_t sd = 0;
    std::vector<double> col[4];
    std::string line;
    bool header = false;
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      if (line[0] == '#') {
        std::istringstream is(line.substr(1));
        std::string tok;
        while (is >> tok) {
          if (tok == "box")
            is >> tok >> bx[0] >> bx[1] >> bx[2];
          else if (tok == "plate_z")
            is >> tok >> plate;
          else if (tok == "seed")
            is >> tok >> sd;
        }
        continue;
      }
      if (!header) {
        header = true;
        continue;
      }
      const std::vector<std::string> f = split_fields(line);
      if (f.size() != 4) throw ConfigError(std::string(path) + ": sphere CSV rows need x,y,z,r");
      double v[4];
      for (int c = 0; c < 4; ++c) v[c] = std::stod(f[c]);
      for (int c = 0; c < 4; ++c) col[c].push_back(v[c]);
      top = std::max(top, v[2] + v[3]);
    }
    if (bx[0] <= 0.0) throw ConfigError(std::string(path) + ": sphere CSV is missing the box header");
    const int64_t n = static_cast<int64_t>(col[0].size());
    *n_spheres = n;
    if (box) std::memcpy(box, bx, sizeof bx);
    if (bottom_plate_z) *bottom_plate_z = plate;
    if (seed) *seed = sd;
    if (achieved_height) *achieved_height = top;
    if (n > capacity) return;
    double* dst[4] = {cx, cy, cz, radius};
    for (int c = 0; c < 4; ++c)
      if (dst[c] && n) std::memcpy(dst[c], col[c].data(), n * sizeof(double));
  });
}

// io.cpp:201-208
int pgpu_write_voxel_file(const char* path, const pgpu_geometry* g) {
  return guard([&] {
    if (!path || !g || !g->flags) throw std::invalid_argument("null argument");
    if (g->slab) throw ConfigError("write_voxel_file: a slab geometry holds one x-range only");
    const std::string h = "porolb-voxel 1 " + std::to_string(g->dims[0]) + " " +
                          std::to_string(g->dims[1]) + " " + std::to_string(g->dims[2]) + " " +
                          (g->periodic[0] ? "1" : "0") + " " + (g->periodic[1] ? "1" : "0") +
                          " " + (g->periodic[2] ? "1" : "0") + "\n";
    OutFile out(path);
    out.put(h);
    out.put(reinterpret_cast<const char*>(g->flags),
            static_cast<size_t>(int64_t(g->dims[0]) * g->dims[1] * g->dims[2]));
    out.close();
  });
}

// io.cpp:210-278: flags from the file, links rebuilt with q = 1/2 in the
// reference's (cell, k) order, no wall planes.
int pgpu_read_voxel_file(const char* path, pgpu_voxel_geometry** out_geom) {
  return guard([&] {
    if (!path || !out_geom) throw std::invalid_argument("null argument");
    *out_geom = nullptr;
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError(std::string("cannot open voxel file: ") + path);
    std::string magic;
    int version = 0, nx = 0, ny = 0, nz = 0, px = 0, py = 0, pz = 0;
    in >> magic >> version >> nx >> ny >> nz >> px >> py >> pz;
    if (magic != "porolb-voxel" || version != 1)
      throw ConfigError(std::string(path) + ": not a porolb voxel file");
    in.get();
    const int64_t cells = int64_t(nx) * ny * nz;
    auto g = std::make_unique<pgpu_voxel_geometry>();
    g->flags.resize(cells);  // a negative count throws like the reference's vector
    in.read(reinterpret_cast<char*>(g->flags.data()), static_cast<std::streamsize>(cells));
    if (in.gcount() != static_cast<std::streamsize>(cells))
      throw ConfigError(std::string(path) + ": truncated voxel data");
    g->dims[0] = nx;
    g->dims[1] = ny;
    g->dims[2] = nz;
    const bool per[3] = {px != 0, py != 0, pz != 0};
    for (int a = 0; a < 3; ++a) g->periodic[a] = per[a] ? 1 : 0;
    g->porosity.assign(nz > 0 ? nz : 0, 0.0);

    struct Part {
      std::vector<int64_t> lf, ls;
      std::vector<int32_t> ld;
      int64_t fluid = 0;
      bool open_face = false;
    };
    const int nt = std::max(1, std::min(hw_threads(), nz));
    std::vector<Part> parts(nt);
    const uint8_t* fl = g->flags.data();
    parallel_for(nz, [&](int64_t z0, int64_t z1, int t) {
      Part& P = parts[t];
      for (int z = (int)z0; z < (int)z1 && !P.open_face; ++z) {
        int64_t fluid = 0;
        for (int y = 0; y < ny && !P.open_face; ++y) {
          for (int x = 0; x < nx; ++x) {
            const int64_t c = (int64_t(z) * ny + y) * nx + x;
            if (fl[c] != 0) continue;
            ++fluid;
            for (int k = 1; k < 19; ++k) {
              const int xn = wrap_or_open(x + kE[k][0], nx, per[0]);
              const int yn = wrap_or_open(y + kE[k][1], ny, per[1]);
              const int zn = wrap_or_open(z + kE[k][2], nz, per[2]);
              if (xn < 0 || yn < 0 || zn < 0) {
                P.open_face = true;
                break;
              }
              if (fl[(int64_t(zn) * ny + yn) * nx + xn] == 0) continue;
              const int xp = wrap_or_open(x - kE[k][0], nx, per[0]);
              const int yp = wrap_or_open(y - kE[k][1], ny, per[1]);
              const int zp = wrap_or_open(z - kE[k][2], nz, per[2]);
              int64_t second = -1;
              if (xp >= 0 && yp >= 0 && zp >= 0) {
                const int64_t sc = (int64_t(zp) * ny + yp) * nx + xp;
                if (fl[sc] == 0) second = sc;
              }
              P.lf.push_back(c);
              P.ls.push_back(second);
              P.ld.push_back(k);
            }
            if (P.open_face) break;
          }
        }
        g->porosity[z] = static_cast<double>(fluid) / (static_cast<double>(nx) * ny);
        P.fluid += fluid;
      }
    }, nt);
    int64_t total = 0;
    for (const Part& P : parts) {
      if (P.open_face)
        throw ConfigError(std::string(path) + ": fluid cell touches a non-periodic open face");
      total += static_cast<int64_t>(P.lf.size());
      g->fluid_cells += P.fluid;
    }
    g->lf.resize(total);
    g->ls.resize(total);
    g->ld.resize(total);
    g->lq.assign(total, 0.5f);
    g->lm.assign(total, 0);
    std::vector<int64_t> off(nt + 1, 0);
    for (int t = 0; t < nt; ++t) off[t + 1] = off[t] + static_cast<int64_t>(parts[t].lf.size());
    parallel_for(nt, [&](int64_t a, int64_t b, int) {
      for (int64_t t = a; t < b; ++t) {
        const Part& P = parts[t];
        std::copy(P.lf.begin(), P.lf.end(), g->lf.begin() + off[t]);
        std::copy(P.ls.begin(), P.ls.end(), g->ls.begin() + off[t]);
        std::copy(P.ld.begin(), P.ld.end(), g->ld.begin() + off[t]);
      }
    });
    if (g->fluid_cells == 0) throw GeometryError(std::string(path) + ": geometry has no fluid cells");
    *out_geom = g.release();
  });
}

}  // extern "C"
