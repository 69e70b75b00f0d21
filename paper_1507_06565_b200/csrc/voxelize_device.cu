// Device voxelizer: the reference voxelize()
// (geometry.cpp:491-632) on the B200, byte-identical to it.
//
//  * sphere images (effective_spheres, geometry.cpp:442-462) and the reject-box
//    grid are built on the host exactly as in voxelize.cpp;
//  * k_vox_flags: one thread per cell; candidate images come from the grid bin
//    of the cell centre (every image whose bounding box holds the cell is in
//    it), then the reference's bounding-box membership and d^2 < r^2 test;
//  * k_vox_count / CUB exclusive scan / k_vox_links: links in ascending
//    (cell, k) order with second_fluid, q from the exact ray-sphere / ray-plane
//    intersections (geometry.cpp:465-487, 604-625).
// Every fp64 operation is an explicit round-to-nearest intrinsic in the
// reference expression order (the host reference has no FMA), so flags, links
// and the fp32 q bits match the host voxelizer bit for bit.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <memory>
#include <sstream>
#include <vector>

#include "host_common.h"
#include "voxel_geometry.h"

namespace pgpu {
namespace {

#define VADD(a, b) __dadd_rn((a), (b))
#define VSUB(a, b) __dsub_rn((a), (b))
#define VMUL(a, b) __dmul_rn((a), (b))
#define VDIV(a, b) __ddiv_rn((a), (b))

using DSph = VoxSph;

struct VoxParams {
  int nx, ny, nz;
  int px, py, pz;
  int wall_lo, wall_hi;
  double plate_z;
  int n_planes;
  double planes[2];
  double q_clamp_min;
  // grid
  double h;
  int gx, gy, gz;
  const int64_t* gstart;
  const int32_t* gitems;
  const DSph* sph;
};

__constant__ int VE[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},   {0, -1, 0},
                              {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                              {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                              {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};

__device__ __forceinline__ int64_t vbin(const VoxParams& v, const double p[3]) {
  int x = (int)floor(VDIV(p[0], v.h));
  int y = (int)floor(VDIV(p[1], v.h));
  int z = (int)floor(VDIV(p[2], v.h));
  x = min(v.gx - 1, max(0, x));
  y = min(v.gy - 1, max(0, y));
  z = min(v.gz - 1, max(0, z));
  return ((int64_t)z * v.gy + y) * v.gx + x;
}

__device__ __forceinline__ int vwrap(int val, int n, int periodic) {
  if (val >= 0 && val < n) return val;
  if (!periodic) return -1;
  return (val % n + n) % n;
}

// geometry.cpp:501-551 for one cell
__global__ void k_vox_flags(VoxParams v, uint8_t* flags) {
  const int64_t cells = (int64_t)v.nx * v.ny * v.nz;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int x = (int)(c % v.nx);
  const int64_t r = c / v.nx;
  const int y = (int)(r % v.ny), z = (int)(r / v.ny);
  uint8_t f = 0;
  if (v.plate_z > 0.0) {  // cells at or below floor(plate - 1/2)
    const int k_max = (int)floor(VSUB(v.plate_z, 0.5));
    if (z <= min(k_max, v.nz - 1)) f = 1;
  }
  if (!f) {
    const double pc[3] = {VADD((double)x, 0.5), VADD((double)y, 0.5), VADD((double)z, 0.5)};
    const int64_t b = vbin(v, pc);
    for (int64_t it = v.gstart[b]; it < v.gstart[b + 1] && !f; ++it) {
      const DSph s = v.sph[v.gitems[it]];
      // bounding box of geometry.cpp:515-520
      const int bx0 = max(0, (int)floor(VSUB(VSUB(s.c[0], s.r), 0.5)));
      const int bx1 = min(v.nx - 1, (int)ceil(VADD(s.c[0], s.r)));
      const int by0 = max(0, (int)floor(VSUB(VSUB(s.c[1], s.r), 0.5)));
      const int by1 = min(v.ny - 1, (int)ceil(VADD(s.c[1], s.r)));
      const int bz0 = max(0, (int)floor(VSUB(VSUB(s.c[2], s.r), 0.5)));
      const int bz1 = min(v.nz - 1, (int)ceil(VADD(s.c[2], s.r)));
      if (x < bx0 || x > bx1 || y < by0 || y > by1 || z < bz0 || z > bz1) continue;
      const double dx = VSUB(VADD((double)x, 0.5), s.c[0]);
      const double dy = VSUB(VADD((double)y, 0.5), s.c[1]);
      const double dz = VSUB(VADD((double)z, 0.5), s.c[2]);
      if (VADD(VADD(VMUL(dx, dx), VMUL(dy, dy)), VMUL(dz, dz)) < VMUL(s.r, s.r)) f = 1;
    }
  }
  if ((v.wall_lo && z == 0) || (v.wall_hi && z == v.nz - 1)) f = 2;  // geometry.cpp:535-551
  flags[c] = f;
}

// Links per fluid cell; flags an open non-periodic face (geometry.cpp:583-588).
__global__ void k_vox_count(VoxParams v, const uint8_t* flags, int64_t* count,
                            unsigned long long* first_open) {
  const int64_t cells = (int64_t)v.nx * v.ny * v.nz;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  int n = 0;
  if (flags[c] == 0) {
    const int x = (int)(c % v.nx);
    const int64_t r = c / v.nx;
    const int y = (int)(r % v.ny), z = (int)(r / v.ny);
    for (int k = 1; k < 19; ++k) {
      const int xn = vwrap(x + VE[k][0], v.nx, v.px);
      const int yn = vwrap(y + VE[k][1], v.ny, v.py);
      const int zn = vwrap(z + VE[k][2], v.nz, v.pz);
      if (xn < 0 || yn < 0 || zn < 0) {
        atomicMin(first_open, (unsigned long long)c);
        continue;
      }
      if (flags[((int64_t)zn * v.ny + yn) * v.nx + xn] != 0) ++n;
    }
  }
  count[c] = n;
}

// geometry.cpp:465-479
__device__ __forceinline__ bool vray_sphere(const double p[3], int k, const DSph& s,
                                            double& t_out) {
  const int e0 = VE[k][0], e1 = VE[k][1], e2 = VE[k][2];
  const double d0 = VSUB(p[0], s.c[0]), d1 = VSUB(p[1], s.c[1]), d2 = VSUB(p[2], s.c[2]);
  const double a = (double)(e0 * e0 + e1 * e1 + e2 * e2);
  const double b = VMUL(2.0, VADD(VADD(VMUL((double)e0, d0), VMUL((double)e1, d1)),
                                  VMUL((double)e2, d2)));
  const double cc =
      VSUB(VADD(VADD(VMUL(d0, d0), VMUL(d1, d1)), VMUL(d2, d2)), VMUL(s.r, s.r));
  const double disc = VSUB(VMUL(b, b), VMUL(VMUL(4.0, a), cc));
  if (disc < 0.0) return false;
  const double sq = __dsqrt_rn(disc);
  const double ts[2] = {VDIV(VSUB(-b, sq), VMUL(2.0, a)), VDIV(VADD(-b, sq), VMUL(2.0, a))};
  bool have = false;
  double best = 0.0;
  for (int i = 0; i < 2; ++i) {
    const double t = ts[i];
    if (t > 0.0 && t <= VADD(1.0, 1e-12) && (!have || t < best)) {
      best = t;
      have = true;
    }
  }
  t_out = best;
  return have;
}

// geometry.cpp:481-487
__device__ __forceinline__ bool vray_plane(const double p[3], int k, double plane, double& t) {
  const int e2 = VE[k][2];
  if (e2 == 0) return false;
  const double tt = VDIV(VSUB(plane, p[2]), (double)e2);
  if (tt > 0.0 && tt <= VADD(1.0, 1e-12)) {
    t = tt;
    return true;
  }
  return false;
}

__global__ void k_vox_links(VoxParams v, const uint8_t* flags, const int64_t* offset,
                            int64_t* lf, int64_t* ls, int32_t* ld, float* lq,
                            unsigned int* q_fallbacks) {
  const int64_t cells = (int64_t)v.nx * v.ny * v.nz;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells || flags[c] != 0) return;
  const int x = (int)(c % v.nx);
  const int64_t r = c / v.nx;
  const int y = (int)(r % v.ny), z = (int)(r / v.ny);
  int64_t o = offset[c];
  unsigned int fb = 0;
  const double pc[3] = {VADD((double)x, 0.5), VADD((double)y, 0.5), VADD((double)z, 0.5)};
  const int64_t b = vbin(v, pc);
  for (int k = 1; k < 19; ++k) {
    const int xn = vwrap(x + VE[k][0], v.nx, v.px);
    const int yn = vwrap(y + VE[k][1], v.ny, v.py);
    const int zn = vwrap(z + VE[k][2], v.nz, v.pz);
    if (xn < 0 || yn < 0 || zn < 0) continue;
    if (flags[((int64_t)zn * v.ny + yn) * v.nx + xn] == 0) continue;
    const int kb = (k & 1) ? k + 1 : k - 1;
    int64_t second = -1;
    const int xp = vwrap(x + VE[kb][0], v.nx, v.px);
    const int yp = vwrap(y + VE[kb][1], v.ny, v.py);
    const int zp = vwrap(z + VE[kb][2], v.nz, v.pz);
    if (xp >= 0 && yp >= 0 && zp >= 0) {
      const int64_t pcell = ((int64_t)zp * v.ny + yp) * v.nx + xp;
      if (flags[pcell] == 0) second = pcell;
    }
    double q = INFINITY, t;
    for (int64_t it = v.gstart[b]; it < v.gstart[b + 1]; ++it) {
      const DSph s = v.sph[v.gitems[it]];
      if (pc[0] < VSUB(VSUB(s.c[0], s.r), 2.0) || pc[0] > VADD(VADD(s.c[0], s.r), 2.0) ||
          pc[1] < VSUB(VSUB(s.c[1], s.r), 2.0) || pc[1] > VADD(VADD(s.c[1], s.r), 2.0) ||
          pc[2] < VSUB(VSUB(s.c[2], s.r), 2.0) || pc[2] > VADD(VADD(s.c[2], s.r), 2.0))
        continue;
      if (vray_sphere(pc, k, s, t)) q = fmin(q, t);
    }
    if (v.plate_z > 0.0 && vray_plane(pc, k, v.plate_z, t)) q = fmin(q, t);
    for (int i = 0; i < v.n_planes; ++i)
      if (vray_plane(pc, k, v.planes[i], t)) q = fmin(q, t);
    if (!isfinite(q)) {
      q = 0.5;
      ++fb;
    }
    const double qc = q < v.q_clamp_min ? v.q_clamp_min : (1.0 < q ? 1.0 : q);  // std::clamp
    lf[o] = c;
    ls[o] = second;
    ld[o] = k;
    lq[o] = __double2float_rn(qc);
    ++o;
  }
  if (fb) atomicAdd(q_fallbacks, fb);
}

#define VCK(call)                                                                     \
  do {                                                                                \
    cudaError_t e__ = (call);                                                         \
    if (e__ != cudaSuccess) throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n) VCK(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
};

}  // namespace

std::unique_ptr<pgpu_voxel_geometry> voxelize_device_impl(const pgpu_sphere_pack& pack,
                                                          const int32_t dims[3],
                                                          const pgpu_voxelize_options& opt,
                                                          int device) {
  if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0) throw ConfigError("voxel dims must be positive");
  VCK(cudaSetDevice(device));
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t cells = (int64_t)nx * ny * nz;
  // host: images and the reject-box grid, identical to voxelize.cpp
  VoxHostGrid hg = build_vox_host_grid(pack, opt.periodic, dims);
  const std::vector<DSph>& sph = hg.spheres;
  DevBuf<DSph> d_sph(sph.size());
  DevBuf<int64_t> d_start(hg.start.size());
  DevBuf<int32_t> d_items(hg.items.size());
  if (!sph.empty()) VCK(cudaMemcpy(d_sph.p, sph.data(), sph.size() * sizeof(DSph), cudaMemcpyHostToDevice));
  VCK(cudaMemcpy(d_start.p, hg.start.data(), hg.start.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (!hg.items.empty())
    VCK(cudaMemcpy(d_items.p, hg.items.data(), hg.items.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  VoxParams v{};
  v.nx = nx;
  v.ny = ny;
  v.nz = nz;
  v.px = opt.periodic[0];
  v.py = opt.periodic[1];
  v.pz = opt.periodic[2];
  v.wall_lo = opt.wall_z_lo ? 1 : 0;
  v.wall_hi = opt.wall_z_hi ? 1 : 0;
  v.plate_z = pack.bottom_plate_z;
  v.q_clamp_min = opt.q_clamp_min;
  v.n_planes = 0;
  if (opt.wall_z_lo) v.planes[v.n_planes++] = 1.0;
  if (opt.wall_z_hi) v.planes[v.n_planes++] = static_cast<double>(nz - 1);
  v.h = hg.h;
  v.gx = hg.gx;
  v.gy = hg.gy;
  v.gz = hg.gz;
  v.gstart = d_start.p;
  v.gitems = d_items.p;
  v.sph = d_sph.p;

  DevBuf<uint8_t> d_flags(cells);
  const unsigned nb = (unsigned)((cells + 255) / 256);
  k_vox_flags<<<nb, 256>>>(v, d_flags.p);
  VCK(cudaGetLastError());
  auto g = std::make_unique<pgpu_voxel_geometry>();
  g->dims[0] = nx;
  g->dims[1] = ny;
  g->dims[2] = nz;
  for (int a = 0; a < 3; ++a) g->periodic[a] = opt.periodic[a] ? 1 : 0;
  g->global_nx = nx;
  g->has_lo = opt.wall_z_lo ? 1 : 0;
  g->lo = 1.0;
  g->has_hi = opt.wall_z_hi ? 1 : 0;
  g->hi = static_cast<double>(nz - 1);
  if (!g->has_lo) g->lo = 0.0;
  if (!g->has_hi) g->hi = 0.0;
  g->flags.resize(cells);
  VCK(cudaMemcpy(g->flags.data(), d_flags.p, cells, cudaMemcpyDeviceToHost));
  // porosity per plane (geometry.cpp:553-565), on the host from the flags
  g->porosity.assign(nz, 0.0);
  std::vector<int64_t> plane_fluid(nz, 0);
  parallel_for(nz, [&](int64_t za, int64_t zb, int) {
    for (int64_t z = za; z < zb; ++z) {
      int64_t fl = 0;
      const uint8_t* f = g->flags.data() + z * (int64_t)nx * ny;
      for (int64_t i = 0; i < (int64_t)nx * ny; ++i) fl += f[i] == 0;
      plane_fluid[z] = fl;
      g->porosity[z] = static_cast<double>(fl) / (static_cast<double>(nx) * ny);
    }
  });
  g->fluid_cells = 0;
  for (int z = 0; z < nz; ++z) g->fluid_cells += plane_fluid[z];
  if (g->fluid_cells == 0) throw GeometryError("geometry has no fluid cells");

  DevBuf<int64_t> d_count(cells);
  DevBuf<int64_t> d_off(cells);
  DevBuf<unsigned long long> d_open(1);
  DevBuf<unsigned int> d_fb(1);
  const unsigned long long none = ~0ull;
  VCK(cudaMemcpy(d_open.p, &none, sizeof(none), cudaMemcpyHostToDevice));
  VCK(cudaMemset(d_fb.p, 0, sizeof(unsigned int)));
  k_vox_count<<<nb, 256>>>(v, d_flags.p, d_count.p, d_open.p);
  VCK(cudaGetLastError());
  unsigned long long first_open;
  VCK(cudaMemcpy(&first_open, d_open.p, sizeof(first_open), cudaMemcpyDeviceToHost));
  if (first_open != none) {
    const int64_t c = (int64_t)first_open;
    std::ostringstream os;
    os << "fluid cell (" << c % nx << "," << (c / nx) % ny << "," << c / ((int64_t)nx * ny)
       << ") touches a non-periodic open face; add a wall layer or periodic axis";
    throw ConfigError(os.str());
  }
  // exclusive scan of the per-cell link counts (int64 offsets)
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_count.p, d_off.p, cells);
  DevBuf<uint8_t> d_tmp(tmp_bytes);
  VCK(cub::DeviceScan::ExclusiveSum(d_tmp.p, tmp_bytes, d_count.p, d_off.p, cells));
  int64_t last_off = 0, last_cnt = 0;
  VCK(cudaMemcpy(&last_off, d_off.p + cells - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
  VCK(cudaMemcpy(&last_cnt, d_count.p + cells - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
  const int64_t nl = last_off + last_cnt;
  DevBuf<int64_t> d_lf(nl), d_ls(nl);
  DevBuf<int32_t> d_ld(nl);
  DevBuf<float> d_lq(nl);
  k_vox_links<<<nb, 256>>>(v, d_flags.p, d_off.p, d_lf.p, d_ls.p, d_ld.p, d_lq.p, d_fb.p);
  VCK(cudaGetLastError());
  g->lf.resize(nl);
  g->ls.resize(nl);
  g->ld.resize(nl);
  g->lq.resize(nl);
  g->lm.assign(nl, 0);
  if (nl) {
    VCK(cudaMemcpy(g->lf.data(), d_lf.p, nl * sizeof(int64_t), cudaMemcpyDeviceToHost));
    VCK(cudaMemcpy(g->ls.data(), d_ls.p, nl * sizeof(int64_t), cudaMemcpyDeviceToHost));
    VCK(cudaMemcpy(g->ld.data(), d_ld.p, nl * sizeof(int32_t), cudaMemcpyDeviceToHost));
    VCK(cudaMemcpy(g->lq.data(), d_lq.p, nl * sizeof(float), cudaMemcpyDeviceToHost));
  }
  unsigned int fb = 0;
  VCK(cudaMemcpy(&fb, d_fb.p, sizeof(fb), cudaMemcpyDeviceToHost));
  g->q_fallback_count = (int32_t)fb;
  return g;
}

}  // namespace pgpu

using namespace pgpu;

extern "C" int pgpu_voxelize_device(const pgpu_sphere_pack* pack, const int32_t dims[3],
                                    const pgpu_voxelize_options* opt, int32_t device,
                                    pgpu_voxel_geometry** out) {
  return guard([&] {
    if (!pack || !dims || !opt || !out) throw std::invalid_argument("null pointer");
    *out = voxelize_device_impl(*pack, dims, *opt, device).release();
  });
}
