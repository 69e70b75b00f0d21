// Shared by the host (voxelize.cpp) and device (voxelize_device.cu) voxelizers.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/porolb_gpu.h"

struct pgpu_voxel_geometry {
  int32_t dims[3];
  uint8_t periodic[3];
  std::vector<uint8_t> flags;
  std::vector<int64_t> lf, ls;
  std::vector<int32_t> ld;
  std::vector<float> lq;
  std::vector<uint8_t> lm;
  std::vector<double> porosity;
  int64_t fluid_cells = 0;
  int32_t q_fallback_count = 0;
  int32_t has_lo = 0, has_hi = 0;
  double lo = 0.0, hi = 0.0;
  int32_t slab = 0, x_offset = 0, global_nx = 0;
  std::vector<uint8_t> ghost_lo, ghost_hi;
};

namespace pgpu {

struct VoxSph {
  double c[3];
  double r;
};

// Sphere images (geometry.cpp:442-462) binned by their reject boxes
// (geometry.cpp:607-611): every image the reference's cheap reject would keep
// for a point p lies in p's bin.
struct VoxHostGrid {
  std::vector<VoxSph> spheres;
  double h = 8.0;
  int gx = 1, gy = 1, gz = 1;
  std::vector<int64_t> start;
  std::vector<int32_t> items;
};
VoxHostGrid build_vox_host_grid(const pgpu_sphere_pack& pack, const uint8_t periodic[3],
                                const int32_t dims[3]);

}  // namespace pgpu
