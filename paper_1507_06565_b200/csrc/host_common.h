// Host-side helpers shared by the C-ABI translation units.  Compiled with
// -ffp-contract=off: every host formula below reproduces the reference
// expression order, so host-derived constants are bit-identical to what the
// reference computes inline.
#pragma once
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/porolb_gpu.h"

namespace pgpu {

// Reference exception types (errors.hpp:9-21) mapped onto status codes.
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalInstability : std::runtime_error {
  explicit NumericalInstability(const std::string& m) : std::runtime_error(m) {}
};
struct GeometryError : std::runtime_error {
  explicit GeometryError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& f) {
  try {
    f();
    return PGPU_OK;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return PGPU_ERR_CONFIG;
  } catch (const NumericalInstability& e) {
    set_last_error(e.what());
    return PGPU_ERR_INSTABILITY;
  } catch (const GeometryError& e) {
    set_last_error(e.what());
    return PGPU_ERR_GEOMETRY;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return PGPU_ERR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PGPU_ERR_INTERNAL;
  }
}

// D3Q19, reference order (lattice.cpp:13-33).
constexpr int kE[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},   {0, -1, 0},
                           {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                           {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                           {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
inline int opposite(int k) { return k == 0 ? 0 : ((k & 1) ? k + 1 : k - 1); }
// lattice.cpp:34-37 weights by speed order.
inline double weight(int k) {
  const int order = std::abs(kE[k][0]) + std::abs(kE[k][1]) + std::abs(kE[k][2]);
  return (order == 0) ? 1.0 / 3.0 : (order == 1) ? 1.0 / 18.0 : 1.0 / 36.0;
}

// Simple fork-join over [0, n) with contiguous chunks, one per hardware thread.
inline void parallel_for(int64_t n, const std::function<void(int64_t, int64_t, int)>& fn,
                         int max_threads = 0) {
  int t = static_cast<int>(std::thread::hardware_concurrency());
  if (t <= 0) t = 1;
  if (max_threads > 0 && t > max_threads) t = max_threads;
  if (n < t) t = static_cast<int>(n > 0 ? n : 1);
  if (t <= 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(t);
  for (int i = 0; i < t; ++i) {
    const int64_t a = n * i / t, b = n * (i + 1) / t;
    th.emplace_back([&fn, a, b, i] { fn(a, b, i); });
  }
  for (auto& x : th) x.join();
}

inline int hw_threads() {
  const int t = static_cast<int>(std::thread::hardware_concurrency());
  return t > 0 ? t : 1;
}

}  // namespace pgpu
