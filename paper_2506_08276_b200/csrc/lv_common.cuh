// lv_common.cuh — shared helpers for the B200 LEANN search library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/leann_b200.h"

namespace lv {

void set_error(const std::string &msg);
// Kernel attributes (e.g. the dynamic shared-memory opt-in) are per device context:
// true the first time this is called for the current device with this flag word,
// which it then marks (launchers keep one word per kernel).
inline bool first_on_device(unsigned long long &done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return false;
  done |= bit;
  return true;
}
// Process-wide count of kernels this library has launched (lv_kernel_launches).
void note_launch(long long n = 1);

struct Status {
  int code;
  std::string msg;
};

#define LV_CHECK_CUDA(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      lv::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                    __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");   \
      return LV_ERR_INTERNAL;                                                      \
    }                                                                              \
  } while (0)

#define LV_REQUIRE(cond, code, msg)   \
  do {                                \
    if (!(cond)) {                    \
      lv::set_error(msg);             \
      return (code);                  \
    }                                 \
  } while (0)

#define LV_TRY(expr)          \
  do {                        \
    int _rc = (expr);         \
    if (_rc != LV_OK) return _rc; \
  } while (0)

constexpr int kMaxLevels = 32;

// Make `dev` current for the lifetime of the guard.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
constexpr int kCentroids = 256;  // pq.py:29 CENTROIDS_PER_SUBSPACE

// ---------------------------------------------------------------------------
// Ordering helpers. Python compares (float, int) tuples with IEEE semantics:
// -0.0 == +0.0, so both map to the same key here (search.py:217-251 tuples).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ord_f32(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) == 0u) u = 0u;  // canonical +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ bool pair_less(float da, int32_t ia, float db, int32_t ib) {
  uint32_t a = ord_f32(da), b = ord_f32(db);
  return a < b || (a == b && ia < ib);
}

__device__ __forceinline__ bool bit_test(const uint32_t *bits, int64_t i) {
  return (bits[i >> 5] >> (i & 31)) & 1u;
}

__device__ __forceinline__ void bit_set(uint32_t *bits, int64_t i) {
  atomicOr(bits + (i >> 5), 1u << (i & 31));
}

}  // namespace lv
