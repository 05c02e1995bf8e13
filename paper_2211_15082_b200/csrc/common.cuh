// Shared helpers for the glint B200 kernels: error plumbing, launch checks,
// small device utilities.  Every extern "C" entry point validates its
// arguments on the host, launches asynchronously on the caller's stream and
// converts CUDA failures into GLINT_ECUDA with a message.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "../../include/glint_b200.h"

namespace glint {

void set_error(const char* fmt, ...);
void clear_error();

// Convert the sticky/last launch error into a status code.
int launch_status(const char* what);

inline cudaStream_t as_stream(glint_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int sm_count();  // cached per current device

int tuning(int key);  // glint_set_tuning knobs (0 = default behaviour)

int fused_debug_counters(uint64_t* host_out, int n, int reset);   // K7 phase counters

constexpr int kWarp = 32;

// Once-per-device guard for host-side kernel configuration
// (cudaFuncSetAttribute is a per-device property; a process-wide flag would
// skip it on the second device a process uses).  Idempotent under races.
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  static uint64_t bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
  }
  bool needed() const { return (done.load(std::memory_order_acquire) & bit()) == 0; }
  void mark() { done.fetch_or(bit(), std::memory_order_release); }
};

}  // namespace glint

#define GLINT_REQUIRE(cond, ...)          \
  do {                                    \
    if (!(cond)) {                        \
      ::glint::set_error(__VA_ARGS__);    \
      return GLINT_EINVAL;                \
    }                                     \
  } while (0)

#define GLINT_CUDA(call)                                                          \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::glint::set_error("%s failed: %s", #call, cudaGetErrorString(_e));         \
      return GLINT_ECUDA;                                                         \
    }                                                                             \
  } while (0)

// Device helpers ------------------------------------------------------------
namespace glint {

__device__ __forceinline__ float4 ldg_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace glint
