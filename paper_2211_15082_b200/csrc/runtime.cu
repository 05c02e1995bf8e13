// Error plumbing and device queries for the C ABI.
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>

#include "common.cuh"

namespace glint {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: kernel launch failed: %s", what, cudaGetErrorString(e));
    return GLINT_ECUDA;
  }
  return GLINT_OK;
}

int sm_count() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
    // The library's stream-ordered scratch (cudaMallocAsync: the GEMM's W
    // panel) comes from the device's default pool; keep freed blocks mapped
    // instead of returning them at every synchronize (re-mapping costs ~ms).
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess && pool) {
      uint64_t keep = 256ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return cached[dev];
}

static int g_tuning[GLINT_TUNE_COUNT] = {0};

int tuning(int key) { return (key >= 0 && key < GLINT_TUNE_COUNT) ? g_tuning[key] : 0; }

}  // namespace glint

extern "C" {

int glint_set_tuning(int key, int value) {
  GLINT_REQUIRE(key >= 0 && key < GLINT_TUNE_COUNT, "set_tuning: unknown key %d", key);
  glint::g_tuning[key] = value;
  return GLINT_OK;
}

int glint_get_tuning(int key) { return glint::tuning(key); }

const char* glint_last_error(void) { return glint::g_last_error.c_str(); }

int glint_abi_version(void) { return 1; }

int glint_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                      size_t* free_bytes, size_t* total_bytes) {
  // cudaDeviceGetAttribute, not cudaGetDeviceProperties: the latter costs
  // milliseconds to tens of ms per call (it gathers every property), and the
  // request path asks for free HBM once per run_inference (budget="device").
  int prev = 0;
  GLINT_CUDA(cudaGetDevice(&prev));
  if (prev != device) GLINT_CUDA(cudaSetDevice(device));
  if (sm_count) GLINT_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  if (cc_major) GLINT_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  if (cc_minor) GLINT_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  if (free_bytes || total_bytes) {
    size_t f = 0, t = 0;
    GLINT_CUDA(cudaMemGetInfo(&f, &t));
    if (free_bytes) *free_bytes = f;
    if (total_bytes) *total_bytes = t;
  }
  if (prev != device) GLINT_CUDA(cudaSetDevice(prev));
  return GLINT_OK;
}

}  // extern "C"
