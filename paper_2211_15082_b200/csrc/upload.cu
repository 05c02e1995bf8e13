// Asynchronous CSR upload with host-side int64 -> int32 narrowing.
//
// The reference hands the engine a host CscGraph with int64 ids
// (storage.py:33-66); the device keeps int32 ids.  Narrowing on the host lets
// the CSR cross PCIe at half the bytes (the e2e path's H2D is its floor), but
// it must not hold the Python thread that launches layer-1 batches: a native
// thread narrows row chunk k on `threads` CPU threads into the caller's pinned
// staging buffer, queues its cudaMemcpyAsync on the copy stream and records
// chunk k's event; consumers wait for "queued" on the host (condition
// variable, no GIL held -- ctypes releases it) and then for the event on
// their stream.
#include <atomic>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace glint {
namespace {

struct Upload {
  std::thread worker;
  int id_bytes = 4;              // 4: int32 ids; 3: 24-bit ids unpacked on the device
  std::vector<cudaEvent_t> events;
  std::vector<int64_t> bounds;   // K+1 edge offsets
  std::vector<int> queued;       // guarded by mu
  std::mutex mu;
  std::condition_variable cv;
  int error = 0;
  int device = 0;
};

void narrow_parallel(const int64_t* src, int32_t* dst, int64_t n, int threads, int64_t* bad) {
  const int t = (n < (1 << 16)) ? 1 : std::max(1, std::min(threads, 64));
  std::vector<int64_t> b(t, 0);
  auto work = [&](int k) {
    const int64_t lo = n * k / t, hi = n * (k + 1) / t;
    int64_t c = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t v = src[i];
      c += (v < INT32_MIN || v > INT32_MAX);
      dst[i] = static_cast<int32_t>(v);
    }
    b[k] = c;
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  for (int64_t c : b) *bad += c;
}

// 24-bit little-endian packing (ids < 2^24): 3 bytes per id cross PCIe
// instead of 4.  Thread k packs ids [lo, hi) with 4-byte stores advancing by
// 3; the last id of a range is written bytewise so no store passes `hi`.
// Branch-free form: 8 ids -> 24 bytes as three 64-bit stores, thread ranges
// aligned to 8 ids; the range check ORs the ids (any id outside [0, 2^24)
// leaves a bit at or above 24).  The e2e call packs 124M ids while the
// features stream over PCIe (host-memory bound): the per-id form spent ~25%
// more time here.
void pack24_fast(const int64_t* src, uint8_t* dst, int64_t n, int threads, int64_t* bad) {
  const int t = (n < (1 << 16)) ? 1 : std::max(1, std::min(threads, 64));
  const int64_t groups = n / 8;
  std::vector<int64_t> b(t, 0);
  auto work = [&](int k) {
    const int64_t g0 = groups * k / t, g1 = groups * (k + 1) / t;
    uint64_t acc = 0;
    for (int64_t g = g0; g < g1; ++g) {
      const int64_t* q = src + 8 * g;
      uint64_t v[8];
      for (int j = 0; j < 8; ++j) {
        v[j] = static_cast<uint64_t>(q[j]);
        acc |= v[j];
      }
      const uint64_t w0 = v[0] | (v[1] << 24) | (v[2] << 48);
      const uint64_t w1 = (v[2] >> 16) | (v[3] << 8) | (v[4] << 32) | (v[5] << 56);
      const uint64_t w2 = (v[5] >> 8) | (v[6] << 16) | (v[7] << 40);
      uint8_t* p = dst + 24 * g;
      std::memcpy(p, &w0, 8);
      std::memcpy(p + 8, &w1, 8);
      std::memcpy(p + 16, &w2, 8);
    }
    if (k == t - 1) {              // tail ids bytewise
      for (int64_t i = 8 * groups; i < n; ++i) {
        const uint64_t u = static_cast<uint64_t>(src[i]);
        acc |= u;
        dst[3 * i] = static_cast<uint8_t>(u);
        dst[3 * i + 1] = static_cast<uint8_t>(u >> 8);
        dst[3 * i + 2] = static_cast<uint8_t>(u >> 16);
      }
    }
    b[k] = (acc >> 24) != 0;
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  for (int64_t c : b) *bad += c;
}

void pack24_parallel(const int64_t* src, uint8_t* dst, int64_t n, int threads, int64_t* bad) {
  if (tuning(GLINT_TUNE_PACK24_LOOP) == 0) {
    pack24_fast(src, dst, n, threads, bad);
    return;
  }
  const int t = (n < (1 << 16)) ? 1 : std::max(1, std::min(threads, 64));
  std::vector<int64_t> b(t, 0);
  auto work = [&](int k) {
    const int64_t lo = n * k / t, hi = n * (k + 1) / t;
    int64_t c = 0;
    uint8_t* p = dst + 3 * lo;
    for (int64_t i = lo; i < hi; ++i, p += 3) {
      const int64_t v = src[i];
      c += (v < 0 || v >= (1LL << 24));
      const uint32_t u = static_cast<uint32_t>(v) & 0xFFFFFFu;
      if (i + 1 < hi) {
        std::memcpy(p, &u, 4);    // the 4th byte is overwritten by id i+1
      } else {
        p[0] = static_cast<uint8_t>(u);
        p[1] = static_cast<uint8_t>(u >> 8);
        p[2] = static_cast<uint8_t>(u >> 16);
      }
    }
    b[k] = c;
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  for (int64_t c : b) *bad += c;
}

// Device side of the 24-bit upload: 4 ids (12 bytes) per thread.
__global__ void unpack24_kernel(const uint8_t* __restrict__ src, int32_t* __restrict__ dst,
                                int64_t n) {
  const int64_t i0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = i0 + j;
    if (i < n) {
      const uint8_t* p = src + 3 * i;
      dst[i] = static_cast<int32_t>(p[0] | (p[1] << 8) | (p[2] << 16));
    }
  }
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

static int upload_start(const int64_t* src_host, int32_t* dst_dev, void* stage_pinned,
                        uint8_t* dev_stage, int id_bytes, const int64_t* chunk_edges,
                        int32_t n_chunks, int32_t threads, glint_stream_t copy_stream,
                        void** handle_out) {
  GLINT_REQUIRE(handle_out && n_chunks >= 0 && chunk_edges, "upload_start: bad argument");
  GLINT_REQUIRE(id_bytes == 4 || id_bytes == 3, "upload_start: id_bytes must be 3 or 4");
  GLINT_REQUIRE(n_chunks == 0 || (src_host && dst_dev && stage_pinned &&
                                  (id_bytes == 4 || dev_stage)),
                "upload_start: null buffer");
  for (int k = 0; k < n_chunks; ++k)
    GLINT_REQUIRE(chunk_edges[k] <= chunk_edges[k + 1] && chunk_edges[k] >= 0,
                  "upload_start: chunk bounds must be non-decreasing");
  auto* u = new Upload();
  u->id_bytes = id_bytes;
  GLINT_CUDA(cudaGetDevice(&u->device));
  u->bounds.assign(chunk_edges, chunk_edges + n_chunks + 1);
  u->queued.assign(n_chunks, 0);
  u->events.resize(n_chunks);
  for (int k = 0; k < n_chunks; ++k)
    GLINT_CUDA(cudaEventCreateWithFlags(&u->events[k], cudaEventDisableTiming));
  cudaStream_t s = as_stream(copy_stream);
  u->worker = std::thread([u, src_host, dst_dev, stage_pinned, dev_stage, threads, s]() {
    cudaSetDevice(u->device);
    for (size_t k = 0; k + 1 < u->bounds.size(); ++k) {
      const int64_t e0 = u->bounds[k], e1 = u->bounds[k + 1];
      int err = 0;
      if (e1 > e0) {
        int64_t bad = 0;
        if (u->id_bytes == 4) {
          int32_t* st = static_cast<int32_t*>(stage_pinned);
          narrow_parallel(src_host + e0, st + e0, e1 - e0, threads, &bad);
          if (bad) err = GLINT_EINVAL;
          else if (cudaMemcpyAsync(dst_dev + e0, st + e0, (e1 - e0) * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s) != cudaSuccess)
            err = GLINT_ECUDA;
        } else {
          uint8_t* st = static_cast<uint8_t*>(stage_pinned);
          pack24_parallel(src_host + e0, st + 3 * e0, e1 - e0, threads, &bad);
          if (bad) {
            err = GLINT_EINVAL;
          } else if (cudaMemcpyAsync(dev_stage + 3 * e0, st + 3 * e0, 3 * (e1 - e0),
                                     cudaMemcpyHostToDevice, s) != cudaSuccess) {
            err = GLINT_ECUDA;
          } else {
            const int64_t blocks = ceil_div(ceil_div(e1 - e0, 4), 256);
            unpack24_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(dev_stage + 3 * e0,
                                                                          dst_dev + e0, e1 - e0);
            if (cudaGetLastError() != cudaSuccess) err = GLINT_ECUDA;
          }
        }
      }
      if (!err && cudaEventRecord(u->events[k], s) != cudaSuccess) err = GLINT_ECUDA;
      {
        std::lock_guard<std::mutex> lk(u->mu);
        if (err) {
          u->error = err;
          for (auto& q : u->queued) q = 1;
        } else {
          u->queued[k] = 1;
        }
      }
      u->cv.notify_all();
      if (err) return;
    }
  });
  *handle_out = u;
  return GLINT_OK;
}

int glint_upload_start(const int64_t* src_host, int32_t* dst_dev, int32_t* stage_pinned,
                       const int64_t* chunk_edges, int32_t n_chunks, int32_t threads,
                       glint_stream_t copy_stream, void** handle_out) {
  return upload_start(src_host, dst_dev, stage_pinned, nullptr, 4, chunk_edges, n_chunks, threads,
                      copy_stream, handle_out);
}

int glint_upload_start_packed(const int64_t* src_host, int32_t* dst_dev, uint8_t* stage_pinned,
                              uint8_t* dev_stage, int32_t id_bytes, const int64_t* chunk_edges,
                              int32_t n_chunks, int32_t threads, glint_stream_t copy_stream,
                              void** handle_out) {
  return upload_start(src_host, dst_dev, stage_pinned, dev_stage, id_bytes, chunk_edges, n_chunks,
                      threads, copy_stream, handle_out);
}

// Row-pitched copy in any direction (cudaMemcpy2DAsync, cudaMemcpyDefault):
// the e2e output sink streams finished rows of a pitched device store straight
// into the caller's dense pinned host array, with no device-side repacking.
int glint_copy_rows_async(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                          int64_t row_bytes, int64_t rows, glint_stream_t stream) {
  GLINT_REQUIRE(rows >= 0 && row_bytes >= 0 && dst_pitch >= row_bytes && src_pitch >= row_bytes,
                "copy_rows_async: bad pitches (dst %lld, src %lld, row %lld)",
                static_cast<long long>(dst_pitch), static_cast<long long>(src_pitch),
                static_cast<long long>(row_bytes));
  if (rows == 0 || row_bytes == 0) return GLINT_OK;
  GLINT_REQUIRE(dst && src, "copy_rows_async: null pointer");
  GLINT_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(dst_pitch), src,
                               static_cast<size_t>(src_pitch), static_cast<size_t>(row_bytes),
                               static_cast<size_t>(rows), cudaMemcpyDefault, as_stream(stream)));
  return GLINT_OK;
}

// Pageable host -> device copy through pinned staging on `threads` host
// threads.  A plain cudaMemcpy from pageable memory goes through the driver's
// own staging at ~10 GB/s (the reference API hands run_inference numpy
// features); here thread t owns a contiguous slice of the source, copies it
// in kStageChunk pieces into its two pinned halves (memcpy on the CPU) and
// queues each piece's cudaMemcpyAsync, waiting for a half's previous copy
// before refilling it.  The staging is allocated once per process (and grown
// on demand) under a mutex that also serialises concurrent callers.  Returns
// after every piece has landed (the synchronous semantics of the pageable copy).
namespace {
constexpr size_t kStageChunk = size_t{4} << 20;
std::mutex g_stage_mu;
uint8_t* g_stage = nullptr;
size_t g_stage_bytes = 0;
}  // namespace

int glint_h2d_pageable(void* dst_dev, const void* src_host, int64_t bytes, int32_t threads,
                       glint_stream_t stream) {
  GLINT_REQUIRE(bytes >= 0 && threads >= 1, "h2d_pageable: bad argument");
  if (bytes == 0) return GLINT_OK;
  GLINT_REQUIRE(dst_dev && src_host, "h2d_pageable: null pointer");
  std::lock_guard<std::mutex> lk(g_stage_mu);
  const int t = static_cast<int>(std::min<int64_t>(
      std::min(threads, 32), std::max<int64_t>(1, bytes / static_cast<int64_t>(kStageChunk))));
  const size_t need = static_cast<size_t>(t) * 2 * kStageChunk;
  if (g_stage_bytes < need) {
    if (g_stage) cudaFreeHost(g_stage);
    g_stage = nullptr;
    g_stage_bytes = 0;
    GLINT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_stage), need, cudaHostAllocDefault));
    g_stage_bytes = need;
  }
  int dev = 0;
  GLINT_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = as_stream(stream);
  std::atomic<int> err{0};
  auto work = [&](int k) {
    cudaSetDevice(dev);
    const int64_t lo = bytes * k / t, hi = bytes * (k + 1) / t;
    uint8_t* half[2] = {g_stage + (2 * k) * kStageChunk, g_stage + (2 * k + 1) * kStageChunk};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    for (int h = 0; h < 2; ++h)
      if (cudaEventCreateWithFlags(&ev[h], cudaEventDisableTiming) != cudaSuccess) err = 1;
    int h = 0;
    for (int64_t off = lo; off < hi && !err; off += static_cast<int64_t>(kStageChunk)) {
      const size_t len = static_cast<size_t>(std::min<int64_t>(kStageChunk, hi - off));
      if (used[h] && cudaEventSynchronize(ev[h]) != cudaSuccess) err = 1;
      std::memcpy(half[h], static_cast<const uint8_t*>(src_host) + off, len);
      if (cudaMemcpyAsync(static_cast<uint8_t*>(dst_dev) + off, half[h], len,
                          cudaMemcpyHostToDevice, s) != cudaSuccess ||
          cudaEventRecord(ev[h], s) != cudaSuccess)
        err = 1;
      used[h] = true;
      h ^= 1;
    }
    for (int q = 0; q < 2; ++q) {
      if (ev[q]) {
        if (used[q] && cudaEventSynchronize(ev[q]) != cudaSuccess) err = 1;
        cudaEventDestroy(ev[q]);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  if (err) {
    set_error("h2d_pageable: CUDA copy failed");
    return GLINT_ECUDA;
  }
  return GLINT_OK;
}

// Blocks until chunk k's copy is queued, then makes `stream` wait for it.
int glint_upload_wait(void* handle, int32_t chunk, glint_stream_t stream) {
  auto* u = static_cast<Upload*>(handle);
  GLINT_REQUIRE(u && chunk >= 0 && chunk < static_cast<int>(u->queued.size()),
                "upload_wait: bad chunk");
  {
    std::unique_lock<std::mutex> lk(u->mu);
    u->cv.wait(lk, [&] { return u->queued[chunk] != 0; });
    if (u->error) {
      set_error("upload: chunk failed (%s)", u->error == GLINT_EINVAL
                ? (u->id_bytes == 3 ? "node ids do not fit 24 bits" : "node ids do not fit int32")
                : "CUDA copy error");
      return u->error;
    }
  }
  GLINT_CUDA(cudaStreamWaitEvent(as_stream(stream), u->events[chunk], 0));
  return GLINT_OK;
}

// 1 when chunk k has been queued and its copy has landed, 0 otherwise.
int glint_upload_query(void* handle, int32_t chunk) {
  auto* u = static_cast<Upload*>(handle);
  GLINT_REQUIRE(u && chunk >= 0 && chunk < static_cast<int>(u->queued.size()),
                "upload_query: bad chunk");
  {
    std::lock_guard<std::mutex> lk(u->mu);
    if (u->error) {
      set_error("upload: a chunk failed");
      return u->error;
    }
    if (!u->queued[chunk]) return 0;
  }
  const cudaError_t e = cudaEventQuery(u->events[chunk]);
  if (e == cudaErrorNotReady) return 0;
  GLINT_CUDA(e);
  return 1;
}

// Joins the worker and releases the events (call once, after the last wait).
int glint_upload_finish(void* handle) {
  auto* u = static_cast<Upload*>(handle);
  if (!u) return GLINT_OK;
  if (u->worker.joinable()) u->worker.join();
  for (auto ev : u->events) cudaEventDestroy(ev);
  const int err = u->error;
  delete u;
  return err ? GLINT_ECUDA : GLINT_OK;
}

}  // extern "C"
