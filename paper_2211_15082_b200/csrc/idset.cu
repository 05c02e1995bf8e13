// K6 integer machinery: sorted id sets (bitmap + per-word rank prefix),
// exclusive scans, degree prefixes, slice gathers, graph relabelling.
//
// Reference: kernels.py:56-88 (gather_slices / build_batch_csc /
// trivial_batch_csc: np.unique + np.searchsorted), storage.py:159-165
// (prefix_for_targets), executor.py:118-121 (_expand), executor.py:270-276
// (_StoreEntry.locate), reorder.py:149-181 (apply_order).
//
// A set over [0, N) is a bitmap of W = ceil(N/32) words plus prefix[w] =
// number of members in words < w.  Members come out ascending by
// construction (np.unique order) and rank(u) = prefix[u>>5] +
// popc(word & lowmask) is exactly np.searchsorted(unique_ids, u) for members.
// All results are integers and bit-exact.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace glint {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int64_t kScanTile = kScanThreads * kScanItems;

inline int64_t scan_tiles(int64_t n) { return ceil_div(std::max<int64_t>(n, 1), kScanTile); }

template <typename F>
__global__ void scan_reduce_kernel(int64_t n, F f, int64_t* partials) {
  using BR = cub::BlockReduce<int64_t, kScanThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + i * kScanThreads + threadIdx.x;
    if (idx < n) s += f(idx);
  }
  const int64_t t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) scan_partials_kernel(int64_t nt, int64_t* partials) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  int64_t carry = 0;
  for (int64_t c0 = 0; c0 < nt; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    int64_t v = i < nt ? partials[i] : 0;
    int64_t x, agg;
    BS(tmp).ExclusiveSum(v, x, agg);
    if (i < nt) partials[i] = x + carry;
    carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[nt] = carry;
}

template <typename F>
__global__ void scan_apply_kernel(int64_t n, F f, const int64_t* partials, int64_t* out) {
  using BS = cub::BlockScan<int64_t, kScanThreads>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int64_t items[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) items[i] = (base + i < n) ? f(base + i) : 0;
  BS(tmp).ExclusiveSum(items, items);
  const int64_t off = partials[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) out[base + i] = items[i] + off;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = partials[gridDim.x];
}

// out[0..n) = exclusive scan of f, out[n] = total.  partials: scan_tiles(n)+1.
template <typename F>
int exclusive_scan(int64_t n, F f, int64_t* out, int64_t* partials, cudaStream_t s) {
  if (n == 0) {
    GLINT_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return GLINT_OK;
  }
  const int64_t nt = scan_tiles(n);
  scan_reduce_kernel<F><<<static_cast<unsigned>(nt), kScanThreads, 0, s>>>(n, f, partials);
  scan_partials_kernel<<<1, 1024, 0, s>>>(nt, partials);
  scan_apply_kernel<F><<<static_cast<unsigned>(nt), kScanThreads, 0, s>>>(n, f, partials, out);
  return launch_status("exclusive_scan");
}

struct DegreeFn {
  const int64_t* indptr;
  const int64_t* targets;
  int64_t base;
  __device__ __forceinline__ int64_t operator()(int64_t j) const {
    const int64_t t = targets ? targets[j] : base + j;
    return indptr[t + 1] - indptr[t];
  }
};

struct HubFn {  // 1 when deg + 1 >= min_degp1
  const int64_t* indptr;
  const int64_t* targets;
  int64_t base;
  int64_t min_degp1;
  __device__ __forceinline__ int64_t operator()(int64_t j) const {
    const int64_t t = targets ? targets[j] : base + j;
    return (indptr[t + 1] - indptr[t] + 1) >= min_degp1 ? 1 : 0;
  }
};

struct PopcFn {
  const uint32_t* bm;
  __device__ __forceinline__ int64_t operator()(int64_t w) const { return __popc(bm[w]); }
};

// ---------------------------------------------------------------- idset --

struct IdSet {
  uint32_t* bm;
  int64_t* prefix;    // W + 1
  int64_t* partials;  // scan_tiles(W) + 1
  int64_t words;
};

inline int64_t words_of(int64_t n) { return ceil_div(std::max<int64_t>(n, 1), 32); }

inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }

IdSet idset_view(void* ws, int64_t n) {
  IdSet s;
  s.words = words_of(n);
  char* p = static_cast<char*>(ws);
  s.bm = reinterpret_cast<uint32_t*>(p);
  p += align8(s.words * sizeof(uint32_t));
  s.prefix = reinterpret_cast<int64_t*>(p);
  p += (s.words + 1) * sizeof(int64_t);
  s.partials = reinterpret_cast<int64_t*>(p);
  return s;
}

__device__ __forceinline__ int64_t idset_rank(const uint32_t* bm, const int64_t* prefix, int64_t u) {
  const uint32_t w = bm[u >> 5];
  const uint32_t bit = 1u << (u & 31);
  if (!(w & bit)) return -1;
  return prefix[u >> 5] + __popc(w & (bit - 1u));
}

__global__ void idset_add_ids_kernel(uint32_t* bm, const int64_t* ids, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t u = ids[i];
    atomicOr(&bm[u >> 5], 1u << (u & 31));
  }
}

// Range [lo, hi): one thread per touched word.
__global__ void idset_add_range_kernel(uint32_t* bm, int64_t lo, int64_t hi) {
  const int64_t w0 = lo >> 5;
  const int64_t w1 = (hi - 1) >> 5;
  for (int64_t w = w0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w <= w1;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t wlo = w << 5;
    const int64_t b0 = (lo > wlo ? lo : wlo) - wlo;
    const int64_t b1 = (hi < wlo + 32 ? hi : wlo + 32) - wlo;  // exclusive
    const uint32_t hi_mask = b1 >= 32 ? 0xffffffffu : ((1u << b1) - 1u);
    const uint32_t lo_mask = ~((1u << b0) - 1u);
    atomicOr(&bm[w], hi_mask & lo_mask);
  }
}

// In-neighbours of a contiguous row range: the edge slice is contiguous.
// Sources inside [skip_lo, skip_hi) are already members (the targets) and
// need no atomic.
__global__ void idset_add_edges_range_kernel(uint32_t* bm, const int64_t* indptr,
                                             const int32_t* indices, int64_t row_lo,
                                             int64_t row_hi) {
  const int64_t e_lo = indptr[row_lo];
  const int64_t e_hi = indptr[row_hi];
  for (int64_t e = e_lo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < e_hi;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t u = indices[e];
    if (u >= row_lo && u < row_hi) continue;
    atomicOr(&bm[u >> 5], 1u << (u & 31));
  }
}

// In-neighbours of an explicit target list: one warp per target.
__global__ void idset_add_edges_list_kernel(uint32_t* bm, const int64_t* indptr,
                                            const int32_t* indices, const int64_t* targets,
                                            int64_t n) {
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
       j += nwarps) {
    const int64_t t = targets[j];
    for (int64_t e = indptr[t] + lane; e < indptr[t + 1]; e += 32) {
      const int64_t u = indices[e];
      atomicOr(&bm[u >> 5], 1u << (u & 31));
    }
  }
}

__global__ void idset_count_out_kernel(const int64_t* prefix, int64_t words, int64_t* count_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *count_out = prefix[words];
}

__global__ void idset_extract_kernel(const uint32_t* bm, const int64_t* prefix, int64_t words,
                                     int64_t* ids) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t bits = bm[w];
    int64_t pos = prefix[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      ids[pos++] = (w << 5) + b;
      bits &= bits - 1u;
    }
  }
}

__global__ void idset_lookup_kernel(const uint32_t* bm, const int64_t* prefix, const int64_t* ids,
                                    const int32_t* ids32, int64_t n, int64_t* pos64,
                                    int32_t* pos32) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t u = ids ? ids[i] : static_cast<int64_t>(ids32[i]);
    const int64_t r = idset_rank(bm, prefix, u);
    if (pos64) pos64[i] = r;
    if (pos32) pos32[i] = static_cast<int32_t>(r);
  }
}

__global__ void idset_rank_map_kernel(const uint32_t* bm, const int64_t* prefix, int64_t n,
                                      int32_t* map) {
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < n;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x)
    map[u] = static_cast<int32_t>(idset_rank(bm, prefix, u));
}

// ------------------------------------------------------------ slices etc --

__global__ void gather_slices_kernel(const int64_t* indptr, const int32_t* indices,
                                     const int64_t* targets, int64_t base, int64_t n,
                                     const int64_t* local_indptr, int64_t* srcs64, int32_t* srcs32,
                                     const uint32_t* bm, const int64_t* prefix, int64_t* local64,
                                     int32_t* local32) {
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
       j += nwarps) {
    const int64_t t = targets ? targets[j] : base + j;
    const int64_t sb = indptr[t];
    const int64_t len = indptr[t + 1] - sb;
    const int64_t db = local_indptr[j];
    for (int64_t k = lane; k < len; k += 32) {
      const int64_t u = indices[sb + k];
      if (srcs64) srcs64[db + k] = u;
      if (srcs32) srcs32[db + k] = static_cast<int32_t>(u);
      if (bm) {
        const int64_t r = idset_rank(bm, prefix, u);
        if (local64) local64[db + k] = r;
        if (local32) local32[db + k] = static_cast<int32_t>(r);
      }
    }
  }
}

__global__ void relabel_kernel(int64_t n, const int64_t* old_indptr, const int32_t* old_indices,
                               const int64_t* perm, const int64_t* inv, const int64_t* new_indptr,
                               int32_t* new_indices) {
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
       j += nwarps) {
    const int64_t old = perm[j];
    const int64_t sb = old_indptr[old];
    const int64_t len = old_indptr[old + 1] - sb;
    const int64_t db = new_indptr[j];
    for (int64_t k = lane; k < len; k += 32)
      new_indices[db + k] = static_cast<int32_t>(inv[old_indices[sb + k]]);
  }
}

__global__ void narrow_kernel(int64_t n, const int64_t* src, int32_t* dst, int64_t limit,
                              unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = src[i];
    if (v < 0 || v >= limit) ++local;
    dst[i] = static_cast<int32_t>(v);
  }
  if (local) atomicAdd(bad, local);
}

inline unsigned grid_for(int64_t work, int threads, int per_sm = 16) {
  const int64_t g = std::min<int64_t>(std::max<int64_t>(ceil_div(work, threads), 1),
                                      static_cast<int64_t>(sm_count()) * per_sm);
  return static_cast<unsigned>(g);
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

size_t glint_scan_workspace_bytes(int64_t n) {
  return static_cast<size_t>(scan_tiles(n) + 1) * sizeof(int64_t);
}

size_t glint_idset_workspace_bytes(int64_t num_nodes) {
  const int64_t w = words_of(num_nodes);
  return align8(w * sizeof(uint32_t)) + (w + 1) * sizeof(int64_t) +
         static_cast<size_t>(scan_tiles(w) + 1) * sizeof(int64_t);
}

int glint_idset_clear(void* ws, int64_t num_nodes, glint_stream_t stream) {
  GLINT_REQUIRE(ws && num_nodes >= 0, "idset_clear: bad argument");
  IdSet s = idset_view(ws, num_nodes);
  GLINT_CUDA(cudaMemsetAsync(s.bm, 0, s.words * sizeof(uint32_t), as_stream(stream)));
  return GLINT_OK;
}

int glint_idset_add_ids(void* ws, int64_t num_nodes, const int64_t* ids, int64_t base, int64_t n,
                        glint_stream_t stream) {
  GLINT_REQUIRE(ws && n >= 0, "idset_add_ids: bad argument");
  if (n == 0) return GLINT_OK;
  IdSet s = idset_view(ws, num_nodes);
  cudaStream_t st = as_stream(stream);
  if (ids) {
    idset_add_ids_kernel<<<grid_for(n, 256), 256, 0, st>>>(s.bm, ids, n);
  } else {
    GLINT_REQUIRE(base >= 0 && base + n <= num_nodes, "idset_add_ids: range out of bounds");
    idset_add_range_kernel<<<grid_for(ceil_div(n, 32) + 1, 256), 256, 0, st>>>(s.bm, base, base + n);
  }
  return launch_status("idset_add_ids");
}

int glint_idset_add_neighbors(void* ws, int64_t num_nodes, const int64_t* indptr,
                              const int32_t* indices, const int64_t* targets, int64_t base,
                              int64_t n, glint_stream_t stream) {
  GLINT_REQUIRE(ws && indptr && indices && n >= 0, "idset_add_neighbors: bad argument");
  if (n == 0) return GLINT_OK;
  IdSet s = idset_view(ws, num_nodes);
  cudaStream_t st = as_stream(stream);
  if (targets) {
    idset_add_edges_list_kernel<<<grid_for(n * 32, 256), 256, 0, st>>>(s.bm, indptr, indices, targets, n);
  } else {
    GLINT_REQUIRE(base >= 0 && base + n <= num_nodes, "idset_add_neighbors: range out of bounds");
    // Sources inside [base, base+n) are skipped: callers add the target range too
    // (build_batch_csc always includes the targets, kernels.py:74).
    idset_add_edges_range_kernel<<<grid_for(int64_t(1) << 30, 256), 256, 0, st>>>(
        s.bm, indptr, indices, base, base + n);
  }
  return launch_status("idset_add_neighbors");
}

int glint_idset_finalize(void* ws, int64_t num_nodes, int64_t* count_out, glint_stream_t stream) {
  GLINT_REQUIRE(ws, "idset_finalize: null workspace");
  IdSet s = idset_view(ws, num_nodes);
  cudaStream_t st = as_stream(stream);
  int rc = exclusive_scan(s.words, PopcFn{s.bm}, s.prefix, s.partials, st);
  if (rc) return rc;
  if (count_out) idset_count_out_kernel<<<1, 32, 0, st>>>(s.prefix, s.words, count_out);
  return launch_status("idset_finalize");
}

int glint_idset_extract(const void* ws, int64_t num_nodes, int64_t* ids_out, glint_stream_t stream) {
  GLINT_REQUIRE(ws && ids_out, "idset_extract: null argument");
  IdSet s = idset_view(const_cast<void*>(ws), num_nodes);
  idset_extract_kernel<<<grid_for(s.words, 256), 256, 0, as_stream(stream)>>>(s.bm, s.prefix, s.words, ids_out);
  return launch_status("idset_extract");
}

int glint_idset_lookup(const void* ws, int64_t num_nodes, const int64_t* ids, const int32_t* ids32,
                       int64_t n, int64_t* pos64, int32_t* pos32, glint_stream_t stream) {
  GLINT_REQUIRE(ws && (ids || ids32 || n == 0) && n >= 0, "idset_lookup: bad argument");
  if (n == 0) return GLINT_OK;
  IdSet s = idset_view(const_cast<void*>(ws), num_nodes);
  idset_lookup_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(s.bm, s.prefix, ids, ids32, n, pos64, pos32);
  return launch_status("idset_lookup");
}

int glint_idset_rank_map(const void* ws, int64_t num_nodes, int32_t* map_out, glint_stream_t stream) {
  GLINT_REQUIRE(ws && map_out && num_nodes < (1LL << 31), "idset_rank_map: bad argument");
  if (num_nodes == 0) return GLINT_OK;
  IdSet s = idset_view(const_cast<void*>(ws), num_nodes);
  idset_rank_map_kernel<<<grid_for(num_nodes, 256), 256, 0, as_stream(stream)>>>(s.bm, s.prefix, num_nodes, map_out);
  return launch_status("idset_rank_map");
}

int glint_degree_prefix(const int64_t* indptr, const int64_t* targets, int64_t base, int64_t n,
                        int64_t* out, void* ws, size_t ws_bytes, glint_stream_t stream) {
  GLINT_REQUIRE(indptr && out && n >= 0, "degree_prefix: bad argument");
  GLINT_REQUIRE(n == 0 || (ws && ws_bytes >= glint_scan_workspace_bytes(n)),
                "degree_prefix: workspace too small");
  return exclusive_scan(n, DegreeFn{indptr, targets, base}, out, static_cast<int64_t*>(ws),
                        as_stream(stream));
}

int glint_hub_prefix(const int64_t* indptr, const int64_t* targets, int64_t base, int64_t n,
                     int64_t min_degp1, int64_t* out, void* ws, size_t ws_bytes,
                     glint_stream_t stream) {
  GLINT_REQUIRE(indptr && out && n >= 0 && min_degp1 >= 0, "hub_prefix: bad argument");
  GLINT_REQUIRE(n == 0 || (ws && ws_bytes >= glint_scan_workspace_bytes(n)),
                "hub_prefix: workspace too small");
  return exclusive_scan(n, HubFn{indptr, targets, base, min_degp1}, out,
                        static_cast<int64_t*>(ws), as_stream(stream));
}

int glint_gather_slices(const int64_t* indptr, const int32_t* indices, const int64_t* targets,
                        int64_t base, int64_t n, const int64_t* local_indptr, int64_t* srcs64,
                        int32_t* srcs32, const void* pos_ws, int64_t num_nodes, int64_t* local64,
                        int32_t* local32, glint_stream_t stream) {
  GLINT_REQUIRE(indptr && indices && local_indptr && n >= 0, "gather_slices: bad argument");
  if (n == 0) return GLINT_OK;
  const uint32_t* bm = nullptr;
  const int64_t* prefix = nullptr;
  if (pos_ws) {
    IdSet s = idset_view(const_cast<void*>(pos_ws), num_nodes);
    bm = s.bm;
    prefix = s.prefix;
  }
  gather_slices_kernel<<<grid_for(n * 32, 256, 32), 256, 0, as_stream(stream)>>>(
      indptr, indices, targets, base, n, local_indptr, srcs64, srcs32, bm, prefix, local64, local32);
  return launch_status("gather_slices");
}

int glint_relabel_csc(int64_t num_nodes, const int64_t* old_indptr, const int32_t* old_indices,
                      const int64_t* perm, const int64_t* inv, const int64_t* new_indptr,
                      int32_t* new_indices, glint_stream_t stream) {
  GLINT_REQUIRE(num_nodes >= 0, "relabel_csc: bad argument");
  if (num_nodes == 0) return GLINT_OK;
  GLINT_REQUIRE(old_indptr && perm && inv && new_indptr, "relabel_csc: null argument");
  relabel_kernel<<<grid_for(num_nodes * 32, 256, 32), 256, 0, as_stream(stream)>>>(
      num_nodes, old_indptr, old_indices, perm, inv, new_indptr, new_indices);
  return launch_status("relabel_csc");
}

int glint_narrow_ids(int64_t n, const int64_t* src, int32_t* dst, int64_t limit, int64_t* bad_out,
                     glint_stream_t stream) {
  GLINT_REQUIRE(n >= 0 && bad_out && limit <= (1LL << 31), "narrow_ids: bad argument");
  cudaStream_t st = as_stream(stream);
  GLINT_CUDA(cudaMemsetAsync(bad_out, 0, sizeof(int64_t), st));
  if (n == 0) return GLINT_OK;
  GLINT_REQUIRE(src && dst, "narrow_ids: null argument");
  narrow_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, src, dst, limit,
                                                 reinterpret_cast<unsigned long long*>(bad_out));
  return launch_status("narrow_ids");
}

}  // extern "C"
