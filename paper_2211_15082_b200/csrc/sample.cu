// Neighbour sampling on the device (reference: executor.py:74-115
// sample_neighbors).  Every in-edge slot s of a selected node v gets the
// priority
//   prio = mix(base ^ mix(v * M1) ^ s),  base = mix(mix(seed) ^ mix(layer * M2))
// (splitmix64 finaliser, wrapping uint64 arithmetic).  The node keeps its
// min(fanout, deg) smallest priorities -- ties by slot, as numpy's stable
// lexsort -- and the kept sources are stored ascending.
//
// Device pipeline (all on the caller's stream, scratch in the caller's
// workspace):
//   1. prio_kernel: one warp per selected node writes (prio, source) for its
//      slots into the node's segment;
//   2. cub::DeviceSegmentedSort::StableSortPairs by priority per segment
//      (stable: equal priorities keep slot order);
//   3. keep_kernel: the first min(fanout, deg) sources of each segment;
//   4. cub::DeviceSegmentedSort::SortKeys per output segment (ascending ids).
#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"

namespace glint {
namespace {

constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;
constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + kGold;
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
  return z ^ (z >> 31);
}

__global__ void prio_kernel(int64_t n_sel, const int64_t* __restrict__ nodes,
                            const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int64_t* __restrict__ local_off, uint64_t base,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_sel) return;
  const int64_t v = nodes ? nodes[w] : w;
  const int64_t beg = indptr[v];
  const int64_t deg = indptr[v + 1] - beg;
  const int64_t out = local_off[w];
  const uint64_t hv = base ^ mix64(static_cast<uint64_t>(v) * kM1);
  for (int64_t s = lane; s < deg; s += 32) {
    keys[out + s] = mix64(hv ^ static_cast<uint64_t>(s));
    vals[out + s] = indices[beg + s];
  }
}

__global__ void keep_kernel(int64_t n_sel, const int64_t* __restrict__ local_off,
                            const int64_t* __restrict__ out_off, const int32_t* __restrict__ sorted,
                            int32_t* __restrict__ kept) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_sel) return;
  const int64_t src = local_off[w];
  const int64_t dst = out_off[w];
  const int64_t cnt = out_off[w + 1] - dst;
  for (int64_t j = lane; j < cnt; j += 32) kept[dst + j] = sorted[src + j];
}

// ---- fanout <= 32: one warp per node selects its fanout smallest (prio, slot)
// keys with warp bitonic sorts -- no segmented sort of every edge --
// then sorts the kept sources ascending.  Same draws and order as the sort
// pipeline below (ties by slot, as numpy's stable lexsort).
//   * A chunk of 32 slots is sorted and merged only if one of its keys beats
//     the current fanout-th smallest (a warp ballot): past the first chunk
//     most chunks of a long row are skipped outright.
//   * Keys carry (prio, slot) only -- 3 shuffles per compare-exchange; the
//     kept sources are loaded by slot at the end.
//   * The kept sources are sorted by a 32-bit id bitonic (1 shuffle per
//     step), skipped when they are ascending already (slices stored sorted).
struct Cand {
  uint64_t prio;
  uint32_t slot;
};

__device__ __forceinline__ bool less(const Cand& a, const Cand& b) {
  return a.prio < b.prio || (a.prio == b.prio && a.slot < b.slot);
}

__device__ __forceinline__ Cand shfl_xor(const Cand& c, int m) {
  Cand o;
  o.prio = __shfl_xor_sync(0xffffffffu, c.prio, m);
  o.slot = __shfl_xor_sync(0xffffffffu, c.slot, m);
  return o;
}

// compare-exchange with the lane `m` away: the lower lane keeps the smaller
// element iff `up`
__device__ __forceinline__ void cmpx(Cand& c, int lane, int m, bool up) {
  const Cand o = shfl_xor(c, m);
  const bool lower = (lane & m) == 0;
  const bool take_min = lower == up;
  const bool o_less = less(o, c);
  if (take_min ? o_less : less(c, o)) c = o;
}

__device__ __forceinline__ void bitonic_sort32(Cand& c, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int m = k >> 1; m > 0; m >>= 1) cmpx(c, lane, m, (lane & k) == 0 || k == 32);
}

// c: a bitonic sequence across the warp -> ascending
__device__ __forceinline__ void bitonic_merge32(Cand& c, int lane) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) cmpx(c, lane, m, true);
}

// ascending 32-bit ids across the warp (0x7fffffff pads the tail)
__device__ __forceinline__ void bitonic_sort32_ids(int32_t& v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int m = k >> 1; m > 0; m >>= 1) {
      const int32_t o = __shfl_xor_sync(0xffffffffu, v, m);
      const bool up = (lane & k) == 0 || k == 32;
      const bool take_min = ((lane & m) == 0) == up;
      v = take_min ? min(v, o) : max(v, o);
    }
}

// 32-bit keys for rows of at most 64 slots: the top 32 bits of the priority
// with the slot as tie-break (2 shuffles per compare-exchange).  Exact unless
// a slot outside the kept set shares the top 32 bits of the fanout-th
// smallest key -- checked by a ballot, and such a row (probability ~deg 2^-32)
// takes the 64-bit path.
struct Key32 {
  uint32_t hi;
  uint32_t slot;
};

__device__ __forceinline__ bool less32(const Key32& a, const Key32& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.slot < b.slot);
}

__device__ __forceinline__ void cmpx32(Key32& c, int lane, int m, bool up) {
  Key32 o;
  o.hi = __shfl_xor_sync(0xffffffffu, c.hi, m);
  o.slot = __shfl_xor_sync(0xffffffffu, c.slot, m);
  const bool take_min = ((lane & m) == 0) == up;
  if (take_min ? less32(o, c) : less32(c, o)) c = o;
}

__device__ __forceinline__ void bitonic_sort32_k(Key32& c, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int m = k >> 1; m > 0; m >>= 1) cmpx32(c, lane, m, (lane & k) == 0 || k == 32);
}

// the fanout smallest of a row with deg <= 64 slots; false if not exact
__device__ __forceinline__ bool select64(uint64_t hv, int64_t deg, int fanout, int lane,
                                         uint32_t* slot_out) {
  const Key32 none{0xffffffffu, 0xffffffffu};
  Key32 a = none, b = none;
  if (lane < deg) a = Key32{static_cast<uint32_t>(mix64(hv ^ static_cast<uint64_t>(lane)) >> 32),
                            static_cast<uint32_t>(lane)};
  if (lane + 32 < deg)
    b = Key32{static_cast<uint32_t>(mix64(hv ^ static_cast<uint64_t>(lane + 32)) >> 32),
              static_cast<uint32_t>(lane + 32)};
  const Key32 a0 = a, b0 = b;
  bitonic_sort32_k(a, lane);
  if (deg > 32) {
    bitonic_sort32_k(b, lane);
    Key32 r;
    r.hi = __shfl_sync(0xffffffffu, b.hi, 31 - lane);
    r.slot = __shfl_sync(0xffffffffu, b.slot, 31 - lane);
    if (less32(r, a)) a = r;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) cmpx32(a, lane, m, true);
  }
  const uint32_t t = __shfl_sync(0xffffffffu, a.hi, fanout - 1);
  const int kept = __popc(__ballot_sync(0xffffffffu, lane < fanout && a.hi == t));
  const int all = __popc(__ballot_sync(0xffffffffu, lane < deg && a0.hi == t)) +
                  __popc(__ballot_sync(0xffffffffu, lane + 32 < deg && b0.hi == t));
  *slot_out = a.slot;
  return kept == all;
}

__global__ void select_kernel(int64_t n_sel, const int64_t* __restrict__ nodes,
                              const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                              const int64_t* __restrict__ out_off, uint64_t base, int fanout,
                              int32_t* __restrict__ out) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_sel) return;
  const int64_t v = nodes ? nodes[w] : w;
  const int64_t beg = indptr[v];
  const int64_t deg = indptr[v + 1] - beg;
  const int64_t dst = out_off[w];
  const uint64_t hv = base ^ mix64(static_cast<uint64_t>(v) * kM1);
  const Cand none{~0ull, 0xffffffffu};
  const int keep = static_cast<int>(deg < fanout ? deg : fanout);
  int32_t id = 0x7fffffff;
  uint32_t slot64 = 0;
  if (deg > fanout && deg <= 64 && select64(hv, deg, fanout, lane, &slot64)) {
    if (lane < keep) id = __ldg(indices + beg + slot64);
  } else if (deg > fanout) {
    Cand best = none;
    for (int64_t c0 = 0; c0 < deg; c0 += 32) {
      const int64_t sl = c0 + lane;
      Cand c = none;
      if (sl < deg) {
        c.prio = mix64(hv ^ static_cast<uint64_t>(sl));
        c.slot = static_cast<uint32_t>(sl);
      }
      if (c0 > 0) {
        // the current fanout-th smallest: a chunk with nothing below it is skipped
        Cand kth;
        kth.prio = __shfl_sync(0xffffffffu, best.prio, fanout - 1);
        kth.slot = __shfl_sync(0xffffffffu, best.slot, fanout - 1);
        if (__ballot_sync(0xffffffffu, less(c, kth)) == 0u) continue;
      }
      bitonic_sort32(c, lane);
      // the 32 smallest of best (ascending) and c (ascending): min against the
      // reversed chunk gives a bitonic sequence holding them
      Cand r;
      r.prio = __shfl_sync(0xffffffffu, c.prio, 31 - lane);
      r.slot = __shfl_sync(0xffffffffu, c.slot, 31 - lane);
      if (less(r, best)) best = r;
      bitonic_merge32(best, lane);
    }
    if (lane < keep) id = __ldg(indices + beg + best.slot);
  } else if (lane < deg) {
    id = __ldg(indices + beg + lane);
  }
  // the kept sources (lanes < keep) ascending by id
  const int32_t prev = __shfl_up_sync(0xffffffffu, id, 1);
  if (__ballot_sync(0xffffffffu, lane > 0 && lane < keep && prev > id) != 0u)
    bitonic_sort32_ids(id, lane);
  if (lane < keep) out[dst + lane] = id;
}

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

struct SampleWs {
  size_t keys, vals, kept, temp, total;
};

int sample_ws(int64_t n_sel, int64_t e_sel, int64_t e_out, SampleWs* ws) {
  size_t t1 = 0, t2 = 0;
  GLINT_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
      nullptr, t1, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
      static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), static_cast<int>(e_sel),
      static_cast<int>(n_sel), static_cast<const int64_t*>(nullptr),
      static_cast<const int64_t*>(nullptr)));
  GLINT_CUDA(cub::DeviceSegmentedSort::SortKeys(
      nullptr, t2, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
      static_cast<int>(e_out), static_cast<int>(n_sel), static_cast<const int64_t*>(nullptr),
      static_cast<const int64_t*>(nullptr)));
  ws->keys = align256(2 * sizeof(uint64_t) * static_cast<size_t>(e_sel));
  ws->vals = align256(2 * sizeof(int32_t) * static_cast<size_t>(e_sel));
  ws->kept = align256(sizeof(int32_t) * static_cast<size_t>(e_out));
  ws->temp = align256(std::max(t1, t2));
  ws->total = ws->keys + ws->vals + ws->kept + ws->temp;
  return GLINT_OK;
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

size_t glint_sample_workspace_bytes(int64_t n_sel, int64_t e_sel, int64_t e_out) {
  if (n_sel < 0 || e_sel < 0 || e_out < 0 || e_sel >= (1LL << 31) || n_sel >= (1LL << 31))
    return 0;
  SampleWs ws{};
  if (sample_ws(n_sel, e_sel, e_out, &ws) != GLINT_OK) return 0;
  return ws.total;
}

int glint_sample_neighbors(const int64_t* indptr, const int32_t* indices, const int64_t* nodes,
                           int64_t n_sel, const int64_t* local_off, int64_t e_sel,
                           const int64_t* out_off, int64_t e_out, int32_t fanout, int64_t seed,
                           int32_t layer, int32_t* out_indices, void* workspace,
                           size_t workspace_bytes, glint_stream_t stream) {
  GLINT_REQUIRE(fanout >= 1, "sample_neighbors: fanout must be >= 1, got %d", fanout);
  GLINT_REQUIRE(n_sel >= 0 && e_sel >= 0 && e_out >= 0 && e_out <= e_sel,
                "sample_neighbors: bad sizes");
  GLINT_REQUIRE(e_sel < (1LL << 31) && n_sel < (1LL << 31),
                "sample_neighbors: more than 2^31 edges or nodes per call");
  if (n_sel == 0 || e_sel == 0) return GLINT_OK;
  GLINT_REQUIRE(indptr && indices && out_off && out_indices, "sample_neighbors: null argument");
  cudaStream_t s = as_stream(stream);
  const uint64_t base0 = mix64(mix64(static_cast<uint64_t>(seed)) ^
                               mix64(static_cast<uint64_t>(static_cast<int64_t>(layer)) * kM2));
  if (fanout <= 32 && tuning(GLINT_TUNE_SAMPLE_SORT) == 0) {   // no workspace, no local_off
    const int64_t blocks = ceil_div(n_sel * 32, 256);
    select_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n_sel, nodes, indptr, indices,
                                                               out_off, base0, fanout, out_indices);
    return launch_status("sample_select");
  }
  GLINT_REQUIRE(local_off && workspace, "sample_neighbors: null argument");
  SampleWs ws{};
  int rc = sample_ws(n_sel, e_sel, e_out, &ws);
  if (rc) return rc;
  GLINT_REQUIRE(workspace_bytes >= ws.total, "sample_neighbors: workspace too small");
  uint8_t* p = static_cast<uint8_t*>(workspace);
  uint64_t* keys_in = reinterpret_cast<uint64_t*>(p);
  uint64_t* keys_out = keys_in + e_sel;
  int32_t* vals_in = reinterpret_cast<int32_t*>(p + ws.keys);
  int32_t* vals_out = vals_in + e_sel;
  int32_t* kept = reinterpret_cast<int32_t*>(p + ws.keys + ws.vals);
  void* temp = p + ws.keys + ws.vals + ws.kept;
  const uint64_t base = base0;
  const int64_t blocks = ceil_div(n_sel * 32, 256);
  prio_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n_sel, nodes, indptr, indices,
                                                             local_off, base, keys_in, vals_in);
  rc = launch_status("sample_prio");
  if (rc) return rc;
  size_t tb = ws.temp;
  GLINT_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
      temp, tb, keys_in, keys_out, vals_in, vals_out, static_cast<int>(e_sel),
      static_cast<int>(n_sel), local_off, local_off + 1, s));
  keep_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n_sel, local_off, out_off, vals_out,
                                                             kept);
  rc = launch_status("sample_keep");
  if (rc) return rc;
  tb = ws.temp;
  GLINT_CUDA(cub::DeviceSegmentedSort::SortKeys(temp, tb, kept, out_indices,
                                                static_cast<int>(e_out), static_cast<int>(n_sel),
                                                out_off, out_off + 1, s));
  return launch_status("sample_sort");
}

}  // extern "C"
