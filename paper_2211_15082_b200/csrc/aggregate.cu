// K1 (mean SpMM) and K4 (GAT edge-softmax SpMM) neighbour aggregation.
//
// Reference semantics: kernels.py:122-135 (agg_mean) and kernels.py:170-203
// (agg_attn).  The mean must be byte-identical to numpy's np.add.at
// accumulation: every output column is ONE sequential fp32 add chain
//   0 + h[u_0] + h[u_1] + ... + h[u_{deg-1}] + h[self]
// in stored edge order, followed by an IEEE division by (float)(deg+1).
// Parallelism therefore comes only from (a) rows, (b) columns and (c) issuing
// many independent row loads ahead of the in-order adds -- never from a
// reduction tree over edges.
//
// Layout of the work:
//   * regular rows: a group of LPR lanes (8/16/32) owns one row; each lane
//     owns VPL 128-bit column chunks; U neighbour rows are loaded ahead of the
//     adds (memory-level parallelism ~ U*VPL*16 B per lane).
//   * hub rows (deg+1 >= hub_min, first n_hub entries of the degree-bucketed
//     schedule): mean_hub_kernel on a side stream, one CTA per (row,
//     64-column slice): a producer warp streams source-row slices into a
//     64 KB shared ring with cp.async.bulk (TMA), one consumer thread per
//     column adds them in stored order.  (Fallback for unaligned layouts: a
//     256-thread CTA per (row, 256 columns) inside mean_kernel with register
//     prefetch.)  Regular rows follow the hubs in descending degree-bucket
//     order (longest-processing-time-first).
#include <cub/block/block_reduce.cuh>

#include <mutex>

#include "common.cuh"

namespace glint {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kHubChunk = 1024;  // staged source offsets per hub iteration
constexpr int kHubUnroll = 32;   // loads in flight per thread on the hub path
constexpr int kMaxHeads = 8;
constexpr int LPR_MIN = 8;  // narrowest lane group of the GAT kernel

struct RowAddr {
  const int64_t* __restrict__ indptr;
  const int32_t* __restrict__ indices;
  const int64_t* __restrict__ row_ids;
  int64_t row_base;
  const int64_t* __restrict__ self_rows;
  const int32_t* __restrict__ col_map;

  __device__ __forceinline__ int64_t csr_row(int64_t r) const {
    return row_ids ? row_ids[r] : row_base + r;
  }
  // Source ids are < 2^31; bit 31 of a stored id may carry the L2 "hot source"
  // annotation (glint_hot_annotate), so every id is masked before use.
  __device__ __forceinline__ int64_t map(int64_t u) const {
    u &= 0x7fffffff;
    return col_map ? static_cast<int64_t>(col_map[u]) : u;
  }
  // 32-bit form for the hot loops (ids and mapped rows are < 2^31)
  __device__ __forceinline__ int32_t map32(int32_t u) const {
    u &= 0x7fffffff;
    return col_map ? __ldg(col_map + u) : u;
  }
  __device__ __forceinline__ int64_t self_row(int64_t r, int64_t rid) const {
    return self_rows ? self_rows[r] : map(rid);
  }
};

struct Sched {
  const int32_t* __restrict__ schedule;
  int64_t n_rows;
  int64_t n_hub;
  int hub_col_blocks;
  int64_t hub_ctas;
};

__device__ __forceinline__ int64_t shfl64(unsigned mask, int64_t v, int src, int width) {
  int lo = __shfl_sync(mask, static_cast<int>(v & 0xffffffffLL), src, width);
  int hi = __shfl_sync(mask, static_cast<int>(v >> 32), src, width);
  return (static_cast<int64_t>(hi) << 32) | static_cast<uint32_t>(lo);
}

// ------------------------------------------------------------------ mean --

struct MeanArgs {
  RowAddr ra;
  Sched sc;
  int dim;
  const float* __restrict__ h;
  int64_t ld_h;
  float* __restrict__ out;
  int64_t ld_out;
  const float* __restrict__ bias;  // optional epilogue: act(mean + bias)
  int act;
  int l2_hint;   // 0 none; 1 hot ids evict_last / others evict_first; 2 hot evict_last only;
                 // 3 all evict_first (GLINT_TUNE_L2_HINT; results never change)
};

__device__ __forceinline__ float mean_epilogue(const MeanArgs& a, float v, int col) {
  if (a.bias) v = __fadd_rn(v, __ldg(a.bias + col));
  if (a.act == GLINT_ACT_RELU) v = (v > 0.0f || v != v) ? v : 0.0f;
  if (a.act == GLINT_ACT_LEAKY_RELU) v = v >= 0.0f ? v : __fmul_rn(0.2f, v);
  return v;
}

template <int VEC>
__device__ __forceinline__ void load_vec(float (&v)[VEC], const float* p) {
  if constexpr (VEC == 4) {
    float4 t = ldg_f4(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    v[0] = __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void store_vec(float* p, const float (&v)[VEC], int valid) {
  if constexpr (VEC == 4) {
    if (valid >= 4) {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < valid) p[c] = v[c];   // static indices: v stays in registers
    }
  } else {
    p[0] = v[0];
  }
}

template <int VEC, int LPR, int VPL, int U>
__device__ __forceinline__ void mean_row_regular(const MeanArgs& a, int64_t r, int lane_g,
                                                 unsigned gmask) {
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self_off = a.ra.self_row(r, rid) * a.ld_h;
  const float degp1 = static_cast<float>(end - beg + 1);
  constexpr int TILE = LPR * VPL * VEC;

  for (int c0 = 0; c0 < a.dim; c0 += TILE) {
    float acc[VPL][VEC];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
      for (int c = 0; c < VEC; ++c) acc[k][c] = 0.0f;

    // the next chunk's source ids are loaded while the current chunk's rows
    // stream in (one dependent index latency per row instead of per chunk)
    int32_t nxt = (beg + lane_g < end) ? __ldg(a.ra.indices + beg + lane_g) : 0;
    for (int64_t e0 = beg; e0 < end; e0 += LPR) {
      const int cnt = static_cast<int>(min(static_cast<int64_t>(LPR), end - e0));
      const int32_t my = (lane_g < cnt) ? a.ra.map32(nxt) : 0;
      if (e0 + LPR + lane_g < end) nxt = __ldg(a.ra.indices + e0 + LPR + lane_g);
      for (int j = 0; j < cnt; j += U) {
        float v[U][VPL][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t off = static_cast<int64_t>(__shfl_sync(gmask, my, (j + u) & (LPR - 1), LPR)) *
                              static_cast<int32_t>(a.ld_h);
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int col = c0 + (lane_g + LPR * k) * VEC;
            if (j + u < cnt && col < a.dim) {
              load_vec<VEC>(v[u][k], a.h + off + col);
            } else {
#pragma unroll
              for (int c = 0; c < VEC; ++c) v[u][k][c] = 0.0f;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (j + u < cnt) {
#pragma unroll
            for (int k = 0; k < VPL; ++k)
#pragma unroll
              for (int c = 0; c < VEC; ++c) acc[k][c] = __fadd_rn(acc[k][c], v[u][k][c]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int col = c0 + (lane_g + LPR * k) * VEC;
      if (col < a.dim) {
        float s[VEC];
        load_vec<VEC>(s, a.h + self_off + col);
#pragma unroll
        for (int c = 0; c < VEC; ++c)
          acc[k][c] = mean_epilogue(a, __fdiv_rn(__fadd_rn(acc[k][c], s[c]), degp1),
                                    col + c < a.dim ? col + c : col);
        store_vec<VEC>(a.out + r * a.ld_out + col, acc[k], a.dim - col);
      }
    }
  }
}

__device__ __forceinline__ void mean_row_hub(const MeanArgs& a, int64_t r, int col_block,
                                             int64_t* s_off) {
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self_off = a.ra.self_row(r, rid) * a.ld_h;
  const float degp1 = static_cast<float>(end - beg + 1);
  const int col = col_block * kThreads + threadIdx.x;
  const bool active = col < a.dim;
  float acc = 0.0f;
  for (int64_t e0 = beg; e0 < end; e0 += kHubChunk) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kHubChunk), end - e0));
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kThreads)
      s_off[t] = a.ra.map(a.ra.indices[e0 + t]) * a.ld_h;
    __syncthreads();
    if (active) {
      for (int j = 0; j < cnt; j += kHubUnroll) {
        float v[kHubUnroll];
#pragma unroll
        for (int u = 0; u < kHubUnroll; ++u)
          v[u] = (j + u < cnt) ? __ldg(a.h + s_off[j + u] + col) : 0.0f;
#pragma unroll
        for (int u = 0; u < kHubUnroll; ++u)
          if (j + u < cnt) acc = __fadd_rn(acc, v[u]);
      }
    }
  }
  if (active) {
    acc = __fadd_rn(acc, __ldg(a.h + self_off + col));
    a.out[r * a.ld_out + col] = mean_epilogue(a, __fdiv_rn(acc, degp1), col);
  }
}

// Hub rows, register path: a 256-thread CTA per (hub row, 256 columns) unit.
// Persistent grid (units strided over the CTAs, longest rows first): launched
// with about one CTA per SM it runs beside the concurrent regular-row kernel
// instead of filling every SM with hub CTAs ahead of it.
__global__ void __launch_bounds__(kThreads) mean_hub_reg_kernel(MeanArgs a) {
  __shared__ int64_t s_off[kHubChunk];
  for (int64_t unit = blockIdx.x; unit < a.sc.hub_ctas; unit += gridDim.x) {
    const int64_t hub = unit / a.sc.hub_col_blocks;
    const int cb = static_cast<int>(unit % a.sc.hub_col_blocks);
    mean_row_hub(a, static_cast<int64_t>(a.sc.schedule[hub]), cb, s_off);
  }
}

// Regular rows (schedule entries n_hub..n_rows): LPR lanes per row.  Hub rows
// run in their own kernel, so this one carries no shared memory and its
// register budget is set by the regular path alone.
template <int VEC, int LPR, int VPL, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) mean_kernel(MeanArgs a) {
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  const int64_t idx = a.sc.n_hub + slot;
  if (idx >= a.sc.n_rows) return;
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  mean_row_regular<VEC, LPR, VPL, U>(a, r, lane_g, gmask);
}

// ------------------------------------------------- hub rows: bulk-copy ring --
//
// One CTA per (hub row, 256-column slice).  Warps 0-7 are consumers, one
// column per thread, adding source rows in stored edge order from a shared
// ring; warp 8 is the producer: it streams whole source-row slices into the
// ring with cp.async.bulk (the TMA engine, completion counted on an mbarrier
// per group of slots).  ~96 KB of row data stay in flight per CTA, so a
// 20K-neighbour hub row is bandwidth- rather than latency-bound, while each
// column keeps its single sequential add chain (bit-exact).
constexpr int kHubRingBytes = 64 * 1024;
constexpr int kHubGroups = 8;               // ring = 8 groups of 32 slots
constexpr int kHubSlice = 64;               // columns per hub CTA
constexpr int kHubConsumerWarps = kHubSlice / 32;
constexpr int kHubThreads = (kHubConsumerWarps + 1) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void hub_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n"
      :
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
}

// Producer warp of the hub ring kernels: streams the [c0, c0+width) slice of
// every source row of edges [beg, end) into ring groups of `spg` slots.  The
// source ids of a whole ring cycle (8 groups) are loaded one cycle ahead, so
// no dependent index load sits between two groups' copies.
//   bulk = true : one cp.async.bulk (TMA) per slot; full_bar count 1 + tx bytes.
//   bulk = false: 16-byte cp.async (LDGSTS) spread over the 32 lanes (many
//                 edges per warp instruction); each lane arrives on full_bar
//                 with cp.async.mbarrier.arrive.noinc (count 32) once its
//                 copies land.  Per-request TMA cost bounds a 20K-edge hub
//                 row in bulk mode; LDGSTS issues 8-32 slices per instruction.
__device__ __forceinline__ void hub_produce(const RowAddr& ra, int64_t beg, int64_t end,
                                            const float* base, int64_t ld, int c0, int width,
                                            int spg, int slice_floats, float* ring,
                                            uint64_t* full_bar, uint64_t* empty_bar, bool bulk) {
  const int lane = threadIdx.x & 31;
  const int64_t deg = end - beg;
  const int64_t ngroups = (deg + spg - 1) / spg;
  const int64_t ncycles = (ngroups + kHubGroups - 1) / kHubGroups;
  const int cps = (width + 3) / 4;  // 16-byte chunks per slot
  const uint32_t slice_bytes = static_cast<uint32_t>(cps * 16);
  auto load_cycle = [&](int64_t c, int64_t (&ids)[kHubGroups]) {
#pragma unroll
    for (int t = 0; t < kHubGroups; ++t) {
      const int64_t e = beg + (c * kHubGroups + t) * spg + lane;
      ids[t] = (lane < spg && e < end) ? ra.map(ra.indices[e]) : 0;
    }
  };
  int64_t cur[kHubGroups], nxt[kHubGroups];
  if (ncycles > 0) load_cycle(0, cur);
  for (int64_t c = 0; c < ncycles; ++c) {
    if (c + 1 < ncycles) load_cycle(c + 1, nxt);
#pragma unroll
    for (int t = 0; t < kHubGroups; ++t) {
      const int64_t gi = c * kHubGroups + t;
      if (gi < ngroups) {
        if (c > 0) hub_mbar_wait(&empty_bar[t], static_cast<uint32_t>(c - 1) & 1u);
        const int64_t e0 = beg + gi * spg;
        const int cnt = static_cast<int>(min(static_cast<int64_t>(spg), end - e0));
        float* grp = ring + static_cast<int64_t>(t) * spg * slice_floats;
        if (bulk) {
          if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(smem_u32(&full_bar[t])), "r"(slice_bytes * cnt) : "memory");
          }
          __syncwarp();
          if (lane < cnt) {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                ::"r"(smem_u32(grp + lane * slice_floats)), "l"(base + cur[t] * ld + c0),
                "r"(slice_bytes), "r"(smem_u32(&full_bar[t]))
                : "memory");
          }
        } else {
          const int total = cnt * cps;
          for (int q0 = 0; q0 < total; q0 += 32) {
            const int q = q0 + lane;
            const int slot = q / cps;
            const int64_t id = shfl64(0xffffffffu, cur[t], slot & 31, 32);
            if (q < total) {
              const int ch = q - slot * cps;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                           ::"r"(smem_u32(grp + slot * slice_floats + ch * 4)),
                           "l"(base + id * ld + c0 + ch * 4)
                           : "memory");
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];"
                       ::"r"(smem_u32(&full_bar[t])) : "memory");
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kHubGroups; ++t) cur[t] = nxt[t];
  }
}

template <int CW>  // consumer warps = columns per CTA / 32
__global__ void __launch_bounds__((CW + 1) * 32) mean_hub_kernel(MeanArgs a, int slots_per_group,
                                                                 int slice_floats, int col_blocks,
                                                                 bool bulk) {
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full_bar[kHubGroups];
  __shared__ __align__(8) uint64_t empty_bar[kHubGroups];
  const int cb = static_cast<int>(blockIdx.x % col_blocks);
  const int64_t r = a.sc.schedule[blockIdx.x / col_blocks];
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int c0 = cb * slice_floats;
  const int width = min(slice_floats, a.dim - c0);
  const int64_t deg = end - beg;
  const int64_t ngroups = (deg + slots_per_group - 1) / slots_per_group;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int g = 0; g < kHubGroups; ++g) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   ::"r"(smem_u32(&full_bar[g])), "r"(bulk ? 1 : 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   ::"r"(smem_u32(&empty_bar[g])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    hub_produce(a.ra, beg, end, a.h, a.ld_h, c0, width, slots_per_group, slice_floats, ring,
                full_bar, empty_bar, bulk);
    return;
  }
  // consumers: thread t owns column c0 + t
  const int col = c0 + threadIdx.x;
  const bool active = threadIdx.x < width;
  float acc = 0.0f;
  for (int64_t gi = 0; gi < ngroups; ++gi) {
    const int g = static_cast<int>(gi % kHubGroups);
    const uint32_t round = static_cast<uint32_t>(gi / kHubGroups);
    hub_mbar_wait(&full_bar[g], round & 1u);
    const int cnt = static_cast<int>(min(static_cast<int64_t>(slots_per_group),
                                         end - (beg + gi * slots_per_group)));
    const float* slot0 = ring + static_cast<int64_t>(g) * slots_per_group * slice_floats;
    if (active) {
      // batches of 8 independent shared loads ahead of the dependent add chain
      int j = 0;
      for (; j + 8 <= cnt; j += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = slot0[(j + u) * slice_floats + threadIdx.x];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
      }
      for (; j < cnt; ++j) acc = __fadd_rn(acc, slot0[j * slice_floats + threadIdx.x]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                                ::"r"(smem_u32(&empty_bar[g])) : "memory");
  }
  if (active) {
    const int64_t self_off = a.ra.self_row(r, rid) * a.ld_h;
    acc = __fadd_rn(acc, __ldg(a.h + self_off + col));
    const float degp1 = static_cast<float>(deg + 1);
    a.out[r * a.ld_out + col] = mean_epilogue(a, __fdiv_rn(acc, degp1), col);
  }
}

struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::mutex mu;   // held from the fork record to the caller's join wait
};

// Library-internal side stream (per device) for the concurrent hub kernel.
int side_stream(SideStream** out) {
  static std::mutex mu;
  static SideStream per_dev[64];
  int dev = 0;
  GLINT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  SideStream& ss = per_dev[dev & 63];
  if (!ss.stream) {
    GLINT_CUDA(cudaStreamCreateWithFlags(&ss.stream, cudaStreamNonBlocking));
    GLINT_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    GLINT_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return GLINT_OK;
}

// Fork/join of the caller's stream with the side stream.  The side stream's
// mutex is held from the fork record until the caller's stream has enqueued
// its wait on the join, so concurrent callers (threads, streams) cannot
// interleave their event records; the destructor always enqueues the join,
// so an error return after the fork never leaves the caller's stream without
// the dependency on work already queued on the side stream.
class SideFork {
 public:
  int begin(cudaStream_t caller) {
    int rc = side_stream(&ss_);
    if (rc) return rc;
    lk_ = std::unique_lock<std::mutex>(ss_->mu);
    caller_ = caller;
    GLINT_CUDA(cudaEventRecord(ss_->fork, caller));
    joined_ = false;
    GLINT_CUDA(cudaStreamWaitEvent(ss_->stream, ss_->fork, 0));
    return GLINT_OK;
  }
  cudaStream_t stream() const { return ss_->stream; }
  int join() {
    if (joined_) return GLINT_OK;
    joined_ = true;
    cudaError_t e1 = cudaEventRecord(ss_->join, ss_->stream);
    cudaError_t e2 = cudaStreamWaitEvent(caller_, ss_->join, 0);
    lk_.unlock();
    cudaError_t e = e1 != cudaSuccess ? e1 : e2;
    if (e != cudaSuccess) {
      set_error("side stream join failed: %s", cudaGetErrorString(e));
      return GLINT_ECUDA;
    }
    return GLINT_OK;
  }
  ~SideFork() { join(); }

 private:
  SideStream* ss_ = nullptr;
  cudaStream_t caller_ = nullptr;
  std::unique_lock<std::mutex> lk_;
  bool joined_ = true;
};

template <int CW>
int launch_hub_cw(const MeanArgs& a, bool bulk, cudaStream_t s) {
  // slices of <= 32*CW columns per CTA (several CTAs per hub row keep more
  // bytes in flight per row)
  constexpr int kSlice = 32 * CW;
  const int width = std::min(kSlice, a.dim);
  const int slice_floats = ((width + 3) / 4) * 4;
  const int col_blocks = static_cast<int>(ceil_div(a.dim, kSlice));
  int per_group = kHubRingBytes / (slice_floats * 4) / kHubGroups;
  per_group = std::max(1, std::min(per_group, 32));  // one producer lane per slot
  const int smem = per_group * kHubGroups * slice_floats * 4;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(mean_hub_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kHubRingBytes + 4096));
    configured.mark();
  }
  const int64_t grid = a.sc.n_hub * col_blocks;
  mean_hub_kernel<CW><<<static_cast<unsigned>(grid), (CW + 1) * 32, smem, s>>>(
      a, per_group, slice_floats, col_blocks, bulk);
  return launch_status("spmm_mean_hub");
}

// Hub ring kernel: 32-column slices with 16-byte cp.async copies (default);
// knob GLINT_TUNE_HUB_INLINE = 3: TMA bulk copies, 4: 64-column slices.
int launch_hub(const MeanArgs& a, cudaStream_t s) {
  const int knob = tuning(GLINT_TUNE_HUB_INLINE);
  if (knob == 4) return launch_hub_cw<2>(a, false, s);
  return launch_hub_cw<1>(a, knob == 3, s);
}

// ------------------------------------- regular rows: per-lane cp.async ring --
//
// Same work split as mean_row_regular (LPR lanes per row, VPL 16-byte column
// chunks per lane) but the neighbour-row loads go through a per-lane ring of
// R shared-memory slots filled with cp.async (LDGSTS): a lane keeps R-1 row
// chunks in flight without holding them in registers, and consumes them in
// stored edge order (one sequential add chain per column -- bit-exact).  The
// source ids of the next LPR edges are prefetched one index chunk ahead of the
// issue cursor, so the issue stream never waits on a dependent index load.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               ::"r"(dst), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// base + u * ld_bytes as ONE 32x32->64 multiply-add (IMAD.WIDE): the hot
// loops' source-row address (row ids < 2^31, row pitch < 2^31 bytes).
__device__ __forceinline__ const float* row_at(const char* base, int32_t u, int32_t ld_bytes) {
  const char* p;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(p) : "r"(u), "r"(ld_bytes), "l"(base));
  return reinterpret_cast<const float*>(p);
}

// MAP = false: no column map (full mode), so the per-edge id needs no lookup.
// HINT: per-edge L2 policy from the id's hot bit (MeanArgs::l2_hint).
template <int LPR, int VPL, int R, int STRIDE = kThreads, int B = 1, bool MAP = true,
          bool HINT = false>
__device__ __forceinline__ void mean_row_async(const MeanArgs& a, int64_t r, int lane_g,
                                               unsigned gmask, float4* ring, int col0 = 0) {
  // ring: this lane's slots, slot (t, k) at ring[(t * VPL + k) * STRIDE]; the
  // lane's column chunks start at col0 (hub units cover one column block)
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const float degp1 = static_cast<float>(end - beg + 1);
  const int deg = static_cast<int>(end - beg);
  bool ok[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) ok[k] = col0 + (lane_g + LPR * k) * 4 < a.dim;
  const uint32_t ring_s = smem_u32(ring);

  const char* hbase = reinterpret_cast<const char*>(a.h + col0 + lane_g * 4);
  const int32_t ldb = static_cast<int32_t>(a.ld_h * 4);
  uint64_t pol_hot = 0, pol_cold = 0;
  if constexpr (HINT) {
    pol_hot = a.l2_hint == 3 ? policy_evict_first() : policy_evict_last();
    pol_cold = a.l2_hint == 2 ? policy_evict_normal() : policy_evict_first();
  }
  // issue cursor: edge `ie`, index chunk [cb, cb+LPR) held in `cur`, next in `nxt`
  int ie = 0, cb = 0;
  int32_t cur = (lane_g < deg) ? __ldg(a.ra.indices + beg + lane_g) : 0;
  int32_t nxt = (LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + LPR + lane_g) : 0;
  auto issue = [&](int slot) {
    if (ie - cb == LPR) {
      cb += LPR;
      cur = nxt;
      nxt = (cb + LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + cb + LPR + lane_g) : 0;
    }
    const int32_t id = __shfl_sync(gmask, cur, ie - cb, LPR);
    const float* src = row_at(hbase, MAP ? a.ra.map32(id) : (id & 0x7fffffff), ldb);
    if constexpr (HINT) {
      const uint64_t pol = id < 0 ? pol_hot : pol_cold;
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (ok[k])
          cp_async16_hint(ring_s + static_cast<uint32_t>((slot * VPL + k) * STRIDE) * 16u,
                          src + LPR * 4 * k, pol);
    } else {
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (ok[k])
          cp_async16(ring_s + static_cast<uint32_t>((slot * VPL + k) * STRIDE) * 16u,
                     src + LPR * 4 * k);
    }
    ++ie;
  };

  float acc[VPL][4];
#pragma unroll
  for (int k = 0; k < VPL; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[k][c] = 0.0f;

  // Edges move in batches of B (one cp.async group each, R/B groups in
  // flight): one wait per batch, B independent shared loads ahead of the
  // in-order adds, so a lone warp (hub rows) is not bound by per-edge latency.
  constexpr int NG = R / B;
  static_assert(NG * B == R, "ring depth must be a multiple of the batch");
#pragma unroll
  for (int g = 0; g < NG; ++g) {
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (ie < deg) issue(g * B + b);
    cp_async_commit();
  }
  int base = 0;
  for (int j0 = 0; j0 < deg; j0 += B) {
    cp_async_wait<NG - 1>();
    float4 v[B][VPL];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        v[b][k] = (ok[k] && j0 + b < deg) ? ring[((base + b) * VPL + k) * STRIDE]
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (j0 + b < deg) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          acc[k][0] = __fadd_rn(acc[k][0], v[b][k].x);
          acc[k][1] = __fadd_rn(acc[k][1], v[b][k].y);
          acc[k][2] = __fadd_rn(acc[k][2], v[b][k].z);
          acc[k][3] = __fadd_rn(acc[k][3], v[b][k].w);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (ie < deg) issue(base + b);
    cp_async_commit();
    base = (base + B == R) ? 0 : base + B;
  }
  cp_async_wait<0>();
  const int64_t self_off = a.ra.self_row(r, rid) * a.ld_h;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int col = col0 + (lane_g + LPR * k) * 4;
    if (!ok[k]) continue;
    float sv[4];
    load_vec<4>(sv, a.h + self_off + col);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      acc[k][c] = mean_epilogue(a, __fdiv_rn(__fadd_rn(acc[k][c], sv[c]), degp1),
                                col + c < a.dim ? col + c : col);
    store_vec<4>(a.out + r * a.ld_out + col, acc[k], a.dim - col);
  }
}

template <int LPR, int VPL, int R, int MINB, int B = 1, bool MAP = true, bool HINT = false>
__global__ void __launch_bounds__(kThreads, MINB) mean_async_kernel(MeanArgs a) {
  extern __shared__ __align__(16) float4 ring_all[];
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  const int64_t idx = a.sc.n_hub + slot;
  if (idx >= a.sc.n_rows) return;
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  mean_row_async<LPR, VPL, R, kThreads, B, MAP, HINT>(a, r, lane_g, gmask, ring_all + threadIdx.x);
}

// Hub rows, per-lane cp.async ring: one warp per (hub row, 128-column block),
// each lane one 16-byte column chunk with kHubR row chunks in flight (a row's
// bytes in flight = 4 d kHubR, so a 20K-neighbour row streams at ~deg/kHubR
// latencies).  Persistent grid of 2 one-warp CTAs per SM walking the hub units
// in the schedule's longest-first order: hub rows never occupy more than a
// sliver of each SM, so the concurrent regular-row kernel keeps the rest.
constexpr int kHubR = 64;

__global__ void __launch_bounds__(32) mean_hub_async_kernel(MeanArgs a, int col_blocks,
                                                            int64_t units) {
  extern __shared__ __align__(16) float4 hring[];
  for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int64_t hub = unit / col_blocks;
    const int cb = static_cast<int>(unit - hub * col_blocks);
    mean_row_async<32, 1, kHubR, 32, 8>(a, static_cast<int64_t>(a.sc.schedule[hub]), threadIdx.x,
                                        0xffffffffu, hring + threadIdx.x, cb * 128);
  }
}

int launch_hub_async(const MeanArgs& a, cudaStream_t s) {
  constexpr int smem = kHubR * 32 * 16;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(mean_hub_async_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.mark();
  }
  const int col_blocks = static_cast<int>(ceil_div(a.dim, 128));
  const int64_t units = a.sc.n_hub * col_blocks;
  const int64_t grid = std::min<int64_t>(units, 2LL * sm_count());
  if (grid <= 0) return GLINT_OK;
  mean_hub_async_kernel<<<static_cast<unsigned>(grid), 32, smem, s>>>(a, col_blocks, units);
  return launch_status("spmm_mean_hub_async");
}

template <int LPR, int VPL, int R, int MINB, int B = 1>
int launch_mean_async(const MeanArgs& a, cudaStream_t s) {
  constexpr int G = 32 / LPR;
  constexpr int smem = R * VPL * kThreads * 16;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(mean_async_kernel<LPR, VPL, R, MINB, B, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    GLINT_CUDA(cudaFuncSetAttribute(mean_async_kernel<LPR, VPL, R, MINB, B, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    GLINT_CUDA(cudaFuncSetAttribute(mean_async_kernel<LPR, VPL, R, MINB, B, false, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.mark();
  }
  const int64_t grid = ceil_div(a.sc.n_rows - a.sc.n_hub, kWarps * G);
  if (grid <= 0) return GLINT_OK;
  if (grid > 0x7fffffffLL) {
    set_error("spmm_mean: grid too large");
    return GLINT_EINVAL;
  }
  if (a.ra.col_map)
    mean_async_kernel<LPR, VPL, R, MINB, B, true><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a);
  else if (a.l2_hint)
    mean_async_kernel<LPR, VPL, R, MINB, B, false, true>
        <<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a);
  else
    mean_async_kernel<LPR, VPL, R, MINB, B, false><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a);
  return launch_status("spmm_mean_async");
}

template <int VEC, int LPR, int VPL, int U, int MINB = 3>
int launch_mean(const MeanArgs& a, cudaStream_t s) {
  constexpr int G = 32 / LPR;
  const int64_t grid = ceil_div(a.sc.n_rows - a.sc.n_hub, kWarps * G);
  if (grid <= 0) return GLINT_OK;
  if (grid > 0x7fffffffLL) {
    set_error("spmm_mean: grid too large");
    return GLINT_EINVAL;
  }
  mean_kernel<VEC, LPR, VPL, U, MINB><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a);
  return launch_status("spmm_mean");
}

int dispatch_regular(const MeanArgs& a, bool vec4, cudaStream_t s);

// Hub rows run on the library side stream (fork/join with events, so the
// caller's stream order is preserved and graph capture works), concurrently
// with the regular rows on the caller's stream.  The bulk-copy ring kernel
// wins when one hub row bounds the launch (small batches, measured up to
// ~10x); on large launches the register path finishes within the regular
// rows' time and leaves shared memory to them (profiles/r01_spmm_sweep*.jsonl).
int dispatch_mean(const MeanArgs& a, bool vec4, cudaStream_t s) {
  if (a.sc.n_hub == 0) return dispatch_regular(a, vec4, s);
  // hub path: 0 auto = producer-warp ring CTAs on small launches (a hub row
  // bounds them; ~35 ns per edge per CTA), register CTAs on large ones (best
  // aggregate throughput, profiles/r01_spmm_sweep_async.jsonl); 1 register
  // CTAs, 2/3/4 ring CTAs (LDGSTS 32-col / TMA 32-col / LDGSTS 64-col),
  // 5 one-warp cp.async units (per-warp request limit: ~116 ns per edge).
  const int knob = tuning(GLINT_TUNE_HUB_INLINE);
  if (tuning(GLINT_TUNE_HUB_AFTER) == 1) {   // hub rows after the regular rows, same stream
    int rc = dispatch_regular(a, vec4, s);
    if (rc) return rc;
    if (vec4 && (knob >= 2 || (knob == 0 && a.sc.n_rows < (1 << 19)))) return launch_hub(a, s);
    mean_hub_reg_kernel<<<static_cast<unsigned>(a.sc.hub_ctas), kThreads, 0, s>>>(a);
    return launch_status("spmm_mean_hub");
  }
  SideFork fork;
  int rc = fork.begin(s);
  if (rc) return rc;
  if (vec4 && knob == 5) {
    rc = launch_hub_async(a, fork.stream());
  } else if (vec4 && (knob >= 2 || (knob == 0 && a.sc.n_rows < (1 << 19)))) {
    rc = launch_hub(a, fork.stream());
  } else {
    // CTAs per SM for the register hub kernel: knob 6 = k caps the grid at
    // k CTAs per SM (persistent); 0 (default) = one CTA per unit, measured
    // best (profiles/r01_spmm_sweep_hub.jsonl: d=48 4.06 ms vs 4.85 at 1/SM)
    const int per_sm = tuning(GLINT_TUNE_HUB_CTAS_PER_SM);
    const int64_t cap = per_sm == 0 ? a.sc.hub_ctas : static_cast<int64_t>(per_sm) * sm_count();
    const int64_t grid = std::min<int64_t>(a.sc.hub_ctas, cap);
    mean_hub_reg_kernel<<<static_cast<unsigned>(grid), kThreads, 0, fork.stream()>>>(a);
    rc = launch_status("spmm_mean_hub");
  }
  if (rc) return rc;
  rc = dispatch_regular(a, vec4, s);
  const int rj = fork.join();
  return rc ? rc : rj;
}

int dispatch_regular(const MeanArgs& a, bool vec4, cudaStream_t s) {
  // Tuning variants (glint_set_tuning(GLINT_TUNE_MEAN_VARIANT, v)) for the
  // widths of the headline workload; 0 is the default.
  // Measured on B200 (tools/sweep_kernels.py, profiles/): 4 CTAs/SM (<= 64
  // registers) beats deeper unrolling at 2-3 CTAs/SM for d=100 and d=256.
  const int variant = tuning(GLINT_TUNE_MEAN_VARIANT);
  if (vec4 && (variant == 0 || variant >= 7)) {
    // cp.async ring kernels (default); variant 0 = best measured on the
    // Products graph (profiles/r01_spmm_sweep_async.jsonl): d=48 5.5 TB/s,
    // d=100 5.8 TB/s, d=256 7.2 TB/s of algorithmic bytes.
    const int d4 = static_cast<int>(ceil_div(a.dim, 4));
    if (d4 <= 8) {
      if (variant == 7) return launch_mean_async<8, 1, 16, 3>(a, s);
      if (variant == 8) return launch_mean_async<4, 2, 8, 3>(a, s);
      return launch_mean_async<8, 1, 8, 4>(a, s);
    }
    if (d4 <= 16) {
      if (variant == 7) return launch_mean_async<16, 1, 16, 3>(a, s);
      if (variant == 8) return launch_mean_async<16, 1, 8, 4>(a, s);
      if (variant == 10) return launch_mean_async<4, 4, 6, 2>(a, s);
      if (variant == 11) return launch_mean_async<16, 1, 12, 3>(a, s);
      if (variant == 9) return launch_mean_async<8, 2, 8, 3>(a, s);
      if (variant == 13) return launch_mean_async<8, 2, 6, 4, 2>(a, s);
      if (variant == 14) return launch_mean_async<16, 1, 6, 5>(a, s);
      if (variant == 15) return launch_mean_async<4, 4, 4, 3>(a, s);
      return launch_mean_async<8, 2, 6, 4>(a, s);   // also variant 12
    }
    if (d4 <= 32) {
      if (variant == 7) return launch_mean_async<32, 1, 16, 3>(a, s);
      if (variant == 9) return launch_mean_async<16, 2, 8, 3>(a, s);
      if (variant == 10) return launch_mean_async<8, 4, 6, 2>(a, s);
      if (variant == 11) return launch_mean_async<32, 1, 12, 3>(a, s);
      if (variant == 12) return launch_mean_async<32, 1, 6, 5>(a, s);
      if (variant == 13) return launch_mean_async<32, 1, 8, 4, 2>(a, s);
      if (variant == 14) return launch_mean_async<16, 2, 6, 4>(a, s);
      if (variant == 15) return launch_mean_async<8, 4, 4, 3>(a, s);
      return launch_mean_async<32, 1, 8, 4>(a, s);   // also variant 8
    }
    if (d4 <= 64) {
      if (variant == 7) return launch_mean_async<32, 2, 8, 3>(a, s);
      if (variant == 9) return launch_mean_async<32, 2, 6, 3>(a, s);
      if (variant == 10) return launch_mean_async<32, 2, 12, 2>(a, s);
      if (variant == 11) return launch_mean_async<32, 2, 10, 2>(a, s);
      if (variant == 12) return launch_mean_async<32, 2, 3, 5>(a, s);
      if (variant == 13) return launch_mean_async<32, 2, 4, 4, 2>(a, s);
      if (variant == 14) return launch_mean_async<16, 4, 4, 3>(a, s);
      if (variant == 15) return launch_mean_async<32, 2, 5, 4>(a, s);
      return launch_mean_async<32, 2, 4, 4>(a, s);   // also variant 8
    }
    if (variant == 0 && d4 <= 128) return launch_mean_async<32, 4, 4, 2>(a, s);
  }
  if (vec4 && variant != 0) {
    const int d4 = static_cast<int>(ceil_div(a.dim, 4));
    if (d4 > 8 && d4 <= 16) {
      if (variant == 1) return launch_mean<4, 8, 2, 8, 4>(a, s);
      if (variant == 2) return launch_mean<4, 16, 1, 16, 3>(a, s);
      if (variant == 3) return launch_mean<4, 4, 4, 8, 4>(a, s);
      if (variant == 4) return launch_mean<4, 8, 2, 4, 6>(a, s);
      if (variant == 5) return launch_mean<4, 8, 2, 4, 8>(a, s);
      if (variant == 6) return launch_mean<4, 16, 1, 4, 6>(a, s);
    }
    if (d4 > 16 && d4 <= 32) {
      if (variant == 1) return launch_mean<4, 32, 1, 8, 3>(a, s);
      if (variant == 2) return launch_mean<4, 32, 1, 16, 2>(a, s);
      if (variant == 3) return launch_mean<4, 16, 2, 8, 2>(a, s);
      if (variant == 4) return launch_mean<4, 32, 1, 4, 6>(a, s);
      if (variant == 5) return launch_mean<4, 32, 1, 4, 8>(a, s);
      if (variant == 6) return launch_mean<4, 32, 1, 6, 5>(a, s);
    }
    if (d4 > 32 && d4 <= 64) {
      if (variant == 1) return launch_mean<4, 32, 2, 4, 3>(a, s);
      if (variant == 2) return launch_mean<4, 32, 2, 8, 2>(a, s);
      if (variant == 3) return launch_mean<4, 16, 4, 4, 2>(a, s);
      if (variant == 4) return launch_mean<4, 32, 2, 2, 6>(a, s);
      if (variant == 5) return launch_mean<4, 32, 2, 2, 8>(a, s);
      if (variant == 6) return launch_mean<4, 32, 2, 3, 5>(a, s);
    }
  }
  if (vec4) {
    const int d4 = static_cast<int>(ceil_div(a.dim, 4));
    // Defaults = best measured variants (profiles/r01_spmm_sweep.jsonl):
    // d=48 4102 GB/s, d=100 4898 GB/s, d=256 6430 GB/s on the Products graph.
    if (d4 <= 8) return launch_mean<4, 8, 1, 4, 6>(a, s);
    if (d4 <= 16) return launch_mean<4, 16, 1, 4, 6>(a, s);
    if (d4 <= 32) return launch_mean<4, 32, 1, 4, 8>(a, s);
    if (d4 <= 64) return launch_mean<4, 32, 2, 3, 5>(a, s);
    if (d4 <= 128) return launch_mean<4, 32, 4, 2>(a, s);
    return launch_mean<4, 32, 8, 2>(a, s);
  }
  if (a.dim <= 32) return launch_mean<1, 32, 1, 8>(a, s);
  if (a.dim <= 64) return launch_mean<1, 32, 2, 8>(a, s);
  if (a.dim <= 128) return launch_mean<1, 32, 4, 4>(a, s);
  return launch_mean<1, 32, 8, 2>(a, s);
}

// ------------------------------------------------------- degree schedule --

__global__ void sched_hist_kernel(int64_t n, RowAddr ra, unsigned long long* hist) {
  __shared__ unsigned int sh[64];
  if (threadIdx.x < 64) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rid = ra.csr_row(r);
    const unsigned long long degp1 =
        static_cast<unsigned long long>(ra.indptr[rid + 1] - ra.indptr[rid] + 1);
    atomicAdd(&sh[63 - __clzll(degp1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 64 && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

__global__ void sched_offsets_kernel(const unsigned long long* hist, unsigned long long* offs,
                                     int hub_log2, int64_t* n_hub_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long run = 0, hubs = 0;
  for (int k = 63; k >= 0; --k) {
    offs[k] = run;
    run += hist[k];
    if (hub_log2 >= 0 && k >= hub_log2) hubs += hist[k];
  }
  *n_hub_out = static_cast<int64_t>(hubs);
}

__global__ void sched_scatter_kernel(int64_t n, RowAddr ra, unsigned long long* offs,
                                     int32_t* schedule) {
  __shared__ unsigned int cnt[64];
  __shared__ unsigned long long base[64];
  for (int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x); t0 < n;
       t0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t r = t0 + threadIdx.x;
    int k = -1;
    unsigned int local = 0;
    if (r < n) {
      const int64_t rid = ra.csr_row(r);
      const unsigned long long degp1 =
          static_cast<unsigned long long>(ra.indptr[rid + 1] - ra.indptr[rid] + 1);
      k = 63 - __clzll(degp1);
      local = atomicAdd(&cnt[k], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 64 && cnt[threadIdx.x])
      base[threadIdx.x] = atomicAdd(&offs[threadIdx.x], static_cast<unsigned long long>(cnt[threadIdx.x]));
    __syncthreads();
    if (k >= 0) schedule[base[k] + local] = static_cast<int32_t>(r);
    __syncthreads();
  }
}

// ------------------------------------------------------------------- GAT --

struct GatArgs {
  RowAddr ra;
  Sched sc;
  int heads;
  int head_dim;
  int head_pitch;  // Z columns per head (multiple of 4)
  const float* __restrict__ Z;
  int64_t ldz;
  const float* __restrict__ s_src;
  const float* __restrict__ s_dst;
  float slope;
  float* __restrict__ out;
  int64_t ld_out;
  int act;
  // two-phase path (glint_gat_aggregate_ws_f32): per-edge softmax weights
  // W[(edge - w_base) * heads + h] and per-row self weights wself[r * heads + h]
  float* __restrict__ w;
  float* __restrict__ wself;
  int64_t w_base;
  int l2_hint;   // source scores evict_last, Z rows evict_first (GLINT_TUNE_GAT_L2 = 1: off)
  int z_first;   // ring prologue before the peak pass (GLINT_TUNE_GAT_PEAK_FIRST = 1: after)
};

__device__ __forceinline__ float gat_epilogue(const GatArgs& a, float v) {
  if (a.act == GLINT_ACT_RELU) v = (v > 0.0f || v != v) ? v : 0.0f;
  if (a.act == GLINT_ACT_LEAKY_RELU) v = v >= 0.0f ? v : __fmul_rn(0.2f, v);
  return v;
}

__device__ __forceinline__ float leaky(float x, float slope) {
  return x >= 0.0f ? x : __fmul_rn(slope, x);
}

// Regular GAT row: a group of LPR lanes owns one row; lane g covers the
// 128-bit chunks g, g+LPR, ... of the head-padded Z row.  H (heads) is a
// compile-time constant so per-head state stays in registers.
//   pass 1: per-head peak over self + edges (lanes over edges, order-free max);
//   pass 2: per chunk of LPR edges, lane i computes the H softmax weights of
//           edge i once into shared memory (w_s[i][h]), then every lane walks
//           the chunk in stored edge order with U neighbour-row loads in
//           flight: den += w; num += w*z (mul then add, as numpy), self last.
template <int H, int LPR, int VPL, int U>
__device__ __forceinline__ void gat_row_regular(const GatArgs& a, int64_t r, int lane_g,
                                                unsigned gmask, float* w_s, float* st) {
  // st: per-group scratch, st[h] = s_dst[self][h], st[H + h] = peak[h]
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  {
    float sdst[H], peak[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      sdst[h] = __ldg(a.s_dst + self * H + h);
      peak[h] = leaky(__fadd_rn(__ldg(a.s_src + self * H + h), sdst[h]), a.slope);
    }
    for (int64_t e = beg + lane_g; e < end; e += LPR) {
      const int64_t u = a.ra.map(a.ra.indices[e]);
#pragma unroll
      for (int h = 0; h < H; ++h)
        peak[h] = fmaxf(peak[h], leaky(__fadd_rn(__ldg(a.s_src + u * H + h), sdst[h]), a.slope));
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1)
        peak[h] = fmaxf(peak[h], __shfl_xor_sync(gmask, peak[h], o, LPR));
    }
    if (lane_g == 0) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        st[h] = sdst[h];
        st[H + h] = peak[h];
      }
    }
    __syncwarp(gmask);
  }

  float num[VPL][4], den[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    den[k] = 0.0f;
#pragma unroll
    for (int c = 0; c < 4; ++c) num[k][c] = 0.0f;
  }
  const int head0 = (lane_g * 4) / a.head_pitch;  // head of chunk k is (zc_k / head_pitch)

  for (int64_t e0 = beg; e0 < end; e0 += LPR) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(LPR), end - e0));
    int32_t my = 0;   // source row id (ids and rows < 2^31): one shuffle per edge
    if (lane_g < cnt) {
      const int32_t u = a.ra.map32(a.ra.indices[e0 + lane_g]);
      my = u;
#pragma unroll
      for (int h = 0; h < H; ++h)
        w_s[lane_g * H + h] = expf(__fsub_rn(
            leaky(__fadd_rn(__ldg(a.s_src + static_cast<int64_t>(u) * H + h), st[h]), a.slope),
            st[H + h]));
    }
    __syncwarp(gmask);
    for (int j = 0; j < cnt; j += U) {
      float4 v[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t off = static_cast<int64_t>(__shfl_sync(gmask, my, (j + u) & (LPR - 1), LPR)) *
                            static_cast<int32_t>(a.ldz);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const int zc = (lane_g + LPR * k) * 4;
          v[u][k] = (j + u < cnt && zc < H * a.head_pitch) ? ldg_f4(a.Z + off + zc)
                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j + u < cnt) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int hk = ((lane_g + LPR * k) * 4) / a.head_pitch;
            const float w = w_s[(j + u) * H + (hk < H ? hk : 0)];
            den[k] = __fadd_rn(den[k], w);
            num[k][0] = __fadd_rn(num[k][0], __fmul_rn(w, v[u][k].x));
            num[k][1] = __fadd_rn(num[k][1], __fmul_rn(w, v[u][k].y));
            num[k][2] = __fadd_rn(num[k][2], __fmul_rn(w, v[u][k].z));
            num[k][3] = __fadd_rn(num[k][3], __fmul_rn(w, v[u][k].w));
          }
        }
      }
    }
    __syncwarp(gmask);
  }
  (void)head0;
  // self term last, then normalise and write the unpadded head columns
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int zc = (lane_g + LPR * k) * 4;
    const int hh = zc / a.head_pitch;
    if (hh >= H) continue;
    const int jc = zc - hh * a.head_pitch;
    const float4 zs = ldg_f4(a.Z + self * a.ldz + zc);
    const float ws = expf(__fsub_rn(
        leaky(__fadd_rn(__ldg(a.s_src + self * H + hh), st[hh]), a.slope), st[H + hh]));
    const float d = __fadd_rn(den[k], ws);
    const float zv[4] = {zs.x, zs.y, zs.z, zs.w};
    float* dst = a.out + r * a.ld_out + hh * a.head_dim + jc;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (jc + c < a.head_dim)
        dst[c] = gat_epilogue(a, __fdiv_rn(__fadd_rn(num[k][c], __fmul_rn(ws, zv[c])), d));
  }
}

// Hub GAT row: a CTA owns (row, 256-column block of padded Z); one column per
// thread; per chunk the CTA computes source offsets and softmax weights into
// shared memory, then each thread walks the chunk in edge order.
constexpr int kGatHubChunk = 256;

__device__ __forceinline__ void gat_row_hub(const GatArgs& a, int64_t r, int col_block,
                                            int64_t* s_off, float (*s_w)[kMaxHeads],
                                            float* s_peak) {
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  const int H = a.heads;
  using BlockReduce = cub::BlockReduce<float, kThreads>;
  __shared__ typename BlockReduce::TempStorage tmp;

  // peak per head: block-wide max over self and all edges
  for (int h = 0; h < H; ++h) {
    const float sd = a.s_dst[self * H + h];
    float m = leaky(__fadd_rn(a.s_src[self * H + h], sd), a.slope);
    for (int64_t e = beg + threadIdx.x; e < end; e += kThreads) {
      const int64_t u = a.ra.map(a.ra.indices[e]);
      m = fmaxf(m, leaky(__fadd_rn(a.s_src[u * H + h], sd), a.slope));
    }
    const float bm = BlockReduce(tmp).Reduce(m, [](float x, float y) { return fmaxf(x, y); });
    if (threadIdx.x == 0) s_peak[h] = bm;
    __syncthreads();
  }
  const int zc = col_block * kThreads + threadIdx.x;
  const int hh = zc / a.head_pitch;
  const int j = zc - hh * a.head_pitch;
  const bool active = hh < H && j < a.head_dim;
  const int hs = active ? hh : 0;
  const float sd_h = a.s_dst[self * H + hs];
  float num = 0.0f, den = 0.0f;
  for (int64_t e0 = beg; e0 < end; e0 += kGatHubChunk) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kGatHubChunk), end - e0));
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kThreads) {
      const int64_t u = a.ra.map(a.ra.indices[e0 + t]);
      s_off[t] = u * a.ldz;
      for (int h = 0; h < H; ++h) {
        const float sd = a.s_dst[self * H + h];
        s_w[t][h] = expf(__fsub_rn(leaky(__fadd_rn(a.s_src[u * H + h], sd), a.slope), s_peak[h]));
      }
    }
    __syncthreads();
    if (active) {
      for (int jj = 0; jj < cnt; jj += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (jj + u < cnt) ? __ldg(a.Z + s_off[jj + u] + zc) : 0.0f;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (jj + u < cnt) {
            const float w = s_w[jj + u][hs];
            den = __fadd_rn(den, w);
            num = __fadd_rn(num, __fmul_rn(w, v[u]));
          }
        }
      }
    }
  }
  (void)sd_h;
  if (active) {
    const float ws = expf(__fsub_rn(leaky(__fadd_rn(a.s_src[self * H + hs], a.s_dst[self * H + hs]), a.slope),
                                    s_peak[hs]));
    const float d = __fadd_rn(den, ws);
    const float n = __fadd_rn(num, __fmul_rn(ws, __ldg(a.Z + self * a.ldz + zc)));
    a.out[r * a.ld_out + hh * a.head_dim + j] = gat_epilogue(a, __fdiv_rn(n, d));
  }
}

// H per-head scores of one node (s_src / s_dst rows are H floats): one vector
// load when the table is aligned for it (vec, warp-uniform).
template <int H>
struct Scores {
  float v[H];
};

template <int H>
__device__ __forceinline__ Scores<H> load_scores(const float* __restrict__ p, bool vec) {
  Scores<H> s;
  if (H == 4 && vec) {
    const float4 t = ldg_f4(p);
    s.v[0] = t.x; s.v[1] = t.y; s.v[2 % H] = t.z; s.v[3 % H] = t.w;
  } else if (H == 2 && vec) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    s.v[0] = t.x; s.v[1 % H] = t.y;
  } else {
#pragma unroll
    for (int h = 0; h < H; ++h) s.v[h] = __ldg(p + h);
  }
  return s;
}

// Regular GAT row through a per-lane cp.async ring (as mean_row_async) -- the
// Z bytes stream continuously with R-1 edges in flight, while the softmax
// weights are computed once per edge and head, a chunk of LPR edges at a time:
//   pass 1: per-head peak over self + edges (order-free max, vector score loads);
//   pass 2: lane g owns the 16-byte Z chunks g, g+LPR, ... and issues them for
//           edge ie into ring slot (ie % R).  When the issue cursor enters edge
//           chunk c, lane i loads the H source scores of edge c*LPR+i into
//           registers; R edges later, when consumption enters chunk c, it
//           turns them into the chunk's weights wbuf[i][h] (the expression of
//           gat_row_regular) -- R <= LPR keeps one chunk of weights live.
// Accumulation: den += w; num += w*z in stored edge order, self last, so the
// bytes equal gat_row_regular's.
// H = 4 source scores (16 bytes) with an L2 policy: per edge the kernel reads
// 16 B of s_src at a random node but DRAM moves 64 B, so keeping the 39 MB
// score table resident in L2 (evict_last, with the streamed Z rows
// evict_first) removes most of that per-edge overfetch.
__device__ __forceinline__ float4 ldg_f4_pol(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}

template <int H>
__device__ __forceinline__ Scores<H> load_scores_hint(const float* __restrict__ p, bool vec,
                                                      bool hint, uint64_t pol) {
  if constexpr (H == 4) {
    if (vec && hint) {
      const float4 t = ldg_f4_pol(p, pol);
      Scores<H> s;
      s.v[0] = t.x; s.v[1] = t.y; s.v[2] = t.z; s.v[3] = t.w;
      return s;
    }
  }
  return load_scores<H>(p, vec);
}

template <int H, int LPR, int VPL, int R>
__device__ __forceinline__ void gat_row_async(const GatArgs& a, int64_t r, int lane_g,
                                              unsigned gmask, float4* zring, float* wbuf) {
  static_assert(R <= LPR, "one chunk of weights is live at a time");
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  const int deg = static_cast<int>(end - beg);
  const bool vec = (reinterpret_cast<uintptr_t>(a.s_src) % (4 * H) == 0) &&
                   (reinterpret_cast<uintptr_t>(a.s_dst) % (4 * H) == 0);
  const bool hint = a.l2_hint != 0;
  uint64_t pol_keep = 0, pol_stream = 0;
  if (hint) {
    pol_keep = policy_evict_last();
    pol_stream = policy_evict_first();
  }

  float sdst[H], peak[H];
  // pass 1 (per-head peak); run before or after the ring prologue (a.z_first):
  // the prologue's Z rows do not depend on it, so issuing them first overlaps
  // their latency with the peak pass's dependent score loads
  auto peak_pass = [&]() {
    const Scores<H> sd = load_scores<H>(a.s_dst + self * H, vec);
    const Scores<H> ss = load_scores<H>(a.s_src + self * H, vec);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      sdst[h] = sd.v[h];
      peak[h] = leaky(__fadd_rn(ss.v[h], sdst[h]), a.slope);
    }
    for (int e = lane_g; e < deg; e += 2 * LPR) {
      const bool two = e + LPR < deg;
      const int32_t u0 = a.ra.map32(__ldg(a.ra.indices + beg + e));
      const int32_t u1 = two ? a.ra.map32(__ldg(a.ra.indices + beg + e + LPR)) : u0;
      const Scores<H> s0 = load_scores_hint<H>(a.s_src + static_cast<int64_t>(u0) * H, vec, hint,
                                               pol_keep);
      const Scores<H> s1 = load_scores_hint<H>(a.s_src + static_cast<int64_t>(u1) * H, vec, hint,
                                               pol_keep);
#pragma unroll
      for (int h = 0; h < H; ++h) {
        peak[h] = fmaxf(peak[h], leaky(__fadd_rn(s0.v[h], sdst[h]), a.slope));
        peak[h] = fmaxf(peak[h], leaky(__fadd_rn(s1.v[h], sdst[h]), a.slope));
      }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1)
        peak[h] = fmaxf(peak[h], __shfl_xor_sync(gmask, peak[h], o, LPR));
    }
  };
  if (!a.z_first) peak_pass();
  bool ok[VPL];
  int hk[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int zc = (lane_g + LPR * k) * 4;
    ok[k] = zc < H * a.head_pitch;
    hk[k] = ok[k] ? zc / a.head_pitch : 0;
  }

  const uint32_t zr = smem_u32(zring);
  const char* zbase = reinterpret_cast<const char*>(a.Z + lane_g * 4);
  const int32_t ldzb = static_cast<int32_t>(a.ldz * 4);
  int ie = 0, cb = 0;
  // ucur: the mapped source row of this lane's edge in chunk cb, with the
  // stored id's bit 31 ("hot" row, kernels.hot_indices) carried along
  auto mapped = [&](int32_t raw) {
    return a.ra.map32(raw) | static_cast<int32_t>(static_cast<uint32_t>(raw) & 0x80000000u);
  };
  int32_t ucur = (lane_g < deg) ? mapped(__ldg(a.ra.indices + beg + lane_g)) : 0;
  int32_t nxt = (LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + LPR + lane_g) : 0;
  Scores<H> sc;                                     // scores of this lane's edge in chunk cb
  if (lane_g < deg)
    sc = load_scores_hint<H>(a.s_src + static_cast<int64_t>(ucur & 0x7fffffff) * H, vec, hint,
                             pol_keep);
  auto issue = [&](int slot) {
    if (ie - cb == LPR) {
      cb += LPR;
      ucur = mapped(nxt);
      nxt = (cb + LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + cb + LPR + lane_g) : 0;
      if (cb + lane_g < deg)
        sc = load_scores_hint<H>(a.s_src + static_cast<int64_t>(ucur & 0x7fffffff) * H, vec,
                                 hint, pol_keep);
    }
    const int32_t uh = __shfl_sync(gmask, ucur, ie - cb, LPR);
    const float* zsrc = row_at(zbase, uh & 0x7fffffff, ldzb);
    const uint64_t pol = uh < 0 ? pol_keep : pol_stream;   // hot Z rows stay in L2
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (ok[k]) {
        const uint32_t o = static_cast<uint32_t>((slot * VPL + k) * kThreads);
        if (hint)
          cp_async16_hint(zr + o * 16u, zsrc + LPR * 4 * k, pol);
        else
          cp_async16(zr + o * 16u, zsrc + LPR * 4 * k);
      }
    }
    ++ie;
  };

  float num[VPL][4], den[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    den[k] = 0.0f;
#pragma unroll
    for (int c = 0; c < 4; ++c) num[k][c] = 0.0f;
  }
#pragma unroll
  for (int t = 0; t < R; ++t) {
    if (ie < deg) issue(t);
    cp_async_commit();
  }
  if (a.z_first) peak_pass();
  int slot = 0, jc = 0;
  for (int j = 0; j < deg; ++j) {
    if (jc == 0) {   // consumption enters a chunk: its weights from the staged scores
      __syncwarp(gmask);   // every lane is done with the previous chunk's weights
      if (j + lane_g < deg) {
#pragma unroll
        for (int h = 0; h < H; ++h)
          wbuf[lane_g * H + h] =
              expf(__fsub_rn(leaky(__fadd_rn(sc.v[h], sdst[h]), a.slope), peak[h]));
      }
      __syncwarp(gmask);   // the chunk's weights are visible
    }
    cp_async_wait<R - 1>();   // this lane's ring slot landed (slots are per lane)
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (ok[k]) {
        const float4 v = zring[(slot * VPL + k) * kThreads];
        const float w = wbuf[jc * H + hk[k]];
        den[k] = __fadd_rn(den[k], w);
        num[k][0] = __fadd_rn(num[k][0], __fmul_rn(w, v.x));
        num[k][1] = __fadd_rn(num[k][1], __fmul_rn(w, v.y));
        num[k][2] = __fadd_rn(num[k][2], __fmul_rn(w, v.z));
        num[k][3] = __fadd_rn(num[k][3], __fmul_rn(w, v.w));
      }
    }
    if (ie < deg) issue(slot);
    cp_async_commit();
    slot = (slot + 1 == R) ? 0 : slot + 1;
    jc = (jc + 1 == LPR) ? 0 : jc + 1;
  }
  cp_async_wait<0>();
  {   // self weights (one per head) through the chunk-weight buffer
    const Scores<H> ssf = load_scores<H>(a.s_src + self * H, vec);
    __syncwarp(gmask);
#pragma unroll
    for (int h = 0; h < H; ++h)
      if (lane_g == h) wbuf[h] = expf(__fsub_rn(leaky(__fadd_rn(ssf.v[h], sdst[h]), a.slope), peak[h]));
    __syncwarp(gmask);
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    if (!ok[k]) continue;
    const int zc = (lane_g + LPR * k) * 4;
    const int hh = hk[k];
    const int jcol = zc - hh * a.head_pitch;
    const float4 zs = ldg_f4(a.Z + self * a.ldz + zc);
    const float ws = wbuf[hh];
    const float d = __fadd_rn(den[k], ws);
    const float zv[4] = {zs.x, zs.y, zs.z, zs.w};
    float* dst = a.out + r * a.ld_out + hh * a.head_dim + jcol;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (jcol + c < a.head_dim)
        dst[c] = gat_epilogue(a, __fdiv_rn(__fadd_rn(num[k][c], __fmul_rn(ws, zv[c])), d));
  }
}

template <int H, int LPR, int VPL, int R, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) gat_async_kernel(GatArgs a) {
  extern __shared__ __align__(16) float4 gring[];
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  const int64_t idx = a.sc.n_hub + slot;
  if (idx >= a.sc.n_rows) return;
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  float* wbuf = reinterpret_cast<float*>(gring + R * VPL * kThreads) + (warp * 32 + group * LPR) * H;
  gat_row_async<H, LPR, VPL, R>(a, r, lane_g, gmask, gring + threadIdx.x, wbuf);
}

// ------------------------------------------------ two-phase GAT (SDDMM + SpMM) --
//
// Phase A, gat_softmax_kernel (edge softmax / SDDMM): LPR lanes per regular
// row compute the per-head peak over self + edges, then every edge's H
// weights w = exp(LeakyReLU(s_src[u] + s_dst[v]) - peak) -- lanes over edges,
// stores coalesced along the row's edge range -- and the self weights.
// Phase B, gat_spmm_async (weighted SpMM): the K1 ring machinery with each
// lane also streaming its head's weight (4 bytes per edge, contiguous per
// row); den += w, num += w z in stored edge order, self last.  Weights and
// accumulation order are those of gat_row_regular, so the bytes match.
template <int H, int LPR>
__global__ void __launch_bounds__(kThreads) gat_softmax_kernel(GatArgs a) {
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t idx = a.sc.n_hub + static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  if (idx >= a.sc.n_rows) return;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  float sdst[H], peak[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    sdst[h] = __ldg(a.s_dst + self * H + h);
    peak[h] = leaky(__fadd_rn(__ldg(a.s_src + self * H + h), sdst[h]), a.slope);
  }
  for (int64_t e = beg + lane_g; e < end; e += LPR) {
    const int64_t u = a.ra.map(a.ra.indices[e]);
#pragma unroll
    for (int h = 0; h < H; ++h)
      peak[h] = fmaxf(peak[h], leaky(__fadd_rn(__ldg(a.s_src + u * H + h), sdst[h]), a.slope));
  }
#pragma unroll
  for (int h = 0; h < H; ++h) {
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1)
      peak[h] = fmaxf(peak[h], __shfl_xor_sync(gmask, peak[h], o, LPR));
  }
  for (int64_t e = beg + lane_g; e < end; e += LPR) {
    const int64_t u = a.ra.map(a.ra.indices[e]);
    float* wp = a.w + (e - a.w_base) * H;
#pragma unroll
    for (int h = 0; h < H; ++h)
      wp[h] = expf(__fsub_rn(leaky(__fadd_rn(__ldg(a.s_src + u * H + h), sdst[h]), a.slope), peak[h]));
  }
  if (lane_g == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h)
      a.wself[r * H + h] =
          expf(__fsub_rn(leaky(__fadd_rn(__ldg(a.s_src + self * H + h), sdst[h]), a.slope), peak[h]));
  }
}

template <int H, int LPR, int VPL, int R>
__device__ __forceinline__ void gat_spmm_row_async(const GatArgs& a, int64_t r, int lane_g,
                                                   unsigned gmask, float4* zring, float* /*unused*/) {
  // Z rows through the per-lane cp.async ring (as K1); the weights of the
  // consume cursor's LPR-edge chunk sit in registers (lane i holds edge i's H
  // weights, the next chunk prefetched) and reach every lane by H shuffles.
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  const int deg = static_cast<int>(end - beg);
  bool ok[VPL];
  int hk[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int zc = (lane_g + LPR * k) * 4;
    ok[k] = zc < H * a.head_pitch;
    hk[k] = ok[k] ? zc / a.head_pitch : 0;
  }
  const uint32_t zr = smem_u32(zring);
  const float* wrow = a.w + (beg - a.w_base) * H;
  auto load_w = [&](int c0, float (&wv)[H]) {
#pragma unroll
    for (int h = 0; h < H; ++h)
      wv[h] = (c0 + lane_g < deg) ? __ldg(wrow + static_cast<int64_t>(c0 + lane_g) * H + h) : 0.0f;
  };
  float wcur[H], wnxt[H];
  load_w(0, wcur);
  load_w(LPR, wnxt);
  int ie = 0, cb = 0;
  int32_t cur = (lane_g < deg) ? __ldg(a.ra.indices + beg + lane_g) : 0;
  int32_t nxt = (LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + LPR + lane_g) : 0;
  auto issue = [&](int slot) {
    if (ie - cb == LPR) {
      cb += LPR;
      cur = nxt;
      nxt = (cb + LPR + lane_g < deg) ? __ldg(a.ra.indices + beg + cb + LPR + lane_g) : 0;
    }
    const int64_t u = a.ra.map(__shfl_sync(gmask, cur, ie - cb, LPR));
    const float* zsrc = a.Z + u * a.ldz + lane_g * 4;
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      if (ok[k])
        cp_async16(zr + static_cast<uint32_t>((slot * VPL + k) * kThreads) * 16u, zsrc + LPR * 4 * k);
    ++ie;
  };
  float num[VPL][4], den[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    den[k] = 0.0f;
#pragma unroll
    for (int c = 0; c < 4; ++c) num[k][c] = 0.0f;
  }
#pragma unroll
  for (int t = 0; t < R; ++t) {
    if (ie < deg) issue(t);
    cp_async_commit();
  }
  int slot = 0, wc = 0;   // wc: consume cursor's position inside its weight chunk
  for (int j = 0; j < deg; ++j) {
    if (wc == LPR) {
      wc = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) wcur[h] = wnxt[h];
      load_w(j + LPR, wnxt);
    }
    float we[H];
#pragma unroll
    for (int h = 0; h < H; ++h) we[h] = __shfl_sync(gmask, wcur[h], wc, LPR);
    ++wc;
    cp_async_wait<R - 1>();
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (ok[k]) {
        float w = we[0];
#pragma unroll
        for (int h = 1; h < H; ++h)
          if (h == hk[k]) w = we[h];
        const float4 v = zring[(slot * VPL + k) * kThreads];
        den[k] = __fadd_rn(den[k], w);
        num[k][0] = __fadd_rn(num[k][0], __fmul_rn(w, v.x));
        num[k][1] = __fadd_rn(num[k][1], __fmul_rn(w, v.y));
        num[k][2] = __fadd_rn(num[k][2], __fmul_rn(w, v.z));
        num[k][3] = __fadd_rn(num[k][3], __fmul_rn(w, v.w));
      }
    }
    if (ie < deg) issue(slot);
    cp_async_commit();
    slot = (slot + 1 == R) ? 0 : slot + 1;
  }
  cp_async_wait<0>();
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    if (!ok[k]) continue;
    const int zc = (lane_g + LPR * k) * 4;
    const int hh = hk[k];
    const int jc = zc - hh * a.head_pitch;
    const float4 zs = ldg_f4(a.Z + self * a.ldz + zc);
    const float ws = a.wself[r * H + hh];
    const float d = __fadd_rn(den[k], ws);
    const float zv[4] = {zs.x, zs.y, zs.z, zs.w};
    float* dst = a.out + r * a.ld_out + hh * a.head_dim + jc;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (jc + c < a.head_dim)
        dst[c] = gat_epilogue(a, __fdiv_rn(__fadd_rn(num[k][c], __fmul_rn(ws, zv[c])), d));
  }
}

template <int H, int LPR, int VPL, int R, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) gat_spmm_async_kernel(GatArgs a) {
  extern __shared__ __align__(16) float4 gring2[];
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t idx = a.sc.n_hub + static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  if (idx >= a.sc.n_rows) return;
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  gat_spmm_row_async<H, LPR, VPL, R>(a, r, lane_g, gmask, gring2 + threadIdx.x, nullptr);
}

// Hub rows (first n_hub schedule entries): one CTA per (row, 256-column block).
__global__ void __launch_bounds__(kThreads) gat_hub_kernel(GatArgs a) {
  __shared__ int64_t s_off[kGatHubChunk];
  __shared__ float s_w[kGatHubChunk][kMaxHeads];
  __shared__ float s_peak[kMaxHeads];
  const int64_t hub = blockIdx.x / a.sc.hub_col_blocks;
  const int cb = static_cast<int>(blockIdx.x % a.sc.hub_col_blocks);
  gat_row_hub(a, static_cast<int64_t>(a.sc.schedule[hub]), cb, s_off, s_w, s_peak);
}

// Hub rows, bulk-copy ring (as mean_hub_kernel): one CTA per (hub row,
// 64-column slice of the padded Z row).  Warp 2 streams the slice of every
// source row into a 64 KB shared ring with cp.async.bulk; warps 0-1 (one
// column per thread) first reduce the per-head peak over self + all edges,
// then, per chunk of kGatWChunk edges, compute the chunk's softmax weights
// into shared memory (consumer-only named barrier) and walk the ring in
// stored edge order: den += w, num += w*z, self last -- the same arithmetic
// and order as gat_row_regular.
constexpr int kGatWChunk = 2048;
template <int CW>   // consumer warps (columns per CTA / 32)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
}

template <int CW>
__global__ void __launch_bounds__((CW + 1) * 32) gat_hub_ring_kernel(GatArgs a, int slots_per_group,
                                                                   int slice_floats,
                                                                   int col_blocks, bool bulk) {
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full_bar[kHubGroups];
  __shared__ __align__(8) uint64_t empty_bar[kHubGroups];
  __shared__ float s_sd[kMaxHeads], s_pk[kMaxHeads];
  __shared__ float s_red[CW][kMaxHeads];
  const int H = a.heads;
  float* w_sm = ring + kHubGroups * slots_per_group * slice_floats;  // [kGatWChunk][H]
  const int cb = static_cast<int>(blockIdx.x % col_blocks);
  const int64_t r = a.sc.schedule[blockIdx.x / col_blocks];
  const int64_t rid = a.ra.csr_row(r);
  const int64_t beg = a.ra.indptr[rid];
  const int64_t end = a.ra.indptr[rid + 1];
  const int64_t self = a.ra.self_row(r, rid);
  const int zw = H * a.head_pitch;
  const int c0 = cb * slice_floats;
  const int width = min(slice_floats, zw - c0);
  const int64_t deg = end - beg;
  const int64_t ngroups = (deg + slots_per_group - 1) / slots_per_group;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int g = 0; g < kHubGroups; ++g) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   ::"r"(smem_u32(&full_bar[g])), "r"(bulk ? 1 : 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   ::"r"(smem_u32(&empty_bar[g])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    hub_produce(a.ra, beg, end, a.Z, a.ldz, c0, width, slots_per_group, slice_floats, ring,
                full_bar, empty_bar, bulk);
    return;
  }

  // consumers: per-head peak over self + edges (order-free max)
  const int tid = threadIdx.x;
  {
    float sd[kMaxHeads], pk[kMaxHeads];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h < H) {
        sd[h] = __ldg(a.s_dst + self * H + h);
        pk[h] = leaky(__fadd_rn(__ldg(a.s_src + self * H + h), sd[h]), a.slope);
      }
    }
    // four independent index -> score chains in flight per thread (a hub row
    // has up to ~2e4 edges: one dependent pair per step would bound the pass)
    constexpr int kStride = CW * 32;
    int64_t e = beg + tid;
    for (; e + 3 * kStride < end; e += 4 * kStride) {
      int64_t u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = a.ra.map(__ldg(a.ra.indices + e + q * kStride));
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
          if (h < H)
            pk[h] = fmaxf(pk[h], leaky(__fadd_rn(__ldg(a.s_src + u[q] * H + h), sd[h]), a.slope));
    }
    for (; e < end; e += kStride) {
      const int64_t u = a.ra.map(a.ra.indices[e]);
#pragma unroll
      for (int h = 0; h < kMaxHeads; ++h)
        if (h < H) pk[h] = fmaxf(pk[h], leaky(__fadd_rn(__ldg(a.s_src + u * H + h), sd[h]), a.slope));
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
      if (h < H) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pk[h] = fmaxf(pk[h], __shfl_xor_sync(0xffffffffu, pk[h], o));
        if (lane == 0) s_red[warp][h] = pk[h];
        if (tid == 0) s_sd[h] = sd[h];
      }
    }
    consumer_sync<CW>();
    if (tid < H) {
      float m = s_red[0][tid];
      for (int w = 1; w < CW; ++w) m = fmaxf(m, s_red[w][tid]);
      s_pk[tid] = m;
    }
    consumer_sync<CW>();
  }
  const int col = c0 + tid;
  const int hh = min(col / a.head_pitch, H - 1);
  const int jc = col - hh * a.head_pitch;
  const bool active = tid < width && col < zw && jc < a.head_dim;
  float num = 0.0f, den = 0.0f;
  const int groups_per_chunk = kGatWChunk / slots_per_group;
  for (int64_t gi = 0; gi < ngroups; ++gi) {
    const int64_t wbase = (gi / groups_per_chunk) * kGatWChunk;
    if (gi % groups_per_chunk == 0) {
      // softmax weights of edges [beg + wbase, +kGatWChunk) for all heads
      consumer_sync<CW>();
      const int64_t e0 = beg + wbase;
      const int cnt = static_cast<int>(min(static_cast<int64_t>(kGatWChunk), end - e0));
      int t = tid;
      for (; t + 3 * (CW * 32) < cnt; t += 4 * (CW * 32)) {   // 4 chains in flight
        int64_t u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = a.ra.map(__ldg(a.ra.indices + e0 + t + q * (CW * 32)));
#pragma unroll
        for (int q = 0; q < 4; ++q)
          for (int h = 0; h < H; ++h)
            w_sm[(t + q * (CW * 32)) * H + h] = expf(__fsub_rn(
                leaky(__fadd_rn(__ldg(a.s_src + u[q] * H + h), s_sd[h]), a.slope), s_pk[h]));
      }
      for (; t < cnt; t += (CW * 32)) {
        const int64_t u = a.ra.map(a.ra.indices[e0 + t]);
        for (int h = 0; h < H; ++h)
          w_sm[t * H + h] = expf(
              __fsub_rn(leaky(__fadd_rn(__ldg(a.s_src + u * H + h), s_sd[h]), a.slope), s_pk[h]));
      }
      consumer_sync<CW>();
    }
    const int g = static_cast<int>(gi % kHubGroups);
    const uint32_t round = static_cast<uint32_t>(gi / kHubGroups);
    hub_mbar_wait(&full_bar[g], round & 1u);
    const int cnt = static_cast<int>(min(static_cast<int64_t>(slots_per_group),
                                         end - (beg + gi * slots_per_group)));
    const float* slot0 = ring + static_cast<int64_t>(g) * slots_per_group * slice_floats;
    const float* wrow = w_sm + (gi * slots_per_group - wbase) * H + hh;
    if (active) {
      int j = 0;
      for (; j + 8 <= cnt; j += 8) {
        float w[8], z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          w[u] = wrow[(j + u) * H];
          z[u] = slot0[(j + u) * slice_floats + tid];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          den = __fadd_rn(den, w[u]);
          num = __fadd_rn(num, __fmul_rn(w[u], z[u]));
        }
      }
      for (; j < cnt; ++j) {
        const float w = wrow[j * H];
        den = __fadd_rn(den, w);
        num = __fadd_rn(num, __fmul_rn(w, slot0[j * slice_floats + tid]));
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                                ::"r"(smem_u32(&empty_bar[g])) : "memory");
  }
  if (active) {
    const float ws = expf(__fsub_rn(
        leaky(__fadd_rn(__ldg(a.s_src + self * H + hh), s_sd[hh]), a.slope), s_pk[hh]));
    const float d = __fadd_rn(den, ws);
    const float n = __fadd_rn(num, __fmul_rn(ws, __ldg(a.Z + self * a.ldz + col)));
    a.out[r * a.ld_out + hh * a.head_dim + jc] = gat_epilogue(a, __fdiv_rn(n, d));
  }
}

template <int CW>
int launch_gat_hub_ring_cw(const GatArgs& a, cudaStream_t s) {
  constexpr int kSlice = 32 * CW;
  const int zw = a.heads * a.head_pitch;
  const int width = std::min(kSlice, zw);
  const int slice_floats = ((width + 3) / 4) * 4;
  const int col_blocks = static_cast<int>(ceil_div(zw, kSlice));
  int per_group = kHubRingBytes / (slice_floats * 4) / kHubGroups;
  per_group = std::max(1, std::min(per_group, 32));
  // weight chunks must cover whole ring groups
  while (kGatWChunk % per_group) --per_group;
  const int smem = per_group * kHubGroups * slice_floats * 4 + kGatWChunk * a.heads * 4;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(gat_hub_ring_kernel<CW>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kHubRingBytes + kGatWChunk * kMaxHeads * 4));
    configured.mark();
  }
  const int64_t grid = a.sc.n_hub * col_blocks;
  // TMA bulk copies by default (one 512 B request per source row slice;
  // measured 25.6 vs 26.3 ms LDGSTS at 4x64 and 21.0 vs 22.3 at 4x47,
  // profiles/r01_gat_sweep.jsonl); knob GLINT_TUNE_HUB_INLINE = 2: LDGSTS
  const bool bulk = tuning(GLINT_TUNE_HUB_INLINE) != 2;
  gat_hub_ring_kernel<CW><<<static_cast<unsigned>(grid), (CW + 1) * 32, smem, s>>>(
      a, per_group, slice_floats, col_blocks, bulk);
  return launch_status("gat_aggregate_hub");
}

// GAT hub rows: 128-column slices by default (the softmax weights, index
// stream and per-request cost are shared by more columns than with 64);
// knob GLINT_TUNE_HUB_INLINE = 4 selects 64-column slices, 1 the register path.
int launch_gat_hub_ring(const GatArgs& a, cudaStream_t s) {
  if (tuning(GLINT_TUNE_HUB_INLINE) == 4) return launch_gat_hub_ring_cw<2>(a, s);
  return launch_gat_hub_ring_cw<4>(a, s);
}

// Regular rows (schedule entries n_hub..n_rows), LPR lanes per row.
template <int H, int LPR, int VPL, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) gat_kernel(GatArgs a) {
  __shared__ float s_w[kThreads * H];
  __shared__ float s_st[kThreads / LPR_MIN][2 * H];
  constexpr int G = 32 / LPR;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int group = lane / LPR;
  const int lane_g = lane % LPR;
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * (kWarps * G) + warp * G + group;
  const int64_t idx = a.sc.n_hub + slot;
  if (idx >= a.sc.n_rows) return;
  const int64_t r = a.sc.schedule ? static_cast<int64_t>(a.sc.schedule[idx]) : idx;
  const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (group * LPR));
  float* w_s = s_w + (warp * 32 + group * LPR) * H;  // LPR x H weights per lane group
  gat_row_regular<H, LPR, VPL, U>(a, r, lane_g, gmask, w_s, s_st[warp * G + group]);
}

// Regular rows on the caller's stream (R == 0: register-staged kernel with U
// loads in flight; R > 0: per-lane cp.async ring of R edges), hub rows on the
// library side stream, concurrently.
template <int H, int LPR, int VPL, int U, int MINB, int R = 0>
int launch_gat(const GatArgs& a, cudaStream_t s) {
  constexpr int G = 32 / LPR;
  const int64_t grid = ceil_div(a.sc.n_rows - a.sc.n_hub, kWarps * G);
  const bool after = tuning(GLINT_TUNE_HUB_AFTER) == 1;
  auto launch_hubs = [&](cudaStream_t hs) -> int {
    if (tuning(GLINT_TUNE_HUB_INLINE) == 1) {   // one-CTA-per-row register path
      gat_hub_kernel<<<static_cast<unsigned>(a.sc.hub_ctas), kThreads, 0, hs>>>(a);
      return launch_status("gat_aggregate_hub");
    }
    return launch_gat_hub_ring(a, hs);
  };
  SideFork fork;
  if (a.sc.hub_ctas > 0 && !after) {
    // hub CTAs on the library side stream, concurrent with the regular rows
    int rc = fork.begin(s);
    if (rc) return rc;
    rc = launch_hubs(fork.stream());
    if (rc) return rc;
  }
  if constexpr (R == 0) {
    if (grid > 0) gat_kernel<H, LPR, VPL, U, MINB><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a);
  } else {
    constexpr int smem = R * VPL * kThreads * 16 + kThreads * H * 4;  // Z ring + chunk weights
    static PerDeviceOnce configured;
    if (configured.needed()) {
      GLINT_CUDA(cudaFuncSetAttribute(gat_async_kernel<H, LPR, VPL, R, MINB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured.mark();
    }
    if (grid > 0)
      gat_async_kernel<H, LPR, VPL, R, MINB><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a);
  }
  int rc = launch_status("gat_aggregate");
  if (rc) return rc;
  if (a.sc.hub_ctas > 0 && after) return launch_hubs(s);
  return fork.join();
}

// Two-phase GAT launch: hub rows on the side stream (one-phase ring kernel),
// regular rows as edge softmax then weighted SpMM on the caller's stream.
template <int H, int LPR_A, int LPR, int VPL, int R, int MINB>
int launch_gat2(const GatArgs& a, cudaStream_t s) {
  SideFork fork;
  if (a.sc.hub_ctas > 0) {
    int rc = fork.begin(s);
    if (rc) return rc;
    rc = launch_gat_hub_ring(a, fork.stream());
    if (rc) return rc;
  }
  const int64_t regular = a.sc.n_rows - a.sc.n_hub;
  if (regular > 0) {
    const int64_t ga = ceil_div(regular, kWarps * (32 / LPR_A));
    gat_softmax_kernel<H, LPR_A><<<static_cast<unsigned>(ga), kThreads, 0, s>>>(a);
    int rc = launch_status("gat_softmax");
    if (rc) return rc;
    constexpr int smem = R * VPL * kThreads * 16;
    static PerDeviceOnce configured;
    if (configured.needed()) {
      GLINT_CUDA(cudaFuncSetAttribute(gat_spmm_async_kernel<H, LPR, VPL, R, MINB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured.mark();
    }
    const int64_t gb = ceil_div(regular, kWarps * (32 / LPR));
    gat_spmm_async_kernel<H, LPR, VPL, R, MINB><<<static_cast<unsigned>(gb), kThreads, smem, s>>>(a);
  }
  const int rc = launch_status("gat_spmm");
  const int rj = fork.join();
  return rc ? rc : rj;
}

// chunks = 128-bit chunks per padded Z row.  Variants (GLINT_TUNE_GAT_VARIANT)
// trade unroll depth against occupancy; 0 = default (best measured).
template <int H>
int dispatch_gat_h(const GatArgs& a, int chunks, cudaStream_t s) {
  const int v = tuning(GLINT_TUNE_GAT_VARIANT);
  if (a.w != nullptr) {   // two-phase path (workspace given); variants 1-3 via the knob
    if (chunks <= 16) return launch_gat2<H, 16, 16, 1, 8, 4>(a, s);
    if (chunks <= 32) return launch_gat2<H, 16, 32, 1, 8, 4>(a, s);
    if (chunks <= 48) {
      if (v == 1) return launch_gat2<H, 16, 16, 3, 4, 3>(a, s);
      if (v == 2) return launch_gat2<H, 16, 32, 2, 6, 3>(a, s);
      if (v == 3) return launch_gat2<H, 8, 32, 2, 4, 4>(a, s);
      return launch_gat2<H, 16, 32, 2, 4, 4>(a, s);
    }
    if (chunks <= 64) {
      if (v == 1) return launch_gat2<H, 16, 32, 2, 3, 5>(a, s);
      if (v == 2) return launch_gat2<H, 16, 32, 2, 6, 3>(a, s);
      if (v == 3) return launch_gat2<H, 8, 32, 2, 4, 4>(a, s);
      return launch_gat2<H, 16, 32, 2, 4, 4>(a, s);
    }
  }
  if (chunks <= 8) return launch_gat<H, 8, 1, 4, 6>(a, s);
  if (chunks <= 16) return launch_gat<H, 16, 1, 4, 6>(a, s);
  if (chunks <= 32) {
    if (v == 1) return launch_gat<H, 32, 1, 8, 4>(a, s);
    if (v == 2) return launch_gat<H, 16, 2, 4, 5>(a, s);
    if (v == 5) return launch_gat<H, 32, 1, 0, 4, 8>(a, s);
    return launch_gat<H, 32, 1, 4, 6>(a, s);
  }
  if (chunks <= 48) {   // 0 and 5-9: cp.async ring (R <= LPR); 1-4: register-staged
    if (v == 1) return launch_gat<H, 16, 3, 2, 4>(a, s);
    if (v == 2) return launch_gat<H, 32, 2, 3, 4>(a, s);
    if (v == 3) return launch_gat<H, 16, 3, 3, 3>(a, s);
    if (v == 4) return launch_gat<H, 16, 3, 2, 5>(a, s);
    if (v == 5) return launch_gat<H, 16, 3, 0, 4, 4>(a, s);
    if (v == 6) return launch_gat<H, 16, 3, 0, 5, 3>(a, s);
    if (v == 7) return launch_gat<H, 16, 3, 0, 3, 6>(a, s);
    if (v == 8) return launch_gat<H, 32, 2, 0, 4, 4>(a, s);
    if (v == 9) return launch_gat<H, 16, 3, 0, 4, 2>(a, s);
    return launch_gat<H, 16, 3, 0, 4, 3>(a, s);
  }
  if (chunks <= 64) {
    if (v == 1) return launch_gat<H, 32, 2, 3, 4>(a, s);
    if (v == 2) return launch_gat<H, 32, 2, 4, 3>(a, s);
    if (v == 3) return launch_gat<H, 32, 2, 2, 5>(a, s);
    if (v == 4) return launch_gat<H, 32, 2, 4, 4>(a, s);
    if (v == 5) return launch_gat<H, 32, 2, 0, 4, 3>(a, s);
    if (v == 6) return launch_gat<H, 32, 2, 0, 5, 3>(a, s);
    if (v == 7) return launch_gat<H, 32, 2, 0, 4, 2>(a, s);
    if (v == 8) return launch_gat<H, 32, 2, 0, 5, 4>(a, s);
    if (v == 9) return launch_gat<H, 32, 2, 0, 3, 6>(a, s);
    return launch_gat<H, 32, 2, 0, 4, 4>(a, s);
  }
  if (chunks <= 128) return launch_gat<H, 32, 4, 2, 3>(a, s);
  return launch_gat<H, 32, 8, 1, 2>(a, s);
}

int dispatch_gat(const GatArgs& a, int chunks, cudaStream_t s) {
  switch (a.heads) {
    case 1: return dispatch_gat_h<1>(a, chunks, s);
    case 2: return dispatch_gat_h<2>(a, chunks, s);
    case 3: return dispatch_gat_h<3>(a, chunks, s);
    case 4: return dispatch_gat_h<4>(a, chunks, s);
    case 5: return dispatch_gat_h<5>(a, chunks, s);
    case 6: return dispatch_gat_h<6>(a, chunks, s);
    case 7: return dispatch_gat_h<7>(a, chunks, s);
    default: return dispatch_gat_h<8>(a, chunks, s);
  }
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

int glint_spmm_mean_f32(int64_t n_rows, int32_t dim, const int64_t* indptr,
                        const int32_t* indices, const int64_t* row_ids, int64_t row_base,
                        const int64_t* self_rows, const int32_t* col_map, const float* h,
                        int64_t ld_h, float* out, int64_t ld_out, const int32_t* schedule,
                        int64_t n_hub, const float* bias, int32_t act,
                        glint_stream_t stream) {
  GLINT_REQUIRE(n_rows >= 0, "spmm_mean: n_rows must be >= 0");
  if (n_rows == 0) return GLINT_OK;
  GLINT_REQUIRE(dim > 0, "spmm_mean: dim must be > 0");
  GLINT_REQUIRE(indptr && h && out, "spmm_mean: null indptr/h/out");
  GLINT_REQUIRE(ld_h >= dim && ld_out >= dim, "spmm_mean: leading dimension < dim");
  GLINT_REQUIRE(ld_h < (1LL << 29), "spmm_mean: ld_h must be < 2^29 (row pitch in bytes < 2^31)");
  GLINT_REQUIRE(n_hub >= 0 && n_hub <= n_rows, "spmm_mean: n_hub out of range");
  GLINT_REQUIRE(schedule || n_hub == 0, "spmm_mean: hub rows need a schedule");
  GLINT_REQUIRE(act >= GLINT_ACT_NONE && act <= GLINT_ACT_LEAKY_RELU, "spmm_mean: bad act %d", act);
  MeanArgs a;
  a.ra = RowAddr{indptr, indices, row_ids, row_base, self_rows, col_map};
  a.dim = dim;
  a.h = h;
  a.ld_h = ld_h;
  a.out = out;
  a.ld_out = ld_out;
  a.bias = bias;
  a.act = act;
  a.l2_hint = tuning(GLINT_TUNE_L2_HINT);
  a.sc.schedule = schedule;
  a.sc.n_rows = n_rows;
  a.sc.n_hub = n_hub;
  a.sc.hub_col_blocks = static_cast<int>(ceil_div(dim, kThreads));
  a.sc.hub_ctas = n_hub * a.sc.hub_col_blocks;
  const bool vec4 = (ld_h % 4 == 0) && (ld_out % 4 == 0) && aligned16(h) && aligned16(out);
  return dispatch_mean(a, vec4, as_stream(stream));
}

size_t glint_degree_schedule_workspace_bytes(void) { return 2 * 64 * sizeof(unsigned long long); }

int glint_degree_schedule(int64_t n_rows, const int64_t* indptr, const int64_t* row_ids,
                          int64_t row_base, int64_t hub_min_degree, int32_t* schedule_out,
                          int64_t* n_hub_out, void* workspace, size_t workspace_bytes,
                          glint_stream_t stream) {
  GLINT_REQUIRE(n_rows >= 0 && n_rows < (1LL << 31), "degree_schedule: n_rows out of range");
  GLINT_REQUIRE(indptr && schedule_out && n_hub_out && workspace, "degree_schedule: null argument");
  GLINT_REQUIRE(workspace_bytes >= glint_degree_schedule_workspace_bytes(),
                "degree_schedule: workspace too small");
  GLINT_REQUIRE(hub_min_degree >= 0 && (hub_min_degree & (hub_min_degree - 1)) == 0,
                "degree_schedule: hub_min_degree must be 0 or a power of two");
  cudaStream_t s = as_stream(stream);
  auto* hist = static_cast<unsigned long long*>(workspace);
  auto* offs = hist + 64;
  GLINT_CUDA(cudaMemsetAsync(hist, 0, 64 * sizeof(unsigned long long), s));
  RowAddr ra{indptr, nullptr, row_ids, row_base, nullptr, nullptr};
  int hub_log2 = -1;
  if (hub_min_degree > 0) hub_log2 = 63 - __builtin_clzll(static_cast<unsigned long long>(hub_min_degree));
  const int grid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(ceil_div(n_rows, 256), 1),
                                                      static_cast<int64_t>(sm_count()) * 8));
  if (n_rows > 0) sched_hist_kernel<<<grid, 256, 0, s>>>(n_rows, ra, hist);
  sched_offsets_kernel<<<1, 32, 0, s>>>(hist, offs, hub_log2, n_hub_out);
  if (n_rows > 0) sched_scatter_kernel<<<grid, 256, 0, s>>>(n_rows, ra, offs, schedule_out);
  return launch_status("degree_schedule");
}

size_t glint_gat_aggregate_workspace_bytes(int64_t n_rows, int64_t edge_span, int32_t heads) {
  if (n_rows < 0 || edge_span < 0 || heads < 1) return 0;
  const size_t w = (static_cast<size_t>(edge_span) * heads * 4 + 255) & ~static_cast<size_t>(255);
  return w + static_cast<size_t>(n_rows) * heads * 4;
}

int glint_gat_aggregate_f32(int64_t n_rows, int32_t heads, int32_t head_dim, int32_t head_pitch,
                            const int64_t* indptr, const int32_t* indices, const int64_t* row_ids,
                            int64_t row_base, const int64_t* self_rows, const int32_t* col_map,
                            const float* Z, int64_t ldz, const float* s_src, const float* s_dst,
                            float slope, float* out, int64_t ld_out, const int32_t* schedule,
                            int64_t n_hub, int32_t act, glint_stream_t stream) {
  return glint_gat_aggregate_ws_f32(n_rows, heads, head_dim, head_pitch, indptr, indices, row_ids,
                                    row_base, self_rows, col_map, Z, ldz, s_src, s_dst, slope, out,
                                    ld_out, schedule, n_hub, act, 0, 0, nullptr, 0, stream);
}

int glint_gat_aggregate_ws_f32(int64_t n_rows, int32_t heads, int32_t head_dim, int32_t head_pitch,
                               const int64_t* indptr, const int32_t* indices, const int64_t* row_ids,
                               int64_t row_base, const int64_t* self_rows, const int32_t* col_map,
                               const float* Z, int64_t ldz, const float* s_src, const float* s_dst,
                               float slope, float* out, int64_t ld_out, const int32_t* schedule,
                               int64_t n_hub, int32_t act, int64_t edge_base, int64_t edge_span,
                               void* workspace, size_t workspace_bytes, glint_stream_t stream) {
  GLINT_REQUIRE(n_rows >= 0, "gat_aggregate: n_rows must be >= 0");
  if (n_rows == 0) return GLINT_OK;
  GLINT_REQUIRE(heads >= 1 && heads <= kMaxHeads, "gat_aggregate: heads must be in [1, %d]", kMaxHeads);
  GLINT_REQUIRE(head_dim >= 1 && head_pitch >= head_dim && head_pitch % 4 == 0,
                "gat_aggregate: head_pitch must be a multiple of 4 and >= head_dim");
  GLINT_REQUIRE(ldz < (1LL << 29), "gat_aggregate: ldz must be < 2^29 (row pitch in bytes < 2^31)");
  GLINT_REQUIRE(ldz % 4 == 0 && ldz >= static_cast<int64_t>(heads) * head_pitch && aligned16(Z),
                "gat_aggregate: Z must be 16B aligned with ldz %% 4 == 0 and ldz >= heads*head_pitch");
  GLINT_REQUIRE(indptr && Z && s_src && s_dst && out, "gat_aggregate: null argument");
  GLINT_REQUIRE(ld_out >= static_cast<int64_t>(heads) * head_dim, "gat_aggregate: ld_out too small");
  GLINT_REQUIRE(n_hub >= 0 && n_hub <= n_rows && (schedule || n_hub == 0),
                "gat_aggregate: bad schedule/n_hub");
  GatArgs a{};
  a.ra = RowAddr{indptr, indices, row_ids, row_base, self_rows, col_map};
  a.l2_hint = tuning(GLINT_TUNE_GAT_L2) == 0;   // default on: cfg3 step 71.1 -> 68.3 ms
  a.z_first = tuning(GLINT_TUNE_GAT_PEAK_FIRST) == 0;
  a.heads = heads;
  a.head_dim = head_dim;
  a.head_pitch = head_pitch;
  a.Z = Z;
  a.ldz = ldz;
  a.s_src = s_src;
  a.s_dst = s_dst;
  a.slope = slope;
  a.out = out;
  a.ld_out = ld_out;
  GLINT_REQUIRE(act >= GLINT_ACT_NONE && act <= GLINT_ACT_LEAKY_RELU, "gat_aggregate: bad act %d", act);
  a.act = act;
  const int zw = heads * head_pitch;
  a.sc.schedule = schedule;
  a.sc.n_rows = n_rows;
  a.sc.n_hub = n_hub;
  a.sc.hub_col_blocks = static_cast<int>(ceil_div(zw, kThreads));
  a.sc.hub_ctas = n_hub * a.sc.hub_col_blocks;
  a.w = nullptr;
  a.wself = nullptr;
  a.w_base = edge_base;
  if (workspace) {
    GLINT_REQUIRE(edge_base >= 0 && edge_span >= 0, "gat_aggregate: bad edge range");
    GLINT_REQUIRE(workspace_bytes >= glint_gat_aggregate_workspace_bytes(n_rows, edge_span, heads),
                  "gat_aggregate: workspace too small");
    const size_t wb = (static_cast<size_t>(edge_span) * heads * 4 + 255) & ~static_cast<size_t>(255);
    a.w = static_cast<float*>(workspace);
    a.wself = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + wb);
  }
  const int chunks = zw / 4;
  cudaStream_t s = as_stream(stream);
  GLINT_REQUIRE(chunks <= 256, "gat_aggregate: heads*head_pitch must be <= 1024");
  return dispatch_gat(a, chunks, s);
}

}  // extern "C"
