// K7: fused aggregate-first ConvMean, out = act(mean(h) W^T + b), in ONE
// kernel.  Reference: model_ir.py:336-338 (ConvMean = agg_mean
// then linear), kernels.py:122-135 (agg_mean) and kernels.py:95-107 (linear).
//
// The unfused path writes the B x d_in aggregate to HBM (K1) and reads it back
// (K2): 2 GB per step on the Products layer 1.  Here a tile of 128 rows goes
// from the gather warps' registers through a shared staging tile into TMEM
// and straight into the tensor core:
//
//   warps 0..NG-1  gather (K1's per-lane cp.async ring, one row per warp at a
//                  time, LPR = 32 lanes x 4 columns).  Rows are taken
//                  dynamically from a per-CTA counter; tiles (128 consecutive
//                  schedule slots) from a global counter, so the longest-first
//                  schedule balances across SMs.  A finished row -- the same
//                  fp32 add chain and division as K1, byte-identical -- is one
//                  contiguous 16-byte-per-lane store into a row-major staging
//                  tile (pitch P floats, P/4 odd: conflict-free both ways).
//   warp NG        W loader: one cp.async.bulk per 8-K block of the pre-split
//                  W panel (hi | lo, canonical no-swizzle K-major layout).
//   warp NG+1      MMA issuer: per k-step lo(A).hi(W), hi(A).lo(W), hi(A).hi(W)
//                  -- K2's 3xTF32 product order -- kind::tf32, M = 128, N = BN,
//                  A from TMEM (the "TS" form), fp32 accumulator in TMEM.
//   warps NG+2..   4 converter / epilogue warps (one per TMEM lane quarter):
//                  thread = tile row: read the staged row, store raw (the TF32
//                  "hi": the tensor core ignores the low mantissa bits) and
//                  lo = a - trunc(a) into TMEM, release the staging tile; once
//                  the MMAs retire, tcgen05.ld the accumulator, bias +
//                  activation, and coalesced stores of each 128-byte row
//                  segment to the row's place in `out` (schedule order).
//
// TMEM: [0, BN) accumulator | [256, +32 ceil(nks/4)) raw A | then lo A (K <= 128).
// The staging tile is released right after the converters' TMEM stores, so a
// gather warp that finishes a row of tile i+1 waits only for that copy, not for
// tile i's MMAs.
#include <cuda.h>

#include "common.cuh"

namespace glint {
namespace {
namespace fused {

constexpr int ROWS = 128;                 // rows per tile (TMEM lanes)
constexpr int NEPI = 4;                   // converter / epilogue warps
constexpr int BK = 8;                     // K per W panel block (one MMA k-step)
constexpr int RS = 2;                     // W ring stages
constexpr int EPI_LD = 36;                // staging pitch (floats), conflict-free
constexpr uint32_t RAW_BASE = 256;        // TMEM column of raw A
constexpr uint32_t TCOLS = 512;
constexpr int MAX_K = 128;                // raw + lo A (2 x 128 columns) beside a 256-wide D

template <int NG>
struct Roles {
  static constexpr int W_LOAD = NG, W_MMA = NG + 1, W_EPI = NG + 2;
  static constexpr int THREADS = (W_EPI + NEPI) * 32;
  static constexpr int GT = NG * 32;      // gather threads (ring stride)
};

// staging pitch (floats): a multiple of 4 with P/4 odd, so a warp's row store
// (contiguous) and the converters' column reads (one row per lane) are both
// conflict-free
inline int stage_pitch(int K) {
  int p = static_cast<int>(ceil_div(K, 4)) * 4;
  if ((p / 4) % 2 == 0) p += 4;
  return p;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nFWAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra FDONE;\nbra FWAIT;\nFDONE:\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ const float* row_at(const char* base, int32_t u, int32_t ld_bytes) {
  const char* p;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(p) : "r"(u), "r"(ld_bytes), "l"(base));
  return reinterpret_cast<const float*>(p);
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

// UMMA shared-memory descriptor (sm_100 format, version bit 46)
__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr) {   // W: no swizzle, K-major
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(((BK / 4) * 128) >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}

template <uint32_t IDESC>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n}\n"
      ::"r"(d), "l"(a), "l"(b), "r"(acc), "n"(IDESC));
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}\n"
      ::"r"(d), "r"(a_tmem), "l"(b), "r"(acc), "n"(IDESC));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
      ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
        "f"(v[7]), "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]),
        "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]),
        "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float lo_of(float v) {
  return __fsub_rn(v, __uint_as_float(__float_as_uint(v) & 0xFFFFE000u));
}

struct FArgs {
  const int64_t* __restrict__ indptr;
  const int32_t* __restrict__ indices;
  const int64_t* __restrict__ row_ids;
  int64_t row_base;
  const int64_t* __restrict__ self_rows;
  const int32_t* __restrict__ col_map;
  const int32_t* __restrict__ schedule;
  int64_t n_rows;
  int K, N;
  const float* __restrict__ h;
  int64_t ld_h;
  const float* __restrict__ bias;
  float* __restrict__ out;
  int64_t ld_out;
  const uint8_t* __restrict__ panel;   // nks blocks of [hi | lo], each BN x BK fp32
  int nks;                             // MMA k-steps of 8 (= W blocks)
  int pitch;                           // staging row pitch (floats)
  int ring_off, stg_off, epi_off, bias_off;
  int64_t num_tiles;
  int max_ctas;                        // persistent CTAs (0: one per SM)
  int pipe;                            // 1: next row prepared ahead (gather_rows_pipelined)
  int* __restrict__ tile_ctr;          // zeroed before the launch
  unsigned long long* __restrict__ prof;   // optional phase counters (diagnostics)
};

// Phase counters (GLINT_TUNE_FUSED_PROF), summed over gather warps: 0 cycles
// in the gather loop, 1 cycles waiting for the staging tile, 2 cycles waiting
// for a tile id, 3 rows, 4 tiles.
__device__ unsigned long long g_fused_prof[8];

// One row's mean, K1's mean_row_async at LPR = 32, VPL = 1, B = 1: lane owns
// columns [4 lane, 4 lane + 4); every column is one fp32 add chain in stored
// edge order, self last, then the IEEE division (byte-identical to K1).
template <int R, int GT, bool MAP>
__device__ __forceinline__ float4 gather_mean_row(const FArgs& a, int64_t r, int lane, bool ok,
                                                  uint32_t ring_s, const float4* ring) {
  const int64_t rid = a.row_ids ? a.row_ids[r] : a.row_base + r;
  const int64_t beg = a.indptr[rid];
  const int64_t end = a.indptr[rid + 1];
  const int deg = static_cast<int>(end - beg);
  const float degp1 = static_cast<float>(end - beg + 1);
  const char* hbase = reinterpret_cast<const char*>(a.h + lane * 4);
  const int32_t ldb = static_cast<int32_t>(a.ld_h * 4);
  int ie = 0, cb = 0;
  int32_t cur = (lane < deg) ? __ldg(a.indices + beg + lane) : 0;
  int32_t nxt = (32 + lane < deg) ? __ldg(a.indices + beg + 32 + lane) : 0;
  auto issue = [&](int slot) {
    if (ie - cb == 32) {
      cb += 32;
      cur = nxt;
      nxt = (cb + 32 + lane < deg) ? __ldg(a.indices + beg + cb + 32 + lane) : 0;
    }
    int32_t id = __shfl_sync(0xffffffffu, cur, ie - cb) & 0x7fffffff;
    if (MAP) id = __ldg(a.col_map + id);
    if (ok) cp_async16(ring_s + static_cast<uint32_t>(slot * GT) * 16u, row_at(hbase, id, ldb));
    ++ie;
  };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int g = 0; g < R; ++g) {
    if (ie < deg) issue(g);
    cp_async_commit();
  }
  int base = 0;
  for (int j = 0; j < deg; ++j) {
    cp_async_wait<R - 1>();
    if (ok) add4(acc, ring[base * GT]);
    if (ie < deg) issue(base);
    cp_async_commit();
    base = (base + 1 == R) ? 0 : base + 1;
  }
  cp_async_wait<0>();
  if (!ok) return make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t self = a.self_rows ? a.self_rows[r] : (rid & 0x7fffffff);
  if (!a.self_rows && MAP) self = __ldg(a.col_map + self);
  const float4 s = ldg_f4(a.h + self * a.ld_h + lane * 4);
  return make_float4(__fdiv_rn(__fadd_rn(acc.x, s.x), degp1), __fdiv_rn(__fadd_rn(acc.y, s.y), degp1),
                     __fdiv_rn(__fadd_rn(acc.z, s.z), degp1), __fdiv_rn(__fadd_rn(acc.w, s.w), degp1));
}

// A gather warp's claimed row (warp-uniform).
struct GRow {
  int seq, slot;
  bool term;        // the tile counter ran out: no more tiles
  bool valid;       // a row of a real tile (false: padding past n_rows)
  int64_t beg;
  int deg;
  int32_t cur, nxt; // this lane's ids of the row's first two 32-edge chunks
  float4 self_v;    // this lane's 4 columns of the self row
};

// The gather warps' loop with the next row prepared ahead: right after a row's
// ring prologue is issued, the warp claims the next row and loads its
// schedule slot, indptr pair, first ids and self row -- a chain of dependent
// loads that now overlaps the current row's in-flight edges instead of
// stalling an empty ring at every row start.  The per-edge loop is K1's
// (gather_mean_row): one fp32 add chain per column in stored edge order, self
// last, then the division -- byte-identical.  Terminal handling and the
// staging hand-off are the per-row loop's.
template <int R, int GT, bool MAP>
__device__ __forceinline__ void gather_rows_pipelined(
    const FArgs& a, int lane, bool ok, uint32_t ring_s, const float4* ring, float* stg,
    int* row_ctr, int* tile_of, int* tile_flag, uint64_t* a_full, uint64_t* stg_empty,
    unsigned long long& t_stg, unsigned long long& n_rows_done, unsigned long long& n_tiles) {
  const char* hbase = reinterpret_cast<const char*>(a.h + lane * 4);
  const int32_t ldb = static_cast<int32_t>(a.ld_h * 4);
  auto prepare = [&](GRow& q) {
    int t = 0;
    if (lane == 0) t = atomicAdd(row_ctr, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    q.seq = t >> 7;
    q.slot = t & (ROWS - 1);
    const int tq = q.seq & 3;
    if (q.slot == 0 && lane == 0) {
      const int tid = atomicAdd(a.tile_ctr, 1);
      tile_of[tq] = tid < a.num_tiles ? tid : -1;
      st_release(&tile_flag[tq], q.seq + 1);
    }
    if (lane == 0)
      while (ld_acquire(&tile_flag[tq]) != q.seq + 1) __nanosleep(32);
    __syncwarp();
    const int tid = *reinterpret_cast<volatile int*>(&tile_of[tq]);
    q.term = tid < 0;
    const int64_t idx = static_cast<int64_t>(tid) * ROWS + q.slot;
    q.valid = !q.term && idx < a.n_rows;
    q.beg = 0;
    q.deg = 0;
    q.cur = q.nxt = 0;
    q.self_v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.prof && q.slot == 0 && !q.term) ++n_tiles;
    if (!q.valid) return;
    const int64_t r = a.schedule ? static_cast<int64_t>(a.schedule[idx]) : idx;
    const int64_t rid = a.row_ids ? a.row_ids[r] : a.row_base + r;
    q.beg = a.indptr[rid];
    q.deg = static_cast<int>(a.indptr[rid + 1] - q.beg);
    int64_t self = a.self_rows ? a.self_rows[r] : (rid & 0x7fffffff);
    if (!a.self_rows && MAP) self = __ldg(a.col_map + self);
    if (ok) q.self_v = ldg_f4(a.h + self * a.ld_h + lane * 4);
    q.cur = (lane < q.deg) ? __ldg(a.indices + q.beg + lane) : 0;
    q.nxt = (32 + lane < q.deg) ? __ldg(a.indices + q.beg + 32 + lane) : 0;
  };

  GRow C, N;
  prepare(C);
  while (true) {
    if (C.term) {
      // the slot-0 taker completes the terminal phase (after the previous
      // tile's) so the converters and the MMA issuer see the end
      if (C.slot == 0) {
        if (C.seq > 0) mbar_wait(stg_empty, static_cast<uint32_t>(C.seq - 1) & 1u);
        if (lane == 0) mbar_arrive_n(a_full, ROWS);
      }
      break;
    }
    const int deg = C.deg;
    const int64_t beg = C.beg;
    int ie = 0, cb = 0;
    int32_t cur = C.cur, nxt = C.nxt;
    auto issue = [&](int slot) {
      if (ie - cb == 32) {
        cb += 32;
        cur = nxt;
        nxt = (cb + 32 + lane < deg) ? __ldg(a.indices + beg + cb + 32 + lane) : 0;
      }
      int32_t id = __shfl_sync(0xffffffffu, cur, ie - cb) & 0x7fffffff;
      if (MAP) id = __ldg(a.col_map + id);
      if (ok) cp_async16(ring_s + static_cast<uint32_t>(slot * GT) * 16u, row_at(hbase, id, ldb));
      ++ie;
    };
#pragma unroll
    for (int g = 0; g < R; ++g) {
      if (ie < deg) issue(g);
      cp_async_commit();
    }
    prepare(N);   // the next row's dependent loads overlap this row's ring
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int base = 0;
    for (int j = 0; j < deg; ++j) {
      cp_async_wait<R - 1>();
      if (ok) add4(acc, ring[base * GT]);
      if (ie < deg) issue(base);
      cp_async_commit();
      base = (base + 1 == R) ? 0 : base + 1;
    }
    cp_async_wait<0>();
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (C.valid && ok) {
      const float degp1 = static_cast<float>(deg + 1);
      v = make_float4(__fdiv_rn(__fadd_rn(acc.x, C.self_v.x), degp1),
                      __fdiv_rn(__fadd_rn(acc.y, C.self_v.y), degp1),
                      __fdiv_rn(__fadd_rn(acc.z, C.self_v.z), degp1),
                      __fdiv_rn(__fadd_rn(acc.w, C.self_v.w), degp1));
    }
    if (a.prof && C.valid) ++n_rows_done;
    const unsigned long long ts = a.prof ? clock64() : 0;
    if (C.seq > 0) mbar_wait(stg_empty, static_cast<uint32_t>(C.seq - 1) & 1u);
    if (a.prof) t_stg += clock64() - ts;
    if (C.valid && ok) *reinterpret_cast<float4*>(stg + C.slot * a.pitch + lane * 4) = v;
    __syncwarp();
    if (lane == 0) mbar_arrive(a_full);
    C = N;
  }
}

template <int ACT>
__device__ __forceinline__ float act_op(float x) {
  if (ACT == GLINT_ACT_RELU) x = (x > 0.0f || x != x) ? x : 0.0f;
  if (ACT == GLINT_ACT_LEAKY_RELU) x = x >= 0.0f ? x : __fmul_rn(0.2f, x);
  return x;
}

template <int BN>
struct Cfg {
  static constexpr int WB = BN * BK * 4;                 // one of W hi / lo per block
  static constexpr int W_OFF = 0;
  static constexpr int FIXED = RS * 2 * WB;              // the ring etc. follow at run-time offsets
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(ROWS >> 4) << 24);
  static_assert(BN % 16 == 0 && BN <= 256, "MMA N: multiple of 16, at most 256");
};

// Shared memory (dynamic, 1 KB aligned): [W ring: RS x (hi | lo)] [gather
// ring: R x GT x 16 B] [staging: 128 x P fp32] [epilogue staging] [bias]
template <int BN, int ACT, bool MAP, int NG, int R>
__global__ void __launch_bounds__(Roles<NG>::THREADS, 1) conv_mean_fused_kernel(FArgs a) {
  using C = Cfg<BN>;
  using RL = Roles<NG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t a_full, stg_empty, lo_full, d_full;
  __shared__ __align__(8) uint64_t w_full[RS], w_empty[RS];
  __shared__ uint32_t tmem_slot;
  __shared__ int row_ctr;
  __shared__ int tile_of[4], tile_flag[4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == RL::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_addr(&tmem_slot)), "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&a_full, ROWS);          // one arrival per tile slot (or 128 at termination)
    mbar_init(&stg_empty, NEPI);       // converters copied the staging tile into TMEM
    mbar_init(&lo_full, NEPI);
    mbar_init(&d_full, 1);
    for (int i = 0; i < RS; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    row_ctr = 0;
    for (int i = 0; i < 4; ++i) tile_flag[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp >= RL::W_EPI)
    for (int i = threadIdx.x - RL::W_EPI * 32; i < BN; i += NEPI * 32)
      reinterpret_cast<float*>(smem + a.bias_off)[i] = (a.bias && i < a.N) ? __ldg(a.bias + i) : 0.f;
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;
  // lo A after raw A, both in whole 32-column chunks (the converters' store width)
  const uint32_t lo_base = RAW_BASE + 32u * static_cast<uint32_t>((a.nks + 3) / 4);
  float* stg = reinterpret_cast<float*>(smem + a.stg_off);

  if (warp < NG) {
    // ------------------------------------------------------------- gather
    const bool ok = lane * 4 < a.K;
    float4* ring = reinterpret_cast<float4*>(smem + a.ring_off) + threadIdx.x;
    const uint32_t ring_s = smem_addr(ring);
    unsigned long long t_loop = 0, t_stg = 0, t_tile = 0, n_rows_done = 0, n_tiles = 0;
    const unsigned long long t0 = a.prof ? clock64() : 0;
    if (a.pipe)
      gather_rows_pipelined<R, RL::GT, MAP>(a, lane, ok, ring_s, ring, stg, &row_ctr, tile_of,
                                            tile_flag, &a_full, &stg_empty, t_stg, n_rows_done,
                                            n_tiles);
    while (!a.pipe) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&row_ctr, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      const int seq = t >> 7, slot = t & (ROWS - 1);
      const int tq = seq & 3;
      if (slot == 0 && lane == 0) {
        const int tid = atomicAdd(a.tile_ctr, 1);
        tile_of[tq] = tid < a.num_tiles ? tid : -1;
        st_release(&tile_flag[tq], seq + 1);
      }
      const unsigned long long tw = a.prof ? clock64() : 0;
      if (lane == 0)
        while (ld_acquire(&tile_flag[tq]) != seq + 1) __nanosleep(32);
      __syncwarp();
      if (a.prof) t_tile += clock64() - tw;
      const int tid = *reinterpret_cast<volatile int*>(&tile_of[tq]);
      if (tid < 0) {
        // the slot-0 taker completes the terminal phase (after the previous
        // tile's) so the converters and the MMA issuer see the end
        if (slot == 0) {
          if (seq > 0) mbar_wait(&stg_empty, static_cast<uint32_t>(seq - 1) & 1u);
          if (lane == 0) mbar_arrive_n(&a_full, ROWS);
        }
        break;
      }
      const int64_t idx = static_cast<int64_t>(tid) * ROWS + slot;
      const bool valid = idx < a.n_rows;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) {
        const int64_t r = a.schedule ? static_cast<int64_t>(a.schedule[idx]) : idx;
        v = gather_mean_row<R, RL::GT, MAP>(a, r, lane, ok, ring_s, ring);
        if (a.prof) ++n_rows_done;
      }
      if (a.prof && slot == 0) ++n_tiles;
      const unsigned long long ts = a.prof ? clock64() : 0;
      if (seq > 0) mbar_wait(&stg_empty, static_cast<uint32_t>(seq - 1) & 1u);
      if (a.prof) t_stg += clock64() - ts;
      if (valid && ok) *reinterpret_cast<float4*>(stg + slot * a.pitch + lane * 4) = v;
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full);
    }
    if (a.prof && lane == 0) {
      t_loop = clock64() - t0;
      atomicAdd(a.prof + 0, t_loop);
      atomicAdd(a.prof + 1, t_stg);
      atomicAdd(a.prof + 2, t_tile);
      atomicAdd(a.prof + 3, n_rows_done);
      atomicAdd(a.prof + 4, n_tiles);
    }
  } else if (warp == RL::W_LOAD) {
    // ------------------------------------------------------------ W loader
    if (lane == 0) {
      int ws = 0;
      uint32_t wph = 0;
      for (int seq = 0;; ++seq) {
        const int tq = seq & 3;
        while (ld_acquire(&tile_flag[tq]) != seq + 1) __nanosleep(64);
        if (*reinterpret_cast<volatile int*>(&tile_of[tq]) < 0) break;
        for (int kb = 0; kb < a.nks; ++kb) {
          mbar_wait(&w_empty[ws], wph ^ 1u);
          mbar_arrive_expect_tx(&w_full[ws], 2 * C::WB);
          bulk_g2s(smem_addr(smem + C::W_OFF + ws * 2 * C::WB),
                   a.panel + static_cast<int64_t>(kb) * 2 * C::WB, 2 * C::WB, &w_full[ws]);
          if (++ws == RS) { ws = 0; wph ^= 1u; }
        }
      }
      // every stage's last use released before the CTA may exit
      for (int i = 0; i < RS; ++i) {
        mbar_wait(&w_empty[ws], wph ^ 1u);
        if (++ws == RS) { ws = 0; wph ^= 1u; }
      }
    }
  } else if (warp == RL::W_MMA) {
    // ------------------------------------------------------------ MMA issue
    int ws = 0;
    uint32_t wph = 0;
    for (int seq = 0;; ++seq) {
      mbar_wait(&lo_full, static_cast<uint32_t>(seq) & 1u);
      fence_after();
      if (*reinterpret_cast<volatile int*>(&tile_of[seq & 3]) < 0) break;
      for (int s = 0; s < a.nks; ++s) {
        mbar_wait(&w_full[ws], wph);
        fence_after();
        const uint32_t w_hi = smem_addr(smem + C::W_OFF + ws * 2 * C::WB);
        const uint64_t dwh = desc_plain(w_hi);
        const uint64_t dwl = desc_plain(w_hi + C::WB);
        const uint32_t raw = tmem + RAW_BASE + 8 * s;
        mma_ts<C::IDESC>(tmem, tmem + lo_base + 8 * s, dwh, s > 0);
        mma_ts<C::IDESC>(tmem, raw, dwl, 1u);
        mma_ts<C::IDESC>(tmem, raw, dwh, 1u);
        commit(&w_empty[ws]);
        if (++ws == RS) { ws = 0; wph ^= 1u; }
      }
      commit(&d_full);
      __syncwarp();
    }
  } else {
    // ------------------------------------- raw / lo A into TMEM + epilogue
    const int q = warp & 3;                   // TMEM lane quarter (tcgen05.ld/st access rule)
    const int slot = q * 32 + lane;           // this thread's tile row
    const uint32_t tq_addr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* stage = reinterpret_cast<float*>(smem + a.epi_off) + (warp - RL::W_EPI) * 32 * EPI_LD;
    const float* bias_s = reinterpret_cast<const float*>(smem + a.bias_off);
    const bool has_bias = a.bias != nullptr;
    const float* my_row = stg + slot * a.pitch;
    for (int seq = 0;; ++seq) {
      mbar_wait(&a_full, static_cast<uint32_t>(seq) & 1u);
      const int tid = *reinterpret_cast<volatile int*>(&tile_of[seq & 3]);
      if (tid < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full);   // releases the MMA issuer
        break;
      }
      // (tile seq-1's MMAs have retired: this warp drained its accumulator)
      for (int c0 = 0; c0 < a.nks * 8; c0 += 32) {
        float v[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int col = c0 + 4 * u;
          const float4 x = col < a.K ? *reinterpret_cast<const float4*>(my_row + col)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * u] = x.x;
          v[4 * u + 1] = x.y;
          v[4 * u + 2] = x.z;
          v[4 * u + 3] = x.w;
        }
        tmem_st32(tq_addr + RAW_BASE + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = lo_of(v[i]);
        tmem_st32(tq_addr + lo_base + c0, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&stg_empty);
        mbar_arrive(&lo_full);
      }

      const int64_t idx = static_cast<int64_t>(tid) * ROWS + slot;
      const bool valid = idx < a.n_rows;
      const int64_t row = valid ? (a.schedule ? static_cast<int64_t>(a.schedule[idx]) : idx) : -1;
      mbar_wait(&d_full, static_cast<uint32_t>(seq) & 1u);
      fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tq_addr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)   // no bias: no add (keeps a -0.0 as K2 does)
          v[i] = act_op<ACT>(has_bias ? __fadd_rn(v[i], bias_s[c0 + i]) : v[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(stage + lane * EPI_LD + 4 * i) =
              make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        __syncwarp();
        // 8 lanes per 128-byte row segment, 4 rows per store instruction
        const int cc = (lane & 7) * 4;
        const int col = c0 + cc;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = (lane >> 3) + 4 * i;
          const int64_t orow = __shfl_sync(0xffffffffu, row, rr);
          if (orow >= 0 && col < a.N) {
            const float4 t = *reinterpret_cast<const float4*>(stage + rr * EPI_LD + cc);
            float* dst = a.out + orow * a.ld_out + col;
            if (col + 3 < a.N) {
              *reinterpret_cast<float4*>(dst) = t;
            } else {
              dst[0] = t.x;
              if (col + 1 < a.N) dst[1] = t.y;
              if (col + 2 < a.N) dst[2] = t.z;
            }
          }
        }
        __syncwarp();
      }
      fence_before();
    }
  }
  fence_before();
  __syncthreads();
  if (warp == RL::W_MMA) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// W (N x K, row pitch ldw) -> panel of nks blocks [hi | lo], each BN rows x
// BK fp32 in the canonical no-swizzle K-major layout (8-row x 16-byte core
// matrices, LBO 128 B along K, SBO BK/4 x 128 B between 8-row groups); zero
// padding beyond N and K.
__global__ void panel_kernel(int N, int K, const float* __restrict__ W, int64_t ldw, int bn,
                             uint8_t* __restrict__ panel) {
  const int kb = blockIdx.x;
  uint8_t* hi = panel + static_cast<int64_t>(kb) * 2 * bn * BK * 4;
  uint8_t* lo = hi + bn * BK * 4;
  for (int item = threadIdx.x; item < bn * (BK / 4); item += blockDim.x) {
    const int n = item / (BK / 4), c = item % (BK / 4);
    const uint32_t off = static_cast<uint32_t>((n & 7) * 16 + c * 128 + (n >> 3) * (BK / 4) * 128);
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = kb * BK + 4 * c + e;
      v[e] = (n < N && k < K) ? W[static_cast<int64_t>(n) * ldw + k] : 0.0f;
    }
    float4 h4, l4;
    float* hp = &h4.x;
    float* lp = &l4.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      hp[e] = __uint_as_float(__float_as_uint(v[e]) & 0xFFFFE000u);
      lp[e] = __fsub_rn(v[e], hp[e]);
    }
    *reinterpret_cast<float4*>(hi + off) = h4;
    *reinterpret_cast<float4*>(lo + off) = l4;
  }
}

int pick_bn(int N) { return N <= 64 ? 64 : N <= 128 ? 128 : N <= 192 ? 192 : 256; }

size_t panel_bytes(int K, int N) {
  return static_cast<size_t>(ceil_div(K, BK)) * 2 * pick_bn(N) * BK * 4;
}

constexpr int SMEM_CAP = 227 * 1024 - 1024;   // dynamic budget: 227 KB less the static barriers

template <int BN, int ACT, bool MAP, int NG, int R>
int launch(FArgs a, cudaStream_t s) {
  using C = Cfg<BN>;
  using RL = Roles<NG>;
  a.ring_off = C::FIXED;
  a.stg_off = a.ring_off + R * RL::GT * 16;
  a.epi_off = a.stg_off + ROWS * a.pitch * 4;
  a.bias_off = a.epi_off + NEPI * 32 * EPI_LD * 4;
  const int smem = a.bias_off + BN * 4 + 1024;   // + 1 KB alignment slack
  if (smem > SMEM_CAP) return GLINT_EUNSUPPORTED;
  auto kern = conv_mean_fused_kernel<BN, ACT, MAP, NG, R>;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_CAP));
    configured.mark();
  }
  const int64_t grid = std::min<int64_t>(a.num_tiles, a.max_ctas > 0 ? std::min(a.max_ctas, sm_count())
                                                                    : sm_count());
  kern<<<static_cast<unsigned>(grid), RL::THREADS, smem, s>>>(a);
  return launch_status("conv_mean_fused");
}

template <int BN, int NG, int R>
int launch_act(const FArgs& a, int act, cudaStream_t s) {
  const bool map = a.col_map != nullptr;
  if (act == GLINT_ACT_RELU)
    return map ? launch<BN, GLINT_ACT_RELU, true, NG, R>(a, s)
               : launch<BN, GLINT_ACT_RELU, false, NG, R>(a, s);
  if (act == GLINT_ACT_LEAKY_RELU)
    return map ? launch<BN, GLINT_ACT_LEAKY_RELU, true, NG, R>(a, s)
               : launch<BN, GLINT_ACT_LEAKY_RELU, false, NG, R>(a, s);
  return map ? launch<BN, GLINT_ACT_NONE, true, NG, R>(a, s)
             : launch<BN, GLINT_ACT_NONE, false, NG, R>(a, s);
}

// gather warps x ring depth (GLINT_TUNE_FUSED_VARIANT; profiles/r02_fused_ab.jsonl):
// 0 = the first of 26 x 8, 26 x 6, 16 x 8 whose shared memory fits (more
// warps beat deeper rings: 16 x 12 11.2 ms, 20 x 10 10.6, 24 x 8 9.4 at
// 100 -> 256); 1 = 24 x 8, 2 = 20 x 10, 3 = 16 x 12
template <int BN>
int launch_variant(const FArgs& a, int act, cudaStream_t s) {
  int rc = GLINT_EUNSUPPORTED;
  switch (tuning(GLINT_TUNE_FUSED_VARIANT)) {
    case 1: rc = launch_act<BN, 24, 8>(a, act, s); break;
    case 2: rc = launch_act<BN, 20, 10>(a, act, s); break;
    case 3: rc = launch_act<BN, 16, 12>(a, act, s); break;
    default: break;
  }
  if (rc != GLINT_EUNSUPPORTED) return rc;
  rc = launch_act<BN, 26, 8>(a, act, s);
  if (rc != GLINT_EUNSUPPORTED) return rc;
  rc = launch_act<BN, 26, 6>(a, act, s);
  if (rc != GLINT_EUNSUPPORTED) return rc;
  return launch_act<BN, 16, 8>(a, act, s);
}

}  // namespace fused
}  // namespace

int fused_debug_counters(uint64_t* host_out, int n, int reset) {
  if (n) GLINT_CUDA(cudaMemcpyFromSymbol(host_out, fused::g_fused_prof, n * sizeof(uint64_t)));
  if (reset) {
    const unsigned long long zeros[8] = {0};
    GLINT_CUDA(cudaMemcpyToSymbol(fused::g_fused_prof, zeros, sizeof(zeros)));
  }
  return GLINT_OK;
}

}  // namespace glint

using namespace glint;

extern "C" size_t glint_conv_mean_workspace_bytes(int32_t dim_in, int32_t dim_out) {
  if (dim_in <= 0 || dim_out <= 0) return 0;
  return 256 + fused::panel_bytes(dim_in, dim_out);
}

extern "C" int glint_conv_mean_supported(int32_t dim_in, int32_t dim_out) {
  return dim_in > 0 && dim_in <= fused::MAX_K && dim_in % 4 == 0 && dim_out > 0 && dim_out <= 256;
}

extern "C" int glint_conv_mean_f32(int64_t n_rows, int32_t dim_in, int32_t dim_out,
                                   const int64_t* indptr, const int32_t* indices,
                                   const int64_t* row_ids, int64_t row_base,
                                   const int64_t* self_rows, const int32_t* col_map,
                                   const float* h, int64_t ld_h, const float* W, int64_t ldw,
                                   const float* bias, int32_t act, float* out, int64_t ld_out,
                                   const int32_t* schedule, int32_t max_ctas, void* workspace,
                                   size_t workspace_bytes, glint_stream_t stream) {
  GLINT_REQUIRE(n_rows >= 0, "conv_mean: n_rows must be >= 0");
  if (n_rows == 0) return GLINT_OK;
  GLINT_REQUIRE(dim_in > 0 && dim_out > 0, "conv_mean: dims must be > 0");
  GLINT_REQUIRE(indptr && h && W && out && workspace, "conv_mean: null argument");
  GLINT_REQUIRE(ld_h >= dim_in && ldw >= dim_in && ld_out >= dim_out,
                "conv_mean: leading dimension < dim");
  GLINT_REQUIRE(ld_h < (1LL << 29), "conv_mean: ld_h must be < 2^29");
  GLINT_REQUIRE(act >= GLINT_ACT_NONE && act <= GLINT_ACT_LEAKY_RELU, "conv_mean: bad act %d", act);
  GLINT_REQUIRE(max_ctas >= 0, "conv_mean: max_ctas must be >= 0");
  GLINT_REQUIRE(workspace_bytes >= glint_conv_mean_workspace_bytes(dim_in, dim_out),
                "conv_mean: workspace too small");
  GLINT_REQUIRE(aligned16(workspace), "conv_mean: workspace must be 16-byte aligned");
  if (!glint_conv_mean_supported(dim_in, dim_out) || ld_h % 4 != 0 || ld_out % 4 != 0 ||
      !aligned16(h) || !aligned16(out) || n_rows > (1LL << 31) * fused::ROWS)
    return GLINT_EUNSUPPORTED;
  cudaStream_t s = as_stream(stream);
  fused::FArgs a{};
  a.indptr = indptr;
  a.indices = indices;
  a.row_ids = row_ids;
  a.row_base = row_base;
  a.self_rows = self_rows;
  a.col_map = col_map;
  a.schedule = schedule;
  a.n_rows = n_rows;
  a.K = dim_in;
  a.N = dim_out;
  a.h = h;
  a.ld_h = ld_h;
  a.bias = bias;
  a.out = out;
  a.ld_out = ld_out;
  a.nks = static_cast<int>(ceil_div(dim_in, fused::BK));
  a.pitch = fused::stage_pitch(dim_in);
  a.max_ctas = max_ctas;
  a.pipe = tuning(GLINT_TUNE_FUSED_PIPE) == 0;   // row-ahead gather (0) or one row at a time (1)
  if (tuning(GLINT_TUNE_FUSED_PROF)) {
    void* p = nullptr;
    GLINT_CUDA(cudaGetSymbolAddress(&p, fused::g_fused_prof));
    a.prof = static_cast<unsigned long long*>(p);
  }
  a.num_tiles = ceil_div(n_rows, fused::ROWS);
  auto* ws = static_cast<uint8_t*>(workspace);
  a.tile_ctr = reinterpret_cast<int*>(ws);
  a.panel = ws + 256;
  const int bn = fused::pick_bn(dim_out);
  GLINT_CUDA(cudaMemsetAsync(ws, 0, 256, s));
  fused::panel_kernel<<<a.nks, 256, 0, s>>>(dim_out, dim_in, W, ldw, bn, ws + 256);
  int rc = launch_status("conv_mean_panel");
  if (rc) return rc;
  switch (bn) {
    case 64: return fused::launch_variant<64>(a, act, s);
    case 128: return fused::launch_variant<128>(a, act, s);
    case 192: return fused::launch_variant<192>(a, act, s);
    default: return fused::launch_variant<256>(a, act, s);
  }
}
