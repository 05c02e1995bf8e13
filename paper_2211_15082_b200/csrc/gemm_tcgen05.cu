// K2 on the 5th-generation tensor cores: C = act(A W^T + b) in split-TF32
// ("3xTF32") with tcgen05.mma kind::tf32 and fp32 accumulators in TMEM.
//
// Reference op: kernels.py:95-107 (linear, fp32 einsum).  Plain TF32 misses
// the rel-L2 1e-4 end-to-end bar (3.4e-4), so each operand is split
// x = hi + lo, hi = x with the low 13 mantissa bits cleared (TF32-exact),
// lo = x - hi (exact in fp32), and the product is lo*hi + hi*lo + hi*hi
// (lo*lo ~ 2^-22 relative is dropped).  Measured ~1e-6 rel-L2 vs fp64.
//
// Persistent, warp-specialised kernel, one CTA per SM (416 threads):
//   warps 0-7  producers, two groups of 4 warps taking alternate K blocks:
//              128-bit global loads of A (256 rows) and W (BN rows) for one
//              BK=16 block, hi/lo split in registers, stores into the
//              canonical no-swizzle K-major UMMA layout (8-row x 16 B core
//              matrices, LBO = 128 B along K, SBO = 512 B between 8-row
//              groups), fence.proxy.async, arrive on the stage's FULL barrier;
//   warp 8     allocates TMEM (2*BN columns: one 128-lane accumulator per
//              M half) and issues 2 k-steps x 2 halves x 3 products of
//              tcgen05.mma (M=128, N=BN, K=8) per block; tcgen05.commit frees
//              the stage (EMPTY barrier) and, after the last block, signals
//              TMEM_FULL;
//   warps 9-12 epilogue: tcgen05.ld 32x32b.x32 (warp%4 owns TMEM lane quarter
//              = 32 tile rows), bias + activation, transpose through a padded
//              shared staging tile, coalesced 128 B global stores, then
//              arrive TMEM_EMPTY.
// A 3-stage shared-memory ring (3 x 64 KB at BN=256) decouples producers from
// the MMA issuer; W tiles are shared by both 128-row halves of a 256-row tile,
// halving W re-reads from L2 per output row.
//
// Row invariance (kernels.py:1-14): an output row depends only on its own A
// row and W with a fixed k order, so any batching of rows gives equal bytes.
#include <cuda.h>

#include "common.cuh"

namespace glint {
namespace {

constexpr int BM = 256;           // rows per tile (two M=128 MMA halves)
constexpr int HALF = 128;
constexpr int BK = 16;            // K per pipeline stage (2 MMA k-steps)
constexpr int STAGES = 3;
constexpr int kProducerWarps = 8;
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
constexpr int kThreads = 13 * 32;
constexpr uint32_t SBO = (BK / 4) * 128;   // bytes between 8-row core-matrix groups
constexpr uint32_t LBO = 128;              // bytes between K-adjacent core matrices
constexpr int EPI_LD = 36;                 // staging row pitch (floats): conflict-free

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((LBO >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((SBO >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100); no swizzle
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
      :
      : "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :
               : "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" : : "r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" : : "r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n"
      :
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
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

template <int BN>
struct Cfg {
  static constexpr uint32_t TCOLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                    : 2 * BN <= 256 ? 256 : 512;
  static constexpr int A_BYTES = BM * BK * 4;  // one of hi / lo
  static constexpr int W_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * W_BYTES;
  static constexpr int EPI_BYTES = 4 * 32 * EPI_LD * 4 + 4 * BN * 4;  // staging + bias copies
  static constexpr int SMEM = STAGES * STAGE + EPI_BYTES;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(HALF >> 4) << 24);
};

struct TcArgs {
  int64_t M;
  int N, K;
  const float* __restrict__ A;
  int64_t lda;
  const int64_t* __restrict__ a_rows;
  const float* __restrict__ W;
  int64_t ldw;
  const float* __restrict__ bias;
  float* __restrict__ C;
  int64_t ldc;
  int64_t num_tiles;
  int n_tiles;
  int nkb;
  bool c_vec4;
  bool raw_hi;               // experiment knob GLINT_TUNE_GEMM_RAWHI (v1 kernel only)
  bool mma_only;             // diagnostics knob GLINT_TUNE_GEMM_PROF == 2 (v2 kernel)
  bool skip_lo;              // diagnostics knob GLINT_TUNE_GEMM_PROF == 3: no lo pass (wrong results)
  // GAT projection epilogue (v2, SC = true): per-head scores of each output row
  const float* attn;         // [heads, 2 * head_dim]
  float* s_src;              // [M, heads]
  float* s_dst;
  int heads, head_dim, head_pitch;
  int sc_mode;               // GLINT_TUNE_GAT_EPI (0 chunked fast path, 1 per-column walk, 2 diagnostic)
  unsigned long long* prof;  // optional phase-cycle counters (GLINT_TUNE_GEMM_PROF)
};

// Phase counters, summed over CTAs: 0 producer wait(empty), 1 producer work,
// 2 mma wait(full), 3 mma wait(tmem_empty), 4 epilogue wait(tmem_full),
// 5 epilogue work, 6 kernel cycles, 7 tiles.
__device__ unsigned long long g_gemm_prof[8];

__device__ __forceinline__ void prof_add(const TcArgs& a, int k, unsigned long long v) {
  if (a.prof) atomicAdd(a.prof + k, v);
}

template <bool VEC>
__device__ __forceinline__ float4 load4(const float* row, int k, int K) {
  if constexpr (VEC) {
    if (k < K) return ldg_f4(row + k);
    return make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    float4 v;
    v.x = k < K ? __ldg(row + k) : 0.f;
    v.y = k + 1 < K ? __ldg(row + k + 1) : 0.f;
    v.z = k + 2 < K ? __ldg(row + k + 2) : 0.f;
    v.w = k + 3 < K ? __ldg(row + k + 3) : 0.f;
    return v;
  }
}

__device__ __forceinline__ void split_store(uint8_t* hi_base, uint8_t* lo_base, uint32_t off,
                                            float4 v) {
  float4 hi, lo;
  hi.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
  hi.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
  hi.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
  hi.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
  lo.x = __fsub_rn(v.x, hi.x);
  lo.y = __fsub_rn(v.y, hi.y);
  lo.z = __fsub_rn(v.z, hi.z);
  lo.w = __fsub_rn(v.w, hi.w);
  *reinterpret_cast<float4*>(hi_base + off) = hi;
  *reinterpret_cast<float4*>(lo_base + off) = lo;
}

// (row r of a 128-row operand half or of W, 16-byte chunk c) -> byte offset
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return static_cast<uint32_t>((r & 7) * 16 + c * 128 + (r >> 3) * SBO);
}

template <int ACT>
__device__ __forceinline__ float epilogue_op(float x, const float* bias_s, bool has_bias) {
  if (has_bias) x = __fadd_rn(x, *bias_s);
  if (ACT == GLINT_ACT_RELU) x = (x > 0.0f || x != x) ? x : 0.0f;
  if (ACT == GLINT_ACT_LEAKY_RELU) x = x >= 0.0f ? x : __fmul_rn(0.2f, x);
  return x;
}

template <int BN, bool VEC, int ACT>
__global__ void __launch_bounds__(kThreads, 1) gemm_3xtf32_kernel(TcArgs a) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tmem_full;
  __shared__ __align__(8) uint64_t tmem_empty;
  __shared__ uint32_t tmem_slot;

  const unsigned long long t_start = clock64();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :
                 : "r"(smem_addr(&tmem_slot)), "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 4);   // one arrive per producer warp of the group
      mbar_init(&empty_bar[s], 1);  // tcgen05.commit
    }
    mbar_init(&tmem_full, 1);
    mbar_init(&tmem_empty, 4);      // one arrive per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;
  const int nkb = a.nkb;

  if (warp < kProducerWarps) {
    // ---------------------------------------------------------- producers
    // Flattened (tile, k-block) steps of this CTA; group g takes steps
    // g, g+2, ...  The loads of a group's next step are issued before it
    // waits for a free stage and splits the current one (register double
    // buffering), so two steps of global loads are in flight per thread.
    const int grp = warp >> 2;
    const int wq = warp & 3;
    const int rsub = lane & 7;
    const int chunk = lane >> 3;  // 0..3: 16-byte chunk within the BK=16 block
    constexpr int WG = (BN / 8 + 3) / 4;
    const int64_t my_tiles = blockIdx.x < a.num_tiles
                                 ? (a.num_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total = my_tiles * nkb;
    unsigned long long t_wait = 0, t_work = 0;

    auto load_a = [&](int64_t idx, float4 (&va)[BM / 32]) {
      const int64_t tile = blockIdx.x + (idx / nkb) * gridDim.x;
      const int kb = static_cast<int>(idx % nkb);
      const int64_t m0 = (tile / a.n_tiles) * BM;
      const int k = kb * BK + 4 * chunk;
#pragma unroll
      for (int i = 0; i < BM / 32; ++i) {
        const int64_t row = m0 + (wq + 4 * i) * 8 + rsub;
        va[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < a.M) va[i] = load4<VEC>(a.A + (a.a_rows ? a.a_rows[row] : row) * a.lda, k, a.K);
      }
    };
    auto store_step = [&](int64_t idx, const float4 (&va)[BM / 32]) {
      // W (L2-resident) is loaded here, A was prefetched one step ahead.
      const int64_t tile = blockIdx.x + (idx / nkb) * gridDim.x;
      const int n0 = static_cast<int>(tile % a.n_tiles) * BN;
      const int k = static_cast<int>(idx % nkb) * BK + 4 * chunk;
      float4 vw[WG];
#pragma unroll
      for (int i = 0; i < WG; ++i) {
        const int r = (wq + 4 * i) * 8 + rsub;
        vw[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < BN && n0 + r < a.N)
          vw[i] = load4<VEC>(a.W + static_cast<int64_t>(n0 + r) * a.ldw, k, a.K);
      }
      const int s = static_cast<int>(idx % STAGES);
      const uint32_t round = static_cast<uint32_t>(idx / STAGES);
      const unsigned long long t0 = clock64();
      mbar_wait(&empty_bar[s], (round & 1u) ^ 1u);
      const unsigned long long t1 = clock64();
      t_wait += t1 - t0;
      uint8_t* a_hi = smem + s * C::STAGE;
      uint8_t* a_lo = a_hi + C::A_BYTES;
      uint8_t* w_hi = a_lo + C::A_BYTES;
      uint8_t* w_lo = w_hi + C::W_BYTES;
#pragma unroll
      for (int i = 0; i < BM / 32; ++i) {
        const int r = (wq + 4 * i) * 8 + rsub;
        const uint32_t off = (r >= HALF ? C::A_BYTES / 2 : 0) + tile_off(r & (HALF - 1), chunk);
        split_store(a_hi, a_lo, off, va[i]);
        if (a.raw_hi)  // experiment: feed the unmasked fp32 as the "hi" operand
          *reinterpret_cast<float4*>(a_hi + off) = va[i];
      }
#pragma unroll
      for (int i = 0; i < WG; ++i) {
        const int r = (wq + 4 * i) * 8 + rsub;
        if (r < BN) split_store(w_hi, w_lo, tile_off(r, chunk), vw[i]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[s]);
      t_work += clock64() - t1;
    };

    float4 va0[BM / 32], va1[BM / 32];
    int64_t idx = grp;
    if (idx < total) load_a(idx, va0);
    while (idx < total) {
      if (idx + 2 < total) load_a(idx + 2, va1);
      store_step(idx, va0);
      idx += 2;
      if (idx >= total) break;
      if (idx + 2 < total) load_a(idx + 2, va0);
      store_step(idx, va1);
      idx += 2;
    }
    if (lane == 0) {
      prof_add(a, 0, t_wait);
      prof_add(a, 1, t_work);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issue
    unsigned long long t_full = 0, t_tmem = 0;
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
      unsigned long long t0 = clock64();
      mbar_wait(&tmem_empty, (static_cast<uint32_t>(it) & 1u) ^ 1u);
      t_tmem += clock64() - t0;
      fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const int64_t idx = it * nkb + kb;
        const int s = static_cast<int>(idx % STAGES);
        const uint32_t round = static_cast<uint32_t>(idx / STAGES);
        t0 = clock64();
        mbar_wait(&full_bar[s], round & 1u);
        t_full += clock64() - t0;
        fence_after();
        if (lane == 0) {
          const uint32_t a_hi = smem_addr(smem + s * C::STAGE);
          const uint32_t a_lo = a_hi + C::A_BYTES;
          const uint32_t w_hi = a_lo + C::A_BYTES;
          const uint32_t w_lo = w_hi + C::W_BYTES;
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint32_t step = j * 256;  // 8 tf32 along K = two 16-byte core matrices
            const uint64_t dwh = umma_desc(w_hi + step);
            const uint64_t dwl = umma_desc(w_lo + step);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t hoff = h * (C::A_BYTES / 2) + step;
              const uint32_t d = tmem + static_cast<uint32_t>(h * BN);
              mma_tf32(d, umma_desc(a_lo + hoff), dwh, C::IDESC, (kb | j) != 0);
              mma_tf32(d, umma_desc(a_hi + hoff), dwl, C::IDESC, 1u);
              mma_tf32(d, umma_desc(a_hi + hoff), dwh, C::IDESC, 1u);
            }
          }
          mma_commit(&empty_bar[s]);
          if (kb == nkb - 1) mma_commit(&tmem_full);
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      prof_add(a, 2, t_full);
      prof_add(a, 3, t_tmem);
      prof_add(a, 7, static_cast<unsigned long long>(it));
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    float* stage = reinterpret_cast<float*>(smem + STAGES * C::STAGE) + (warp - kEpiWarp0) * 32 * EPI_LD;
    float* bias_s = reinterpret_cast<float*>(smem + STAGES * C::STAGE) + 4 * 32 * EPI_LD +
                    (warp - kEpiWarp0) * BN;
    const bool has_bias = a.bias != nullptr;
    int bias_n0 = -1;
    unsigned long long t_wait = 0, t_work = 0;
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
      const int64_t m0 = (tile / a.n_tiles) * BM;
      const int n0 = static_cast<int>(tile % a.n_tiles) * BN;
      if (has_bias && n0 != bias_n0) {   // this warp's copy of bias[n0, n0+BN)
        __syncwarp();
        for (int i = lane; i < BN; i += 32) bias_s[i] = n0 + i < a.N ? __ldg(a.bias + n0 + i) : 0.f;
        __syncwarp();
        bias_n0 = n0;
      }
      const unsigned long long t0 = clock64();
      mbar_wait(&tmem_full, static_cast<uint32_t>(it) & 1u);
      const unsigned long long t1 = clock64();
      t_wait += t1 - t0;
      fence_after();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int64_t row_base = m0 + h * HALF + q * 32;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + h * BN + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = n0 + c0 + i;
            v[i] = col < a.N ? epilogue_op<ACT>(v[i], bias_s + c0 + i, has_bias) : 0.0f;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4*>(stage + lane * EPI_LD + 4 * i) =
                make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          __syncwarp();
          const int cc = (lane & 7) * 4;
          const int col = n0 + c0 + cc;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = (lane >> 3) + 4 * i;
            const int64_t row = row_base + rr;
            if (row < a.M && col < a.N) {
              const float4 t = *reinterpret_cast<const float4*>(stage + rr * EPI_LD + cc);
              float* dst = a.C + row * a.ldc + col;
              if (a.c_vec4 && col + 3 < a.N) {
                *reinterpret_cast<float4*>(dst) = t;
              } else {
                dst[0] = t.x;
                if (col + 1 < a.N) dst[1] = t.y;
                if (col + 2 < a.N) dst[2] = t.z;
                if (col + 3 < a.N) dst[3] = t.w;
              }
            }
          }
          __syncwarp();
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty);
      t_work += clock64() - t1;
    }
    if (lane == 0) {
      prof_add(a, 4, t_wait);
      prof_add(a, 5, t_work);
    }
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x == 0) prof_add(a, 6, clock64() - t_start);
  if (warp == kMmaWarp) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" : : "r"(tmem), "r"(C::TCOLS));
  }
}

template <int BN, bool VEC, int ACT>
int launch_tc(TcArgs a, cudaStream_t s) {
  using C = Cfg<BN>;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(gemm_3xtf32_kernel<BN, VEC, ACT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    configured.mark();
  }
  a.n_tiles = static_cast<int>(ceil_div(a.N, BN));
  a.num_tiles = ceil_div(a.M, BM) * a.n_tiles;
  a.nkb = static_cast<int>(ceil_div(a.K, BK));
  const int64_t grid = std::min<int64_t>(a.num_tiles, sm_count());
  gemm_3xtf32_kernel<BN, VEC, ACT><<<static_cast<unsigned>(grid), kThreads, C::SMEM, s>>>(a);
  return launch_status("linear_3xtf32");
}

template <int BN, bool VEC>
int launch_act(const TcArgs& a, int act, cudaStream_t s) {
  if (act == GLINT_ACT_RELU) return launch_tc<BN, VEC, GLINT_ACT_RELU>(a, s);
  if (act == GLINT_ACT_LEAKY_RELU) return launch_tc<BN, VEC, GLINT_ACT_LEAKY_RELU>(a, s);
  return launch_tc<BN, VEC, GLINT_ACT_NONE>(a, s);
}

template <bool VEC>
int launch_bn(const TcArgs& a, int act, cudaStream_t s) {
  if (a.N <= 32) return launch_act<32, VEC>(a, act, s);
  if (a.N <= 48) return launch_act<48, VEC>(a, act, s);
  if (a.N <= 64) return launch_act<64, VEC>(a, act, s);
  if (a.N <= 128) return launch_act<128, VEC>(a, act, s);
  if (a.N <= 192) return launch_act<192, VEC>(a, act, s);
  return launch_act<256, VEC>(a, act, s);
}

// ============================================================== v2 kernel --
//
// Same split-TF32 products and k order as the kernel above, restructured for
// the two limits measured on it (phase counters, ncu source stalls): the
// producers stalled on A's DRAM latency with only ~1 stage of lookahead, and
// the epilogue serialised with the MMAs.
//   * The tensor core truncates fp32 operands of kind::tf32 to TF32 (ignores
//     the low 13 mantissa bits; verified bit-for-bit, tools/tf32_trunc_probe.py),
//     so the raw fp32 A tile IS the "hi" operand: producers cp.async (LDGSTS)
//     raw A rows straight into the canonical K-major UMMA layout RA-1 k-steps
//     ahead (no registers held), then compute only lo = a - trunc(a) into a
//     small lo ring just before the MMA needs it.
//   * W is pre-split once per call (w_panel_kernel) into hi/lo blocks already in
//     the UMMA layout; a loader warp streams one block per k-step with ONE
//     cp.async.bulk (TMA engine, mbarrier tx-count), RW steps ahead.
//   * Tiles are 256 rows x BN <= 128 columns; TMEM holds TWO accumulators
//     (2 x 2 halves x BN <= 512 columns): the MMA warp starts tile i+1 while the
//     epilogue warps drain tile i.
#ifndef GLINT_GEMM_RA1
#define GLINT_GEMM_RA1 8
#endif
#ifndef GLINT_GEMM_RL1
#define GLINT_GEMM_RL1 2
#endif
#ifndef GLINT_GEMM_RL2
#define GLINT_GEMM_RL2 2
#endif
#ifndef GLINT_GEMM_RW1
#define GLINT_GEMM_RW1 3
#endif
namespace v2 {

constexpr int kEpiWarps2 = 8;
constexpr int kScMaxN = 512;               // widest Z row with the fused score epilogue

// Warp roles: PW producer warps, then the MMA warp, the W loader and 8
// epilogue warps.  8 producer warps measured faster than 4 for both tile
// shapes, although 18 warps cap the kernel at 96 registers (the fused GAT
// score epilogue then spills a little; profiles/r01_gemm_sweep.jsonl).
template <int MH>
struct Roles {
  static constexpr int PW = 8;
  static constexpr int MMA = PW;
  static constexpr int WL = PW + 1;
  static constexpr int EPI = PW + 2;
  static constexpr int THREADS = (PW + 2 + kEpiWarps2) * 32;
  static constexpr int PT = PW * 32;
};

template <int BN, int MH = 2>   // MH: 128-row M halves per tile (2: 256 x BN, 1: 128 x BN)
struct Cfg2 {
  static constexpr int TM = MH * HALF;           // tile rows
  // raw-A ring (cp.async, also the TF32 "hi" operand): 128-row tiles have the
  // shared memory for a deeper ring (more loads in flight per SM)
  static constexpr int RA = MH == 1 ? GLINT_GEMM_RA1 : 6;
  // A "lo" ring (computed by the producers): the producer of lo(k) waits for
  // the MMAs of k - RL to retire, so RL bounds how far lo runs ahead of the
  // tensor pipe; W panel ring (TMA bulk copies from L2)
  static constexpr int RL = MH == 1 ? GLINT_GEMM_RL1 : (BN <= 96 ? GLINT_GEMM_RL2 : 2);
  static constexpr int RW = MH == 1 ? GLINT_GEMM_RW1 : 3;
  static constexpr int A_BYTES = TM * BK * 4;  // one raw / lo slot (TM x 16 fp32)
  static constexpr int W_BYTES = BN * BK * 4;  // one of W hi / lo
  static constexpr int RAW_OFF = 0;
  static constexpr int LO_OFF = RA * A_BYTES;
  static constexpr int W_OFF = LO_OFF + RL * A_BYTES;
  static constexpr int EPI_OFF = W_OFF + RW * 2 * W_BYTES;
  static constexpr uint32_t ACC = MH * BN;     // TMEM columns of one accumulator
  static constexpr uint32_t TCOLS = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128
                                    : 2 * ACC <= 256 ? 256 : 512;
  static constexpr int EPI_BYTES = kEpiWarps2 * 32 * EPI_LD * 4 + kEpiWarps2 * BN * 4;
  static constexpr int SC_OFF = EPI_OFF + EPI_BYTES;      // score tables (SC kernels only)
  static constexpr int SMEM = EPI_OFF + EPI_BYTES;
  static constexpr int SMEM_SC = SC_OFF + 2 * kScMaxN * 4;   // a_src | a_dst
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(HALF >> 4) << 24);
};

__global__ void w_panel_kernel(int N, int K, const float* __restrict__ W, int64_t ldw, int bn,
                               int nkb, uint8_t* __restrict__ panel) {
  const int blk = blockIdx.x;
  const int nt = blk / nkb;
  const int kb = blk - nt * nkb;
  uint8_t* hi = panel + static_cast<int64_t>(blk) * 2 * bn * BK * 4;
  uint8_t* lo = hi + bn * BK * 4;
  for (int item = threadIdx.x; item < bn * 4; item += blockDim.x) {
    const int r = item >> 2, c = item & 3;
    const int n = nt * bn + r;
    const int k = kb * BK + 4 * c;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n < N) v = load4<false>(W + static_cast<int64_t>(n) * ldw, k, K);
    split_store(hi, lo, tile_off(r, c), v);
  }
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Epilogue of one CW-column chunk (CW = 32 or 16) of a 32-row TMEM lane quarter.
// Running per-row GAT score state of the fused projection epilogue: the lane
// walks its row's columns in order; a head's dot products with a_src / a_dst
// are sequential fmaf chains over j, written out when the head ends.
struct ScoreAcc {
  int h;
  float ps, pd;
};

__device__ __forceinline__ void score_flush(const TcArgs& a, ScoreAcc& st, int64_t row) {
  if (st.h >= 0 && row < a.M) {
    a.s_src[row * a.heads + st.h] = st.ps;
    a.s_dst[row * a.heads + st.h] = st.pd;
  }
}

template <int CW, int ACT, bool SC = false>
__device__ __forceinline__ void epi_chunk(const TcArgs& a, uint32_t taddr, float* stage,
                                          const float* bias_s, bool has_bias, int64_t row_base,
                                          int col0, int lane, const float* sc_tab,
                                          ScoreAcc& st) {
  float v[CW];
  if constexpr (CW == 32) tmem_ld32(taddr, v);
  else tmem_ld16(taddr, v);
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    const int col = col0 + i;
    v[i] = col < a.N ? epilogue_op<ACT>(v[i], bias_s + i, has_bias) : 0.0f;
  }
  if constexpr (SC) {
    // sc_tab: [0, N) a_src per column, [kScMaxN, +N) a_dst.  The columns of a
    // head are contiguous, so the chunk splits into at most a few head runs:
    // the head changes at warp-uniform positions (no per-element lookup or
    // divergence); each head's dot products stay one sequential fmaf chain.
    const int64_t row = row_base + lane;
    if (a.sc_mode == 2) {
      // diagnostic: no score math
    } else if (a.sc_mode != 1 && a.head_pitch % 16 == 0 && col0 + CW <= a.N) {
      // every 16-column half of the chunk lies in one head (chunks start at
      // multiples of 16): no per-column head or bounds checks, a_src / a_dst
      // as 128-bit broadcast loads; the same fmaf chain order, so the same bits
#pragma unroll
      for (int hb = 0; hb < CW / 16; ++hb) {
        const int cc = col0 + 16 * hb;
        const int h = cc / a.head_pitch;
        if (h != st.h) {
          score_flush(a, st, row);
          st.h = h;
          st.ps = 0.0f;
          st.pd = 0.0f;
        }
        const float4* ts = reinterpret_cast<const float4*>(sc_tab + cc);
        const float4* td = reinterpret_cast<const float4*>(sc_tab + kScMaxN + cc);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 s4 = ts[q4];
          const float4 d4 = td[q4];
          const float* vv = v + 16 * hb + 4 * q4;
          st.ps = fmaf(vv[0], s4.x, st.ps);
          st.pd = fmaf(vv[0], d4.x, st.pd);
          st.ps = fmaf(vv[1], s4.y, st.ps);
          st.pd = fmaf(vv[1], d4.y, st.pd);
          st.ps = fmaf(vv[2], s4.z, st.ps);
          st.pd = fmaf(vv[2], d4.z, st.pd);
          st.ps = fmaf(vv[3], s4.w, st.ps);
          st.pd = fmaf(vv[3], d4.w, st.pd);
        }
      }
    } else {
      int h = min(col0 / a.head_pitch, a.heads - 1);
      int next = (h + 1) * a.head_pitch;      // first column of the following head
      if (h != st.h) {
        score_flush(a, st, row);
        st.h = h;
        st.ps = 0.0f;
        st.pd = 0.0f;
      }
#pragma unroll
      for (int i = 0; i < CW; ++i) {
        const int col = col0 + i;
        if (col >= a.N) break;
        if (col == next && h + 1 < a.heads) {
          score_flush(a, st, row);
          ++h;
          next += a.head_pitch;
          st.h = h;
          st.ps = 0.0f;
          st.pd = 0.0f;
        }
        st.ps = fmaf(v[i], sc_tab[col], st.ps);
        st.pd = fmaf(v[i], sc_tab[kScMaxN + col], st.pd);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < CW / 4; ++i)
    *reinterpret_cast<float4*>(stage + lane * EPI_LD + 4 * i) =
        make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  __syncwarp();
  constexpr int LPRW = CW / 4;          // lanes per row segment
  constexpr int RPI = 32 / LPRW;        // rows per store instruction
  const int cc = (lane % LPRW) * 4;
  const int col = col0 + cc;
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int rr = lane / LPRW + RPI * i;
    const int64_t row = row_base + rr;
    if (row < a.M && col < a.N) {
      const float4 t = *reinterpret_cast<const float4*>(stage + rr * EPI_LD + cc);
      float* dst = a.C + row * a.ldc + col;
      if (a.c_vec4 && col + 3 < a.N) {
        *reinterpret_cast<float4*>(dst) = t;
      } else {
        dst[0] = t.x;
        if (col + 1 < a.N) dst[1] = t.y;
        if (col + 2 < a.N) dst[2] = t.z;
        if (col + 3 < a.N) dst[3] = t.w;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

template <int BN, int ACT, bool SC = false, int MH = 2>
__global__ void __launch_bounds__(Roles<MH>::THREADS, 1) gemm_v2_kernel(TcArgs a, const uint8_t* __restrict__ panel) {
  using C = Cfg2<BN, MH>;
  using Rl = Roles<MH>;
  constexpr int PER = C::TM * 4 / Rl::PT;   // 16-byte chunks per producer thread
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t raw_empty[C::RA];
  __shared__ __align__(8) uint64_t lo_full[C::RL], lo_empty[C::RL];
  __shared__ __align__(8) uint64_t w_full[C::RW], w_empty[C::RW];
  __shared__ __align__(8) uint64_t tmem_full[2];
  __shared__ __align__(8) uint64_t tmem_empty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == Rl::MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :
                 : "r"(smem_addr(&tmem_slot)), "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::RA; ++i) mbar_init(&raw_empty[i], 1);           // tcgen05.commit
    for (int i = 0; i < C::RL; ++i) {
      mbar_init(&lo_full[i], Rl::PW);                           // one per producer warp
      mbar_init(&lo_empty[i], 1);
    }
    for (int i = 0; i < C::RW; ++i) {
      mbar_init(&w_full[i], 1);                                         // expect_tx arrive
      mbar_init(&w_empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], kEpiWarps2);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;
  const int nkb = a.nkb;
  const int64_t my_tiles = blockIdx.x < a.num_tiles
                               ? (a.num_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nkb;

  if (a.mma_only && (warp < Rl::PW || warp == Rl::WL)) {
    // diagnostics: no operand traffic
  } else if (warp < Rl::PW) {
    // ---------------------------------------------------------- producers
    // Thread t owns 16-byte chunks q = t + 256 i (i < 4) of every k-step:
    // row q >> 2, k-chunk q & 3 -- it copies them (cp.async) and later turns
    // the same chunks into lo, so it only ever waits on its own copies.
    const int t = threadIdx.x;
    int rows[PER], chs[PER];
    uint32_t offs[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int q = t + Rl::PT * i;
      rows[i] = q >> 2;
      chs[i] = q & 3;
      offs[i] = (rows[i] / HALF) * (HALF * BK * 4) + tile_off(rows[i] & (HALF - 1), chs[i]);
    }
    const uint32_t raw_base = smem_addr(smem + C::RAW_OFF);
    auto issue = [&](int64_t idx) {
      const int slot = static_cast<int>(idx % C::RA);
      const uint32_t use = static_cast<uint32_t>(idx / C::RA);
      mbar_wait(&raw_empty[slot], (use & 1u) ^ 1u);
      const int64_t tile = blockIdx.x + (idx / nkb) * gridDim.x;
      const int kb = static_cast<int>(idx % nkb);
      const int64_t m0 = (tile / a.n_tiles) * C::TM;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int64_t row = m0 + rows[i];
        const int k = kb * BK + 4 * chs[i];
        const bool ok = row < a.M && k < a.K;
        const float* src = ok ? a.A + (a.a_rows ? a.a_rows[row] : row) * a.lda + k : a.A;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                     ::"r"(raw_base + slot * C::A_BYTES + offs[i]), "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    };
    for (int64_t d = 0; d < C::RA - 1; ++d) {
      if (d < total) issue(d);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t idx = 0; idx < total; ++idx) {
      asm volatile("cp.async.wait_group %0;" ::"n"(C::RA - 2) : "memory");  // own copies of idx landed
      const int rs = static_cast<int>(idx % C::RA);
      const int ls = static_cast<int>(idx % C::RL);
      const uint32_t luse = static_cast<uint32_t>(idx / C::RL);
      mbar_wait(&lo_empty[ls], (luse & 1u) ^ 1u);
      const uint8_t* raw = smem + C::RAW_OFF + rs * C::A_BYTES;
      uint8_t* lo = smem + C::LO_OFF + ls * C::A_BYTES;
#pragma unroll
      for (int i = 0; i < PER && !a.skip_lo; ++i) {   // a.skip_lo: diagnostics only
        const float4 v = *reinterpret_cast<const float4*>(raw + offs[i]);
        float4 l;
        l.x = __fsub_rn(v.x, __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
        l.y = __fsub_rn(v.y, __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
        l.z = __fsub_rn(v.z, __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
        l.w = __fsub_rn(v.w, __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
        *reinterpret_cast<float4*>(lo + offs[i]) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&lo_full[ls]);
      if (idx + C::RA - 1 < total) issue(idx + C::RA - 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (warp == Rl::WL) {
    // ------------------------------------------------- W panel loader (TMA)
    if (lane == 0) {
      for (int64_t idx = 0; idx < total; ++idx) {
        const int64_t tile = blockIdx.x + (idx / nkb) * gridDim.x;
        const int nt = static_cast<int>(tile % a.n_tiles);
        const int kb = static_cast<int>(idx % nkb);
        const int s = static_cast<int>(idx % C::RW);
        const uint32_t use = static_cast<uint32_t>(idx / C::RW);
        mbar_wait(&w_empty[s], (use & 1u) ^ 1u);
        mbar_arrive_expect_tx(&w_full[s], 2 * C::W_BYTES);
        bulk_g2s(smem + C::W_OFF + s * 2 * C::W_BYTES,
                 panel + (static_cast<int64_t>(nt) * nkb + kb) * 2 * C::W_BYTES, 2 * C::W_BYTES,
                 &w_full[s]);
      }
    }
  } else if (warp == Rl::MMA) {
    // ------------------------------------------------------------ MMA issue
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
      const int buf = static_cast<int>(it & 1);
      const uint32_t tuse = static_cast<uint32_t>(it >> 1);
      mbar_wait(&tmem_empty[buf], (tuse & 1u) ^ 1u);
      fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const int64_t idx = it * nkb + kb;
        const int rs = static_cast<int>(idx % C::RA);
        const int ls = static_cast<int>(idx % C::RL);
        const int ws = static_cast<int>(idx % C::RW);
        if (!a.mma_only) {   // a.mma_only: diagnostics, MMA issue rate without operand waits
          mbar_wait(&lo_full[ls], static_cast<uint32_t>(idx / C::RL) & 1u);
          mbar_wait(&w_full[ws], static_cast<uint32_t>(idx / C::RW) & 1u);
        }
        fence_after();
        if (lane == 0) {
          const uint32_t a_hi = smem_addr(smem + C::RAW_OFF + rs * C::A_BYTES);
          const uint32_t a_lo = smem_addr(smem + C::LO_OFF + ls * C::A_BYTES);
          const uint32_t w_hi = smem_addr(smem + C::W_OFF + ws * 2 * C::W_BYTES);
          const uint32_t w_lo = w_hi + C::W_BYTES;
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint32_t step = j * 256;
            const uint64_t dwh = umma_desc(w_hi + step);
            const uint64_t dwl = umma_desc(w_lo + step);
#pragma unroll
            for (int h = 0; h < MH; ++h) {
              const uint32_t hoff = h * (HALF * BK * 4) + step;
              const uint32_t d = tmem + static_cast<uint32_t>(buf * C::ACC + h * BN);
              mma_tf32(d, umma_desc(a_lo + hoff), dwh, C::IDESC, (kb | j) != 0);
              mma_tf32(d, umma_desc(a_hi + hoff), dwl, C::IDESC, 1u);
              mma_tf32(d, umma_desc(a_hi + hoff), dwh, C::IDESC, 1u);
            }
          }
          mma_commit(&raw_empty[rs]);
          mma_commit(&lo_empty[ls]);
          mma_commit(&w_empty[ws]);
          if (kb == nkb - 1) mma_commit(&tmem_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    // 8 warps: warp w drains TMEM lane quarter (w % 4) (the tcgen05.ld access
    // rule); pair index p = (w - Rl::EPI) / 4 picks the M half (MH = 2: 32 rows x
    // BN columns) or the column half (MH = 1: 32 rows x BN/2 columns).
    const int q = warp & 3;
    const int p = (warp - Rl::EPI) >> 2;
    const int h = MH == 2 ? p : 0;
    constexpr int CW_SPAN = MH == 2 ? BN : BN / 2;    // columns this warp drains
    const int cbase = MH == 2 ? 0 : p * CW_SPAN;
    float* stage = reinterpret_cast<float*>(smem + C::EPI_OFF) + (warp - Rl::EPI) * 32 * EPI_LD;
    float* bias_s = reinterpret_cast<float*>(smem + C::EPI_OFF) + kEpiWarps2 * 32 * EPI_LD +
                    (warp - Rl::EPI) * BN;
    const bool has_bias = a.bias != nullptr;
    float* sc_tab = reinterpret_cast<float*>(smem + C::SC_OFF);
    if constexpr (SC) {
      // per-column a_src / a_dst tables, shared by the 8 epilogue warps
      for (int c = threadIdx.x - Rl::EPI * 32; c < a.N; c += kEpiWarps2 * 32) {
        const int hh = c / a.head_pitch;
        const int j = c - hh * a.head_pitch;
        const bool live = hh < a.heads && j < a.head_dim;
        sc_tab[c] = live ? __ldg(a.attn + hh * 2 * a.head_dim + j) : 0.0f;
        sc_tab[kScMaxN + c] = live ? __ldg(a.attn + hh * 2 * a.head_dim + a.head_dim + j) : 0.0f;
      }
      asm volatile("bar.sync 2, %0;" ::"r"(kEpiWarps2 * 32) : "memory");
    }
    int bias_n0 = -1;
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++it) {
      const int buf = static_cast<int>(it & 1);
      const uint32_t tuse = static_cast<uint32_t>(it >> 1);
      const int64_t m0 = (tile / a.n_tiles) * C::TM;
      const int n0 = static_cast<int>(tile % a.n_tiles) * BN;
      if (has_bias && n0 != bias_n0) {
        __syncwarp();
        for (int i = lane; i < BN; i += 32) bias_s[i] = n0 + i < a.N ? __ldg(a.bias + n0 + i) : 0.f;
        __syncwarp();
        bias_n0 = n0;
      }
      mbar_wait(&tmem_full[buf], tuse & 1u);
      fence_after();
      {
        const int64_t row_base = m0 + h * HALF + q * 32;
        const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(buf * C::ACC + h * BN + cbase);
        ScoreAcc st{-1, 0.0f, 0.0f};
        if constexpr (SC) {
          // 16-column chunks: the score chains need registers the 32-wide
          // chunk would take (96 per thread at 18 warps)
#pragma unroll 1
          for (int c0 = 0; c0 + 16 <= CW_SPAN; c0 += 16)
            epi_chunk<16, ACT, SC>(a, tbase + c0, stage, bias_s + cbase + c0, has_bias, row_base,
                                   n0 + cbase + c0, lane, sc_tab, st);
        } else {
#pragma unroll 1
          for (int c0 = 0; c0 + 32 <= CW_SPAN; c0 += 32)
            epi_chunk<32, ACT, SC>(a, tbase + c0, stage, bias_s + cbase + c0, has_bias, row_base,
                                   n0 + cbase + c0, lane, sc_tab, st);
        }
        if constexpr (!SC && CW_SPAN % 32 == 16)
          epi_chunk<16, ACT, SC>(a, tbase + (CW_SPAN - 16), stage, bias_s + cbase + CW_SPAN - 16,
                                 has_bias, row_base, n0 + cbase + CW_SPAN - 16, lane, sc_tab, st);
        if constexpr (SC) score_flush(a, st, row_base + lane);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == Rl::MMA) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" : : "r"(tmem), "r"(C::TCOLS));
  }
}

template <int BN, int ACT, bool SC = false, int MH = 2>
int launch_v2(TcArgs a, cudaStream_t s) {
  using C = Cfg2<BN, MH>;
  constexpr int smem = SC ? C::SMEM_SC : C::SMEM;
  static_assert(smem <= 227 * 1024, "v2 GEMM shared memory over the per-CTA limit");
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(gemm_v2_kernel<BN, ACT, SC, MH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured.mark();
  }
  a.n_tiles = static_cast<int>(ceil_div(a.N, BN));
  a.num_tiles = ceil_div(a.M, C::TM) * a.n_tiles;
  a.nkb = static_cast<int>(ceil_div(a.K, BK));
  const size_t panel_bytes = static_cast<size_t>(a.n_tiles) * a.nkb * 2 * C::W_BYTES;
  void* panel = nullptr;
  GLINT_CUDA(cudaMallocAsync(&panel, panel_bytes, s));
  w_panel_kernel<<<a.n_tiles * a.nkb, 128, 0, s>>>(a.N, a.K, a.W, a.ldw, BN, a.nkb,
                                                   static_cast<uint8_t*>(panel));
  int rc = launch_status("linear_3xtf32_panel");
  if (rc == GLINT_OK) {
    const int64_t grid = std::min<int64_t>(a.num_tiles, sm_count());
    gemm_v2_kernel<BN, ACT, SC, MH><<<static_cast<unsigned>(grid), Roles<MH>::THREADS, smem, s>>>(
        a, static_cast<const uint8_t*>(panel));
    rc = launch_status("linear_3xtf32");
  }
  GLINT_CUDA(cudaFreeAsync(panel, s));
  return rc;
}

template <int BN, int MH = 2>
int launch_v2_act(const TcArgs& a, int act, cudaStream_t s) {
  if (act == GLINT_ACT_RELU) return launch_v2<BN, GLINT_ACT_RELU, false, MH>(a, s);
  if (act == GLINT_ACT_LEAKY_RELU) return launch_v2<BN, GLINT_ACT_LEAKY_RELU, false, MH>(a, s);
  return launch_v2<BN, GLINT_ACT_NONE, false, MH>(a, s);
}

// N in (128, 256]: 128-row tiles with ONE N = BN MMA per product (each A row
// is loaded and split once for all columns; knob GLINT_TUNE_GEMM_WIDE = 2
// forces the 256-row x N/2 tiles).  N <= 128: 256-row tiles, BN = N rounded
// up to an instantiated width.
int launch_v2_bn(const TcArgs& a, int act, cudaStream_t s) {
  if (a.N > 128 && a.N <= 256 && tuning(GLINT_TUNE_GEMM_WIDE) != 2) {
    if (a.N <= 192) return launch_v2_act<192, 1>(a, act, s);
    return launch_v2_act<256, 1>(a, act, s);
  }
  if (a.N <= 128 && tuning(GLINT_TUNE_GEMM_WIDE) == 3) {   // experiment: 128-row tiles
    if (a.N <= 48) return launch_v2_act<48, 1>(a, act, s);
    if (a.N <= 64) return launch_v2_act<64, 1>(a, act, s);
    return launch_v2_act<128, 1>(a, act, s);
  }
  const int nt = static_cast<int>(ceil_div(a.N, 128));
  const int per = static_cast<int>(ceil_div(a.N, nt));
  if (per <= 32) return launch_v2_act<32>(a, act, s);
  if (per <= 48) return launch_v2_act<48>(a, act, s);
  if (per <= 64) return launch_v2_act<64>(a, act, s);
  if (per <= 96) return launch_v2_act<96>(a, act, s);
  return launch_v2_act<128>(a, act, s);
}

// GAT projection with fused scores: needs every head inside one n-tile.
int launch_v2_scores(const TcArgs& a, cudaStream_t s) {
  if (a.N > 128 && a.N <= 256 && tuning(GLINT_TUNE_GEMM_WIDE) != 2) {
    if (a.N <= 192) return launch_v2<192, GLINT_ACT_NONE, true, 1>(a, s);
    return launch_v2<256, GLINT_ACT_NONE, true, 1>(a, s);
  }
  const int nt = static_cast<int>(ceil_div(a.N, 128));
  const int per = static_cast<int>(ceil_div(a.N, nt));
  auto fits = [&](int bn) { return ceil_div(a.N, bn) == 1 || bn % a.head_pitch == 0; };
  if (per <= 32 && fits(32)) return launch_v2<32, GLINT_ACT_NONE, true>(a, s);
  if (per <= 48 && fits(48)) return launch_v2<48, GLINT_ACT_NONE, true>(a, s);
  if (per <= 64 && fits(64)) return launch_v2<64, GLINT_ACT_NONE, true>(a, s);
  if (per <= 96 && fits(96)) return launch_v2<96, GLINT_ACT_NONE, true>(a, s);
  if (fits(128)) return launch_v2<128, GLINT_ACT_NONE, true>(a, s);
  return GLINT_EUNSUPPORTED;
}

}  // namespace v2

// ============================================================== v3 kernel --
//
// Same split-TF32 products, k order and epilogue as v2, with the operand path
// rebuilt around the Blackwell copy engines:
//   * A and W tiles arrive by TMA tensor copies (cp.async.bulk.tensor, SASS
//     UTMALDG) into the 128-byte-swizzled K-major UMMA layout: 32 fp32 of K
//     per row per chunk (one swizzle atom row), 8-row groups 1 KB apart.  One
//     elected thread issues every copy, so no warp spends issue slots on
//     address generation (v2's 8 LDGSTS producer warps).
//   * The raw fp32 tile is the TF32 "hi" operand (the tensor core ignores the
//     low 13 mantissa bits, tools/tf32_trunc_probe.py).  Four converter warps
//     compute lo = x - trunc(x) elementwise over the same swizzled bytes (the
//     layout is a byte permutation, so lo lands in the identical layout), for
//     A and for W: no W panel kernel, no workspace, no allocation.
//   * N > 64: a CTA pair (cluster of 2, tcgen05 cta_group::2).  The pair
//     computes a 256-row tile with one M = 256 MMA per product; each CTA
//     loads its own 128 A rows and HALF of the W rows (B split along N across
//     the pair, tools/probes/umma2_probe.cu), which halves the per-SM W traffic
//     from L2 and the shared-memory B reads.  The leader's thread issues the
//     MMAs and commits to both CTAs' barriers (multicast); the peer's
//     converters and epilogue warps arrive on the leader's barriers remotely.
//   * N <= 64 (the narrowing layer-3 transform, 256 -> 47): W (raw + lo) stays
//     resident in shared memory for the whole persistent CTA, so only A
//     streams and the kernel runs at the A-read (HBM) rate.
//   * TMEM holds two accumulators: the MMA issuer starts tile i+1 while the
//     epilogue warps drain tile i.
namespace v3 {

constexpr int BKC = 32;                     // fp32 K per chunk = one 128 B swizzle row
constexpr int ROWS = 128;                   // A rows per CTA per tile
constexpr int A_BYTES = ROWS * BKC * 4;     // 16 KB
constexpr int NCONV = 4;                    // converter warps per group (one per lane quarter)
// One converter group: a second group taking alternate chunks measured no
// faster, and with an odd stage count two consumers of one stage ring make
// the mbarrier parity waits ambiguous (a waiter can see the previous phase of
// the same parity as complete) -- tools/gemm_det_check.py caught exactly that.
constexpr int NGRP = 1;
constexpr int W_TMA = 0, W_MMA = 1, W_CONV = 2, W_EPI = W_CONV + NGRP * NCONV;
// epilogue warps: 4 (one per TMEM lane quarter); the GAT score epilogue uses
// 8 (two per quarter, split at a head boundary: its per-row score chains are
// the long pole there)
// epilogue warps: the score-fused BN = 256 tiles drain faster with 8 (100 -> 4x64:
// 0.93 vs 1.07 ms); at BN = 192 four keep a 4th operand stage (256 -> 4x47: 1.21
// vs 1.30 ms; profiles/r02c_gemm_sc_epi_warps.jsonl)
template <int BN, bool SC>
constexpr int nepi() { return SC && BN == 256 ? 8 : 4; }
template <int BN, bool SC>
constexpr int threads3() { return (W_EPI + nepi<BN, SC>()) * 32; }
constexpr int RL = 2;                       // A lo ring depth (shared memory, pair kernels)
constexpr int RT = 4;                       // A hi/lo TMEM slots (resident-W kernels)
constexpr uint32_t TS_BASE = 256;           // first TMEM column of the A slots
constexpr int MAX_RS = 8;
constexpr int SMEM_CAP = 227 * 1024 - 2048;   // dynamic budget: 227 KB less the static barriers
constexpr uint64_t POLICY_EVICT_FIRST = 0x12F0000000000000ull;
constexpr uint64_t POLICY_EVICT_LAST = 0x14F0000000000000ull;

template <int BN, bool PAIR>
struct Cfg3 {
  static constexpr int BNH = PAIR ? BN / 2 : BN;     // W rows one CTA holds
  static constexpr int WB = BNH * BKC * 4;           // one W chunk (raw or lo)
  static constexpr uint32_t TCOLS = PAIR ? (2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128
                                             ? 128 : 2 * BN <= 256 ? 256 : 512)
                                         : 512;   // single CTAs: accumulators + A slots
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>((PAIR ? 2 * ROWS : ROWS) >> 4) << 24);
  static_assert(BNH % 8 == 0, "W rows per CTA must fill 8-row swizzle groups");
  static_assert(2 * BN <= 512, "two accumulators must fit TMEM");
};

// Shared-memory plan (dynamic, every buffer 1 KB aligned for the swizzle):
//   [RS stages: A raw | W raw | W lo (streamed W only)] [RL A lo] [resident W
//   raw/lo chunks] [epilogue staging | bias | score tables]
struct Plan3 {
  int rs = 0, stage = 0, lo_off = 0, wres_off = 0, epi_off = 0, smem = 0;
};

// staging tiles + per-warp bias copies + score tables
template <int BN, bool SC>
constexpr int epi_bytes() {
  // two score tables (a_src | a_dst): at BN = 256 this keeps the epilogue at 48 KB,
  // so the score-fused pair kernel holds 3 operand stages like the plain one
  return nepi<BN, SC>() * (32 * EPI_LD + BN) * 4 + (SC ? 2 * v2::kScMaxN * 4 : 0);
}

template <int BN, bool PAIR, bool RESW, bool SC>
Plan3 plan3(int nkc) {
  using C = Cfg3<BN, PAIR>;
  constexpr int EPI = epi_bytes<BN, SC>();
  Plan3 p;
  p.stage = A_BYTES + (RESW ? 0 : 2 * C::WB);
  const int wres = RESW ? nkc * 2 * C::WB : 0;
  // resident-W kernels keep A hi/lo in TMEM, so only the pair kernels need
  // the shared-memory lo ring
  const int fixed = (RESW ? 0 : RL * A_BYTES) + wres + EPI + 1024;   // +1 KB align slack
  p.rs = std::min(MAX_RS, (SMEM_CAP - fixed) / p.stage);
  p.lo_off = p.rs * p.stage;
  p.wres_off = p.lo_off + (RESW ? 0 : RL * A_BYTES);
  p.epi_off = p.wres_off + wres;
  p.smem = p.epi_off + EPI + 1024;
  return p;
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;                   // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;           // SBO: 8-row groups 1 KB apart
  d |= static_cast<uint64_t>(1) << 46;                   // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                   // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t num_clusters() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}


// arrive on the pair leader's copy of `bar` (CTA rank 0 of the cluster)
template <bool PAIR>
__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t rank) {
  // default (.release.cta) semantics, as CUTLASS's ClusterBarrier: a
  // .cluster-scope release compiles to MEMBAR.GPU + L1 invalidation (CCTL.IVALL)
  // per arrive, measured as ~23% of the stall samples of the first v3 build
  if (!PAIR || rank == 0) {
    mbar_arrive(bar);
  } else {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_addr(bar)));
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar)),
        "l"(policy)
      : "memory");
}

// L2 prefetch of one box (no shared memory, no barrier): tiles ahead of the
// shared-memory ring, so the ring's TMA loads hit L2
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1) : "memory");
}

// The MMA issuer is a whole warp running a convergent loop over warp-uniform
// values; elect.sync INSIDE the asm picks the one issuing lane.  With the
// instruction descriptor an immediate and the k-steps unrolled at constant
// descriptor offsets, the compiler keeps every operand in uniform registers:
// tools/probes/mma_rate_probe.cu measures this form at the M*N/256-cycle
// formula (TS: 24 cycles at N = 48), where a lane-0-only loop with a runtime
// descriptor cost ~100 cycles per MMA (R2UR + ELECT waterfall per issue).
template <bool PAIR, uint32_t IDESC>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
  if constexpr (PAIR) {
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %4, p;\n}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(accumulate), "n"(IDESC));
  } else {
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(accumulate), "n"(IDESC));
  }
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}\n"
      ::"r"(d), "r"(a_tmem), "l"(b), "r"(accumulate), "n"(IDESC));
}

// tcgen05.commit (one elected lane) to `bar` in this CTA or in both CTAs of the pair
template <bool PAIR>
__device__ __forceinline__ void commit3(uint64_t* bar) {
  if constexpr (PAIR) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n}\n" ::"r"(smem_addr(bar)), "h"(static_cast<uint16_t>(3)) : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
        ::"r"(smem_addr(bar)) : "memory");
  }
}

// lo = x - trunc_tf32(x) over n16 16-byte words (same byte offsets)
__device__ __forceinline__ float lo_of(float v) {
  return __fsub_rn(v, __uint_as_float(__float_as_uint(v) & 0xFFFFE000u));
}
__device__ __forceinline__ float4 lo_of(float4 v) {
  return make_float4(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w));
}
// four loads in flight per thread before the dependent math and stores
__device__ __forceinline__ void split_lo(const uint8_t* src, uint8_t* dst, int n16, int t) {
  constexpr int T = NCONV * 32;
  int q = t;
  for (; q + 3 * T < n16; q += 4 * T) {
    float4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = *reinterpret_cast<const float4*>(src + (q + i * T) * 16);
#pragma unroll
    for (int i = 0; i < 4; ++i) *reinterpret_cast<float4*>(dst + (q + i * T) * 16) = lo_of(v[i]);
  }
  for (; q < n16; q += T)
    *reinterpret_cast<float4*>(dst + q * 16) = lo_of(*reinterpret_cast<const float4*>(src + q * 16));
}

// tcgen05.st of 32 consecutive TMEM columns of this warp's lane quarter
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

// A operand from TMEM (the "TS" form): D[tmem] += A[tmem] . B[smem]
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

struct V3Args {
  int rs, stage, lo_off, wres_off, epi_off;
  int nkc;              // K chunks of 32
  int pf_tiles;         // L2 prefetch distance of A, in this CTA's tiles (0 = off)
  int n_tiles;          // column tiles of BN
  int64_t num_tiles;    // m tiles (of 128 or 256 rows) x n tiles
};

template <int BN, int ACT, bool SC, bool PAIR, bool RESW>
__global__ void __launch_bounds__(threads3<BN, SC>(), 1)
gemm_v3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
               TcArgs a, V3Args g) {
  using C = Cfg3<BN, PAIR>;
  constexpr int NEPI = nepi<BN, SC>();
  extern __shared__ uint8_t smem_raw[];
  // 1 KB alignment for the 128 B swizzle atoms
  // (offset arithmetic on the __shared__ array keeps the state-space provenance,
  // so the converters and the epilogue get LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[MAX_RS], empty[MAX_RS], rdy[MAX_RS];
  __shared__ __align__(8) uint64_t lo_empty[RT];   // A lo slots (RL) or A TMEM slots (RT)
  __shared__ __align__(8) uint64_t tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t wres_full, wres_rdy;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cta_rank() : 0;
  const uint32_t cid = PAIR ? cluster_id() : blockIdx.x;
  const uint32_t ncl = PAIR ? num_clusters() : gridDim.x;
  constexpr uint32_t NPEER = PAIR ? 2 : 1;
  const int rs = g.rs;

  if (warp == W_MMA) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_addr(&tmem_slot)), "r"(C::TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_addr(&tmem_slot)), "r"(C::TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    for (int i = 0; i < rs; ++i) {
      mbar_init(&full[i], 1);                 // producer arrive + TMA bytes
      mbar_init(&empty[i], RESW ? NCONV : 1);  // converters (A now in TMEM) or MMA commit
      mbar_init(&rdy[i], NCONV * NPEER);      // converters of both CTAs (leader's copy)
    }
    for (int i = 0; i < (RESW ? RT : RL); ++i) mbar_init(&lo_empty[i], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], NEPI * NPEER);
    }
    mbar_init(&wres_full, 1);
    mbar_init(&wres_rdy, NGRP * NCONV);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;
  const int nkc = g.nkc;
  const int64_t my_tiles = cid < g.num_tiles ? (g.num_tiles - 1 - cid) / ncl + 1 : 0;
  const int64_t total = my_tiles * nkc;
  constexpr int TM = PAIR ? 2 * ROWS : ROWS;   // rows per (pair) tile

  if (warp == W_TMA) {
    // ------------------------------------------------------------ TMA issue
    if (lane == 0) {
      if constexpr (RESW) {
        v2::mbar_arrive_expect_tx(&wres_full, static_cast<uint32_t>(nkc * C::WB));
        for (int c = 0; c < nkc; ++c)
          tma_load_2d(smem_addr(smem + g.wres_off + c * 2 * C::WB), &tmW, c * BKC, 0, &wres_full,
                      POLICY_EVICT_LAST);
      }
      int s = 0;
      uint32_t ph = 0;
      int64_t tile = cid;
      int c = 0;
      for (int64_t idx = 0; idx < total; ++idx) {
        if (c == 0 && g.pf_tiles > 0) {
          // this CTA's A rows of tile + pf_tiles * ncl into L2
          const int64_t pt = tile + static_cast<int64_t>(g.pf_tiles) * ncl;
          if (pt < g.num_tiles && (pt % g.n_tiles) == 0) {
            const int pm = static_cast<int>((pt / g.n_tiles) * TM + rank * ROWS);
            for (int k = 0; k < nkc; ++k) tma_prefetch_2d(&tmA, k * BKC, pm);
          }
        }
        mbar_wait(&empty[s], ph ^ 1u);
        const int64_t m0 = (tile / g.n_tiles) * TM + rank * ROWS;
        const int n0 = static_cast<int>(tile % g.n_tiles) * BN + static_cast<int>(rank) * C::BNH;
        uint8_t* st = smem + s * g.stage;
        v2::mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(A_BYTES + (RESW ? 0 : C::WB)));
        tma_load_2d(smem_addr(st), &tmA, c * BKC, static_cast<int>(m0), &full[s],
                    POLICY_EVICT_FIRST);
        if constexpr (!RESW)
          tma_load_2d(smem_addr(st + A_BYTES), &tmW, c * BKC, n0, &full[s], POLICY_EVICT_LAST);
        if (++s == rs) { s = 0; ph ^= 1u; }
        if (++c == nkc) { c = 0; tile += ncl; }
      }
      // drain: every stage's last use is released (the MMA commits target
      // this CTA's barriers) before the CTA may exit
      for (int64_t idx = total > rs ? total - rs : 0; idx < total; ++idx)
        mbar_wait(&empty[idx % rs], static_cast<uint32_t>(idx / rs) & 1u);
    }
  } else if (warp >= W_CONV && warp < W_EPI) {
    // ----------------------------------------------------------- converters
    const int grp = (warp - W_CONV) / NCONV;
    const int t = threadIdx.x - (W_CONV + grp * NCONV) * 32;   // thread within the group
    if constexpr (RESW) {
      mbar_wait(&wres_full, 0);
      for (int c = grp; c < nkc; c += NGRP)
        split_lo(smem + g.wres_off + c * 2 * C::WB, smem + g.wres_off + c * 2 * C::WB + C::WB,
                 C::WB / 16, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&wres_rdy);
    }
    constexpr int NL = RESW ? RT : RL;
    for (int64_t idx = grp; idx < total; idx += NGRP) {
      const int s = static_cast<int>(idx % rs);
      const uint32_t ph = static_cast<uint32_t>(idx / rs) & 1u;
      const int l = static_cast<int>(idx % NL);
      const uint32_t lph = static_cast<uint32_t>(idx / NL) & 1u;
      mbar_wait(&full[s], ph);
      mbar_wait(&lo_empty[l], lph ^ 1u);
      uint8_t* st = smem + s * g.stage;
      if constexpr (RESW) {
        // thread = A row (this warp's TMEM lane quarter): read the row's 32
        // floats out of the swizzled tile, release the stage to the TMA at
        // once, then store hi (= raw) and lo into the TMEM slot
        const int row = (warp & 3) * 32 + lane;
        const uint8_t* rp = st + row * 128;
        float v[32];
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const float4 x = *reinterpret_cast<const float4*>(rp + ((c16 ^ (row & 7)) << 4));
          v[4 * c16] = x.x;
          v[4 * c16 + 1] = x.y;
          v[4 * c16 + 2] = x.z;
          v[4 * c16 + 3] = x.w;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const uint32_t ta = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + TS_BASE +
                            static_cast<uint32_t>(l * 64);
        tmem_st32(ta, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = lo_of(v[i]);
        tmem_st32(ta + 32, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_before();
      } else {
        split_lo(st, smem + g.lo_off + l * A_BYTES, A_BYTES / 16, t);
        split_lo(st + A_BYTES, st + A_BYTES + C::WB, C::WB / 16, t);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0) arrive_leader<PAIR>(&rdy[s], rank);
    }
    // drain the lo slots (their last commits target this CTA's barriers)
    for (int64_t idx = total > NL ? total - NL : 0; idx < total; ++idx)
      if (idx % NGRP == grp) mbar_wait(&lo_empty[idx % NL], static_cast<uint32_t>(idx / NL) & 1u);
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issue
    if (!PAIR || rank == 0) {
      if constexpr (RESW) mbar_wait(&wres_rdy, 0);
      int s = 0, l = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      for (int64_t tile = cid; tile < g.num_tiles; tile += ncl, ++it) {
        const int buf = static_cast<int>(it & 1);
        mbar_wait(&tempty[buf], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
        fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf * BN);
        for (int c = 0; c < nkc; ++c) {
          mbar_wait(&rdy[s], ph);
          fence_after();
          {
            const uint8_t* st = smem + s * g.stage;
            const uint32_t w_hi = RESW ? smem_addr(smem + g.wres_off + c * 2 * C::WB)
                                       : smem_addr(st + A_BYTES);
            const uint64_t dwh = desc_sw128(w_hi);
            const uint64_t dwl = desc_sw128(w_hi + C::WB);
            const int nks = min(BKC / 8, (a.K - c * BKC + 7) / 8);
            const uint32_t acc0 = c != 0;
            if constexpr (RESW) {
              const uint32_t ta = tmem + TS_BASE + static_cast<uint32_t>(l * 64);
#pragma unroll
              for (int j = 0; j < BKC / 8; ++j) {
                if (j < nks) {   // descriptor start address advances 32 B per k-step
                  mma_ts<C::IDESC>(d, ta + 32 + 8 * j, dwh + 2 * j, acc0 | j);
                  mma_ts<C::IDESC>(d, ta + 8 * j, dwl + 2 * j, 1u);
                  mma_ts<C::IDESC>(d, ta + 8 * j, dwh + 2 * j, 1u);
                }
              }
              commit3<false>(&lo_empty[l]);
            } else {
              const uint64_t dah = desc_sw128(smem_addr(st));
              const uint64_t dal = desc_sw128(smem_addr(smem + g.lo_off + l * A_BYTES));
#pragma unroll
              for (int j = 0; j < BKC / 8; ++j) {
                if (j < nks) {
                  mma_ss<PAIR, C::IDESC>(d, dal + 2 * j, dwh + 2 * j, acc0 | j);
                  mma_ss<PAIR, C::IDESC>(d, dah + 2 * j, dwl + 2 * j, 1u);
                  mma_ss<PAIR, C::IDESC>(d, dah + 2 * j, dwh + 2 * j, 1u);
                }
              }
              commit3<PAIR>(&empty[s]);
              commit3<PAIR>(&lo_empty[l]);
            }
            if (c == nkc - 1) commit3<PAIR>(&tfull[buf]);
          }
          __syncwarp();
          if (++s == rs) { s = 0; ph ^= 1u; }
          if (++l == (RESW ? RT : RL)) l = 0;
        }
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    // warp (q, p): TMEM lane quarter q (the tcgen05.ld access rule), column
    // part p: halves of BN (multiples of 16), or for the GAT score epilogue
    // the first / last ceil(H/2) heads; a part that cannot split runs on p = 0
    const int q = warp & 3;
    const int p = (warp - W_EPI) >> 2;
    float* epi = reinterpret_cast<float*>(smem + g.epi_off);
    float* stage = epi + (warp - W_EPI) * 32 * EPI_LD;
    float* bias_s = epi + NEPI * 32 * EPI_LD + (warp - W_EPI) * BN;
    float* sc_tab = epi + NEPI * (32 * EPI_LD + BN);
    const bool has_bias = a.bias != nullptr;
    int bias_n0 = -1;
    int cbeg = 0, cend = BN;
    if constexpr (SC) {
      const int split = ((a.heads + 1) / 2) * a.head_pitch;
      if (NEPI == 8 && split % 16 == 0 && split < BN) {
        cbeg = p ? split : 0;
        cend = p ? BN : split;
      } else if (p) {
        cend = 0;
      }
      for (int c = threadIdx.x - W_EPI * 32; c < a.N; c += NEPI * 32) {
        const int hh = c / a.head_pitch;
        const int j = c - hh * a.head_pitch;
        const bool live = hh < a.heads && j < a.head_dim;
        sc_tab[c] = live ? __ldg(a.attn + hh * 2 * a.head_dim + j) : 0.0f;
        sc_tab[v2::kScMaxN + c] = live ? __ldg(a.attn + hh * 2 * a.head_dim + a.head_dim + j) : 0.0f;
      }
      asm volatile("bar.sync 2, %0;" ::"r"(NEPI * 32) : "memory");
    } else if constexpr (NEPI == 8) {
      constexpr int HALF_BN = BN / 2;
      if constexpr (HALF_BN % 16 == 0) {
        cbeg = p * HALF_BN;
        cend = cbeg + HALF_BN;
      } else {
        if (p) cend = 0;
      }
    }
    int64_t it = 0;
    for (int64_t tile = cid; tile < g.num_tiles; tile += ncl, ++it) {
      const int buf = static_cast<int>(it & 1);
      const int64_t m0 = (tile / g.n_tiles) * TM + rank * ROWS;
      const int n0 = static_cast<int>(tile % g.n_tiles) * BN;
      if (has_bias && n0 != bias_n0) {   // this warp's copy of the tile's bias (LDS broadcasts)
        __syncwarp();
        for (int i = lane; i < BN; i += 32) bias_s[i] = n0 + i < a.N ? __ldg(a.bias + n0 + i) : 0.f;
        __syncwarp();
        bias_n0 = n0;
      }
      mbar_wait(&tfull[buf], static_cast<uint32_t>(it >> 1) & 1u);
      fence_after();
      const int64_t row_base = m0 + q * 32;
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) +
                             static_cast<uint32_t>(buf * BN);
      const float* bias_g = bias_s;
      v2::ScoreAcc sa{-1, 0.0f, 0.0f};
      if constexpr (SC) {
        int c0 = cbeg;
        if (a.sc_mode == 0 || a.sc_mode == 2) {   // 32-column chunks (1, 3: 16)
#pragma unroll 1
          for (; c0 + 32 <= cend; c0 += 32)
            v2::epi_chunk<32, ACT, SC>(a, tbase + c0, stage, bias_g + c0, has_bias, row_base,
                                       n0 + c0, lane, sc_tab, sa);
        }
#pragma unroll 1
        for (; c0 + 16 <= cend; c0 += 16)
          v2::epi_chunk<16, ACT, SC>(a, tbase + c0, stage, bias_g + c0, has_bias, row_base,
                                     n0 + c0, lane, sc_tab, sa);
        if (cend > cbeg) v2::score_flush(a, sa, row_base + lane);
      } else {
        int c0 = cbeg;
#pragma unroll 1
        for (; c0 + 32 <= cend; c0 += 32)
          v2::epi_chunk<32, ACT, SC>(a, tbase + c0, stage, bias_g + c0, has_bias, row_base,
                                     n0 + c0, lane, sc_tab, sa);
        if (c0 + 16 <= cend)
          v2::epi_chunk<16, ACT, SC>(a, tbase + c0, stage, bias_g + c0, has_bias, row_base,
                                     n0 + c0, lane, sc_tab, sa);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader<PAIR>(&tempty[buf], rank);
    }
  }
  fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  if (warp == W_MMA) {
    fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
  }
}

// ---------------------------------------------------------------- host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D fp32 map over a row-major [rows x cols] matrix with row pitch ld
// (elements); box = 32 columns (128 B) x box_rows rows, 128 B swizzle, zero fill
int make_map(CUtensorMap* m, const float* base, int64_t rows, int cols, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("linear: cuTensorMapEncodeTiled unavailable from the driver");
    return GLINT_ECUDA;
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BKC), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("linear: cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%d ld=%lld", static_cast<int>(r),
              static_cast<long long>(rows), cols, static_cast<long long>(ld));
    return GLINT_ECUDA;
  }
  return GLINT_OK;
}

template <int BN, int ACT, bool SC, bool PAIR, bool RESW>
int launch_v3(TcArgs a, cudaStream_t s) {
  using C = Cfg3<BN, PAIR>;
  V3Args g{};
  g.nkc = static_cast<int>(ceil_div(a.K, BKC));
  const Plan3 p = plan3<BN, PAIR, RESW, SC>(g.nkc);
  if (p.rs < 2) return GLINT_EUNSUPPORTED;
  g.rs = p.rs;
  g.stage = p.stage;
  g.lo_off = p.lo_off;
  g.wres_off = p.wres_off;
  g.epi_off = p.epi_off;
  g.n_tiles = static_cast<int>(ceil_div(a.N, BN));
  {
    const int knob = tuning(GLINT_TUNE_GEMM_PF);   // 0 default (1 tile ahead), -1 off, k > 0
    g.pf_tiles = knob < 0 ? 0 : knob == 0 ? 1 : knob;
  }
  constexpr int TM = PAIR ? 2 * ROWS : ROWS;
  g.num_tiles = ceil_div(a.M, TM) * g.n_tiles;
  CUtensorMap ma, mw;
  int rc = make_map(&ma, a.A, a.M, a.K, a.lda, ROWS);
  if (rc) return rc;
  rc = make_map(&mw, a.W, a.N, a.K, a.ldw, RESW ? BN : C::BNH);
  if (rc) return rc;
  auto kern = gemm_v3_kernel<BN, ACT, SC, PAIR, RESW>;
  static PerDeviceOnce configured;
  if (configured.needed()) {
    GLINT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_CAP));
    configured.mark();
  }
  const int sms = sm_count();
  int64_t ctas = PAIR ? std::min<int64_t>(g.num_tiles, sms / 2) * 2
                      : std::min<int64_t>(g.num_tiles, sms);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(ctas));
  cfg.blockDim = dim3(threads3<BN, SC>());
  cfg.dynamicSmemBytes = static_cast<size_t>(p.smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mw, a, g);
  if (e != cudaSuccess) {
    set_error("linear_3xtf32 (v3) launch failed: %s", cudaGetErrorString(e));
    return GLINT_ECUDA;
  }
  return launch_status("linear_3xtf32_v3");
}

template <int BN, bool SC, bool PAIR, bool RESW>
int launch_v3_act(const TcArgs& a, int act, cudaStream_t s) {
  if constexpr (SC) {
    return launch_v3<BN, GLINT_ACT_NONE, true, PAIR, RESW>(a, s);
  } else {
    if (act == GLINT_ACT_RELU) return launch_v3<BN, GLINT_ACT_RELU, false, PAIR, RESW>(a, s);
    if (act == GLINT_ACT_LEAKY_RELU) return launch_v3<BN, GLINT_ACT_LEAKY_RELU, false, PAIR, RESW>(a, s);
    return launch_v3<BN, GLINT_ACT_NONE, false, PAIR, RESW>(a, s);
  }
}

// Shape dispatch.  N <= 64: single CTAs with W resident (K <= 512);
// otherwise CTA pairs with BN = N rounded up to 64 (<= 256; wider N tiles by
// 256).  Score epilogues need every head in one column tile (N <= 256).
// Returns GLINT_EUNSUPPORTED when no v3 shape applies (caller uses v2).
template <bool SC>
int dispatch_v3(const TcArgs& a, int act, cudaStream_t s) {
  if (a.a_rows) return GLINT_EUNSUPPORTED;   // row-gathered A: no tensor map (v2 path)
  // with the per-column score walk (GLINT_TUNE_GAT_EPI 1) short-K score
  // projections are epilogue-bound and v2's 128-row tiles were faster there;
  // the chunked score path runs them on v3 (100 -> 4x64: 0.99 vs 1.75 ms,
  // profiles/r02_gemm_sc_modes.jsonl)
  if (SC && a.K < 192 && a.sc_mode == 1) return GLINT_EUNSUPPORTED;
  if (a.N <= 64 && a.K <= 512) {
    // resident W: falls through to the pair kernel when W raw + lo leave
    // fewer than 2 A stages of shared memory (e.g. N = 64, K = 512)
    int rc;
    if (a.N <= 16) rc = launch_v3_act<16, SC, false, true>(a, act, s);
    else if (a.N <= 32) rc = launch_v3_act<32, SC, false, true>(a, act, s);
    else if (a.N <= 48) rc = launch_v3_act<48, SC, false, true>(a, act, s);
    else rc = launch_v3_act<64, SC, false, true>(a, act, s);
    if (rc != GLINT_EUNSUPPORTED) return rc;
  }
  if (a.N <= 64) return launch_v3_act<64, SC, true, false>(a, act, s);
  if (a.N <= 128) return launch_v3_act<128, SC, true, false>(a, act, s);
  if (a.N <= 192) return launch_v3_act<192, SC, true, false>(a, act, s);
  if (SC && a.N > 256) return GLINT_EUNSUPPORTED;
  return launch_v3_act<256, SC, true, false>(a, act, s);
}

}  // namespace v3

}  // namespace

// Z = A W_pad^T (3xTF32) with s_src / s_dst computed in the epilogue; returns
// GLINT_EUNSUPPORTED when the shape does not fit (the caller falls back).
int launch_gat_project_3xtf32(int64_t M, int heads, int head_dim, int head_pitch, int K,
                              const float* A, int64_t lda, const int64_t* a_rows, const float* W,
                              int64_t ldw, const float* attn, float* Z, int64_t ldz, float* s_src,
                              float* s_dst, cudaStream_t s) {
  const int N = heads * head_pitch;
  const bool vec = (lda % 4 == 0) && (ldw % 4 == 0) && (K % 4 == 0) && aligned16(A) && aligned16(W);
  if (!vec || N > v2::kScMaxN || tuning(GLINT_TUNE_GEMM_V1) != 0) return GLINT_EUNSUPPORTED;
  TcArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.lda = lda;
  a.a_rows = a_rows;
  a.W = W;
  a.ldw = ldw;
  a.C = Z;
  a.ldc = ldz;
  a.c_vec4 = (ldz % 4 == 0) && aligned16(Z);
  a.attn = attn;
  a.s_src = s_src;
  a.s_dst = s_dst;
  a.heads = heads;
  a.head_dim = head_dim;
  a.head_pitch = head_pitch;
  a.sc_mode = tuning(GLINT_TUNE_GAT_EPI);
  if (tuning(GLINT_TUNE_GEMM_V3) == 0) {
    const int rc = v3::dispatch_v3<true>(a, GLINT_ACT_NONE, s);
    if (rc != GLINT_EUNSUPPORTED) return rc;
  }
  return v2::launch_v2_scores(a, s);
}

int launch_linear_3xtf32(int64_t M, int N, int K, const float* A, int64_t lda,
                         const int64_t* a_rows, const float* W, int64_t ldw, const float* bias,
                         int act, float* C, int64_t ldc, cudaStream_t s) {
  TcArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.lda = lda;
  a.a_rows = a_rows;
  a.W = W;
  a.ldw = ldw;
  a.bias = bias;
  a.C = C;
  a.ldc = ldc;
  a.c_vec4 = (ldc % 4 == 0) && aligned16(C);
  a.raw_hi = tuning(GLINT_TUNE_GEMM_RAWHI) != 0;
  a.mma_only = tuning(GLINT_TUNE_GEMM_PROF) == 2;
  a.skip_lo = tuning(GLINT_TUNE_GEMM_PROF) == 3;
  a.prof = nullptr;
  if (tuning(GLINT_TUNE_GEMM_PROF) == 1) {
    void* p = nullptr;
    GLINT_CUDA(cudaGetSymbolAddress(&p, g_gemm_prof));
    a.prof = static_cast<unsigned long long*>(p);
  }
  // 16-byte pitched rows: v3's tensor maps cover exactly K columns (the box
  // beyond K is zero-filled by the TMA), so K need not be a multiple of 4 there;
  // v2/v1's vector loads would read the pad columns, so they also need K % 4 == 0
  const bool pitched = (lda % 4 == 0) && (ldw % 4 == 0) && aligned16(A) && aligned16(W);
  const bool vec = pitched && (K % 4 == 0);
  // v3 (tensor-map TMA, CTA pairs / resident W), then v2 (row-gathered A),
  // unless the knobs ask for an older kernel
  if (pitched && tuning(GLINT_TUNE_GEMM_V1) == 0 && tuning(GLINT_TUNE_GEMM_V3) == 0) {
    const int rc = v3::dispatch_v3<false>(a, act, s);
    if (rc != GLINT_EUNSUPPORTED) return rc;
  }
  if (vec && tuning(GLINT_TUNE_GEMM_V1) == 0) return v2::launch_v2_bn(a, act, s);
  return vec ? launch_bn<true>(a, act, s) : launch_bn<false>(a, act, s);
}

}  // namespace glint

extern "C" int glint_debug_counters(int which, uint64_t* host_out, int n, int reset) {
  GLINT_REQUIRE((which == 0 || which == 1) && n >= 0 && n <= 8 && (host_out || n == 0),
                "debug_counters: bad argument");
  if (which == 1) return glint::fused_debug_counters(host_out, n, reset);
  if (n) GLINT_CUDA(cudaMemcpyFromSymbol(host_out, glint::g_gemm_prof, n * sizeof(uint64_t)));
  if (reset) {
    const unsigned long long zeros[8] = {0};
    GLINT_CUDA(cudaMemcpyToSymbol(glint::g_gemm_prof, zeros, sizeof(zeros)));
  }
  return GLINT_OK;
}
