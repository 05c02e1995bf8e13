// K2 on the 5th-generation tensor cores: C = act(A W^T + b) in split-TF32
// ("3xTF32") with tcgen05.mma kind::tf32, fp32 accumulators in TMEM.
//
// Reference op: kernels.py:95-107 (linear, fp32 einsum).  Plain TF32 misses
// the rel-L2 1e-4 end-to-end bar (3.4e-4), so every operand is
// split into a TF32-exact high part and a residual, x = hi + lo with
// hi = x with the low 13 mantissa bits cleared and lo = x - hi (exact in fp32),
// and the product is hi*hi + hi*lo + lo*hi (lo*lo ~ 2^-22 relative is dropped).
// Measured error of the scheme ~1e-7 rel-L2.
//
// Tiling: one CTA (4 warps) per 128-row M tile x BN columns; K advances in
// 32-element blocks through a 2-stage shared-memory ring.  Every thread loads
// A / W with 128-bit loads, splits hi/lo in registers and writes both parts
// into the canonical no-swizzle K-major UMMA layout (8-row x 16-byte core
// matrices: LBO = 128 B along K, SBO = 1024 B between 8-row groups).  One
// thread issues 3 x (BK/8) tcgen05.mma (M=128, N=BN, K=8) per block and
// commits them to the stage's mbarrier, which gates reuse of that stage.  The
// epilogue reads the accumulator with tcgen05.ld (warp w owns TMEM lanes
// 32w..32w+31 = tile rows), adds bias, applies the activation and stores.
//
// Row invariance (kernels.py:1-14): each output row depends only on its own
// A row and W, with a fixed k order, so any batching of rows gives the same
// bytes.
#include "common.cuh"

namespace glint {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int kTcThreads = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tcgen05 shared-memory matrix descriptor, SWIZZLE_NONE, K-major.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                             // base offset 0, layout type 0 (no swizzle)
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

template <int BN>
struct TmemCols {
  static constexpr uint32_t value = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
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
};

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

// Canonical no-swizzle K-major offset of (row r, 16-byte chunk c) in a tile
// whose K extent is BK: core matrix = 8 rows x 16 B (128 B), K-adjacent core
// matrices 128 B apart (LBO), 8-row groups BK*32 B apart (SBO).
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return static_cast<uint32_t>((r & 7) * 16 + c * 128 + (r >> 3) * (BK / 4) * 128);
}

template <int BN, bool VEC, int ACT>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_3xtf32_kernel(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_slot;
  constexpr int A_BYTES = BM * BK * 4;
  constexpr int W_BYTES = BN * BK * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * W_BYTES;
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  constexpr uint32_t SBO = (BK / 4) * 128;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                             (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(BM >> 4) << 24);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :
                 : "r"(smem_addr(&tmem_slot)), "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_slot;

  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int nkb = (a.K + BK - 1) / BK;

  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    uint8_t* a_hi = smem + s * STAGE;
    uint8_t* a_lo = a_hi + A_BYTES;
    uint8_t* w_hi = a_lo + A_BYTES;
    uint8_t* w_lo = w_hi + W_BYTES;
    if (kb >= 2) mbar_wait(&bars[s], static_cast<uint32_t>(((kb >> 1) - 1) & 1));
    const int kbase = kb * BK;
    // A tile: warp w fills 8-row groups w, w+4, w+8, w+12; lane -> (row in group, chunk)
#pragma unroll
    for (int i = 0; i < BM / 32; ++i) {
      const int r = (warp + 4 * i) * 8 + (lane & 7);
      const int64_t row = m0 + r;
      const float* src = nullptr;
      if (row < a.M) src = a.A + (a.a_rows ? a.a_rows[row] : row) * a.lda;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = (lane >> 3) + 4 * h;
        const float4 v = src ? load4<VEC>(src, kbase + 4 * c, a.K) : make_float4(0.f, 0.f, 0.f, 0.f);
        split_store(a_hi, a_lo, tile_off(r, c), v);
      }
    }
    // W tile: BN rows
    for (int gidx = warp; gidx < BN / 8; gidx += 4) {
      const int r = gidx * 8 + (lane & 7);
      const int n = n0 + r;
      const float* src = n < a.N ? a.W + static_cast<int64_t>(n) * a.ldw : nullptr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = (lane >> 3) + 4 * h;
        const float4 v = src ? load4<VEC>(src, kbase + 4 * c, a.K) : make_float4(0.f, 0.f, 0.f, 0.f);
        split_store(w_hi, w_lo, tile_off(r, c), v);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_after();
      const uint32_t ah = smem_addr(a_hi), al = smem_addr(a_lo);
      const uint32_t wh = smem_addr(w_hi), wl = smem_addr(w_lo);
#pragma unroll
      for (int j = 0; j < BK / 8; ++j) {
        const uint32_t step = j * 256;  // 8 tf32 along K = two 16-byte core matrices
        const uint64_t d_ah = umma_desc(ah + step, 128, SBO);
        const uint64_t d_al = umma_desc(al + step, 128, SBO);
        const uint64_t d_wh = umma_desc(wh + step, 128, SBO);
        const uint64_t d_wl = umma_desc(wl + step, 128, SBO);
        mma_tf32(tmem, d_al, d_wh, IDESC, (kb | j) != 0);
        mma_tf32(tmem, d_ah, d_wl, IDESC, 1);
        mma_tf32(tmem, d_ah, d_wh, IDESC, 1);
      }
      mma_commit(&bars[s]);
    }
  }
  const int last = nkb - 1;
  mbar_wait(&bars[last & 1], static_cast<uint32_t>((last >> 1) & 1));
  fence_after();

  // epilogue: warp w <-> TMEM lanes 32w.., thread <-> one tile row
  const int64_t row = m0 + warp * 32 + lane;
  const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(lane_addr + c0, v);
    if (row < a.M) {
      float* dst = a.C + row * a.ldc;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = n0 + c0 + i;
        if (col < a.N) {
          float x = v[i];
          if (a.bias) x = __fadd_rn(x, a.bias[col]);
          if (ACT == GLINT_ACT_RELU) x = (x > 0.0f || x != x) ? x : 0.0f;
          if (ACT == GLINT_ACT_LEAKY_RELU) x = x >= 0.0f ? x : __fmul_rn(0.2f, x);
          dst[col] = x;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" : : "r"(tmem), "r"(TCOLS));
  }
}

template <int BN, bool VEC, int ACT>
int launch_tc(const TcArgs& a, cudaStream_t s) {
  constexpr int smem_bytes = 2 * (2 * BM * BK * 4 + 2 * BN * BK * 4);
  static bool configured = false;
  if (!configured) {
    GLINT_CUDA(cudaFuncSetAttribute(gemm_3xtf32_kernel<BN, VEC, ACT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    configured = true;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(a.M, BM)), static_cast<unsigned>(ceil_div(a.N, BN)));
  gemm_3xtf32_kernel<BN, VEC, ACT><<<grid, kTcThreads, smem_bytes, s>>>(a);
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
  return launch_act<256, VEC>(a, act, s);
}

}  // namespace

int launch_linear_3xtf32(int64_t M, int N, int K, const float* A, int64_t lda,
                         const int64_t* a_rows, const float* W, int64_t ldw, const float* bias,
                         int act, float* C, int64_t ldc, cudaStream_t s) {
  GLINT_REQUIRE(ceil_div(M, BM) < (1LL << 31), "linear_3xtf32: M too large");
  TcArgs a{M, N, K, A, lda, a_rows, W, ldw, bias, C, ldc};
  const bool vec = (lda % 4 == 0) && (ldw % 4 == 0) && (K % 4 == 0) && aligned16(A) && aligned16(W);
  return vec ? launch_bn<true>(a, act, s) : launch_bn<false>(a, act, s);
}

}  // namespace glint
