// K2 dense per-layer transform C = act(A W^T + b) and the GAT score epilogue.
//
// Reference: kernels.py:95-107 (linear: einsum "ij,kj->ik" + bias) and
// kernels.py:188-189 (s_src / s_dst = einsum "ij,j->i").
//
// GLINT_PREC_FP32: CUDA-core fp32 with one FMA chain per output element over
// k = 0..K-1 in fixed order -> every row is independent of M and of its
// position (batch invariance, kernels.py:1-14).
// GLINT_PREC_3XTF32: tcgen05 tensor-core path (gemm_tcgen05.cu).
#include <algorithm>

#include "common.cuh"

namespace glint {

int launch_linear_3xtf32(int64_t M, int N, int K, const float* A, int64_t lda,
                         const int64_t* a_rows, const float* W, int64_t ldw, const float* bias,
                         int act, float* C, int64_t ldc, cudaStream_t s);
int launch_gat_project_3xtf32(int64_t M, int heads, int head_dim, int head_pitch, int K,
                              const float* A, int64_t lda, const int64_t* a_rows, const float* W,
                              int64_t ldw, const float* attn, float* Z, int64_t ldz, float* s_src,
                              float* s_dst, cudaStream_t s);

namespace {

constexpr int BM = 128, BN = 64, BK = 16, TM = 8, TN = 4;

template <int ACT>
__device__ __forceinline__ float activate(float v) {
  if constexpr (ACT == GLINT_ACT_RELU) return (v > 0.0f || v != v) ? v : 0.0f;
  if constexpr (ACT == GLINT_ACT_LEAKY_RELU) return v >= 0.0f ? v : __fmul_rn(0.2f, v);
  return v;
}

template <int ACT>
__global__ void __launch_bounds__(256) sgemm_nt_kernel(int64_t M, int N, int K,
                                                       const float* __restrict__ A, int64_t lda,
                                                       const int64_t* __restrict__ a_rows,
                                                       const float* __restrict__ W, int64_t ldw,
                                                       const float* __restrict__ bias,
                                                       float* __restrict__ C, int64_t ldc) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Ws[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15;
  const int ty = tid >> 4;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;

  const int a_row = tid >> 1;
  const int a_k = (tid & 1) * 8;
  const int64_t grow = m0 + a_row;
  const bool a_ok = grow < M;
  const float* a_ptr = a_ok ? A + (a_rows ? a_rows[grow] : grow) * lda : A;
  const int w_row = tid >> 2;
  const int w_k = (tid & 3) * 4;
  const bool w_ok = n0 + w_row < N;
  const float* w_ptr = W + static_cast<int64_t>(w_ok ? n0 + w_row : 0) * ldw;

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = k0 + a_k + i;
      As[a_k + i][a_row] = (a_ok && k < K) ? __ldg(a_ptr + k) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = k0 + w_k + i;
      Ws[w_k + i][w_row] = (w_ok && k < K) ? __ldg(w_ptr + k) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Ws[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = m0 + ty * TM + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = n0 + tx * TN + j;
      if (col < N) {
        float v = acc[i][j];
        if (bias) v = __fadd_rn(v, bias[col]);
        C[row * ldc + col] = activate<ACT>(v);
      }
    }
  }
}

// s_src / s_dst: one warp per row, lanes over the head's columns.
__global__ void gat_scores_kernel(int64_t M, int heads, int head_dim, int head_pitch,
                                  const float* __restrict__ Z, int64_t ldz,
                                  const float* __restrict__ attn, float* __restrict__ s_src,
                                  float* __restrict__ s_dst) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* z = Z + row * ldz;
  for (int h = 0; h < heads; ++h) {
    const float* a = attn + static_cast<int64_t>(h) * 2 * head_dim;
    float ps = 0.0f, pd = 0.0f;
    for (int j = lane; j < head_dim; j += 32) {
      const float zv = z[h * head_pitch + j];
      ps = fmaf(zv, a[j], ps);
      pd = fmaf(zv, a[head_dim + j], pd);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ps += __shfl_xor_sync(0xffffffffu, ps, o);
      pd += __shfl_xor_sync(0xffffffffu, pd, o);
    }
    if (lane == 0) {
      s_src[row * heads + h] = ps;
      s_dst[row * heads + h] = pd;
    }
  }
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

int glint_linear_f32(int64_t M, int32_t N, int32_t K, const float* A, int64_t lda,
                     const int64_t* a_rows, const float* W, int64_t ldw, const float* bias,
                     int32_t act, float* C, int64_t ldc, int32_t precision,
                     glint_stream_t stream) {
  GLINT_REQUIRE(M >= 0 && N >= 1 && K >= 1, "linear: bad shape M=%lld N=%d K=%d",
                static_cast<long long>(M), N, K);
  if (M == 0) return GLINT_OK;
  GLINT_REQUIRE(A && W && C, "linear: null A/W/C");
  GLINT_REQUIRE(lda >= K && ldw >= K && ldc >= N, "linear: leading dimension too small");
  GLINT_REQUIRE(act >= GLINT_ACT_NONE && act <= GLINT_ACT_LEAKY_RELU, "linear: bad activation %d", act);
  cudaStream_t s = as_stream(stream);
  if (precision == GLINT_PREC_3XTF32) {
    return launch_linear_3xtf32(M, N, K, A, lda, a_rows, W, ldw, bias, act, C, ldc, s);
  }
  GLINT_REQUIRE(precision == GLINT_PREC_FP32, "linear: unknown precision %d", precision);
  const int64_t gx = ceil_div(M, BM);
  GLINT_REQUIRE(gx < (1LL << 31), "linear: M too large");
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(ceil_div(N, BN)));
  switch (act) {
    case GLINT_ACT_RELU:
      sgemm_nt_kernel<GLINT_ACT_RELU><<<grid, 256, 0, s>>>(M, N, K, A, lda, a_rows, W, ldw, bias, C, ldc);
      break;
    case GLINT_ACT_LEAKY_RELU:
      sgemm_nt_kernel<GLINT_ACT_LEAKY_RELU><<<grid, 256, 0, s>>>(M, N, K, A, lda, a_rows, W, ldw, bias, C, ldc);
      break;
    default:
      sgemm_nt_kernel<GLINT_ACT_NONE><<<grid, 256, 0, s>>>(M, N, K, A, lda, a_rows, W, ldw, bias, C, ldc);
  }
  return launch_status("linear_f32");
}

int glint_gat_scores_f32(int64_t M, int32_t heads, int32_t head_dim, int32_t head_pitch,
                         const float* Z, int64_t ldz, const float* attn, float* s_src,
                         float* s_dst, glint_stream_t stream) {
  GLINT_REQUIRE(M >= 0 && heads >= 1 && head_dim >= 1 && head_pitch >= head_dim,
                "gat_scores: bad shape");
  if (M == 0) return GLINT_OK;
  GLINT_REQUIRE(Z && attn && s_src && s_dst, "gat_scores: null argument");
  GLINT_REQUIRE(ldz >= static_cast<int64_t>(heads) * head_pitch, "gat_scores: ldz too small");
  const int64_t grid = ceil_div(M * 32, 256);
  gat_scores_kernel<<<static_cast<unsigned>(grid), 256, 0, as_stream(stream)>>>(
      M, heads, head_dim, head_pitch, Z, ldz, attn, s_src, s_dst);
  return launch_status("gat_scores");
}

int glint_gat_project_f32(int64_t M, int32_t heads, int32_t head_dim, int32_t head_pitch,
                          int32_t K, const float* A, int64_t lda, const int64_t* a_rows,
                          const float* W_pad, int64_t ldw, const float* attn, float* Z,
                          int64_t ldz, float* s_src, float* s_dst, int32_t precision,
                          glint_stream_t stream) {
  GLINT_REQUIRE(M >= 0 && heads >= 1 && head_dim >= 1 && head_pitch >= head_dim && K >= 1,
                "gat_project: bad shape");
  if (M == 0) return GLINT_OK;
  GLINT_REQUIRE(A && W_pad && attn && Z && s_src && s_dst, "gat_project: null argument");
  const int N = heads * head_pitch;
  GLINT_REQUIRE(lda >= K && ldw >= K && ldz >= N, "gat_project: leading dimension too small");
  cudaStream_t s = as_stream(stream);
  // GLINT_TUNE_GAT_PROJ: 0 scores in the GEMM epilogue, 1 GEMM then the score
  // kernel, 2 the latter for short K (< 192) only
  const int split = tuning(GLINT_TUNE_GAT_PROJ);
  if (precision == GLINT_PREC_3XTF32 && split != 1 && !(split == 2 && K < 192)) {
    const int rc = launch_gat_project_3xtf32(M, heads, head_dim, head_pitch, K, A, lda, a_rows,
                                             W_pad, ldw, attn, Z, ldz, s_src, s_dst, s);
    if (rc != GLINT_EUNSUPPORTED) return rc;
  }
  const int rc = glint_linear_f32(M, N, K, A, lda, a_rows, W_pad, ldw, nullptr, GLINT_ACT_NONE, Z,
                                  ldz, precision, stream);
  if (rc) return rc;
  return glint_gat_scores_f32(M, heads, head_dim, head_pitch, Z, ldz, attn, s_src, s_dst, stream);
}

}  // extern "C"
