// K5 per-row operators and row copies.
// Reference: kernels.py:206-231 (elementwise), kernels.py:234-239 (concat),
// storage.py:224-246 (EmbeddingStore gather/scatter), executor.py:351-384
// (target restriction of input-domain operands through target_pos).
#include "common.cuh"

namespace glint {
namespace {

constexpr int kMaxOperands = 8;

struct EwArgs {
  int kind;
  int64_t n_rows;
  int dim;
  int n_in;
  const float* in[kMaxOperands];
  int64_t ld[kMaxOperands];
  const int64_t* rows[kMaxOperands];
  float* out;
  int64_t ld_out;
};

__device__ __forceinline__ const float* operand_row(const EwArgs& a, int k, int64_t i) {
  const int64_t r = a.rows[k] ? a.rows[k][i] : i;
  return a.in[k] + r * a.ld[k];
}

__global__ void ew_pointwise_kernel(EwArgs a) {
  const int64_t total = a.n_rows * a.dim;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / a.dim;
    const int c = static_cast<int>(t - i * a.dim);
    float v = operand_row(a, 0, i)[c];
    switch (a.kind) {
      case GLINT_EW_RELU:
        v = (v > 0.0f || v != v) ? v : 0.0f;  // np.maximum(x, 0): -0.0 -> +0.0, NaN kept
        break;
      case GLINT_EW_LEAKY_RELU:
        v = v >= 0.0f ? v : __fmul_rn(0.2f, v);
        break;
      case GLINT_EW_ADD:
        for (int k = 1; k < a.n_in; ++k) v = __fadd_rn(v, operand_row(a, k, i)[c]);
        break;
      default:
        break;  // DropoutIdentity: copy
    }
    a.out[i * a.ld_out + c] = v;
  }
}

// The pointwise kinds by rows and 16-byte chunks: LPR lanes per row, lane g
// takes chunks g, g+LPR, ...  Used when every operand row and the output row
// are 16-byte aligned with room for the last chunk (ld >= 4 ceil(dim/4)): the
// last chunk may read pad columns, whose results are never stored.  Same
// per-element arithmetic (and Add order) as ew_pointwise_kernel.
__device__ __forceinline__ float ew_unary(int kind, float v) {
  if (kind == GLINT_EW_RELU) return (v > 0.0f || v != v) ? v : 0.0f;
  if (kind == GLINT_EW_LEAKY_RELU) return v >= 0.0f ? v : __fmul_rn(0.2f, v);
  return v;
}

template <int LPR>
__global__ void ew_rows_kernel(EwArgs a, int c4) {
  constexpr int G = 32 / LPR;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t i = warp * G + lane / LPR;
  if (i >= a.n_rows) return;
  for (int c = lane % LPR; c < c4; c += LPR) {
    const int col = 4 * c;
    float4 v = ldg_f4(operand_row(a, 0, i) + col);
    if (a.kind == GLINT_EW_ADD) {
      for (int k = 1; k < a.n_in; ++k) {
        const float4 w = ldg_f4(operand_row(a, k, i) + col);
        v.x = __fadd_rn(v.x, w.x);
        v.y = __fadd_rn(v.y, w.y);
        v.z = __fadd_rn(v.z, w.z);
        v.w = __fadd_rn(v.w, w.w);
      }
    } else {
      v.x = ew_unary(a.kind, v.x);
      v.y = ew_unary(a.kind, v.y);
      v.z = ew_unary(a.kind, v.z);
      v.w = ew_unary(a.kind, v.w);
    }
    float* o = a.out + i * a.ld_out + col;
    if (col + 4 <= a.dim) {
      *reinterpret_cast<float4*>(o) = v;
    } else {
      const float t[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; col + j < a.dim; ++j) o[j] = t[j];
    }
  }
}

// Norm: x / sqrt(sum(x*x) + 1e-12), one warp per row (kernels.py:227-230).
__global__ void ew_norm_kernel(EwArgs a) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= a.n_rows) return;
  const float* x = operand_row(a, 0, i);
  float ss = 0.0f;
  for (int c = lane; c < a.dim; c += 32) ss = __fadd_rn(ss, __fmul_rn(x[c], x[c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  const float den = __fsqrt_rn(__fadd_rn(ss, 1e-12f));
  for (int c = lane; c < a.dim; c += 32) a.out[i * a.ld_out + c] = __fdiv_rn(x[c], den);
}

template <bool VEC4>
__global__ void copy_rows_kernel(int64_t n_rows, int dim, const float* __restrict__ src,
                                 int64_t ld_src, const int64_t* __restrict__ src_rows,
                                 float* __restrict__ dst, int64_t ld_dst,
                                 const int64_t* __restrict__ dst_rows) {
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_rows; i += nwarps) {
    const float* s = src + (src_rows ? src_rows[i] : i) * ld_src;
    float* d = dst + (dst_rows ? dst_rows[i] : i) * ld_dst;
    if constexpr (VEC4) {
      const int d4 = dim >> 2;
      for (int c = lane; c < d4; c += 32)
        reinterpret_cast<float4*>(d)[c] = ldg_f4(s + 4 * c);
      for (int c = 4 * d4 + lane; c < dim; c += 32) d[c] = s[c];
    } else {
      for (int c = lane; c < dim; c += 32) d[c] = s[c];
    }
  }
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" {

int glint_elementwise_f32(int32_t kind, int64_t n_rows, int32_t dim, int32_t n_inputs,
                          const float* const* inputs, const int64_t* ld_inputs,
                          const int64_t* const* input_rows, float* out, int64_t ld_out,
                          glint_stream_t stream) {
  GLINT_REQUIRE(kind >= GLINT_EW_RELU && kind <= GLINT_EW_DROPOUT_IDENTITY,
                "elementwise: unknown kind %d", kind);
  GLINT_REQUIRE(n_rows >= 0 && dim >= 1, "elementwise: bad shape");
  GLINT_REQUIRE(n_inputs >= 1 && n_inputs <= kMaxOperands, "elementwise: 1..%d operands", kMaxOperands);
  GLINT_REQUIRE(kind == GLINT_EW_ADD ? n_inputs >= 2 : n_inputs == 1,
                kind == GLINT_EW_ADD ? "Add needs at least two operands"
                                     : "elementwise: this kind takes exactly one operand");
  GLINT_REQUIRE(inputs && ld_inputs && out && ld_out >= dim, "elementwise: null argument");
  if (n_rows == 0) return GLINT_OK;
  EwArgs a{};
  a.kind = kind;
  a.n_rows = n_rows;
  a.dim = dim;
  a.n_in = n_inputs;
  for (int k = 0; k < n_inputs; ++k) {
    GLINT_REQUIRE(inputs[k] && ld_inputs[k] >= dim, "elementwise: operand %d invalid", k);
    a.in[k] = inputs[k];
    a.ld[k] = ld_inputs[k];
    a.rows[k] = input_rows ? input_rows[k] : nullptr;
  }
  a.out = out;
  a.ld_out = ld_out;
  cudaStream_t s = as_stream(stream);
  if (kind == GLINT_EW_NORM) {
    ew_norm_kernel<<<static_cast<unsigned>(ceil_div(n_rows * 32, 256)), 256, 0, s>>>(a);
  } else {
    const int c4 = static_cast<int>(ceil_div(dim, 4));
    bool vec = ld_out % 4 == 0 && aligned16(out);
    for (int k = 0; k < n_inputs; ++k)
      vec = vec && a.ld[k] % 4 == 0 && a.ld[k] >= 4 * c4 && aligned16(a.in[k]);
    if (vec) {
      const int lpr = c4 <= 4 ? 4 : c4 <= 8 ? 8 : c4 <= 16 ? 16 : 32;
      const int64_t grid = ceil_div(ceil_div(n_rows, 32 / lpr) * 32, 256);
      if (grid > 0x7fffffffLL) {
        set_error("elementwise: grid too large");
        return GLINT_EINVAL;
      }
      const unsigned g = static_cast<unsigned>(grid);
      if (lpr == 4) ew_rows_kernel<4><<<g, 256, 0, s>>>(a, c4);
      else if (lpr == 8) ew_rows_kernel<8><<<g, 256, 0, s>>>(a, c4);
      else if (lpr == 16) ew_rows_kernel<16><<<g, 256, 0, s>>>(a, c4);
      else ew_rows_kernel<32><<<g, 256, 0, s>>>(a, c4);
    } else {
      const int64_t total = n_rows * dim;
      const int64_t grid = std::min<int64_t>(ceil_div(total, 256), static_cast<int64_t>(sm_count()) * 16);
      ew_pointwise_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(a);
    }
  }
  return launch_status("elementwise");
}

int glint_copy_rows_f32(int64_t n_rows, int32_t dim, const float* src, int64_t ld_src,
                        const int64_t* src_rows, float* dst, int64_t ld_dst,
                        const int64_t* dst_rows, glint_stream_t stream) {
  GLINT_REQUIRE(n_rows >= 0 && dim >= 0, "copy_rows: bad shape");
  if (n_rows == 0 || dim == 0) return GLINT_OK;
  GLINT_REQUIRE(src && dst && ld_src >= dim && ld_dst >= dim, "copy_rows: bad argument");
  cudaStream_t s = as_stream(stream);
  const int64_t grid = std::min<int64_t>(ceil_div(n_rows * 32, 256), static_cast<int64_t>(sm_count()) * 32);
  const bool vec4 = ld_src % 4 == 0 && ld_dst % 4 == 0 && aligned16(src) && aligned16(dst);
  if (vec4)
    copy_rows_kernel<true><<<static_cast<unsigned>(grid), 256, 0, s>>>(n_rows, dim, src, ld_src, src_rows, dst, ld_dst, dst_rows);
  else
    copy_rows_kernel<false><<<static_cast<unsigned>(grid), 256, 0, s>>>(n_rows, dim, src, ld_src, src_rows, dst, ld_dst, dst_rows);
  return launch_status("copy_rows");
}

}  // extern "C"
