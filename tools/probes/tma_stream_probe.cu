// TMA streaming probe: DRAM read throughput of cp.async.bulk.tensor for the
// box shapes a K2 A-operand loader can use, on a [M x K] fp32 row-major
// matrix larger than L2.  Each persistent CTA (one per SM) streams its own
// row blocks through RS shared-memory stages; one thread issues, waits, and
// re-issues (no compute), so the number is the copy engine's rate.
//   mode 0: 2-D box {32 fp32, 128 rows}, SWIZZLE_128B   (v3 today: 128 B per row)
//   mode 1: 2-D box {32 fp32, 256 rows}, SWIZZLE_128B
//   mode 2: 3-D box {32, 8 chunks, 16 rows} of a (k_in, chunk, row) view,
//           SWIZZLE_128B: 16 full 1 KB rows = 16 KB contiguous per box
//   mode 3: 2-D box {256 fp32, 16 rows}, no swizzle (16 KB contiguous)
//   mode 4: plain cp.async.bulk (1-D) of 16 KB contiguous
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_stream_probe tma_stream_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int K = 256;
constexpr int STAGE = 16384;

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32, 1) stream(const __grid_constant__ CUtensorMap map, const float* base,
                                                int mode, int rs, int64_t units, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < rs; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int bytes = mode == 1 ? 2 * STAGE : STAGE;
  // unit u = one box; CTA b takes units b, b + grid, ...
  auto issue = [&](int64_t u, int s) {
    uint8_t* dst = smem + s * bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(sa(&full[s])), "r"(bytes) : "memory");
    const uint64_t m = reinterpret_cast<uint64_t>(&map);
    if (mode == 0) {   // unit = (row block of 128, chunk)
      int c = static_cast<int>(u % 8), r = static_cast<int>(u / 8) * 128;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(dst)), "l"(m), "r"(c * 32), "r"(r), "r"(sa(&full[s])) : "memory");
    } else if (mode == 1) {
      int c = static_cast<int>(u % 8), r = static_cast<int>(u / 8) * 256;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(dst)), "l"(m), "r"(c * 32), "r"(r), "r"(sa(&full[s])) : "memory");
    } else if (mode == 2) {
      int r = static_cast<int>(u) * 16;
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(dst)), "l"(m), "r"(0), "r"(0), "r"(r), "r"(sa(&full[s])) : "memory");
    } else if (mode == 3) {
      int r = static_cast<int>(u) * 16;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(dst)), "l"(m), "r"(0), "r"(r), "r"(sa(&full[s])) : "memory");
    } else {
      const float* src = base + u * (STAGE / 4);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(dst)), "l"(src), "r"(STAGE), "r"(sa(&full[s])) : "memory");
    }
  };
  int64_t mine = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) ++mine;
  int64_t issued = 0;
  for (; issued < rs && issued < mine; ++issued) issue(blockIdx.x + issued * gridDim.x, static_cast<int>(issued));
  int acc = 0;
  for (int64_t i = 0; i < mine; ++i) {
    const int s = static_cast<int>(i % rs);
    const uint32_t ph = static_cast<uint32_t>(i / rs) & 1u;
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n"
                 ::"r"(sa(&full[s])), "r"(ph) : "memory");
    acc += smem[s * bytes + 5];
    if (issued < mine) { issue(blockIdx.x + issued * gridDim.x, s); ++issued; }
  }
  if (acc == 12345) *sink = acc;
}

using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                         CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t M = 2449029 / 256 * 256;   // whole 256-row blocks
  float* a;
  int* sink;
  cudaMalloc(&a, M * K * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 0, M * K * 4);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2 * STAGE > 200000 ? 200 * 1024 : 16 * 2 * STAGE);
  for (int mode = 0; mode <= 4; ++mode) {
    for (int rs : {4, 6, 8, 12}) {
      if (mode == 1 && rs > 6) continue;
      CUtensorMap map{};
      CUresult r = CUDA_SUCCESS;
      int64_t units = 0;
      if (mode == 0 || mode == 1) {
        const int br = mode == 0 ? 128 : 256;
        cuuint64_t dims[2] = {K, (cuuint64_t)M};
        cuuint64_t str[1] = {K * 4};
        cuuint32_t box[2] = {32, (cuuint32_t)br}, es[2] = {1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        units = M / br * 8;
      } else if (mode == 2) {
        cuuint64_t dims[3] = {32, 8, (cuuint64_t)M};
        cuuint64_t str[2] = {128, K * 4};
        cuuint32_t box[3] = {32, 8, 16}, es[3] = {1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        units = M / 16;
      } else if (mode == 3) {
        cuuint64_t dims[2] = {K, (cuuint64_t)M};
        cuuint64_t str[1] = {K * 4};
        cuuint32_t box[2] = {256, 16}, es[2] = {1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        units = M / 16;
      } else {
        units = M * K * 4 / STAGE;
      }
      if (r != CUDA_SUCCESS) { printf("{\"mode\": %d, \"encode_error\": %d}\n", mode, (int)r); continue; }
      const size_t smem = (size_t)rs * (mode == 1 ? 2 : 1) * STAGE;
      if (smem > 200 * 1024) continue;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      stream<<<sms, 32, smem>>>(map, a, mode, rs, units, sink);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) stream<<<sms, 32, smem>>>(map, a, mode, rs, units, sink);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("{\"mode\": %d, \"stages\": %d, \"stage_kb\": %d, \"ms\": %.4f, \"gbs\": %.1f, \"err\": \"%s\"}\n", mode, rs,
             (mode == 1 ? 32 : 16), ms, (double)M * K * 4 / ms / 1e6, cudaGetErrorString(err));
    }
  }
  return 0;
}
