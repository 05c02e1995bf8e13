// tcgen05.mma kind::tf32 issue-rate probe: one CTA per SM issues a chain of
// `reps` MMAs (M = 128, K = 8, N = n) into one TMEM accumulator from fixed
// shared-memory (SS) or TMEM-A (TS) operands, commits once, and reports
// clock cycles per MMA.  Answers: is a chain of small-N MMAs bound by a
// per-instruction floor rather than by the M*N/256-cycle formula?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_rate_probe mma_rate_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {   // SWIZZLE_128B K-major
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

template <int n, int ts>
__global__ void __launch_bounds__(128, 1) probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];   // A 16 KB, B up to 32 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    // the whole warp runs the issue loop with warp-uniform operands; elect.sync
    // inside the asm picks the one issuing lane (no divergent region, so the
    // compiler keeps descriptors in uniform registers: no R2UR/ELECT waterfall)
    const uint64_t da = desc(sa(smem)), db = desc(sa(smem + 16384));
    t0 = clock64();
    // 12 MMAs per iteration (4 k-steps x 3 products, the v3 chunk), constant
    // descriptor offsets: what a fully unrolled issue loop costs
    for (int i = 0; i < reps; i += 12) {
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const uint32_t o = (j & 3) * 2;
        if (ts) {
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tmem), "r"(tmem + 256 + 8 * (j & 3)), "l"(db + o), "n"(idesc), "r"(i | j));
        } else {
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(da + o), "l"(db + o), "n"(idesc), "r"(i | j));
        }
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                 ::"r"(sa(&bar)) : "memory");
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n"
                 ::"r"(sa(&bar)) : "memory");
    t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int n, int ts) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int reps = 4092;
    cudaMemset(d, 0, 8);
    kern<<<sms, 128, 64 * 1024>>>(reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"ts\": %d, \"n\": %d, \"cycles_per_mma\": %.1f, \"formula\": %.1f, \"err\": \"%s\"}\n", ts, n,
           (double)cyc / sms / reps, 128.0 * n / 256.0, cudaGetErrorString(e));
  };
  run(probe<16, 0>, 16, 0); run(probe<48, 0>, 48, 0); run(probe<64, 0>, 64, 0); run(probe<128, 0>, 128, 0);
  run(probe<256, 0>, 256, 0);
  run(probe<16, 1>, 16, 1); run(probe<48, 1>, 48, 1); run(probe<64, 1>, 64, 1); run(probe<128, 1>, 128, 1);
  run(probe<256, 1>, 256, 1);
  return 0;
}
