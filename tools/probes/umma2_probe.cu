// Probe of the cta_group::2 tcgen05 programming model (groundwork for a paired-SM
// K2): one CTA pair computes D[256 x 64] = A[256 x 16] B[64 x 16]^T
// with two kind::tf32 MMAs (K = 8 each) issued by the leader CTA.  Each CTA holds
// its 128 rows of A in the canonical no-swizzle K-major layout; B is placed either
// split (CTA r holds B rows [32 r, 32 r + 32)) or whole in both CTAs.  Each CTA
// drains its own TMEM (its 128 rows) after a multicast commit.  The host compares
// both placements with an fp64 reference (inputs are exact in tf32).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma2_probe umma2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 256, N = 64, K = 16;
constexpr uint32_t SBO = (K / 4) * 128, LBO = 128;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return static_cast<uint32_t>((r & 7) * 16 + c * 128 + (r >> 3) * SBO);
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((a >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((LBO >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((SBO >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const float* A, const float* B, float* D, int split) {
  __shared__ __align__(1024) uint8_t a_s[128 * K * 4];
  __shared__ __align__(1024) uint8_t b_s[N * K * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // operands: A rows [128 rank, +128); B rows [32 rank, +32) (split) or all 64
  for (int i = tid; i < 128 * (K / 4); i += 128) {
    const int r = i / (K / 4), c = i % (K / 4);
    *reinterpret_cast<float4*>(a_s + tile_off(r, c)) =
        *reinterpret_cast<const float4*>(A + (128 * rank + r) * K + 4 * c);
  }
  const int brows = split ? N / 2 : N;
  for (int i = tid; i < brows * (K / 4); i += 128) {
    const int r = i / (K / 4), c = i % (K / 4);
    const int src = split ? (N / 2) * rank + r : r;
    *reinterpret_cast<float4*>(b_s + tile_off(r, c)) =
        *reinterpret_cast<const float4*>(B + src * K + 4 * c);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(saddr(&tslot)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // idesc: D f32, A/B tf32, N >> 3, M >> 4 (M = 256 for the pair)
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
  if (rank == 0 && tid == 0) {
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t da = desc(saddr(a_s) + j * 256), db = desc(saddr(b_s) + j * 256);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(j));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(saddr(&bar)), "h"(static_cast<uint16_t>(3)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n"
               ::"r"(saddr(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 32) {
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
        : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 128 * rank + warp * 32 + lane;
    for (int i = 0; i < 32; ++i) D[row * N + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = static_cast<float>((i * 7 % 13) - 6) / 4.0f;
  for (int i = 0; i < N * K; ++i) B[i] = static_cast<float>((i * 5 % 11) - 5) / 8.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int split = 1; split >= 0; --split) {
    cudaMemset(dD, 0xff, D.size() * 4);
    probe<<<2, 128>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"split\": %d, \"error\": \"%s\"}\n", split, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0; int bad = 0, bad_lo = 0, bad_hi = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += static_cast<double>(A[m * K + k]) * B[n * K + k];
        const double err = std::fabs(ref - D[m * N + n]);
        maxerr = std::fmax(maxerr, err);
        if (err > 1e-4) { ++bad; if (n < N / 2) ++bad_lo; else ++bad_hi; }
      }
    printf("{\"split\": %d, \"max_abs_err\": %g, \"bad\": %d, \"bad_cols_lo\": %d, \"bad_cols_hi\": %d}\n",
           split, maxerr, bad, bad_lo, bad_hi);
  }
  return 0;
}
