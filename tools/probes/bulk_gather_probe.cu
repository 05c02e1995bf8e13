// Bulk-copy row gather probe: can one cp.async.bulk (TMA) per edge gather small
// rows (192 B: K1's reassociated layer 3; 768 B: K4's 4x47 Z rows) faster
// than K1's per-lane 16-byte cp.async ring, whose d=48 kernel is request-rate
// bound (profiles/r02_ncu_k1_d48.md)?
//
// N source rows of ROWB bytes (pitch = ROWB), B output rows of DEG random
// in-neighbours each (uniform ids).  A warp owns one output row at a time:
// each chunk of up to 32 edges is one cp.async.bulk per lane into the warp's
// ring (G groups x 32 slots x ROWB, one mbarrier per group), the next chunk
// is in flight while the lanes sum the current one in edge order (one add
// chain per column, like K1).  Prints gathered GB/s (DEG * ROWB per row).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o bulk_gather_probe bulk_gather_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n"
               ::"r"(bar), "r"(par) : "memory");
}

template <int ROWB, int G, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) bulk_gather(const float* __restrict__ h,
                                                          const int32_t* __restrict__ idx, int deg,
                                                          int64_t rows, float* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[WARPS][G];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * G * 32 * ROWB;
  if (lane < G) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][lane])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  constexpr int L = ROWB / 16;   // consuming lanes (16 B each)
  uint32_t phase_bits = 0;       // bit g: parity of group g's next completion
  int gq = 0;                    // next group to issue into
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * WARPS;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * WARPS + warp; r < rows; r += nwarps) {
    const int32_t* ids = idx + r * deg;
    const int nch = (deg + 31) / 32;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto issue = [&](int c, int g) {
      const int cnt = min(32, deg - 32 * c);
      const uint32_t b = sa(&bar[warp][g]);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(b), "r"(cnt * ROWB) : "memory");
      __syncwarp();
      if (lane < cnt) {
        const float* src = h + static_cast<int64_t>(__ldg(ids + 32 * c + lane)) * (ROWB / 4);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(ring + (g * 32 + lane) * ROWB)), "l"(src), "r"(ROWB), "r"(b) : "memory");
      }
    };
    // prologue: up to G chunks in flight
    int issued = 0;
    int gfirst = gq;
    for (; issued < nch && issued < G; ++issued) { issue(issued, gq); gq = (gq + 1) % G; }
    int gc = gfirst;
    for (int c = 0; c < nch; ++c) {
      const int cnt = min(32, deg - 32 * c);
      mbar_wait(sa(&bar[warp][gc]), (phase_bits >> gc) & 1u);
      phase_bits ^= 1u << gc;
      if (lane < L) {
        const uint8_t* base = ring + gc * 32 * ROWB + lane * 16;
        for (int j = 0; j < cnt; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(base + j * ROWB);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      __syncwarp();                       // group gc consumed: reusable
      if (issued < nch) { issue(issued, gc); ++issued; gq = (gc + 1) % G; }
      gc = (gc + 1) % G;
    }
    gq = gc;
    if (lane < L) reinterpret_cast<float4*>(out + r * (ROWB / 4))[lane] = acc;
  }
}

template <int ROWB, int G, int WARPS, int CTAS_PER_SM>
void run(const char* name, int64_t n_src, int deg, int64_t rows) {
  float* h;
  int32_t* idx;
  float* out;
  cudaMalloc(&h, n_src * ROWB);
  cudaMalloc(&idx, rows * deg * 4);
  cudaMalloc(&out, rows * ROWB);
  cudaMemset(h, 0, n_src * ROWB);
  std::vector<int32_t> hidx(rows * deg);
  uint64_t s = 88172645463325252ull;
  for (auto& v : hidx) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; v = static_cast<int32_t>(s % n_src); }
  cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice);
  const int smem = WARPS * G * 32 * ROWB;
  auto k = bulk_gather<ROWB, G, WARPS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * CTAS_PER_SM;
  k<<<grid, WARPS * 32, smem>>>(h, idx, deg, rows, out);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k<<<grid, WARPS * 32, smem>>>(h, idx, deg, rows, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = static_cast<double>(rows) * deg * ROWB;
  printf("{\"kernel\": \"%s\", \"row_bytes\": %d, \"groups\": %d, \"warps\": %d, \"ctas_per_sm\": %d, "
         "\"rows\": %lld, \"deg\": %d, \"ms\": %.4f, \"gathered_gbs\": %.1f, \"err\": \"%s\"}\n",
         name, ROWB, G, WARPS, CTAS_PER_SM, static_cast<long long>(rows), deg, ms, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(h);
  cudaFree(idx);
  cudaFree(out);
}

int main() {
  const int64_t n_src = 2449029;
  const int deg = 50;
  const int64_t rows = 2449029;
  run<192, 2, 8, 2>("bulk", n_src, deg, rows);
  run<192, 3, 8, 1>("bulk", n_src, deg, rows);
  run<192, 2, 4, 4>("bulk", n_src, deg, rows);
  run<768, 1, 8, 1>("bulk", n_src, deg, rows);
  run<768, 2, 4, 1>("bulk", n_src, deg, rows);
  return 0;
}
