// Shared-memory (LSU) pipe microbenchmark for the traversal roofline
// (SURVEY.md §8(d) "SMEM LDS throughput"): one CTA of 512 threads per SM, each
// thread issues LDS.64 loads in a dependent-free unrolled loop.
//   conflict-free: lane-consecutive 8-byte words (2 wavefronts per warp LDS.64)
//   random:        per-lane pseudo-random 8-byte words in a 16 KB region
// Output: JSON with achieved shared-memory bytes/s and per-SM bytes/clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool RANDOM>
__global__ void __launch_bounds__(512, 1) lds_kernel(int iters, unsigned long long* sink) {
  extern __shared__ uint2 buf[];
  const int n = 2048;  // 16 KB of 8-byte words
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint2(i, i * 3);
  __syncthreads();
  uint32_t idx = (threadIdx.x * 2654435761u) & (n - 1);
  uint32_t acc = 0;
  const uint32_t lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      uint32_t a = RANDOM ? ((idx + u * 977u) * 2246822519u >> 21) & (n - 1) : ((lane + 32u * ((it + u) & 63)) & (n - 1));
      const uint2 v = buf[a];
      acc += v.x ^ v.y;
    }
    idx += acc & 1;
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double res[2];
  for (int r = 0; r < 2; ++r) {
    auto k = r ? lds_kernel<true> : lds_kernel<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    k<<<sms, 512, 16384>>>(100, sink);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k<<<sms, 512, 16384>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double bytes = (double)sms * 512 * iters * 16 * 8;
    res[r] = bytes / (best / 1e3);
  }
  printf("{\"smem_lds64_conflict_free_GBps\": %.1f, \"smem_lds64_random_GBps\": %.1f, \"sms\": %d, "
         "\"clock_mhz_attr\": %d, \"per_sm_bytes_per_clk_at_1965\": %.2f, "
         "\"how\": \"tools/smem_peak.cu: 1 CTA x 512 threads per SM, unrolled LDS.64, best of 5\"}\n",
         res[0] / 1e9, res[1] / 1e9, sms, clk / 1000, res[0] / sms / 1.965e9);
  return 0;
}
