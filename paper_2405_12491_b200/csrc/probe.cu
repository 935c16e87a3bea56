// Roofline probe of the shared-memory (LSU) pipe, measured live by bench.py on
// the box it runs on (the traversal's binding resource, DESIGN.md §6 K4
// "Roofline").  One CTA of 512 threads per SM issues unrolled, dependence-free
// LDS.64: lane-consecutive words (conflict free: 2 wavefronts per warp load =
// the 128 B/clk/SM unit rate) and per-lane pseudo-random words in a 16 KB
// region (the random-index rate the deep tree levels see).  Best of 5
// CUDA-event-timed launches each.  Not on the inference path.
#include <cuda_runtime.h>

#include <cstdint>

#include "bridger_internal.h"

namespace bridger {

template <bool RANDOM>
__global__ void __launch_bounds__(512, 1) lds_probe_kernel(int iters, unsigned long long* sink) {
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
      const uint32_t a = RANDOM ? ((idx + u * 977u) * 2246822519u >> 21) & (n - 1)
                                : ((lane + 32u * ((it + u) & 63)) & (n - 1));
      const uint2 v = buf[a];
      acc += v.x ^ v.y;
    }
    idx += acc & 1;
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

}  // namespace bridger

using namespace bridger;

extern "C" bridger_status bridger_probe_smem_bandwidth(int32_t cuda_device, double* conflict_free_gbps,
                                                       double* random_gbps) {
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(BRIDGER_E_CUDA, "invalid cuda_device");
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  unsigned long long* sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaMalloc(&sink, 8);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  const int iters = 20000;
  double res[2] = {0.0, 0.0};
  for (int r = 0; r < 2 && e == cudaSuccess; ++r) {
    auto k = r ? lds_probe_kernel<true> : lds_probe_kernel<false>;
    k<<<sms, 512, 16384>>>(100, sink);
    e = cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
      cudaEventRecord(e0);
      k<<<sms, 512, 16384>>>(iters, sink);
      cudaEventRecord(e1);
      e = cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    res[r] = (double)sms * 512 * iters * 16 * 8 / (best / 1e3) / 1e9;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(sink);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(BRIDGER_E_CUDA, std::string("smem probe: ") + cudaGetErrorString(e));
  if (conflict_free_gbps) *conflict_free_gbps = res[0];
  if (random_gbps) *random_gbps = res[1];
  return BRIDGER_OK;
}
