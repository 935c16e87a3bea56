// Probe: leaf-vector gather rate of the tree-streamed walk (C4 shape: 1000 trees
// x 4096 leaves x 8 fp32 classes = 131 MB, one 32-byte leaf vector per
// (row, tree), every CTA on the same tree at about the same time).
//   A: each lane loads its leaf vector with two 16-byte global loads (the LSU /
//      L1 path the K4s kernel uses: 32 distinct sectors per warp instruction);
//   B: the TMA engine gathers it: per warp and tree 8 x
//      cp.async.bulk.tensor.2d.tile::gather4 (4 leaf rows each) into shared
//      memory, one mbarrier per warp buffer, double-buffered over trees.
// Leaf indices are a hash of (row, tree); prints ms per 1M rows for each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe tools/gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kLeaves = 4096, kK = 8, kWarps = 16;

__device__ __forceinline__ uint32_t hsh(uint32_t r, uint32_t t) {
  uint32_t h = r * 0x9E3779B1u ^ (t * 0x85EBCA77u + 0x165667B1u);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  return h;
}
__device__ __forceinline__ uint32_t s2u(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512) gather_ldg(const float4* __restrict__ tab, int n_rows, int T, float* out) {
  for (int base = blockIdx.x * 512; base < n_rows; base += gridDim.x * 512) {
    const uint32_t row = base + threadIdx.x;
    float acc = 0.f;
    uint32_t li = hsh(row, 0) & (kLeaves - 1);
    float4 a = __ldg(tab + (size_t)li * 2), b = __ldg(tab + (size_t)li * 2 + 1);
    for (int t = 0; t < T; ++t) {
      float4 na = a, nb = b;
      if (t + 1 < T) {
        const size_t g = (size_t)(t + 1) * kLeaves + (hsh(row, t + 1) & (kLeaves - 1));
        na = __ldg(tab + g * 2);
        nb = __ldg(tab + g * 2 + 1);
      }
      acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
      a = na;
      b = nb;
    }
    if (row < (uint32_t)n_rows) out[row] = acc;
  }
}

__global__ void __launch_bounds__(512) gather_tma(const __grid_constant__ CUtensorMap tm, int n_rows, int T, float* out) {
  __shared__ __align__(128) float slot[kWarps][2][32 * kK];
  __shared__ __align__(8) uint64_t bar[kWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&bar[warp][b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t ph[2] = {0, 0};
  for (int base = blockIdx.x * 512; base < n_rows; base += gridDim.x * 512) {
    const uint32_t row = base + threadIdx.x;
    float acc = 0.f;
    auto issue = [&](int t, int b) {
      const int gi = t * kLeaves + (int)(hsh(row, t) & (kLeaves - 1));
      const int i0 = __shfl_sync(0xffffffffu, gi, (lane & 7) * 4 + 0);
      const int i1 = __shfl_sync(0xffffffffu, gi, (lane & 7) * 4 + 1);
      const int i2 = __shfl_sync(0xffffffffu, gi, (lane & 7) * 4 + 2);
      const int i3 = __shfl_sync(0xffffffffu, gi, (lane & 7) * 4 + 3);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s2u(&bar[warp][b])), "r"(32 * kK * 4)
                     : "memory");
      __syncwarp();
      if (lane < 8)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(s2u(&slot[warp][b][lane * 4 * kK])),
            "l"(&tm), "r"(s2u(&bar[warp][b])), "r"(0), "r"(i0), "r"(i1), "r"(i2), "r"(i3)
            : "memory");
    };
    issue(0, 0);
    for (int t = 0; t < T; ++t) {
      const int b = t & 1;
      if (t + 1 < T) issue(t + 1, b ^ 1);
      asm volatile(
          "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n}\n" ::"r"(
              s2u(&bar[warp][b])),
          "r"(ph[b])
          : "memory");
      ph[b] ^= 1;
      const float4 a = *reinterpret_cast<const float4*>(&slot[warp][b][lane * kK]);
      const float4 c = *reinterpret_cast<const float4*>(&slot[warp][b][lane * kK + 4]);
      acc += a.x + a.y + a.z + a.w + c.x + c.y + c.z + c.w;
      __syncwarp();
    }
    if (row < (uint32_t)n_rows) out[row] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int T = 1000, n_rows = 1 << 20;
  const size_t n = (size_t)T * kLeaves * kK;
  float* tab;
  float* out;
  cudaMalloc(&tab, n * 4);
  cudaMalloc(&out, n_rows * 4);
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
  cudaMemcpy(tab, h.data(), n * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  CUtensorMap tm;
  cuuint64_t gdim[2] = {kK, (cuuint64_t)T * kLeaves};
  cuuint64_t gstr[1] = {kK * 4};
  cuuint32_t box[2] = {kK, 1}, es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  std::vector<float> o1(n_rows), o2(n_rows);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid_mul = 1; grid_mul <= 2; ++grid_mul) {
    for (int k = 0; k < 2; ++k) {
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (k == 0)
          gather_ldg<<<148 * grid_mul, 512>>>((const float4*)tab, n_rows, T, out);
        else
          gather_tma<<<148 * grid_mul, 512>>>(tm, n_rows, T, out);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("kernel %d failed: %s\n", k, cudaGetErrorString(err));
          return 1;
        }
        cudaEventElapsedTime(&ms, e0, e1);
      }
      cudaMemcpy(k == 0 ? o1.data() : o2.data(), out, n_rows * 4, cudaMemcpyDeviceToHost);
      printf("%s grid %d: %.3f ms per %d rows x %d trees (%.1f G leaf gathers/s)\n", k == 0 ? "ldg" : "tma gather4",
             148 * grid_mul, ms, n_rows, T, (double)n_rows * T / ms * 1e-6);
    }
    int bad = 0;
    for (int i = 0; i < n_rows; ++i) bad += o1[i] != o2[i];
    printf("mismatches ldg vs tma: %d\n", bad);
  }
  return 0;
}
