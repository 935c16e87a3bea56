// Probe: 2-D TMA tile loads from X [n][F] fp32 viewed as [n/R][R*F], box
// {FG, 32/R}, at column starts that are / are not 16-byte aligned.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ uint32_t s2u(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int col, int srow, int nbytes, float* out) {
  __shared__ __align__(128) float buf[32 * 8];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s2u(&bar)), "r"(nbytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            s2u(buf)),
        "l"(&tm), "r"(col), "r"(srow), "r"(s2u(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}\n" ::"r"(
            s2u(&bar))
        : "memory");
    for (int i = 0; i < nbytes / 4; ++i) out[i] = buf[i];
  }
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  struct Case { int F, R, FG, col; };
  Case cases[] = {{28, 1, 4, 0}, {28, 1, 4, 4}, {90, 2, 8, 0}, {90, 2, 8, 8}, {90, 2, 8, 90}, {90, 2, 8, 98}, {21, 4, 4, 0}, {21, 4, 4, 21}};
  const int n = 4096;
  float* X; float* out;
  cudaMalloc(&X, (size_t)n * 90 * 4); cudaMalloc(&out, 4096);
  std::vector<float> h((size_t)n * 90);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  cudaMemcpy(X, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (auto c : cases) {
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)c.R * c.F, (cuuint64_t)(n / c.R)};
    cuuint64_t gstr[1] = {(cuuint64_t)c.R * c.F * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.FG, (cuuint32_t)(32 / c.R)}, es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("F %d R %d FG %d col %d: encode %d", c.F, c.R, c.FG, c.col, (int)r);
    k<<<1, 32>>>(tm, c.col, 1, 32 * c.FG * 4 / c.R, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf(" -> %s", cudaGetErrorString(e));
    if (e != cudaSuccess) { printf("\n"); return 1; }
    float o[4]; cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("  first %g %g (want %g)\n", o[0], o[1], (double)(1 * c.R * c.F + c.col));
  }
  return 0;
}
