// Probe of tcgen05.mma.sp ... kind::i8 (sm_100a) semantics, run once on a B200
// to pin the 2:4 metadata layout before the sparse path-contraction kernel
// (gemm_path.cu pcs_kernel) relies on it.  One CTA, M = 128, N = 64, K = 64
// (logical; A stored compressed, 32 bytes per row).  B = identity (B[n][k] =
// [k == n]) so D[m][n] = A_logical[m][n], i.e. D shows where every compressed
// element landed.  Compressed A[m][j] = j + 1.  Metadata per row m (64 bits,
// written to TMEM lane m at column E0 and E0+1 with tcgen05.st):
//   row parity 0: nibble 0x4 in every group (kept positions 0,1)
//   row parity 1: nibble 0xE in every group (kept positions 2,3)
// Hypothesis H: group g = logical k 4g..4g+3 uses metadata bits [4g, 4g+4)
// (low 2 bits: position of compressed element 2g, high 2 bits: of 2g+1).
// Prints D rows 0 and 1 and a verdict per (sparse_id2, E column) tried.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o sparse_probe tools/sparse_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

__device__ __forceinline__ uint32_t s2u(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void probe(int32_t* out, int e_col, int id2, int meta_mode) {
  __shared__ __align__(1024) int8_t sA[2 * 128 * 16];  // [kc=2][128 rows][16 B]
  __shared__ __align__(1024) int8_t sB[4 * 64 * 16];   // [kc=4][64 rows][16 B]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    const int m = i / 32, j = i % 32;
    sA[(j / 16) * 2048 + m * 16 + (j % 16)] = (int8_t)(j + 1);
  }
  for (int i = tid; i < 64 * 64; i += blockDim.x) {
    const int n = i / 64, k = i % 64;
    sB[(k / 16) * 1024 + n * 16 + (k % 16)] = (int8_t)(k == n ? 1 : 0);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(s2u(&tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_holder;
  // metadata: thread = TMEM lane = row m (4 warps x 32 lanes)
  {
    const int m = tid;
    uint32_t nib;
    if (meta_mode == 0) nib = (m & 1) ? 0xEu : 0x4u;
    else if (meta_mode == 1) nib = (m & 1) ? 0x8u : 0x4u;   // 0x8 = positions {0, 2}
    else nib = (m & 1) ? 0xDu : 0x4u;                       // 0xD = positions {1, 3}
    uint32_t w = 0, w1 = 0;
    for (int g = 0; g < 8; ++g) w |= nib << (4 * g);
    // mode 3: column E0 = 0x4 groups, column E0+1 = 0xE groups (every row)
    if (meta_mode == 3) {
      w = 0x44444444u;
      w1 = 0xEEEEEEEEu;
    } else {
      w1 = w;
    }
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)e_col;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(w), "r"(w1), "r"(w),
                 "r"(w1)
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    // idesc: sparse id2 [0,2), sparse flag [2], D s32 [4,6)=2, A s8 [7,10)=1, B s8 [10,13)=1, N>>3 [17,23), M>>4 [24,29)
    const uint32_t idesc = (uint32_t)id2 | (1u << 2) | (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) |
                           ((128u >> 4) << 24);
    const uint64_t ad = smem_desc(s2u(sA), 2048, 128);
    const uint64_t bd = smem_desc(s2u(sB), 1024, 128);
    const uint32_t te = tmem + (uint32_t)e_col;
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %5, {%6, %6, %6, %6}, p;\n\t}\n" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(te), "r"(0u), "r"(idesc), "r"(z)
        : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s2u(&bar))
                 : "memory");
  }
  // wait for the MMA
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}\n" ::"r"(
          s2u(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int cb = 0; cb < 64; cb += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) out[tid * 64 + cb + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  int32_t* d;
  cudaMalloc(&d, 128 * 64 * 4);
  int32_t h[128 * 64];
  const uint32_t nibs[4][2] = {{0x4, 0xE}, {0x4, 0x8}, {0x4, 0xD}, {0x4, 0xE}};
  for (int mode = 0; mode < 4; ++mode)
    for (int e_col = 64; e_col <= 132; e_col += (e_col == 64 ? 64 : 4))
      for (int id2 = 0; id2 < 1; ++id2) {
        cudaMemset(d, 0xFF, 128 * 64 * 4);
        probe<<<1, 128>>>(d, e_col, id2, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("mode %d e_col %d id2 %d: CUDA error %s\n", mode, e_col, id2, cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        // expected under H for each row
        int bad = 0;
        for (int m = 0; m < 128; ++m) {
          for (int n = 0; n < 64; ++n) {
            const uint32_t nib = mode == 3 ? nibs[3][n >= 32] : nibs[mode][m & 1];
            const int g = n / 4, pos = n % 4;
            int want = 0;
            if ((int)(nib & 3) == pos) want = 2 * g + 1;
            if ((int)((nib >> 2) & 3) == pos) want = 2 * g + 2;
            if (h[m * 64 + n] != want) ++bad;
          }
        }
        printf("mode %d e_col %d id2 %d: mismatches vs H = %d\n", mode, e_col, id2, bad);
        if (bad)
          for (int m = 0; m < 2; ++m) {
            printf("  row %d:", m);
            for (int n = 0; n < 32; ++n) printf(" %d", h[m * 64 + n]);
            printf("\n");
          }
      }
  return 0;
}
