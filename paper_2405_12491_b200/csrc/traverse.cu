// K4 traversal: host-side dispatch (trav_run) and finalize of caller-provided
// accumulators.  The kernel templates live in traverse.cuh and are
// instantiated in trav_inst_*.cu (compiled in parallel).
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "traverse.cuh"
#include "ptx.cuh"

namespace bridger {

cudaError_t launch_trav_deep(const TravParams& p, int K, bool ml, int wm, int grid, int block, int smem,
                             cudaStream_t st);
int trav_deep_smem(int chunk_cap, int code_buf, int nb);

#define BRIDGER_TRAV_EXTERN(ACC, ML, GT, FMT)                                                                           \
  extern template cudaError_t launch_trav_t<1, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<2, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<4, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<8, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<16, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_trav_t<64, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);
BRIDGER_TRAV_EXTERN(long long, false, false, 0)
BRIDGER_TRAV_EXTERN(long long, true, false, 0)
BRIDGER_TRAV_EXTERN(double, false, false, 0)
BRIDGER_TRAV_EXTERN(double, true, false, 0)
BRIDGER_TRAV_EXTERN(long long, false, false, 1)
BRIDGER_TRAV_EXTERN(long long, true, false, 1)
BRIDGER_TRAV_EXTERN(double, false, false, 1)
BRIDGER_TRAV_EXTERN(double, true, false, 1)
BRIDGER_TRAV_EXTERN(long long, false, true, 0)
BRIDGER_TRAV_EXTERN(long long, true, true, 0)
BRIDGER_TRAV_EXTERN(double, false, true, 0)
BRIDGER_TRAV_EXTERN(double, true, true, 0)
BRIDGER_TRAV_EXTERN(long long, false, false, 3)
BRIDGER_TRAV_EXTERN(long long, true, false, 3)
BRIDGER_TRAV_EXTERN(double, false, false, 3)
BRIDGER_TRAV_EXTERN(double, true, false, 3)
BRIDGER_TRAV_EXTERN(long long, false, false, 4)
BRIDGER_TRAV_EXTERN(long long, true, false, 4)
BRIDGER_TRAV_EXTERN(double, false, false, 4)
BRIDGER_TRAV_EXTERN(double, true, false, 4)
BRIDGER_TRAV_EXTERN(long long, false, false, 5)
BRIDGER_TRAV_EXTERN(long long, true, false, 5)
BRIDGER_TRAV_EXTERN(double, false, false, 5)
BRIDGER_TRAV_EXTERN(double, true, false, 5)
#define BRIDGER_STREAM_EXTERN_W(ACC, ML, W, SPL)                                                                         \
  extern template cudaError_t launch_stream_t<1, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<2, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<4, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<8, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<16, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_stream_t<64, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_stream_t<1, ACC, ML, W, true, SPL>(const TravParams&, int, int, int, cudaStream_t);
#define BRIDGER_STREAM_EXTERN_S(SPL)                \
  BRIDGER_STREAM_EXTERN_W(long long, false, 1, SPL) \
  BRIDGER_STREAM_EXTERN_W(long long, true, 1, SPL)  \
  BRIDGER_STREAM_EXTERN_W(double, false, 1, SPL)    \
  BRIDGER_STREAM_EXTERN_W(double, true, 1, SPL)     \
  BRIDGER_STREAM_EXTERN_W(long long, false, 2, SPL) \
  BRIDGER_STREAM_EXTERN_W(long long, true, 2, SPL)  \
  BRIDGER_STREAM_EXTERN_W(double, false, 2, SPL)    \
  BRIDGER_STREAM_EXTERN_W(double, true, 2, SPL)
BRIDGER_STREAM_EXTERN_S(0)
BRIDGER_STREAM_EXTERN_S(1)
BRIDGER_STREAM_EXTERN_S(2)
BRIDGER_STREAM_EXTERN_W(long long, false, 3, 2)
BRIDGER_STREAM_EXTERN_W(long long, true, 3, 2)
BRIDGER_STREAM_EXTERN_W(double, false, 3, 2)
BRIDGER_STREAM_EXTERN_W(double, true, 3, 2)
BRIDGER_TRAV_EXTERN(long long, false, true, 2)
BRIDGER_TRAV_EXTERN(long long, true, true, 2)
BRIDGER_TRAV_EXTERN(double, false, true, 2)
BRIDGER_TRAV_EXTERN(double, true, true, 2)

// Threshold-bin coding of the input (§8(f2)): X [N][F] fp32 row-major ->
// codes [n_blocks][F2/2][32][2] u16 (F2 = F rounded up to even; feature pairs
// interleaved per lane so that the traversal's per-lane code loads hit bank
// `lane` for ANY feature), code = #{u in U_f : u < x}, NaN -> 0xFFFF.
// lane = row; each warp bulk-copies dense [32][F] blocks (double buffered) and
// descends, for NP feature pairs at a time (2 NP independent chains, passes
// sized so no chain is wasted: C2's 14 pairs = 2 passes of 7), the features'
// k-level Eytzinger search trees in shared memory: i <- 2i + 1 + [E_f[i] < x]
// (all lanes of a warp search the same feature, so the top levels are
// broadcasts).  The leaf reached, i - (2^k - 1), is the code (lowering.cpp).
template <int NP, int V>
__global__ void __launch_bounds__(512, 1) bin_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                     const float* __restrict__ table, int32_t k,
                                                     uint32_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  // programmatic dependent launch: the walk kernel that consumes the codes may
  // be scheduled (and run its prologue) as SMs free up; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int P = (1 << k) - 1;
  const int F2h = (F + 1) >> 1;  // feature pairs
  const size_t tab_bytes = ((size_t)F * P * 4 + 127) / 128 * 128;
  const uint32_t blk_bytes = 128u * (uint32_t)F;  // dense [32][F] fp32
  float* stage = reinterpret_cast<float*>(smem + tab_bytes + (size_t)warp * 2 * blk_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tab_bytes + (size_t)NW * 2 * blk_bytes) + 2 * warp;
  {
    const float4* src = reinterpret_cast<const float4*>(table);
    float4* dst = reinterpret_cast<float4*>(smem);
    const int n4 = (F * P) / 4;
    for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    for (int i = n4 * 4 + threadIdx.x; i < F * P; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = table[i];
  }
  if (lane == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t tab_s = ptx::s2u(smem);
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t gstride = (int64_t)gridDim.x * NW;
  int64_t blk = (int64_t)blockIdx.x * NW + warp;
  auto issue = [&](int64_t b, int buf) {
    if (lane == 0 && b < n_blocks && (b + 1) * 32 <= n_rows) {
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(&bars[buf], blk_bytes);
      ptx::bulk_g2s(stage + (size_t)buf * 32 * F, X + b * 32 * (int64_t)F, blk_bytes, &bars[buf]);
    }
  };
  issue(blk, 0);
  uint32_t phase = 0;  // bit b: parity of buffer b
  for (int it = 0; blk < n_blocks; blk += gstride, ++it) {
    const int buf = it & 1;
    float* St = stage + (size_t)buf * 32 * F;
    const int64_t row0 = blk * 32;
    if (row0 + 32 <= n_rows) {
      ptx::mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      const int rows = (int)(n_rows - row0);
      const float* src = X + row0 * F;
      for (int e = lane; e < 32 * F; e += 32) St[e] = e < rows * F ? src[e] : 0.f;
      __syncwarp();
    }
    issue(blk + gstride, buf ^ 1);  // the other buffer was drained by the previous block
    const float* xr = St + (size_t)lane * F;
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
    for (int f0 = 0; f0 < 2 * F2h; f0 += 2 * NP) {
      float x[2 * NP];
#pragma unroll
      for (int u = 0; u < 2 * NP; u += 2) {
        if (V == 2 && f0 + u + 1 < F) {
          const float2 v = *reinterpret_cast<const float2*>(xr + f0 + u);  // F even: 8-byte aligned
          x[u] = v.x;
          x[u + 1] = v.y;
        } else {
          x[u] = f0 + u < F ? xr[f0 + u] : 0.f;
          x[u + 1] = f0 + u + 1 < F ? xr[f0 + u + 1] : 0.f;
        }
      }
      // shared address A of the current search-tree node; A' = 2A + c4 (+ 4 if E < x)
      uint32_t A[2 * NP], c4[2 * NP];
#pragma unroll
      for (int u = 0; u < 2 * NP; ++u) {
        A[u] = tab_s + (uint32_t)(min(f0 + u, F - 1) * P) * 4u;
        c4[u] = 4u - A[u];
      }
      for (int s = 0; s < k; ++s) {
#pragma unroll
        for (int u = 0; u < 2 * NP; ++u) {
          const float e = ptx::lds_f32(A[u]);
          A[u] = 2u * A[u] + c4[u];
          if (e < x[u]) A[u] += 4u;
        }
      }
#pragma unroll
      for (int u = 0; u < 2 * NP; u += 2) {
        if (f0 + u < 2 * F2h) {
          // leaf byte offset A + c4 - 4 = 4 (2^k - 1 + code)
          const uint32_t c0 = isnan(x[u]) ? 0xFFFFu : ((A[u] + c4[u] - 4u) >> 2) - (uint32_t)P;
          const uint32_t c1 = f0 + u + 1 >= F ? 0u
                              : isnan(x[u + 1]) ? 0xFFFFu : ((A[u + 1] + c4[u + 1] - 4u) >> 2) - (uint32_t)P;
          dst[(size_t)((f0 + u) >> 1) * 32] = c0 | (c1 << 16);
        }
      }
    }
    __syncwarp();
  }
}

// Cooperative binning for search tables too large to leave room for per-warp
// staging (C3: 90 features x 511-slot trees = 184 KB): the CTA's 16 warps share
// one double-buffered dense [32][F] block (bulk copy, mbarrier) and split its
// feature pairs; lane = row as above, up to 8 chains (4 pairs) per warp pass.
template <int NP>
__global__ void __launch_bounds__(512, 1) bin_coop_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                          const float* __restrict__ table, int32_t k,
                                                          uint32_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  // programmatic dependent launch: the walk kernel that consumes the codes may
  // be scheduled (and run its prologue) as SMs free up; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int P = (1 << k) - 1;
  const int F2h = (F + 1) >> 1;
  const size_t tab_bytes = ((size_t)F * P * 4 + 127) / 128 * 128;
  const uint32_t blk_bytes = 128u * (uint32_t)F;
  float* stage = reinterpret_cast<float*>(smem + tab_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tab_bytes + 2 * (size_t)blk_bytes);
  uint32_t* done = reinterpret_cast<uint32_t*>(bars + 2);  // [2] warps finished with buffer b
  {
    const float4* src = reinterpret_cast<const float4*>(table);
    float4* dst = reinterpret_cast<float4*>(smem);
    const int n4 = (F * P) / 4;
    for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    for (int i = n4 * 4 + threadIdx.x; i < F * P; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = table[i];
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    done[0] = done[1] = 0;
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t tab_s = ptx::s2u(smem);
  const int64_t n_blocks = (n_rows + 31) / 32;
  auto issue = [&](int64_t b, int buf) {
    if (threadIdx.x == 0 && b < n_blocks && (b + 1) * 32 <= n_rows) {
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(&bars[buf], blk_bytes);
      ptx::bulk_g2s(stage + (size_t)buf * 32 * F, X + b * 32 * (int64_t)F, blk_bytes, &bars[buf]);
    }
  };
  issue(blockIdx.x, 0);
  issue((int64_t)blockIdx.x + gridDim.x, 1);
  // this warp's pairs when one pass covers them all (F2h <= NP * NW): block-
  // independent chain constants hoisted out of the block loop
  const bool single = F2h <= NP * NW;
  const int npairs = warp < F2h ? min(NP, (F2h - 1 - warp) / NW + 1) : 0;
  uint32_t xoff[2 * NP], A0[2 * NP], c4[2 * NP], hi_mask[NP];
#pragma unroll
  for (int u = 0; u < 2 * NP; ++u) {
    const int f = min(2 * (warp + (u >> 1) * NW) + (u & 1), F - 1);
    xoff[u] = 4u * (uint32_t)f;
    A0[u] = tab_s + (uint32_t)(f * P) * 4u;
    c4[u] = 4u - A0[u];
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) hi_mask[q] = 2 * (warp + q * NW) + 1 >= F ? 0u : 0xFFFFFFFFu;
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x, ++it) {
    const int buf = it & 1;
    float* St = stage + (size_t)buf * 32 * F;
    const int64_t row0 = blk * 32;
    if (row0 + 32 <= n_rows) {
      ptx::mbar_wait(&bars[buf], (uint32_t)(it >> 1) & 1u);
    } else {
      // the tail block (never bulk-copied): every warp is past the buffer's
      // previous use before it is filled by hand
      __syncthreads();
      const int rows = (int)(n_rows - row0);
      const float* src = X + row0 * F;
      for (int e = threadIdx.x; e < 32 * F; e += blockDim.x) St[e] = e < rows * F ? src[e] : 0.f;
      __syncthreads();
    }
    const uint32_t xs = ptx::s2u(St) + 4u * (uint32_t)(lane * F);
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
    if (single) {
      // one pass: the per-chain constants (features, search-tree bases) are
      // block independent and live in registers (hoisted below)
      float x[2 * NP];
      uint32_t A[2 * NP];
#pragma unroll
      for (int u = 0; u < 2 * NP; ++u) {
        x[u] = ptx::lds_f32(xs + xoff[u]);
        A[u] = A0[u];
      }
      for (int s = 0; s < k; ++s) {
#pragma unroll
        for (int u = 0; u < 2 * NP; ++u) {
          const float e = ptx::lds_f32(A[u]);
          A[u] = 2u * A[u] + c4[u];
          if (e < x[u]) A[u] += 4u;
        }
      }
#pragma unroll
      for (int u = 0; u < 2 * NP; u += 2) {
        if (u / 2 < npairs) {
          // leaf byte offset A + c4 - 4 = 4 (2^k - 1 + code)
          const uint32_t c0 = isnan(x[u]) ? 0xFFFFu : ((A[u] + c4[u]) >> 2) - 1u - (uint32_t)P;
          uint32_t c1 = isnan(x[u + 1]) ? 0xFFFFu : ((A[u + 1] + c4[u + 1]) >> 2) - 1u - (uint32_t)P;
          c1 &= hi_mask[u / 2];
          dst[(size_t)(warp + (u >> 1) * NW) * 32] = c0 | (c1 << 16);
        }
      }
    } else {
    const float* xr = St + (size_t)lane * F;
    // this warp's pairs warp, warp + NW, ...: NP pairs (2 NP chains) per pass
    for (int p0 = warp; p0 < F2h; p0 += NP * NW) {
      float x[2 * NP];
      uint32_t A[2 * NP], c4l[2 * NP];
#pragma unroll
      for (int u = 0; u < 2 * NP; ++u) {
        const int f = min(2 * (p0 + (u >> 1) * NW) + (u & 1), F - 1);
        x[u] = xr[f];
        A[u] = tab_s + (uint32_t)(f * P) * 4u;
        c4l[u] = 4u - A[u];
      }
      for (int s = 0; s < k; ++s) {
#pragma unroll
        for (int u = 0; u < 2 * NP; ++u) {
          const float e = ptx::lds_f32(A[u]);
          A[u] = 2u * A[u] + c4l[u];
          if (e < x[u]) A[u] += 4u;
        }
      }
#pragma unroll
      for (int u = 0; u < 2 * NP; u += 2) {
        const int pr = p0 + (u >> 1) * NW;
        if (pr < F2h) {
          const uint32_t c0 = isnan(x[u]) ? 0xFFFFu : ((A[u] + c4l[u] - 4u) >> 2) - (uint32_t)P;
          const uint32_t c1 = 2 * pr + 1 >= F ? 0u
                              : isnan(x[u + 1]) ? 0xFFFFu : ((A[u + 1] + c4l[u + 1] - 4u) >> 2) - (uint32_t)P;
          dst[(size_t)pr * 32] = c0 | (c1 << 16);
        }
      }
    }
    }
    // no CTA-wide barrier per block (it would drain the pipeline): the last
    // warp to finish with this buffer refills it, the others run ahead
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[buf], 1u) == (uint32_t)NW - 1u) {
        done[buf] = 0;
        if (blk + 2 * (int64_t)gridDim.x < n_blocks && (blk + 2 * (int64_t)gridDim.x + 1) * 32 <= n_rows) {
          ptx::fence_proxy_async();
          ptx::mbar_arrive_expect_tx(&bars[buf], blk_bytes);
          ptx::bulk_g2s(stage + (size_t)buf * 32 * F, X + (blk + 2 * (int64_t)gridDim.x) * 32 * (int64_t)F, blk_bytes,
                        &bars[buf]);
        }
      }
    }
  }
}

// Bucketed binning (round 2; TravLayout::bkt_blob, lowering.cpp
// build_bucket_table): code(x) = cum_f[b_f(x)] + lower_bound of x in the
// window U_f[cum .. cum + 2^s_f - 1) -- one u16 load plus s_f <= 4 search
// steps instead of the k = 9..10 levels of the Eytzinger descent.  The
// bucket map b_f(x) = clamp(floor((x - lo_f) * iw_f), 0, NB - 1) is evaluated
// with the same IEEE fp32 operations the host used (monotone: exact).  CTA
// layout as bin_coop_kernel: the whole blob resident, 16 warps share one
// double-buffered dense [32][F] block, the last warp done with a buffer
// refills it; every warp owns fixed feature pairs (chain constants hoisted).
template <int NP>
// nbuf (2 or 3) staged row blocks: the DRAM reads in flight per SM are what
// the kernel waits on once the window search is cheap; feature f's U row sits
// at word offset prm_f[3] (rows of their own length: lowering.cpp).
__global__ void __launch_bounds__(512, 1) bin_bucket_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                            const uint8_t* __restrict__ blob, int32_t blob_bytes,
                                                            int32_t NB, int32_t nbuf,
                                                            uint32_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  // programmatic dependent launch: the walk kernel that consumes the codes may
  // be scheduled (and run its prologue) as SMs free up; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int F2h = (F + 1) >> 1;
  const size_t tab_bytes = ((size_t)blob_bytes + 127) / 128 * 128;
  const uint32_t blk_bytes = 128u * (uint32_t)F;
  float* stage = reinterpret_cast<float*>(smem + tab_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tab_bytes + (size_t)nbuf * blk_bytes);
  uint32_t* done = reinterpret_cast<uint32_t*>(bars + nbuf);
  {
    const float4* src = reinterpret_cast<const float4*>(blob);
    float4* dst = reinterpret_cast<float4*>(smem);
    for (int i = threadIdx.x; i < blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbuf; ++b) {
      ptx::mbar_init(&bars[b], 1);
      done[b] = 0;
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t sbase = ptx::s2u(smem);
  const uint32_t cum_row = (uint32_t)(((NB + 2) * 2 + 3) / 4 * 4);
  const uint32_t cum0 = sbase + 16u * (uint32_t)F, u0 = cum0 + cum_row * (uint32_t)F;
  const int64_t n_blocks = (n_rows + 31) / 32;
  auto issue = [&](int64_t b, int buf) {
    if (threadIdx.x == 0 && b < n_blocks && (b + 1) * 32 <= n_rows) {
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(&bars[buf], blk_bytes);
      ptx::bulk_g2s(stage + (size_t)buf * 32 * F, X + b * 32 * (int64_t)F, blk_bytes, &bars[buf]);
    }
  };
  for (int b = 0; b < nbuf; ++b) issue((int64_t)blockIdx.x + (int64_t)b * gridDim.x, b);
  // this warp's pairs warp, warp + NW, ... (one pass covers all: NP * NW >= F2h)
  const int npairs = warp < F2h ? min(NP, (F2h - 1 - warp) / NW + 1) : 0;
  uint32_t xoff[2 * NP], cumb[2 * NP], ub[2 * NP], hi_mask[NP];
  float lo[2 * NP], iw[2 * NP];
  const float nbm1 = (float)(NB - 1);
#pragma unroll
  for (int u = 0; u < 2 * NP; ++u) {
    // pair index clamped to the last pair, so (for even F) the pair's first
    // feature stays even and its 8-byte LDS.64 aligned
    const int f = min(2 * min(warp + (u >> 1) * NW, F2h - 1) + (u & 1), F - 1);
    xoff[u] = 4u * (uint32_t)f;
    lo[u] = ptx::lds_f32(sbase + 16u * f);
    iw[u] = ptx::lds_f32(sbase + 16u * f + 4u);
    cumb[u] = cum0 + cum_row * (uint32_t)f;
    ub[u] = u0 + 4u * ptx::lds_u32(sbase + 16u * f + 12u);
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) hi_mask[q] = 2 * (warp + q * NW) + 1 >= F ? 0u : 0xFFFFFFFFu;
  const bool even_f = (F & 1) == 0;  // pairs (2p, 2p+1) are 8-byte aligned in a row
  int it = 0;
  int buf = 0;
  uint32_t par = 0;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x, ++it) {
    float* St = stage + (size_t)buf * 32 * F;
    const int64_t row0 = blk * 32;
    if (row0 + 32 <= n_rows) {
      ptx::mbar_wait(&bars[buf], par);
    } else {
      __syncthreads();
      const int rows = (int)(n_rows - row0);
      const float* src = X + row0 * F;
      for (int e = threadIdx.x; e < 32 * F; e += blockDim.x) St[e] = e < rows * F ? src[e] : 0.f;
      __syncthreads();
    }
    const uint32_t xs = ptx::s2u(St) + 4u * (uint32_t)(lane * F);
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
    float x[2 * NP];
    uint32_t pos[2 * NP];
    if (even_f) {
      // both values of a feature pair with one LDS.64: lanes' rows start at
      // lane * 4F bytes, so the 16 lanes of a half-warp phase hit 16 distinct
      // even banks (conflict-free; two LDS.32 of odd-stride rows conflict 2-way)
#pragma unroll
      for (int u = 0; u < 2 * NP; u += 2) {
        float a, b;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(xs + xoff[u]));
        x[u] = a;
        x[u + 1] = b;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 2 * NP; ++u) x[u] = ptx::lds_f32(xs + xoff[u]);
    }
#pragma unroll
    for (int u = 0; u < 2 * NP; ++u) {
      float t = __fmul_rn(__fsub_rn(x[u], lo[u]), iw[u]);
      t = fminf(fmaxf(t, 0.f), nbm1);
      const uint32_t b = (uint32_t)t;
      pos[u] = ub[u] + 4u * ptx::lds_u16(cumb[u] + 2u * b);
    }
    // branch-free lower_bound over the 15-element window (every bucket holds
    // <= 15 thresholds; positions past the bucket hold larger ones or +inf)
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
      for (int u = 0; u < 2 * NP; ++u) {
        const float e = ptx::lds_f32(pos[u] + 4u * (uint32_t)(h - 1));
        if (e < x[u]) pos[u] += 4u * (uint32_t)h;
      }
    }
#pragma unroll
    for (int u = 0; u < 2 * NP; u += 2) {
      if (u / 2 < npairs) {
        const uint32_t c0 = isnan(x[u]) ? 0xFFFFu : (pos[u] - ub[u]) >> 2;
        uint32_t c1 = isnan(x[u + 1]) ? 0xFFFFu : (pos[u + 1] - ub[u + 1]) >> 2;
        c1 &= hi_mask[u / 2];
        dst[(size_t)(warp + (u >> 1) * NW) * 32] = c0 | (c1 << 16);
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[buf], 1u) == (uint32_t)NW - 1u) {
        done[buf] = 0;
        const int64_t nb2 = blk + (int64_t)nbuf * gridDim.x;
        if (nb2 < n_blocks && (nb2 + 1) * 32 <= n_rows) {
          ptx::fence_proxy_async();
          ptx::mbar_arrive_expect_tx(&bars[buf], blk_bytes);
          ptx::bulk_g2s(stage + (size_t)buf * 32 * F, X + nb2 * 32 * (int64_t)F, blk_bytes, &bars[buf]);
        }
      }
    }
    if (++buf == nbuf) {
      buf = 0;
      par ^= 1u;
    }
  }
}

// Bucketed binning per feature group (wide inputs whose tables do not fit all
// at once: C5-shaped 200 features x ~6.4K thresholds, NB = 8192 buckets): a
// CTA holds FG features' parameter, cum and threshold rows and a slice of row
// blocks; lane = row reads its FG values (one 16-byte load when FG = 4 and
// F % 4 == 0), then the same bucket map + 4-step window search as
// bin_bucket_kernel (5 random shared loads instead of the 13 levels of the
// Eytzinger descent).
template <int FG>
__global__ void __launch_bounds__(512, 1) bin_bucket_fg_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                               const uint8_t* __restrict__ blob, int32_t NB,
                                                               int32_t stride, uint32_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  // programmatic dependent launch: the walk kernel that consumes the codes may
  // be scheduled (and run its prologue) as SMs free up; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int F2h = (F + 1) >> 1;
  const int n_fg = (F + FG - 1) / FG;
  const int fg = blockIdx.x % n_fg;
  const int slice = blockIdx.x / n_fg, n_slices = gridDim.x / n_fg;
  const int f0 = fg * FG;
  const int nf = min(FG, F - f0);
  const uint32_t cum_row = (uint32_t)(((NB + 2) * 2 + 3) / 4 * 4);
  const uint32_t urow = 4u * (uint32_t)stride;
  // shared: params [FG][16 B] | cum [FG][cum_row] | U [FG][urow]
  uint8_t* s_cum = smem + 16 * FG;
  uint8_t* s_u = s_cum + (size_t)FG * cum_row;
  {
    const uint32_t* g = reinterpret_cast<const uint32_t*>(blob);
    const size_t g_cum = ((size_t)F * 16) / 4, g_u = ((size_t)F * 16 + (size_t)F * cum_row) / 4;
    for (int i = threadIdx.x; i < nf * 4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(smem)[i] = g[(size_t)f0 * 4 + i];
    const int cw = (int)(cum_row / 4), uw = (int)(urow / 4);
    for (int i = threadIdx.x; i < nf * cw; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_cum)[i] = g[g_cum + (size_t)(f0 + i / cw) * cw + i % cw];
    for (int i = threadIdx.x; i < nf * uw; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_u)[i] = g[g_u + (size_t)(f0 + i / uw) * uw + i % uw];
  }
  __syncthreads();
  float lo[FG], iw[FG];
  uint32_t cumb[FG], ub[FG];
#pragma unroll
  for (int q = 0; q < FG; ++q) {
    const int qq = min(q, nf - 1);
    lo[q] = reinterpret_cast<const float*>(smem)[4 * qq];
    iw[q] = reinterpret_cast<const float*>(smem)[4 * qq + 1];
    cumb[q] = ptx::s2u(s_cum) + cum_row * (uint32_t)qq;
    ub[q] = ptx::s2u(s_u) + urow * (uint32_t)qq;
  }
  const float nbm1 = (float)(NB - 1);
  const bool vec4 = FG == 4 && nf == 4 && (F & 3) == 0;
  const int64_t n_blocks = (n_rows + 31) / 32;
  for (int64_t blk = (int64_t)slice * NW + warp; blk < n_blocks; blk += (int64_t)n_slices * NW) {
    const int64_t row = blk * 32 + lane;
    const float* xr = X + (row < n_rows ? row : blk * 32) * (int64_t)F + f0;
    float x[FG];
    if (vec4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xr));
      x[0] = v.x;
      x[FG > 1 ? 1 : 0] = v.y;
      x[FG > 2 ? 2 : 0] = v.z;
      x[FG > 3 ? 3 : 0] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < FG; ++q) x[q] = q < nf ? __ldg(xr + q) : 0.f;
    }
    uint32_t pos[FG];
#pragma unroll
    for (int q = 0; q < FG; ++q) {
      float t = __fmul_rn(__fsub_rn(x[q], lo[q]), iw[q]);
      t = fminf(fmaxf(t, 0.f), nbm1);
      pos[q] = ub[q] + 4u * ptx::lds_u16(cumb[q] + 2u * (uint32_t)t);
    }
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
      for (int q = 0; q < FG; ++q) {
        const float e = ptx::lds_f32(pos[q] + 4u * (uint32_t)(h - 1));
        if (e < x[q]) pos[q] += 4u * (uint32_t)h;
      }
    }
    uint32_t cd[FG];
#pragma unroll
    for (int q = 0; q < FG; ++q) cd[q] = q >= nf ? 0u : isnan(x[q]) ? 0xFFFFu : (pos[q] - ub[q]) >> 2;
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
    if (FG == 1) {
      reinterpret_cast<uint16_t*>(dst + (size_t)(f0 >> 1) * 32)[f0 & 1] = (uint16_t)cd[0];
    } else {
#pragma unroll
      for (int q = 0; q < FG; q += 2)
        if (f0 + q < 2 * F2h) dst[(size_t)((f0 + q) >> 1) * 32] = cd[q] | (cd[q + 1 < FG ? q + 1 : q] << 16) * (q + 1 < FG);
    }
  }
}

// Bucket-entry binning (round 2; TravLayout::bke_blob, lowering.cpp
// build_entry_table): step a1's threshold-bin codes with ONE random 16-byte
// shared load per value.  b = clamp(floor((x - lo) * iw), 0, NB - 1) (the
// host's IEEE fp32 map: monotone, exact), entry e_b = {cum | cnt << 16, t0,
// t1, t2}; code = cum + [t0 < x] + [t1 < x] + [t2 < x] (pads +inf) when
// cnt <= 3, else the branch-free 4-step search in the 15-wide window of U
// from cum (rare: the map puts ~3+ buckets per threshold).  The previous
// bucketed kernel issued 5 dependent random 4-byte loads per value (~16
// shared wavefronts per warp-value, 58% of them bank conflicts).
// A CTA holds FG features' tables (~210 KB) and a slice of the 32-row blocks;
// each warp owns its blocks and double-buffers their [32][FG] fp32 tiles,
// moved by the TMA engine (cp.async.bulk.tensor.2d, no LSU wavefronts) from X
// viewed as [n_rows / R][R * F] (R = 1, 2, 4: the smallest super-row whose
// pitch is a multiple of 16 B), R boxes of {W, 32 / R} per block.  A box's
// first column must sit on a 16-byte boundary (measured: an unaligned start
// is an illegal instruction, tools/tma_probe.cu), so for R > 1 the boxes
// start at the aligned column at or below r * F + f0 and are W = FG + 4 wide.
// Rows past the last whole super-row (n_rows % R) are read directly.
// Row-tile width W (values staged per row): a box must start on a 16-byte
// column, so it begins d = (r F + f0) mod 4 values before the group when
// that is not 0 (R > 1, or FG = 2) and is rounded up to 4 values.
__host__ __device__ constexpr int bin_tile_w(int FG, int R) {
  return R == 1 ? (FG < 4 ? 4 : FG) : ((FG + (R == 2 ? 2 : 3) + 3) / 4) * 4;
}

// TAB = 2: the Eytzinger search trees (TravLayout::bin_table, 2^k - 1 slots
// per feature) for tables too large for any bucket form (C4: up to 63K
// thresholds per feature, k = 16): the top T levels of FG features' trees in
// shared memory, the k - T deeper ones read from L2 (NB := k, stride := T).
// TAB = 1: the same TMA-staged pipeline over the bucketed tables instead
// (TravLayout::bkt_blob built for feature groups: u16 cum + the 15-wide
// window search; wide inputs such as the C5 shard, whose ~6.4K thresholds per
// feature leave no room for entries) -- it replaces bin_bucket_fg_kernel's
// per-lane global row loads (32 sectors per warp load, latency-bound).
// Lockstep (epochs != nullptr; grid co-resident, launched cooperatively): the
// ceil(F / FG) feature-group CTAs of one row range otherwise drift apart on
// inputs larger than L2 and each group's sectors come from DRAM again (C3:
// 9.2 GB read for a 3.6 GB input).  Every `ipe` block iterations a CTA
// publishes its epoch (a counter per epoch) and waits until every CTA has
// finished the epoch before the previous one: at most ~2 epochs (~2 x 24 MB
// of X) are in flight, so the groups share each row's sectors through L2.
template <int FG, int R, int TAB>
__global__ void __launch_bounds__(1024, 1) bin_entry_kernel(const __grid_constant__ CUtensorMap tmx,
                                                           const float* __restrict__ X, int64_t n_rows, int64_t n_tma,
                                                           int32_t F, const uint8_t* __restrict__ blob, int32_t NB,
                                                           int32_t stride, uint32_t* __restrict__ codes,
                                                           uint32_t* __restrict__ epochs, int32_t ipe,
                                                           int32_t n_epochs) {
  extern __shared__ __align__(128) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int W = bin_tile_w(FG, R);       // staged values per row
  constexpr uint32_t kTile = 32u * W * 4u;   // bytes of one staged block
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int F2h = (F + 1) >> 1;
  const int n_fg = (F + FG - 1) / FG;
  const int fg = blockIdx.x % n_fg;
  const int slice = blockIdx.x / n_fg, n_slices = gridDim.x / n_fg;
  const int f0 = fg * FG;
  const int nf = min(FG, F - f0);
  // per feature: entries [NB][16 B] (TAB 0), cum [NB + 2] u16 rounded to 4 B
  // (TAB 1), or the top T levels of the search tree (TAB 2; no U: stride = T)
  const int P = TAB == 2 ? (1 << NB) - 1 : 1, Pt = TAB == 2 ? (1 << stride) - 1 : 1;
  const uint32_t sec2 = TAB == 0 ? 16u * (uint32_t)NB
                        : TAB == 1 ? (uint32_t)(((NB + 2) * 2 + 3) / 4 * 4)
                                   : 4u * (uint32_t)Pt;
  const int ustride = TAB == 2 ? 0 : stride;
  // shared: stage [NW][2][32][W] fp32 | params [FG][16 B] | entries / cum [FG][sec2] | U [FG][stride] | bars
  uint8_t* stage = smem;
  uint8_t* s_prm = smem + (size_t)NW * 2 * kTile;
  uint8_t* s_ent = s_prm + 16 * FG;
  uint8_t* s_u = s_ent + (size_t)FG * sec2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_u + (size_t)FG * ustride * 4);  // [NW][2] + [1] table
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NW + 1; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (TAB == 2) {  // top T levels of this group's search trees
    const float* tab = reinterpret_cast<const float*>(blob);
    float* dst = reinterpret_cast<float*>(s_ent);
    for (int i = threadIdx.x; i < nf * Pt; i += blockDim.x) dst[i] = tab[(size_t)(f0 + i / Pt) * P + i % Pt];
    if (threadIdx.x == 0) ptx::mbar_arrive(&bars[2 * NW]);
    __syncthreads();
  } else if (TAB == 1) {  // cum rows are 4-byte multiples: a plain cooperative copy of this group's tables
    const uint32_t* g = reinterpret_cast<const uint32_t*>(blob);
    const size_t g_cum = (size_t)F * 4, g_u = ((size_t)F * 16 + (size_t)F * sec2) / 4;
    const int cw = (int)(sec2 / 4), uw = stride;
    for (int i = threadIdx.x; i < nf * 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s_prm)[i] = g[(size_t)f0 * 4 + i];
    for (int i = threadIdx.x; i < nf * cw; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_ent)[i] = g[g_cum + (size_t)f0 * cw + i];
    for (int i = threadIdx.x; i < nf * uw; i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_u)[i] = g[g_u + (size_t)f0 * uw + i];
    if (threadIdx.x == 0) ptx::mbar_arrive(&bars[2 * NW]);
    __syncthreads();
  } else if (threadIdx.x == 0) {  // this group's tables: three contiguous bulk copies
    const uint32_t pb = 16u * nf, eb = 16u * (uint32_t)nf * NB, ub = 4u * (uint32_t)nf * stride;
    ptx::mbar_arrive_expect_tx(&bars[2 * NW], pb + eb + ub);
    ptx::bulk_g2s(s_prm, blob + (size_t)f0 * 16, pb, &bars[2 * NW]);
    const uint8_t* ge = blob + (size_t)F * 16 + (size_t)f0 * NB * 16;
    for (uint32_t o = 0; o < eb;) {  // <= 1 MB per bulk copy
      const uint32_t n = min(eb - o, 1u << 20);
      ptx::bulk_g2s(s_ent + o, ge + o, n, &bars[2 * NW]);
      o += n;
    }
    ptx::bulk_g2s(s_u, blob + (size_t)F * 16 + (size_t)F * NB * 16 + (size_t)f0 * stride * 4, ub, &bars[2 * NW]);
  }
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t step = (int64_t)n_slices * NW;
  const uint32_t st0 = ptx::s2u(stage) + (uint32_t)warp * 2u * kTile;
  uint64_t* wb = bars + 2 * warp;
  auto issue = [&](int64_t b, int buf) {
    if (b >= n_blocks) return;
    ptx::mbar_arrive_expect_tx(&wb[buf], kTile);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t dst = st0 + (uint32_t)buf * kTile + (uint32_t)r * (kTile / R);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              dst),
          "l"(&tmx), "r"((r * F + f0) & ~3), "r"((int)(b * (32 / R))), "r"(ptx::s2u(&wb[buf]))
          : "memory");
    }
  };
  int64_t blk = (int64_t)slice * NW + warp;
  if (lane == 0) {
    issue(blk, 0);
    issue(blk + step, 1);
  }
  ptx::mbar_wait(&bars[2 * NW], 0);
  float lo[FG], iw[FG];
  uint32_t eb_[FG], ub_[FG];
#pragma unroll
  for (int q = 0; q < FG; ++q) {
    const int qq = min(q, nf - 1);
    lo[q] = TAB == 2 ? 0.f : reinterpret_cast<const float*>(s_prm)[4 * qq];
    iw[q] = TAB == 2 ? 0.f : reinterpret_cast<const float*>(s_prm)[4 * qq + 1];
    eb_[q] = ptx::s2u(s_ent) + sec2 * (uint32_t)qq;
    ub_[q] = ptx::s2u(s_u) + 4u * (uint32_t)stride * (uint32_t)qq;
  }
  const float nbm1 = (float)(NB - 1);
  // lane's row within the block: box r = lane % R, super-row s = lane / R,
  // its first value d = (r * F + f0) % 4 columns into the box row
  const int xr = lane % R;
  const uint32_t xoff = ((uint32_t)xr * (32 / R) + (uint32_t)(lane / R)) * W * 4u + 4u * (uint32_t)((xr * F + f0) & 3);
  // every warp of the CTA runs the same iteration count (the first warp's:
  // the largest), so the epoch barriers below see all of them
  const int64_t first = (int64_t)slice * NW;
  const int64_t n_iter = first < n_blocks ? (n_blocks - 1 - first) / step + 1 : 0;
  for (int it = 0; it < n_iter; blk += step, ++it) {
    if (epochs != nullptr && it > 0 && it % ipe == 0) {
      const int e = it / ipe;  // epoch e begins: this CTA finished epoch e - 1
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(epochs + (e - 1)) : "memory");
        if (e >= 2) {  // wait until every CTA finished epoch e - 2
          uint32_t v = 0;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(epochs + (e - 2)) : "memory");
            if (v >= gridDim.x) break;
            __nanosleep(64);
          }
        }
      }
      __syncthreads();
    }
    if (blk >= n_blocks) continue;  // this warp's blocks ran out (the CTA's last iteration)
    const int buf = it & 1;
    ptx::mbar_wait(&wb[buf], (uint32_t)(it >> 1) & 1u);
    const uint32_t xa = st0 + (uint32_t)buf * kTile + xoff;
    float x[FG];
    if (R == 1 && FG % 4 == 0) {  // 16-byte aligned
#pragma unroll
      for (int q = 0; q < FG; q += 4)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x[q]), "=f"(x[q + (FG > 1 ? 1 : 0)]), "=f"(x[q + (FG > 2 ? 2 : 0)]),
                       "=f"(x[q + (FG > 3 ? 3 : 0)])
                     : "r"(xa + 4u * q));
    } else if (R <= 2 && FG % 2 == 0) {  // d in {0, 2}: 8-byte aligned
#pragma unroll
      for (int q = 0; q < FG; q += 2)
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x[q]), "=f"(x[q + 1]) : "r"(xa + 4u * q));
    } else {
#pragma unroll
      for (int q = 0; q < FG; ++q) x[q] = ptx::lds_f32(xa + 4u * q);
    }
    const int64_t row = blk * 32 + lane;
    if (row >= n_tma && row < n_rows) {  // past the last whole super-row
#pragma unroll
      for (int q = 0; q < FG; ++q) x[q] = q < nf ? __ldg(X + row * F + f0 + q) : 0.f;
    }
    __syncwarp();
    if (lane == 0) {  // every lane holds its values: refill this buffer
      ptx::fence_proxy_async();
      issue(blk + 2 * step, buf);
    }
    uint32_t cd[FG];
    if (TAB == 2) {  // Eytzinger descents, the FG chains interleaved: T levels in shared memory, then L2
      uint32_t A[FG], c4[FG];
#pragma unroll
      for (int q = 0; q < FG; ++q) {
        A[q] = eb_[q];
        c4[q] = 4u - eb_[q];
      }
      for (int l = 0; l < stride; ++l) {
#pragma unroll
        for (int q = 0; q < FG; ++q) {
          const float e = ptx::lds_f32(A[q]);
          A[q] = 2u * A[q] + c4[q];
          if (e < x[q]) A[q] += 4u;
        }
      }
      uint32_t i[FG];
      const float* tg[FG];
#pragma unroll
      for (int q = 0; q < FG; ++q) {
        i[q] = (A[q] + c4[q] - 4u) >> 2;
        tg[q] = reinterpret_cast<const float*>(blob) + (size_t)(f0 + min(q, nf - 1)) * P;
      }
      for (int l = stride; l < NB; ++l) {
#pragma unroll
        for (int q = 0; q < FG; ++q) i[q] = 2u * i[q] + 1u + (__ldg(tg[q] + i[q]) < x[q] ? 1u : 0u);
      }
#pragma unroll
      for (int q = 0; q < FG; ++q) cd[q] = q >= nf ? 0u : isnan(x[q]) ? 0xFFFFu : i[q] - (uint32_t)P;
    }
#pragma unroll
    for (int q = 0; q < FG; ++q) {
      if (TAB == 2) continue;
      float t = __fmul_rn(__fsub_rn(x[q], lo[q]), iw[q]);
      t = fminf(fmaxf(t, 0.f), nbm1);
      if (TAB == 1) {  // cum[b] + lower_bound in the 15-wide window
        uint32_t pos = ub_[q] + 4u * ptx::lds_u16(eb_[q] + 2u * (uint32_t)t);
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
          if (ptx::lds_f32(pos + 4u * (uint32_t)(h - 1)) < x[q]) pos += 4u * (uint32_t)h;
        cd[q] = q >= nf ? 0u : isnan(x[q]) ? 0xFFFFu : (pos - ub_[q]) >> 2;
        continue;
      }
      uint32_t e0, e1, e2, e3;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3)
                   : "r"(eb_[q] + 16u * (uint32_t)t));
      uint32_t c = (e0 & 0xFFFFu) + (__uint_as_float(e1) < x[q] ? 1u : 0u) + (__uint_as_float(e2) < x[q] ? 1u : 0u) +
                   (__uint_as_float(e3) < x[q] ? 1u : 0u);
      if (e0 > 0x3FFFFu) {  // cnt > 3: lower_bound in the 15-wide window from cum
        uint32_t pos = ub_[q] + 4u * (e0 & 0xFFFFu);
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
          if (ptx::lds_f32(pos + 4u * (uint32_t)(h - 1)) < x[q]) pos += 4u * (uint32_t)h;
        c = (pos - ub_[q]) >> 2;
      }
      cd[q] = q >= nf ? 0u : isnan(x[q]) ? 0xFFFFu : c;
    }
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
#pragma unroll
    for (int q = 0; q < FG; q += 2)
      if (q < nf) dst[(size_t)((f0 + q) >> 1) * 32] = cd[q] | (cd[q + 1] << 16);
  }
  if (epochs != nullptr) {  // the epochs this CTA did not publish in the loop: done
    __syncthreads();
    if (threadIdx.x == 0)
      for (int e = n_iter > 0 ? (int)((n_iter - 1) / ipe) : 0; e < n_epochs; ++e)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(epochs + e) : "memory");
  }
}

// Feature-group binning for search tables too large to hold for all features
// at once (C5-shaped shards: 200 features x 8191-slot trees = 6.5 MB): a CTA
// owns FG features and a range of 32-row blocks; lane = row reads its row's FG
// contiguous values straight from global memory and descends FG search trees
// (FG chains).  The top T levels of each tree -- the first 2^T - 1 slots of the
// Eytzinger array -- sit in shared memory; deeper levels (T < k: tables of
// 2^16 - 1 slots, 256 KB per feature) are read from global memory (L2).  FG is
// 4 or 2 (whole code pairs: one coalesced u32 store per pair), or 1 (u16 stores).
template <int FG>
__global__ void __launch_bounds__(512, 1) bin_fg_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                        const float* __restrict__ table, int32_t k, int32_t T,
                                                        uint32_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  // programmatic dependent launch: the walk kernel that consumes the codes may
  // be scheduled (and run its prologue) as SMs free up; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int P = (1 << k) - 1, Pt = (1 << T) - 1;
  const int F2h = (F + 1) >> 1;
  const int n_fg = (F + FG - 1) / FG;
  const int fg = blockIdx.x % n_fg;
  const int slice = blockIdx.x / n_fg, n_slices = gridDim.x / n_fg;
  const int f0 = fg * FG;
  const int nf = min(FG, F - f0);
  {
    float* dst = reinterpret_cast<float*>(smem);
    for (int i = threadIdx.x; i < nf * Pt; i += blockDim.x) dst[i] = table[(size_t)(f0 + i / Pt) * P + i % Pt];
  }
  __syncthreads();
  const uint32_t tab_s = ptx::s2u(smem);
  const int64_t n_blocks = (n_rows + 31) / 32;
  for (int64_t blk = (int64_t)slice * NW + warp; blk < n_blocks; blk += (int64_t)n_slices * NW) {
    const int64_t row = blk * 32 + lane;
    const float* xr = X + (row < n_rows ? row : blk * 32) * (int64_t)F + f0;
    float x[FG];
#pragma unroll
    for (int u = 0; u < FG; ++u) x[u] = u < nf ? __ldg(xr + u) : 0.f;
    uint32_t A[FG], c4[FG];
#pragma unroll
    for (int u = 0; u < FG; ++u) {
      A[u] = tab_s + (uint32_t)(min(u, nf - 1) * Pt) * 4u;
      c4[u] = 4u - A[u];
    }
    for (int s = 0; s < T; ++s) {
#pragma unroll
      for (int u = 0; u < FG; ++u) {
        const float e = ptx::lds_f32(A[u]);
        A[u] = 2u * A[u] + c4[u];
        if (e < x[u]) A[u] += 4u;
      }
    }
    uint32_t i[FG];  // Eytzinger index after T levels
#pragma unroll
    for (int u = 0; u < FG; ++u) i[u] = (A[u] + c4[u] - 4u) >> 2;
    for (int s = T; s < k; ++s) {
#pragma unroll
      for (int u = 0; u < FG; ++u) {
        const float e = __ldg(table + (size_t)(f0 + min(u, nf - 1)) * P + i[u]);
        i[u] = 2u * i[u] + 1u + (e < x[u] ? 1u : 0u);
      }
    }
    uint32_t cd[FG];
#pragma unroll
    for (int u = 0; u < FG; ++u) cd[u] = u >= nf ? 0u : isnan(x[u]) ? 0xFFFFu : i[u] - (uint32_t)P;
    uint32_t* dst = codes + (size_t)blk * F2h * 32 + lane;
    if (FG == 1) {
      reinterpret_cast<uint16_t*>(dst + (size_t)(f0 >> 1) * 32)[f0 & 1] = (uint16_t)cd[0];
    } else {
#pragma unroll
      for (int u = 0; u < FG; u += 2)
        if (f0 + u < 2 * F2h) dst[(size_t)((f0 + u) >> 1) * 32] = cd[u] | (cd[u + 1 < FG ? u + 1 : u] << 16) * (u + 1 < FG);
    }
  }
}

// Pre-transposed input (FMT_HEAP_T): X [N][F] fp32 row-major -> [n_blocks][F][32]
// fp32, the traversal's feature-major 32-row block layout, written once so
// that every chunk CTA bulk-copies blocks with no per-chunk transpose.
__global__ void __launch_bounds__(512) xpose_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                    float* __restrict__ XT) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int S = F | 1;
  float* St = reinterpret_cast<float*>(smem) + (size_t)warp * 32 * S;
  const int64_t n_blocks = (n_rows + 31) / 32;
  for (int64_t blk = (int64_t)blockIdx.x * NW + warp; blk < n_blocks; blk += (int64_t)gridDim.x * NW) {
    const int64_t row0 = blk * 32;
    const int rows = (int)(n_rows - row0 < 32 ? n_rows - row0 : 32);
    const float* src = X + row0 * F;
    for (int r = 0; r < 32; ++r)
      for (int f = lane; f < F; f += 32) {
        const uint32_t dsts = ptx::s2u(St + r * S + f);
        const float* g = src + (int64_t)(r < rows ? r : 0) * F + f;
        const uint32_t nbytes = r < rows ? 4u : 0u;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dsts), "l"(g), "r"(nbytes) : "memory");
      }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    float* dst = XT + blk * 32 * (int64_t)F;
    for (int f = 0; f < F; ++f) dst[f * 32 + lane] = St[lane * S + f];
    __syncwarp();
  }
}

// ------------------------------------------------------------- launchers ----
static std::atomic<uint64_t> g_xpose_smem{0};  // xpose_kernel's shared-memory opt-in, per device

static int64_t l2_bytes(int dev) {
  static std::atomic<int64_t> cached[64];
  if (dev >= 0 && dev < 64 && cached[dev].load()) return cached[dev].load();
  int b = 0;
  cudaDeviceGetAttribute(&b, cudaDevAttrL2CacheSize, dev);
  if (dev >= 0 && dev < 64) cached[dev].store(b);
  return b;
}

static int num_sms(int dev) {
  static std::atomic<int> cached[64];  // per device; concurrent predicts may fill it
  if (dev >= 0 && dev < 64) {
    const int c = cached[dev].load(std::memory_order_relaxed);
    if (c) return c;
  }
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev].store(n, std::memory_order_relaxed);
  return n;
}

// Tensor map of X [n_rows][F] fp32 viewed as [n_sr][R * F] (pitch R * F * 4,
// a multiple of 16 B), box {W, 32 / R}: bin_entry_kernel's row tiles.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static cudaError_t encode_x_map(CUtensorMap* tm, const float* X, int F, int R, int64_t n_sr, int W) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn || n_sr <= 0) return cudaErrorNotSupported;
  const cuuint64_t gdim[2] = {(cuuint64_t)R * F, (cuuint64_t)n_sr};
  const cuuint64_t gstr[1] = {(cuuint64_t)R * F * 4};
  const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)(32 / R)}, es[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorNotSupported;
}

// Row slices per feature group for one-CTA-per-SM binning grids of n_fg x
// slices CTAs: the fewest slices whose waves keep >= 90% of the SMs busy
// (C5 shard: 50 groups -> 8 slices, 400 CTAs in 3 waves; 100 CTAs would idle
// a third of the SMs and 150 would leave 2 CTAs for a second wave).
static int64_t pick_slices(int n_fg, int sms, int64_t max_slices) {
  max_slices = std::max<int64_t>(1, max_slices);
  for (int64_t s = std::max(1, sms / n_fg); s <= std::min<int64_t>(max_slices, 64); ++s) {
    const int64_t ctas = (int64_t)n_fg * s, waves = (ctas + sms - 1) / sms;
    if (ctas * 10 >= waves * sms * 9) return s;
  }
  return std::max<int64_t>(1, std::min<int64_t>(max_slices, std::max(1, sms / n_fg)));
}

// Runs the traversal over all rows.  want: 0 predict, 1 proba, 2 raw, 3 apply.
// Step a1 in coded form: bin the rows once into [n_blocks][F2/2][32][2] u16
// code blocks (stream-ordered allocation, returned in *codes_out).
static cudaError_t launch_binning(const bridger_model* m, const TravLayout& L, const float* X, int64_t n_rows, int sms,
                                  cudaStream_t st, void** codes_out) {
  void* codes = nullptr;
  cudaError_t err = cudaSuccess;
  // step a1 in coded form: bin the rows once (all chunks reuse the codes)
  const int64_t nbk = (n_rows + 31) / 32;
  const int F2 = (m->F + 1) & ~1;
  err = cudaMallocAsync(&codes, (size_t)nbk * 32 * F2 * 2, st);
  if (err != cudaSuccess) return err;
  // Bucketed binning where the per-warp-staged Eytzinger kernel does not fit
  // (wide tables, e.g. C3): measured on B200, C3 2.39 -> 2.23 ms; C2 (staged
  // kernel fits) 0.095 ms Eytzinger vs 0.15 bucketed -- both are bound by
  // random shared-memory wavefronts (~15-17 per warp-value either way).
  // BRIDGER_BIN: tests force a variant ('b' bucketed, 'f'/'c' Eytzinger).
  const char* bin_env = std::getenv("BRIDGER_BIN");
  const int P0 = (1 << L.bin_k) - 1;
  const bool staged_fits = (m->F * P0 * 4 + 127) / 128 * 128 + 8 * (2 * 128 * m->F + 16) <= 232448;
  const bool want_bkt = bin_env ? (bin_env[0] == 'b' || bin_env[0] == 'g') : !staged_fits;
  // bucket-entry kernel (TMA-staged row tiles) when built and X is 16-byte
  // aligned; BRIDGER_BIN=e forces it, any other BRIDGER_BIN value avoids it
  // (BRIDGER_BIN=E: required -- an error when it cannot run; tests)
  // Default only where it measured faster: 16-byte-aligned rows (R = 1) and
  // an input no larger than L2, which stays resident while the ceil(F / FG)
  // feature-group CTAs each read their columns of every row (C2, 112 MB:
  // binning 0.080 -> 0.067 ms, step 0.390 -> 0.375 ms).  On C3
  // (10M x 90, 3.6 GB) the groups drift apart and every group's sectors come
  // from DRAM (9.2 GB read vs 3.6), so despite 23% fewer shared wavefronts it
  // ties the all-features bucketed kernel (2.04 ms each).
  const int R = (m->F * 4) % 16 == 0 ? 1 : (m->F * 8) % 16 == 0 ? 2 : 4;
  const bool fits_l2 = (double)n_rows * m->F * 4 <= (double)l2_bytes(m->device);
  const char* lock_env = std::getenv("BRIDGER_BIN_LOCK");
  const bool lock_ok = !fits_l2 && !(lock_env && lock_env[0] == '0');
  const bool want_bke = bin_env ? (bin_env[0] == 'e' || bin_env[0] == 'E')
                                : (R == 1 && fits_l2) || (lock_ok && lock_env && lock_env[0] == '1');
  if (L.bke_nb > 0 && !L.stream && want_bke && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && n_rows >= 128) {
    const int64_t n_sr = n_rows / R;
    CUtensorMap tm;
    err = encode_x_map(&tm, X, m->F, R, n_sr, bin_tile_w(L.bke_fg, R));
    if (err == cudaSuccess) {
      const int FG = L.bke_fg;
      const int n_fg = (m->F + FG - 1) / FG;
      // as many warps (chains in flight) as fit next to the tables: 32, else 16
      auto bsm_of = [&](int w) {
        return w * 2 * 32 * bin_tile_w(FG, R) * 4 + 16 * FG + FG * L.bke_nb * 16 + FG * L.bke_stride * 4 + 8 * (2 * w + 1);
      };
      int nw = 32;
      if (const char* e = std::getenv("BRIDGER_BIN_WARPS")) nw = std::atoi(e) >= 32 ? 32 : 16;
      if (bsm_of(nw) > 232448) nw = 16;
      const int bsm = bsm_of(nw);
      const int64_t slices = pick_slices(n_fg, sms, (nbk + nw - 1) / nw);
      using BinE = void (*)(const CUtensorMap, const float*, int64_t, int64_t, int32_t, const uint8_t*, int32_t, int32_t,
                            uint32_t*, uint32_t*, int32_t, int32_t);
      BinE k = nullptr;
      if (FG == 8)
        k = R == 1 ? bin_entry_kernel<8, 1, 0> : R == 2 ? bin_entry_kernel<8, 2, 0> : bin_entry_kernel<8, 4, 0>;
      else
        k = R == 1 ? bin_entry_kernel<4, 1, 0> : R == 2 ? bin_entry_kernel<4, 2, 0> : bin_entry_kernel<4, 4, 0>;
      static std::atomic<uint64_t> attr_e[6];
      smem_opt_in(reinterpret_cast<const void*>(k), attr_e[(FG == 8 ? 3 : 0) + (R == 1 ? 0 : R == 2 ? 1 : 2)]);
      const int grid = (int)(n_fg * slices);
      uint32_t* epochs = nullptr;
      int32_t ipe = 1, n_epochs = 0;
      if (lock_ok && grid <= sms) {
        // lockstep epochs of ~24 MB of X (see the kernel); co-residency of
        // every CTA is guaranteed by the cooperative launch below
        const int64_t step = slices * nw;
        const int64_t n_iter = (nbk + step - 1) / step;
        ipe = (int32_t)std::max<int64_t>(1, (24LL << 20) / std::max<int64_t>(1, step * 32 * m->F * 4));
        n_epochs = (int32_t)((n_iter + ipe - 1) / ipe);
        if (cudaMallocAsync(reinterpret_cast<void**>(&epochs), (size_t)std::max(1, n_epochs) * 4, st) != cudaSuccess ||
            cudaMemsetAsync(epochs, 0, (size_t)std::max(1, n_epochs) * 4, st) != cudaSuccess) {
          cudaGetLastError();
          if (epochs) cudaFreeAsync(epochs, st);
          epochs = nullptr;
        }
      }
      uint32_t* codes32 = static_cast<uint32_t*>(codes);
      const uint8_t* bke = m->d_bke;
      const int64_t n_tma_rows = n_sr * R;
      const int32_t Fi = m->F, nbi = L.bke_nb, sti = L.bke_stride;
      if (epochs) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(nw * 32);
        cfg.dynamicSmemBytes = bsm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        err = cudaLaunchKernelEx(&cfg, k, tm, X, n_rows, n_tma_rows, Fi, bke, nbi, sti, codes32, epochs, ipe, n_epochs);
        cudaFreeAsync(epochs, st);
        if (err != cudaSuccess) {  // not co-resident (e.g. a shared GPU): the free-running kernel
          cudaGetLastError();
          k<<<grid, nw * 32, bsm, st>>>(tm, X, n_rows, n_tma_rows, Fi, bke, nbi, sti, codes32, nullptr, 1, 0);
          err = cudaSuccess;
        }
      } else {
        k<<<grid, nw * 32, bsm, st>>>(tm, X, n_rows, n_tma_rows, Fi, bke, nbi, sti, codes32, nullptr, 1, 0);
        err = cudaSuccess;
      }
      count_launch();
      if (err == cudaSuccess) err = cudaGetLastError();
      if (err != cudaSuccess) {
        cudaFreeAsync(codes, st);
        return err;
      }
      *codes_out = codes;
      return cudaSuccess;
    }
    err = cudaSuccess;  // no tensor map (driver entry point missing): the other kernels
  }
  if (bin_env && bin_env[0] == 'E') {
    cudaFreeAsync(codes, st);
    return cudaErrorNotSupported;
  }
  if (L.bkt_nb > 0 && L.bkt_fg == 4 && !L.stream && want_bkt && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
      n_rows >= 128 && !(bin_env && bin_env[0] == 'g')) {
    // per-feature-group bucketed tables with TMA-staged row tiles
    // (bin_entry_kernel<4, R, 1>) when they fit next to the staging;
    // BRIDGER_BIN=g keeps the direct-load kernel below
    const int R = (m->F * 4) % 16 == 0 ? 1 : (m->F * 8) % 16 == 0 ? 2 : 4;
    const int W = bin_tile_w(4, R);
    const int n_fg = (m->F + 3) / 4;
    const int cum_row = ((L.bkt_nb + 2) * 2 + 3) / 4 * 4;
    int nw = 32;
    if (const char* e = std::getenv("BRIDGER_BIN_WARPS")) nw = std::atoi(e) >= 32 ? 32 : 16;
    auto bsm_of = [&](int w) { return w * 2 * 32 * W * 4 + 4 * (16 + cum_row + 4 * L.bkt_stride) + 8 * (2 * w + 1); };
    while (nw > 4 && bsm_of(nw) > 232448) nw /= 2;
    CUtensorMap tm;
    const int64_t n_sr = n_rows / R;
    if (bsm_of(nw) <= 232448 && encode_x_map(&tm, X, m->F, R, n_sr, W) == cudaSuccess) {
      using BinE = void (*)(const CUtensorMap, const float*, int64_t, int64_t, int32_t, const uint8_t*, int32_t, int32_t,
                            uint32_t*, uint32_t*, int32_t, int32_t);
      BinE k = R == 1 ? bin_entry_kernel<4, 1, 1> : R == 2 ? bin_entry_kernel<4, 2, 1> : bin_entry_kernel<4, 4, 1>;
      static std::atomic<uint64_t> attr_t[3];
      smem_opt_in(reinterpret_cast<const void*>(k), attr_t[R == 1 ? 0 : R == 2 ? 1 : 2]);
      const int64_t slices = pick_slices(n_fg, sms, (nbk + nw - 1) / nw);
      k<<<(int)(n_fg * slices), nw * 32, bsm_of(nw), st>>>(
          tm, X, n_rows, n_sr * R, m->F, m->d_bkt, L.bkt_nb, L.bkt_stride, static_cast<uint32_t*>(codes), nullptr, 1, 0);
      count_launch();
      err = cudaGetLastError();
      if (err != cudaSuccess) {
        cudaFreeAsync(codes, st);
        return err;
      }
      *codes_out = codes;
      return cudaSuccess;
    }
  }
  if (L.bkt_nb > 0 && L.bkt_fg > 0 && !L.stream && want_bkt) {
    // per-feature-group bucketed binning
    const int FG = L.bkt_fg;  // 4
    const int n_fg = (m->F + FG - 1) / FG;
    const int cum_row = ((L.bkt_nb + 2) * 2 + 3) / 4 * 4;
    const int bsm = FG * (16 + cum_row + 4 * L.bkt_stride) + 64;
    const int64_t slices = std::max<int64_t>(1, std::min<int64_t>((2 * sms + n_fg - 1) / n_fg, (nbk + 15) / 16));
    static std::atomic<uint64_t> attr_fg{0};
    smem_opt_in(reinterpret_cast<const void*>(bin_bucket_fg_kernel<4>), attr_fg);
    bin_bucket_fg_kernel<4><<<(int)(n_fg * slices), 512, bsm, st>>>(X, n_rows, m->F, m->d_bkt, L.bkt_nb,
                                                                      L.bkt_stride, static_cast<uint32_t*>(codes));
    count_launch();
    err = cudaGetLastError();
    if (err != cudaSuccess) {
      cudaFreeAsync(codes, st);
      return err;
    }
    *codes_out = codes;
    return cudaSuccess;
  }
  if (L.bkt_nb > 0 && L.bkt_fg == 0 && !L.stream && want_bkt) {
    // bucketed binning (all features' tables + one shared double-buffered block)
    const int f2h = (m->F + 1) >> 1;
    // >= 3 pairs (6 search chains) per warp when the feature count allows
    int nw = std::max(4, std::min(16, (f2h + 2) / 3));
    if (const char* e = std::getenv("BRIDGER_BIN_WARPS")) nw = std::max(1, std::min(16, std::atoi(e)));
    const int np = (f2h + nw - 1) / nw;  // pairs per warp: one pass
    const int blob = (int)L.bkt_blob.size();
    // three staged blocks when they fit (more DRAM reads in flight), else two
    int nbuf = (blob + 127) / 128 * 128 + 3 * 128 * m->F + 48 <= 232448 ? 3 : 2;
    if (const char* e = std::getenv("BRIDGER_BIN_NBUF")) nbuf = std::max(2, std::min(nbuf, std::atoi(e)));
    const int bsm = (blob + 127) / 128 * 128 + nbuf * 128 * m->F + 16 * nbuf;
    using BinB = void (*)(const float*, int64_t, int32_t, const uint8_t*, int32_t, int32_t, int32_t, uint32_t*);
    const BinB bks[8] = {bin_bucket_kernel<1>, bin_bucket_kernel<2>, bin_bucket_kernel<3>, bin_bucket_kernel<4>,
                         bin_bucket_kernel<5>, bin_bucket_kernel<6>, bin_bucket_kernel<7>, bin_bucket_kernel<8>};
    if (np <= 8 && bsm <= 232448) {
      auto bk = bks[np - 1];
      static std::atomic<uint64_t> attr[8];
      smem_opt_in(reinterpret_cast<const void*>(bk), attr[np - 1]);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nbk, sms));
      bk<<<grid, nw * 32, bsm, st>>>(X, n_rows, m->F, m->d_bkt, blob, L.bkt_nb, nbuf, static_cast<uint32_t*>(codes));
      count_launch();
      err = cudaGetLastError();
      if (err != cudaSuccess) {
        cudaFreeAsync(codes, st);
        return err;
      }
      *codes_out = codes;
      return cudaSuccess;
    }
  }
  const int P = (1 << L.bin_k) - 1;
  const int fixed = (m->F * P * 4 + 127) / 128 * 128;
  // per-warp staging (bulk-copied dense blocks) when the table leaves room
  // for >= 8 warps of double-buffered staging, else one CTA-shared block
  int nwb = 16;
  while (nwb > 1 && fixed + nwb * (2 * 128 * m->F + 16) > 232448) --nwb;
  bool stage = nwb >= 8;
  bool coop = !stage && fixed + 2 * 128 * m->F + 32 <= 232448;
  if (const char* e = std::getenv("BRIDGER_BIN")) {  // tests: force a binning variant where it fits
    if (e[0] == 'f') stage = coop = false;
    if (e[0] == 'c' && fixed + 2 * 128 * m->F + 32 <= 232448) { stage = false; coop = true; }
  }
  if (!stage) nwb = 16;
  // cooperative binning: 16 warps (measured on B200 for C3, 45 feature pairs:
  // 16 warps x 3 pairs 2.6 ms, 12 x 4 2.8, 8 x 6 3.1, 6 x 8 5.0 -- latency,
  // not per-block overhead, bounds it); BRIDGER_BIN_WARPS overrides
  if (coop) {
    if (const char* e = std::getenv("BRIDGER_BIN_WARPS")) nwb = std::max(1, std::min(16, std::atoi(e)));
  }
  const int bsmem = fixed + (stage ? nwb * (2 * 128 * m->F + 16) : coop ? 2 * 128 * m->F + 32 : 0);
  // staged kernel: NP pairs per pass, passes sized so that no chain is wasted
  const int f2h = (m->F + 1) >> 1;
  const int npass = (f2h + 6) / 7;
  const int nps = (f2h + npass - 1) / npass;  // 1..7
  using BinK = void (*)(const float*, int64_t, int32_t, const float*, int32_t, uint32_t*);
  const BinK kerns[2][7] = {
      {bin_kernel<1, 1>, bin_kernel<2, 1>, bin_kernel<3, 1>, bin_kernel<4, 1>, bin_kernel<5, 1>, bin_kernel<6, 1>,
       bin_kernel<7, 1>},
      {bin_kernel<1, 2>, bin_kernel<2, 2>, bin_kernel<3, 2>, bin_kernel<4, 2>, bin_kernel<5, 2>, bin_kernel<6, 2>,
       bin_kernel<7, 2>}};
  const int np = std::min(6, (f2h + nwb - 1) / nwb);  // pairs per warp pass (coop)
  const BinK coops[6] = {bin_coop_kernel<1>, bin_coop_kernel<2>, bin_coop_kernel<3>, bin_coop_kernel<4>,
                         bin_coop_kernel<5>, bin_coop_kernel<6>};
  auto bk = coop ? coops[np - 1] : kerns[m->F % 2 == 0 ? 1 : 0][nps - 1];
  int bsm = bsmem;
  int64_t want_ctas = coop ? nbk : (nbk + nwb - 1) / nwb;
  int fgsz = 0, fg_levels = 0;
  if (!stage && !coop) {
    // feature groups: FG features' tables per CTA, whole code pairs when they
    // fit; 2^16-slot tables: pairs with their top 14 levels in shared memory
    fgsz = 4 * P * 4 <= 200 * 1024 ? 4 : 2 * P * 4 <= 200 * 1024 ? 2 : P * 4 <= 200 * 1024 ? 1 : 2;
    fg_levels = L.bin_k;
    while (fgsz * ((1 << fg_levels) - 1) * 4 > 200 * 1024) --fg_levels;
    bsm = fgsz * ((1 << fg_levels) - 1) * 4;
    const int n_fg = (m->F + fgsz - 1) / fgsz;
    // slices of row blocks per feature group: fill the SMs, each slice >= 16 blocks
    const int64_t slices = std::max<int64_t>(1, std::min<int64_t>((2 * sms + n_fg - 1) / n_fg, (nbk + 15) / 16));
    want_ctas = n_fg * slices;
    nwb = 16;
  }
  cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bk, nwb * 32, bsm);
  const int bgrid = fgsz ? (int)want_ctas
                         : (int)std::max<int64_t>(1, std::min<int64_t>(want_ctas, (int64_t)sms * std::max(1, occ)));
  if (fgsz == 2 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && n_rows >= 128 && !(bin_env && bin_env[0] == 'g')) {
    // the same feature groups with TMA-staged row tiles (bin_entry_kernel<2, R, 2>)
    const int R = (m->F * 4) % 16 == 0 ? 1 : (m->F * 8) % 16 == 0 ? 2 : 4;
    const int W = bin_tile_w(2, R);
    const int n_fg = (m->F + 1) / 2;
    int nw = 32;
    if (const char* e = std::getenv("BRIDGER_BIN_WARPS")) nw = std::atoi(e) >= 32 ? 32 : 16;
    auto bsm_of = [&](int w) { return w * 2 * 32 * W * 4 + 2 * 16 + bsm + 8 * (2 * w + 1); };
    while (nw > 4 && bsm_of(nw) > 232448) nw /= 2;
    CUtensorMap tm;
    const int64_t n_sr = n_rows / R;
    if (bsm_of(nw) <= 232448 && encode_x_map(&tm, X, m->F, R, n_sr, W) == cudaSuccess) {
      using BinE = void (*)(const CUtensorMap, const float*, int64_t, int64_t, int32_t, const uint8_t*, int32_t, int32_t,
                            uint32_t*, uint32_t*, int32_t, int32_t);
      BinE k = R == 1 ? bin_entry_kernel<2, 1, 2> : R == 2 ? bin_entry_kernel<2, 2, 2> : bin_entry_kernel<2, 4, 2>;
      static std::atomic<uint64_t> attr_y[3];
      smem_opt_in(reinterpret_cast<const void*>(k), attr_y[R == 1 ? 0 : R == 2 ? 1 : 2]);
      const int64_t slices = pick_slices(n_fg, sms, (nbk + nw - 1) / nw);
      k<<<(int)(n_fg * slices), nw * 32, bsm_of(nw), st>>>(tm, X, n_rows, n_sr * R, m->F,
                                                            reinterpret_cast<const uint8_t*>(m->d_bin_table), L.bin_k,
                                                            fg_levels, static_cast<uint32_t*>(codes), nullptr, 1, 0);
      count_launch();
      err = cudaGetLastError();
      if (err != cudaSuccess) {
        cudaFreeAsync(codes, st);
        return err;
      }
      *codes_out = codes;
      return cudaSuccess;
    }
  }
  if (fgsz) {
    auto fk = fgsz == 4 ? bin_fg_kernel<4> : fgsz == 2 ? bin_fg_kernel<2> : bin_fg_kernel<1>;
    cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    fk<<<bgrid, nwb * 32, bsm, st>>>(X, n_rows, m->F, m->d_bin_table, L.bin_k, fg_levels,
                                     static_cast<uint32_t*>(codes));
  } else {
    bk<<<bgrid, nwb * 32, bsm, st>>>(X, n_rows, m->F, m->d_bin_table, L.bin_k, static_cast<uint32_t*>(codes));
  }
  count_launch();
  err = cudaGetLastError();
  if (err != cudaSuccess) {
    cudaFreeAsync(codes, st);
    return err;
  }
  *codes_out = codes;
  return cudaSuccess;
}

cudaError_t trav_run(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                     int32_t total_trees, cudaStream_t st, void* const* scatter, int64_t rows_per_rank) {
  const TravLayout& L = m->trav;
  const int n_chunks = (int)L.chunks.size();
  TravParams p{};
  p.X = X;
  p.n_rows = n_rows;
  p.F = m->F;
  p.K = m->K;
  p.data = static_cast<const uint8_t*>(m->d_trav_data);
  p.chunks = static_cast<const TravChunk*>(m->d_trav_chunks);
  p.n_chunks = n_chunks;
  const int sms = num_sms(m->device);
  int32_t maxc = 0;
  for (auto& c : L.chunks) maxc = std::max(maxc, c.bytes);
  p.chunk_cap = L.global_trees ? 0 : (maxc + 127) / 128 * 128;
  p.slot_tree = m->d_slot_tree;
  p.sparse = static_cast<const SparseTree*>(m->d_sparse_trees);
  p.sparse_nodes = static_cast<const uint4*>(m->d_sparse_nodes);
  p.hyb_nodes = static_cast<const uint2*>(m->d_hyb_nodes);
  p.hyb_leaves = m->d_hyb_leaves;
  p.slot_leafid_off = m->d_slot_leafid_off;
  p.leaf_ids = m->d_leaf_ids;
  p.T = m->T;
  FinalizeArgs fin{};
  fin.task = m->task;
  fin.agg = m->agg;
  fin.post = m->post;
  fin.K = m->K;
  fin.total_trees = total_trees;
  fin.q = m->ex.q;
  fin.acc_int = m->acc_int ? 1 : 0;
  fin.want = want;
  fin.leaf_scale = m->leaf_scale;
  fin.base = m->d_base;
  fin.out = out;
  p.fin = fin;
  if (L.stream) {
    // tree-streamed mode: X transposed once into feature-major 32-row blocks
    // (or binned into code blocks), then row tiles resident / chunk node
    // records streamed (traverse.cuh K4s)
    const int64_t nbk = (n_rows + 31) / 32;
    void* xt = nullptr;
    cudaError_t err = cudaSuccess;
    if (L.codes) {
      err = launch_binning(m, L, X, n_rows, sms, st, &xt);
      if (err != cudaSuccess) return err;
    } else {
      err = cudaMallocAsync(&xt, (size_t)nbk * 32 * m->F * 4, st);
      if (err != cudaSuccess) return err;
      int nwx = 16;
      while (nwx > 1 && nwx * 32 * (m->F | 1) * 4 > 200 * 1024) --nwx;
      const int xsmem = nwx * 32 * (m->F | 1) * 4;
      smem_opt_in(reinterpret_cast<const void*>(xpose_kernel), g_xpose_smem);
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xpose_kernel, nwx * 32, xsmem);
      const int xgrid = (int)std::max<int64_t>(1, std::min<int64_t>((nbk + nwx - 1) / nwx, (int64_t)sms * std::max(1, occ)));
      xpose_kernel<<<xgrid, nwx * 32, xsmem, st>>>(X, n_rows, m->F, static_cast<float*>(xt));
      count_launch();
      err = cudaGetLastError();
    }
    if (err == cudaSuccess) {
      p.X = static_cast<const float*>(xt);
      p.mode = want == 3 ? TRAV_APPLY : TRAV_FINAL;
      p.out_leaf = static_cast<int32_t*>(out);
      p.stream_ns = L.stream_ns;
      p.stream_stage = L.stream_stage;
      const int rb = L.stream_warps * 32;
      p.stream_x_bytes = L.codes ? (L.stream_warps + 1) * code_buf_bytes(m->F) : rb * m->F * 4;
      p.code_buf = L.codes ? code_buf_bytes(m->F) : 0;
      p.k2 = 2u;
      p.k16 = 65536u;
      const int W = L.stream_w;
      p.stream_lbuf_bytes = (rb * W * m->K * 4 + 15) / 16 * 16;
      // ring | landing slots | [split: slack for the walk's discarded last-level child loads] | barriers
      const int smem_s = p.stream_x_bytes + L.stream_ns * L.stream_stage + p.stream_lbuf_bytes + L.stream_slack +
                         (1 + 2 * L.stream_ns) * 8 + 16;
      p.stream_lbuf_bytes += L.stream_slack;  // barriers sit after the slack
      const int64_t n_tiles = (n_rows + rb - 1) / rb;
      const int grid_s = (int)std::max<int64_t>(1, std::min<int64_t>(n_tiles, sms));
      const int block_s = (L.stream_warps + 1) * 32;
      const bool w2 = W == 2;
      const bool ml = L.has_missing;
      const int sf = L.codes ? 2 : L.stream_split ? 1 : 0;
#define BRIDGER_STA(ML, W)                                                                             \
  (sf == 2 ? launch_stream_t<1, long long, ML, W, true, 2>(p, grid_s, block_s, smem_s, st)             \
   : sf == 1 ? launch_stream_t<1, long long, ML, W, true, 1>(p, grid_s, block_s, smem_s, st)           \
             : launch_stream_t<1, long long, ML, W, true, 0>(p, grid_s, block_s, smem_s, st))
#define BRIDGER_STW(ACC, ML, W)                                                                        \
  (sf == 2 ? launch_stream_t<KT, ACC, ML, W, false, 2>(p, grid_s, block_s, smem_s, st)                 \
   : sf == 1 ? launch_stream_t<KT, ACC, ML, W, false, 1>(p, grid_s, block_s, smem_s, st)               \
             : launch_stream_t<KT, ACC, ML, W, false, 0>(p, grid_s, block_s, smem_s, st))
      if (W == 3) {  // codes only
        if (want == 3) {
          err = ml ? launch_stream_t<1, long long, true, 3, true, 2>(p, grid_s, block_s, smem_s, st)
                   : launch_stream_t<1, long long, false, 3, true, 2>(p, grid_s, block_s, smem_s, st);
        } else {
#define BRIDGER_ST3(ACC)                                                                    \
  (ml ? launch_stream_t<KT, ACC, true, 3, false, 2>(p, grid_s, block_s, smem_s, st)        \
      : launch_stream_t<KT, ACC, false, 3, false, 2>(p, grid_s, block_s, smem_s, st))
          BRIDGER_DISPATCH_KT(m->K, { err = m->acc_int ? BRIDGER_ST3(long long) : BRIDGER_ST3(double); });
#undef BRIDGER_ST3
        }
      } else if (want == 3) {
        err = ml ? (w2 ? BRIDGER_STA(true, 2) : BRIDGER_STA(true, 1)) : (w2 ? BRIDGER_STA(false, 2) : BRIDGER_STA(false, 1));
      } else {
#define BRIDGER_ST(ACC) \
  (ml ? (w2 ? BRIDGER_STW(ACC, true, 2) : BRIDGER_STW(ACC, true, 1)) : (w2 ? BRIDGER_STW(ACC, false, 2) : BRIDGER_STW(ACC, false, 1)))
        BRIDGER_DISPATCH_KT(m->K, { err = m->acc_int ? BRIDGER_ST(long long) : BRIDGER_ST(double); });
#undef BRIDGER_ST
      }
#undef BRIDGER_STA
#undef BRIDGER_STW
    }
    cudaFreeAsync(xt, st);
    return err;
  }
  const int NW = L.n_warps, G = L.group, NB = NW / G;
  const int block = NW * 32;
  p.group = G;
  p.red_off = p.chunk_cap + trav_x_region(L.codes, m->F, NB) + trav_bar_bytes(NB);
  p.code_buf = L.codes ? code_buf_bytes(m->F) : 0;
  p.k2 = 2u;
  p.k16 = 65536u;
  p.slot_off = p.red_off + trav_red_bytes(NB, G, m->K);
  int smem = p.slot_off;
  int cluster = 1;
  void* partial = nullptr;
  // K4d (trav_deep.cu): coded chunks, several of them, exact int64 tiers ->
  // per-warp red.global.add into one accumulator instead of per-chunk partials
  // + combine (BRIDGER_DEEP=0 keeps K4's partials, for comparison)
  const char* deep_env = std::getenv("BRIDGER_DEEP");
  const bool deep = L.codes && !L.global_trees && want != 3 && m->acc_int && n_chunks >= deep_min_chunks() &&
                    !(deep_env && deep_env[0] == '0');
  if (want == 3) {
    p.mode = TRAV_APPLY;
    p.out_leaf = static_cast<int32_t*>(out);
  } else if (n_chunks == 1 || L.global_trees) {
    p.mode = TRAV_FINAL;
  } else if (L.use_cluster && n_chunks <= 8 && smem + trav_slot_bytes(NB, n_chunks, m->K) <= 232448) {
    p.mode = TRAV_CLUSTER;
    cluster = n_chunks;
    smem += trav_slot_bytes(NB, n_chunks, m->K);
  } else if (!deep) {
    p.mode = TRAV_PARTIAL;
    cudaError_t e = cudaMallocAsync(&partial, (size_t)n_chunks * n_rows * m->K * 8, st);
    if (e != cudaSuccess) return e;
    p.partial = partial;
  }
  // global-tree mode: every CTA walks every chunk -> the grid is one chunk-group
  if (L.global_trees) p.n_chunks_grid = 1;
  else p.n_chunks_grid = n_chunks;
  // persistent grid ~ one CTA per SM, but never more CTAs per chunk than there
  // are row-block groups to hand out (small batches: C1 is one CTA)
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t groups_needed = (n_blocks + NB - 1) / NB;
  const int cpc = (int)std::max<int64_t>(1, std::min<int64_t>(sms / p.n_chunks_grid, groups_needed));
  const int grid = p.n_chunks_grid * cpc;
  cudaError_t err = cudaSuccess;
  void* codes = nullptr;
  // K4d accumulator: zeroed BEFORE the binning kernel, so the walk -- launched
  // as a programmatic dependent of the binning grid -- only waits on that grid
  void* deep_acc = nullptr;
  if (deep && !scatter) {
    deep_acc = want == 2 ? out : nullptr;
    if (!deep_acc) err = cudaMallocAsync(&deep_acc, (size_t)n_rows * m->K * 8, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(deep_acc, 0, (size_t)n_rows * m->K * 8, st);
    if (err != cudaSuccess) return err;
  }
  if (L.codes) {
    err = launch_binning(m, L, X, n_rows, sms, st, &codes);
    if (err != cudaSuccess) return err;
    p.X = static_cast<const float*>(codes);
  } else if (L.hybrid || (L.pretransposed && want != 3)) {
    const int64_t nbk = (n_rows + 31) / 32;
    err = cudaMallocAsync(&codes, (size_t)nbk * 32 * m->F * 4, st);
    if (err != cudaSuccess) return err;
    int nwx = 16;
    while (nwx > 1 && nwx * 32 * (m->F | 1) * 4 > 200 * 1024) --nwx;
    const int xsmem = nwx * 32 * (m->F | 1) * 4;
    smem_opt_in(reinterpret_cast<const void*>(xpose_kernel), g_xpose_smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xpose_kernel, nwx * 32, xsmem);
    const int64_t want_ctas = (nbk + nwx - 1) / nwx;
    const int xgrid = (int)std::max<int64_t>(1, std::min<int64_t>(want_ctas, (int64_t)sms * std::max(1, occ)));
    xpose_kernel<<<xgrid, nwx * 32, xsmem, st>>>(X, n_rows, m->F, static_cast<float*>(codes));
    count_launch();
    err = cudaGetLastError();
    if (err != cudaSuccess) {
      cudaFreeAsync(codes, st);
      return err;
    }
    p.X = static_cast<const float*>(codes);
  }
  if (scatter && !deep) {
    if (codes) cudaFreeAsync(codes, st);
    return cudaErrorNotSupported;
  }
  if (deep) {
    void* acc = deep_acc;
    if (scatter) {
      p.scatter = scatter;  // the caller zeroed the ranks' slices
      p.scatter_blocks = (int32_t)(rows_per_rank / 32);
    }
    if (err == cudaSuccess) {
      p.mode = TRAV_PARTIAL;
      p.partial = acc;
      // child-pair speculation from this depth on (latency-bound deep chunks)
      p.spec_min_d = 9;
      if (const char* e = std::getenv("BRIDGER_SPEC_D")) p.spec_min_d = std::atoi(e);
      const int dsmem = trav_deep_smem(p.chunk_cap, p.code_buf, NB);
      // wm = 1 when every chunk takes the speculative walk (as
      // trav_deep_kernel decides it): the kernel built with only that walk
      int wm = 1;
      const int KT = m->K <= 1 ? 1 : m->K <= 2 ? 2 : m->K <= 4 ? 4 : m->K <= 8 ? 8 : m->K <= 16 ? 16 : 64;
      for (const TravChunk& ch : L.chunks)
        if (!(ch.depth >= p.spec_min_d && m->K == KT && ch.depth >= 1)) wm = 0;
      if (const char* e = std::getenv("BRIDGER_DEEP_WM"))
        if (e[0] == '0') wm = 0;  // A/B: the kernel with every walk (runtime choice)
      err = launch_trav_deep(p, m->K, L.has_missing, std::max(wm, 0), grid, block, dsmem, st);
    }
    if (err == cudaSuccess && want != 2) {
      const int tb = 256;
      const int g = (int)((n_rows + tb - 1) / tb);
      BRIDGER_DISPATCH_KT(m->K, {
        trav_combine_kernel<KT, long long><<<g, tb, 0, st>>>(static_cast<const long long*>(acc), 1, n_rows, fin);
      });
      count_launch();
      err = cudaGetLastError();
    }
    if (acc && want != 2) cudaFreeAsync(acc, st);
    if (codes) cudaFreeAsync(codes, st);
    return err;
  }
  BRIDGER_DISPATCH_KT(m->K, {
    auto launch = [&]() {
      if (L.sparse) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, true, 2>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, true, 2>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, true, 2>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, true, 2>(p, grid, block, smem, cluster, st);
      }
      if (L.split) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, false, 5>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, false, 5>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, false, 5>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, false, 5>(p, grid, block, smem, cluster, st);
      }
      if (L.hybrid) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, false, 4>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, false, 4>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, false, 4>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, false, 4>(p, grid, block, smem, cluster, st);
      }
      if (L.pretransposed && want != 3) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, false, 3>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, false, 3>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, false, 3>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, false, 3>(p, grid, block, smem, cluster, st);
      }
      if (L.codes) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, false, 1>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, false, 1>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, false, 1>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, false, 1>(p, grid, block, smem, cluster, st);
      }
      if (L.global_trees) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, true, 0>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, true, 0>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, true, 0>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, true, 0>(p, grid, block, smem, cluster, st);
      }
      if (m->acc_int)
        return L.has_missing ? launch_trav_t<KT, long long, true, false, 0>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, long long, false, false, 0>(p, grid, block, smem, cluster, st);
      return L.has_missing ? launch_trav_t<KT, double, true, false, 0>(p, grid, block, smem, cluster, st)
                           : launch_trav_t<KT, double, false, false, 0>(p, grid, block, smem, cluster, st);
    };
    err = launch();
    if (err != cudaSuccess && p.mode == TRAV_CLUSTER) {
      // clusters of this size cannot be co-resident at this shared-memory
      // footprint: fall back to per-chunk partials + combine
      cudaGetLastError();
      p.mode = TRAV_PARTIAL;
      cluster = 1;
      smem = p.slot_off;
      err = cudaMallocAsync(&partial, (size_t)n_chunks * n_rows * m->K * 8, st);
      p.partial = partial;
      if (err == cudaSuccess) err = launch();
    }
    if (err == cudaSuccess && p.mode == TRAV_PARTIAL) {
      const int tb = 256;
      const int g = (int)((n_rows + tb - 1) / tb);
      if (m->acc_int)
        trav_combine_kernel<KT, long long><<<g, tb, 0, st>>>(static_cast<const long long*>(partial), n_chunks, n_rows, fin);
      else
        trav_combine_kernel<KT, double><<<g, tb, 0, st>>>(static_cast<const double*>(partial), n_chunks, n_rows, fin);
      count_launch();
      err = cudaGetLastError();
    }
  });
  if (partial) cudaFreeAsync(partial, st);
  if (codes) cudaFreeAsync(codes, st);
  return err;
}

// finalize of caller-provided accumulators (bridger_finalize)
cudaError_t finalize_run(const bridger_model* m, const void* acc, int64_t n_rows, int32_t total_trees,
                         void* out, int want, cudaStream_t st) {
  FinalizeArgs fin{};
  fin.task = m->task;
  fin.agg = m->agg;
  fin.post = m->post;
  fin.K = m->K;
  fin.total_trees = total_trees;
  fin.q = m->ex.q;
  fin.acc_int = m->acc_int ? 1 : 0;
  fin.want = want;
  fin.leaf_scale = m->leaf_scale;
  fin.base = m->d_base;
  fin.out = out;
  const int tb = 256;
  const int g = (int)((n_rows + tb - 1) / tb);
  cudaError_t err = cudaSuccess;
  BRIDGER_DISPATCH_KT(m->K, {
    if (m->acc_int)
      trav_combine_kernel<KT, long long><<<g, tb, 0, st>>>(static_cast<const long long*>(acc), 1, n_rows, fin);
    else
      trav_combine_kernel<KT, double><<<g, tb, 0, st>>>(static_cast<const double*>(acc), 1, n_rows, fin);
    count_launch();
    err = cudaGetLastError();
  });
  return err;
}

}  // namespace bridger
