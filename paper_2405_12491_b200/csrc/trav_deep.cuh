// K4d: traversal of threshold-bin-coded ensembles split over several resident
// chunks (C5-shaped deep forests: 74 chunks of ~17 depth-10 trees per 1250-tree
// shard; also C2/C3's 2-3 chunks), steps a4' + a5 + a6 of SURVEY.md §8(a).
//
// Same per-visit walk as K4 (walk_trees, CODES branch: one LDS of the 4-byte
// node word, one conflict-free LDS of the lane's u16 input code, 7
// instructions), but the per-row-block bookkeeping is rebuilt for many chunks:
//  * the G warps that share a 32-row code block do NOT meet at a barrier and do
//    not combine partial sums in shared memory: each warp adds its own per-row
//    int64 fixed-point partial straight into the caller's accumulator with
//    red.global.add.u64 (exact and order-free, reading c9 -- no per-chunk
//    partial arrays, no combine pass; round 1's K4 wrote 74 x 8 B per row);
//  * a code buffer is refilled by the LAST warp of its group to finish with it
//    (shared-memory counter, as in bin_coop_kernel), so a warp that ran ahead
//    never waits for a slower one except when both buffers are still in use;
//  * the chunk's trees are dealt to the G warps in shares that ROTATE with the
//    block index (share r = (gw + i) mod G), so a chunk whose tree count is not
//    a multiple of G costs every warp the same work on average (round 1's
//    fixed split left 1/3 of the warps idle at the group barrier for C5);
//  * everything that does not depend on the block (share sizes, pass plan) is
//    computed once per kernel (round 1's K4 recomputed two integer divisions
//    per warp per block: ~50% of the C5 kernel's issue slots, ncu
//    profiles/r2_c5_trav_*.txt).
// The accumulator is zeroed by the launcher; finalize (a7) is one pass of
// trav_combine_kernel over it, or nothing for predict_raw (the accumulator IS
// the output).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "traverse.cuh"

namespace bridger {

// fire-and-forget 64-bit add in L2 (RED, no return value)
__device__ __forceinline__ void red_add_u64(unsigned long long* a, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

// Child-pair speculation for deep coded trees (D >= p.spec_min_d): per level
// the lane's input code of the current node AND the node words of BOTH its
// children (one LDS.64: children 2i+1, 2i+2 are an 8-byte-aligned pair behind
// the tree's pad word, lowering.cpp) are loaded together; the compare then
// selects the child word already in registers.  The dependent chain per level
// shrinks from node LDS -> code LDS -> compare to code LDS -> compare -> select
// (one shared-memory latency instead of two).  At the last level the "children"
// are the two leaf values (adjacent: leaves 2i+1-I, 2i+2-I), loaded as one
// vector and selected the same way, so the leaf gather costs no extra latency.
// Tree u = j + v of the chunk: pad word at T = nodes + 4 (j+v)(I+1), node idx at
// T + 4 (idx + 1); with A the current node's address, the children pair is at
// 2A - T = 2A + cb (cb = -T) and the leaf pair of a last-level node at
// leaves_u + 2K (A - T - 4) + 4K (1 - I).
template <int NI, int KT, bool ML>
__device__ __forceinline__ void walk_codes_spec(const TravParams& p, uint32_t nodes_s, uint32_t leaves_s,
                                                uint32_t xb, int j, int I, int L, int D, long long (&acc)[KT]) {
  const uint32_t mask = (uint32_t)p.code_buf - 2u;
  const uint32_t k2 = p.k2, k16 = p.k16;
  uint32_t A[NI], cb[NI], a[NI];
#pragma unroll
  for (int v = 0; v < NI; ++v) {
    const uint32_t T = nodes_s + 4u * (uint32_t)((j + v) * (I + 1));
    A[v] = T + 4u;
    cb[v] = 0u - T;
    a[v] = ptx::lds_u32(A[v]);
  }
  for (int lvl = 0; lvl + 1 < D; ++lvl) {
    uint32_t x[NI], c0[NI], c1[NI];
#pragma unroll
    for (int v = 0; v < NI; ++v) x[v] = ptx::lds_u16(xb | (a[v] & mask));
#pragma unroll
    for (int v = 0; v < NI; ++v) {
      A[v] = A[v] * k2 + cb[v];  // left child's address; the pair {left, right}
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(c0[v]), "=r"(c1[v]) : "r"(A[v]));
    }
#pragma unroll
    for (int v = 0; v < NI; ++v) {
      bool r = x[v] * k16 > a[v];  // code(x) > j  <=>  !(x <= t); NaN code 0xFFFF -> right
      if (ML) r = r && !((a[v] & 1u) && x[v] == 0xFFFFu);
      a[v] = r ? c1[v] : c0[v];
      if (r) A[v] += 4u;
    }
  }
  // last internal level: its children are leaves
  uint32_t x[NI];
#pragma unroll
  for (int v = 0; v < NI; ++v) x[v] = ptx::lds_u16(xb | (a[v] & mask));
#pragma unroll
  for (int v = 0; v < NI; ++v) {
    const uint32_t lu = leaves_s + 4u * (uint32_t)((j + v) * L * KT);
    const uint32_t la = lu + 2u * KT * (A[v] + cb[v] - 4u) + 4u * KT - 4u * KT * (uint32_t)I;
    bool r = x[v] * k16 > a[v];
    if (ML) r = r && !((a[v] & 1u) && x[v] == 0xFFFFu);
    if (KT == 1) {
      // one leaf value after the compare: a random LDS.32 costs about half the
      // wavefronts of the leaf pair (the walk is LSU-bound here)
      acc[0] += leaf_to_acc<long long>(ptx::lds_f32(la + (r ? 4u : 0u)));
    } else if (KT == 2) {
      float v0, v1, v2, v3;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(la));
      acc[0] += leaf_to_acc<long long>(r ? v2 : v0);
      acc[KT > 1 ? 1 : 0] += leaf_to_acc<long long>(r ? v3 : v1);
    } else {
      const uint32_t lr = la + (r ? 4u * KT : 0u);
#pragma unroll
      for (int k = 0; k < KT; ++k) acc[k] += leaf_to_acc<long long>(ptx::lds_f32(lr + 4u * k));
    }
  }
}

template <int KT, bool ML, int MAXNI>
__device__ __forceinline__ void walk_spec_tail(int n, const TravParams& p, uint32_t nodes_s, uint32_t leaves_s,
                                               uint32_t xb, int j, int I, int L, int D, long long (&acc)[KT]) {
  switch (n) {
#define BRIDGER_SPEC_TAIL(N) \
  case N: if (N <= MAXNI) walk_codes_spec<(N <= MAXNI ? N : 1), KT, ML>(p, nodes_s, leaves_s, xb, j, I, L, D, acc); break;
    BRIDGER_SPEC_TAIL(1) BRIDGER_SPEC_TAIL(2) BRIDGER_SPEC_TAIL(3) BRIDGER_SPEC_TAIL(4) BRIDGER_SPEC_TAIL(5)
    BRIDGER_SPEC_TAIL(6) BRIDGER_SPEC_TAIL(7) BRIDGER_SPEC_TAIL(8) BRIDGER_SPEC_TAIL(9) BRIDGER_SPEC_TAIL(10)
#undef BRIDGER_SPEC_TAIL
    default: break;
  }
}

// SC: the fused tree-sharding reduce (partials scattered to the owner rank's
// slice); a separate instantiation -- the branch in the common kernel cost the
// C5 shard walk 4% (7.89 -> 8.23 ms, register allocation of the pass loop)
// WM = 1: every chunk takes the speculative walk, and the kernel holds only
// that walk (C5 shard walk 7.86 -> 7.73 ms); 0 chooses per chunk at run time.
// (A WM for the compile-time-depth walks measured slower on C3: 8.55 -> 8.73.)
template <int KT, bool ML, bool SC, int WM>
__global__ void __launch_bounds__(512, 1) trav_deep_kernel(const TravParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int G = p.group, NB = NW / G;
  const int grp = warp / G, gw = warp % G;
  const int chunk_id = blockIdx.x % p.n_chunks_grid;
  const int cta_in_chunk = blockIdx.x / p.n_chunks_grid;
  const TravChunk c = p.chunks[chunk_id];
  const int K = p.K;
  const uint32_t cbuf = (uint32_t)p.code_buf;
  const uint32_t a0 = ptx::s2u(smem + p.chunk_cap);
  uint8_t* Cb = smem + p.chunk_cap + (((a0 + cbuf - 1u) & ~(cbuf - 1u)) - a0);  // [NB][2] 2^b-aligned buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(Cb + (size_t)NB * 2 * cbuf);     // [0] chunk, [1 + 2 grp + s] full
  uint32_t* done = reinterpret_cast<uint32_t*>(bars + 1 + 2 * NB);              // [NB][2] warps done with a buffer
  if (threadIdx.x == 0) {
    for (int b = 0; b < 1 + 2 * NB; ++b) ptx::mbar_init(&bars[b], 1);
    for (int b = 0; b < 2 * NB; ++b) done[b] = 0;
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bars[0], (uint32_t)c.bytes);
    const uint8_t* src = p.data + c.offset;
    for (int32_t o = 0; o < c.bytes; o += 65536)
      ptx::bulk_g2s(smem + o, src + o, (uint32_t)min(65536, c.bytes - o), &bars[0]);
  }
  const int64_t n_rows = p.n_rows;
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t stride = (int64_t)p.cpc * NB;
  const int64_t blk0 = (int64_t)cta_in_chunk * NB + grp;
  const int64_t n_mine = blk0 < n_blocks ? (n_blocks - 1 - blk0) / stride + 1 : 0;
  const int F2 = (p.F + 1) & ~1;
  const uint32_t cbytes = 64u * (uint32_t)F2;  // one [F2/2][32][2] u16 code block
  const uint8_t* codes = reinterpret_cast<const uint8_t*>(p.X);
  uint64_t* full = bars + 1 + 2 * grp;
  uint8_t* gbuf = Cb + (size_t)grp * 2 * cbuf;
  auto issue = [&](int64_t i, int s) {
    ptx::fence_proxy_async();
    ptx::mbar_arrive_expect_tx(&full[s], cbytes);
    ptx::bulk_g2s(gbuf + (size_t)s * cbuf, codes + (blk0 + i * stride) * (int64_t)cbytes, cbytes, &full[s]);
  };
  // programmatic dependent launch: everything above (barrier init, the chunk's
  // bulk copy) overlapped the binning grid's tail; the codes it writes are
  // read from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (gw == 0 && lane == 0) {
    if (n_mine > 0) issue(0, 0);
    if (n_mine > 1) issue(1, 1);
  }
  ptx::mbar_wait(&bars[0], 0);  // chunk resident

  // per-kernel share plan: share r of the chunk's n trees = [r*base + min(r, rem), + base + (r < rem))
  constexpr int NI_MAX = (!ML && KT <= 8) ? 12 : 4;
  const int D = c.depth, I = (1 << D) - 1, L = 1 << D;
  const int n = c.n_trees;
  const int base = n / G, rem = n % G;
  const float* leaves = reinterpret_cast<const float*>(smem + c.leaf_offset);
  // speculative walk (K == KT layouts only: vector leaf pairs) for deep chunks
  constexpr int SPEC_NI = (!ML && KT <= 2) ? 10 : 4;
  const bool spec = D >= p.spec_min_d && K == KT && D >= 1;
  const int ni_max = spec ? SPEC_NI : NI_MAX;
  const uint32_t nodes_s = ptx::s2u(smem), leaves_s = ptx::s2u(leaves);
  // pass plans of the two share sizes (base, base + 1): n_pass passes of
  // (nearly) equal width <= ni_max, the first `big` of them one tree wider
  int np_[2], sz_[2], big_[2];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int cnt = base + b;
    np_[b] = (cnt + ni_max - 1) / ni_max;
    sz_[b] = np_[b] ? cnt / np_[b] : 0;
    big_[b] = np_[b] ? cnt - sz_[b] * np_[b] : 0;
  }
  int r = gw;  // rotating share index (gw + i) mod G
  for (int64_t i = 0; i < n_mine; ++i) {
    const int s = (int)(i & 1);
    ptx::mbar_wait_sleep(&full[s], (uint32_t)(i >> 1) & 1u, 32);
    const void* xl = gbuf + (size_t)s * cbuf + 4 * lane;
    const int b1 = r < rem ? 1 : 0;
    int j = r * base + min(r, rem);
    const int64_t row = (blk0 + i * stride) * 32 + lane;
    long long acc[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) acc[k] = 0;
    const int n_pass = b1 ? np_[1] : np_[0], sz0 = b1 ? sz_[1] : sz_[0], nbig = b1 ? big_[1] : big_[0];
    for (int q = 0; q < n_pass; ++q) {
      const int sz = sz0 + (q < nbig ? 1 : 0);
      if (WM == 1 || (WM == 0 && spec))
        walk_spec_tail<KT, ML, SPEC_NI>(sz, p, nodes_s, leaves_s, ptx::s2u(xl), j, I, L, D, acc);
      else if (!ML && KT <= 8 && D == 6)
        walk_tail<KT, long long, ML, true, NI_MAX, false, 6>(sz, p, c, smem, leaves, xl, j, I, L, D, K, row, acc);
      else if (!ML && KT <= 8 && D == 8)
        walk_tail<KT, long long, ML, true, NI_MAX, false, 8>(sz, p, c, smem, leaves, xl, j, I, L, D, K, row, acc);
      else
        walk_tail<KT, long long, ML, true, NI_MAX>(sz, p, c, smem, leaves, xl, j, I, L, D, K, row, acc);
      j += sz;
    }
    const int cnt = base + b1;
    if (cnt > 0 && row < n_rows) {
      unsigned long long* dst;
      if (SC) {
        // the reduce of tree sharding fused into the walk: this row's partial
        // goes straight into the owner rank's slice (own or peer memory)
        const int32_t gb = (int32_t)(blk0 + i * stride);           // global 32-row block (warp-uniform)
        const int32_t rk = gb / p.scatter_blocks;
        dst = static_cast<unsigned long long*>(p.scatter[rk]) +
              ((int64_t)(gb - rk * p.scatter_blocks) * 32 + lane) * K;
      } else {
        dst = static_cast<unsigned long long*>(p.partial) + row * K;
      }
#pragma unroll
      for (int k = 0; k < KT; ++k)
        if (k < K) red_add_u64(dst + k, static_cast<unsigned long long>(acc[k]));
    }
    // release the buffer: the group's last warp to finish refills it
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[grp * 2 + s], 1u) == (uint32_t)G - 1u) {
        done[grp * 2 + s] = 0;
        if (i + 2 < n_mine) issue(i + 2, s);
      }
    }
    if (++r == G) r = 0;
  }
}

// Launch one instantiation (SC: fused scatter, WM: walk mode).  The kernels
// are compiled in parallel translation units (trav_deep_inst_*.cu); the
// dispatcher (trav_deep.cu) only declares them.
template <int KT, bool ML, bool SC, int WM>
cudaError_t launch_deep_k(const TravParams& p, int grid, int block, int smem, cudaStream_t st) {
  auto kern = trav_deep_kernel<KT, ML, SC, WM>;
  static std::atomic<uint64_t> configured{0};  // per instantiation, per device
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(kern), configured);
  if (e != cudaSuccess) return e;
  TravParams q = p;
  q.cpc = grid / p.n_chunks_grid;
  if (std::getenv("BRIDGER_DEBUG"))
    std::fprintf(stderr, "[bridger] trav_deep_kernel<%d,%d,%d,%d> grid=%d block=%d smem=%d chunks=%d cpc=%d G=%d\n",
                 KT, (int)ML, (int)SC, WM, grid, block, smem, q.n_chunks, q.cpc, q.group);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // programmatic dependent launch: see the griddepcontrol.wait in the kernel
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  const char* pdl = std::getenv("BRIDGER_PDL");
  cfg.numAttrs = (pdl && pdl[0] == '0') ? 0 : 1;
  cudaEvent_t ev;
  hot_begin(st, &ev);
  e = cudaLaunchKernelEx(&cfg, kern, q);
  hot_end(st, ev);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

#define BRIDGER_DEEP_DECL(PREFIX, KT, ML, SC, WM) \
  PREFIX template cudaError_t launch_deep_k<KT, ML, SC, WM>(const TravParams&, int, int, int, cudaStream_t);
// every KT of BRIDGER_DISPATCH_KT
#define BRIDGER_DEEP_ALL_KT(PREFIX, ML, SC, WM)                                                        \
  BRIDGER_DEEP_DECL(PREFIX, 1, ML, SC, WM) BRIDGER_DEEP_DECL(PREFIX, 2, ML, SC, WM)                    \
  BRIDGER_DEEP_DECL(PREFIX, 4, ML, SC, WM) BRIDGER_DEEP_DECL(PREFIX, 8, ML, SC, WM)                    \
  BRIDGER_DEEP_DECL(PREFIX, 16, ML, SC, WM) BRIDGER_DEEP_DECL(PREFIX, 64, ML, SC, WM)
// the speculative-walk-only kernels (WM = 1): !ML, no scatter, KT <= 8
#define BRIDGER_DEEP_WM1(PREFIX)                                                                       \
  BRIDGER_DEEP_DECL(PREFIX, 1, false, false, 1) BRIDGER_DEEP_DECL(PREFIX, 2, false, false, 1)          \
  BRIDGER_DEEP_DECL(PREFIX, 4, false, false, 1) BRIDGER_DEEP_DECL(PREFIX, 8, false, false, 1)
#define BRIDGER_DEEP_EXTERN_ALL()                                                                      \
  BRIDGER_DEEP_ALL_KT(extern, false, false, 0) BRIDGER_DEEP_ALL_KT(extern, true, false, 0)             \
  BRIDGER_DEEP_ALL_KT(extern, false, true, 0) BRIDGER_DEEP_ALL_KT(extern, true, true, 0)               \
  BRIDGER_DEEP_WM1(extern)

}  // namespace bridger
