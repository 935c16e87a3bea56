#pragma once
// Traversal kernel templates (K4); instantiated in trav_inst_*.cu.
// K4 traversal kernel (step a4' + a5 + a6 [+ a7 fused]).
//
// The COR form of a tree executed as the SPEC.md:283 template:
//   idx <- 0; repeat D: idx <- 2 idx + 1 + [not (X[r, feat[idx]] <= thr[idx])]
//   leaf = idx - I;  acc += E[leaf]
// on perfect, heap-ordered trees (lowering.cpp).  B200 mapping:
//  * A chunk of trees (nodes {thr, feature} 8 B + leaf values) is copied ONCE
//    into a CTA's shared memory by the TMA engine (cp.async.bulk) and stays
//    resident; the grid is persistent, n_chunks x ctas_per_chunk ~= #SMs.
//  * lane = row.  Each warp streams its own 32-row blocks of X: a bulk copy
//    lands the dense [32][F] block in a staging buffer (double buffering: the
//    next block is in flight while the current one is walked), then the warp
//    transposes it to a feature-major [F][32] block, so x = Xs[f*32 + lane]
//    hits bank `lane` for ANY per-lane feature: the data-dependent feature
//    gather is bank-conflict free.  Node loads are broadcast at the top levels
//    and random-but-narrow below.
//  * Each thread walks 4 trees at once (ILP) and accumulates leaf values in
//    int64 fixed point (exact, order-free; reading c9) or fp64.
//  * One chunk: finalize fused (a7).  Several chunks: per-chunk partials
//    [chunk][row][K], combined in chunk order by trav_combine_kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "bridger_internal.h"
#include "finalize.cuh"
#include "ptx.cuh"

namespace bridger {

void count_launch();
void hot_begin(cudaStream_t st, cudaEvent_t* ev);
void hot_end(cudaStream_t st, cudaEvent_t start);

// FINAL: one chunk, finalize fused.  PARTIAL: per-chunk partials to global.
// APPLY: leaf ids.  CLUSTER: the n_chunks CTAs of a thread-block cluster hold
// the n chunks of the model and walk the SAME row blocks; peers push their
// per-row partial sums into the leader CTA's shared memory over DSMEM
// (st.shared::cluster + remote mbarrier arrive), the leader adds them in rank
// order and finalizes -- no global partials, no second kernel.
enum TravFmt : int { FMT_HEAP = 0, FMT_CODES = 1, FMT_SPARSE = 2, FMT_HEAP_T = 3, FMT_HYBRID = 4, FMT_SPLIT = 5 };
enum TravMode : int32_t { TRAV_FINAL = 0, TRAV_PARTIAL = 1, TRAV_APPLY = 2, TRAV_CLUSTER = 3 };

struct TravParams {
  const float* X;
  int64_t n_rows;
  int32_t F;
  int32_t K;
  const uint8_t* data;
  const TravChunk* chunks;
  int32_t n_chunks;
  int32_t n_chunks_grid;  // chunks the grid is split over (1 in global-tree mode)
  int32_t cpc;        // CTAs per chunk
  int32_t chunk_cap;  // bytes reserved for the chunk in shared memory
  int32_t mode;
  void* partial;      // [n_chunks][n_rows][K] ACC   (TRAV_PARTIAL)
  int32_t* out_leaf;  // [n_rows][T]                 (TRAV_APPLY)
  const int32_t* slot_tree;
  const int64_t* slot_leafid_off;
  const int32_t* leaf_ids;
  int32_t T;
  const SparseTree* sparse;  // FMT_SPARSE: per-slot tree descriptors
  const uint4* sparse_nodes; //             16-byte node records
  const uint2* hyb_nodes;    // FMT_HYBRID: deep levels of every tree (global)
  const float* hyb_leaves;   //             leaf values (global)
  int32_t hyb_pret;          //             input pre-transposed (bulk-copied blocks)
  int32_t group;      // warps sharing one 32-row block (tree split)
  int32_t red_off;    // byte offset of the intra-group partials
  int32_t slot_off;   // byte offset of the DSMEM reduction slots (TRAV_CLUSTER)
  int32_t stream_ns;      // tree-streamed mode: node-record ring depth
  int32_t stream_stage;   //                     bytes per ring slot
  int32_t stream_x_bytes; //                     X tile bytes (rows_per_tile * F * 4)
  int32_t stream_lbuf_bytes; //                  leaf-value landing slots (rows_per_tile * W * K * 4)
  int32_t code_buf;   // codes: bytes (2^b) of one aligned code-block buffer
  uint32_t k2, k16;   // 2 and 65536, opaque to the compiler: keeps the walk's
                      // multiplies on the FMA pipe (IMAD) instead of the ALU pipe
  int32_t spec_min_d; // trav_deep: chunks of depth >= this walk with child-pair speculation
  void* const* scatter;      // trav_deep, bridger_predict_raw_scatter: per-rank accumulator slices
  int32_t scatter_blocks;    //   32-row blocks per rank slice (rows_per_rank / 32)
  FinalizeArgs fin;   // (TRAV_FINAL, TRAV_CLUSTER)
};

template <typename ACC>
__device__ __forceinline__ ACC leaf_to_acc(float v);
template <>
__device__ __forceinline__ long long leaf_to_acc<long long>(float v) {
  return __float2ll_rz(v);  // v is an integer-valued float (pre-scaled by 2^-q): exact
}
template <>
__device__ __forceinline__ double leaf_to_acc<double>(float v) {
  return (double)v;
}

template <bool ML>
__device__ __forceinline__ int go_right(float x, uint2 nd) {
  const float t = __uint_as_float(nd.x);
  int r = !(x <= t);  // NaN -> right (reading c2 default)
  if (ML) r &= !((nd.y >> 31) & isnan(x));
  return r;
}

// Walk NI trees [j, j+NI) of the chunk for this thread's row (NI independent
// dependency chains for ILP), then gather and accumulate their leaf values.
// DT > 0: the depth is a compile-time constant (coded walks of the common
// depths: the level loop unrolls fully -- no loop counter / branch / register
// shuffling per level); DT == 0: runtime depth D.
template <int NI, int KT, typename ACC, bool ML, bool CODES, bool SPLIT = false, int DT = 0>
__device__ __forceinline__ void walk_trees(const TravParams& p, const TravChunk& c, const void* nodes,
                                           const float* leaves, const void* xl, int j, int I, int L, int D,
                                           int K, int64_t row, ACC (&acc)[KT]) {
  int idx[NI];
#pragma unroll
  for (int u = 0; u < NI; ++u) idx[u] = 0;
  if (SPLIT) {
    // split node arrays: fp32 thresholds [n][I], then 1-byte features [n][I]
    // (bit 7 = missing_left).  Byte loads of nearby nodes share 4-byte words,
    // so the feature loads stay bank-conflict free through level 7.
    const float* tb = static_cast<const float*>(nodes) + (size_t)j * I;
    const uint8_t* fb = static_cast<const uint8_t*>(nodes) + (((size_t)c.n_trees * I * 4 + 15) & ~(size_t)15) + (size_t)j * I;
    const float* xf = static_cast<const float*>(xl);
    for (int lvl = 0; lvl < D; ++lvl) {
      uint32_t f[NI];
      float t[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        f[u] = fb[u * I + idx[u]];
        t[u] = tb[u * I + idx[u]];
      }
      float x[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) x[u] = xf[(f[u] & 0x7Fu) * 32];
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        int r = !(x[u] <= t[u]);
        if (ML) r &= !((f[u] >> 7) & isnan(x[u]));
        idx[u] = 2 * idx[u] + 1 + r;
      }
    }
  } else if (CODES) {
    // 4-byte node: code index j (31..16) | feature byte offset (14..1, even)
    // within a lane's view of a [F/2][32][2] u16 code block | missing (0).
    // xl is this lane's 4-byte column of a 2^b-aligned block buffer, so the
    // code address is (xl | (a & (2^b - 2))): bank `lane` for any feature, one LOP3.
    // code(x) > j  <=>  x * 2^16 > a  (the low half of a is < 2^16), so the
    // compare needs no field extraction.  Node addresses are shared-window byte
    // addresses: node idx of tree u at A = base_u + 4 idx, and
    // idx' = 2 idx + 1 + r  <=>  A' = 2 A + (r ? 8 : 4) - base_u.
    // The two multiplies use opaque constants (p.k2, p.k16) so they issue on
    // the FMA pipe; the LOP3 / compare / select use the ALU pipe.
    // tree u of the chunk at words [(j+u)(I+1), ...): a pad word, then nodes
    // 0..I-1 (lowering.cpp), so node 0 of tree u sits at nb + 4 (u (I+1))
    const uint32_t nb = ptx::s2u(nodes) + 4u * (uint32_t)(j * (I + 1)) + 4u;
    const uint32_t xb = ptx::s2u(xl);
    const uint32_t mask = (uint32_t)p.code_buf - 2u;  // feature offset bits, not the missing bit
    const uint32_t k2 = p.k2, k16 = p.k16;
    uint32_t A[NI], cb[NI];  // cb = 4 - base_u:  A' = A * 2 + cb (+ 4 if right)
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      A[u] = nb + 4u * (uint32_t)(u * (I + 1));  // shared address of tree u's current node
      cb[u] = 4u - A[u];
    }
    const int DD = DT > 0 ? DT : D;
#pragma unroll (DT > 0 ? DT : 1)
    for (int lvl = 0; lvl < DD; ++lvl) {
      uint32_t a[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) a[u] = ptx::lds_u32(A[u]);
      uint32_t x[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) x[u] = ptx::lds_u16(xb | (a[u] & mask));
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        bool r = x[u] * k16 > a[u];  // code(x) > j  <=>  !(x <= t);  NaN code 0xFFFF -> right
        if (ML) r = r && !((a[u] & 1u) && x[u] == 0xFFFFu);
        A[u] = A[u] * k2 + cb[u];
        if (r) A[u] += 4u;
      }
    }
    if (p.mode != TRAV_APPLY && KT == K) {
      // leaf values straight from the final node address: leaf l = idx - I,
      // idx = (A - base_u) / 4, value address = leaves_u + 4 K l
      //   = K * A + (leaves_u - K (base_u + 4 I)),  base_u = 4 - cb_u
      const uint32_t lb = ptx::s2u(leaves) + 4u * (uint32_t)(j * L * KT);
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        const uint32_t la = (uint32_t)KT * (A[u] + cb[u] - 4u - 4u * (uint32_t)I) + lb + 4u * (uint32_t)(u * L * KT);
        if (KT == 2) {
          float v0, v1;
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(la));
          acc[0] += leaf_to_acc<ACC>(v0);
          acc[KT > 1 ? 1 : 0] += leaf_to_acc<ACC>(v1);
        } else if (KT == 4) {
          float v0, v1, v2, v3;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(la));
          acc[0] += leaf_to_acc<ACC>(v0);
          acc[KT > 1 ? 1 : 0] += leaf_to_acc<ACC>(v1);
          acc[KT > 2 ? 2 : 0] += leaf_to_acc<ACC>(v2);
          acc[KT > 3 ? 3 : 0] += leaf_to_acc<ACC>(v3);
        } else {
#pragma unroll
          for (int k = 0; k < KT; ++k) acc[k] += leaf_to_acc<ACC>(ptx::lds_f32(la + 4u * k));
        }
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < NI; ++u) idx[u] = (int)((A[u] + cb[u] - 4u) >> 2);
  } else {
    constexpr uint32_t kFeatMask = ML ? 0x7fffffffu : 0xffffffffu;
    const uint2* nb = static_cast<const uint2*>(nodes) + (size_t)j * I;
    const float* xf = static_cast<const float*>(xl);
    for (int lvl = 0; lvl < D; ++lvl) {
      uint2 a[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) a[u] = nb[u * I + idx[u]];
      float x[NI];
#pragma unroll
      for (int u = 0; u < NI; ++u) x[u] = xf[(a[u].y & kFeatMask) * 32];
#pragma unroll
      for (int u = 0; u < NI; ++u) idx[u] = 2 * idx[u] + 1 + go_right<ML>(x[u], a[u]);
    }
  }
  if (p.mode == TRAV_APPLY) {
    if (row < p.n_rows) {
      int32_t* o = p.out_leaf + row * p.T;
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        const int s = c.first_slot + j + u;
        o[p.slot_tree[s]] = p.leaf_ids[p.slot_leafid_off[s] + idx[u] - I];
      }
    }
    return;
  }
  if (KT == K && (KT == 2 || KT == 4)) {
    // K == KT: one vector load per tree (8/16-byte aligned leaf records)
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      const float* e = leaves + ((size_t)(j + u) * L + (idx[u] - I)) * KT;
      if (KT == 2) {
        const float2 v = *reinterpret_cast<const float2*>(e);
        acc[0] += leaf_to_acc<ACC>(v.x);
        acc[KT > 1 ? 1 : 0] += leaf_to_acc<ACC>(v.y);
      } else {
        const float4 v = *reinterpret_cast<const float4*>(e);
        acc[0] += leaf_to_acc<ACC>(v.x);
        acc[KT > 1 ? 1 : 0] += leaf_to_acc<ACC>(v.y);
        acc[KT > 2 ? 2 : 0] += leaf_to_acc<ACC>(v.z);
        acc[KT > 3 ? 3 : 0] += leaf_to_acc<ACC>(v.w);
      }
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const float* e = leaves + ((size_t)(j + u) * L + (idx[u] - I)) * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) acc[k] += leaf_to_acc<ACC>(e[k]);
  }
}

// one pass over r (<= 12) trees with ILP = r
template <int KT, typename ACC, bool ML, bool CODES, int MAXNI, bool SPLIT = false, int DT = 0>
__device__ __forceinline__ void walk_tail(int r, const TravParams& p, const TravChunk& c, const void* nodes,
                                          const float* leaves, const void* xl, int j, int I, int L, int D, int K,
                                          int64_t row, ACC (&acc)[KT]) {
  switch (r) {
#define BRIDGER_TAIL(N) \
  case N: if (N <= MAXNI) walk_trees<(N <= MAXNI ? N : 1), KT, ACC, ML, CODES, SPLIT, DT>(p, c, nodes, leaves, xl, j, I, L, D, K, row, acc); break;
    BRIDGER_TAIL(1) BRIDGER_TAIL(2) BRIDGER_TAIL(3) BRIDGER_TAIL(4) BRIDGER_TAIL(5) BRIDGER_TAIL(6)
    BRIDGER_TAIL(7) BRIDGER_TAIL(8) BRIDGER_TAIL(9) BRIDGER_TAIL(10) BRIDGER_TAIL(11) BRIDGER_TAIL(12)
#undef BRIDGER_TAIL
    default: break;
  }
}

// Barrier among the G warps that share one row block (named barrier 1+group).
__device__ __forceinline__ void group_sync(int group, int G) {
  if (G == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(G * 32) : "memory");
  }
}

// Hybrid heap format for trees too large for shared memory (C4: depth 12,
// 8-class leaves): the top `top` levels of the chunk's trees are resident in
// shared memory (where the walk is broadcast-heavy and conflict-light), the
// deeper levels and the leaves are read from global memory (L1/L2).
template <int NI, int KT, typename ACC, bool ML>
__device__ __forceinline__ void walk_hybrid(const TravParams& p, const TravChunk& c, const uint2* top_nodes,
                                            const float* xf, int j, int K, int64_t row, ACC (&acc)[KT]) {
  const int D = c.depth, top = c.top_levels;
  const int It = (1 << top) - 1, I = (1 << D) - 1, L = 1 << D, Ib = I - It;
  const uint2* nt = top_nodes + (size_t)j * It;
  const uint2* nbm = p.hyb_nodes + c.g_nodes + (int64_t)j * Ib;
  int idx[NI];
#pragma unroll
  for (int u = 0; u < NI; ++u) idx[u] = 0;
  for (int lvl = 0; lvl < top; ++lvl) {
    uint2 a[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) a[u] = nt[u * It + idx[u]];
    float x[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) x[u] = xf[(a[u].y & (ML ? 0x7fffffffu : 0xffffffffu)) * 32];
#pragma unroll
    for (int u = 0; u < NI; ++u) idx[u] = 2 * idx[u] + 1 + go_right<ML>(x[u], a[u]);
  }
  for (int lvl = top; lvl < D; ++lvl) {
    uint2 a[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) a[u] = __ldg(nbm + (int64_t)u * Ib + (idx[u] - It));
    float x[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) x[u] = xf[(a[u].y & (ML ? 0x7fffffffu : 0xffffffffu)) * 32];
#pragma unroll
    for (int u = 0; u < NI; ++u) idx[u] = 2 * idx[u] + 1 + go_right<ML>(x[u], a[u]);
  }
  if (p.mode == TRAV_APPLY) {
    if (row < p.n_rows) {
      int32_t* o = p.out_leaf + row * p.T;
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        const int s = c.first_slot + j + u;
        o[p.slot_tree[s]] = p.leaf_ids[p.slot_leafid_off[s] + idx[u] - I];
      }
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const float* e = p.hyb_leaves + c.g_leaves + ((int64_t)(j + u) * L + (idx[u] - I)) * K;
    if (KT == K && (KT == 4 || KT == 8)) {
#pragma unroll
      for (int k4 = 0; k4 < KT; k4 += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(e) + k4 / 4);
        acc[k4 + 0 < KT ? k4 + 0 : 0] += leaf_to_acc<ACC>(v.x);
        acc[k4 + 1 < KT ? k4 + 1 : 0] += leaf_to_acc<ACC>(v.y);
        acc[k4 + 2 < KT ? k4 + 2 : 0] += leaf_to_acc<ACC>(v.z);
        acc[k4 + 3 < KT ? k4 + 3 : 0] += leaf_to_acc<ACC>(v.w);
      }
    } else {
#pragma unroll
      for (int k = 0; k < KT; ++k)
        if (k < K) acc[k] += leaf_to_acc<ACC>(__ldg(e + k));
    }
  }
}

template <int KT, typename ACC, bool ML>
__device__ __forceinline__ void walk_hybrid_tail(int r, const TravParams& p, const TravChunk& c, const uint2* top,
                                                 const float* xf, int j, int K, int64_t row, ACC (&acc)[KT]) {
  switch (r) {
#define BRIDGER_HTAIL(N) \
  case N: walk_hybrid<N, KT, ACC, ML>(p, c, top, xf, j, K, row, acc); break;
    BRIDGER_HTAIL(1) BRIDGER_HTAIL(2) BRIDGER_HTAIL(3) BRIDGER_HTAIL(4) BRIDGER_HTAIL(5) BRIDGER_HTAIL(6)
    BRIDGER_HTAIL(7) BRIDGER_HTAIL(8)
#undef BRIDGER_HTAIL
    default: break;
  }
}

// Sparse (pointer) format for unbounded / unbalanced trees (§8(f3)): BFS order,
// the two children of a node adjacent; record {threshold, feature | missing<<30
// | leaf<<31, left-child index or leaf index, -}.  NI trees walk together;
// lanes that reached a leaf idle until the pass's deepest tree is done.
template <int NI, int KT, typename ACC, bool ML>
__device__ __forceinline__ void walk_sparse(const TravParams& p, int t0, const float* xl, int K, int64_t row,
                                            ACC (&acc)[KT]) {
  int64_t base[NI];
  int32_t idx[NI], leaf[NI];
  int steps = 0;
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const SparseTree td = p.sparse[t0 + u];
    base[u] = td.node_off;
    idx[u] = 0;
    leaf[u] = -1;
    steps = max(steps, td.depth + 1);
  }
  for (int s = 0; s < steps; ++s) {
#pragma unroll
    for (int u = 0; u < NI; ++u)
      if (leaf[u] < 0) {
        const uint4 r = __ldg(p.sparse_nodes + base[u] + idx[u]);
        if (r.y >> 31) {
          leaf[u] = (int32_t)r.z;
        } else {
          const float x = xl[(r.y & 0x3FFFFFFFu) * 32];
          int go = !(x <= __uint_as_float(r.x));
          if (ML) go &= !(((r.y >> 30) & 1u) & isnan(x));
          idx[u] = (int32_t)r.z + go;
        }
      }
  }
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const SparseTree td = p.sparse[t0 + u];
    if (p.mode == TRAV_APPLY) {
      if (row < p.n_rows) p.out_leaf[row * p.T + td.slot_tree] = p.leaf_ids[td.leafid_off + leaf[u]];
    } else {
      const float* e = reinterpret_cast<const float*>(p.data) + td.leaf_off + (int64_t)leaf[u] * K;
#pragma unroll
      for (int k = 0; k < KT; ++k)
        if (k < K) acc[k] += leaf_to_acc<ACC>(__ldg(e + k));
    }
  }
}

template <int KT, typename ACC, bool ML>
__device__ __forceinline__ void walk_sparse_tail(int r, const TravParams& p, int t0, const float* xl, int K,
                                                 int64_t row, ACC (&acc)[KT]) {
  switch (r) {
#define BRIDGER_STAIL(N) \
  case N: walk_sparse<N, KT, ACC, ML>(p, t0, xl, K, row, acc); break;
    BRIDGER_STAIL(1) BRIDGER_STAIL(2) BRIDGER_STAIL(3) BRIDGER_STAIL(4) BRIDGER_STAIL(5) BRIDGER_STAIL(6)
    BRIDGER_STAIL(7) BRIDGER_STAIL(8)
#undef BRIDGER_STAIL
    default: break;
  }
}

template <int KT, typename ACC, bool ML, bool GT, int FMT>
__global__ void __launch_bounds__(512, 1) trav_kernel(const TravParams p) {
  constexpr bool CODES = FMT == FMT_CODES;
  constexpr bool SPARSE = FMT == FMT_SPARSE;
  // PRE: the input arrives pre-laid-out as feature-major [F][32] blocks (u16
  // codes or pre-transposed fp32), bulk-copied into two buffers per group
  constexpr bool HYB = FMT == FMT_HYBRID;
  constexpr bool PRE = CODES || FMT == FMT_HEAP_T || HYB;  // hybrid always takes pre-transposed input
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int G = p.group, NB = NW / G;          // G warps share each of NB row blocks
  const int grp = warp / G, gw = warp % G;     // row-block group, warp within the group
  const int chunk_id = blockIdx.x % p.n_chunks_grid;
  const int cta_in_chunk = blockIdx.x / p.n_chunks_grid;
  const TravChunk c = p.chunks[chunk_id];
  const int F = p.F;
  const int K = p.K;

  uint8_t* cdata = smem;
  // per row-block group: fp32 mode  Xs [F][32] float + St [32][F] float (256*F B)
  //                      codes mode Cb[2] [F2/2][32][2] u16 in 2^b-aligned buffers, double buffered
  const int F2 = (F + 1) & ~1;  // codes: feature pairs interleaved per lane, [F2/2][32][2] u16
  // codes: two 2^b-aligned buffers of code_buf bytes per group (trav_x_region)
  const size_t xblk = CODES ? (size_t)2 * p.code_buf : (size_t)256 * F;  // HEAP_T: 2 x 128F, same as Xs + St
  float* Xs = reinterpret_cast<float*>(smem + p.chunk_cap + (size_t)grp * xblk);  // [F][32]
  float* St = Xs + 32 * F;                                                         // [32][F]
  uint8_t* Cb = nullptr;
  if (CODES) {
    const uint32_t a0 = ptx::s2u(smem + p.chunk_cap);
    const uint32_t al = (a0 + (uint32_t)p.code_buf - 1u) & ~((uint32_t)p.code_buf - 1u);
    Cb = smem + p.chunk_cap + (al - a0) + (size_t)grp * xblk;
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.chunk_cap + trav_x_region(CODES, F, NB));
  uint64_t* red = reinterpret_cast<uint64_t*>(smem + p.red_off);  // [NB][G-1][32][K] intra-group partials

  const bool clustered = p.mode == TRAV_CLUSTER;
  const int nC = p.n_chunks;
  uint64_t* full_bar = bars + 1 + NB;        // [NB][2] (leader): peers' partials landed
  uint64_t* empty_bar = bars + 1 + 3 * NB;   // [NB][2] (peers): leader consumed the slot
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars[0], 1);
    for (int b = 0; b < NB; ++b) ptx::mbar_init(&bars[1 + b], 1);
    for (int b = 0; b < NB; ++b) ptx::mbar_init(&bars[1 + 5 * NB + b], 1);  // codes: 2nd buffer
    if (clustered)
      for (int b = 0; b < 2 * NB; ++b) {
        ptx::mbar_init(&full_bar[b], 32 * (nC - 1));
        ptx::mbar_init(&empty_bar[b], 32);
      }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (clustered) ptx::cluster_sync();
  else __syncthreads();
  if (!GT && threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bars[0], (uint32_t)c.bytes);
    const uint8_t* src = p.data + c.offset;
    for (int32_t o = 0; o < c.bytes; o += 65536) {
      const uint32_t n = (uint32_t)min(65536, c.bytes - o);
      ptx::bulk_g2s(cdata + o, src + o, n, &bars[0]);
    }
  }

  const int64_t n_rows = p.n_rows;
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t stride = (int64_t)p.cpc * NB;
  int64_t blk = (int64_t)cta_in_chunk * NB + grp;
  uint64_t* sbar = &bars[1 + grp];
  uint32_t sphase = 0;
  const uint32_t block_bytes = 32u * (uint32_t)F * 4u;

  auto issue = [&](int64_t b) {  // warp 0 of the group, lane 0: next block -> staging
    if (gw == 0 && lane == 0 && b < n_blocks && (b + 1) * 32 <= n_rows) {
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(sbar, block_bytes);
      ptx::bulk_g2s(St, p.X + b * 32 * (int64_t)F, block_bytes, sbar);
    }
  };
  // codes mode: blocks of the binned input are [F][32] u16, always complete
  const uint8_t* codes = reinterpret_cast<const uint8_t*>(p.X);
  const uint32_t code_block_bytes = CODES ? 64u * (uint32_t)F2 : 128u * (uint32_t)F;
  auto issue_codes = [&](int64_t b, int s) {
    if (gw == 0 && lane == 0 && b < n_blocks) {
      uint64_t* bar = s ? &bars[1 + 5 * NB + grp] : sbar;
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(bar, code_block_bytes);
      uint8_t* dst = CODES ? Cb + (size_t)s * p.code_buf : reinterpret_cast<uint8_t*>(Xs) + (size_t)s * code_block_bytes;
      ptx::bulk_g2s(dst, codes + b * (int64_t)code_block_bytes, code_block_bytes, bar);
    }
  };
  if (PRE) issue_codes(blk, 0);
  else issue(blk);
  if (!GT) ptx::mbar_wait(&bars[0], 0);  // chunk resident

  // feature share of the transpose
  const int f_lo = F * gw / G, f_hi = F * (gw + 1) / G;
  uint64_t* slots = reinterpret_cast<uint64_t*>(smem + p.slot_off);  // [NB][2][nC-1][32][K]
  uint32_t it = 0;

  uint32_t itx = 0;  // blocks consumed by this group (codes double buffer)
  while (blk < n_blocks) {
    const int64_t row0 = blk * 32;
    const int64_t next = blk + stride;
    const void* xptr;
    if (PRE) {
      const int sb = itx & 1;
      ptx::mbar_wait(sb ? &bars[1 + 5 * NB + grp] : sbar, (itx >> 1) & 1);
      ++itx;
      issue_codes(next, sb ^ 1);  // the other buffer was released by the previous block's group sync
      xptr = (CODES ? Cb + (size_t)sb * p.code_buf : reinterpret_cast<const uint8_t*>(Xs) + (size_t)sb * code_block_bytes) +
             4 * lane;
    } else {
      const bool full = row0 + 32 <= n_rows;
      if (full) {
        ptx::mbar_wait(sbar, sphase);
        sphase ^= 1;
      } else {
        const int rows = (int)(n_rows - row0);
        const float* src = p.X + row0 * F;
        if (gw == 0)
          for (int e = lane; e < rows * F; e += 32) St[e] = src[e];
        group_sync(grp, G);
      }
      // transpose staging [32][F] -> feature-major [F][32] (features split over
      // the group's warps).  Every write hits bank `lane`; reads of row `lane`
      // start at a lane-dependent feature so one instruction spreads over banks.
      if ((F & 3) == 0 && G == 1) {
        const float4* srow = reinterpret_cast<const float4*>(St + lane * F);
#pragma unroll 2
        for (int f4 = 0; f4 < F / 4; ++f4) {
          const float4 v = srow[f4];
          Xs[(4 * f4 + 0) * 32 + lane] = v.x;
          Xs[(4 * f4 + 1) * 32 + lane] = v.y;
          Xs[(4 * f4 + 2) * 32 + lane] = v.z;
          Xs[(4 * f4 + 3) * 32 + lane] = v.w;
        }
      } else {
        const float* srow = St + lane * F;
        const int span = f_hi - f_lo;
        if (span > 0) {
          int f = f_lo + lane % span;
#pragma unroll 4
          for (int f0 = 0; f0 < span; ++f0) {
            Xs[f * 32 + lane] = srow[f];
            f = (f + 1 == f_hi) ? f_lo : f + 1;
          }
        }
      }
      group_sync(grp, G);  // Xs ready, staging free
      issue(next);
      xptr = Xs + lane;
    }

    const int64_t row = row0 + lane;
    ACC acc[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) acc[k] = ACC(0);

    // ceil(nt / NI_MAX) passes of (nearly) equal size: each pass walks its
    // trees as independent dependency chains (ILP); a pass costs about the same
    // latency whatever its width, so the pass count is what matters.  Full ILP
    // range for the common int64 / no-missing / K <= 8 kernels, passes of <= 4
    // for the rare variants (compile time).
    auto run_chunk = [&](const TravChunk& cc, const uint8_t* base) {
      constexpr int NI_MAX = (!ML && KT <= 8 && !std::is_same<ACC, double>::value) ? 12 : 4;
      const int D = cc.depth;
      const int I = (1 << D) - 1, L = 1 << D;
      const void* nodes = base;
      const float* leaves = reinterpret_cast<const float*>(base + cc.leaf_offset);
      // this warp's share of the chunk's trees
      const int t0 = (int)((int64_t)cc.n_trees * gw / G), t1 = (int)((int64_t)cc.n_trees * (gw + 1) / G);
      const int nt = t1 - t0;
      const int n_pass = (nt + NI_MAX - 1) / NI_MAX;
      int j = t0;
      for (int q = 0; q < n_pass; ++q) {
        const int sz = nt / n_pass + (q < nt % n_pass ? 1 : 0);
        constexpr bool kFixedD = CODES && !ML && KT <= 8 && std::is_same<ACC, long long>::value;
        if (kFixedD && D == 8)
          walk_tail<KT, ACC, ML, CODES, NI_MAX, false, 8>(sz, p, cc, nodes, leaves, xptr, j, I, L, D, K, row, acc);
        else if (kFixedD && D == 6)
          walk_tail<KT, ACC, ML, CODES, NI_MAX, false, 6>(sz, p, cc, nodes, leaves, xptr, j, I, L, D, K, row, acc);
        else
          walk_tail<KT, ACC, ML, CODES, NI_MAX, FMT == FMT_SPLIT>(sz, p, cc, nodes, leaves, xptr, j, I, L, D, K, row, acc);
        j += sz;
      }
    };
    if (HYB) {
      const int nt = (int)((int64_t)c.n_trees * (gw + 1) / G) - (int)((int64_t)c.n_trees * gw / G);
      const int t0 = (int)((int64_t)c.n_trees * gw / G);
      const int n_pass = (nt + 7) / 8;
      int j = t0;
      for (int q = 0; q < n_pass; ++q) {
        const int sz = nt / n_pass + (q < nt % n_pass ? 1 : 0);
        walk_hybrid_tail<KT, ACC, ML>(sz, p, c, reinterpret_cast<const uint2*>(cdata), static_cast<const float*>(xptr),
                                      j, K, row, acc);
        j += sz;
      }
    } else if (SPARSE) {
      // pointer-format trees from global memory: every CTA walks every tree
      const int T = c.n_trees;
      const int t0 = (int)((int64_t)T * gw / G), t1 = (int)((int64_t)T * (gw + 1) / G);
      const int nt = t1 - t0;
      const int n_pass = (nt + 7) / 8;
      int j = t0;
      for (int q = 0; q < n_pass; ++q) {
        const int sz = nt / n_pass + (q < nt % n_pass ? 1 : 0);
        walk_sparse_tail<KT, ACC, ML>(sz, p, j, static_cast<const float*>(xptr), K, row, acc);
        j += sz;
      }
    } else if (GT) {
      // trees too large for shared memory: every CTA walks all chunks from
      // global memory (L1/L2), no cross-CTA combine
      for (int ci = 0; ci < nC; ++ci) {
        const TravChunk cc = p.chunks[ci];
        run_chunk(cc, p.data + cc.offset);
      }
    } else {
      run_chunk(c, cdata);
    }

    if (p.mode != TRAV_APPLY) {
      // combine the group's warps (exact int64 / fixed order)
      uint64_t* gred = red + (size_t)grp * (G - 1) * 32 * K;
      if (gw > 0) {
        uint64_t* dst = gred + ((size_t)(gw - 1) * 32 + lane) * K;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < K) dst[k] = reinterpret_cast<const uint64_t&>(acc[k]);
      }
      group_sync(grp, G);
      if (gw == 0) {
        for (int q = 0; q < G - 1; ++q) {
          const uint64_t* src = gred + ((size_t)q * 32 + lane) * K;
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (k < K) acc[k] += reinterpret_cast<const ACC&>(src[k]);
        }
        if (clustered) {
          const int s = it & 1;
          const uint32_t ph = (it >> 1) & 1;
          ++it;
          uint64_t* slot = slots + (size_t)(grp * 2 + s) * (nC - 1) * 32 * K;
          if (chunk_id != 0) {
            ptx::mbar_wait_cluster(&empty_bar[grp * 2 + s], ph ^ 1);
            const uint32_t dst = ptx::mapa(ptx::s2u(slot + ((size_t)(chunk_id - 1) * 32 + lane) * K), 0);
#pragma unroll
            for (int k = 0; k < KT; ++k)
              if (k < K) ptx::st_cluster_u64(dst + 8 * k, reinterpret_cast<const uint64_t&>(acc[k]));
            ptx::mbar_arrive_remote(ptx::mapa(ptx::s2u(&full_bar[grp * 2 + s]), 0));
          } else {
            ptx::mbar_wait_cluster(&full_bar[grp * 2 + s], ph);
            for (int q = 0; q < nC - 1; ++q) {
              const uint64_t* src = slot + ((size_t)q * 32 + lane) * K;
#pragma unroll
              for (int k = 0; k < KT; ++k)
                if (k < K) acc[k] += reinterpret_cast<const ACC&>(src[k]);
            }
            for (int q = 1; q < nC; ++q)
              ptx::mbar_arrive_remote(ptx::mapa(ptx::s2u(&empty_bar[grp * 2 + s]), q));
            if (row < n_rows) finalize_row<KT, ACC>(p.fin, row, acc);
          }
        } else if (row < n_rows) {
          if (p.mode == TRAV_PARTIAL) {
            ACC* o = static_cast<ACC*>(p.partial) + ((size_t)chunk_id * n_rows + row) * K;
#pragma unroll
            for (int k = 0; k < KT; ++k)
              if (k < K) o[k] = acc[k];
          } else {
            finalize_row<KT, ACC>(p.fin, row, acc);
          }
        }
      }
    } else {
      group_sync(grp, G);  // keep the group's barrier sequence uniform
    }
    blk = next;
  }
  if (clustered) ptx::cluster_sync();  // no CTA leaves while peers may touch its shared memory
}

// Sum per-chunk partials in chunk order (exact for int64) and finalize.
template <int KT, typename ACC>
__global__ void __launch_bounds__(256) trav_combine_kernel(const ACC* partial, int32_t n_chunks,
                                                            int64_t n_rows, FinalizeArgs fin) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n_rows) return;
  const int K = fin.K;
  ACC acc[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) acc[k] = ACC(0);
  for (int c = 0; c < n_chunks; ++c) {
    const ACC* src = partial + ((size_t)c * n_rows + row) * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) acc[k] += src[k];
  }
  finalize_row<KT, ACC>(fin, row, acc);
}

template <int KT, typename ACC, bool ML, bool GT, int FMT>
cudaError_t launch_trav_t(const TravParams& p, int grid_ctas, int block, int smem, int cluster,
                                 cudaStream_t st) {
  auto kern = trav_kernel<KT, ACC, ML, GT, FMT>;
  static std::atomic<uint64_t> configured{0};  // per instantiation, per device
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(kern), configured);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int grid = grid_ctas;
  if (cluster > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cluster);
    int max_clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&max_clusters, (void*)kern, &cfg);
    if (std::getenv("BRIDGER_DEBUG"))
      std::fprintf(stderr, "[bridger] cluster=%d smem=%d max_active_clusters=%d (%s)\n", cluster, smem,
                   max_clusters, cudaGetErrorString(e));
    if (e != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      return cudaErrorNotSupported;  // caller falls back to partials
    }
    grid = std::min(grid_ctas, max_clusters * cluster);
    grid = std::max(cluster, grid / cluster * cluster);
  }
  cfg.gridDim = dim3(grid);
  TravParams q = p;
  q.cpc = grid / p.n_chunks_grid;
  if (std::getenv("BRIDGER_DEBUG"))
    std::fprintf(stderr, "[bridger] trav_kernel mode=%d grid=%d block=%d smem=%d cluster=%d chunks=%d cpc=%d\n", q.mode,
                 grid, block, smem, cluster, q.n_chunks, q.cpc);
  cudaEvent_t ev;
  hot_begin(st, &ev);
  e = cudaLaunchKernelEx(&cfg, kern, q);
  hot_end(st, ev);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Tree-streamed traversal (K4s) for ensembles too large for shared-memory
// residency (C4: depth-12 trees of 32 KB nodes + 128 KB 8-class leaves, 164 MB
// in total).  The loop order is the transpose of the resident kernel's: a CTA
// keeps a TILE of rows (one row per thread, 512 rows) resident in shared memory
// -- feature-major 32-row blocks of the pre-transposed input, so x = Xs[f*32 +
// lane] is conflict free -- and STREAMS every chunk's node records through a
// ring of bulk copies (TMA engine) issued by a dedicated loader warp.  Per-row
// accumulators stay in registers across the whole ensemble: no per-chunk
// partials, no combine pass.  Leaf values are read from global memory (L2):
// every CTA walks the same chunk at about the same time, so a chunk's nodes and
// leaves are L2-resident while it is in flight.  Leaf gathers are
// software-pipelined by one pass (loads of pass p land while pass p+1 walks).
template <int W, bool ML>
__device__ __forceinline__ void stream_walk(const uint2* nb, const float* xl, int I, int D, int (&idx)[W]) {
  // nb: tree 0's node 0; tree u at nb + u (I + 1) (8-byte front pad per tree,
  // lowering.cpp), so the children pair {2i+1, 2i+2} of every node is one
  // 16-byte-aligned LDS.128.  Child-pair speculation: at each level the
  // feature value of the current node and BOTH children's records are loaded
  // together (independent addresses), the compare then selects the child
  // record already in registers -- one shared-memory latency per level
  // instead of two (node record, then the feature value it names).
  constexpr uint32_t kFeatMask = ML ? 0x7fffffffu : 0xffffffffu;
  uint2 a[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    idx[u] = 0;
    a[u] = nb[u * (I + 1)];
  }
  for (int lvl = 0; lvl < D; ++lvl) {
    float x[W];
    uint4 pr[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
      x[u] = xl[(a[u].y & kFeatMask) * 32];
      if (lvl + 1 < D) pr[u] = *reinterpret_cast<const uint4*>(nb + u * (I + 1) + 2 * idx[u] + 1);
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int r = go_right<ML>(x[u], a[u]);
      idx[u] = 2 * idx[u] + 1 + r;
      if (lvl + 1 < D) a[u] = r ? make_uint2(pr[u].z, pr[u].w) : make_uint2(pr[u].x, pr[u].y);
    }
  }
#pragma unroll
  for (int u = 0; u < W; ++u) idx[u] -= I;  // leaf index
}

// Split node format for streamed trees (F <= 127): per tree [pad][thresholds
// 0..I-1] fp32 then [pad][features 0..I-1] u8 (bit 7 = missing_left), 5 * 2^D
// bytes (vs 8 * 2^D): two trees fit a ring slot where one 8-byte-node tree
// did, so every thread walks two trees at once.  Same child-pair speculation:
// the children's thresholds (8 B) and features (2 B) are loaded with the
// current node's feature value.
template <int W, bool ML>
__device__ __forceinline__ void stream_walk_split(const uint8_t* t0, int tb, const float* xl, int I, int D,
                                                  int (&idx)[W]) {
  float at[W];
  uint32_t af[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    idx[u] = 0;
    at[u] = reinterpret_cast<const float*>(t0 + u * tb)[1];
    af[u] = (t0 + u * tb + (4 << D))[1];
  }
#pragma unroll 4
  for (int lvl = 0; lvl < D; ++lvl) {
    float x[W];
    float2 tp[W];
    uint32_t fp[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
      x[u] = xl[(af[u] & 0x7Fu) * 32];
      // unconditional (no branch in the level loop): at the last level the
      // "children" are read past the tree's arrays -- still inside the ring /
      // landing region of shared memory -- and discarded
      tp[u] = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(t0 + u * tb) + 2 * idx[u] + 2);
      fp[u] = *reinterpret_cast<const uint16_t*>(t0 + u * tb + (4 << D) + 2 * idx[u] + 2);
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {
      int r = !(x[u] <= at[u]);  // NaN -> right (reading c2 default)
      if (ML) r &= !((af[u] >> 7) & isnan(x[u]));
      idx[u] = 2 * idx[u] + 1 + r;
      at[u] = r ? tp[u].y : tp[u].x;
      af[u] = r ? (fp[u] >> 8) : (fp[u] & 0xFFu);
    }
  }
#pragma unroll
  for (int u = 0; u < W; ++u) idx[u] -= I;  // leaf index
}

// Threshold-bin codes for streamed trees: 4-byte node words (code index j <<
// 16 | feature byte offset | missing) behind a pad word per tree (tree stride
// 4 (I + 1), node idx at T + 4 (idx + 1), lowering.cpp); xb = this lane's
// column of its warp's 2^b-aligned code block.  Child-pair speculation (as in
// trav_deep.cu): per level the lane's code of the current node and the words
// of BOTH children (one LDS.64) are loaded together and the compare selects
// the child already in registers -- one shared-memory latency per level
// instead of two (the depth-12 streamed walk is latency-bound).
template <int W, bool ML>
__device__ __forceinline__ void stream_walk_codes(uint32_t nb, int tstride, int umax, uint32_t xb, uint32_t mask,
                                                  uint32_t k2, uint32_t k16, int I, int D, int (&idx)[W]) {
  uint32_t A[W], cb[W], a[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    A[u] = nb + (uint32_t)(min(u, umax) * tstride);  // node 0; chunks with < W trees re-walk their last tree
    cb[u] = 4u - A[u];
    a[u] = ptx::lds_u32(A[u]);
  }
  for (int lvl = 0; lvl + 1 < D; ++lvl) {
    uint32_t x[W], c0[W], c1[W];
#pragma unroll
    for (int u = 0; u < W; ++u) x[u] = ptx::lds_u16(xb | (a[u] & mask));
#pragma unroll
    for (int u = 0; u < W; ++u) {
      A[u] = A[u] * k2 + cb[u];  // left child (the pair {left, right} is 8-byte aligned)
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(c0[u]), "=r"(c1[u]) : "r"(A[u]));
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {
      bool r = x[u] * k16 > a[u];  // code(x) > j; NaN code 0xFFFF -> right
      if (ML) r = r && !((a[u] & 1u) && x[u] == 0xFFFFu);
      a[u] = r ? c1[u] : c0[u];
      if (r) A[u] += 4u;
    }
  }
#pragma unroll
  for (int u = 0; u < W; ++u) {
    const uint32_t x = ptx::lds_u16(xb | (a[u] & mask));
    bool r = x * k16 > a[u];
    if (ML) r = r && !((a[u] & 1u) && x == 0xFFFFu);
    A[u] = A[u] * k2 + cb[u];
    if (r) A[u] += 4u;
    idx[u] = (int)((A[u] + cb[u] - 4u) >> 2) - I;  // leaf index
  }
}

// W: trees walked together per pass (= the chunk width chosen at lowering; a
// chunk's last pass masks trees past its end).  The steady-state loop has no
// divergent branch: ptxas drains every load scoreboard at one, which would
// serialise the leaf-gather latency the pipelining hides.
// SF: streamed node format -- 0: 8-byte records, 1: split (fp32 thresholds +
// u8 features), 2: threshold-bin codes (4-byte words, u16 input codes)
template <int KT, typename ACC, bool ML, int W, bool APPLY, int SF = 0>
// Coded walks with K <= 8: up to 20 walking warps + the loader (672 threads;
// C4: 16 -> 20 warps, 13.27 -> 12.2 ms per 1M rows -- an 800-thread bound
// forces spills at 72 registers); other formats keep 16 + 1 (their larger
// per-thread state spills under the 672-thread register cap).
__global__ void __launch_bounds__((SF == 2 && KT <= 8) ? 672 : 544, 1) trav_stream_kernel(const TravParams p) {
  constexpr bool SPL = SF == 1;
  constexpr bool SCODES = SF == 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NWc = (blockDim.x >> 5) - 1;  // walking warps; the last warp is the loader
  const int RB = NWc * 32;                // rows per tile
  const int NS = p.stream_ns, F = p.F, K = p.K, nC = p.n_chunks;
  float* Xs = reinterpret_cast<float*>(smem);
  // codes: per-warp code-block buffers aligned to their power-of-two size
  uint8_t* xcodes = smem;
  if (SCODES) {
    const uint32_t a0 = ptx::s2u(smem);
    xcodes = smem + (((a0 + (uint32_t)p.code_buf - 1u) & ~((uint32_t)p.code_buf - 1u)) - a0);
  }
  uint8_t* ring = smem + p.stream_x_bytes;
  // per-thread landing slot of the previous pass's leaf values (cp.async)
  float* lbuf_all = reinterpret_cast<float*>(ring + (size_t)NS * p.stream_stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(lbuf_all) + p.stream_lbuf_bytes);
  uint64_t* xbar = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + NS;
  if (threadIdx.x == 0) {
    ptx::mbar_init(xbar, 1);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], RB);  // every walking thread arrives (no elected-lane branch)
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  __syncthreads();
  const int64_t n_rows = p.n_rows;
  const int64_t n_tiles = (n_rows + RB - 1) / RB;
  const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_items = my_tiles * nC;

  if (warp == NWc) {
    // loader: chunk node records, in item order, into the ring.  Each slot =
    // [64-byte header: the chunk descriptor][node records]; the header is
    // written with plain stores before the (release) arrive, so the walkers
    // never issue a global load for it.
    if (lane == 0) {
      int s = 0, c_i = 0;
      uint32_t ph = 0;
      for (int64_t k = 0; k < n_items; ++k) {
        const TravChunk c = p.chunks[c_i];
        if (++c_i == nC) c_i = 0;
        ptx::mbar_wait_sleep(&empty[s], ph ^ 1, 256);
        uint8_t* slot = ring + (size_t)s * p.stream_stage;
        *reinterpret_cast<TravChunk*>(slot) = c;
        ptx::fence_proxy_async();
        ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)c.leaf_offset);
        ptx::bulk_g2s(slot + 64, p.data + c.offset, (uint32_t)c.leaf_offset, &full[s]);
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  const int64_t n_blocks = (n_rows + 31) / 32;
  uint32_t xphase = 0;
  // ring position kept incrementally: no 64-bit division in the loop
  int s = 0;
  uint32_t ph = 0;
  for (int64_t ti = 0; ti < my_tiles; ++ti) {
    const int64_t tile = blockIdx.x + ti * gridDim.x;
    const int64_t blk0 = tile * (RB / 32);
    const int nblk = (int)(n_blocks - blk0 < RB / 32 ? n_blocks - blk0 : RB / 32);
    // every walking warp is done with the previous tile: reload X
    asm volatile("bar.sync 1, %0;" ::"r"(RB) : "memory");
    if (threadIdx.x == 0) {
      ptx::fence_proxy_async();
      if (SCODES) {
        // one code block (64 * F2 bytes) per walking warp, into its 2^b-aligned buffer
        const uint32_t cbytes = 64u * (uint32_t)((F + 1) & ~1);
        ptx::mbar_arrive_expect_tx(xbar, (uint32_t)nblk * cbytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.X) + blk0 * (int64_t)cbytes;
        for (int w = 0; w < nblk; ++w)
          ptx::bulk_g2s(xcodes + (size_t)w * p.code_buf, src + (size_t)w * cbytes, cbytes, xbar);
      } else {
        const uint32_t bytes = (uint32_t)nblk * 32u * (uint32_t)F * 4u;
        ptx::mbar_arrive_expect_tx(xbar, bytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.X) + blk0 * 32 * (int64_t)F * 4;
        for (uint32_t o = 0; o < bytes; o += 65536u)
          ptx::bulk_g2s(reinterpret_cast<uint8_t*>(Xs) + o, src + o, min(65536u, bytes - o), xbar);
      }
    }
    ptx::mbar_wait(xbar, xphase);
    xphase ^= 1;
    const int64_t row = tile * RB + warp * 32 + lane;
    const float* xl = Xs + (size_t)warp * F * 32 + lane;
    const uint32_t xcl = SCODES ? ptx::s2u(xcodes + (size_t)warp * p.code_buf) + 4u * lane : 0u;
    ACC acc[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) acc[q] = ACC(0);
    // The previous pass's leaf values land in this thread's shared-memory slot
    // through cp.async: their completion is tracked by the async-copy group,
    // not by a register scoreboard, so the walk's loops and branches (where
    // ptxas drains outstanding loads) do not serialise the gather latency.
    // element-major: value v of this thread at lbuf[v * RB] (float4 units when
    // K % 4 == 0), so a warp's copies and reads touch consecutive words
    constexpr bool V4 = (KT % 4) == 0;
    const bool v4 = V4 && KT == K;
    float* lbuf = lbuf_all + (size_t)threadIdx.x * (v4 ? 4 : 1);
    uint32_t pmask[W];
#pragma unroll
    for (int u = 0; u < W; ++u) pmask[u] = 0u;
    auto flush = [&]() {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const uint32_t m = pmask[u];
        if (v4) {
#pragma unroll
          for (int q = 0; q < KT; q += 4) {
            const float4 v = *reinterpret_cast<const float4*>(lbuf + (size_t)(u * (KT / 4) + q / 4) * RB * 4);
            acc[q] += leaf_to_acc<ACC>(__uint_as_float(__float_as_uint(v.x) & m));
            acc[q + 1 < KT ? q + 1 : 0] += leaf_to_acc<ACC>(__uint_as_float(__float_as_uint(v.y) & m));
            acc[q + 2 < KT ? q + 2 : 0] += leaf_to_acc<ACC>(__uint_as_float(__float_as_uint(v.z) & m));
            acc[q + 3 < KT ? q + 3 : 0] += leaf_to_acc<ACC>(__uint_as_float(__float_as_uint(v.w) & m));
          }
        } else {
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < K) acc[q] += leaf_to_acc<ACC>(__uint_as_float(__float_as_uint(lbuf[(size_t)(u * K + q) * RB]) & m));
        }
        pmask[u] = 0u;
      }
    };
    ptx::mbar_wait(&full[s], ph);
    for (int c = 0; c < nC; ++c) {
      const uint8_t* slot = ring + (size_t)s * p.stream_stage;
      const TravChunk ch = *reinterpret_cast<const TravChunk*>(slot);
      const int D = ch.depth, I = (1 << D) - 1, L = 1 << D;
      const uint2* nodes = reinterpret_cast<const uint2*>(slot + 64);
      const float* leaves = reinterpret_cast<const float*>(p.data + ch.offset + ch.leaf_offset);
      for (int j = 0; j < ch.n_trees; j += W) {
        int idx[W];
        // trees past the chunk's end re-walk its last tree (masked below)
        const int jw = min(j, ch.n_trees - W < 0 ? 0 : ch.n_trees - W);
        if (SCODES) {
          stream_walk_codes<W, ML>(ptx::s2u(nodes) + 4u * (uint32_t)(jw * (I + 1)) + 4u, 4 * (I + 1), ch.n_trees - 1 - jw, xcl,
                                   (uint32_t)p.code_buf - 2u, p.k2, p.k16, I, D, idx);
        } else if (SPL) {
          const int tb = ((5 << D) + 15) & ~15;
          stream_walk_split<W, ML>(reinterpret_cast<const uint8_t*>(nodes) + (size_t)jw * tb, tb, xl, I, D, idx);
        } else {
          stream_walk<W, ML>(nodes + (size_t)jw * (I + 1) + 1, xl, I, D, idx);
        }
        if (APPLY) {
#pragma unroll
          for (int u = 0; u < W; ++u) {
            const int t = jw + u;
            if (t >= j && t < ch.n_trees && row < n_rows) {
              const int sl = ch.first_slot + t;
              p.out_leaf[row * p.T + p.slot_tree[sl]] = p.leaf_ids[p.slot_leafid_off[sl] + idx[u]];
            }
          }
        } else {
          flush();  // the previous pass's leaf values have landed by now
          const bool last_pass = j + W >= ch.n_trees;
          if (last_pass && c + 1 < nC) {
            // next slot's node records: waited for while no leaf load is in flight
            const int s2 = s + 1 == NS ? 0 : s + 1;
            ptx::mbar_wait(&full[s2], s2 == 0 ? ph ^ 1 : ph);
          }
#pragma unroll
          for (int u = 0; u < W; ++u) {
            const int t = jw + u;
            pmask[u] = (t >= j && t < ch.n_trees) ? 0xffffffffu : 0u;
            const float* e = leaves + ((size_t)min(t, ch.n_trees - 1) * L + idx[u]) * K;
            if (v4) {
#pragma unroll
              for (int q = 0; q < KT; q += 4) {
                const uint32_t d = ptx::s2u(lbuf + (size_t)(u * (KT / 4) + q / 4) * RB * 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(e + q) : "memory");
              }
            } else {
#pragma unroll
              for (int q = 0; q < KT; ++q)
                if (q < K) {
                  const uint32_t d = ptx::s2u(lbuf + (size_t)(u * K + q) * RB);
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(e + q) : "memory");
                }
            }
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
      }
      ptx::mbar_arrive(&empty[s]);  // this thread is done with the slot
      if (APPLY && c + 1 < nC) ptx::mbar_wait(&full[s + 1 == NS ? 0 : s + 1], s + 1 == NS ? ph ^ 1 : ph);
      if (++s == NS) {
        s = 0;
        ph ^= 1;
      }
    }
    if (!APPLY) {
      flush();
      if (row < n_rows) finalize_row<KT, ACC>(p.fin, row, acc);
    }
  }
}

template <int KT, typename ACC, bool ML, int W, bool APPLY, int SPL>
cudaError_t launch_stream_t(const TravParams& p, int grid, int block, int smem, cudaStream_t st) {
  auto kern = trav_stream_kernel<KT, ACC, ML, W, APPLY, SPL>;
  static std::atomic<uint64_t> configured{0};  // per instantiation, per device
  cudaError_t e0 = smem_opt_in(reinterpret_cast<const void*>(kern), configured);
  if (e0 != cudaSuccess) return e0;
  if (std::getenv("BRIDGER_DEBUG"))
    std::fprintf(stderr, "[bridger] trav_stream_kernel W=%d grid=%d block=%d smem=%d chunks=%d ns=%d stage=%d\n", W,
                 grid, block, smem, p.n_chunks, p.stream_ns, p.stream_stage);
  cudaEvent_t ev;
  hot_begin(st, &ev);
  kern<<<grid, block, smem, st>>>(p);
  hot_end(st, ev);
  count_launch();
  return cudaGetLastError();
}

#define BRIDGER_STREAM_INSTANTIATE_W(ACC, ML, W, SPL)                                                                  \
  template cudaError_t launch_stream_t<1, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  template cudaError_t launch_stream_t<2, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  template cudaError_t launch_stream_t<4, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  template cudaError_t launch_stream_t<8, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);  \
  template cudaError_t launch_stream_t<16, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t); \
  template cudaError_t launch_stream_t<64, ACC, ML, W, false, SPL>(const TravParams&, int, int, int, cudaStream_t);
#define BRIDGER_STREAM_INSTANTIATE(ACC, ML, SPL)                                                                   \
  BRIDGER_STREAM_INSTANTIATE_W(ACC, ML, 1, SPL)                                                                    \
  BRIDGER_STREAM_INSTANTIATE_W(ACC, ML, 2, SPL)                                                                    \
  template cudaError_t launch_stream_t<1, ACC, ML, 1, true, SPL>(const TravParams&, int, int, int, cudaStream_t); \
  template cudaError_t launch_stream_t<1, ACC, ML, 2, true, SPL>(const TravParams&, int, int, int, cudaStream_t);

#define BRIDGER_TRAV_INSTANTIATE(ACC, ML, GT, FMT)                                                                  \
  template cudaError_t launch_trav_t<1, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  template cudaError_t launch_trav_t<2, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  template cudaError_t launch_trav_t<4, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  template cudaError_t launch_trav_t<8, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  template cudaError_t launch_trav_t<16, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t); \
  template cudaError_t launch_trav_t<64, ACC, ML, GT, FMT>(const TravParams&, int, int, int, int, cudaStream_t);

}  // namespace bridger
