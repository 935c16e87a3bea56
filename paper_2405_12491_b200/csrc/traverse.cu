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
enum TravMode : int32_t { TRAV_FINAL = 0, TRAV_PARTIAL = 1, TRAV_APPLY = 2, TRAV_CLUSTER = 3 };

struct TravParams {
  const float* X;
  int64_t n_rows;
  int32_t F;
  int32_t K;
  const uint8_t* data;
  const TravChunk* chunks;
  int32_t n_chunks;
  int32_t cpc;        // CTAs per chunk
  int32_t chunk_cap;  // bytes reserved for the chunk in shared memory
  int32_t mode;
  void* partial;      // [n_chunks][n_rows][K] ACC   (TRAV_PARTIAL)
  int32_t* out_leaf;  // [n_rows][T]                 (TRAV_APPLY)
  const int32_t* slot_tree;
  const int64_t* slot_leafid_off;
  const int32_t* leaf_ids;
  int32_t T;
  int32_t slot_off;   // byte offset of the DSMEM reduction slots (TRAV_CLUSTER)
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
template <int NI, int KT, typename ACC, bool ML>
__device__ __forceinline__ void walk_trees(const TravParams& p, const TravChunk& c, const uint2* nodes,
                                           const float* leaves, const float* xl, int j, int I, int L, int D,
                                           int K, int64_t row, ACC (&acc)[KT]) {
  constexpr uint32_t kFeatMask = ML ? 0x7fffffffu : 0xffffffffu;
  int idx[NI];
#pragma unroll
  for (int u = 0; u < NI; ++u) idx[u] = 0;
  const uint2* nb = nodes + (size_t)j * I;
  for (int lvl = 0; lvl < D; ++lvl) {
    uint2 a[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) a[u] = nb[u * I + idx[u]];
    float x[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) x[u] = xl[(a[u].y & kFeatMask) * 32];
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
    const float* e = leaves + ((size_t)(j + u) * L + (idx[u] - I)) * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) acc[k] += leaf_to_acc<ACC>(e[k]);
  }
}

template <int KT, typename ACC, bool ML>
__global__ void __launch_bounds__(256, 1) trav_kernel(const TravParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int chunk_id = blockIdx.x % p.n_chunks;
  const int cta_in_chunk = blockIdx.x / p.n_chunks;
  const TravChunk c = p.chunks[chunk_id];
  const int F = p.F;

  uint8_t* cdata = smem;
  float* Xs = reinterpret_cast<float*>(smem + p.chunk_cap) + (size_t)warp * 64 * F;  // [F][32]
  float* St = Xs + 32 * F;                                                           // [32][F]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.chunk_cap + (size_t)NW * 256 * F);

  const bool clustered = p.mode == TRAV_CLUSTER;
  const int nC = p.n_chunks;
  uint64_t* full_bar = bars + 1 + NW;        // [NW][2] (leader): peers' partials landed
  uint64_t* empty_bar = bars + 1 + 3 * NW;   // [NW][2] (peers): leader consumed the slot
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars[0], 1);
    for (int w = 0; w < NW; ++w) ptx::mbar_init(&bars[1 + w], 1);
    if (clustered)
      for (int w = 0; w < 2 * NW; ++w) {
        ptx::mbar_init(&full_bar[w], 32 * (nC - 1));
        ptx::mbar_init(&empty_bar[w], 32);
      }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (clustered) ptx::cluster_sync();
  else __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bars[0], (uint32_t)c.bytes);
    const uint8_t* src = p.data + c.offset;
    for (int32_t o = 0; o < c.bytes; o += 65536) {
      const uint32_t n = (uint32_t)min(65536, c.bytes - o);
      ptx::bulk_g2s(cdata + o, src + o, n, &bars[0]);
    }
  }

  const int64_t n_rows = p.n_rows;
  const int64_t n_blocks = (n_rows + 31) / 32;
  const int64_t stride = (int64_t)p.cpc * NW;
  int64_t blk = (int64_t)cta_in_chunk * NW + warp;
  uint64_t* wbar = &bars[1 + warp];
  uint32_t wphase = 0;
  const uint32_t block_bytes = 32u * (uint32_t)F * 4u;
  const int lane_mod_F = lane % F;

  auto issue = [&](int64_t b) {
    if (b < n_blocks && (b + 1) * 32 <= n_rows && lane == 0) {
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(wbar, block_bytes);
      ptx::bulk_g2s(St, p.X + b * 32 * (int64_t)F, block_bytes, wbar);
    }
  };
  issue(blk);

  ptx::mbar_wait(&bars[0], 0);  // chunk resident

  const int D = c.depth;
  const int I = (1 << D) - 1, L = 1 << D;
  const int K = p.K;
  const int nt = c.n_trees;
  const uint2* nodes = reinterpret_cast<const uint2*>(cdata);
  const float* leaves = reinterpret_cast<const float*>(cdata + c.leaf_offset);
  const float* xl = Xs + lane;
  uint64_t* slots = reinterpret_cast<uint64_t*>(smem + p.slot_off);  // [NW][2][nC-1][32][K]
  uint32_t it = 0;

  while (blk < n_blocks) {
    const int64_t row0 = blk * 32;
    const bool full = row0 + 32 <= n_rows;
    if (full) {
      ptx::mbar_wait(wbar, wphase);
      wphase ^= 1;
    } else {
      const int rows = (int)(n_rows - row0);
      const float* src = p.X + row0 * F;
      for (int e = lane; e < rows * F; e += 32) St[e] = src[e];
      __syncwarp();
    }
    // transpose staging [32][F] -> feature-major [F][32].  Lane l walks the
    // features of row l starting at (l mod F) and wrapping, so one staging read
    // instruction touches 32 different (row, feature) words spread over the
    // banks; every write hits bank `lane`.
    {
      const float* srow = St + lane * F;
      int f = lane_mod_F;
#pragma unroll 4
      for (int f0 = 0; f0 < F; ++f0) {
        Xs[f * 32 + lane] = srow[f];
        f = (f + 1 == F) ? 0 : f + 1;
      }
    }
    __syncwarp();
    const int64_t next = blk + stride;
    issue(next);

    const int64_t row = row0 + lane;
    ACC acc[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) acc[k] = ACC(0);

    int j = 0;
    for (; j + 8 <= nt; j += 8) walk_trees<8, KT, ACC, ML>(p, c, nodes, leaves, xl, j, I, L, D, K, row, acc);
    for (; j + 4 <= nt; j += 4) walk_trees<4, KT, ACC, ML>(p, c, nodes, leaves, xl, j, I, L, D, K, row, acc);
    for (; j < nt; ++j) walk_trees<1, KT, ACC, ML>(p, c, nodes, leaves, xl, j, I, L, D, K, row, acc);

    if (clustered) {
      const int s = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      ++it;
      uint64_t* slot = slots + (size_t)(warp * 2 + s) * (nC - 1) * 32 * K;
      if (chunk_id != 0) {
        ptx::mbar_wait_cluster(&empty_bar[warp * 2 + s], ph ^ 1);
        const uint32_t dst = ptx::mapa(ptx::s2u(slot + ((size_t)(chunk_id - 1) * 32 + lane) * K), 0);
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < K) ptx::st_cluster_u64(dst + 8 * k, reinterpret_cast<const uint64_t&>(acc[k]));
        ptx::mbar_arrive_remote(ptx::mapa(ptx::s2u(&full_bar[warp * 2 + s]), 0));
      } else {
        ptx::mbar_wait_cluster(&full_bar[warp * 2 + s], ph);
        for (int q = 0; q < nC - 1; ++q) {
          const uint64_t* src = slot + ((size_t)q * 32 + lane) * K;
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (k < K) acc[k] += reinterpret_cast<const ACC&>(src[k]);
        }
        for (int q = 1; q < nC; ++q) ptx::mbar_arrive_remote(ptx::mapa(ptx::s2u(&empty_bar[warp * 2 + s]), q));
        if (row < n_rows) finalize_row<KT, ACC>(p.fin, row, acc);
      }
    } else if (row < n_rows) {
      if (p.mode == TRAV_PARTIAL) {
        ACC* o = static_cast<ACC*>(p.partial) + ((size_t)chunk_id * n_rows + row) * K;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < K) o[k] = acc[k];
      } else if (p.mode == TRAV_FINAL) {
        finalize_row<KT, ACC>(p.fin, row, acc);
      }
    }
    blk = next;
    __syncwarp();
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

// ------------------------------------------------------------- launchers ----
static int num_sms(int dev) {
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

template <int KT, typename ACC, bool ML>
static cudaError_t launch_trav_t(const TravParams& p, int grid_ctas, int block, int smem, int cluster,
                                 cudaStream_t st) {
  auto kern = trav_kernel<KT, ACC, ML>;
  static int configured_smem = 0;  // per instantiation
  cudaError_t e;
  if (configured_smem < smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured_smem = 232448;
  }
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
    if (e != cudaSuccess) return e;
    if (max_clusters < 1) return cudaErrorNotSupported;  // caller falls back to partials
    grid = std::min(grid_ctas, max_clusters * cluster);
    grid = std::max(cluster, grid / cluster * cluster);
  }
  cfg.gridDim = dim3(grid);
  TravParams q = p;
  q.cpc = grid / p.n_chunks;
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

// Runs the traversal over all rows.  want: 0 predict, 1 proba, 2 raw, 3 apply.
cudaError_t trav_run(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                     int32_t total_trees, cudaStream_t st) {
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
  p.chunk_cap = (maxc + 127) / 128 * 128;
  p.slot_tree = m->d_slot_tree;
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
  const int NW = L.n_warps;
  const int block = NW * 32;
  const int bars_bytes = ((1 + 5 * NW) * 8 + 15) / 16 * 16;
  p.slot_off = p.chunk_cap + NW * 256 * m->F + bars_bytes;
  int smem = p.slot_off;
  int cluster = 1;
  void* partial = nullptr;
  if (want == 3) {
    p.mode = TRAV_APPLY;
    p.out_leaf = static_cast<int32_t*>(out);
  } else if (n_chunks == 1) {
    p.mode = TRAV_FINAL;
  } else if (n_chunks <= 8) {
    p.mode = TRAV_CLUSTER;
    cluster = n_chunks;
    smem += trav_slot_bytes(NW, n_chunks, m->K);
  } else {
    p.mode = TRAV_PARTIAL;
    cudaError_t e = cudaMallocAsync(&partial, (size_t)n_chunks * n_rows * m->K * 8, st);
    if (e != cudaSuccess) return e;
    p.partial = partial;
  }
  const int cpc = std::max(1, sms / n_chunks);
  const int grid = n_chunks * cpc;
  cudaError_t err = cudaSuccess;
  BRIDGER_DISPATCH_KT(m->K, {
    auto launch = [&]() {
      if (m->acc_int)
        return L.has_missing ? launch_trav_t<KT, long long, true>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, long long, false>(p, grid, block, smem, cluster, st);
      return L.has_missing ? launch_trav_t<KT, double, true>(p, grid, block, smem, cluster, st)
                           : launch_trav_t<KT, double, false>(p, grid, block, smem, cluster, st);
    };
    err = launch();
    if (err == cudaErrorNotSupported && p.mode == TRAV_CLUSTER) {
      // clusters of this size cannot be co-resident at this shared-memory
      // footprint: fall back to per-chunk partials + combine
      cudaGetLastError();
      p.mode = TRAV_PARTIAL;
      cluster = 1;
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
