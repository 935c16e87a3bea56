// K4 traversal: host-side dispatch (trav_run) and finalize of caller-provided
// accumulators.  The kernel templates live in traverse.cuh and are
// instantiated in trav_inst_*.cu (compiled in parallel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "traverse.cuh"

namespace bridger {

#define BRIDGER_TRAV_EXTERN(ACC, ML, GT)                                                                           \
  extern template cudaError_t launch_trav_t<1, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<2, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<4, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<8, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_trav_t<16, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_trav_t<64, ACC, ML, GT>(const TravParams&, int, int, int, int, cudaStream_t);
BRIDGER_TRAV_EXTERN(long long, false, false)
BRIDGER_TRAV_EXTERN(long long, true, false)
BRIDGER_TRAV_EXTERN(double, false, false)
BRIDGER_TRAV_EXTERN(double, true, false)
BRIDGER_TRAV_EXTERN(long long, false, true)
BRIDGER_TRAV_EXTERN(long long, true, true)
BRIDGER_TRAV_EXTERN(double, false, true)
BRIDGER_TRAV_EXTERN(double, true, true)

// ------------------------------------------------------------- launchers ----
static int num_sms(int dev) {
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
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
  p.chunk_cap = L.global_trees ? 0 : (maxc + 127) / 128 * 128;
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
  const int NW = L.n_warps, G = L.group, NB = NW / G;
  const int block = NW * 32;
  p.group = G;
  p.red_off = p.chunk_cap + NB * 256 * m->F + trav_bar_bytes(NB);
  p.slot_off = p.red_off + trav_red_bytes(NB, G, m->K);
  int smem = p.slot_off;
  int cluster = 1;
  void* partial = nullptr;
  if (want == 3) {
    p.mode = TRAV_APPLY;
    p.out_leaf = static_cast<int32_t*>(out);
  } else if (n_chunks == 1 || L.global_trees) {
    p.mode = TRAV_FINAL;
  } else if (L.use_cluster && n_chunks <= 8 && smem + trav_slot_bytes(NB, n_chunks, m->K) <= 232448) {
    p.mode = TRAV_CLUSTER;
    cluster = n_chunks;
    smem += trav_slot_bytes(NB, n_chunks, m->K);
  } else {
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
  BRIDGER_DISPATCH_KT(m->K, {
    auto launch = [&]() {
      if (L.global_trees) {
        if (m->acc_int)
          return L.has_missing ? launch_trav_t<KT, long long, true, true>(p, grid, block, smem, cluster, st)
                               : launch_trav_t<KT, long long, false, true>(p, grid, block, smem, cluster, st);
        return L.has_missing ? launch_trav_t<KT, double, true, true>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, double, false, true>(p, grid, block, smem, cluster, st);
      }
      if (m->acc_int)
        return L.has_missing ? launch_trav_t<KT, long long, true, false>(p, grid, block, smem, cluster, st)
                             : launch_trav_t<KT, long long, false, false>(p, grid, block, smem, cluster, st);
      return L.has_missing ? launch_trav_t<KT, double, true, false>(p, grid, block, smem, cluster, st)
                           : launch_trav_t<KT, double, false, false>(p, grid, block, smem, cluster, st);
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
