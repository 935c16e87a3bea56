// K4 traversal: host-side dispatch (trav_run) and finalize of caller-provided
// accumulators.  The kernel templates live in traverse.cuh and are
// instantiated in trav_inst_*.cu (compiled in parallel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "traverse.cuh"
#include "ptx.cuh"

namespace bridger {

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
#define BRIDGER_STREAM_EXTERN_W(ACC, ML, W)                                                                         \
  extern template cudaError_t launch_stream_t<1, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<2, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<4, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<8, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t);  \
  extern template cudaError_t launch_stream_t<16, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_stream_t<64, ACC, ML, W, false>(const TravParams&, int, int, int, cudaStream_t); \
  extern template cudaError_t launch_stream_t<1, ACC, ML, W, true>(const TravParams&, int, int, int, cudaStream_t);
BRIDGER_STREAM_EXTERN_W(long long, false, 1)
BRIDGER_STREAM_EXTERN_W(long long, true, 1)
BRIDGER_STREAM_EXTERN_W(double, false, 1)
BRIDGER_STREAM_EXTERN_W(double, true, 1)
BRIDGER_STREAM_EXTERN_W(long long, false, 2)
BRIDGER_STREAM_EXTERN_W(long long, true, 2)
BRIDGER_STREAM_EXTERN_W(double, false, 2)
BRIDGER_STREAM_EXTERN_W(double, true, 2)
BRIDGER_TRAV_EXTERN(long long, false, true, 2)
BRIDGER_TRAV_EXTERN(long long, true, true, 2)
BRIDGER_TRAV_EXTERN(double, false, true, 2)
BRIDGER_TRAV_EXTERN(double, true, true, 2)

// Threshold-bin coding of the input (§8(f2)): X [N][F] fp32 row-major ->
// codes [n_blocks][F][32] u16, code = #{u in U_f : u < x} (binary search over
// the feature's sorted distinct thresholds, all in shared memory), NaN ->
// 0xFFFF.  The output is already in the traversal kernel's feature-major
// 32-row block layout, so the traversal bulk-copies it with no transpose.
__global__ void __launch_bounds__(512) bin_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                  const float* __restrict__ table, const int32_t* __restrict__ offs,
                                                  int32_t table_n, uint16_t* __restrict__ codes) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* U = reinterpret_cast<float*>(smem);
  int32_t* O = reinterpret_cast<int32_t*>(smem + (size_t)table_n * 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int S = F | 1;  // odd staging stride: St[lane*S + f] is bank-conflict free for a uniform f
  float* St = reinterpret_cast<float*>(smem + (size_t)table_n * 4 + (size_t)(F + 1) * 4) + (size_t)warp * 32 * S;
  for (int i = threadIdx.x; i < table_n; i += blockDim.x) U[i] = table[i];
  for (int i = threadIdx.x; i <= F; i += blockDim.x) O[i] = offs[i];
  __syncthreads();
  const int64_t n_blocks = (n_rows + 31) / 32;
  for (int64_t blk = (int64_t)blockIdx.x * NW + warp; blk < n_blocks; blk += (int64_t)gridDim.x * NW) {
    const int64_t row0 = blk * 32;
    const int rows = (int)(n_rows - row0 < 32 ? n_rows - row0 : 32);
    const float* src = X + row0 * F;
    // row-major copy into the odd-stride staging block: async 4-byte copies,
    // all in flight at once (zero-filled past the last row)
    for (int r = 0; r < 32; ++r)
      for (int f = lane; f < F; f += 32) {
        const uint32_t dsts = ptx::s2u(St + r * S + f);
        const float* g = src + (int64_t)(r < rows ? r : 0) * F + f;
        const uint32_t nbytes = r < rows ? 4u : 0u;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dsts), "l"(g), "r"(nbytes) : "memory");
      }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    uint16_t* dst = codes + blk * 32 * (int64_t)F;
    // lower_bound over the feature's sorted distinct thresholds; 4 features per
    // pass give 4 independent dependency chains per thread, and lane = row
    // with a warp-uniform feature makes the first search steps broadcasts
    for (int f0 = 0; f0 < F; f0 += 4) {
      float x[4];
      int lo[4], len[4], base[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = min(f0 + u, F - 1);
        x[u] = St[lane * S + f];
        base[u] = O[f];
        len[u] = O[f + 1] - base[u];
        lo[u] = 0;
      }
      bool any = true;
      while (any) {
        any = false;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (len[u] > 0) {
            const int half = len[u] >> 1;
            const bool less = U[base[u] + lo[u] + half] < x[u];
            lo[u] = less ? lo[u] + half + 1 : lo[u];
            len[u] = less ? len[u] - half - 1 : half;
            any = true;
          }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (f0 + u < F) dst[(f0 + u) * 32 + lane] = isnan(x[u]) ? (uint16_t)0xFFFF : (uint16_t)lo[u];
    }
    __syncwarp();
  }
}

// Pre-transposed input (FMT_HEAP_T): X [N][F] fp32 row-major -> [n_blocks][F][32]
// fp32, the traversal's feature-major 32-row block layout, written once so
// that every chunk CTA bulk-copies blocks with no per-chunk transpose.
__global__ void __launch_bounds__(512) xpose_kernel(const float* __restrict__ X, int64_t n_rows, int32_t F,
                                                    float* __restrict__ XT) {
  extern __shared__ __align__(16) uint8_t smem[];
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
    // tree-streamed mode: X transposed once into feature-major 32-row blocks,
    // then row tiles resident / chunk node records streamed (traverse.cuh K4s)
    const int64_t nbk = (n_rows + 31) / 32;
    void* xt = nullptr;
    cudaError_t err = cudaMallocAsync(&xt, (size_t)nbk * 32 * m->F * 4, st);
    if (err != cudaSuccess) return err;
    int nwx = 16;
    while (nwx > 1 && nwx * 32 * (m->F | 1) * 4 > 200 * 1024) --nwx;
    const int xsmem = nwx * 32 * (m->F | 1) * 4;
    static bool x_attr_s = false;
    if (!x_attr_s) {
      cudaFuncSetAttribute(xpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      x_attr_s = true;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xpose_kernel, nwx * 32, xsmem);
    const int xgrid = (int)std::max<int64_t>(1, std::min<int64_t>((nbk + nwx - 1) / nwx, (int64_t)sms * std::max(1, occ)));
    xpose_kernel<<<xgrid, nwx * 32, xsmem, st>>>(X, n_rows, m->F, static_cast<float*>(xt));
    count_launch();
    err = cudaGetLastError();
    if (err == cudaSuccess) {
      p.X = static_cast<const float*>(xt);
      p.mode = want == 3 ? TRAV_APPLY : TRAV_FINAL;
      p.out_leaf = static_cast<int32_t*>(out);
      p.stream_ns = L.stream_ns;
      p.stream_stage = L.stream_stage;
      const int rb = L.stream_warps * 32;
      p.stream_x_bytes = rb * m->F * 4;
      const int W = L.stream_w;
      p.stream_lbuf_bytes = (rb * W * m->K * 4 + 15) / 16 * 16;
      const int smem_s = p.stream_x_bytes + L.stream_ns * L.stream_stage + p.stream_lbuf_bytes + (1 + 2 * L.stream_ns) * 8 + 16;
      const int64_t n_tiles = (n_rows + rb - 1) / rb;
      const int grid_s = (int)std::max<int64_t>(1, std::min<int64_t>(n_tiles, sms));
      const int block_s = (L.stream_warps + 1) * 32;
      const bool w2 = W == 2;
      const bool ml = L.has_missing;
      if (want == 3) {
        err = ml ? (w2 ? launch_stream_t<1, long long, true, 2, true>(p, grid_s, block_s, smem_s, st)
                       : launch_stream_t<1, long long, true, 1, true>(p, grid_s, block_s, smem_s, st))
                 : (w2 ? launch_stream_t<1, long long, false, 2, true>(p, grid_s, block_s, smem_s, st)
                       : launch_stream_t<1, long long, false, 1, true>(p, grid_s, block_s, smem_s, st));
      } else {
#define BRIDGER_ST(ACC)                                                                      \
  (ml ? (w2 ? launch_stream_t<KT, ACC, true, 2, false>(p, grid_s, block_s, smem_s, st)      \
            : launch_stream_t<KT, ACC, true, 1, false>(p, grid_s, block_s, smem_s, st))     \
      : (w2 ? launch_stream_t<KT, ACC, false, 2, false>(p, grid_s, block_s, smem_s, st)     \
            : launch_stream_t<KT, ACC, false, 1, false>(p, grid_s, block_s, smem_s, st)))
        BRIDGER_DISPATCH_KT(m->K, { err = m->acc_int ? BRIDGER_ST(long long) : BRIDGER_ST(double); });
#undef BRIDGER_ST
      }
    }
    cudaFreeAsync(xt, st);
    return err;
  }
  const int NW = L.n_warps, G = L.group, NB = NW / G;
  const int block = NW * 32;
  p.group = G;
  const int xblk = L.codes ? 128 * m->F : 256 * m->F;
  p.red_off = p.chunk_cap + NB * xblk + trav_bar_bytes(NB);
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
  void* codes = nullptr;
  if (L.codes) {
    // step a1 in coded form: bin the rows once (all chunks reuse the codes)
    const int64_t nbk = (n_rows + 31) / 32;
    err = cudaMallocAsync(&codes, (size_t)nbk * 32 * m->F * 2, st);
    if (err != cudaSuccess) return err;
    const int table_n = (int)L.bin_table.size();
    const int fixed = table_n * 4 + (m->F + 1) * 4;
    int nwb = 16;
    while (nwb > 1 && fixed + nwb * 32 * (m->F | 1) * 4 > 232448) --nwb;
    const int bsmem = fixed + nwb * 32 * (m->F | 1) * 4;
    static bool bin_attr = false;
    if (!bin_attr) {
      cudaFuncSetAttribute(bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      bin_attr = true;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bin_kernel, nwb * 32, bsmem);
    const int64_t want_ctas = (nbk + nwb - 1) / nwb;
    const int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(want_ctas, (int64_t)sms * std::max(1, occ)));
    bin_kernel<<<bgrid, nwb * 32, bsmem, st>>>(X, n_rows, m->F, m->d_bin_table, m->d_bin_offsets, table_n,
                                                 static_cast<uint16_t*>(codes));
    count_launch();
    err = cudaGetLastError();
    if (err != cudaSuccess) {
      cudaFreeAsync(codes, st);
      return err;
    }
    p.X = static_cast<const float*>(codes);
  } else if (L.hybrid || (L.pretransposed && want != 3)) {
    const int64_t nbk = (n_rows + 31) / 32;
    err = cudaMallocAsync(&codes, (size_t)nbk * 32 * m->F * 4, st);
    if (err != cudaSuccess) return err;
    int nwx = 16;
    while (nwx > 1 && nwx * 32 * (m->F | 1) * 4 > 200 * 1024) --nwx;
    const int xsmem = nwx * 32 * (m->F | 1) * 4;
    static bool x_attr = false;
    if (!x_attr) {
      cudaFuncSetAttribute(xpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      x_attr = true;
    }
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
