// GEMM form of steps a1..a4 -- the tensor-operator lowering
// of a tree (COR) that the paper's framework generates: an exact
// feature gather, a threshold compare, the path-matrix contraction (matmul,
// PAPER.md:588) and the leaf-count compare (equal), then the
// leaf-value gather and the per-tree reduction.
//
//   K1 gc_kernel  a1+a2  P[t][r][i] = [X[r, A_t[i]] <= B_t[i]]  (exact fp32 gather,
//                        never a one-hot GEMM; NaN -> missing_left)   int8 0/1
//   K2 pc_kernel  a3+a4  S = P . C_D on tcgen05 (kind::i8, M=128, N=L_pad,
//                        K=32 per instruction), accumulator in TMEM; the
//                        epilogue tcgen05.ld's each row and keeps the unique l
//                        with S[l] == D_D[l]                            int16 leaf
//   K3 lg_kernel  a5+a6+a7  acc += E_t[leaf] (int64 fixed point), finalize
//
// C_D is universal per depth (host lowering); P tiles are written by K1
// directly in the UMMA canonical K-major "interleaved" layout
// [k-chunk of 16 B][128 rows][16 B], so K2 stages each (tree, 128-row tile)
// operand with ONE bulk copy (TMA engine) and describes it with LBO = 2048 B
// (next 16-byte K chunk), SBO = 128 B (next 8-row core matrix).  Rows are
// processed in blocks so the decision scratch stays bounded.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "bridger_internal.h"
#include "finalize.cuh"
#include "ptx.cuh"

namespace bridger {

void count_launch();
void hot_begin(cudaStream_t st, cudaEvent_t* ev);
void hot_end(cudaStream_t st, cudaEvent_t start);
void hot_end_id(cudaStream_t st, cudaEvent_t start, int id);

struct GemmClassDev {
  int32_t depth, i_pad, l_pad, n_trees;
  int64_t feat_off;   // int32 [n][i_pad]  feature | missing_left << 31
  int64_t thr_off;    // float [n][i_pad]
  int64_t cmat_off;   // int8  [i_pad/16][l_pad][16]  C_D in canonical K-major layout
  int64_t dv_off;     // int32 [l_pad]  D_D (127 for padding columns: never matches)
  int64_t leaf_off;   // float [n][L][K]  leaf values (fixed-point scaled when exact)
  int32_t first_slot; // index of the class's first tree in slot order
  int32_t pad_;
  int64_t node_off;   // uint2 [n][i_pad] {feature | missing<<31, threshold} (K5; row I = constant-1 node)
  int64_t cmat2_off;  // int8 C'_D canonical K-major: C_D plus row I = popc(l) (K5, a4 folded in)
  // 2:4-sparse form (K2s): K regrouped by level (sparse_pos), k_sp = round_up(2^D, 64),
  // m_sp = round_up(2^D, 128) leaves as the MMA's M (the A operand is C_sp^T)
  int32_t k_sp, m_sp;
  int64_t feat_sp_off;  // int32 [n][k_sp]  nodes at sparse_pos(i), dummies elsewhere
  int64_t thr_sp_off;   // float [n][k_sp]
  int64_t asp_off;      // int8  [m_sp/128][k_sp/64][2][128][16]  compressed C_sp^T (2 of every 4 K values)
  int64_t meta_off;     // u32   [m_sp/128][128][k_sp/64][2]     2:4 metadata per leaf row (TMEM layout)
};

struct GemmHost {
  std::vector<GemmClassDev> classes;
  std::vector<int32_t> slot_tree;      // slot -> original tree
  std::vector<int32_t> tree_slot;      // original tree -> slot
  std::vector<int32_t> tree_class;     // original tree -> class index
  int64_t max_p_per_row = 0;           // max over classes of n_trees * i_pad
  int64_t max_psp_per_row = 0;         // ... of n_trees * k_sp (sparse form)
  int32_t max_trees = 0;
  bool has_missing = false;            // any real node with missing_left (K5 ML instantiation)
};

static constexpr int kSmemMax = 232448;

// ------------------------------------------------------------------ K1 -----
// grid (row tiles of the block, tree groups), 128 threads = 128 rows.
// out layout TILED: P[t][rt][kc][128][16]; PLAIN: P[t][row][i_pad].
// ML: the model has missing_left nodes (else the NaN test per decision is
// compiled out: NaN compares false -> 0 -> right, reading c2).
template <bool PLAIN, bool ML>
__global__ void __launch_bounds__(128) gc_kernel(const float* __restrict__ X, int64_t row0, int32_t rows, int32_t F,
                                                 const uint8_t* __restrict__ gbase, GemmClassDev cls,
                                                 int32_t tree_begin, int32_t trees_per_cta, int32_t tree_end,
                                                 int8_t* __restrict__ P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int r = threadIdx.x;
  const int rt = blockIdx.x;
  const int n_rt = gridDim.x;
  const int ip = cls.i_pad;
  const int S = 129;  // padded feature-major X tile: bank (f*129 + r) % 32 = (f + r) % 32
  // [2][ip] {feature | missing<<31, threshold} node records of the current tree
  // (double buffered: one __syncthreads per tree), then the X tile
  uint2* nd = reinterpret_cast<uint2*>(smem);
  float* Xs = reinterpret_cast<float*>(smem + (size_t)2 * ip * 8);
  // coalesced load of the 128-row tile, transposed into Xs[f][r]
  const int64_t tile_row0 = row0 + (int64_t)rt * 128;
  const int tile_rows = max(0, min(128, (int)(row0 + rows - tile_row0)));
  const float* src = X + tile_row0 * F;
  for (int e = r; e < 128 * F; e += 128) {
    const int rr = e / F, f = e - rr * F;
    Xs[f * S + rr] = rr < tile_rows ? src[e] : 0.0f;
  }
  const int32_t* feat = reinterpret_cast<const int32_t*>(gbase + cls.feat_off);
  const float* thr = reinterpret_cast<const float*>(gbase + cls.thr_off);
  const int t_lo = tree_begin + blockIdx.y * trees_per_cta;
  const int t_hi = min(tree_end, t_lo + trees_per_cta);
  const float* xr = Xs + r;
  for (int t = t_lo, buf = 0; t < t_hi; ++t, buf ^= 1) {
    uint2* ndb = nd + buf * ip;
    for (int i = r; i < ip; i += 128)
      ndb[i] = make_uint2((uint32_t)feat[(size_t)t * ip + i], __float_as_uint(thr[(size_t)t * ip + i]));
    __syncthreads();  // node records (and, first time, the X tile) visible
    const int64_t t_local = t - tree_begin;
    for (int kc = 0; kc < ip / 16; ++kc) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; b += 2) {
          // two node records per broadcast read (16 B)
          const uint4 n2 = *reinterpret_cast<const uint4*>(&ndb[kc * 16 + q * 4 + b]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t nf = h ? n2.z : n2.x, nt = h ? n2.w : n2.y;
            const float x = xr[(ML ? (nf & 0x7fffffffu) : nf) * S];  // exact fp32 gather (a1)
            uint32_t d = (x <= __uint_as_float(nt)) ? 1u : 0u;      // a2: less_equal
            if (ML && (int32_t)nf < 0 && isnan(x)) d = 1u;          // missing_left
            word |= d << (8 * (b + h));
          }
        }
        w[q] = word;
      }
      if (PLAIN) {
        const int64_t row = (int64_t)rt * 128 + r;
        if (r < tile_rows)
          *reinterpret_cast<uint4*>(P + (t_local * rows + row) * ip + kc * 16) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        int8_t* dst = P + ((t_local * n_rt + rt) * (int64_t)ip * 128) + (int64_t)kc * 2048 + r * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

// plain [rows][i_pad] -> tiled [rt][kc][128][16] (step-level test entry only)
__global__ void tile_kernel(const int8_t* __restrict__ in, int64_t rows, int32_t ip, int8_t* __restrict__ out) {
  const int64_t n16 = (rows + 127) / 128 * 128 * (ip / 16);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n16; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / (ip / 16);
    const int kc = (int)(e % (ip / 16));
    const int64_t rt = row / 128;
    const int r = (int)(row % 128);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < rows) v = *reinterpret_cast<const uint4*>(in + row * ip + kc * 16);
    *reinterpret_cast<uint4*>(out + rt * 128 * ip + (int64_t)kc * 2048 + r * 16) = v;
  }
}

// ------------------------------------------------------------------ K2 -----
namespace umma {
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // sm_100 shared-memory matrix descriptor, SWIZZLE_NONE, K-major canonical layout
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout type 0 (no swizzle)
}
// kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(ptx::s2u(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
}  // namespace umma

struct PcParams {
  const int8_t* P;       // tiled decisions [n_trees][n_rt][i_pad/16][128][16]
  const uint8_t* gbase;  // class data (C_D tile, D_D)
  GemmClassDev cls;
  int32_t n_trees;       // trees in this launch (class-local, starting at 0 of P)
  int32_t n_rt;          // 128-row tiles
  int32_t rows;          // valid rows of the block
  int32_t tmem_cols;     // allocated columns (power of 2): 2 accumulator stages
  int32_t b_bytes;       // i_pad * l_pad
  int32_t stages;        // depth of the A-operand ring
  int32_t mode;          // 0: int16 leaf index, 1: int32 S rows
  int16_t* leaf;         // [n_trees][rows]
  int32_t* S;            // [n_trees][rows][l_pad]
};

// Warp-specialised tcgen05 pipeline (18 warps):
//   warps 0-15 epilogue: warp w reads TMEM lanes 32(w%4)..+31 (= rows of the
//              tile) and column quarter w/4 with tcgen05.ld, a4 leaf-count
//              compare; the leaf is unique, so exactly one quarter writes it;
//              then release the TMEM stage (4 warps per SMSP hide the LDTM and
//              compare latencies: measured 4x faster than 1 warp per SMSP)
//   warp 16    producer: bulk copies (TMA engine) of C_D once and of each
//              (tree, 128-row) decision tile into a `stages`-deep ring
//   warp 17    MMA issuer: one thread issues I_pad/32 tcgen05.mma kind::i8 per
//              tile into one of two TMEM accumulators; tcgen05.commit frees the
//              A stage and signals the epilogue
constexpr int kPcEpiWarps = 16;
constexpr int kPcThreads = (kPcEpiWarps + 2) * 32;

__global__ void __launch_bounds__(kPcThreads, 1) pc_kernel(const PcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ip = p.cls.i_pad, lp = p.cls.l_pad, D = p.cls.depth;
  const int NS = p.stages;
  const uint32_t a_bytes = 128u * (uint32_t)ip;
  uint8_t* sB = smem;
  uint8_t* sA = smem + ((p.b_bytes + 1023) / 1024) * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + (size_t)NS * a_bytes);
  uint64_t* bfull = bars;               // [1]
  uint64_t* afull = bars + 1;           // [NS]
  uint64_t* aempty = bars + 1 + NS;     // [NS]
  uint64_t* tfull = bars + 1 + 2 * NS;  // [2]
  uint64_t* tempty = bars + 3 + 2 * NS; // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 5 + 2 * NS);

  if (tid == 0) {
    ptx::mbar_init(bfull, 1);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kPcEpiWarps * 32);
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (warp == kPcEpiWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::s2u(tmem_holder)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_holder;
  const int n_items = p.n_trees * p.n_rt;
  const int grid = gridDim.x;

  if (warp == kPcEpiWarps) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bfull, (uint32_t)p.b_bytes);
      for (int o = 0; o < p.b_bytes; o += 32768)
        ptx::bulk_g2s(sB + o, p.gbase + p.cls.cmat_off + o, (uint32_t)min(32768, p.b_bytes - o), bfull);
      int k = 0;
      for (int item = blockIdx.x; item < n_items; item += grid, ++k) {
        const int s = k % NS;
        ptx::mbar_wait(&aempty[s], ((k / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&afull[s], a_bytes);
        ptx::bulk_g2s(sA + (size_t)s * a_bytes, p.P + (size_t)item * a_bytes, a_bytes, &afull[s]);
      }
    }
  } else if (warp == kPcEpiWarps + 1) {
    if (lane == 0) {
      ptx::mbar_wait(bfull, 0);
      const uint32_t idesc = umma::idesc_i8(lp);
      const uint32_t sA_u = ptx::s2u(sA), sB_u = ptx::s2u(sB);
      int k = 0;
      for (int item = blockIdx.x; item < n_items; item += grid, ++k) {
        const int s = k % NS, acc = k & 1;
        ptx::mbar_wait(&tempty[acc], ((k >> 1) & 1) ^ 1);   // epilogue drained this accumulator
        ptx::mbar_wait(&afull[s], (k / NS) & 1);             // decision tile landed
        umma::fence_after();
        const uint32_t a0 = sA_u + (uint32_t)s * a_bytes;
        for (int ks = 0; ks < ip / 32; ++ks) {
          const uint64_t ad = umma::smem_desc(a0 + (uint32_t)ks * 2u * 2048u, 2048u, 128u);
          const uint64_t bd = umma::smem_desc(sB_u + (uint32_t)ks * 2u * (uint32_t)lp * 16u, (uint32_t)lp * 16u, 128u);
          umma::mma_i8(tmem + (uint32_t)(acc * lp), ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
        umma::commit(&aempty[s]);   // A stage free once these MMAs have read it
        umma::commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // epilogue warps: thread = row of the tile (TMEM lane), a quarter of the columns
    const int quad = warp & 3, part = warp >> 2;
    const int n_parts = lp >= 64 ? 4 : lp / 16;      // 16-column tcgen05.ld granularity
    const int cols = lp / n_parts;
    const bool active = part < n_parts;
    int k = 0;
    for (int item = blockIdx.x; item < n_items; item += grid, ++k) {
      const int acc = k & 1;
      ptx::mbar_wait(&tfull[acc], (k >> 1) & 1);
      umma::fence_after();
      const int t = item / p.n_rt, rt = item % p.n_rt;
      const int row = rt * 128 + quad * 32 + lane;
      const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * lp);
      int leaf = -1;
      const int L = 1 << D;
      if (active) {
        for (int cb = part * cols; cb < (part + 1) * cols; cb += 16) {
          uint32_t v[16];
          umma::ld16(tbase + cb, v);
          umma::wait_ld();
          if (p.mode == 0) {
            // a4: D_D[l] = D - popc(l); popc(cb + j) = popc(cb) + popc(j) for j < 16
            const int base = D - __popc(cb);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if ((int32_t)v[j] + __popc(j) == base && cb + j < L) leaf = cb + j;
          } else if (row < p.rows) {
            int4* o = reinterpret_cast<int4*>(p.S + ((size_t)t * p.rows + row) * lp + cb);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              o[j] = make_int4((int)v[4 * j], (int)v[4 * j + 1], (int)v[4 * j + 2], (int)v[4 * j + 3]);
          }
        }
      }
      umma::fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      if (p.mode == 0 && leaf >= 0 && row < p.rows) p.leaf[(size_t)t * p.rows + row] = (int16_t)leaf;
    }
  }
  __syncthreads();
  umma::fence_after();
  if (warp == kPcEpiWarps)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

// ----------------------------------------------------------------- K2s -----
// 2:4-sparse path contraction ("sparse operator replacing", PAPER.md:502,
// Table 2).  The transposed product
//     S^T[l][r] = sum_k C_sp^T[l][k] P[r][k]
// puts the constant path matrix on the SPARSE operand: A = C_sp^T (M = leaves,
// K = internal nodes regrouped by level so every group of 4 consecutive K
// positions holds <= 2 ancestors of a leaf, bridger_path_matrix_sparse),
// stored compressed (2 of every 4 K values, 32 B per row per 64-K step) in
// shared memory once per CTA, its 2:4 metadata written once into TMEM (lane =
// leaf, 2 columns per 64-K step; nibble g = positions p0 | p1 << 2 of group g,
// pinned on B200 by tools/sparse_probe.cu); B = the decision tile P (N = 128
// rows, K-major canonical, the same tiles K1 writes).  tcgen05.mma.sp
// .cta_group::1.kind::i8 (M = 128, N = 128, K = 64): half the MACs of the
// dense K2 per logical product.  Warp roles as in pc_kernel:
//   warps 0-15 epilogue: thread = leaf (TMEM lane), a quarter of the tile's 128
//              row columns: tcgen05.ld 2 x 16 columns, a4 (S == D_D[leaf]) ->
//              this leaf is that row's leaf (unique), store it
//   warp 16    producer: compressed A + metadata once, then decision tiles
//   warp 17    MMA issuer: per (tile, M-tile) item k_sp/64 sparse MMAs into
//              one of kSpSlots 128-column TMEM accumulators
constexpr int kSpSlots = 3;
struct PcsParams {
  const int8_t* P;       // tiled decisions [n_trees][n_rt][k_sp/16][128][16]
  const uint8_t* gbase;
  GemmClassDev cls;
  int32_t n_trees, n_rt, rows;
  int32_t stages;        // B (decision tile) ring depth
  int32_t mode;          // 0: int16 leaf index, 1: int32 S rows [n_trees][rows][l_pad]
  int16_t* leaf;
  int32_t* S;
};

__device__ __forceinline__ void mma_sp_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                          uint32_t idesc, uint32_t acc) {
  const uint32_t z = 0u;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %5, {%6, %6, %6, %6}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(acc), "r"(idesc), "r"(z)
      : "memory");
}

__global__ void __launch_bounds__(kPcThreads, 1) pcs_kernel(const PcsParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = p.cls.depth, L = 1 << D, lp = p.cls.l_pad;
  const int ks_n = p.cls.k_sp / 64, mt_n = p.cls.m_sp / 128;
  const int NS = p.stages;
  const uint32_t a_bytes = (uint32_t)mt_n * ks_n * 4096u;  // compressed C_sp^T
  const uint32_t b_bytes = 128u * (uint32_t)p.cls.k_sp;    // one decision tile
  uint8_t* sA = smem;
  uint8_t* sB = smem + ((a_bytes + 1023) / 1024) * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)NS * b_bytes);
  uint64_t* afull = bars;                      // [1]
  uint64_t* bfull = bars + 1;                  // [NS]
  uint64_t* bempty = bars + 1 + NS;            // [NS]
  uint64_t* tfull = bars + 1 + 2 * NS;         // [kSpSlots]
  uint64_t* tempty = tfull + kSpSlots;         // [kSpSlots]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + kSpSlots);
  constexpr uint32_t kMetaCol = kSpSlots * 128;  // metadata after the accumulator slots

  if (tid == 0) {
    ptx::mbar_init(afull, 1);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < kSpSlots; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kPcEpiWarps * 32);
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (warp == kPcEpiWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::s2u(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_holder;
  // 2:4 metadata of every (M-tile, K-step) into TMEM: warp quadrant q writes lanes 32q..32q+31
  if (warp < 4) {
    const uint32_t* meta = reinterpret_cast<const uint32_t*>(p.gbase + p.cls.meta_off);
    for (int mt = 0; mt < mt_n; ++mt)
      for (int ks = 0; ks < ks_n; ++ks) {
        const int r = warp * 32 + lane;
        const uint32_t w0 = meta[((size_t)(mt * 128 + r) * ks_n + ks) * 2 + 0];
        const uint32_t w1 = meta[((size_t)(mt * 128 + r) * ks_n + ks) * 2 + 1];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + kMetaCol + (uint32_t)(mt * ks_n + ks) * 4u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(w0), "r"(w1)
                     : "memory");
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const int n_tiles = p.n_trees * p.n_rt;
  const int grid = gridDim.x;

  if (warp == kPcEpiWarps) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(afull, a_bytes);
      for (uint32_t o = 0; o < a_bytes; o += 32768u)
        ptx::bulk_g2s(sA + o, p.gbase + p.cls.asp_off + o, min(32768u, a_bytes - o), afull);
      int k = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += grid, ++k) {
        const int s = k % NS;
        ptx::mbar_wait(&bempty[s], ((k / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bfull[s], b_bytes);
        ptx::bulk_g2s(sB + (size_t)s * b_bytes, p.P + (size_t)tile * b_bytes, b_bytes, &bfull[s]);
      }
    }
  } else if (warp == kPcEpiWarps + 1) {
    if (lane == 0) {
      ptx::mbar_wait(afull, 0);
      // idesc: sparse (bit 2), D s32, A s8, B s8, K-major both, N = 128, M = 128
      const uint32_t idesc = (1u << 2) | (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t sA_u = ptx::s2u(sA), sB_u = ptx::s2u(sB);
      int k = 0, item = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += grid, ++k) {
        const int s = k % NS;
        ptx::mbar_wait(&bfull[s], (k / NS) & 1);
        const uint32_t b0 = sB_u + (uint32_t)s * b_bytes;
        for (int mt = 0; mt < mt_n; ++mt, ++item) {
          const int slot = item % kSpSlots;
          ptx::mbar_wait(&tempty[slot], ((item / kSpSlots) & 1) ^ 1);  // epilogue drained the slot
          umma::fence_after();
          for (int ks = 0; ks < ks_n; ++ks) {
            const uint64_t ad = umma::smem_desc(sA_u + (uint32_t)(mt * ks_n + ks) * 4096u, 2048u, 128u);
            const uint64_t bd = umma::smem_desc(b0 + (uint32_t)ks * 4u * 2048u, 2048u, 128u);
            mma_sp_i8(tmem + (uint32_t)slot * 128u, ad, bd, tmem + kMetaCol + (uint32_t)(mt * ks_n + ks) * 4u, idesc,
                      ks > 0 ? 1u : 0u);
          }
          umma::commit(&tfull[slot]);
        }
        umma::commit(&bempty[s]);  // decision tile free once every M-tile's MMAs have read it
      }
    }
  } else {
    // epilogue: thread = leaf (TMEM lane) of the M-tile, 32 of the tile's 128 row columns
    const int quad = warp & 3, part = warp >> 2;
    const int32_t* dv = reinterpret_cast<const int32_t*>(p.gbase + p.cls.dv_off);
    int32_t want_mt[2];  // D_D of this thread's leaf in each M-tile (padding leaves never match)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int l = mt * 128 + quad * 32 + lane;
      want_mt[mt] = (mt < mt_n && l < L) ? dv[l] : 0x7fffffff;
    }
    int item = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += grid) {
      const int t = tile / p.n_rt, rt = tile % p.n_rt;
      for (int mt = 0; mt < mt_n; ++mt, ++item) {
        const int slot = item % kSpSlots;
        ptx::mbar_wait(&tfull[slot], (item / kSpSlots) & 1);
        umma::fence_after();
        const int l = mt * 128 + quad * 32 + lane;
        const int32_t want = mt ? want_mt[1] : want_mt[0];
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)slot * 128u + (uint32_t)(part * 32);
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tbase));
        umma::wait_ld();
        umma::fence_before();
        ptx::mbar_arrive(&tempty[slot]);
        const int row0 = rt * 128 + part * 32;
        if (p.mode == 0) {
          // a4: S <= D_D[l] with equality iff the row reaches leaf l, so with
          // w1 = D_D - 1, max(S, w1) = w1 + hit bit and (mod 2^32)
          //   sum_j max(S_j, w1) << j = hit - w1
          // -- two instructions per value (VIMNMX + IMAD); a few of the 32
          // rows reach this leaf: store those
          const int32_t w1 = want - 1;
          uint32_t hit = (uint32_t)w1;
#pragma unroll
          for (int j = 0; j < 32; ++j) hit += (uint32_t)max((int32_t)v[j], w1) << j;
          while (hit) {
            const int j = __ffs(hit) - 1;
            hit &= hit - 1;
            if (row0 + j < p.rows) p.leaf[(size_t)t * p.rows + row0 + j] = (int16_t)l;
          }
        } else if (l < lp) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (row0 + j < p.rows) p.S[((size_t)t * p.rows + row0 + j) * lp + l] = (int32_t)v[j];
        }
      }
    }
  }
  __syncthreads();
  umma::fence_after();
  if (warp == kPcEpiWarps)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ K3 -----
template <int KT, typename ACC>
__global__ void __launch_bounds__(256) lg_kernel(const int16_t* __restrict__ leaf, int32_t rows, int32_t n_trees,
                                                 const float* __restrict__ E, int32_t L, int32_t K,
                                                 ACC* __restrict__ accbuf, int32_t first, int32_t last,
                                                 int64_t row0, FinalizeArgs fin) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  ACC acc[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) acc[k] = (first || k >= K) ? ACC(0) : accbuf[(size_t)r * K + k];
#pragma unroll 4
  for (int t = 0; t < n_trees; ++t) {
    const int l = leaf[(size_t)t * rows + r];
    const float* e = E + ((size_t)t * L + l) * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) {
        const float v = __ldg(e + k);
        if (std::is_same<ACC, long long>::value) acc[k] += (ACC)__float2ll_rz(v);
        else acc[k] += (ACC)v;
      }
  }
  if (last) {
    finalize_row<KT, ACC>(fin, row0 + r, acc);
  } else {
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) accbuf[(size_t)r * K + k] = acc[k];
  }
}

// ------------------------------------------------------------------ K5 -----
// Fused, warp-specialised GEMM form: a1..a7 in ONE kernel,
// decisions never leave shared memory.  Persistent CTAs own 128-row tiles; per
// tile every tree of the depth class is one pipeline item:
//   producer warps (kFzProd) a1+a2: the X tile sits feature-major in SMEM
//        (stride 129: conflict-free transpose stores AND gathers); a warp keeps
//        16 node records of one K chunk in registers and writes the packed
//        decisions of 32 rows straight into the UMMA canonical K-major A stage
//   loader warp   C'_D once, then each tree's node records into a small ring
//                 (bulk copies, TMA engine)
//   MMA warp      a3: I_pad/32 tcgen05.mma kind::i8 per item into one of two
//                 TMEM accumulators (as K2)
//   epilogue warps (kFzEpi) a4..a7: tcgen05.ld, leaf select, leaf-value gather
//        and int64 accumulation in registers across the tile's trees; at the
//        tile's last tree the column parts are summed in SMEM and finalized.
// a4 is folded into the contraction: the padding K row I (always present,
// since 2^D - 1 is odd and I_pad a multiple of 32) carries a constant decision
// 1 (feature F = a constant-zero row of the X tile, threshold +inf) and C'_D[I][l] = popc(l) (-64 for padding
// columns), so S'[l] = S[l] + popc(l) = D exactly at the reached leaf
// (D_D[l] = D - popc(l), reading c14) and < D everywhere else.
constexpr int kFzProd = 8;
constexpr int kFzEpi = 8;
constexpr int kFzThreads = (kFzProd + kFzEpi + 2) * 32;
constexpr int kFzNodeMax = 32;  // node-record ring depth cap (sized by bytes in fz_plan)
constexpr int kFzXStride = 129;

struct FzParams {
  const float* X;
  int64_t n_rows;
  int32_t F, K, L;
  int32_t n_tiles;
  const uint8_t* gbase;
  GemmClassDev cls;
  int32_t stages;     // A ring depth
  int32_t nstages;    // node-record ring depth
  int32_t tstages;    // TMEM accumulator ring depth
  int32_t tmem_cols;
  int32_t b_bytes;
  int32_t x_off, a_off, n_off, red_off, bar_off, smem;  // shared-memory carve-up (fz_plan)
  int32_t first, last;  // depth-class position (accbuf in/out)
  void* accbuf;         // [n_rows][K] ACC, when the model has several depth classes
  FinalizeArgs fin;
};

template <int KT, typename ACC, bool ML>
__global__ void __launch_bounds__(kFzThreads, 1) fz_kernel(const FzParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ip = p.cls.i_pad, lp = p.cls.l_pad, D = p.cls.depth, nt = p.cls.n_trees;
  const int NS = p.stages, F = p.F;
  const uint32_t a_bytes = 128u * (uint32_t)ip;
  uint8_t* sB = smem;
  float* Xs = reinterpret_cast<float*>(smem + p.x_off);
  uint8_t* sA = smem + p.a_off;
  uint2* sN = reinterpret_cast<uint2*>(smem + p.n_off);  // [nstages][ip]
  const int NN = p.nstages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* bfull = bars;                      // [1]
  uint64_t* afull = bars + 1;                  // [NS]
  uint64_t* aempty = afull + NS;               // [NS]
  const int NT = p.tstages;
  uint64_t* tfull = aempty + NS;               // [NT]
  uint64_t* tempty = tfull + NT;               // [NT]
  uint64_t* nfull = tempty + NT;               // [NN]
  uint64_t* nempty = nfull + NN;               // [NN]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(nempty + NN);
  constexpr int kLoader = kFzProd, kMma = kFzProd + 1, kEpi0 = kFzProd + 2;

  if (tid == 0) {
    ptx::mbar_init(bfull, 1);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&afull[i], kFzProd * 32);
      ptx::mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < NT; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kFzEpi * 32);
    }
    for (int i = 0; i < NN; ++i) {
      ptx::mbar_init(&nfull[i], 1);
      ptx::mbar_init(&nempty[i], kFzProd);
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (warp == kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::s2u(tmem_holder)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_holder;
  const int grid = gridDim.x;
  const int my_tiles = p.n_tiles > (int)blockIdx.x ? (p.n_tiles - 1 - (int)blockIdx.x) / grid + 1 : 0;
  const int n_items = my_tiles * nt;

  if (warp < kFzProd) {
    // ---------------------------------------------------------- producers --
    const int n_kc = ip / 16;
    const int n_pairs = n_kc * 4;  // (K chunk, 32-row group)
    const int per = (n_pairs + kFzProd - 1) / kFzProd;
    const int p_lo = warp * per, p_hi = min(n_pairs, p_lo + per);
    int k = 0;
    for (int ti = 0; ti < my_tiles; ++ti) {
      const int64_t tile_row0 = (int64_t)(blockIdx.x + ti * grid) * 128;
      const int tile_rows = (int)(p.n_rows - tile_row0 < 128 ? p.n_rows - tile_row0 : 128);
      // the previous tile's decisions are all written: reload the X tile
      asm volatile("bar.sync 1, %0;" ::"r"(kFzProd * 32) : "memory");
      if (ti == 0)
        for (int e = tid; e < 128; e += kFzProd * 32) Xs[F * kFzXStride + e] = 0.0f;  // row F: constant node
      const float* src = p.X + tile_row0 * F;
      if (tile_rows == 128) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        for (int e4 = tid; e4 < 32 * F; e4 += kFzProd * 32) {
          const float4 v = __ldg(s4 + e4);
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = 4 * e4 + q, rr = e / F, f = e - rr * F;
            Xs[f * kFzXStride + rr] = vv[q];
          }
        }
      } else {
        for (int e = tid; e < 128 * F; e += kFzProd * 32) {
          const int rr = e / F, f = e - rr * F;
          Xs[f * kFzXStride + rr] = rr < tile_rows ? __ldg(src + e) : 0.0f;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kFzProd * 32) : "memory");
      for (int t = 0; t < nt; ++t, ++k) {
        const int s = k % NS, ns = k % NN;
        ptx::mbar_wait(&nfull[ns], (k / NN) & 1);              // node records of tree t
        ptx::mbar_wait(&aempty[s], ((k / NS) & 1) ^ 1);        // A stage free
        const uint2* nd = sN + (size_t)ns * ip;
        uint8_t* a = sA + (size_t)s * a_bytes;
        // this warp's pairs are consecutive: runs of row groups [rg0, rg1) of one K chunk
        for (int pr = p_lo; pr < p_hi;) {
          const int kc = pr >> 2, rg0 = pr & 3;
          const int rg1 = min(4, rg0 + (p_hi - pr));
          pr += rg1 - rg0;
          // 16 node records (broadcast loads) -> per-node shared address of this
          // lane's x in row group rg0; the other row groups are +128 B immediates
          uint32_t xa[16];
          float th[16];
          uint32_t mlm = 0;  // missing-left nodes (bit b)
          const uint4* n4 = reinterpret_cast<const uint4*>(nd + kc * 16);
          const uint32_t xbase = ptx::s2u(Xs) + (uint32_t)(rg0 * 32 + lane) * 4u;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const uint4 v = n4[b];
            xa[2 * b] = xbase + (v.x & 0x7fffffffu) * (uint32_t)(kFzXStride * 4);
            xa[2 * b + 1] = xbase + (v.z & 0x7fffffffu) * (uint32_t)(kFzXStride * 4);
            th[2 * b] = __uint_as_float(v.y);
            th[2 * b + 1] = __uint_as_float(v.w);
            if (ML) mlm |= (v.x >> 31) << (2 * b) | (v.z >> 31) << (2 * b + 1);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (j < rg1 - rg0) {
              uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int b = 0; b < 16; ++b) {
                float x;  // a1: exact fp32 gather (feature-major tile, conflict-free)
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(xa[b] + (uint32_t)(j * 128)));
                uint32_t msk;  // a2: less_equal as an all-ones mask (NaN -> 0, goes right)
                asm("set.le.u32.f32 %0, %1, %2;" : "=r"(msk) : "f"(x), "f"(th[b]));
                if (ML) {  // missing-left node: unordered (NaN) compares true
                  uint32_t mu;
                  asm("set.leu.u32.f32 %0, %1, %2;" : "=r"(mu) : "f"(x), "f"(th[b]));
                  msk |= mu & (0u - ((mlm >> b) & 1u));
                }
                w[b >> 2] |= msk & (1u << (8 * (b & 3)));
              }
              *reinterpret_cast<uint4*>(a + (size_t)kc * 2048 + ((rg0 + j) * 32 + lane) * 16) =
                  make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&nempty[ns]);
        ptx::fence_proxy_async();  // generic-proxy stores -> tensor-core (async proxy) reads
        ptx::mbar_arrive(&afull[s]);
      }
    }
  } else if (warp == kLoader) {
    // -------------------------------------------------- bulk-copy loader --
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bfull, (uint32_t)p.b_bytes);
      for (int o = 0; o < p.b_bytes; o += 32768)
        ptx::bulk_g2s(sB + o, p.gbase + p.cls.cmat2_off + o, (uint32_t)min(32768, p.b_bytes - o), bfull);
      const uint8_t* nodes = p.gbase + p.cls.node_off;
      const uint32_t nb = 8u * (uint32_t)ip;
      for (int k = 0; k < n_items; ++k) {
        const int ns = k % NN, t = k % nt;
        ptx::mbar_wait(&nempty[ns], ((k / NN) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&nfull[ns], nb);
        ptx::bulk_g2s(sN + (size_t)ns * ip, nodes + (size_t)t * nb, nb, &nfull[ns]);
      }
    }
  } else if (warp == kMma) {
    // ---------------------------------------------------------- MMA issue --
    if (lane == 0) {
      ptx::mbar_wait(bfull, 0);
      const uint32_t idesc = umma::idesc_i8(lp);
      const uint32_t sA_u = ptx::s2u(sA), sB_u = ptx::s2u(sB);
      for (int k = 0; k < n_items; ++k) {
        const int s = k % NS, acc = k % NT;
        ptx::mbar_wait(&tempty[acc], ((k / NT) & 1) ^ 1);
        ptx::mbar_wait(&afull[s], (k / NS) & 1);
        umma::fence_after();
        const uint32_t a0 = sA_u + (uint32_t)s * a_bytes;
        for (int ks = 0; ks < ip / 32; ++ks) {
          const uint64_t ad = umma::smem_desc(a0 + (uint32_t)ks * 2u * 2048u, 2048u, 128u);
          const uint64_t bd = umma::smem_desc(sB_u + (uint32_t)ks * 2u * (uint32_t)lp * 16u, (uint32_t)lp * 16u, 128u);
          umma::mma_i8(tmem + (uint32_t)(acc * lp), ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
        umma::commit(&aempty[s]);
        umma::commit(&tfull[acc]);
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue --
    const int ew = warp - kEpi0;
    // tcgen05.ld: warp w may only touch TMEM lanes 32*(w%4)..+31, so the row
    // quadrant follows the hardware warp id (epilogue warps start at kEpi0)
    const int quad = warp & 3, part = ew >> 2;            // TMEM lane quadrant, column half
    const int n_parts = lp >= 32 ? 2 : 1;
    const int cols = lp / n_parts;
    const bool active = part < n_parts;
    const int r_in = quad * 32 + lane;
    const int K = p.K, L = p.L;
    const float* E = reinterpret_cast<const float*>(p.gbase + p.cls.leaf_off);
    ACC* red = reinterpret_cast<ACC*>(smem + p.red_off);  // [128][KT] part-1 partials
    ACC acc[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) acc[q] = ACC(0);
    // a5 is software-pipelined: the leaf values of item k are loaded while
    // item k+1's accumulator is read from TMEM, and added one item later
    float pv[KT];
    bool pend = false;
    auto add_pending = [&]() {
      if (pend) {
#pragma unroll
        for (int q = 0; q < KT; ++q)
          if (q < K) {
            if (std::is_same<ACC, long long>::value) acc[q] += (ACC)__float2ll_rz(pv[q]);
            else acc[q] += (ACC)pv[q];
          }
      }
      pend = false;
    };
    int k = 0;
    for (int ti = 0; ti < my_tiles; ++ti) {
      const int64_t row = (int64_t)(blockIdx.x + ti * grid) * 128 + r_in;
      for (int t = 0; t < nt; ++t, ++k) {
        const int sacc = k % NT;
        ptx::mbar_wait(&tfull[sacc], (k / NT) & 1);
        umma::fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(sacc * lp);
        int leaf = -1;
        if (active) {
          int cb = part * cols;
          const int ce = cb + cols;
          for (; cb + 32 <= ce; cb += 32) {
            uint32_t v[16], w[16];
            umma::ld16(tbase + cb, v);
            umma::ld16(tbase + cb + 16, w);
            umma::wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if ((int32_t)v[j] == D) leaf = cb + j;  // a4: S'[l] == D at the reached leaf only
              if ((int32_t)w[j] == D) leaf = cb + 16 + j;
            }
          }
          if (cb < ce) {
            uint32_t v[16];
            umma::ld16(tbase + cb, v);
            umma::wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if ((int32_t)v[j] == D) leaf = cb + j;
          }
        }
        umma::fence_before();
        ptx::mbar_arrive(&tempty[sacc]);
        add_pending();
        if (leaf >= 0) {  // a5 + a6: leaf-value gather, exact fixed-point accumulation
          const float* e = E + ((size_t)t * L + leaf) * K;
#pragma unroll
          for (int q = 0; q < KT; ++q) pv[q] = q < K ? __ldg(e + q) : 0.0f;
          pend = true;
        }
      }
      add_pending();
      // tile done: sum the two column parts, then finalize (a7) or hand on
      if (n_parts > 1 && part == 1) {
#pragma unroll
        for (int q = 0; q < KT; ++q) red[r_in * KT + q] = acc[q];
      }
      asm volatile("bar.sync 2, %0;" ::"r"(kFzEpi * 32) : "memory");
      if (part == 0 && row < p.n_rows) {
        if (n_parts > 1) {
#pragma unroll
          for (int q = 0; q < KT; ++q) acc[q] += red[r_in * KT + q];
        }
        ACC* ab = static_cast<ACC*>(p.accbuf);
        if (!p.first) {
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < K) acc[q] += ab[row * K + q];
        }
        if (p.last) {
          finalize_row<KT, ACC>(p.fin, row, acc);
        } else {
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < K) ab[row * K + q] = acc[q];
        }
      }
      asm volatile("bar.sync 2, %0;" ::"r"(kFzEpi * 32) : "memory");
#pragma unroll
      for (int q = 0; q < KT; ++q) acc[q] = ACC(0);
    }
  }
  __syncthreads();
  umma::fence_after();
  if (warp == kMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

// ------------------------------------------------------------- host side ----
static int dev_sms(int dev) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

bool gemm_build(bridger_model* m, const bridger_model_desc* d, const std::vector<int32_t>& depth, std::string* why) {
  m->gemm_ok = false;
  const int32_t T = d->n_trees, K = d->n_outputs;
  for (int32_t t = 0; t < T; ++t)
    if (depth[t] > 8) {
      if (why) *why = "GEMM path supports depth <= 8 (path matrix N = 2^D <= 256)";
      return false;
    }
  auto* h = new GemmHost();
  std::vector<int32_t> order(T);
  for (int32_t t = 0; t < T; ++t) order[t] = t;
  auto eff = [&](int32_t t) { return std::max(1, depth[t]); };
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return eff(a) < eff(b); });
  h->slot_tree = order;
  h->tree_slot.assign(T, 0);
  h->tree_class.assign(T, 0);
  std::vector<uint8_t> buf;
  auto align = [&](size_t a) { buf.resize((buf.size() + a - 1) / a * a, 0); };
  PaddedTree pt;
  int32_t s = 0;
  while (s < T) {
    const int32_t D = eff(order[s]);
    int32_t n = 0;
    while (s + n < T && eff(order[s + n]) == D) ++n;
    GemmClassDev c{};
    c.depth = D;
    c.i_pad = gemm_i_pad(D);
    c.l_pad = gemm_l_pad(D);
    c.n_trees = n;
    c.first_slot = s;
    const int32_t I = (1 << D) - 1, L = 1 << D;
    align(256);
    c.cmat_off = (int64_t)buf.size();
    {
      std::vector<int8_t> Cm((size_t)c.i_pad * c.l_pad);
      std::vector<int32_t> Dv(L);
      path_matrix(D, c.i_pad, c.l_pad, Cm.data(), Dv.data());
      buf.resize(buf.size() + (size_t)c.i_pad * c.l_pad);
      int8_t* dst = reinterpret_cast<int8_t*>(buf.data() + c.cmat_off);
      for (int32_t kc = 0; kc < c.i_pad / 16; ++kc)
        for (int32_t l = 0; l < c.l_pad; ++l)
          for (int32_t b = 0; b < 16; ++b) dst[((size_t)kc * c.l_pad + l) * 16 + b] = Cm[(size_t)(kc * 16 + b) * c.l_pad + l];
      align(16);
      c.dv_off = (int64_t)buf.size();
      buf.resize(buf.size() + 4 * (size_t)c.l_pad);
      int32_t* dv = reinterpret_cast<int32_t*>(buf.data() + c.dv_off);
      for (int32_t l = 0; l < c.l_pad; ++l) dv[l] = l < L ? Dv[l] : 127;
    }
    align(256);
    c.cmat2_off = (int64_t)buf.size();
    {
      std::vector<int8_t> Cm((size_t)c.i_pad * c.l_pad);
      path_matrix(D, c.i_pad, c.l_pad, Cm.data(), nullptr);
      for (int32_t l = 0; l < c.l_pad; ++l) Cm[(size_t)I * c.l_pad + l] = l < L ? (int8_t)__builtin_popcount(l) : (int8_t)-64;
      buf.resize(buf.size() + (size_t)c.i_pad * c.l_pad);
      int8_t* dst = reinterpret_cast<int8_t*>(buf.data() + c.cmat2_off);
      for (int32_t kc = 0; kc < c.i_pad / 16; ++kc)
        for (int32_t l = 0; l < c.l_pad; ++l)
          for (int32_t b = 0; b < 16; ++b) dst[((size_t)kc * c.l_pad + l) * 16 + b] = Cm[(size_t)(kc * 16 + b) * c.l_pad + l];
    }
    align(16);
    c.node_off = (int64_t)buf.size();
    buf.resize(buf.size() + 8 * (size_t)n * c.i_pad);
    align(16);
    c.feat_off = (int64_t)buf.size();
    buf.resize(buf.size() + 4 * (size_t)n * c.i_pad);
    align(16);
    c.thr_off = (int64_t)buf.size();
    buf.resize(buf.size() + 4 * (size_t)n * c.i_pad);
    align(16);
    c.leaf_off = (int64_t)buf.size();
    buf.resize(buf.size() + 4 * (size_t)n * L * K);
    for (int32_t j = 0; j < n; ++j) {
      const int32_t t = order[s + j];
      h->tree_slot[t] = s + j;
      h->tree_class[t] = (int32_t)h->classes.size();
      pad_tree(d, t, D, &pt);
      int32_t* fe = reinterpret_cast<int32_t*>(buf.data() + c.feat_off) + (size_t)j * c.i_pad;
      float* th = reinterpret_cast<float*>(buf.data() + c.thr_off) + (size_t)j * c.i_pad;
      for (int32_t i = 0; i < c.i_pad; ++i) {
        if (i < I) {
          fe[i] = pt.feature[i] | (pt.missing[i] ? (int32_t)0x80000000 : 0);
          if (pt.missing[i]) h->has_missing = true;
          th[i] = pt.threshold[i];
        } else {
          fe[i] = 0;  // padding: x <= NaN is false, so P[i >= I] == 0 exactly
          th[i] = std::numeric_limits<float>::quiet_NaN();
        }
      }
      uint32_t* nr = reinterpret_cast<uint32_t*>(buf.data() + c.node_off) + (size_t)j * c.i_pad * 2;
      for (int32_t i = 0; i < c.i_pad; ++i) {
        float tv = th[i];
        uint32_t fv = (uint32_t)fe[i];
        if (i == I) {  // K5 constant-1 decision: the X tile's extra row F is all zeros, 0 <= +inf
          tv = std::numeric_limits<float>::infinity();
          fv = (uint32_t)d->n_features;
        }
        std::memcpy(&nr[2 * i + 1], &tv, 4);
        nr[2 * i] = fv;
      }
      float* lv = reinterpret_cast<float*>(buf.data() + c.leaf_off) + (size_t)j * L * K;
      for (int32_t l = 0; l < L * K; ++l) lv[l] = m->acc_int ? std::ldexp(pt.leaf_value[l], -m->ex.q) : pt.leaf_value[l];
    }
    // ---- 2:4-sparse form: regrouped node arrays, compressed C_sp^T + metadata
    c.k_sp = gemm_k_sp(D);
    c.m_sp = gemm_m_sp(D);
    {
      const int32_t ks_n = c.k_sp / 64, mt_n = c.m_sp / 128;
      std::vector<int8_t> Csp((size_t)c.k_sp * c.m_sp);
      path_matrix_sparse(D, Csp.data());
      align(1024);
      c.asp_off = (int64_t)buf.size();
      buf.resize(buf.size() + (size_t)mt_n * ks_n * 4096, 0);
      align(16);
      c.meta_off = (int64_t)buf.size();
      buf.resize(buf.size() + (size_t)mt_n * 128 * ks_n * 2 * 4, 0);
      int8_t* asp = reinterpret_cast<int8_t*>(buf.data() + c.asp_off);
      uint32_t* meta = reinterpret_cast<uint32_t*>(buf.data() + c.meta_off);
      for (int32_t mt = 0; mt < mt_n; ++mt)
        for (int32_t r = 0; r < 128; ++r)
          for (int32_t ks = 0; ks < ks_n; ++ks) {
            const int32_t l = mt * 128 + r;
            uint32_t w[2] = {0u, 0u};
            for (int32_t g = 0; g < 16; ++g) {
              const int32_t k0 = ks * 64 + 4 * g;
              int8_t v[4];
              int32_t nz[4], nnz = 0;
              for (int32_t q = 0; q < 4; ++q) {
                v[q] = Csp[(size_t)(k0 + q) * c.m_sp + l];
                if (v[q]) nz[nnz++] = q;
              }
              if (nnz > 2) {
                delete h;
                if (why) *why = "internal: path matrix not 2:4 structured";
                return false;
              }
              // two kept positions p0 < p1 (the non-zeros, padded with zeros)
              int32_t p0 = 0, p1 = 1;
              if (nnz == 2) { p0 = nz[0]; p1 = nz[1]; }
              else if (nnz == 1) { p0 = nz[0] < 3 ? nz[0] : 2; p1 = p0 + 1; }
              const int32_t j = 2 * g;  // compressed index within the K-step (0..31)
              int8_t* a = asp + (size_t)(mt * ks_n + ks) * 4096;
              a[(j >> 4) * 2048 + r * 16 + (j & 15)] = v[p0];
              a[((j + 1) >> 4) * 2048 + r * 16 + ((j + 1) & 15)] = v[p1];
              w[g >> 3] |= (uint32_t)(p0 | (p1 << 2)) << (4 * (g & 7));
            }
            meta[((size_t)(mt * 128 + r) * ks_n + ks) * 2 + 0] = w[0];
            meta[((size_t)(mt * 128 + r) * ks_n + ks) * 2 + 1] = w[1];
          }
      align(16);
      c.feat_sp_off = (int64_t)buf.size();
      buf.resize(buf.size() + 4 * (size_t)n * c.k_sp, 0);
      align(16);
      c.thr_sp_off = (int64_t)buf.size();
      buf.resize(buf.size() + 4 * (size_t)n * c.k_sp, 0);
      const int32_t* fe_all = reinterpret_cast<const int32_t*>(buf.data() + c.feat_off);
      const float* th_all = reinterpret_cast<const float*>(buf.data() + c.thr_off);
      for (int32_t j = 0; j < n; ++j) {
        int32_t* fe = reinterpret_cast<int32_t*>(buf.data() + c.feat_sp_off) + (size_t)j * c.k_sp;
        float* th = reinterpret_cast<float*>(buf.data() + c.thr_sp_off) + (size_t)j * c.k_sp;
        for (int32_t k = 0; k < c.k_sp; ++k) {
          fe[k] = 0;
          th[k] = std::numeric_limits<float>::quiet_NaN();  // dummy: decision 0 (C_sp is zero there anyway)
        }
        for (int32_t i = 0; i < I; ++i) {
          fe[sparse_pos(i)] = fe_all[(size_t)j * c.i_pad + i];
          th[sparse_pos(i)] = th_all[(size_t)j * c.i_pad + i];
        }
      }
    }
    h->max_psp_per_row = std::max<int64_t>(h->max_psp_per_row, (int64_t)n * c.k_sp);
    h->max_p_per_row = std::max<int64_t>(h->max_p_per_row, (int64_t)n * c.i_pad);
    h->max_trees = std::max(h->max_trees, n);
    h->classes.push_back(c);
    s += n;
  }
  void* dbuf = nullptr;
  if (cudaMalloc(&dbuf, buf.size()) != cudaSuccess || cudaMemcpy(dbuf, buf.data(), buf.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(dbuf);
    delete h;
    if (why) *why = "GEMM layout upload failed";
    return false;
  }
  m->d_gemm = dbuf;
  m->gemm_host = h;
  m->gemm_ok = true;
  for (auto& c : h->classes) m->gemm_classes.push_back({c.depth, c.i_pad, c.l_pad, c.first_slot, c.n_trees});
  return true;
}

void gemm_free(bridger_model* m) {
  cudaFree(m->d_gemm);
  m->d_gemm = nullptr;
  delete static_cast<GemmHost*>(m->gemm_host);
  m->gemm_host = nullptr;
}

static cudaError_t launch_gc(const float* X, int64_t row0, int32_t rows, int32_t F, const uint8_t* gbase,
                             const GemmClassDev& c, int32_t t_begin, int32_t t_end, int8_t* P, bool plain, bool ml,
                             int sms, cudaStream_t st) {
  const int n_rt = (rows + 127) / 128;
  const int n_t = t_end - t_begin;
  const int smem = 129 * F * 4 + 2 * c.i_pad * 8;
  // spread trees over enough 4-warp CTAs to keep ~12 resident per SM (round
  // 1 aimed at 4: ncu showed 23% of the warp slots active, issue-latency
  // bound); each tree group re-reads its 128-row X tile (from L2)
  const int per_sm = std::max(1, std::min(12, (int)(kSmemMax / std::max(1, smem + 1024))));
  int tpc = std::max(1, (int)((int64_t)n_t * n_rt / ((int64_t)per_sm * sms)));
  tpc = std::min(tpc, n_t);
  dim3 grid(n_rt, (n_t + tpc - 1) / tpc);
  auto k = plain ? (ml ? gc_kernel<true, true> : gc_kernel<true, false>)
                 : (ml ? gc_kernel<false, true> : gc_kernel<false, false>);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  cudaEvent_t ev;
  hot_begin(st, &ev);
  k<<<grid, 128, smem, st>>>(X, row0, rows, F, gbase, c, t_begin, tpc, t_end, P);
  hot_end_id(st, ev, 1);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_pc(const int8_t* P, const uint8_t* gbase, const GemmClassDev& c, int32_t n_trees,
                             int32_t rows, int mode, int16_t* leaf, int32_t* S, int dev, cudaStream_t st) {
  PcParams p{};
  p.P = P;
  p.gbase = gbase;
  p.cls = c;
  p.n_trees = n_trees;
  p.n_rt = (rows + 127) / 128;
  p.rows = rows;
  int cols = 32;
  while (cols < 2 * c.l_pad) cols *= 2;
  p.tmem_cols = cols;
  p.b_bytes = c.i_pad * c.l_pad;
  p.mode = mode;
  p.leaf = leaf;
  p.S = S;
  const int a_bytes = 128 * c.i_pad;
  const int b_al = (p.b_bytes + 1023) / 1024 * 1024;
  // as deep an A ring as fits next to C_D (2..8 stages)
  int stages = 8;
  while (stages > 2 && b_al + stages * a_bytes + 256 > kSmemMax) --stages;
  p.stages = stages;
  int smem = b_al + stages * a_bytes + (5 + 2 * stages) * 8 + 16 + 64;
  // co-resident CTAs must fit in the 512 TMEM columns of an SM: pad the
  // shared-memory request so no more CTAs than that are placed per SM
  const int tmem_occ = std::max(1, 512 / cols);
  smem = std::max(smem, kSmemMax / tmem_occ - 1024);
  cudaError_t e = cudaFuncSetAttribute(pc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pc_kernel, kPcThreads, smem);
  occ = std::max(1, std::min(occ, tmem_occ));
  const int n_items = n_trees * p.n_rt;
  const int grid = std::max(1, std::min(n_items, dev_sms(dev) * occ));
  cudaEvent_t ev;
  hot_begin(st, &ev);
  pc_kernel<<<grid, kPcThreads, smem, st>>>(p);
  hot_end(st, ev);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_pcs(const int8_t* P, const uint8_t* gbase, const GemmClassDev& c, int32_t n_trees,
                              int32_t rows, int mode, int16_t* leaf, int32_t* S, int dev, cudaStream_t st) {
  PcsParams p{};
  p.P = P;
  p.gbase = gbase;
  p.cls = c;
  p.n_trees = n_trees;
  p.n_rt = (rows + 127) / 128;
  p.rows = rows;
  p.mode = mode;
  p.leaf = leaf;
  p.S = S;
  const int a_al = ((c.m_sp / 128) * (c.k_sp / 64) * 4096 + 1023) / 1024 * 1024;
  const int b_bytes = 128 * c.k_sp;
  const int bar_bytes = (1 + 2 * 8 + 2 * kSpSlots) * 8 + 16;
  int stages = 6;
  while (stages > 2 && a_al + stages * b_bytes + bar_bytes > kSmemMax) --stages;
  p.stages = stages;
  // one CTA per SM: the kernel allocates all 512 TMEM columns
  const int smem = std::max(a_al + stages * b_bytes + bar_bytes, kSmemMax / 2 + 1024);
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(pcs_kernel), configured);
  if (e != cudaSuccess) return e;
  const int n_tiles = n_trees * p.n_rt;
  const int grid = std::max(1, std::min(n_tiles, dev_sms(dev)));
  cudaEvent_t ev;
  hot_begin(st, &ev);
  pcs_kernel<<<grid, kPcThreads, smem, st>>>(p);
  hot_end(st, ev);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t gemm_run_impl(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                                 int32_t total_trees, cudaStream_t st, bool sparse) {
  const GemmHost* h = static_cast<const GemmHost*>(m->gemm_host);
  const uint8_t* gbase = static_cast<const uint8_t*>(m->d_gemm);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  // row blocks: decision scratch <= 1 GB (large blocks keep every kernel's grid
  // full); BRIDGER_GEMM_SCRATCH_MB sets it (e.g. L2-resident blocks)
  const int64_t per_row = sparse ? h->max_psp_per_row : h->max_p_per_row;
  int64_t scratch = (int64_t)1 << 30;
  if (const char* ev = std::getenv("BRIDGER_GEMM_SCRATCH_MB")) scratch = (int64_t)std::max(1, std::atoi(ev)) << 20;
  int64_t rb = scratch / std::max<int64_t>(1, per_row);
  rb = std::max<int64_t>(128, rb / 128 * 128);
  rb = std::min<int64_t>(rb, (n_rows + 127) / 128 * 128);
  int8_t* P = nullptr;
  int16_t* leaf = nullptr;
  void* accbuf = nullptr;
  cudaError_t e = cudaMallocAsync(&P, (size_t)rb * per_row, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&leaf, (size_t)rb * h->max_trees * 2, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&accbuf, (size_t)rb * m->K * 8, st);
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
  const int nc = (int)h->classes.size();
  for (int64_t r0 = 0; e == cudaSuccess && r0 < n_rows; r0 += rb) {
    const int32_t rows = (int32_t)std::min<int64_t>(rb, n_rows - r0);
    for (int ci = 0; ci < nc && e == cudaSuccess; ++ci) {
      const GemmClassDev& c = h->classes[ci];
      if (sparse) {
        // K1 on the level-regrouped node arrays (K = k_sp), then the 2:4-sparse K2s
        GemmClassDev csp = c;
        csp.i_pad = c.k_sp;
        csp.feat_off = c.feat_sp_off;
        csp.thr_off = c.thr_sp_off;
        e = launch_gc(X, r0, rows, m->F, gbase, csp, 0, c.n_trees, P, false, h->has_missing, sms, st);
        if (e == cudaSuccess) e = launch_pcs(P, gbase, c, c.n_trees, rows, 0, leaf, nullptr, m->device, st);
      } else {
        e = launch_gc(X, r0, rows, m->F, gbase, c, 0, c.n_trees, P, false, h->has_missing, sms, st);
        if (e == cudaSuccess) e = launch_pc(P, gbase, c, c.n_trees, rows, 0, leaf, nullptr, m->device, st);
      }
      if (e != cudaSuccess) break;
      const int tb = 256, g = (rows + tb - 1) / tb;
      const float* E = reinterpret_cast<const float*>(gbase + c.leaf_off);
      cudaEvent_t ev3;
      hot_begin(st, &ev3);
      BRIDGER_DISPATCH_KT(m->K, {
        if (m->acc_int)
          lg_kernel<KT, long long><<<g, tb, 0, st>>>(leaf, rows, c.n_trees, E, 1 << c.depth, m->K,
                                                      static_cast<long long*>(accbuf), ci == 0, ci == nc - 1, r0, fin);
        else
          lg_kernel<KT, double><<<g, tb, 0, st>>>(leaf, rows, c.n_trees, E, 1 << c.depth, m->K,
                                                   static_cast<double*>(accbuf), ci == 0, ci == nc - 1, r0, fin);
      });
      hot_end_id(st, ev3, 2);
      count_launch();
      e = cudaGetLastError();
    }
  }
  cudaFreeAsync(P, st);
  cudaFreeAsync(leaf, st);
  cudaFreeAsync(accbuf, st);
  return e;
}

cudaError_t gemm_run(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want, int32_t total_trees,
                     cudaStream_t st) {
  return gemm_run_impl(m, X, n_rows, out, want, total_trees, st, false);
}

cudaError_t gemm_run_sparse(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                            int32_t total_trees, cudaStream_t st) {
  return gemm_run_impl(m, X, n_rows, out, want, total_trees, st, true);
}

// Shared-memory carve-up of K5: C'_D | X tile | A ring | node ring | partials | barriers.
static bool fz_plan(const GemmClassDev& c, int32_t F, int32_t K, FzParams* p) {
  int KT = 1;
  while (KT < K) KT *= 2;
  if (KT > 16) KT = 64;
  const int a_bytes = 128 * c.i_pad;
  p->b_bytes = c.i_pad * c.l_pad;
  // TMEM accumulator ring: as many L_pad-column stages as fit in 512 columns (<= 4)
  p->tstages = std::max(2, std::min(4, 512 / c.l_pad));
  int cols = 32;
  while (cols < p->tstages * c.l_pad) cols *= 2;
  p->tmem_cols = cols;
  int off = (p->b_bytes + 1023) / 1024 * 1024;
  p->x_off = off;
  off += (kFzXStride * (F + 1) * 4 + 1023) / 1024 * 1024;  // + constant-zero row F
  p->a_off = off;
  // node ring: ~16 KB in flight covers the L2 latency of the per-tree bulk copies
  p->nstages = std::max(4, std::min(kFzNodeMax, 16384 / (8 * c.i_pad)));
  const int fixed = off + p->nstages * c.i_pad * 8 + 128 * KT * 8 + 512;
  int stages = 6;
  while (stages > 2 && fixed + stages * a_bytes > kSmemMax) --stages;
  if (fixed + stages * a_bytes > kSmemMax) return false;  // X tile too wide for this depth
  p->stages = stages;
  off += stages * a_bytes;
  p->n_off = off;
  off += p->nstages * c.i_pad * 8;
  p->red_off = off;
  off += 128 * KT * 8;
  p->bar_off = off;
  off += (1 + 2 * stages + 2 * p->tstages + 2 * p->nstages) * 8 + 16;
  p->smem = off;
  return true;
}

// K5: one fused launch per depth class (accumulators carried in HBM between
// classes only when the model mixes depths).
cudaError_t gemm_run_fused(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                           int32_t total_trees, cudaStream_t st) {
  const GemmHost* h = static_cast<const GemmHost*>(m->gemm_host);
  const uint8_t* gbase = static_cast<const uint8_t*>(m->d_gemm);
  const int nc = (int)h->classes.size();
  for (const GemmClassDev& c : h->classes) {
    FzParams probe{};
    if (!fz_plan(c, m->F, m->K, &probe))  // input too wide to stage next to C'_D: staged K1->K2->K3
      return gemm_run(m, X, n_rows, out, want, total_trees, st);
  }
  void* accbuf = nullptr;
  cudaError_t e = cudaSuccess;
  if (nc > 1) e = cudaMallocAsync(&accbuf, (size_t)n_rows * m->K * 8, st);
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
  const int64_t n_tiles64 = (n_rows + 127) / 128;
  if (n_tiles64 > INT32_MAX) return cudaErrorInvalidValue;
  for (int ci = 0; ci < nc && e == cudaSuccess; ++ci) {
    const GemmClassDev& c = h->classes[ci];
    FzParams p{};
    p.X = X;
    p.n_rows = n_rows;
    p.F = m->F;
    p.K = m->K;
    p.L = 1 << c.depth;
    p.n_tiles = (int32_t)n_tiles64;
    p.gbase = gbase;
    p.cls = c;
    p.first = ci == 0;
    p.last = ci == nc - 1;
    p.accbuf = accbuf;
    p.fin = fin;
    if (!fz_plan(c, m->F, m->K, &p)) return cudaErrorInvalidConfiguration;
    const int smem = p.smem;
    const int grid = (int)std::min<int64_t>(n_tiles64, dev_sms(m->device));
    cudaEvent_t ev;
    hot_begin(st, &ev);
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
      kern<<<grid, kFzThreads, smem, st>>>(p);
    };
    BRIDGER_DISPATCH_KT(m->K, {
      if (m->acc_int) {
        if (h->has_missing) launch(fz_kernel<KT, long long, true>);
        else launch(fz_kernel<KT, long long, false>);
      } else {
        if (h->has_missing) launch(fz_kernel<KT, double, true>);
        else launch(fz_kernel<KT, double, false>);
      }
    });
    hot_end_id(st, ev, 3);
    count_launch();
    e = cudaGetLastError();
  }
  if (accbuf) cudaFreeAsync(accbuf, st);
  return e;
}

cudaError_t gemm_step_decisions(const bridger_model* m, const float* X, int64_t n_rows, int32_t tree0, int32_t n_trees,
                                int8_t* out, cudaStream_t st, std::string* why) {
  const GemmHost* h = static_cast<const GemmHost*>(m->gemm_host);
  if (tree0 < 0 || n_trees < 1 || tree0 + n_trees > m->T) {
    *why = "tree range out of bounds";
    return cudaErrorInvalidValue;
  }
  const int ci = h->tree_class[tree0];
  const GemmClassDev& c = h->classes[ci];
  for (int32_t t = tree0; t < tree0 + n_trees; ++t)
    if (h->tree_class[t] != ci || h->tree_slot[t] != h->tree_slot[tree0] + (t - tree0)) {
      *why = "trees must be consecutive members of one depth class";
      return cudaErrorInvalidValue;
    }
  if (n_rows > INT32_MAX) {
    *why = "too many rows";
    return cudaErrorInvalidValue;
  }
  const int32_t t_begin = h->tree_slot[tree0] - c.first_slot;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
  return launch_gc(X, 0, (int32_t)n_rows, m->F, static_cast<const uint8_t*>(m->d_gemm), c, t_begin,
                   t_begin + n_trees, out, true, h->has_missing, sms, st);
}

cudaError_t gemm_step_scores(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows, int32_t* out,
                             cudaStream_t st, std::string* why) {
  const GemmHost* h = static_cast<const GemmHost*>(m->gemm_host);
  const GemmClassDev* c = nullptr;
  for (auto& cc : h->classes)
    if (cc.depth == depth) c = &cc;
  if (!c) {
    *why = "model has no trees of that depth";
    return cudaErrorInvalidValue;
  }
  if (rows > INT32_MAX) {
    *why = "too many rows";
    return cudaErrorInvalidValue;
  }
  const int64_t n_rt = (rows + 127) / 128;
  int8_t* tiled = nullptr;
  cudaError_t e = cudaMallocAsync(&tiled, (size_t)n_rt * 128 * c->i_pad, st);
  if (e != cudaSuccess) return e;
  tile_kernel<<<256, 256, 0, st>>>(P, rows, c->i_pad, tiled);
  count_launch();
  e = cudaGetLastError();
  if (e == cudaSuccess)
    e = launch_pc(tiled, static_cast<const uint8_t*>(m->d_gemm), *c, 1, (int32_t)rows, 1, nullptr, out, m->device, st);
  cudaFreeAsync(tiled, st);
  return e;
}

cudaError_t gemm_step_scores_sparse(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows, int32_t* out,
                                    cudaStream_t st, std::string* why) {
  const GemmHost* h = static_cast<const GemmHost*>(m->gemm_host);
  const GemmClassDev* c = nullptr;
  for (auto& cc : h->classes)
    if (cc.depth == depth) c = &cc;
  if (!c) {
    *why = "model has no trees of that depth";
    return cudaErrorInvalidValue;
  }
  if (rows > INT32_MAX) {
    *why = "too many rows";
    return cudaErrorInvalidValue;
  }
  const int64_t n_rt = (rows + 127) / 128;
  int8_t* tiled = nullptr;
  cudaError_t e = cudaMallocAsync(&tiled, (size_t)n_rt * 128 * c->k_sp, st);
  if (e != cudaSuccess) return e;
  tile_kernel<<<256, 256, 0, st>>>(P, rows, c->k_sp, tiled);
  count_launch();
  e = cudaGetLastError();
  if (e == cudaSuccess)
    e = launch_pcs(tiled, static_cast<const uint8_t*>(m->d_gemm), *c, 1, (int32_t)rows, 1, nullptr, out, m->device, st);
  cudaFreeAsync(tiled, st);
  return e;
}

}  // namespace bridger
