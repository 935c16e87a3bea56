// Internal declarations shared by the library's translation units (host
// lowering, kernels, C ABI).  Not installed; the public surface is
// include/bridger.h.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bridger.h"

namespace bridger {

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
bridger_status fail(bridger_status s, const std::string& msg);

// ------------------------------------------------------------ lowering -------
// One tree padded to a perfect tree of depth D in heap order (step a0,
// SURVEY.md §8(a)): children of heap node i are 2i+1 / 2i+2; leaves are heap
// nodes I..2I (I = 2^D - 1) and leaf index l = heap - I.  A leaf of the
// original tree at depth d < D is REPLICATED into all 2^(D-d) heap leaves under
// its heap position, and the internal heap nodes below it get a dummy split
// (feature 0, threshold 0): both subtrees are identical, so any routing of a
// dummy (NaN included) reaches the same value and the same original leaf id
// (reading c11; the leaf self-loop of SPEC.md:283 made static).
struct PaddedTree {
  int32_t depth = 0;
  std::vector<int32_t> feature;   // [I]
  std::vector<float> threshold;   // [I]
  std::vector<uint8_t> missing;   // [I] (0 when the desc has no missing_left)
  std::vector<int32_t> leaf_id;   // [L] original tree-local node id
  std::vector<float> leaf_value;  // [L*K]
};

bridger_status validate_desc(const bridger_model_desc* d);

// A validated desc with per-tree scalar outputs (tree_output, reading c15)
// rewritten to K-vector leaves that are zero outside the tree's output: every
// later stage sees one layout.  Sums are unchanged (x + 0.0 == x exactly).
struct ExpandedDesc {
  explicit ExpandedDesc(const bridger_model_desc* d);
  const bridger_model_desc* get() const { return &desc; }
  bridger_model_desc desc;
  std::vector<float> value;
};
int32_t tree_depth(const bridger_model_desc* d, int32_t t);  // desc must be valid
void pad_tree(const bridger_model_desc* d, int32_t t, int32_t D, PaddedTree* out);

struct Exactness {
  int32_t q = 0;        // every leaf value is an integer multiple of 2^q
  int32_t tier = BRIDGER_EXACT_E53;
  double log2_M = -1.0; // log2 of max_k sum_t max_leaf |v| 2^-q  (-1 when M == 0)
};
Exactness analyze_exactness(const bridger_model_desc* d);

// Universal path matrix of depth D (step a0/a3): C[i][l] in {+1,-1,0},
// Dv[l] = number of left turns on leaf l's root path.
void path_matrix(int32_t D, int32_t i_pad, int32_t l_pad, int8_t* C, int32_t* Dv);
inline int32_t gemm_i_pad(int32_t D) { int32_t I = (1 << D) - 1; return ((I + 31) / 32) * 32; }
inline int32_t gemm_l_pad(int32_t D) { int32_t L = 1 << D; int32_t p = ((L + 15) / 16) * 16; return p < 16 ? 16 : p; }
// 2:4-sparse form (include/bridger.h bridger_path_matrix_sparse): K position of
// heap node i, K extent (multiple of the sparse MMA's 64), M extent (leaves,
// multiple of the MMA's 128 rows)
inline int32_t sparse_pos(int32_t i) { return i >= 3 ? i + 1 : i; }
inline int32_t gemm_k_sp(int32_t D) { return ((1 << D) + 63) / 64 * 64; }
inline int32_t gemm_m_sp(int32_t D) { return ((1 << D) + 127) / 128 * 128; }
void path_matrix_sparse(int32_t D, int8_t* C);  // [gemm_k_sp(D)][gemm_m_sp(D)]

// ----------------------------------------------- traversal (K4) layout -------
// A chunk is a contiguous set of trees (same padded depth) resident in one
// CTA's shared memory for the whole kernel.  In global memory (and SMEM) a
// chunk is:  nodes  [n_trees][I] {float threshold; int32 feature | missing<<31}
//            leaves [n_trees][L][K] float (fixed-point scaled when exact)
struct TravChunk {
  int64_t offset;      // byte offset of the chunk inside the packed buffer
  int32_t bytes;       // total bytes (multiple of 16)
  int32_t n_trees;
  int32_t depth;
  int32_t leaf_offset; // byte offset of the leaves inside the chunk
  int32_t first_slot;  // index of the chunk's first tree slot (slot -> original tree)
  int32_t top_levels;  // hybrid: heap levels resident in shared memory
  int64_t g_nodes;     // hybrid: first deep-level record of the chunk (global)
  int64_t g_leaves;    // hybrid: first leaf value of the chunk (global)
};
static_assert(sizeof(TravChunk) <= 64, "tree-streamed ring slots carry a chunk descriptor in a 64-byte header");

// Sparse (pointer) tree descriptor (§8(f3)): unbounded / unbalanced trees.
struct SparseTree {
  int64_t node_off;    // first 16-byte node record of the tree
  int64_t leaf_off;    // first leaf value (float index) of the tree
  int64_t leafid_off;  // first original leaf id of the tree
  int32_t depth;       // longest root-to-leaf path (internal nodes)
  int32_t slot_tree;   // original tree index
};

struct TravLayout {
  int32_t n_warps = 16;         // warps per CTA
  int32_t group = 2;            // warps sharing one 32-row X block (they split the chunk's trees)
  bool use_cluster = false;     // cross-chunk reduction over DSMEM (else global partials)
  bool global_trees = false;    // trees too large for shared memory: walked from global memory
  bool codes = false;           // threshold-bin codes: 4-byte nodes, u16 X codes (see lowering.cpp)
  bool sparse = false;          // pointer-format trees (deep / unbalanced), walked from global memory
  bool pretransposed = false;   // fp32 input transposed once into feature-major blocks (wide X, many chunks)
  bool hybrid = false;          // top levels in shared memory, deep levels + leaves in global memory
  bool split = false;           // split nodes: fp32 threshold array + 1-byte feature array (F <= 127)
  bool stream = false;          // tree-streamed: row tiles resident, chunk node records streamed (K4s)
  int32_t stream_ns = 0;        //   node-record ring depth
  int32_t stream_stage = 0;     //   bytes per ring slot (>= every chunk's node bytes)
  int32_t stream_warps = 0;     //   walking warps (rows per tile / 32)
  int32_t stream_w = 1;         //   trees walked together per pass
  bool stream_split = false;    //   split node records (fp32 thresholds + u8 features, 5 * 2^D B per tree)
  int32_t stream_slack = 0;     //   bytes after the ring the split walk's last-level child loads may read
  std::vector<uint32_t> hyb_nodes;  // [records][2] deep levels of every tree (slot order)
  std::vector<float> hyb_leaves;    // [slots][L][K]
  std::vector<SparseTree> sparse_trees;
  std::vector<uint32_t> sparse_nodes;   // [n][4] records
  std::vector<std::vector<float>> bin_sorted;  // host: sorted distinct thresholds per feature (U_f)
  std::vector<float> bin_table;     // device: [F][2^bin_k - 1] Eytzinger (BFS) search trees of U_f, +inf padded
  int32_t bin_k = 0;                // levels of every feature's search tree
  // Bucketed binning (round 2, built when it fits and pays): per feature an
  // affine fp32 bucket map b(x) = clamp(floor((x - lo) * iw), 0, NB-1)
  // (monotone in x), cum[b] = #{u : b(u) < b}, and the sorted U_f padded with
  // +inf; code(x) = cum[b(x)] + a fixed s_f-step search in a window of
  // 2^s_f - 1 >= max bucket count (lowering.cpp build_bucket_table).  Blob:
  // [F] {lo, iw, s, 0} 16 B | [F][NB+2] u16 cum | [F][bkt_stride] fp32 U
  std::vector<uint8_t> bkt_blob;
  int32_t bkt_nb = 0, bkt_stride = 0;
  int32_t bkt_fg = 0;               // > 0: tables sized for the feature-group kernel (that many features per CTA)
  // Bucket-entry binning (round 2): the same monotone bucket map, but each
  // bucket is one 16-byte entry {cum | cnt << 16, t0, t1, t2} holding its
  // first three thresholds (+inf padded), so code(x) = cum + #{t_i < x} with
  // ONE shared load when cnt <= 3 (the window search over U only when a
  // bucket holds more).  Tables for bke_fg features per CTA (row tiles staged
  // by TMA).  Blob: [F] {lo, iw, 0, 0} 16 B | [F][NB] 16 B entries |
  // [F][bke_stride] fp32 U (+inf padded)   (lowering.cpp build_entry_table)
  std::vector<uint8_t> bke_blob;
  int32_t bke_nb = 0, bke_stride = 0, bke_fg = 0;
  int32_t smem_bytes = 0;       // dynamic shared memory per CTA
  int32_t chunk_budget = 0;     // max bytes of one chunk
  bool has_missing = false;
  std::vector<TravChunk> chunks;
  std::vector<uint8_t> data;        // packed chunks
  std::vector<int32_t> slot_tree;   // [slots] original tree index
  std::vector<int64_t> slot_leafid_off; // [slots] offset into leaf_ids
  std::vector<int32_t> leaf_ids;    // concatenated [L] per slot (original ids)
};

// Shared-memory carve-up of the traversal kernel after the chunk:
//   [NB row blocks x (feature-major X + staging) = NB*256*F][mbarriers]
//   [intra-group partials NB*(G-1)*32*K*8][cluster DSMEM slots NB*2*(nC-1)*32*K*8]
// Codes mode: each 32-row code block ([F2/2][32][2] u16, 64*F2 bytes) lands in
// a buffer of 2^b >= 64*F2 bytes aligned to 2^b, so a lane's code address is
// (buffer | lane*4 | feature offset) -- one LOP3 (traverse.cuh).  The region
// holds NB groups x 2 buffers plus 2^b bytes of alignment slack.
#ifdef __CUDACC__
#define BRIDGER_HD __host__ __device__
#else
#define BRIDGER_HD
#endif
BRIDGER_HD inline int32_t code_buf_bytes(int32_t F) {
  const int32_t need = 64 * ((F + 1) & ~1);
  int32_t b = 128;
  while (b < need) b <<= 1;
  return b;
}
BRIDGER_HD inline int32_t trav_x_region(bool codes, int32_t F, int32_t nb) {
  return codes ? (2 * nb + 1) * code_buf_bytes(F) : nb * 256 * F;
}
inline int32_t trav_bar_bytes(int32_t nb) { return ((1 + 6 * nb) * 8 + 15) / 16 * 16; }
inline int32_t trav_red_bytes(int32_t nb, int32_t g, int32_t K) { return nb * (g - 1) * 32 * K * 8; }
inline int32_t trav_slot_bytes(int32_t nb, int32_t n_chunks, int32_t K) {
  return (n_chunks >= 2 && n_chunks <= 8) ? nb * 2 * (n_chunks - 1) * 32 * K * 8 : 0;
}

// Builds the resident-chunk layout; returns false (with reason) when a single
// tree does not fit the shared-memory budget.
bool build_trav_layout(const bridger_model_desc* d, const std::vector<int32_t>& depth,
                       const Exactness& ex, bool acc_int, int32_t sms, TravLayout* out, std::string* why);

// --------------------------------------------------- GEMM-path layout -------
struct GemmClass {
  int32_t depth, i_pad, l_pad;
  int32_t first_tree, n_trees;   // trees of this depth class (in sorted order)
};

// ------------------------------------------------ launch configuration -----
// K4d (trav_deep.cu) serves coded models of at least this many chunks
// (measured on B200: C3's 3 chunks 8.47 vs 8.50 ms in K4; C2's 2 chunks
// 0.392 vs 0.401 ms per step); BRIDGER_DEEP_MIN overrides
inline int deep_min_chunks() {
  const char* e = std::getenv("BRIDGER_DEEP_MIN");
  return e ? std::atoi(e) : 2;
}
#ifdef __CUDACC__
// Opt a kernel in to the full 227 KB of dynamic shared memory on the CURRENT
// device.  The attribute belongs to one device's context, so the cache is a
// per-device bitmask (one per kernel, passed by the caller as a function-local
// static), updated atomically: safe when models on several GPUs launch from
// several threads.  Devices >= 64 are simply configured on every launch.
inline cudaError_t smem_opt_in(const void* kern, std::atomic<uint64_t>& dev_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (uint64_t)1 << dev : 0;
  if (bit && (dev_mask.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  if (e == cudaSuccess && bit) dev_mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}
#endif

// ------------------------------------------------------------- finalize -----
struct FinalizeArgs {
  int32_t task, agg, post, K;
  int32_t total_trees;
  int32_t q;          // raw = acc * 2^q
  int32_t acc_int;    // accumulators are int64 fixed point (else double)
  int32_t want;       // 0 predict, 1 proba, 2 raw
  double leaf_scale;
  const double* base; // device [K] or nullptr
  void* out;
};

}  // namespace bridger

struct bridger_model {
  int device = 0;
  int32_t T = 0, F = 0, K = 0, task = 0, agg = 0, post = 0;
  double leaf_scale = 1.0;
  std::vector<double> base;
  bridger::Exactness ex;
  bool acc_int = true;
  int32_t max_depth = 0;
  int32_t variant = BRIDGER_VARIANT_AUTO;
  int32_t resolved_variant = BRIDGER_VARIANT_TRAVERSE;

  // traversal layout on device
  bridger::TravLayout trav;
  bool trav_ok = false;
  void* d_trav_data = nullptr;
  void* d_trav_chunks = nullptr;
  int32_t* d_slot_tree = nullptr;
  int64_t* d_slot_leafid_off = nullptr;
  int32_t* d_leaf_ids = nullptr;
  double* d_base = nullptr;
  void* d_hyb_nodes = nullptr;       // TravLayout::hybrid
  float* d_hyb_leaves = nullptr;
  void* d_sparse_trees = nullptr;    // SparseTree[T] (TravLayout::sparse)
  void* d_sparse_nodes = nullptr;    // uint4 records
  float* d_bin_table = nullptr;      // threshold-bin codes (TravLayout::codes)
  uint8_t* d_bkt = nullptr;          // bucketed binning tables (TravLayout::bkt_blob)
  uint8_t* d_bke = nullptr;          // bucket-entry binning tables (TravLayout::bke_blob)

  // GEMM-path layout on device (filled by gemm_path.cu)
  bool gemm_ok = false;
  std::vector<bridger::GemmClass> gemm_classes;
  void* d_gemm = nullptr;   // opaque device block owned by gemm_path.cu
  void* gemm_host = nullptr;

  // bridger_predict_host pipeline context (streams + staging buffers), lazily built
  std::mutex host_mu;
  void* host_ctx = nullptr;
};
