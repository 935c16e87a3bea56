/*
 * bridger.h -- C ABI of the B200-native tree-ensemble inference library
 * (libbridger.so).  Hot path of arxiv 2405.12491 ("bridger") for classical ML:
 * tree / forest / boosted-tree inference expressed as primitive tensor
 * operators (COR, §4.2; primitive operators Table 4,
 * PAPER.md:564-593), code-generated here by hand for sm_100a instead of TVM
 * (PAPER.md:614).  The step decomposition:
 *   a0 lowering (host, once)           -- bridger_model_load
 *   a1 feature-select  G = X[:, A]     -- gather
 *   a2 threshold compare P = G <= B    -- less_equal
 *   a3 path contraction S = P . C_D    -- matmul
 *   a4 leaf-count compare S == D_D     -- equal/argmax
 *   a4' traversal (replaces a1..a4)    -- loop/gather/where
 *   a5 leaf value gather  E[leaf]      -- gather
 *   a6 per-tree reduction              -- sum
 *   a7 finalize (mean / base+scale*sum, sigmoid, argmax)
 *
 * Conventions (all entry points):
 *  - Every call returns a bridger_status; on a non-OK status
 *    bridger_last_error() returns a thread-local message for the calling thread.
 *  - Argument errors are detected synchronously, before anything is enqueued.
 *  - Device entry points take CALLER-OWNED DEVICE pointers on the model's device
 *    (X: contiguous row-major fp32 [n_rows x n_features], 16-byte aligned) and a
 *    cudaStream_t passed as void* (NULL = legacy default stream).  Work is
 *    enqueued on that stream and the call returns without synchronising;
 *    launch failures return BRIDGER_E_CUDA, asynchronous faults surface at the
 *    caller's next synchronisation.
 *  - n_rows == 0 is a no-op returning BRIDGER_OK.
 *  - A model is immutable after load (except bridger_model_set_variant, which
 *    must not race with predicts); concurrent predicts on different streams
 *    are safe.  Scratch memory is stream-ordered (cudaMallocAsync).
 *  - There is no CPU fallback: every compute step runs in this library's CUDA
 *    kernels; without a usable sm_100 device the calls fail with E_CUDA.
 */
#ifndef BRIDGER_H
#define BRIDGER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bridger_model bridger_model; /* opaque; owns device buffers on ONE device */

typedef enum {
  BRIDGER_OK = 0,
  BRIDGER_E_NULL_ARG = 1,     /* a required pointer was NULL */
  BRIDGER_E_SHAPE = 2,        /* n_features mismatch, negative sizes, size overflow */
  BRIDGER_E_INVALID_TREE = 3, /* node arrays do not describe valid binary trees */
  BRIDGER_E_UNSUPPORTED = 4,  /* valid but outside what is implemented (see notes) */
  BRIDGER_E_CUDA = 5,         /* CUDA runtime / launch error */
  BRIDGER_E_OOM = 6           /* device or host allocation failed */
} bridger_status;

typedef enum { BRIDGER_TASK_REGRESSION = 0, BRIDGER_TASK_CLASSIFICATION = 1 } bridger_task;
/* MEAN: s = sum_t v_t / T (decision tree, random forest).
 * SUM : s = base_score + leaf_scale * sum_t v_t (gradient boosting).   Reading c6. */
typedef enum { BRIDGER_AGG_MEAN = 0, BRIDGER_AGG_SUM = 1 } bridger_agg;
/* SOFTMAX (multiclass boosting, reading c15): proba_k = exp(s_k - max s) / sum_j exp(s_j - max s),
 * fp64, labels from s (pre-transform, exact). */
typedef enum { BRIDGER_POST_IDENTITY = 0, BRIDGER_POST_SIGMOID = 1, BRIDGER_POST_SOFTMAX = 2 } bridger_post;

/* Which lowering of steps a1..a4 runs. */
typedef enum {
  BRIDGER_VARIANT_AUTO = 0,     /* per-depth choice from measured throughput */
  BRIDGER_VARIANT_TRAVERSE = 1, /* a4': traversal kernels (group-resident or streamed) */
  BRIDGER_VARIANT_GEMM = 2,     /* a1..a7 fused (K5): producer warps write the int8
                                   decisions straight into shared memory, int8 tcgen05 path contraction
                                   into TMEM, leaf select + gather + reduce in the epilogue warps */
  BRIDGER_VARIANT_GEMM_STAGED = 3, /* the same operator form staged through HBM: K1 gather-compare ->
                                   K2 tcgen05 contraction -> K3 leaf gather/reduce (step-level kernels) */
  BRIDGER_VARIANT_GEMM_SPARSE = 4 /* staged, with K2 replaced by the 2:4-sparse path contraction
                                   (tcgen05.mma.sp kind::i8, "sparse operator replacing" PAPER.md:502,
                                   Table 2): S^T = C_sp^T . P^T with the level-regrouped
                                   path matrix as the compressed sparse A operand, metadata in TMEM */
} bridger_variant;

/*
 * Model description: T trees as concatenated node arrays (SPEC.md:264-265
 * ModelSpec tree arrays; sklearn tree_ layout).  Node ids are TREE-LOCAL inside
 * [tree_offsets[t], tree_offsets[t+1]); the root of every tree is local id 0.
 * load() deep-copies everything; the caller may free the desc on return.
 */
typedef struct {
  int32_t n_trees;             /* T >= 1 */
  int32_t n_features;          /* F >= 1 */
  int32_t n_outputs;           /* K in [1, 64]: classes (DT/RF classifier) or 1 */
  const int64_t* tree_offsets; /* [T+1], strictly increasing, tree_offsets[0] == 0 */
  const int32_t* feature;      /* [n_nodes] split feature in [0,F); ignored at leaves */
  const float* threshold;      /* [n_nodes] go LEFT iff x <= threshold (reading c1); not NaN */
  const int32_t* left;         /* [n_nodes] tree-local left child, -1 at leaves */
  const int32_t* right;        /* [n_nodes] tree-local right child, -1 at leaves */
  const float* value;          /* [n_nodes * K] read at leaves only; must be finite there
                                  ([n_nodes] scalars when tree_output is given) */
  const uint8_t* missing_left; /* optional [n_nodes]: NaN goes left iff != 0; NULL => NaN right (c2) */
  int32_t task;                /* bridger_task */
  int32_t agg;                 /* bridger_agg */
  int32_t post;                /* bridger_post (SIGMOID requires task CLASSIFICATION, K == 1) */
  const double* base_score;    /* optional [K], SUM only; NULL => 0 */
  double leaf_scale;           /* SUM only (e.g. learning rate); 1.0 if already folded */
  /* Tree sharding support: force the fixed-point exponent q and exactness tier
   * computed over the WHOLE ensemble (bridger_analyze_exactness) so that int64
   * partial sums of different shards add exactly.  force_fixed_point == 0 =>
   * analyse this desc alone. */
  int32_t force_fixed_point;
  int32_t forced_scale_exp;    /* q */
  int32_t forced_tier;         /* bridger_exact_tier */
  /* Optional [T] (multiclass boosting, reading c15; sklearn
   * GradientBoostingClassifier / XGBoost / LightGBM multiclass): tree t has ONE
   * scalar value per node and adds it to output tree_output[t] in [0, K).
   * NULL => every leaf carries a K-vector.  Lowered at load to K-vectors that are
   * zero outside tree_output[t] (identical sums: adding +0 is exact). */
  const int32_t* tree_output;
} bridger_model_desc;

/* Exactness tiers (reading c9).  q = min over non-zero leaf values of the
 * exponent of their lowest set bit, so every value is an integer multiple of
 * 2^q; M = max_k sum_t max_leaf |v| 2^-q.
 *  E53: M < 2^53  -> int64 fixed-point sums, bit-identical to any fp64 order.
 *  E63: M < 2^63  -> int64 fixed-point sums exact and order-free.
 *  F64: otherwise -> fp64 accumulation (deterministic per launch config). */
typedef enum { BRIDGER_EXACT_E53 = 0, BRIDGER_EXACT_E63 = 1, BRIDGER_EXACT_F64 = 2 } bridger_exact_tier;

/* Lowering (step a0): validate, pad every tree to a perfect tree of its depth
 * by leaf replication, heap order, pack per-variant device layouts, analyse
 * exactness, upload to cuda_device.  Errors: E_NULL_ARG, E_SHAPE (T<1, F<1,
 * K outside [1,64]), E_INVALID_TREE (offsets not increasing; exactly one of
 * left/right == -1; child out of range or == self; a node with != 1 parent or
 * unreachable from 0; feature outside [0,F); NaN threshold; non-finite leaf
 * value), E_UNSUPPORTED (SIGMOID with K != 1 or regression), E_CUDA, E_OOM.
 * Any depth is accepted: trees deeper than 14 levels or too unbalanced to pad
 * into perfect heaps use the sparse pointer layout (DESIGN.md §6, §8(f3)).
 * *out is set only on success. */
bridger_status bridger_model_load(const bridger_model_desc* desc, int cuda_device, bridger_model** out);
bridger_status bridger_model_free(bridger_model* m); /* NULL is OK; synchronises the device */

/* max_depth: deepest padded tree; exact_tier: bridger_exact_tier;
 * acc_is_int64: 1 if raw accumulators are int64 fixed point, 0 if double;
 * acc_scale_exp: q (raw value = acc * 2^q).  Any output pointer may be NULL. */
bridger_status bridger_model_info(const bridger_model* m, int32_t* max_depth, int32_t* exact_tier,
                                  int32_t* acc_is_int64, int32_t* acc_scale_exp);
bridger_status bridger_model_set_variant(bridger_model* m, int32_t variant); /* bridger_variant */
/* Traversal layout chosen at load: number of tree chunks,
 * node format (*coded: 0 heap fp32, 1 threshold-bin codes, 2 sparse pointer
 * layout for deep / unbalanced trees, 3 heap fp32 with the input transposed
 * once into feature-major blocks, 4 hybrid top-levels-resident, 6 tree-streamed:
 * row tiles resident, chunk node records streamed through shared memory, 7 tree-streamed in
 * threshold-bin codes), global-tree mode
 * (trees too large for shared memory), warps per CTA and warps per row block.
 * Any output pointer may be NULL. */
bridger_status bridger_model_layout(const bridger_model* m, int32_t* n_chunks, int32_t* coded, int32_t* global_trees,
                                    int32_t* n_warps, int32_t* group);
int32_t bridger_model_variant(const bridger_model* m); /* variant that predicts will run */

/* predict: regression -> float out[n_rows * K] (s cast to fp32);
 * classification -> int32 labels out[n_rows] (argmax s, lowest index on ties;
 * K == 1: label = s > 0). */
bridger_status bridger_predict(const bridger_model* m, const float* X, int64_t n_rows,
                               int32_t n_features, void* out, void* stream);
/* predict_proba: classification only (else E_UNSUPPORTED).  float out[n_rows*C],
 * C = K, or C = 2 for K == 1 sigmoid models ([1-p, p]). */
bridger_status bridger_predict_proba(const bridger_model* m, const float* X, int64_t n_rows,
                                     int32_t n_features, float* out, void* stream);
/* apply: int32 out_leaf[n_rows * T] = ORIGINAL tree-local leaf id reached in
 * each tree (sklearn apply), original tree order. */
bridger_status bridger_apply(const bridger_model* m, const float* X, int64_t n_rows,
                             int32_t n_features, int32_t* out_leaf, void* stream);
/* predict_raw: acc[n_rows * K] = sum over THIS model's trees of the leaf values,
 * int64 fixed point (value * 2^-q) when acc_is_int64, else double.  Used by
 * tree sharding: partials of disjoint tree sets add (exactly under E53/E63). */
bridger_status bridger_predict_raw(const bridger_model* m, const float* X, int64_t n_rows,
                                   int32_t n_features, void* acc, void* stream);
/* finalize: acc (layout of predict_raw, summed over shards) -> predict output
 * (want_proba == 0) or predict_proba output (want_proba == 1).  total_trees is
 * the ensemble size used by MEAN aggregation. */
/* Tree sharding with the cross-rank reduce fused into the walk (SURVEY.md
 * §8(e); the "compute followed by a collective" written as one kernel over
 * peer memory): like bridger_predict_raw, but every row's int64 fixed-point
 * partial sum is added with red.global.add straight into the accumulator
 * slice of the rank that owns the row -- dest[r] (HOST array of n_dest device
 * pointers: this device's own memory or a peer's, mapped through CUDA IPC and
 * reached over NVLink P2P) is rank r's slice, int64 [rows_per_rank][n_outputs],
 * row i belongs to rank i / rows_per_rank.  int64 addition is associative, so
 * the slices end bitwise equal to an NCCL reduce-scatter of predict_raw
 * outputs.  The caller zeroes every slice before any rank launches and reads
 * its own only after every rank's kernel has completed (host barriers; the
 * library never makes one rank wait for another).  rows_per_rank: a positive
 * multiple of 32 with rows_per_rank * n_dest >= n_rows; n_rows < 2^31.
 * Exact tiers and the multi-chunk coded layout only (else
 * BRIDGER_E_UNSUPPORTED: use predict_raw + a collective). */
bridger_status bridger_predict_raw_scatter(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                                           void* const* dest, int32_t n_dest, int64_t rows_per_rank, void* stream);
bridger_status bridger_finalize(const bridger_model* m, const void* acc, int64_t n_rows,
                                int32_t total_trees, void* out, int32_t want_proba, void* stream);

/* End-to-end host-buffer entry (the e2e metric): X_host / out_host are HOST
 * pointers (pinned memory recommended); the call copies X in chunks over two
 * streams, overlapping H2D, compute and D2H, and returns after out_host is
 * complete.  want_proba as in bridger_finalize. */
bridger_status bridger_predict_host(const bridger_model* m, const float* X_host, int64_t n_rows,
                                    int32_t n_features, void* out_host, int32_t want_proba);

/* --- step-level entry points (parity tests of individual §8(a) rows) ------- */
/* a1+a2 (K1): decisions P[t][r][i] (int8 0/1, i < I_pad of tree t's padded
 * depth, zero-padded beyond I) for trees [tree0, tree0+n_trees) of the model's
 * GEMM lowering, rows [0, n_rows).  out_P is [n_trees][n_rows][i_pad] where
 * i_pad = the model's GEMM K stride for that depth class (see
 * bridger_gemm_geometry); trees must share one depth class. */
bridger_status bridger_step_decisions(const bridger_model* m, const float* X, int64_t n_rows,
                                      int32_t n_features, int32_t tree0, int32_t n_trees,
                                      int8_t* out_P, void* stream);
/* a3 (K2): S[r][l] = sum_i P[r][i] * C_D[i][l] on the tcgen05 int8 tensor cores
 * for a P laid out as bridger_step_decisions writes it; rows = n_trees*n_rows.
 * out_S int32 [rows][l_pad]. */
bridger_status bridger_step_path_scores(const bridger_model* m, int32_t depth, const int8_t* P,
                                        int64_t rows, int32_t* out_S, void* stream);
/* geometry of the GEMM lowering for a depth: I_pad (K), L_pad (N). */
bridger_status bridger_gemm_geometry(int32_t depth, int32_t* i_pad, int32_t* l_pad);
/* a3 on the 2:4-sparse form (K2s, variant GEMM_SPARSE): S[r][l] = sum_k P[r][k] *
 * C_sp[k][l] for P given in the SPARSE K order of bridger_path_matrix_sparse
 * (int8 0/1 [rows][k_sp], row-major; values at the pad positions are ignored
 * because C_sp is zero there).  out_S int32 [rows][l_pad] (l_pad as in
 * bridger_gemm_geometry).  Errors: depth not in the model -> BRIDGER_E_SHAPE. */
bridger_status bridger_step_path_scores_sparse(const bridger_model* m, int32_t depth, const int8_t* P,
                                               int64_t rows, int32_t* out_S, void* stream);

/* --- host-only helpers (no device needed) ---------------------------------- */
/* Universal path matrix of depth D (step a0): C[i*l_pad + l] = +1 if leaf l is
 * in the left subtree of heap node i, -1 if in the right subtree, else 0
 * (i < I_pad, rows >= I zero); Dv[l] = number of left turns on l's path
 * (D - popcount(l)), l < L.  C has i_pad*l_pad entries, Dv has 2^D. */
bridger_status bridger_path_matrix(int32_t depth, int8_t* C, int32_t* Dv);
/* The path matrix with its K dimension (internal nodes) regrouped for 2:4
 * structured sparsity ("sparse operator replacing",
 * PAPER.md:502): heap node i sits at K position pos(i) = i + [i >= 3] (one zero
 * row after the two level-1 nodes, so levels 0+1 share the first group of four
 * and every deeper level starts on a group boundary).  A leaf has exactly one
 * ancestor per level, hence <= 2 non-zeros in the first group and <= 1 in every
 * other group of 4 consecutive K positions.  C[k*m_sp + l] for k < k_sp =
 * round_up(2^D, 64), l < m_sp = round_up(2^D, 128) (zero outside pos(i), l < L).
 * C may be NULL (dimensions only).  depth in [1, 8] else BRIDGER_E_UNSUPPORTED. */
bridger_status bridger_path_matrix_sparse(int32_t depth, int8_t* C, int32_t* k_sp, int32_t* m_sp);
/* Padded perfect form of tree t (step a0): depth, then heap arrays feature[I],
 * threshold[I], missing_left[I], leaf_id[L] (original ids), leaf_value[L*K].
 * Call with all arrays NULL to query *depth first. */
bridger_status bridger_lower_tree(const bridger_model_desc* desc, int32_t tree, int32_t* depth,
                                  int32_t* feature, float* threshold, uint8_t* missing_left,
                                  int32_t* leaf_id, float* leaf_value);
/* Exactness analysis of a whole desc (reading c9): q, tier, log2(M) (or -1 if M == 0). */
bridger_status bridger_analyze_exactness(const bridger_model_desc* desc, int32_t* scale_exp,
                                         int32_t* tier, double* log2_M);
/* Validation only (E_INVALID_TREE etc. exactly as load). */
bridger_status bridger_validate(const bridger_model_desc* desc);
/* Host emulation of step a1's threshold-bin codes from the tables the load
 * would build ("data type rewriting"; DESIGN.md §6 bucketed /
 * bucket-entry binning), for CPU tests of the table construction: code(x) =
 * #{distinct thresholds of feature f < x}, 0xFFFF for NaN.  method 1: the
 * bucketed table (cum + 15-wide window search), 2: the bucket-entry table
 * ({cum | cnt, t0, t1, t2} + the window when cnt > 3).  X host [n_rows][F]
 * fp32, codes host [n_rows][F] u16 (caller-owned).  *nb = the table's bucket
 * count, 0 when the load would not build that table (codes untouched).
 * E_UNSUPPORTED when the model would not use threshold-bin codes. */
bridger_status bridger_bin_codes_host(const bridger_model_desc* desc, const float* X, int64_t n_rows,
                                      int32_t n_features, int32_t method, uint16_t* codes, int32_t* nb);

/* ---------------------------------------------------------------------------
 * Linear models (the paper's other GPU-evaluated classical-ML
 * models, PAPER.md:800-801, 861-862 -- LogisticRegression, SGDClassifier,
 * LinearRegression, Ridge -- optionally behind a StandardScaler).  What is
 * computed (oracle.c oracle_linear_run is the definition):
 *   x'_f = ((float)x_f - (float)mean_f) / (float)scale_f   fp32 ops (reading c16),
 *                                                          only with a scaler
 *   s_k  = intercept_k + sum_{f=0..F-1} coef[k][f] * x'_f   fp64, f ascending, no FMA
 *   regression: out[r,k] = (float) s_k
 *   classification K == 1: label = [s_0 > 0]; proba = [1-p, p], p = sigmoid(s_0)
 *   classification K >= 2: label = lowest k maximising s_k; proba = softmax
 *                          (post SOFTMAX) or (float) s_k (post IDENTITY)
 * Scores are bit-identical to the oracle's (same fp64 operation order), so
 * labels are exact; sigmoid/softmax probabilities agree within 1e-5 (c10).
 * HBM-bound: one pass over X, the weights broadcast from shared memory.
 * --------------------------------------------------------------------------- */
typedef struct bridger_linear bridger_linear; /* opaque; immutable after load; owns device memory */
typedef struct {
  int32_t n_features;         /* F >= 1 */
  int32_t n_outputs;          /* K in [1, 64] (K = 1: binary classifier or single-target regressor) */
  const double* coef;         /* [K * F] row-major, finite */
  const double* intercept;    /* optional [K]; NULL => 0 */
  const double* scaler_mean;  /* optional [F] StandardScaler mean_ (with scaler_scale) */
  const double* scaler_scale; /* optional [F] StandardScaler scale_; both or neither */
  int32_t task;               /* bridger_task */
  int32_t post;               /* IDENTITY; SIGMOID (classification, K == 1); SOFTMAX (classification, K >= 2) */
} bridger_linear_desc;

/* Deep-copies the desc to the device.  E_NULL_ARG (NULL desc/coef/out),
 * E_SHAPE (F < 1, K out of range, only one scaler array), E_INVALID_TREE
 * (non-finite coefficient, scale == 0), E_UNSUPPORTED (post/task mismatch). */
bridger_status bridger_linear_load(const bridger_linear_desc* desc, int cuda_device, bridger_linear** out);
bridger_status bridger_linear_free(bridger_linear* m); /* NULL ok */
/* predict: regression -> float out[n_rows * K]; classification -> int32 labels out[n_rows]. */
bridger_status bridger_linear_predict(const bridger_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                                      void* out, void* stream);
/* classification only: float out[n_rows * C], C = K, or 2 for K == 1 ([1-p, p]). */
bridger_status bridger_linear_predict_proba(const bridger_linear* m, const float* X, int64_t n_rows,
                                            int32_t n_features, float* out, void* stream);
/* raw scores s: double out[n_rows * K] (sklearn decision_function / predict in fp64). */
bridger_status bridger_linear_decision(const bridger_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                                       double* out, void* stream);

const char* bridger_last_error(void);
const char* bridger_status_string(bridger_status s);
/* Number of kernel launches this thread has issued through the library (for
 * the bench's gpu_launches claim). */
int64_t bridger_launch_count(void);
/* Hot-kernel timing (bench roofline): while enabled, the library brackets each
 * launch of the dominant kernel (traversal or path-contraction kernel) with
 * CUDA events on the launching stream.  bridger_hot_kernel_time synchronises
 * those events, returns the summed milliseconds and the number of launches
 * since the last query, and clears them. */
bridger_status bridger_hot_kernel_timing(int32_t enable);
bridger_status bridger_hot_kernel_time(double* total_ms, int64_t* launches);
/* Same for a kernel id: 0 = dominant kernel (traversal / path contraction K2,
 * linear-model kernel), 1 = gather-compare K1, 2 = leaf gather / reduce K3,
 * 3 = fused GEMM-form K5. */
bridger_status bridger_hot_kernel_time_by(int32_t kernel, double* total_ms, int64_t* launches);
/* Roofline probe (bench.py, live on the measuring box): shared-memory (LSU)
 * pipe bandwidth on `cuda_device` in GB/s -- one 512-thread CTA per SM issuing
 * unrolled LDS.64 with lane-consecutive (conflict-free, the 128 B/clk/SM unit
 * rate) and per-lane random addresses; best of 5 launches each.  Synchronises
 * the device; runs ~0.2 s.  Errors: invalid device / launch -> BRIDGER_E_CUDA.
 * Not part of the inference path (the traversal is bound by this pipe,
 * SURVEY.md §8(d) "Which roofline bounds what"). */
bridger_status bridger_probe_smem_bandwidth(int32_t cuda_device, double* conflict_free_gbps, double* random_gbps);

#ifdef __cplusplus
}
#endif
#endif /* BRIDGER_H */
