// C ABI of libbridger.so (include/bridger.h).  Argument checking, model
// ownership, device selection, variant dispatch.  Every compute step runs in
// this library's CUDA kernels; there is no host fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bridger_internal.h"
#include "variant_table.h"

namespace bridger {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
bridger_status fail(bridger_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
void count_launch() { ++g_launches; }

static thread_local bool g_timing = false;
static thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events[4];
// bracket kernels of a predict with events (bench roofline); id 0 = dominant
// kernel (traversal / path contraction), 1 = gather-compare, 2 = leaf gather
void hot_begin(cudaStream_t st, cudaEvent_t* ev) {
  *ev = nullptr;
  if (!g_timing) return;
  cudaEventCreate(ev);
  cudaEventRecord(*ev, st);
}
void hot_end_id(cudaStream_t st, cudaEvent_t start, int id) {
  if (!g_timing || !start) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_events[id & 3].push_back({start, e});
}
void hot_end(cudaStream_t st, cudaEvent_t start) { hot_end_id(st, start, 0); }

cudaError_t trav_run(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                     int32_t total_trees, cudaStream_t st, void* const* scatter = nullptr,
                     int64_t rows_per_rank = 0);
cudaError_t finalize_run(const bridger_model* m, const void* acc, int64_t n_rows, int32_t total_trees,
                         void* out, int want, cudaStream_t st);
// GEMM path (gemm_path.cu)
bool gemm_build(bridger_model* m, const bridger_model_desc* d, const std::vector<int32_t>& depth,
                std::string* why);
void gemm_free(bridger_model* m);
cudaError_t gemm_run(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                     int32_t total_trees, cudaStream_t st);
cudaError_t gemm_run_fused(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                           int32_t total_trees, cudaStream_t st);
cudaError_t gemm_step_decisions(const bridger_model* m, const float* X, int64_t n_rows, int32_t tree0,
                                int32_t n_trees, int8_t* out, cudaStream_t st, std::string* why);
cudaError_t gemm_step_scores(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows,
                             int32_t* out, cudaStream_t st, std::string* why);
cudaError_t gemm_step_scores_sparse(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows,
                                    int32_t* out, cudaStream_t st, std::string* why);
cudaError_t gemm_run_sparse(const bridger_model* m, const float* X, int64_t n_rows, void* out, int want,
                            int32_t total_trees, cudaStream_t st);

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

static bridger_status cuda_fail(cudaError_t e, const char* what) {
  return fail(BRIDGER_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
static cudaError_t upload(T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), n * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
}

constexpr int kHostStages = 3;
struct HostCtx {
  cudaStream_t st[kHostStages] = {};
  float* dX[kHostStages] = {};
  void* dO[kHostStages] = {};
  int stages = 2;
  int64_t rows = 0;       // capacity in rows per stage
  size_t out_row = 0;     // capacity in output bytes per row
};

static void free_host_ctx(HostCtx* c) {
  if (!c) return;
  for (int i = 0; i < kHostStages; ++i) {
    if (c->st[i]) cudaStreamSynchronize(c->st[i]);
    cudaFree(c->dX[i]);
    cudaFree(c->dO[i]);
    if (c->st[i]) cudaStreamDestroy(c->st[i]);
  }
  delete c;
}

static void free_model(bridger_model* m) {
  if (!m) return;
  DeviceGuard g(m->device);
  cudaDeviceSynchronize();
  free_host_ctx(static_cast<HostCtx*>(m->host_ctx));
  cudaFree(m->d_trav_data);
  cudaFree(m->d_trav_chunks);
  cudaFree(m->d_slot_tree);
  cudaFree(m->d_slot_leafid_off);
  cudaFree(m->d_leaf_ids);
  cudaFree(m->d_base);
  cudaFree(m->d_bin_table);
  cudaFree(m->d_bkt);
  cudaFree(m->d_bke);
  cudaFree(m->d_sparse_trees);
  cudaFree(m->d_hyb_nodes);
  cudaFree(m->d_hyb_leaves);
  cudaFree(m->d_sparse_nodes);
  gemm_free(m);
  delete m;
}

static int32_t resolve_variant(const bridger_model* m, int32_t v) {
  if (v == BRIDGER_VARIANT_TRAVERSE) return m->trav_ok ? v : -1;
  if (v == BRIDGER_VARIANT_GEMM || v == BRIDGER_VARIANT_GEMM_STAGED || v == BRIDGER_VARIANT_GEMM_SPARSE)
    return m->gemm_ok ? v : -1;
  // AUTO: the per-depth table measured on B200 (variant_table.h, generated
  // from profiles/variant_table.json by tools/variant_table.py +
  // tools/gen_variant_table.py; DESIGN.md §6 "Variant table"), indexed by the
  // model's deepest padded tree; a variant the model cannot run falls back to
  // the other form.
  const int32_t d = m->max_depth < 0 ? 0 : m->max_depth > 15 ? 15 : m->max_depth;
  const int32_t want = kVariantByDepth[d];
  if ((want == BRIDGER_VARIANT_GEMM || want == BRIDGER_VARIANT_GEMM_STAGED || want == BRIDGER_VARIANT_GEMM_SPARSE) &&
      m->gemm_ok)
    return want;
  if (m->trav_ok) return BRIDGER_VARIANT_TRAVERSE;
  if (m->gemm_ok) return BRIDGER_VARIANT_GEMM;
  return -1;
}

static bridger_status check_rows(const bridger_model* m, const void* X, int64_t n_rows, int32_t n_features,
                                 const void* out) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (n_rows < 0) return fail(BRIDGER_E_SHAPE, "n_rows < 0");
  if (n_features != m->F)
    return fail(BRIDGER_E_SHAPE, "n_features " + std::to_string(n_features) + " != model's " + std::to_string(m->F));
  if (n_rows == 0) return BRIDGER_OK;
  if (!X || !out) return fail(BRIDGER_E_NULL_ARG, "X or out is NULL");
  if (n_rows > (int64_t)1 << 40 || n_rows * (int64_t)n_features > ((int64_t)1 << 46))
    return fail(BRIDGER_E_SHAPE, "n_rows * n_features overflows");
  if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) return fail(BRIDGER_E_UNSUPPORTED, "X must be 16-byte aligned");
  return BRIDGER_OK;
}

// want: 0 predict, 1 proba, 2 raw, 3 apply
static bridger_status run(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features, void* out,
                          int want, void* stream) {
  bridger_status s = check_rows(m, X, n_rows, n_features, out);
  if (s != BRIDGER_OK || n_rows == 0) return s;
  if (want == 1 && m->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "predict_proba needs a classifier");
  DeviceGuard g(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  const int32_t v = m->resolved_variant;
  if (v == BRIDGER_VARIANT_GEMM && want != 3)
    e = gemm_run_fused(m, X, n_rows, out, want, m->T, st);
  else if (v == BRIDGER_VARIANT_GEMM_STAGED && want != 3)
    e = gemm_run(m, X, n_rows, out, want, m->T, st);
  else if (v == BRIDGER_VARIANT_GEMM_SPARSE && want != 3)
    e = gemm_run_sparse(m, X, n_rows, out, want, m->T, st);
  else if (m->trav_ok)
    e = trav_run(m, X, n_rows, out, want, m->T, st);
  else if (m->gemm_ok)
    e = gemm_run(m, X, n_rows, out, want, m->T, st);
  else
    return fail(BRIDGER_E_UNSUPPORTED, "no kernel variant supports this model");
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return BRIDGER_OK;
}

}  // namespace bridger

using namespace bridger;

extern "C" {

const char* bridger_last_error(void) { return g_err.c_str(); }

bridger_status bridger_hot_kernel_timing(int32_t enable) {
  g_timing = enable != 0;
  return BRIDGER_OK;
}

bridger_status bridger_hot_kernel_time_by(int32_t kernel, double* total_ms, int64_t* launches) {
  if (kernel < 0 || kernel > 3) return fail(BRIDGER_E_SHAPE, "kernel id must be in [0,3]");
  double sum = 0.0;
  auto& v = g_events[kernel];
  for (auto& pr : v) {
    float ms = 0.f;
    cudaEventSynchronize(pr.second);
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    sum += ms;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (total_ms) *total_ms = sum;
  if (launches) *launches = (int64_t)v.size();
  v.clear();
  return BRIDGER_OK;
}

bridger_status bridger_hot_kernel_time(double* total_ms, int64_t* launches) {
  return bridger_hot_kernel_time_by(0, total_ms, launches);
}
int64_t bridger_launch_count(void) { return g_launches; }

const char* bridger_status_string(bridger_status s) {
  switch (s) {
    case BRIDGER_OK: return "BRIDGER_OK";
    case BRIDGER_E_NULL_ARG: return "BRIDGER_E_NULL_ARG";
    case BRIDGER_E_SHAPE: return "BRIDGER_E_SHAPE";
    case BRIDGER_E_INVALID_TREE: return "BRIDGER_E_INVALID_TREE";
    case BRIDGER_E_UNSUPPORTED: return "BRIDGER_E_UNSUPPORTED";
    case BRIDGER_E_CUDA: return "BRIDGER_E_CUDA";
    case BRIDGER_E_OOM: return "BRIDGER_E_OOM";
  }
  return "unknown";
}

bridger_status bridger_validate(const bridger_model_desc* d) { return validate_desc(d); }

bridger_status bridger_analyze_exactness(const bridger_model_desc* d, int32_t* scale_exp, int32_t* tier,
                                         double* log2_M) {
  bridger_status s = validate_desc(d);
  if (s != BRIDGER_OK) return s;
  const ExpandedDesc ed(d);
  Exactness ex = analyze_exactness(ed.get());
  if (scale_exp) *scale_exp = ex.q;
  if (tier) *tier = ex.tier;
  if (log2_M) *log2_M = ex.log2_M;
  return BRIDGER_OK;
}

bridger_status bridger_path_matrix(int32_t depth, int8_t* C, int32_t* Dv) {
  if (depth < 1 || depth > 8) return fail(BRIDGER_E_UNSUPPORTED, "path matrix depth must be in [1,8]");
  if (!C) return fail(BRIDGER_E_NULL_ARG, "C is NULL");
  path_matrix(depth, gemm_i_pad(depth), gemm_l_pad(depth), C, Dv);
  return BRIDGER_OK;
}

bridger_status bridger_path_matrix_sparse(int32_t depth, int8_t* C, int32_t* k_sp, int32_t* m_sp) {
  if (depth < 1 || depth > 8) return fail(BRIDGER_E_UNSUPPORTED, "sparse path matrix depth must be in [1,8]");
  if (k_sp) *k_sp = gemm_k_sp(depth);
  if (m_sp) *m_sp = gemm_m_sp(depth);
  if (C) path_matrix_sparse(depth, C);
  return BRIDGER_OK;
}

bridger_status bridger_gemm_geometry(int32_t depth, int32_t* i_pad, int32_t* l_pad) {
  if (depth < 1 || depth > 8) return fail(BRIDGER_E_UNSUPPORTED, "GEMM path supports depth 1..8");
  if (i_pad) *i_pad = gemm_i_pad(depth);
  if (l_pad) *l_pad = gemm_l_pad(depth);
  return BRIDGER_OK;
}

bridger_status bridger_lower_tree(const bridger_model_desc* d, int32_t tree, int32_t* depth, int32_t* feature,
                                  float* threshold, uint8_t* missing_left, int32_t* leaf_id, float* leaf_value) {
  bridger_status s = validate_desc(d);
  if (s != BRIDGER_OK) return s;
  const ExpandedDesc ed(d);
  d = ed.get();
  if (tree < 0 || tree >= d->n_trees) return fail(BRIDGER_E_SHAPE, "tree index out of range");
  if (!depth) return fail(BRIDGER_E_NULL_ARG, "depth is NULL");
  const int32_t D = tree_depth(d, tree);
  *depth = D;
  if (!feature && !threshold && !missing_left && !leaf_id && !leaf_value) return BRIDGER_OK;
  if (D > 14) return fail(BRIDGER_E_UNSUPPORTED, "padded depth > 14");
  PaddedTree pt;
  pad_tree(d, tree, D, &pt);
  const int32_t I = (1 << D) - 1, L = 1 << D, K = d->n_outputs;
  if (feature) std::memcpy(feature, pt.feature.data(), sizeof(int32_t) * I);
  if (threshold) std::memcpy(threshold, pt.threshold.data(), sizeof(float) * I);
  if (missing_left) std::memcpy(missing_left, pt.missing.data(), I);
  if (leaf_id) std::memcpy(leaf_id, pt.leaf_id.data(), sizeof(int32_t) * L);
  if (leaf_value) std::memcpy(leaf_value, pt.leaf_value.data(), sizeof(float) * L * K);
  return BRIDGER_OK;
}

bridger_status bridger_bin_codes_host(const bridger_model_desc* d_in, const float* X, int64_t n_rows,
                                      int32_t n_features, int32_t method, uint16_t* codes, int32_t* nb) {
  if (!nb || (n_rows > 0 && (!X || !codes))) return fail(BRIDGER_E_NULL_ARG, "X, codes or nb is NULL");
  bridger_status s = validate_desc(d_in);
  if (s != BRIDGER_OK) return s;
  if (n_features != d_in->n_features) return fail(BRIDGER_E_SHAPE, "n_features does not match the model");
  if (method != 1 && method != 2) return fail(BRIDGER_E_UNSUPPORTED, "method must be 1 (bucketed) or 2 (entries)");
  const ExpandedDesc ed(d_in);
  const bridger_model_desc* d = ed.get();
  std::vector<int32_t> depth(d->n_trees);
  for (int32_t t = 0; t < d->n_trees; ++t) depth[t] = tree_depth(d, t);
  const Exactness ex = analyze_exactness(d);
  TravLayout L;
  std::string why;
  if (!build_trav_layout(d, depth, ex, ex.tier != BRIDGER_EXACT_F64, 148, &L, &why) || !L.codes)
    return fail(BRIDGER_E_UNSUPPORTED, "the model would not use threshold-bin codes");
  const int32_t F = d->n_features;
  const int32_t NB = method == 1 ? L.bkt_nb : L.bke_nb;
  *nb = NB;
  if (NB == 0) return BRIDGER_OK;
  const uint8_t* blob = method == 1 ? L.bkt_blob.data() : L.bke_blob.data();
  const int32_t stride = method == 1 ? L.bkt_stride : L.bke_stride;
  const size_t cum_row = ((size_t)(NB + 2) * 2 + 3) / 4 * 4;
  const float nbm1 = (float)(NB - 1);
  for (int32_t f = 0; f < F; ++f) {
    const float* prm = reinterpret_cast<const float*>(blob + (size_t)f * 16);
    const float lo = prm[0], iw = prm[1];
    // bucketed tables: U row at word offset prm[3]; entry tables: fixed stride
    const float* U = reinterpret_cast<const float*>(
                         blob + (size_t)F * 16 + (size_t)F * (method == 1 ? cum_row : (size_t)NB * 16)) +
                     (method == 1 ? (size_t)reinterpret_cast<const uint32_t*>(prm)[3] : (size_t)f * stride);
    for (int64_t r = 0; r < n_rows; ++r) {
      const float x = X[r * F + f];
      uint16_t& c = codes[r * F + f];
      if (std::isnan(x)) {
        c = 0xFFFF;
        continue;
      }
      float t = (x - lo) * iw;  // fp32, as the kernels (__fsub_rn, __fmul_rn)
      t = std::fmin(std::fmax(t, 0.f), nbm1);  // fmax(NaN, 0) = 0, as fmaxf
      const uint32_t b = (uint32_t)t;
      uint32_t pos;
      if (method == 1) {
        pos = reinterpret_cast<const uint16_t*>(blob + (size_t)F * 16 + (size_t)f * cum_row)[b];
      } else {
        const uint32_t* e = reinterpret_cast<const uint32_t*>(blob + (size_t)F * 16 + ((size_t)f * NB + b) * 16);
        float t3[3];
        std::memcpy(t3, e + 1, 12);
        pos = (e[0] & 0xFFFFu) + (t3[0] < x) + (t3[1] < x) + (t3[2] < x);
        if ((e[0] >> 16) <= 3) {
          c = (uint16_t)pos;
          continue;
        }
        pos = e[0] & 0xFFFFu;
      }
      for (int h = 8; h >= 1; h >>= 1)  // branch-free lower_bound in the 15-wide window
        if (U[pos + h - 1] < x) pos += h;
      c = (uint16_t)pos;
    }
  }
  return BRIDGER_OK;
}

bridger_status bridger_model_load(const bridger_model_desc* d_in, int cuda_device, bridger_model** out) {
  if (!out) return fail(BRIDGER_E_NULL_ARG, "out is NULL");
  bridger_status s = validate_desc(d_in);
  if (s != BRIDGER_OK) return s;
  const ExpandedDesc ed(d_in);  // per-tree scalar outputs -> K-vector leaves (reading c15)
  const bridger_model_desc* d = ed.get();
  const int32_t T = d->n_trees;
  std::vector<int32_t> depth(T);
  int32_t Dmax = 0;
  for (int32_t t = 0; t < T; ++t) {
    depth[t] = tree_depth(d, t);
    Dmax = std::max(Dmax, depth[t]);
  }
  if (Dmax > 1000000) return fail(BRIDGER_E_UNSUPPORTED, "tree depth > 1e6");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (cuda_device < 0 || cuda_device >= ndev) return fail(BRIDGER_E_CUDA, "invalid cuda_device");

  bridger_model* m = new (std::nothrow) bridger_model();
  if (!m) return fail(BRIDGER_E_OOM, "host allocation failed");
  m->device = cuda_device;
  m->T = T;
  m->F = d->n_features;
  m->K = d->n_outputs;
  m->task = d->task;
  m->agg = d->agg;
  m->post = d->post;
  m->leaf_scale = d->leaf_scale;
  m->max_depth = Dmax;
  m->base.assign(m->K, 0.0);
  if (d->base_score)
    for (int k = 0; k < m->K; ++k) m->base[k] = d->base_score[k];
  m->ex = analyze_exactness(d);
  if (d->force_fixed_point) {
    // shards of one ensemble must share q and the tier of the WHOLE ensemble
    Exactness own = m->ex;
    if (own.log2_M >= 0 && own.q < d->forced_scale_exp) {
      delete m;
      return fail(BRIDGER_E_UNSUPPORTED, "forced fixed-point exponent is coarser than this shard's leaf values");
    }
    m->ex.q = d->forced_scale_exp;
    m->ex.tier = d->forced_tier;
  }
  m->acc_int = m->ex.tier != BRIDGER_EXACT_F64;

  std::string why;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  m->trav_ok = build_trav_layout(d, depth, m->ex, m->acc_int, sms, &m->trav, &why);
  std::string why_gemm;
  DeviceGuard g(cuda_device);
  {
    // stream-ordered scratch (cudaMallocAsync) must not be returned to the OS
    // at every synchronisation: keep the default pool's memory cached
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (m->trav_ok) {
    const TravLayout& L = m->trav;
    if ((e = upload(reinterpret_cast<uint8_t**>(&m->d_trav_data), L.data.data(), L.data.size())) != cudaSuccess ||
        (e = upload(reinterpret_cast<TravChunk**>(&m->d_trav_chunks), L.chunks.data(), L.chunks.size())) != cudaSuccess ||
        (e = upload(&m->d_slot_tree, L.slot_tree.data(), L.slot_tree.size())) != cudaSuccess ||
        (e = upload(&m->d_slot_leafid_off, L.slot_leafid_off.data(), L.slot_leafid_off.size())) != cudaSuccess ||
        (e = upload(&m->d_leaf_ids, L.leaf_ids.data(), L.leaf_ids.size())) != cudaSuccess ||
        (e = upload(&m->d_bin_table, L.bin_table.data(), L.bin_table.size())) != cudaSuccess ||
        (e = upload(&m->d_bkt, L.bkt_blob.data(), L.bkt_blob.size())) != cudaSuccess ||
        (e = upload(&m->d_bke, L.bke_blob.data(), L.bke_blob.size())) != cudaSuccess ||
        (e = upload(reinterpret_cast<SparseTree**>(&m->d_sparse_trees), L.sparse_trees.data(), L.sparse_trees.size())) != cudaSuccess ||
        (e = upload(reinterpret_cast<uint32_t**>(&m->d_hyb_nodes), L.hyb_nodes.data(), L.hyb_nodes.size())) != cudaSuccess ||
        (e = upload(&m->d_hyb_leaves, L.hyb_leaves.data(), L.hyb_leaves.size())) != cudaSuccess ||
        (e = upload(reinterpret_cast<uint32_t**>(&m->d_sparse_nodes), L.sparse_nodes.data(), L.sparse_nodes.size())) != cudaSuccess) {
      free_model(m);
      return e == cudaErrorMemoryAllocation ? fail(BRIDGER_E_OOM, "device allocation failed") : cuda_fail(e, "upload");
    }
  }
  if ((e = upload(&m->d_base, m->base.data(), m->base.size())) != cudaSuccess) {
    free_model(m);
    return cuda_fail(e, "upload base");
  }
  m->gemm_ok = gemm_build(m, d, depth, &why_gemm);
  if (!m->trav_ok && !m->gemm_ok) {
    free_model(m);
    return fail(BRIDGER_E_UNSUPPORTED, "no kernel variant supports this model: " + why + "; " + why_gemm);
  }
  int32_t v = BRIDGER_VARIANT_AUTO;
  if (const char* env = std::getenv("BRIDGER_VARIANT")) {
    if (!std::strcmp(env, "traverse")) v = BRIDGER_VARIANT_TRAVERSE;
    else if (!std::strcmp(env, "gemm")) v = BRIDGER_VARIANT_GEMM;
    else if (!std::strcmp(env, "gemm_staged")) v = BRIDGER_VARIANT_GEMM_STAGED;
    else if (!std::strcmp(env, "gemm_sparse")) v = BRIDGER_VARIANT_GEMM_SPARSE;
  }
  m->variant = v;
  m->resolved_variant = resolve_variant(m, v);
  if (m->resolved_variant < 0) m->resolved_variant = resolve_variant(m, BRIDGER_VARIANT_AUTO);
  *out = m;
  return BRIDGER_OK;
}

bridger_status bridger_model_free(bridger_model* m) {
  free_model(m);
  return BRIDGER_OK;
}

bridger_status bridger_model_info(const bridger_model* m, int32_t* max_depth, int32_t* exact_tier,
                                  int32_t* acc_is_int64, int32_t* acc_scale_exp) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (max_depth) *max_depth = m->max_depth;
  if (exact_tier) *exact_tier = m->ex.tier;
  if (acc_is_int64) *acc_is_int64 = m->acc_int ? 1 : 0;
  if (acc_scale_exp) *acc_scale_exp = m->ex.q;
  return BRIDGER_OK;
}

bridger_status bridger_model_set_variant(bridger_model* m, int32_t variant) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (variant < 0 || variant > 4) return fail(BRIDGER_E_UNSUPPORTED, "unknown variant");
  const int32_t r = resolve_variant(m, variant);
  if (r < 0) return fail(BRIDGER_E_UNSUPPORTED, "variant not available for this model");
  m->variant = variant;
  m->resolved_variant = r;
  return BRIDGER_OK;
}

int32_t bridger_model_variant(const bridger_model* m) { return m ? m->resolved_variant : -1; }

bridger_status bridger_model_layout(const bridger_model* m, int32_t* n_chunks, int32_t* coded, int32_t* global_trees,
                                    int32_t* n_warps, int32_t* group) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (n_chunks) *n_chunks = m->trav_ok ? (int32_t)m->trav.chunks.size() : 0;
  if (coded) {
    // 8: threshold-bin codes walked by the many-chunk K4d kernel (trav_deep.cu)
    const char* de = std::getenv("BRIDGER_DEEP");
    const bool deep = m->trav.codes && !m->trav.stream && !m->trav.global_trees && m->acc_int &&
                      (int)m->trav.chunks.size() >= deep_min_chunks() && !(de && de[0] == '0');
    *coded = !m->trav_ok ? 0 : m->trav.stream ? (m->trav.codes ? 7 : 6) : deep ? 8 : m->trav.codes ? 1
           : m->trav.sparse ? 2 : m->trav.hybrid ? 4 : m->trav.pretransposed ? 3 : 0;
  }
  if (global_trees) *global_trees = m->trav_ok && m->trav.global_trees ? 1 : 0;
  if (n_warps) *n_warps = m->trav.n_warps;
  if (group) *group = m->trav.group;
  return BRIDGER_OK;
}

bridger_status bridger_predict(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                               void* out, void* stream) {
  return run(m, X, n_rows, n_features, out, 0, stream);
}

bridger_status bridger_predict_proba(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                                     float* out, void* stream) {
  if (m && m->task != BRIDGER_TASK_CLASSIFICATION) return fail(BRIDGER_E_UNSUPPORTED, "predict_proba needs a classifier");
  return run(m, X, n_rows, n_features, out, 1, stream);
}

bridger_status bridger_apply(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                             int32_t* out_leaf, void* stream) {
  return run(m, X, n_rows, n_features, out_leaf, 3, stream);
}

bridger_status bridger_predict_raw(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                                   void* acc, void* stream) {
  return run(m, X, n_rows, n_features, acc, 2, stream);
}

bridger_status bridger_predict_raw_scatter(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                                           void* const* dest, int32_t n_dest, int64_t rows_per_rank, void* stream) {
  bridger_status s = check_rows(m, X, n_rows, n_features, dest);
  if (s != BRIDGER_OK || n_rows == 0) return s;
  if (n_dest < 1 || n_dest > 1024) return fail(BRIDGER_E_SHAPE, "n_dest must be in [1, 1024]");
  if (rows_per_rank < 32 || rows_per_rank % 32 != 0)
    return fail(BRIDGER_E_SHAPE, "rows_per_rank must be a positive multiple of 32");
  if (rows_per_rank * n_dest < n_rows) return fail(BRIDGER_E_SHAPE, "rows_per_rank * n_dest < n_rows");
  if (n_rows >= ((int64_t)1 << 31)) return fail(BRIDGER_E_SHAPE, "scatter: n_rows must be < 2^31");
  for (int32_t r = 0; r < n_dest; ++r)
    if (!dest[r]) return fail(BRIDGER_E_NULL_ARG, "dest pointer is NULL");
  const bool deep = m->trav_ok && m->trav.codes && !m->trav.stream && !m->trav.global_trees && m->acc_int &&
                    (int)m->trav.chunks.size() >= deep_min_chunks();
  if (!deep)
    return fail(BRIDGER_E_UNSUPPORTED,
                "fused scatter needs an exact-tier model in the multi-chunk coded layout (use predict_raw + a collective)");
  DeviceGuard g(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void** d_dest = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_dest), sizeof(void*) * n_dest, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_dest, dest, sizeof(void*) * n_dest, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = trav_run(m, X, n_rows, nullptr, 2, m->T, st, d_dest, rows_per_rank);
  if (d_dest) cudaFreeAsync(d_dest, st);
  if (e != cudaSuccess) return cuda_fail(e, "predict_raw_scatter");
  return BRIDGER_OK;
}

bridger_status bridger_finalize(const bridger_model* m, const void* acc, int64_t n_rows, int32_t total_trees,
                                void* out, int32_t want_proba, void* stream) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (n_rows < 0) return fail(BRIDGER_E_SHAPE, "n_rows < 0");
  if (n_rows == 0) return BRIDGER_OK;
  if (!acc || !out) return fail(BRIDGER_E_NULL_ARG, "acc or out is NULL");
  if (total_trees < 1) return fail(BRIDGER_E_SHAPE, "total_trees < 1");
  if (want_proba && m->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "proba needs a classifier");
  DeviceGuard g(m->device);
  cudaError_t e = finalize_run(m, acc, n_rows, total_trees, out, want_proba ? 1 : 0,
                               static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "finalize");
  return BRIDGER_OK;
}

bridger_status bridger_predict_host(const bridger_model* m, const float* X_host, int64_t n_rows, int32_t n_features,
                                    void* out_host, int32_t want_proba) {
  bridger_status s = check_rows(m, X_host, n_rows, n_features, out_host);
  if (s != BRIDGER_OK || n_rows == 0) return s;
  if (want_proba && m->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "proba needs a classifier");
  DeviceGuard g(m->device);
  const int want = want_proba ? 1 : 0;
  size_t out_row_bytes;
  if (m->task == BRIDGER_TASK_REGRESSION) out_row_bytes = 4 * (size_t)m->K;
  else if (want) out_row_bytes = 4 * (size_t)(m->K == 1 ? 2 : m->K);
  else out_row_bytes = 4;
  // stages of ~32 MiB of X: each H2D is large, and compute of stage i overlaps
  // the copies of stage i+1 on the other stream
  int64_t stage_mb = 32;
  int stages = 2;
  if (const char* ev = std::getenv("BRIDGER_H2D_MB")) stage_mb = std::max(1, std::atoi(ev));  // experiments
  if (const char* ev = std::getenv("BRIDGER_H2D_STAGES")) stages = std::max(2, std::min(kHostStages, std::atoi(ev)));
  int64_t chunk = std::max<int64_t>(1024, (stage_mb << 20) / (4 * (int64_t)m->F));
  chunk = (chunk + 31) / 32 * 32;
  if (chunk > n_rows) chunk = (n_rows + 31) / 32 * 32;
  bridger_model* mm = const_cast<bridger_model*>(m);
  std::lock_guard<std::mutex> lock(mm->host_mu);
  HostCtx* c = static_cast<HostCtx*>(mm->host_ctx);
  cudaError_t e = cudaSuccess;
  if (!c || c->rows < chunk || c->out_row < out_row_bytes || c->stages != stages) {
    free_host_ctx(c);
    c = new HostCtx();
    mm->host_ctx = c;
    c->rows = std::max<int64_t>(chunk, c->rows);
    c->out_row = std::max<size_t>(out_row_bytes, 4 * (size_t)(m->K < 2 ? 2 : m->K));
    c->stages = stages;
    for (int i = 0; i < stages && e == cudaSuccess; ++i) {
      e = cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaMalloc(&c->dX[i], (size_t)c->rows * m->F * 4);
      if (e == cudaSuccess) e = cudaMalloc(&c->dO[i], (size_t)c->rows * c->out_row);
    }
    if (e != cudaSuccess) {
      free_host_ctx(c);
      mm->host_ctx = nullptr;
      return cuda_fail(e, "predict_host setup");
    }
  }
  bridger_status rs = BRIDGER_OK;
  for (int64_t r0 = 0, i = 0; e == cudaSuccess && r0 < n_rows; r0 += chunk, ++i) {
    const int64_t rows = std::min(chunk, n_rows - r0);
    const int b = (int)(i % c->stages);
    e = cudaMemcpyAsync(c->dX[b], X_host + r0 * m->F, (size_t)rows * m->F * 4, cudaMemcpyHostToDevice, c->st[b]);
    if (e != cudaSuccess) break;
    rs = run(m, c->dX[b], rows, n_features, c->dO[b], want, c->st[b]);
    if (rs != BRIDGER_OK) break;
    e = cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + r0 * out_row_bytes, c->dO[b], (size_t)rows * out_row_bytes,
                        cudaMemcpyDeviceToHost, c->st[b]);
  }
  for (int i = 0; i < c->stages; ++i) {
    cudaError_t e2 = cudaStreamSynchronize(c->st[i]);
    if (e == cudaSuccess) e = e2;
  }
  if (rs != BRIDGER_OK) return rs;
  if (e != cudaSuccess) return cuda_fail(e, "predict_host");
  return BRIDGER_OK;
}

bridger_status bridger_step_decisions(const bridger_model* m, const float* X, int64_t n_rows, int32_t n_features,
                                      int32_t tree0, int32_t n_trees, int8_t* out_P, void* stream) {
  bridger_status s = check_rows(m, X, n_rows, n_features, out_P);
  if (s != BRIDGER_OK || n_rows == 0) return s;
  if (!m->gemm_ok) return fail(BRIDGER_E_UNSUPPORTED, "model has no GEMM lowering");
  DeviceGuard g(m->device);
  std::string why;
  cudaError_t e = gemm_step_decisions(m, X, n_rows, tree0, n_trees, out_P, static_cast<cudaStream_t>(stream), &why);
  if (!why.empty()) return fail(BRIDGER_E_SHAPE, why);
  if (e != cudaSuccess) return cuda_fail(e, "step_decisions");
  return BRIDGER_OK;
}

bridger_status bridger_step_path_scores_sparse(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows,
                                               int32_t* out_S, void* stream) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (rows < 0) return fail(BRIDGER_E_SHAPE, "rows < 0");
  if (rows == 0) return BRIDGER_OK;
  if (!P || !out_S) return fail(BRIDGER_E_NULL_ARG, "P or out_S is NULL");
  if (!m->gemm_ok) return fail(BRIDGER_E_UNSUPPORTED, "model has no GEMM lowering");
  DeviceGuard g(m->device);
  std::string why;
  cudaError_t e = gemm_step_scores_sparse(m, depth, P, rows, out_S, static_cast<cudaStream_t>(stream), &why);
  if (!why.empty()) return fail(BRIDGER_E_SHAPE, why);
  if (e != cudaSuccess) return cuda_fail(e, "step_path_scores_sparse");
  return BRIDGER_OK;
}

bridger_status bridger_step_path_scores(const bridger_model* m, int32_t depth, const int8_t* P, int64_t rows,
                                        int32_t* out_S, void* stream) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (rows < 0) return fail(BRIDGER_E_SHAPE, "rows < 0");
  if (rows == 0) return BRIDGER_OK;
  if (!P || !out_S) return fail(BRIDGER_E_NULL_ARG, "P or out_S is NULL");
  if (!m->gemm_ok) return fail(BRIDGER_E_UNSUPPORTED, "model has no GEMM lowering");
  DeviceGuard g(m->device);
  std::string why;
  cudaError_t e = gemm_step_scores(m, depth, P, rows, out_S, static_cast<cudaStream_t>(stream), &why);
  if (!why.empty()) return fail(BRIDGER_E_SHAPE, why);
  if (e != cudaSuccess) return cuda_fail(e, "step_path_scores");
  return BRIDGER_OK;
}

}  // extern "C"
