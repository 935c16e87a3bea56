// Host-side lowering (step a0): validation, padding to
// perfect heap-ordered trees, exactness analysis (reading c9), the universal
// path matrix C_D / D_D, and the packed device layouts of the traversal
// kernels.  The COR view of a tree becomes five tensors per
// tree: A (feature index), B (threshold), C_D/D_D (per depth, universal) and E
// (leaf values); CML "data type rewriting" and "redundant operator
// elimination" (Table 2) show up as the int8 path matrix and the
// exact gather that replaces a one-hot feature-selection matmul.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "bridger_internal.h"

namespace bridger {

static inline bool finite_f(float v) { return std::isfinite(v); }

ExpandedDesc::ExpandedDesc(const bridger_model_desc* d) : desc(*d) {
  if (!d->tree_output) return;
  const int32_t K = d->n_outputs;
  const int64_t n = d->tree_offsets[d->n_trees];
  value.assign((size_t)n * K, 0.0f);
  for (int32_t t = 0; t < d->n_trees; ++t)
    for (int64_t g = d->tree_offsets[t]; g < d->tree_offsets[t + 1]; ++g)
      value[(size_t)g * K + d->tree_output[t]] = d->value[g];
  desc.value = value.data();
  desc.tree_output = nullptr;
}

bridger_status validate_desc(const bridger_model_desc* d) {
  if (!d) return fail(BRIDGER_E_NULL_ARG, "desc is NULL");
  if (!d->tree_offsets || !d->feature || !d->threshold || !d->left || !d->right || !d->value)
    return fail(BRIDGER_E_NULL_ARG, "desc has a NULL required array");
  if (d->n_trees < 1) return fail(BRIDGER_E_SHAPE, "n_trees must be >= 1");
  if (d->n_features < 1) return fail(BRIDGER_E_SHAPE, "n_features must be >= 1");
  if (d->n_outputs < 1 || d->n_outputs > 64) return fail(BRIDGER_E_SHAPE, "n_outputs must be in [1,64]");
  if (d->task != BRIDGER_TASK_REGRESSION && d->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "unknown task");
  if (d->agg != BRIDGER_AGG_MEAN && d->agg != BRIDGER_AGG_SUM) return fail(BRIDGER_E_UNSUPPORTED, "unknown agg");
  if (d->post != BRIDGER_POST_IDENTITY && d->post != BRIDGER_POST_SIGMOID && d->post != BRIDGER_POST_SOFTMAX)
    return fail(BRIDGER_E_UNSUPPORTED, "unknown post");
  if (d->post == BRIDGER_POST_SOFTMAX && (d->task != BRIDGER_TASK_CLASSIFICATION || d->n_outputs < 2))
    return fail(BRIDGER_E_UNSUPPORTED, "softmax post-transform needs a K >= 2 classifier");
  if (d->tree_output)
    for (int32_t t = 0; t < d->n_trees; ++t)
      if (d->tree_output[t] < 0 || d->tree_output[t] >= d->n_outputs)
        return fail(BRIDGER_E_SHAPE, "tree_output[" + std::to_string(t) + "] out of [0,K)");
  if (d->post == BRIDGER_POST_SIGMOID && (d->task != BRIDGER_TASK_CLASSIFICATION || d->n_outputs != 1))
    return fail(BRIDGER_E_UNSUPPORTED, "sigmoid post-transform needs a K == 1 classifier");
  if (!std::isfinite(d->leaf_scale)) return fail(BRIDGER_E_SHAPE, "leaf_scale not finite");
  if (d->tree_offsets[0] != 0) return fail(BRIDGER_E_INVALID_TREE, "tree_offsets[0] != 0");
  const int32_t F = d->n_features, K = d->tree_output ? 1 : d->n_outputs;  // values stored per node
  std::vector<int32_t> parents;
  std::vector<uint8_t> seen;
  std::vector<int32_t> stack;
  for (int32_t t = 0; t < d->n_trees; ++t) {
    const int64_t a = d->tree_offsets[t], b = d->tree_offsets[t + 1];
    if (b <= a) return fail(BRIDGER_E_INVALID_TREE, "tree_offsets not strictly increasing at tree " + std::to_string(t));
    if (b - a > (int64_t)1 << 30) return fail(BRIDGER_E_UNSUPPORTED, "tree too large");
    const int32_t n = (int32_t)(b - a);
    parents.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) {
      const int32_t l = d->left[a + i], r = d->right[a + i];
      if ((l == -1) != (r == -1))
        return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " node " + std::to_string(i) + ": exactly one child is -1");
      if (l == -1) {
        for (int32_t k = 0; k < K; ++k)
          if (!finite_f(d->value[(a + i) * K + k]))
            return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " leaf " + std::to_string(i) + ": non-finite value");
        continue;
      }
      if (l <= 0 || r <= 0 || l >= n || r >= n || l == i || r == i || l == r)
        return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " node " + std::to_string(i) + ": child out of range");
      const int32_t f = d->feature[a + i];
      if (f < 0 || f >= F)
        return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " node " + std::to_string(i) + ": feature out of [0,F)");
      if (std::isnan(d->threshold[a + i]))
        return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " node " + std::to_string(i) + ": NaN threshold");
      parents[l]++;
      parents[r]++;
    }
    for (int32_t i = 1; i < n; ++i)
      if (parents[i] != 1)
        return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + " node " + std::to_string(i) + ": must have exactly one parent");
    seen.assign(n, 0);
    stack.clear();
    stack.push_back(0);
    int32_t count = 0;
    while (!stack.empty()) {
      const int32_t i = stack.back();
      stack.pop_back();
      if (seen[i]) return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + ": cycle");
      seen[i] = 1;
      ++count;
      if (d->left[a + i] != -1) {
        stack.push_back(d->left[a + i]);
        stack.push_back(d->right[a + i]);
      }
    }
    if (count != n) return fail(BRIDGER_E_INVALID_TREE, "tree " + std::to_string(t) + ": unreachable nodes");
  }
  return BRIDGER_OK;
}

int32_t tree_depth(const bridger_model_desc* d, int32_t t) {
  const int64_t a = d->tree_offsets[t];
  int32_t best = 0;
  std::vector<std::pair<int32_t, int32_t>> st{{0, 0}};
  while (!st.empty()) {
    auto [i, dep] = st.back();
    st.pop_back();
    if (d->left[a + i] == -1) {
      best = std::max(best, dep);
    } else {
      st.push_back({d->left[a + i], dep + 1});
      st.push_back({d->right[a + i], dep + 1});
    }
  }
  return best;
}

void pad_tree(const bridger_model_desc* d, int32_t t, int32_t D, PaddedTree* out) {
  const int64_t a = d->tree_offsets[t];
  const int32_t K = d->n_outputs;
  const int32_t I = (1 << D) - 1, L = 1 << D;
  out->depth = D;
  out->feature.assign(I, 0);
  out->threshold.assign(I, 0.0f);
  out->missing.assign(I, 0);
  out->leaf_id.assign(L, -1);
  out->leaf_value.assign((size_t)L * K, 0.0f);
  struct E { int32_t n; int32_t h; int32_t dep; };
  std::vector<E> st{{0, 0, 0}};
  while (!st.empty()) {
    E e = st.back();
    st.pop_back();
    const int64_t g = a + e.n;
    if (d->left[g] == -1) {
      const int32_t span = 1 << (D - e.dep);
      const int32_t first = e.h * span + (span - 1) - I;  // leftmost heap leaf under h, as leaf index
      for (int32_t j = 0; j < span; ++j) {
        out->leaf_id[first + j] = e.n;
        for (int32_t k = 0; k < K; ++k) out->leaf_value[(size_t)(first + j) * K + k] = d->value[g * K + k];
      }
    } else {
      out->feature[e.h] = d->feature[g];
      out->threshold[e.h] = d->threshold[g];
      out->missing[e.h] = d->missing_left ? (d->missing_left[g] != 0) : 0;
      st.push_back({d->left[g], 2 * e.h + 1, e.dep + 1});
      st.push_back({d->right[g], 2 * e.h + 2, e.dep + 1});
    }
  }
}

// exponent of the lowest set bit of a non-zero finite float
static int32_t lsb_exp(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  const uint32_t E = (u >> 23) & 0xFF, M = u & 0x7FFFFF;
  if (E == 0) return -149 + __builtin_ctz(M);
  return (int32_t)E - 150 + __builtin_ctz(M | 0x800000u);
}

Exactness analyze_exactness(const bridger_model_desc* d) {
  Exactness ex;
  const int32_t K = d->n_outputs;
  int32_t q = INT32_MAX;
  for (int32_t t = 0; t < d->n_trees; ++t)
    for (int64_t g = d->tree_offsets[t]; g < d->tree_offsets[t + 1]; ++g)
      if (d->left[g] == -1)
        for (int32_t k = 0; k < K; ++k) {
          const float v = d->value[g * K + k];
          if (v != 0.0f) q = std::min(q, lsb_exp(v));
        }
  if (q == INT32_MAX) {  // every leaf value is zero
    ex.q = 0;
    ex.tier = BRIDGER_EXACT_E53;
    ex.log2_M = -1.0;
    return ex;
  }
  ex.q = q;
  bool overflow = false;
  unsigned __int128 worst = 0;
  std::vector<unsigned __int128> sum(K, 0);
  for (int32_t t = 0; t < d->n_trees && !overflow; ++t)
    for (int32_t k = 0; k < K && !overflow; ++k) {
      float mx = 0.0f;
      for (int64_t g = d->tree_offsets[t]; g < d->tree_offsets[t + 1]; ++g)
        if (d->left[g] == -1) mx = std::max(mx, std::fabs(d->value[g * K + k]));
      const long double term = std::ldexp((long double)mx, -q);  // exact: an integer
      if (term >= std::ldexp(1.0L, 63)) { overflow = true; break; }
      sum[k] += (unsigned __int128)(uint64_t)term;
    }
  if (overflow) {
    ex.tier = BRIDGER_EXACT_F64;
    ex.log2_M = 64.0;
    return ex;
  }
  for (int32_t k = 0; k < K; ++k) worst = std::max(worst, sum[k]);
  const long double Mf = (long double)worst;
  ex.log2_M = worst == 0 ? -1.0 : (double)std::log2(Mf);
  if (worst < ((unsigned __int128)1 << 53)) ex.tier = BRIDGER_EXACT_E53;
  else if (worst < ((unsigned __int128)1 << 63)) ex.tier = BRIDGER_EXACT_E63;
  else ex.tier = BRIDGER_EXACT_F64;
  return ex;
}

void path_matrix(int32_t D, int32_t i_pad, int32_t l_pad, int8_t* C, int32_t* Dv) {
  const int32_t I = (1 << D) - 1, L = 1 << D;
  std::memset(C, 0, (size_t)i_pad * l_pad);
  for (int32_t l = 0; l < L; ++l) {
    // walk the root path of leaf l: bit (D-1-k) of l is the turn at depth k (1 = right)
    int32_t h = 0, lefts = 0;
    for (int32_t k = 0; k < D; ++k) {
      const int32_t right = (l >> (D - 1 - k)) & 1;
      C[(size_t)h * l_pad + l] = right ? -1 : +1;
      lefts += !right;
      h = 2 * h + 1 + right;
    }
    if (Dv) Dv[l] = lefts;
    (void)I;
  }
}

// 2:4-sparse regrouping of C_D's K dimension (bridger.h bridger_path_matrix_sparse)
void path_matrix_sparse(int32_t D, int8_t* C) {
  const int32_t I = (1 << D) - 1, ks = gemm_k_sp(D), ms = gemm_m_sp(D);
  std::vector<int8_t> dense((size_t)std::max(I, 1) * ms);
  path_matrix(D, std::max(I, 1), ms, dense.data(), nullptr);
  std::memset(C, 0, (size_t)ks * ms);
  for (int32_t i = 0; i < I; ++i)
    std::memcpy(C + (size_t)sparse_pos(i) * ms, dense.data() + (size_t)i * ms, (size_t)ms);
}

// ------------------------------------------------------ traversal layout ----
static constexpr int32_t kSmemMax = 232448;  // 227 KB opt-in per block (sm_100)

// Threshold-bin codes (§8(f2), "data type rewriting" PAPER.md:502): per
// feature f the sorted distinct thresholds U_f; x becomes
// code(x) = #{u in U_f : u < x} (NaN -> 0xFFFF), and a node's threshold t =
// U_f[j] becomes j.  For every non-NaN x:  x <= U_f[j]  <=>  code(x) <= j
// (the thresholds below x are exactly U_f[0..code(x)-1]), so the comparison is
// unchanged bit for bit.  Eligible when F <= 512 and every |U_f| <= 65534
// (codes and node indices fit 15 bits).  The device search structure is, per
// feature, U_f laid out as a complete binary search tree in BFS (Eytzinger)
// order with 2^k - 1 slots (k uniform over the features so every lane of a
// warp takes the same k steps), padded with +inf: descending
// i <- 2i + 1 + [E[i] < x] for k levels ends at leaf i - (2^k - 1) = #{u < x}
// (the padding never counts: +inf < x is false for every x).
static void eytzinger_fill(const std::vector<float>& sorted, std::vector<float>& out, size_t base, int64_t i,
                           int64_t size, int64_t& next) {
  if (i >= size) return;
  eytzinger_fill(sorted, out, base, 2 * i + 1, size, next);
  out[base + i] = next < (int64_t)sorted.size() ? sorted[next] : INFINITY;
  ++next;
  eytzinger_fill(sorted, out, base, 2 * i + 2, size, next);
}

static bool build_bin_table(const bridger_model_desc* d, TravLayout* out) {
  const int32_t F = d->n_features;
  out->bin_sorted.clear();
  out->bin_table.clear();
  out->bin_k = 0;
  if (F > 512) return false;
  std::vector<std::vector<float>>& u = out->bin_sorted;
  u.assign(F, {});
  for (int32_t t = 0; t < d->n_trees; ++t)
    for (int64_t g = d->tree_offsets[t]; g < d->tree_offsets[t + 1]; ++g)
      if (d->left[g] != -1) u[d->feature[g]].push_back(d->threshold[g]);
  size_t nmax = 0;
  for (int32_t f = 0; f < F; ++f) {
    auto& v = u[f];
    std::sort(v.begin(), v.end());
    // -0.0 and +0.0 compare equal: keep one
    v.erase(std::unique(v.begin(), v.end(), [](float a, float b) { return a == b; }), v.end());
    if (v.size() > 65534) return false;  // codes 0..|U_f| and NaN = 0xFFFF in 16 bits
    nmax = std::max(nmax, v.size());
  }
  int32_t k = 1;
  while (((size_t)1 << k) - 1 < nmax) ++k;
  const size_t P = ((size_t)1 << k) - 1;
  out->bin_k = k;
  out->bin_table.assign((size_t)F * P, INFINITY);
  for (int32_t f = 0; f < F; ++f) {
    int64_t next = 0;
    eytzinger_fill(u[f], out->bin_table, (size_t)f * P, 0, (int64_t)P, next);
  }
  return true;
}

// Bucketed binning tables (see TravLayout::bkt_blob).  Exactness: b(x) is
// monotone non-decreasing in x (fp32 subtraction and multiplication by a
// positive constant round monotonically, floor and clamp are monotone; the
// device evaluates the identical fp32 expression, __fsub_rn / __fmul_rn /
// fmaxf / fminf, host built with -ffp-contract=off), so thresholds in lower
// buckets are < x and thresholds in higher buckets are > x: code(x) =
// #{u < x} = cum[b(x)] + #{u in bucket b(x) : u < x}, the second term a
// lower_bound in the window U[cum[b] .. cum[b] + 2^s - 1) (positions past the
// bucket hold larger thresholds or +inf padding).  Built only if every
// feature's max bucket count <= 15 (s <= 4) for the chosen NB and the tables
// fit next to the staging buffers.
// fg_features > 0: tables for the feature-group kernel (bin_bucket_fg_kernel),
// which holds only fg_features features' rows per CTA -- the fit test is per
// group, not for the whole blob (C5-shaped: 200 features x ~6.4K thresholds).
static void build_bucket_table(int32_t F, TravLayout* out, int32_t staging_bytes, int32_t fg_features = 0) {
  out->bkt_blob.clear();
  out->bkt_nb = 0;
  out->bkt_stride = 0;
  out->bkt_fg = 0;
  const auto& u = out->bin_sorted;
  if ((int32_t)u.size() != F || F == 0) return;
  size_t nmax = 0;
  for (auto& v : u) nmax = std::max(nmax, v.size());
  const int32_t stride = (int32_t)((nmax + 16 + 3) / 4 * 4);  // + 15 +inf pad (window overrun), 16-B rows
  // U rows: all-features tables give each feature a row of its own length
  // (count + 16, 16-byte multiple; word offset in prm[3]) -- the freed bytes
  // buy the kernel a third staged block; feature-group tables keep one stride
  // (a group's rows are copied as one contiguous range)
  std::vector<uint32_t> uoff(F + 1, 0);
  for (int32_t f = 0; f < F; ++f)
    uoff[f + 1] = uoff[f] + (fg_features > 0 ? (uint32_t)stride : (uint32_t)((u[f].size() + 16 + 3) / 4 * 4));
  for (int32_t NB : {256, 512, 1024, 2048, 4096, 8192, 16384}) {
    const size_t cum_row = ((size_t)(NB + 2) * 2 + 3) / 4 * 4;
    const size_t bytes = (size_t)F * 16 + (size_t)F * cum_row + (size_t)uoff[F] * 4;
    if (fg_features > 0) {
      if ((size_t)fg_features * (16 + cum_row + (size_t)stride * 4) + 64 > (size_t)kSmemMax) break;
    } else if (bytes + (size_t)staging_bytes + 64 > (size_t)kSmemMax) {
      break;
    }
    std::vector<uint8_t> blob(bytes, 0);
    bool ok = true;
    for (int32_t f = 0; f < F && ok; ++f) {
      const std::vector<float>& v = u[f];
      float lo = v.empty() ? 0.f : v.front();
      float hi = v.empty() ? 0.f : v.back();
      const float span = hi - lo;
      const float iw = span > 0.f ? (float)NB / span : (v.size() > 1 ? 0.f : INFINITY);
      if (!(std::isfinite(lo) && std::isfinite(hi)) || iw == 0.f) { ok = false; break; }
      const float nbm1 = (float)(NB - 1);
      auto bucket = [&](float x) {
        float t = (x - lo) * iw;
        t = std::fmin(std::fmax(t, 0.f), nbm1);
        return (int32_t)t;
      };
      std::vector<int32_t> cnt(NB, 0);
      int32_t prev = -1;
      for (float x : v) {
        const int32_t b = bucket(x);
        if (b < prev) { ok = false; break; }  // monotonicity (holds by construction; checked)
        prev = b;
        ++cnt[b];
      }
      int32_t mx = 0;
      for (int32_t c : cnt) mx = std::max(mx, c);
      int32_t sf = 0;
      while (((1 << sf) - 1) < mx) ++sf;
      if (sf > 4) { ok = false; break; }
      float* prm = reinterpret_cast<float*>(blob.data() + (size_t)f * 16);
      prm[0] = lo;
      prm[1] = iw;
      reinterpret_cast<uint32_t*>(prm)[2] = (uint32_t)sf;
      reinterpret_cast<uint32_t*>(prm)[3] = uoff[f];
      uint16_t* cum = reinterpret_cast<uint16_t*>(blob.data() + (size_t)F * 16 + (size_t)f * cum_row);
      int32_t run = 0;
      for (int32_t b = 0; b < NB; ++b) {
        cum[b] = (uint16_t)run;
        run += cnt[b];
      }
      cum[NB] = (uint16_t)run;
      float* U = reinterpret_cast<float*>(blob.data() + (size_t)F * 16 + (size_t)F * cum_row) + uoff[f];
      for (int32_t i = 0; i < (int32_t)(uoff[f + 1] - uoff[f]); ++i) U[i] = i < (int32_t)v.size() ? v[i] : INFINITY;
    }
    if (!ok) continue;
    out->bkt_blob.swap(blob);
    out->bkt_nb = NB;
    out->bkt_stride = stride;
    out->bkt_fg = fg_features;
    return;
  }
}

// Bucket-entry tables (TravLayout::bke_blob) for bin_entry_kernel: FG
// features per CTA (FG * 4 B = the TMA box width, >= 16 B), 16 warps each
// double-buffering a [32][FG] fp32 row tile; NB = the most buckets that fit
// the rest of shared memory.  FG = 8 when that leaves >= 3 buckets per
// threshold of the densest feature, else 4.  Same monotone map as
// build_bucket_table (exact: thresholds in earlier buckets are < x, in later
// ones > x); every bucket must hold <= 15 thresholds (the overflow window).
static void build_entry_table(int32_t F, TravLayout* out) {
  out->bke_blob.clear();
  out->bke_nb = out->bke_stride = out->bke_fg = 0;
  const auto& u = out->bin_sorted;
  if ((int32_t)u.size() != F || F == 0) return;
  size_t nmax = 0;
  for (auto& v : u) nmax = std::max(nmax, v.size());
  if (nmax == 0) return;
  const int32_t stride = (int32_t)((nmax + 16 + 3) / 4 * 4);
  // row tile width: FG values, or FG + 4 when rows are not 16-byte aligned
  // (R > 1 super-rows: TMA box starts must be 16-byte aligned, so the box
  // begins up to 3 values early; traverse.cu bin_entry_kernel)
  const bool rows_aligned = (F * 4) % 16 == 0;
  auto nb_for = [&](int32_t fg) {
    const int64_t w = rows_aligned ? fg : fg + 4;
    // 32 warps of double-buffered tiles where rows are aligned (the
    // L2-resident default case, C2), else 16 (bin_entry_kernel's launcher
    // falls back to 16 when 32 do not fit)
    const int64_t nwarps = rows_aligned ? 32 : 16;
    const int64_t staging = nwarps * 2 * 32 * w * 4 + nwarps * 2 * 8 + 64;
    const int64_t per_f = (kSmemMax - staging) / fg - 16 - 4LL * stride;
    return (int32_t)std::max<int64_t>(0, per_f / 16 / 32 * 32);
  };
  int32_t FG = 8, NB = nb_for(8);
  if ((size_t)NB < 3 * nmax) {
    FG = 4;
    NB = nb_for(4);
  }
  if (NB < 64 || (size_t)NB * 3 < 2 * nmax) return;  // too few buckets: keep the other binning kernels
  std::vector<uint8_t> blob((size_t)F * 16 + (size_t)F * NB * 16 + (size_t)F * stride * 4, 0);
  const float nbm1 = (float)(NB - 1);
  for (int32_t f = 0; f < F; ++f) {
    const std::vector<float>& v = u[f];
    float* prm = reinterpret_cast<float*>(blob.data() + (size_t)f * 16);
    uint32_t* ent = reinterpret_cast<uint32_t*>(blob.data() + (size_t)F * 16 + (size_t)f * NB * 16);
    float* U = reinterpret_cast<float*>(blob.data() + (size_t)F * 16 + (size_t)F * NB * 16) + (size_t)f * stride;
    for (int32_t i = 0; i < stride; ++i) U[i] = i < (int32_t)v.size() ? v[i] : INFINITY;
    float lo = 0.f, iw = INFINITY;  // no threshold: every x -> bucket 0 (code 0)
    if (!v.empty()) {
      lo = v.front();
      const float span = v.back() - lo;
      iw = span > 0.f ? (float)NB / span : INFINITY;
      if (!(std::isfinite(lo) && std::isfinite(v.back()))) return;
    }
    prm[0] = lo;
    prm[1] = iw;
    std::vector<int32_t> cnt(NB, 0);
    int32_t prev = -1;
    for (float x : v) {
      float t = (x - lo) * iw;  // IEEE fp32, as the kernel (__fsub_rn, __fmul_rn)
      if (std::isnan(t)) t = 0.f;  // inf * 0 (single threshold): the kernel's fmaxf(NaN, 0) = 0
      t = std::fmin(std::fmax(t, 0.f), nbm1);
      const int32_t b = (int32_t)t;
      if (b < prev) return;  // monotone by construction; checked
      prev = b;
      if (++cnt[b] > 15) return;
    }
    int32_t run = 0;
    for (int32_t b = 0; b < NB; ++b) {
      uint32_t* e = ent + 4 * (size_t)b;
      e[0] = (uint32_t)run | ((uint32_t)cnt[b] << 16);
      for (int32_t j = 0; j < 3; ++j) {
        const float t = j < cnt[b] ? v[run + j] : INFINITY;
        std::memcpy(&e[1 + j], &t, 4);
      }
      run += cnt[b];
    }
  }
  out->bke_blob.swap(blob);
  out->bke_nb = NB;
  out->bke_stride = stride;
  out->bke_fg = FG;
}

static uint32_t code_of_threshold(const TravLayout& L, int32_t f, float t) {
  const std::vector<float>& v = L.bin_sorted[f];
  return (uint32_t)(std::lower_bound(v.begin(), v.end(), t) - v.begin());  // t is present: exact index
}

// Sparse (pointer) layout (§8(f3)): each tree in BFS order with the two
// children of a node adjacent, 16-byte records {threshold, feature |
// missing<<30 | leaf<<31, left-child index | leaf index, 0}, leaf values per
// tree.  Used for trees deeper than the heap layouts allow or so unbalanced
// that padding them to perfect trees would blow up (sklearn max_depth=None).
static void build_sparse_layout(const bridger_model_desc* d, const Exactness& ex, bool acc_int, TravLayout* out) {
  const int32_t T = d->n_trees, F = d->n_features, K = d->n_outputs;
  out->sparse = true;
  out->global_trees = true;
  out->codes = false;
  out->bin_table.clear();
  out->bin_sorted.clear();
  out->sparse_trees.assign(T, SparseTree{});
  out->sparse_nodes.clear();
  out->slot_tree.assign(T, 0);
  out->slot_leafid_off.assign(T, 0);
  out->leaf_ids.clear();
  std::vector<float> leaves;
  std::vector<std::pair<int32_t, int32_t>> q;
  for (int32_t t = 0; t < T; ++t) {
    const int64_t a = d->tree_offsets[t];
    SparseTree& st = out->sparse_trees[t];
    st.node_off = (int64_t)(out->sparse_nodes.size() / 4);
    st.leaf_off = (int64_t)leaves.size();
    st.leafid_off = (int64_t)out->leaf_ids.size();
    st.slot_tree = t;
    int32_t dmax = 0, n_leaf = 0;
    q.clear();
    q.push_back({0, 0});
    for (size_t i = 0; i < q.size(); ++i) {
      const int32_t n = q[i].first, dep = q[i].second;
      const int64_t g = a + n;
      uint32_t rec[4] = {0, 0, 0, 0};
      if (d->left[g] == -1) {
        rec[1] = 1u << 31;
        rec[2] = (uint32_t)n_leaf++;
        for (int32_t k = 0; k < K; ++k) {
          const float v = d->value[g * K + k];
          leaves.push_back(acc_int ? std::ldexp(v, -ex.q) : v);
        }
        out->leaf_ids.push_back(n);
        dmax = std::max(dmax, dep);
      } else {
        std::memcpy(&rec[0], &d->threshold[g], 4);
        rec[1] = (uint32_t)d->feature[g] | ((d->missing_left && d->missing_left[g]) ? (1u << 30) : 0u);
        rec[2] = (uint32_t)q.size();
        q.push_back({d->left[g], dep + 1});
        q.push_back({d->right[g], dep + 1});
      }
      out->sparse_nodes.insert(out->sparse_nodes.end(), rec, rec + 4);
    }
    st.depth = dmax;
    out->slot_leafid_off[t] = st.leafid_off;
    out->slot_tree[t] = t;
  }
  out->data.assign(reinterpret_cast<const uint8_t*>(leaves.data()),
                   reinterpret_cast<const uint8_t*>(leaves.data()) + leaves.size() * 4);
  out->data.resize((out->data.size() + 127) / 128 * 128 + 128, 0);
  TravChunk c{};
  c.offset = 0;
  c.bytes = (int32_t)std::min<size_t>(out->data.size(), INT32_MAX / 2);
  c.n_trees = T;
  c.depth = 0;
  c.leaf_offset = 0;
  c.first_slot = 0;
  out->chunks.assign(1, c);
  int32_t nb = 16;
  while (nb > 1 && nb * 256 * F > 200 * 1024) nb /= 2;
  out->n_warps = 16;
  out->group = 16 / nb;
  out->chunk_budget = 0;
  out->smem_bytes = nb * 256 * F + 1024 + trav_bar_bytes(nb) + trav_red_bytes(nb, 16 / nb, K);
}

bool build_trav_layout(const bridger_model_desc* d, const std::vector<int32_t>& depth,
                       const Exactness& ex, bool acc_int, int32_t sms, TravLayout* out, std::string* why) {
  const int32_t T = d->n_trees, F = d->n_features, K = d->n_outputs;
  {
    // deep or badly unbalanced trees -> sparse pointer layout
    int64_t orig = 0, padded = 0;
    int32_t dmax = 0;
    for (int32_t t = 0; t < T; ++t) {
      orig += d->tree_offsets[t + 1] - d->tree_offsets[t];
      dmax = std::max(dmax, depth[t]);
      padded += depth[t] > 30 ? ((int64_t)1 << 40) : ((int64_t)2 << depth[t]) - 1;
    }
    const char* env = std::getenv("BRIDGER_SPARSE");
    const bool sparse = env ? env[0] != '0' : (dmax > 14 || padded > 4 * orig + 4096);
    out->has_missing = d->missing_left != nullptr;
    out->use_cluster = false;
    if (sparse) {
      build_sparse_layout(d, ex, acc_int, out);
      return true;
    }
    out->sparse = false;
    out->sparse_trees.clear();
    out->sparse_nodes.clear();
  }
  out->has_missing = d->missing_left != nullptr;
  out->use_cluster = std::getenv("BRIDGER_CLUSTER") != nullptr;
  // coded nodes pay for the separate binning pass (~k search steps per input
  // value) when each input value is reused by enough node visits: measured on
  // B200 C2 (800 visits/row over 28 features) 0.478 -> 0.431 ms
  // and C3 (3000 over 90) 15.06 -> 14.25 ms with codes, so the default is codes
  // iff sum_t D_t >= 12 * F (and >= 64) and the search tables fit in shared
  // memory.  BRIDGER_CODES=0/1 forces either format.
  const char* codes_env = std::getenv("BRIDGER_CODES");
  int64_t visits = 0;
  for (int32_t t = 0; t < T; ++t) visits += std::max(1, depth[t]);
  bool want_codes = codes_env ? codes_env[0] != '0' : (visits >= 12 * (int64_t)F && visits >= 64);
  const bool codes_requested = want_codes;
  if (want_codes) {
    want_codes = build_bin_table(d, out);
    // (tables of any size: the binning kernel keeps all of them, or a group of
    // features' tables, in shared memory; one feature's is <= 128 KB)
  }
  std::vector<int32_t> order(T);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return depth[a] < depth[b]; });
  const int32_t Dmax = depth[order.back()];

  struct Run { int32_t start, n, D; };
  std::vector<Run> bal;
  int32_t budget = 0, nb = 16, nw = 16, G = 1, node_bytes = 8, xw = 0, misc = 0;

  // plan with a node format; false if one tree of the deepest class does not fit
  auto plan = [&](bool codes) -> bool {
    node_bytes = codes ? 4 : (out->split ? 5 : 8);
    // per 32-row block: codes mode = two u16 feature-major buffers (double
    // buffered, filled straight by bulk copy); fp32 mode = feature-major block
    // + dense staging block
    xw = codes ? 2 * code_buf_bytes(F) : 2 * 32 * F * 4;
    // 16 warps; NB = largest power of two with NB * xw <= the x budget below (measured on
    // B200: C2 best at NB=16/G=1, C3 at NB=4/G=4 in fp32 mode)
    nw = 16;
    nb = 16;
    // measured on B200: C3 codes (16 KB per group) best at NB=8 (12.59 vs 13.11
    // ms at NB=4), C5 shard codes (32 KB per group) best at NB=2 (14.6 vs 15.3)
    int32_t xbudget = (codes && xw <= 16 * 1024) ? 144 * 1024 : 120 * 1024;
    if (const char* e = std::getenv("BRIDGER_XBUDGET")) xbudget = 1024 * std::atoi(e);  // experiments
    while (nb > 1 && nb * xw > xbudget) nb /= 2;
    // wide coded inputs (>= 16 KB code blocks, C5-shaped): 12 warps, measured
    // on B200 with the K4d kernel (1250-tree shard, 1M rows: 7.94 ms vs 8.29 at
    // 16 and 8.47 at 8 warps; profiles/r2_deep_sweep.jsonl)
    if (codes && code_buf_bytes(F) >= 16 * 1024) nw = 12;
    if (const char* e = std::getenv("BRIDGER_WARPS")) nw = std::max(1, std::min(16, std::atoi(e)));  // experiments
    if (const char* e = std::getenv("BRIDGER_BLOCKS")) nb = std::max(1, std::min(16, std::atoi(e)));
    nb = std::min(nb, nw);
    while (nw % nb) --nb;
    G = nw / nb;
    misc = 1024 + trav_bar_bytes(nb) + trav_red_bytes(nb, G, K);
    const int32_t base_budget = kSmemMax - misc - trav_x_region(codes, F, nb);
    auto chunk_bytes = [&](int32_t n, int32_t D) -> int64_t {
      // codes: [pad word][I node words] per tree (2^D words, see the packing below)
      const int64_t nodes = codes ? (int64_t)n * (1 << D) * 4
                                  : (int64_t)n * ((1 << D) - 1) * node_bytes + (node_bytes == 5 ? 16 : 0);
      return (nodes + 31) / 32 * 32 + ((int64_t)n * (1 << D) * K * 4 + 15) / 16 * 16;
    };
    out->global_trees = false;
    int32_t n_prev = 1;
    for (int iter = 0; iter < 4; ++iter) {
      budget = base_budget - (out->use_cluster ? trav_slot_bytes(nb, n_prev, K) : 0);
      if (chunk_bytes(1, Dmax) > budget) {
        if (codes) return false;
        // global-tree mode: chunks are runs of equal depth of any size, read from
        // global memory by every CTA (no shared-memory residency, no partials)
        out->global_trees = true;
        budget = INT32_MAX / 2;
      }
      std::vector<Run> runs;
      int32_t s = 0;
      while (s < T) {
        int32_t Dc = depth[order[s]], n = 1;
        while (s + n < T) {
          const int32_t Dn = std::max(Dc, depth[order[s + n]]);
          if (out->global_trees ? (Dn != Dc || chunk_bytes(n + 1, Dn) > (1 << 30)) : (chunk_bytes(n + 1, Dn) > budget))
            break;
          Dc = Dn;
          ++n;
        }
        runs.push_back({s, n, Dc});
        s += n;
      }
      bal.clear();
      for (size_t i = 0; i < runs.size();) {
        size_t j = i;
        int32_t total = 0;
        while (j < runs.size() && runs[j].D == runs[i].D) total += runs[j++].n;
        int32_t nc = (int32_t)(j - i);
        // many chunks of one depth: round the count up to a multiple of the SM
        // count so the one-CTA-per-chunk grid fills every SM (C5-like models)
        if (!out->global_trees && sms > 0 && nc > sms / 2 && nc % sms != 0) {
          const int32_t nc2 = (nc + sms - 1) / sms * sms;
          if (nc2 <= total) nc = nc2;
        } else if (!out->global_trees && sms > 0 && sms % 2 == 0 && nc > sms / 4 && nc < sms / 2 && sms / 2 <= total) {
          // ... or up to half the SM count: two CTAs per chunk fill every SM
          // (C5 shard in codes: 70 chunks of 18 trees -> 74 x 2 CTAs = 148)
          nc = sms / 2;
        }
        int32_t st = runs[i].start;
        for (int32_t c = 0; c < nc; ++c) {
          const int32_t n = total / nc + (c < total % nc ? 1 : 0);
          bal.push_back({st, n, runs[i].D});
          st += n;
        }
        i = j;
      }
      if (out->global_trees || (int32_t)bal.size() <= n_prev) break;
      n_prev = (int32_t)bal.size();
    }
    return true;
  };
  {
    // split node arrays (fp32 thresholds + 1-byte features): opt-in until
    // measured better (BRIDGER_SPLIT=1); needs F <= 127 (bit 7 = missing_left)
    const char* env = std::getenv("BRIDGER_SPLIT");
    out->split = !want_codes && F <= 127 && env && env[0] == '1';
  }
  out->codes = want_codes && plan(true);
  // bucketed binning where it fits next to the cooperative kernel's staging
  // (two dense [32][F] fp32 blocks); BRIDGER_BUCKET=0 keeps the Eytzinger search
  {
    const char* be = std::getenv("BRIDGER_BUCKET");
    if (out->codes && !(be && be[0] == '0')) {
      build_bucket_table(F, out, 2 * 128 * F + 64);
      if (out->bkt_nb == 0) build_bucket_table(F, out, 0, 4);  // per-feature-group tables (wide inputs)
    } else {
      out->bkt_blob.clear();
      out->bkt_nb = 0;
    }
    out->bke_blob.clear();
    out->bke_nb = 0;
    if (out->codes && !(be && be[0] == '0')) build_entry_table(F, out);
  }
  if (!out->codes) {
    out->bin_table.clear();
    out->bin_sorted.clear();
    plan(false);
  }
  if (out->split && out->global_trees) {  // split nodes only for shared-memory-resident chunks
    out->split = false;
    plan(false);
  }
  out->hybrid = false;
  out->hyb_nodes.clear();
  out->hyb_leaves.clear();
  const char* hyb_env = std::getenv("BRIDGER_HYBRID");
  const bool uniform = depth[order.front()] == Dmax;
  // measured on B200: slower than global-tree mode for C4 at
  // every shared-memory split tried, so opt-in (BRIDGER_HYBRID=1)
  if (out->global_trees && uniform && Dmax >= 6 && hyb_env && hyb_env[0] == '1') {
    // Hybrid: the top `top` levels of a chunk of trees resident in shared
    // memory, deep levels + leaves in global memory; input pre-transposed.
    int64_t base_budget = kSmemMax - misc - (int64_t)nb * xw;
    if (const char* e = std::getenv("BRIDGER_HYB_BUDGET")) base_budget = std::min<int64_t>(base_budget, 1024LL * std::atoi(e));
    int32_t top = std::min(Dmax - 1, 11);
    int64_t n_fit = 0;
    for (; top >= 3; --top) {
      n_fit = base_budget / (((int64_t)1 << top) - 1) / 8;
      if (n_fit >= 32 || n_fit >= T) break;
    }
    if (top >= 3 && n_fit >= 1) {
      out->hybrid = true;
      out->global_trees = false;
      out->pretransposed = false;
      const int32_t It = (1 << top) - 1, I = (1 << Dmax) - 1, L = 1 << Dmax;
      int32_t nc = (int32_t)((T + n_fit - 1) / n_fit);
      if (sms > 0 && nc > sms / 2 && nc % sms != 0) nc = std::min<int32_t>(T, (nc + sms - 1) / sms * sms);
      out->chunks.clear();
      out->data.clear();
      out->slot_tree.assign(T, 0);
      out->slot_leafid_off.assign(T, 0);
      out->leaf_ids.clear();
      PaddedTree pt;
      int64_t off = 0;
      int32_t s0 = 0;
      for (int32_t ci = 0; ci < nc; ++ci) {
        const int32_t n = T / nc + (ci < T % nc ? 1 : 0);
        TravChunk c{};
        c.offset = off;
        c.n_trees = n;
        c.depth = Dmax;
        c.first_slot = s0;
        c.top_levels = top;
        c.g_nodes = (int64_t)s0 * (I - It);
        c.g_leaves = (int64_t)s0 * L * K;
        c.leaf_offset = 0;
        c.bytes = (int32_t)(((int64_t)n * It * 8 + 15) / 16 * 16);
        out->data.resize(off + c.bytes, 0);
        uint32_t* nd = reinterpret_cast<uint32_t*>(out->data.data() + off);
        for (int32_t j = 0; j < n; ++j) {
          const int32_t t = order[s0 + j];
          pad_tree(d, t, Dmax, &pt);
          for (int32_t i = 0; i < I; ++i) {
            uint32_t tb;
            std::memcpy(&tb, &pt.threshold[i], 4);
            const uint32_t fw = (uint32_t)pt.feature[i] | ((uint32_t)pt.missing[i] << 31);
            if (i < It) {
              nd[2 * ((size_t)j * It + i)] = tb;
              nd[2 * ((size_t)j * It + i) + 1] = fw;
            } else {
              out->hyb_nodes.push_back(tb);
              out->hyb_nodes.push_back(fw);
            }
          }
          for (int32_t l = 0; l < L * K; ++l)
            out->hyb_leaves.push_back(acc_int ? std::ldexp(pt.leaf_value[l], -ex.q) : pt.leaf_value[l]);
          out->slot_tree[s0 + j] = t;
          out->slot_leafid_off[s0 + j] = (int64_t)out->leaf_ids.size();
          out->leaf_ids.insert(out->leaf_ids.end(), pt.leaf_id.begin(), pt.leaf_id.end());
        }
        out->chunks.push_back(c);
        off += (c.bytes + 127) / 128 * 128;
        out->data.resize(off, 0);
        s0 += n;
      }
      out->n_warps = nw;
      out->group = G;
      out->chunk_budget = (int32_t)base_budget;
      int32_t maxc = 0;
      for (auto& c : out->chunks) maxc = std::max(maxc, c.bytes);
      out->smem_bytes = maxc + nb * xw + misc;
      return true;
    }
  }
  out->n_warps = nw;
  out->group = G;
  out->chunk_budget = budget;
  out->stream = false;
  out->stream_split = false;
  out->stream_slack = 0;
  if (out->global_trees && !out->sparse) {
    // Tree-streamed mode (traverse.cuh K4s): rows resident, node records of
    // chunks of <= 4 equal-depth trees streamed through a 3-slot ring; leaves
    // stay in global memory.  Default on (BRIDGER_STREAM=0 keeps the older
    // global-tree walker for comparison).
    const char* env = std::getenv("BRIDGER_STREAM");
    const bool want_stream = !(env && env[0] == '0');
    // streamed trees are stored with an 8-byte front pad ([pad][node 0..I-1],
    // 2^D * 8 bytes): the two children 2i+1, 2i+2 of every node then form one
    // 16-byte-aligned pair (one LDS.128 in the speculative walk).  With
    // F <= 127 the split format ([pad][thresholds] fp32 + [pad][features] u8,
    // 5 * 2^D bytes) lets two trees share a slot of a 2-slot ring, so every
    // thread walks two trees at once (BRIDGER_STREAM_SPLIT=0 keeps 8-byte nodes)
    // Threshold-bin codes for streamed trees (when the tables can be built:
    // <= 65534 distinct thresholds per feature, F <= 512): 4-byte node words,
    // u16 code blocks as the row tile (half the fp32 tile); BRIDGER_STREAM_CODES=0
    // keeps the fp32 formats
    const char* cenv = std::getenv("BRIDGER_STREAM_CODES");
    const bool scodes = codes_requested && F <= 512 && !(cenv && cenv[0] == '0') && build_bin_table(d, out);
    if (!scodes) {
      out->bin_table.clear();
      out->bin_sorted.clear();
    }
    const char* senv = std::getenv("BRIDGER_STREAM_SPLIT");
    const bool spl = !scodes && F <= 127 && !(senv && senv[0] == '0');
    auto tree_bytes = [&](int32_t D) -> int64_t {
      return scodes ? (((((int64_t)1 << D) - 1) * 4 + 15) / 16 * 16)
                    : spl ? ((((int64_t)5 << D) + 15) / 16 * 16) : ((int64_t)1 << D) * 8;
    };
    const int64_t tree_nodes = tree_bytes(Dmax);
    // codes: two trees per slot of a 3-slot ring; three per slot of a 2-slot
    // ring (BRIDGER_STREAM_W=3) measured slower on C4 (16.1 vs 14.1 ms)
    int32_t per_slot = (spl || scodes) ? 2 : 1;
    if (scodes) {
      if (const char* e = std::getenv("BRIDGER_STREAM_W")) per_slot = std::max(2, std::min(3, std::atoi(e)));
    }
    int32_t ns = (spl || per_slot == 3) ? 2 : 3;
    if (const char* e = std::getenv("BRIDGER_STREAM_NS")) ns = std::max(2, std::min(3, std::atoi(e)));
    // one slot = 64-byte chunk header + node records
    const int64_t stage = std::max<int64_t>(per_slot > 1 ? per_slot * tree_nodes : (tree_nodes + 15) / 16 * 16, 16384) + 64;
    std::vector<Run> pieces;
    int32_t min_n = INT32_MAX;
    for (const Run& r : bal) {
      const int64_t per = std::max<int64_t>(1, std::min<int64_t>(4, (stage - 64) / tree_bytes(r.D)));
      // pieces of `per` trees; a remainder of 1 behind a full piece is
      // rebalanced (3 + 1 -> 2 + 2) so that no chunk holds a single tree
      std::vector<int32_t> sizes;
      for (int32_t s0 = 0; s0 < r.n; s0 += (int32_t)per) sizes.push_back((int32_t)std::min<int64_t>(per, r.n - s0));
      if (sizes.size() >= 2 && sizes.back() == 1 && sizes[sizes.size() - 2] >= 3) {
        sizes[sizes.size() - 2] -= 1;
        sizes.back() += 1;
      }
      int32_t s0 = 0;
      for (int32_t sz : sizes) {
        pieces.push_back({r.start + s0, sz, r.D});
        min_n = std::min(min_n, sz);
        s0 += sz;
      }
    }
    // trees per pass (every chunk holds >= w)
    // (codes walk clamps chunks that hold fewer than w trees; the fp32 walks need >= w)
    const int32_t w = scodes ? per_slot : (min_n >= 2 && K <= 8) ? 2 : 1;
    // shared memory: X tile (32 rows per warp) + ring + per-thread leaf slots
    auto fits = [&](int32_t wp) {
      const int64_t landing = (int64_t)wp * 32 * w * K * 4;
      // split walk: the discarded last-level child loads read <= 3*2^D bytes
      // past a tree, i.e. into the landing slots after the ring; pad if short
      const int64_t slack = spl ? std::max<int64_t>(0, ((int64_t)3 << Dmax) + 64 - landing) : 0;
      const int64_t xtile = scodes ? (int64_t)(wp + 1) * code_buf_bytes(F) : (int64_t)wp * 32 * F * 4;
      return xtile + ns * stage + landing + slack + 1024 <= kSmemMax;
    };
    // walking warps: as many as fit, up to 20 (the kernel's launch bound:
    // more chains hide the shared-memory and leaf-gather latency; measured
    // on C4 codes: 16 warps 13.27 ms, 18 12.68, 20 12.21 per 1M rows)
    const int32_t max_warps = (scodes && K <= 8) ? 20 : 16;  // trav_stream_kernel's launch bound
    int32_t warps = max_warps;
    if (const char* e = std::getenv("BRIDGER_STREAM_WARPS")) warps = std::max(4, std::min(max_warps, std::atoi(e)));
    while (warps > 4 && !fits(warps)) --warps;
    if (want_stream && fits(warps)) {
      out->stream = true;
      out->stream_ns = ns;
      out->stream_stage = (int32_t)stage;
      out->stream_warps = warps;
      out->stream_w = w;
      out->stream_split = spl;
      out->codes = scodes;
      out->stream_slack = spl ? (int32_t)std::max<int64_t>(0, ((int64_t)3 << Dmax) + 64 - (int64_t)warps * 32 * w * K * 4) : 0;
      bal.swap(pieces);
    } else if (scodes) {
      out->bin_table.clear();
      out->bin_sorted.clear();
    }
  }
  {
    // wide inputs walked by many chunks: transpose X once into feature-major
    // blocks instead of once per chunk CTA (measured: C5-shaped models)
    const char* env = std::getenv("BRIDGER_PRET");
    const int64_t work = (int64_t)F * (int64_t)bal.size();
    out->pretransposed = !out->codes && !out->split && !out->global_trees && (env ? env[0] != '0' : work >= 1024);
  }
  out->chunks.clear();
  out->data.clear();
  out->slot_tree.assign(T, 0);
  out->slot_leafid_off.assign(T, 0);
  out->leaf_ids.clear();
  PaddedTree pt;
  int64_t off = 0;
  for (const Run& r : bal) {
    const int32_t D = r.D, I = (1 << D) - 1, L = 1 << D;
    TravChunk c{};
    c.offset = off;
    c.n_trees = r.n;
    c.depth = D;
    c.first_slot = r.start;
    const int64_t nodes = out->split ? (((int64_t)r.n * I * 4 + 15) / 16 * 16 + (int64_t)r.n * I)
                          : (out->stream && out->codes) ? (int64_t)r.n * (I + 1) * 4
                          : out->codes ? (int64_t)r.n * (I + 1) * 4
                          : out->stream ? (int64_t)r.n * (out->stream_split ? ((((int64_t)5 << D) + 15) / 16 * 16) : (int64_t)(I + 1) * 8)
                                        : (int64_t)r.n * I * node_bytes;
    c.leaf_offset = (int32_t)((nodes + 31) / 32 * 32);  // 32-byte aligned leaf vectors (256-bit gathers)
    c.bytes = (int32_t)(c.leaf_offset + ((int64_t)r.n * L * K * 4 + 15) / 16 * 16);
    out->data.resize(off + c.bytes, 0);
    uint8_t* base = out->data.data() + off;
    for (int32_t j = 0; j < r.n; ++j) {
      const int32_t t = order[r.start + j];
      pad_tree(d, t, D, &pt);
      if (out->codes) {
        // node word: code index j (bits 16..31) | byte offset of the feature's
        // code within a lane's view of a [F/2][32][2] u16 code block (bits
        // 1..14: (f/2)*128 + (f%2)*2, always even, F <= 512) | missing (bit 0).
        // Tree j at words [j (I + 1), (j + 1)(I + 1)): a pad word, then nodes
        // 0..I-1, so that the two children 2i+1, 2i+2 of every node form one
        // 8-byte-aligned pair (the speculative walks of trav_deep.cu and of
        // the tree-streamed kernel load both with one LDS.64).
        uint32_t* nd = reinterpret_cast<uint32_t*>(base) + (size_t)j * (I + 1) + 1;
        for (int32_t i = 0; i < I; ++i) {
          // real nodes: t is in U_f, exact index; dummy nodes under replicated
          // leaves (feature 0, threshold 0): any code routes to identical leaves
          const int32_t f = pt.feature[i];
          const uint32_t code = code_of_threshold(*out, f, pt.threshold[i]);
          const uint32_t foff = (uint32_t)(f >> 1) * 128u + (uint32_t)(f & 1) * 2u;
          nd[i] = (code << 16) | foff | (uint32_t)pt.missing[i];
        }
      } else if (out->split) {
        float* th = reinterpret_cast<float*>(base) + (size_t)j * I;
        uint8_t* fe = base + (((size_t)r.n * I * 4 + 15) / 16 * 16) + (size_t)j * I;
        for (int32_t i = 0; i < I; ++i) {
          th[i] = pt.threshold[i];
          fe[i] = (uint8_t)(pt.feature[i] | (pt.missing[i] << 7));
        }
      } else if (out->stream && out->stream_split) {
        // streamed split: tree j at j * tb: [pad][thr 0..I-1] fp32, [pad][feature | missing << 7] u8
        const size_t tb = (((size_t)5 << D) + 15) / 16 * 16;
        float* th = reinterpret_cast<float*>(base + (size_t)j * tb);
        uint8_t* fe = base + (size_t)j * tb + ((size_t)4 << D);
        for (int32_t i = 0; i < I; ++i) {
          th[1 + i] = pt.threshold[i];
          fe[1 + i] = (uint8_t)(pt.feature[i] | (pt.missing[i] << 7));
        }
      } else {
        // streamed: tree j at [(I + 1) j + 1] (front pad), else [I j]
        uint32_t* nd = reinterpret_cast<uint32_t*>(base) + (out->stream ? ((size_t)j * (I + 1) + 1) * 2 : (size_t)j * I * 2);
        for (int32_t i = 0; i < I; ++i) {
          uint32_t tb;
          std::memcpy(&tb, &pt.threshold[i], 4);
          nd[2 * i] = tb;
          nd[2 * i + 1] = (uint32_t)pt.feature[i] | ((uint32_t)pt.missing[i] << 31);
        }
      }
      float* lv = reinterpret_cast<float*>(base + c.leaf_offset) + (size_t)j * L * K;
      // v * 2^-q: an integer-valued float < 2^63 (exact: a power-of-two scale
      // of a 24-bit significand, done in double, which holds 2^-q for any q
      // of the int64 tiers; the product is an integer, never subnormal) --
      // one multiply instead of a std::ldexp call per leaf value (C4: 33M)
      const double sq = std::ldexp(1.0, -ex.q);
      for (int32_t l = 0; l < L * K; ++l) {
        const float v = pt.leaf_value[l];
        lv[l] = acc_int ? (float)((double)v * sq) : v;
      }
      out->slot_tree[r.start + j] = t;
      out->slot_leafid_off[r.start + j] = (int64_t)out->leaf_ids.size();
      out->leaf_ids.insert(out->leaf_ids.end(), pt.leaf_id.begin(), pt.leaf_id.end());
    }
    out->chunks.push_back(c);
    off += (c.bytes + 127) / 128 * 128;
    out->data.resize(off, 0);
  }
  int32_t maxc = 0;
  for (auto& c : out->chunks) maxc = std::max(maxc, c.bytes);
  out->smem_bytes = (maxc + 127) / 128 * 128 + trav_x_region(out->codes, F, out->n_warps / out->group) + misc;
  (void)why;
  return true;
}

}  // namespace bridger
