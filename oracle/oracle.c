/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  A plain, slow, obviously correct CPU
 * node-by-node tree-ensemble walker.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or layout with the CUDA path (paper_2405_12491_b200/):
 * it reads the ORIGINAL (unpadded) node arrays and walks them pointer by pointer.
 *
 * What it computes is the definition the paper's operator form reaches exactly
 * (SURVEY.md §8(c)): trees are combinations of comparison, conditional,
 * assignment and aggregation operators (COR, §4.2); the tree
 * template is SPEC.md:283 (loop: f = gather(feature, node); t = gather(threshold,
 * node); branch; node = where(...); out = gather(leaf_values, node)).
 *
 *   for each row r:
 *     acc[0..K) = 0.0 (double)
 *     for t in 0..T-1 (tree order):                 aggregation
 *       n = 0
 *       while left_t[n] != -1:                       loop, Table 4
 *         x = X[r, feature_t[n]]                     gather
 *         go_left = isnan(x) ? (missing_left ? missing_left_t[n] : 0)
 *                            : (x <= threshold_t[n]) less_equal, PAPER.md:576 (readings c1, c2)
 *         n = go_left ? left_t[n] : right_t[n]       where
 *       leaf[r,t] = n
 *       acc[k] += (double) value_t[n*K + k]         sum, fp64 accumulation SPEC.md:167,243
 *     s[k] = agg == MEAN ? acc[k] / T : base[k] + leaf_scale * acc[k]     (reading c6)
 *     regression:        pred[r,k] = (float) s[k]
 *     classif. K >= 2:   label = smallest k maximising s[k]; proba = (float) s
 *     classif. K == 1:   p = 1/(1+exp(-s0)); label = (s0 > 0) (reading c7);
 *                        proba = [(float)(1-p), (float)p]
 *     post == SOFTMAX:   proba[k] = (float)(exp(s[k] - max s) / sum_j exp(s[j] - max s))
 *                        (exp / divide, Table 4; reading c15)
 *
 * Multiclass boosting (reading c15, sklearn _gradient_boosting.pyx
 * predict_stages: out[i, k] += scale * tree[stage, k](x)): when tree_output is
 * given, every tree has ONE scalar value per node (value[n_nodes]) and adds it
 * to output tree_output[t] only:  acc[tree_output[t]] += (double) value_t[n].
 *
 * Built with -O2 -ffp-contract=off and no fast-math: no FMA contraction of
 * base + scale*acc, IEEE compares (reading c3).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n_trees, n_features, n_outputs;
  const int64_t* tree_offsets;   /* [n_trees+1] */
  const int32_t* feature;        /* [n_nodes] */
  const float*   threshold;      /* [n_nodes] */
  const int32_t* left;           /* [n_nodes] tree-local, -1 at leaves */
  const int32_t* right;          /* [n_nodes] */
  const float*   value;          /* [n_nodes * n_outputs] */
  const uint8_t* missing_left;   /* [n_nodes] or NULL */
  int32_t task;                  /* 0 regression, 1 classification */
  int32_t agg;                   /* 0 MEAN, 1 SUM */
  int32_t post;                  /* 0 identity, 1 sigmoid */
  const double* base_score;      /* [n_outputs] or NULL */
  double leaf_scale;
  const int32_t* tree_output;    /* [n_trees] or NULL (then value is [n_nodes * n_outputs]) */
} oracle_model;

typedef struct {
  const oracle_model* m;
  const float* X;
  int64_t r0, r1;
  int32_t F;
  int32_t* leaf; double* acc; double* s; int32_t* label; float* proba; float* pred;
  int err;
} job_t;

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  const oracle_model* m = j->m;
  const int32_t T = m->n_trees, K = m->n_outputs;
  double a[64];
  for (int64_t r = j->r0; r < j->r1; ++r) {
    const float* x = j->X + r * (int64_t)j->F;
    for (int k = 0; k < K; ++k) a[k] = 0.0;
    for (int32_t t = 0; t < T; ++t) {
      const int64_t base = m->tree_offsets[t];
      const int64_t size = m->tree_offsets[t + 1] - base;
      int64_t n = 0, steps = 0;
      while (m->left[base + n] != -1) {
        const float xv = x[m->feature[base + n]];
        int go_left;
        if (isnan(xv)) go_left = m->missing_left ? (m->missing_left[base + n] != 0) : 0;
        else           go_left = (xv <= m->threshold[base + n]);
        n = go_left ? m->left[base + n] : m->right[base + n];
        if (n < 0 || n >= size || ++steps > size) { j->err = 1; return NULL; }
      }
      if (j->leaf) j->leaf[r * T + t] = (int32_t)n;
      if (m->tree_output) a[m->tree_output[t]] += (double)m->value[base + n];
      else for (int k = 0; k < K; ++k) a[k] += (double)m->value[(base + n) * K + k];
    }
    if (j->acc) for (int k = 0; k < K; ++k) j->acc[r * K + k] = a[k];
    double s[64];
    for (int k = 0; k < K; ++k) {
      if (m->agg == 0) s[k] = a[k] / (double)T;
      else {
        const double prod = m->leaf_scale * a[k];
        s[k] = (m->base_score ? m->base_score[k] : 0.0) + prod;
      }
    }
    if (j->s) for (int k = 0; k < K; ++k) j->s[r * K + k] = s[k];
    if (m->task == 0) {
      if (j->pred) for (int k = 0; k < K; ++k) j->pred[r * K + k] = (float)s[k];
    } else if (K == 1) {
      if (j->label) j->label[r] = s[0] > 0.0 ? 1 : 0;
      if (j->proba) {
        const double p = 1.0 / (1.0 + exp(-s[0]));
        j->proba[r * 2 + 0] = (float)(1.0 - p);
        j->proba[r * 2 + 1] = (float)p;
      }
    } else {
      if (j->label) {
        int best = 0;
        for (int k = 1; k < K; ++k) if (s[k] > s[best]) best = k;
        j->label[r] = best;
      }
      if (j->proba && m->post == 2) {
        double mx = s[0], e[64], z = 0.0;
        for (int k = 1; k < K; ++k) if (s[k] > mx) mx = s[k];
        for (int k = 0; k < K; ++k) { e[k] = exp(s[k] - mx); z += e[k]; }
        for (int k = 0; k < K; ++k) j->proba[r * K + k] = (float)(e[k] / z);
      } else if (j->proba) {
        for (int k = 0; k < K; ++k) j->proba[r * K + k] = (float)s[k];
      }
    }
  }
  return NULL;
}

/* Returns 0 on success, 1 on a malformed tree (walk left its node range), 2 on
 * bad arguments.  Every output pointer may be NULL. */
int oracle_run(const oracle_model* m, const float* X, int64_t n_rows, int32_t n_features,
               int n_threads, int32_t* leaf, double* acc, double* s, int32_t* label,
               float* proba, float* pred) {
  if (!m || (!X && n_rows > 0) || n_features != m->n_features || m->n_outputs < 1 ||
      m->n_outputs > 64 || m->n_trees < 1)
    return 2;
  if (m->tree_output)
    for (int32_t t = 0; t < m->n_trees; ++t)
      if (m->tree_output[t] < 0 || m->tree_output[t] >= m->n_outputs) return 2;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n_rows) n_threads = n_rows > 0 ? (int)n_rows : 1;
  job_t* jobs = (job_t*)calloc((size_t)n_threads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
  for (int i = 0; i < n_threads; ++i) {
    job_t* j = &jobs[i];
    j->m = m; j->X = X; j->F = n_features;
    j->r0 = n_rows * i / n_threads; j->r1 = n_rows * (i + 1) / n_threads;
    j->leaf = leaf; j->acc = acc; j->s = s; j->label = label; j->proba = proba; j->pred = pred;
  }
  for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, run_rows, &jobs[i]);
  run_rows(&jobs[0]);
  for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
  int err = 0;
  for (int i = 0; i < n_threads; ++i) err |= jobs[i].err;
  free(jobs); free(th);
  return err ? 1 : 0;
}

/* ------------------------------------------------------------------------ *
 * Linear models (the paper's other GPU-evaluated CML models,
 * PAPER.md:800-801, 861-862; LogisticRegression / SGDClassifier / LinearRegression
 * / Ridge, optionally behind a StandardScaler).  Plain definition, fp64:
 *
 *   scaler (optional, reading c16 = sklearn 1.9 StandardScaler.transform on an
 *   fp32 X: X -= mean_.astype(float32); X /= scale_.astype(float32)):
 *     x'_f = ((float)x_f - (float)mean_f) / (float)scale_f      (fp32 ops)
 *   s_k = intercept_k + sum_{f = 0..F-1} coef[k][f] * x'_f     (fp64, f in order,
 *                                                                no FMA)
 *   regression:   pred[k] = (float) s_k
 *   classif K==1: label = (s_0 > 0); proba = sigmoid (reading c7, c10)
 *   classif K>=2: label = smallest k maximising s_k; proba = softmax (c15)
 *                 (post = IDENTITY: proba = (float) s_k)
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t n_features, n_outputs;
  const double* coef;       /* [K][F] */
  const double* intercept;  /* [K] or NULL */
  const double* mean;       /* [F] or NULL (no scaler) */
  const double* scale;      /* [F] or NULL */
  int32_t task, post;
} oracle_linear;

int oracle_linear_run(const oracle_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                      double* s_out, int32_t* label, float* proba, float* pred) {
  if (!m || n_features != m->n_features || m->n_outputs < 1 || m->n_outputs > 64) return 2;
  const int32_t F = m->n_features, K = m->n_outputs;
  for (int64_t r = 0; r < n_rows; ++r) {
    const float* x = X + r * (int64_t)F;
    double s[64];
    for (int k = 0; k < K; ++k) {
      double acc = m->intercept ? m->intercept[k] : 0.0;
      for (int f = 0; f < F; ++f) {
        float xv = x[f];
        if (m->mean) {
          const float m32 = (float)m->mean[f], s32 = (float)m->scale[f];
          const float c = xv - m32;  /* fp32 subtract (FLT_EVAL_METHOD 0) */
          xv = c / s32;              /* fp32 divide */
        }
        const double prod = m->coef[(int64_t)k * F + f] * (double)xv;
        acc = acc + prod;
      }
      s[k] = acc;
      if (s_out) s_out[r * K + k] = acc;
    }
    if (m->task == 0) {
      if (pred) for (int k = 0; k < K; ++k) pred[r * K + k] = (float)s[k];
    } else if (K == 1) {
      if (label) label[r] = s[0] > 0.0 ? 1 : 0;
      if (proba) {
        const double p = 1.0 / (1.0 + exp(-s[0]));
        proba[r * 2 + 0] = (float)(1.0 - p);
        proba[r * 2 + 1] = (float)p;
      }
    } else {
      if (label) {
        int best = 0;
        for (int k = 1; k < K; ++k) if (s[k] > s[best]) best = k;
        label[r] = best;
      }
      if (proba) {
        if (m->post == 2) {
          double mx = s[0], e[64], z = 0.0;
          for (int k = 1; k < K; ++k) if (s[k] > mx) mx = s[k];
          for (int k = 0; k < K; ++k) { e[k] = exp(s[k] - mx); z += e[k]; }
          for (int k = 0; k < K; ++k) proba[r * K + k] = (float)(e[k] / z);
        } else {
          for (int k = 0; k < K; ++k) proba[r * K + k] = (float)s[k];
        }
      }
    }
  }
  return 0;
}
