// Linear models on the same GPU path (include/bridger.h
// "Linear models").  The definition is oracle.c oracle_linear_run:
//   x'_f = ((float)x_f - (float)mean_f) / (float)scale_f        (reading c16)
//   s_k  = intercept_k + sum_f coef[k][f] * x'_f  (fp64, f ascending, no FMA)
// then identity / sigmoid / softmax / argmax exactly as finalize.cuh does for
// tree ensembles (readings c7, c10, c15).
//
// B200 mapping: HBM-bound (4F bytes of input per row against K*F fp64 MACs).
// Persistent CTAs of W warps; each warp streams 32-row blocks of X through a
// double-buffered shared-memory staging block filled by cp.async (coalesced
// 16-, 8- or 4-byte copies, the widest F and X's alignment allow; row stride
// odd in copy vectors so that lane = row vector reads are conflict free)
// while it computes the previous block; the weights sit in shared memory
// and are read as warp-wide broadcasts.  fp64 arithmetic costs nothing here:
// the kernel is bound by the X stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <vector>

#include "bridger_internal.h"
#include "finalize.cuh"
#include "ptx.cuh"

struct bridger_linear {
  int device = 0;
  int32_t F = 0, K = 0, task = 0, post = 0;
  bool scaler = false;
  int sms = 148;
  // per staging width (vw = 4, 2, 1): occupancy of the kernel that width
  // selects, measured on first use (0 = not yet); the launch then makes no
  // attribute or occupancy queries
  mutable std::atomic<int> occ[3] = {0, 0, 0};
  double* d_w = nullptr;      // [F][K] coef (feature-major), then [K] intercept
  float* d_scale = nullptr;   // [2F] fp32 mean, scale (reading c16: cast to the input dtype)
};

namespace bridger {

void count_launch();
void hot_begin(cudaStream_t st, cudaEvent_t* ev);
void hot_end(cudaStream_t st, cudaEvent_t start);

struct LinParams {
  const float* X;
  int64_t n_rows;
  int32_t F, K, S;      // S = staging row stride (odd)
  const double* w;      // [F][K] coef (feature-major) then [K] intercept
  const float* sc;      // [2F] or nullptr
  int32_t want;         // 0 predict, 1 proba, 2 decision (fp64 scores)
  int32_t bulk;         // S == F and X 16-B aligned: whole blocks by one cp.async.bulk
  FinalizeArgs fin;     // task / post / K / out
};

template <int KT, bool SCALER, int VW, bool FULL>  // FULL: K == KT
__global__ void __launch_bounds__(512) linear_kernel(const LinParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  const int F = p.F, K = FULL ? KT : p.K, S = p.S;
  double* W = reinterpret_cast<double*>(smem);                 // [F][K] + [K]
  float* SC = reinterpret_cast<float*>(W + (((size_t)K * F + K + 1) & ~(size_t)1));  // [2F]
  float* St = SC + ((2 * F + 3) & ~3);                          // [NW][2][32*S], 16-B aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(St + (size_t)NW * 2 * 32 * S) + 2 * warp;  // [NW][2]
  if (lane == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < K * F + K; i += blockDim.x) W[i] = p.w[i];
  if (SCALER)
    for (int i = threadIdx.x; i < 2 * F; i += blockDim.x) SC[i] = p.sc[i];
  __syncthreads();
  float* st0 = St + (size_t)warp * 2 * 32 * S;
  const int64_t n_blocks = (p.n_rows + 31) / 32;
  const int64_t stride = (int64_t)gridDim.x * NW;
  int64_t blk = (int64_t)blockIdx.x * NW + warp;
  // The contiguous [rows][F] block is copied in VW-float vectors (VW = 4, 2
  // or 1: the largest that divides F and the alignment of X): vector e =
  // lane + 32 j goes to row e / FV, vector column e % FV of the staging block,
  // whose row stride S = VW * (FV | 1) is odd in vector units, so the lane =
  // row reads below are conflict free.  (row, column) advance incrementally
  // (32 = q FV + r): no division in the copy loop.  When FV is odd already
  // (S == F: F = 28, 90, ...) the staging block is the dense [32][F] block, so
  // whole blocks are fetched by one bulk copy (TMA engine, mbarrier) issued by
  // lane 0; the ragged tail block always takes the per-lane path.
  const int FV = F / VW, q = 32 / FV, r = 32 - q * FV;
  const int rr0 = lane / FV, c0 = lane - rr0 * FV;
  auto stage = [&](int64_t b, int buf) {
    if (b < n_blocks) {
      const int rows = (int)(p.n_rows - b * 32 < 32 ? p.n_rows - b * 32 : 32);
      const float* src = p.X + b * 32 * (int64_t)F;
      const uint32_t dst = ptx::s2u(st0 + (size_t)buf * 32 * S);
      if (p.bulk && rows == 32) {
        if (lane == 0) {
          ptx::fence_proxy_async();  // this warp's generic reads of the buffer precede the async write
          ptx::mbar_arrive_expect_tx(&bars[buf], 128u * (uint32_t)F);
          ptx::bulk_g2s(st0 + (size_t)buf * 32 * S, src, 128u * (uint32_t)F, &bars[buf]);
        }
      } else {
      int rr = rr0, c = c0;
      for (int e = lane; e < rows * FV; e += 32) {
        const uint32_t d = dst + (uint32_t)(rr * S + c * VW) * 4u;
        if constexpr (VW == 4)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + (size_t)e * 4) : "memory");
        else if constexpr (VW == 2)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + (size_t)e * 2) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + e) : "memory");
        rr += q;
        c += r;
        if (c >= FV) {
          c -= FV;
          ++rr;
        }
      }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(blk, 0);
  uint32_t phase = 0;  // bit b: parity of buffer b's mbarrier
  for (int buf = 0; blk < n_blocks; blk += stride, buf ^= 1) {
    stage(blk + stride, buf ^ 1);                                // next block in flight
    if (p.bulk && blk * 32 + 32 <= p.n_rows) {
      ptx::mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      asm volatile("cp.async.wait_group 1;" ::: "memory");      // this block landed
    }
    __syncwarp();
    const float* xr = st0 + (size_t)buf * 32 * S + lane * S;
    double acc[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) acc[k] = k < K ? W[(size_t)K * F + k] : 0.0;  // intercept
    for (int f0 = 0; f0 < F; f0 += VW) {
      float xs[4];
      if constexpr (VW == 4) {
        const float4 v = *reinterpret_cast<const float4*>(xr + f0);
        xs[0] = v.x, xs[1] = v.y, xs[2] = v.z, xs[3] = v.w;
      } else if constexpr (VW == 2) {
        const float2 v = *reinterpret_cast<const float2*>(xr + f0);
        xs[0] = v.x, xs[1] = v.y;
      } else {
        xs[0] = xr[f0];
      }
#pragma unroll
      for (int u = 0; u < VW; ++u) {  // features in ascending order
        const int f = f0 + u;
        float xv = xs[u];
        if (SCALER) xv = __fdiv_rn(__fsub_rn(xv, SC[f]), SC[F + f]);  // fp32 ops (c16)
        const double xd = (double)xv;
        const double* wf = W + f * K;  // the K weights of feature f: immediate offsets below
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (FULL || k < K) acc[k] = __dadd_rn(acc[k], __dmul_rn(wf[k], xd));  // no FMA
      }
    }
    const int64_t row = blk * 32 + lane;
    if (row < p.n_rows) {
      if (p.want == 2) {
        double* o = static_cast<double*>(p.fin.out) + row * K;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < K) o[k] = acc[k];
      } else {
        // the same finalize as the tree path: SUM with base 0, scale 1, q = 0
        finalize_row<KT, double>(p.fin, row, acc);
      }
    }
    __syncwarp();  // staging buffer `buf` is re-filled two blocks later
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

static bridger_status lin_cuda_fail(cudaError_t e, const char* what) {
  return fail(BRIDGER_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct LinDeviceGuard {
  int prev = -1;
  explicit LinDeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~LinDeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static bridger_status linear_run(const bridger_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                                 void* out, int want, void* stream) {
  if (!m) return fail(BRIDGER_E_NULL_ARG, "model is NULL");
  if (n_rows < 0) return fail(BRIDGER_E_SHAPE, "n_rows < 0");
  if (n_features != m->F)
    return fail(BRIDGER_E_SHAPE, "n_features " + std::to_string(n_features) + " != model's " + std::to_string(m->F));
  if (n_rows == 0) return BRIDGER_OK;
  if (!X || !out) return fail(BRIDGER_E_NULL_ARG, "X or out is NULL");
  if (n_rows > (int64_t)1 << 40 || n_rows * (int64_t)n_features > ((int64_t)1 << 46))
    return fail(BRIDGER_E_SHAPE, "n_rows * n_features overflows");
  if (want == 1 && m->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "predict_proba needs a classifier");
  LinDeviceGuard g(m->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LinParams p{};
  p.X = X;
  p.n_rows = n_rows;
  p.F = m->F;
  p.K = m->K;
  // vector width of the staging copies: the largest of 4, 2, 1 dividing F and
  // the alignment of X; staging row stride odd in vectors (conflict-free reads)
  int vw = 4;
  while (vw > 1 && (m->F % vw != 0 || reinterpret_cast<uintptr_t>(X) % (4u * vw) != 0)) vw >>= 1;
  p.S = vw * ((m->F / vw) | 1);
  p.w = m->d_w;
  p.sc = m->d_scale;
  p.want = want;
  p.bulk = p.S == m->F && reinterpret_cast<uintptr_t>(X) % 16 == 0;
  FinalizeArgs fin{};
  fin.task = m->task;
  fin.agg = BRIDGER_AGG_SUM;
  fin.post = m->post;
  fin.K = m->K;
  fin.total_trees = 1;
  fin.q = 0;
  fin.acc_int = 0;
  fin.want = want == 2 ? 0 : want;
  fin.leaf_scale = 1.0;
  fin.base = nullptr;
  fin.out = out;
  p.fin = fin;
  const size_t fixed = (((size_t)m->K * m->F + m->K + 1) & ~(size_t)1) * 8 + (size_t)((2 * m->F + 3) & ~3) * 4;
  const size_t per_warp = (size_t)2 * 32 * p.S * 4 + 16;  // two staging blocks + two mbarriers
  int nw = 16;
  while (nw > 1 && fixed + nw * per_warp > 232448) --nw;
  if (fixed + per_warp > 232448) return fail(BRIDGER_E_UNSUPPORTED, "model too wide for the linear kernel");
  const int smem = (int)(fixed + nw * per_warp);
  const int dev_sms = m->sms;
  const int64_t n_blocks = (n_rows + 31) / 32;
  // persistent: as many CTAs as fit (up to 4 per SM), never more than row blocks need
  cudaError_t e = cudaSuccess;
  BRIDGER_DISPATCH_KT(m->K, {
    const bool full = m->K == KT;
    auto pick = [&](auto f_full, auto f_part) { return full ? f_full : f_part; };
    auto kern = vw == 4 ? (m->scaler ? pick(linear_kernel<KT, true, 4, true>, linear_kernel<KT, true, 4, false>)
                                     : pick(linear_kernel<KT, false, 4, true>, linear_kernel<KT, false, 4, false>))
                : vw == 2 ? (m->scaler ? pick(linear_kernel<KT, true, 2, true>, linear_kernel<KT, true, 2, false>)
                                       : pick(linear_kernel<KT, false, 2, true>, linear_kernel<KT, false, 2, false>))
                          : (m->scaler ? pick(linear_kernel<KT, true, 1, true>, linear_kernel<KT, true, 1, false>)
                                       : pick(linear_kernel<KT, false, 1, true>, linear_kernel<KT, false, 1, false>));
    const int vi = vw == 4 ? 0 : vw == 2 ? 1 : 2;
    int occ = m->occ[vi].load(std::memory_order_relaxed);
    if (occ == 0) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nw * 32, smem);
      if (e == cudaSuccess) m->occ[vi].store(std::max(1, occ), std::memory_order_relaxed);
    }
    if (e == cudaSuccess) {
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_blocks + nw - 1) / nw,
                                                                   (int64_t)dev_sms * std::max(1, std::min(occ, 4))));
      cudaEvent_t ev;
      hot_begin(st, &ev);
      kern<<<grid, nw * 32, smem, st>>>(p);
      hot_end(st, ev);
      count_launch();
      e = cudaGetLastError();
    }
  });
  if (e != cudaSuccess) return lin_cuda_fail(e, "linear kernel launch");
  return BRIDGER_OK;
}

}  // namespace bridger

using namespace bridger;

extern "C" {

bridger_status bridger_linear_load(const bridger_linear_desc* d, int cuda_device, bridger_linear** out) {
  if (!out) return fail(BRIDGER_E_NULL_ARG, "out is NULL");
  *out = nullptr;
  if (!d || !d->coef) return fail(BRIDGER_E_NULL_ARG, "desc or coef is NULL");
  const int32_t F = d->n_features, K = d->n_outputs;
  if (F < 1) return fail(BRIDGER_E_SHAPE, "n_features must be >= 1");
  if (K < 1 || K > 64) return fail(BRIDGER_E_SHAPE, "n_outputs must be in [1,64]");
  if ((d->scaler_mean == nullptr) != (d->scaler_scale == nullptr))
    return fail(BRIDGER_E_SHAPE, "scaler_mean and scaler_scale must both be given or both NULL");
  if (d->task != BRIDGER_TASK_REGRESSION && d->task != BRIDGER_TASK_CLASSIFICATION)
    return fail(BRIDGER_E_UNSUPPORTED, "unknown task");
  if (d->post == BRIDGER_POST_SIGMOID && (d->task != BRIDGER_TASK_CLASSIFICATION || K != 1))
    return fail(BRIDGER_E_UNSUPPORTED, "sigmoid post-transform needs a K == 1 classifier");
  if (d->post == BRIDGER_POST_SOFTMAX && (d->task != BRIDGER_TASK_CLASSIFICATION || K < 2))
    return fail(BRIDGER_E_UNSUPPORTED, "softmax post-transform needs a K >= 2 classifier");
  if (d->post < BRIDGER_POST_IDENTITY || d->post > BRIDGER_POST_SOFTMAX)
    return fail(BRIDGER_E_UNSUPPORTED, "unknown post");
  std::vector<double> w((size_t)K * F + K, 0.0);
  for (size_t i = 0; i < (size_t)K * F; ++i) {
    if (!std::isfinite(d->coef[i])) return fail(BRIDGER_E_INVALID_TREE, "non-finite coefficient");
    w[(i % F) * K + i / F] = d->coef[i];  // feature-major: the kernel reads W[f][0..K)
  }
  for (int32_t k = 0; k < K; ++k) {
    const double b = d->intercept ? d->intercept[k] : 0.0;
    if (!std::isfinite(b)) return fail(BRIDGER_E_INVALID_TREE, "non-finite intercept");
    w[(size_t)K * F + k] = b;
  }
  std::vector<float> sc;
  if (d->scaler_mean) {
    sc.resize(2 * (size_t)F);
    for (int32_t f = 0; f < F; ++f) {
      sc[f] = (float)d->scaler_mean[f];   // reading c16: the transform runs in the input dtype
      sc[F + f] = (float)d->scaler_scale[f];
      if (!std::isfinite(sc[f]) || !std::isfinite(sc[F + f]) || sc[F + f] == 0.0f)
        return fail(BRIDGER_E_INVALID_TREE, "scaler mean/scale not finite or scale == 0");
    }
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return lin_cuda_fail(e, "cudaGetDeviceCount");
  if (cuda_device < 0 || cuda_device >= ndev) return fail(BRIDGER_E_CUDA, "invalid cuda_device");
  LinDeviceGuard g(cuda_device);
  bridger_linear* m = new bridger_linear();
  m->device = cuda_device;
  m->F = F;
  m->K = K;
  m->task = d->task;
  m->post = d->post;
  m->scaler = !sc.empty();
  cudaDeviceGetAttribute(&m->sms, cudaDevAttrMultiProcessorCount, cuda_device);
  e = cudaMalloc(&m->d_w, w.size() * 8);
  if (e == cudaSuccess) e = cudaMemcpy(m->d_w, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && m->scaler) {
    e = cudaMalloc(&m->d_scale, sc.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(m->d_scale, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(m->d_w);
    cudaFree(m->d_scale);
    delete m;
    return e == cudaErrorMemoryAllocation ? fail(BRIDGER_E_OOM, "device allocation failed")
                                          : lin_cuda_fail(e, "linear upload");
  }
  *out = m;
  return BRIDGER_OK;
}

bridger_status bridger_linear_free(bridger_linear* m) {
  if (!m) return BRIDGER_OK;
  LinDeviceGuard g(m->device);
  cudaDeviceSynchronize();
  cudaFree(m->d_w);
  cudaFree(m->d_scale);
  delete m;
  return BRIDGER_OK;
}

bridger_status bridger_linear_predict(const bridger_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                                      void* out, void* stream) {
  return linear_run(m, X, n_rows, n_features, out, 0, stream);
}

bridger_status bridger_linear_predict_proba(const bridger_linear* m, const float* X, int64_t n_rows,
                                            int32_t n_features, float* out, void* stream) {
  return linear_run(m, X, n_rows, n_features, out, 1, stream);
}

bridger_status bridger_linear_decision(const bridger_linear* m, const float* X, int64_t n_rows, int32_t n_features,
                                       double* out, void* stream) {
  return linear_run(m, X, n_rows, n_features, out, 2, stream);
}

}  // extern "C"
