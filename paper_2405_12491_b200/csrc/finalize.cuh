// Steps a6/a7: turn the per-row accumulators of the
// per-tree reduction into the outputs.  Matches the definition the oracle
// writes out (reading c6, c7, c9, c10):
//   a   = acc * 2^q            (int64 fixed point -> fp64, exact under E53)
//   s   = MEAN ? a / T : base + leaf_scale * a     (fp64, explicit _rn: no FMA)
//   regression      -> (float) s
//   classification  -> label = argmax s (lowest index wins ties); K == 1: s > 0
//   proba           -> (float) s, or sigmoid for K == 1: [(float)(1-p), (float)p],
//                      or softmax (POST_SOFTMAX, reading c15)
#pragma once
#include <cstdint>

#include "bridger_internal.h"

namespace bridger {

template <typename ACC>
__device__ __forceinline__ double acc_to_double(ACC a, double scale_q);
template <>
__device__ __forceinline__ double acc_to_double<long long>(long long a, double scale_q) {
  return __dmul_rn(__ll2double_rn(a), scale_q);
}
template <>
__device__ __forceinline__ double acc_to_double<double>(double a, double) {
  return a;
}

template <int KT, typename ACC>
__device__ __forceinline__ void finalize_row(const FinalizeArgs& f, int64_t row, const ACC (&acc)[KT]) {
  const int K = f.K;
  if (f.want == 2) {
    ACC* o = static_cast<ACC*>(f.out) + row * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) o[k] = acc[k];
    return;
  }
  // 2^q built from its bit pattern (exact; the int64 tiers have q in
  // [-149, 127], always a normal double -- the F64 tier never uses it)
  const double scale_q = __longlong_as_double((long long)(f.q + 1023) << 52);
  double s[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k < K) {
      const double a = acc_to_double<ACC>(acc[k], scale_q);
      if (f.agg == BRIDGER_AGG_MEAN) {
        s[k] = __ddiv_rn(a, (double)f.total_trees);
      } else {
        const double b = f.base ? f.base[k] : 0.0;
        s[k] = __dadd_rn(b, __dmul_rn(f.leaf_scale, a));
      }
    } else {
      s[k] = 0.0;
    }
  }
  if (f.task == BRIDGER_TASK_REGRESSION) {
    float* o = static_cast<float*>(f.out) + row * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) o[k] = __double2float_rn(s[k]);
    return;
  }
  if (f.want == 0) {
    int32_t label = 0;
    if (K == 1) {
      label = s[0] > 0.0 ? 1 : 0;
    } else {
      double best = s[0];
#pragma unroll
      for (int k = 1; k < KT; ++k)
        if (k < K && s[k] > best) {
          best = s[k];
          label = k;
        }
    }
    static_cast<int32_t*>(f.out)[row] = label;
    return;
  }
  if (f.post == BRIDGER_POST_SOFTMAX) {  // reading c15: fp64, max-shifted
    double mx = s[0];
#pragma unroll
    for (int k = 1; k < KT; ++k)
      if (k < K && s[k] > mx) mx = s[k];
    double e[KT], z = 0.0;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      e[k] = k < K ? exp(s[k] - mx) : 0.0;
      z += e[k];
    }
    float* o = static_cast<float*>(f.out) + row * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) o[k] = __double2float_rn(e[k] / z);
  } else if (K == 1) {
    const double p = 1.0 / (1.0 + exp(-s[0]));
    float* o = static_cast<float*>(f.out) + row * 2;
    o[0] = __double2float_rn(1.0 - p);
    o[1] = __double2float_rn(p);
  } else {
    float* o = static_cast<float*>(f.out) + row * K;
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (k < K) o[k] = __double2float_rn(s[k]);
  }
}

// Dispatch a runtime K to the register-array capacity KT.
#define BRIDGER_DISPATCH_KT(K, ...)                     \
  do {                                                  \
    if ((K) <= 1) { constexpr int KT = 1; __VA_ARGS__; } \
    else if ((K) <= 2) { constexpr int KT = 2; __VA_ARGS__; } \
    else if ((K) <= 4) { constexpr int KT = 4; __VA_ARGS__; } \
    else if ((K) <= 8) { constexpr int KT = 8; __VA_ARGS__; } \
    else if ((K) <= 16) { constexpr int KT = 16; __VA_ARGS__; } \
    else { constexpr int KT = 64; __VA_ARGS__; }         \
  } while (0)

}  // namespace bridger
