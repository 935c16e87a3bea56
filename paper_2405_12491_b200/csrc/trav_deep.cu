// K4d dispatcher: picks the trav_deep_kernel instantiation (trav_deep.cuh;
// compiled in trav_deep_inst_*.cu) for K, missing-value routing, the fused
// scatter and the walk mode.
#include "trav_deep.cuh"

namespace bridger {

BRIDGER_DEEP_EXTERN_ALL()

template <int KT, bool ML>
static cudaError_t launch_deep_t(const TravParams& p, int wm, int grid, int block, int smem, cudaStream_t st) {
  if (p.scatter) return launch_deep_k<KT, ML, true, 0>(p, grid, block, smem, st);
  if constexpr (!ML && KT <= 8) {
    if (wm == 1) return launch_deep_k<KT, false, false, 1>(p, grid, block, smem, st);
  }
  return launch_deep_k<KT, ML, false, 0>(p, grid, block, smem, st);
}

// wm: the walk every chunk takes (traverse.cu deep_walk_mode), 0 if mixed
cudaError_t launch_trav_deep(const TravParams& p, int K, bool ml, int wm, int grid, int block, int smem,
                             cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  BRIDGER_DISPATCH_KT(K, { e = ml ? launch_deep_t<KT, true>(p, wm, grid, block, smem, st)
                                  : launch_deep_t<KT, false>(p, wm, grid, block, smem, st); });
  return e;
}

// shared memory of the deep kernel: chunk + alignment slack + NB x 2 buffers + barriers + counters
int trav_deep_smem(int chunk_cap, int code_buf, int nb) {
  return chunk_cap + code_buf + nb * 2 * code_buf + (1 + 2 * nb) * 8 + nb * 2 * 4;
}

}  // namespace bridger
