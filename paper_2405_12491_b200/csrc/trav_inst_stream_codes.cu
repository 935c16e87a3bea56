// Instantiations of the tree-streamed traversal kernel, threshold-bin codes (traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_STREAM_INSTANTIATE(long long, false, 2)
BRIDGER_STREAM_INSTANTIATE(long long, true, 2)
BRIDGER_STREAM_INSTANTIATE(double, false, 2)
BRIDGER_STREAM_INSTANTIATE(double, true, 2)
// three trees per pass (codes only)
#define BRIDGER_STREAM_INSTANTIATE_W3(ACC, ML)                                                                \
  BRIDGER_STREAM_INSTANTIATE_W(ACC, ML, 3, 2)                                                                 \
  template cudaError_t launch_stream_t<1, ACC, ML, 3, true, 2>(const TravParams&, int, int, int, cudaStream_t);
BRIDGER_STREAM_INSTANTIATE_W3(long long, false)
BRIDGER_STREAM_INSTANTIATE_W3(long long, true)
BRIDGER_STREAM_INSTANTIATE_W3(double, false)
BRIDGER_STREAM_INSTANTIATE_W3(double, true)
}  // namespace bridger
