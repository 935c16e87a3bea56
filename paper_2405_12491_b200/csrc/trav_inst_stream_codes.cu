// Instantiations of the tree-streamed traversal kernel, threshold-bin codes (traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_STREAM_INSTANTIATE(long long, false, 2)
BRIDGER_STREAM_INSTANTIATE(long long, true, 2)
BRIDGER_STREAM_INSTANTIATE(double, false, 2)
BRIDGER_STREAM_INSTANTIATE(double, true, 2)
}  // namespace bridger
