// Instantiations of the tree-streamed traversal kernel (traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_STREAM_INSTANTIATE(long long, false)
BRIDGER_STREAM_INSTANTIATE(long long, true)
BRIDGER_STREAM_INSTANTIATE(double, false)
BRIDGER_STREAM_INSTANTIATE(double, true)
}  // namespace bridger
