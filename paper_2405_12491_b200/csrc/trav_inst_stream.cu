// Instantiations of the tree-streamed traversal kernel (traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_STREAM_INSTANTIATE(long long, false, false)
BRIDGER_STREAM_INSTANTIATE(long long, true, false)
BRIDGER_STREAM_INSTANTIATE(double, false, false)
BRIDGER_STREAM_INSTANTIATE(double, true, false)
}  // namespace bridger
