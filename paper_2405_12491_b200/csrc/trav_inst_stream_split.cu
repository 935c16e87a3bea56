// Instantiations of the tree-streamed traversal kernel, split node format (traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_STREAM_INSTANTIATE(long long, false, true)
BRIDGER_STREAM_INSTANTIATE(long long, true, true)
BRIDGER_STREAM_INSTANTIATE(double, false, true)
BRIDGER_STREAM_INSTANTIATE(double, true, true)
}  // namespace bridger
