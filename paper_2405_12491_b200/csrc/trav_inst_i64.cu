// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(long long, false, false, false)
BRIDGER_TRAV_INSTANTIATE(long long, false, false, true)
}  // namespace bridger
