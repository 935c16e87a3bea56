// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(long long, true, false, false)
BRIDGER_TRAV_INSTANTIATE(long long, true, false, true)
}  // namespace bridger
