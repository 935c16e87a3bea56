// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(long long, true, false, 0)
BRIDGER_TRAV_INSTANTIATE(long long, true, false, 1)
BRIDGER_TRAV_INSTANTIATE(long long, true, false, 3)
}  // namespace bridger
