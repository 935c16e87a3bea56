// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(long long, false, true, 2)
BRIDGER_TRAV_INSTANTIATE(long long, true, true, 2)
BRIDGER_TRAV_INSTANTIATE(double, false, true, 2)
BRIDGER_TRAV_INSTANTIATE(double, true, true, 2)
}  // namespace bridger
