// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(long long, false, false, 5)
BRIDGER_TRAV_INSTANTIATE(long long, true, false, 5)
BRIDGER_TRAV_INSTANTIATE(double, false, false, 5)
BRIDGER_TRAV_INSTANTIATE(double, true, false, 5)
}  // namespace bridger
