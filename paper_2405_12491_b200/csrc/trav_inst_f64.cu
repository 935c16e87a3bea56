// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(double, false, false, 0)
BRIDGER_TRAV_INSTANTIATE(double, true, false, 0)
BRIDGER_TRAV_INSTANTIATE(double, false, false, 1)
BRIDGER_TRAV_INSTANTIATE(double, true, false, 1)
BRIDGER_TRAV_INSTANTIATE(double, false, false, 3)
BRIDGER_TRAV_INSTANTIATE(double, true, false, 3)
}  // namespace bridger
