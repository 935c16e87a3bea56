// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(double, false, false, false)
BRIDGER_TRAV_INSTANTIATE(double, true, false, false)
BRIDGER_TRAV_INSTANTIATE(double, false, false, true)
BRIDGER_TRAV_INSTANTIATE(double, true, false, true)
}  // namespace bridger
