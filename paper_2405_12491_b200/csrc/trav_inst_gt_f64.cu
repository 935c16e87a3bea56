// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(double, false, true, 0)
BRIDGER_TRAV_INSTANTIATE(double, true, true, 0)
}  // namespace bridger
