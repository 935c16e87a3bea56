// Explicit instantiations of the traversal kernel (see traverse.cuh).
#include "traverse.cuh"

namespace bridger {
BRIDGER_TRAV_INSTANTIATE(double, false, true, false)
BRIDGER_TRAV_INSTANTIATE(double, true, true, false)
}  // namespace bridger
