// Explicit instantiations of the K4d kernel launchers (trav_deep.cuh).
#include "trav_deep.cuh"

namespace bridger {
BRIDGER_DEEP_ALL_KT(, true, false, 0)
}  // namespace bridger
