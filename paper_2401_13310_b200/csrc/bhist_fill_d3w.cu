// Fill-kernel instantiations for DIM = 3, weighted fills (see bhist_launch.cuh).
#define BH_FILL_TU
#include "bhist_launch.cuh"

namespace bh {
BH_DEFINE_FILL_TU(3, true)
}  // namespace bh
