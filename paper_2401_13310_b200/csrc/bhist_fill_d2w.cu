// Fill-kernel instantiations for DIM = 2, weighted fills (see bhist_launch.cuh).
#define BH_FILL_TU
#include "bhist_launch.cuh"

namespace bh {
BH_DEFINE_FILL_TU(2, true)
}  // namespace bh
