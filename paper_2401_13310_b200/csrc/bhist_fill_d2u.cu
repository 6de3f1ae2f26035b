// Fill-kernel instantiations for DIM = 2, unit fills (see bhist_launch.cuh).
#define BH_FILL_TU
#include "bhist_launch.cuh"

namespace bh {
BH_DEFINE_FILL_TU(2, false)
}  // namespace bh
