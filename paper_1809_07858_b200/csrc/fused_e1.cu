// Explicit instantiations of the fused width-4 kernel for E in [1, 9, 17, 25]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(1)
SB_INSTANTIATE_FUSED(9)
SB_INSTANTIATE_FUSED(17)
SB_INSTANTIATE_FUSED(25)
