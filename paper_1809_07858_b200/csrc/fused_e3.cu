// Explicit instantiations of the fused width-4 kernel for E in [3, 11, 19, 27]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(3)
SB_INSTANTIATE_FUSED(11)
SB_INSTANTIATE_FUSED(19)
SB_INSTANTIATE_FUSED(27)
