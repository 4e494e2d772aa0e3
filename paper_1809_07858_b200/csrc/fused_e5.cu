// Explicit instantiations of the fused width-4 kernel for E in [5, 13, 21, 29]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(5)
SB_INSTANTIATE_FUSED(13)
SB_INSTANTIATE_FUSED(21)
SB_INSTANTIATE_FUSED(29)
