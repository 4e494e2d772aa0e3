// Explicit instantiations of the fused width-4 kernel for E in [7, 15, 23, 31]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(7)
SB_INSTANTIATE_FUSED(15)
SB_INSTANTIATE_FUSED(23)
SB_INSTANTIATE_FUSED(31)
