// Explicit instantiations of the fused width-4 kernel for E in [0, 8, 16, 24]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(0)
SB_INSTANTIATE_FUSED(8)
SB_INSTANTIATE_FUSED(16)
SB_INSTANTIATE_FUSED(24)
