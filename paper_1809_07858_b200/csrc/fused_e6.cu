// Explicit instantiations of the fused width-4 kernel for E in [6, 14, 22, 30]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(6)
SB_INSTANTIATE_FUSED(14)
SB_INSTANTIATE_FUSED(22)
SB_INSTANTIATE_FUSED(30)
