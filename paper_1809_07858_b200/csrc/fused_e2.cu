// Explicit instantiations of the fused width-4 kernel for E in [2, 10, 18, 26]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(2)
SB_INSTANTIATE_FUSED(10)
SB_INSTANTIATE_FUSED(18)
SB_INSTANTIATE_FUSED(26)
