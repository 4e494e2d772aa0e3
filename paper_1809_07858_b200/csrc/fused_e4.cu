// Explicit instantiations of the fused width-4 kernel for E in [4, 12, 20, 28]
// (split across units so they compile in parallel).
#include "fused.cuh"

SB_INSTANTIATE_FUSED(4)
SB_INSTANTIATE_FUSED(12)
SB_INSTANTIATE_FUSED(20)
SB_INSTANTIATE_FUSED(28)
