// Instantiations of the blocked any-width search (wsearch.cuh) and its launcher.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "wsearch.cuh"

namespace sb {

namespace {

template <int W, int NC>
cudaError_t launch_w(const FilterArgs& a, cudaStream_t s) {
    const long long ngroups = (a.n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + 127) / 128);
    shouji_wsearch<W, NC><<<grid, 128, 0, s>>>(a.planes, a.n, a.m, static_cast<int>(a.e), a.accept,
                                               a.estimates, a.outplanes, a.nflags);
    count_launch();
    return cudaGetLastError();
}

template <int NC>
cudaError_t launch_nc(const FilterArgs& a, cudaStream_t s) {
    switch (a.width) {
        case 3: return launch_w<3, NC>(a, s);
        case 4: return launch_w<4, NC>(a, s);
        case 5: return launch_w<5, NC>(a, s);
        case 6: return launch_w<6, NC>(a, s);
        case 7: return launch_w<7, NC>(a, s);
        case 8: return launch_w<8, NC>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

bool wsearch_applies(const FilterArgs& a) { return a.m <= 4095 && a.width >= 3 && a.width <= 8; }

cudaError_t launch_wsearch(const FilterArgs& a, cudaStream_t s) {
    return a.m <= 255 ? launch_nc<8>(a, s) : launch_nc<12>(a, s);
}

}  // namespace sb
