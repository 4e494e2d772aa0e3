// Stage 1: ASCII records -> pair-sliced planes (see pack.cuh for the layout).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"

namespace sb {

namespace {

// One CTA per tile of GROUPS x 32 pairs (pack_one_tile, pack_tile.cuh).
template <int GROUPS, int ALIGN, bool NIB>
__global__ void __launch_bounds__(kPackNT)
pack_tile_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                 size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ err_flag) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    const uint32_t err = pack_one_tile<ALIGN, kPackNT, NIB>(
        sm, &bar, 0, GROUPS, static_cast<long long>(blockIdx.x) * GROUPS, text, pattern, pitch, n, m,
        planes);
    if (!NIB && err) atomicOr(err_flag, 1u);
}

// Long records (tile does not fit in shared memory): each thread gathers one
// (group, chunk, sequence) tile straight from global memory.
__global__ void __launch_bounds__(kPackNT)
pack_direct_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                   size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                   uint32_t* __restrict__ err_flag) {
    const long long ngroups = (n + 31) / 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const int C = (mc + CH - 1) / CH;
    const long long items = 2 * ngroups * C;
    const long long it = static_cast<long long>(blockIdx.x) * kPackNT + threadIdx.x;
    if (it >= items) return;
    const int c = static_cast<int>(it % C);
    const long long g = (it / C) % ngroups;
    const int s = static_cast<int>(it / (C * ngroups));
    uint32_t sink[CH * 3];
    uint32_t* dst = planes ? planes + plane_index(s, g, c * CH, 0, nblocks, mc) : sink;
    const int stride = planes ? kPackGroups : 1;
    const uint32_t err = produce_chunk(s == 0 ? text : pattern, pitch, g * 32, n, c, m, dst, stride);
    if (err) atomicOr(err_flag, 1u);
}

}  // namespace

template <int GROUPS, int ALIGN, bool NIB = false>
static cudaError_t launch_tile(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                               long long n, int m, uint32_t* planes, uint32_t* err_flag,
                               cudaStream_t s) {
    const cudaError_t st = ensure_smem_attr<pack_tile_kernel<GROUPS, ALIGN, NIB>>(110 * 1024);
    if (st != cudaSuccess) return st;
    const long long ngroups = (n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + GROUPS - 1) / GROUPS);
    pack_tile_kernel<GROUPS, ALIGN, NIB><<<grid, kPackNT, tile_smem(pitch, GROUPS), s>>>(
        text, pattern, pitch, n, m, planes, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                        int m, uint32_t* planes, uint32_t* err_flag, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (pitch % 4 != 0) return cudaErrorInvalidValue;
    const int groups = tile_groups(pitch);
    const size_t smem = tile_smem(pitch, groups);
    cudaError_t st;
    if (smem <= 110 * 1024) {
        const bool a16 = pitch % 16 == 0;
        if (groups == 8)
            st = a16 ? launch_tile<8, 16>(text, pattern, pitch, n, m, planes, err_flag, s)
                     : launch_tile<8, 4>(text, pattern, pitch, n, m, planes, err_flag, s);
        else
            st = a16 ? launch_tile<4, 16>(text, pattern, pitch, n, m, planes, err_flag, s)
                     : launch_tile<4, 4>(text, pattern, pitch, n, m, planes, err_flag, s);
    } else {
        const long long items = 2 * ((n + 31) / 32) * ((plane_cols(m) + CH - 1) / CH);
        pack_direct_kernel<<<static_cast<unsigned>((items + kPackNT - 1) / kPackNT), kPackNT, 0,
                             s>>>(text, pattern, pitch, n, m, planes, err_flag);
        st = cudaGetLastError();
    }
    count_launch();
    return st;
}

bool nibble_pack_fits(int m) {
    const size_t np = nibble_pitch(m);
    return tile_smem(np, tile_groups(np)) <= 110 * 1024;
}

cudaError_t launch_pack_nibbles(const uint8_t* text, const uint8_t* pattern, long long n, int m,
                                uint32_t* planes, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!nibble_pack_fits(m) || planes == nullptr) return cudaErrorInvalidValue;
    const size_t np = nibble_pitch(m);
    const cudaError_t st = tile_groups(np) == 8
                               ? launch_tile<8, 4, true>(text, pattern, np, n, m, planes, nullptr, s)
                               : launch_tile<4, 4, true>(text, pattern, np, n, m, planes, nullptr, s);
    count_launch();
    return st;
}

// ---- dibit records (host-packed upload format, pack.cuh) ---------------------------
namespace {

// One CTA per pair block (8 groups): a bulk copy per sequence brings the
// block's dibit rows (and, for chunks with N, its N-plane rows) into shared
// memory, then each thread gathers one (chunk, group, sequence) item.
template <bool HAS_N>
__global__ void __launch_bounds__(kPackNT)
pack_dibit_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                  const uint8_t* __restrict__ ntext, const uint8_t* __restrict__ npattern,
                  long long n, int m, uint32_t* __restrict__ planes) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const int dp = static_cast<int>(dibit_pitch(m));
    const int np = static_cast<int>(nplane_pitch(m));
    const long long row0 = static_cast<long long>(blockIdx.x) * kPackPairs;
    const int rows = static_cast<int>(n - row0 < kPackPairs ? n - row0 : kPackPairs);
    uint8_t* dib[2] = {sm, sm + kPackPairs * dp};
    uint8_t* nrow[2] = {sm + 2 * kPackPairs * dp, sm + 2 * kPackPairs * dp + kPackPairs * np};
    const uint32_t dbytes = static_cast<uint32_t>(rows * dp), dbulk = dbytes & ~15u;
    const uint32_t nbytes = static_cast<uint32_t>(rows * np), nbulk = nbytes & ~15u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, 2 * dbulk + (HAS_N ? 2 * nbulk : 0u));
        for (int s = 0; s < 2; ++s) {
            if (dbulk) bulk_g2s(dib[s], (s ? pattern : text) + row0 * dp, dbulk, &bar);
            if (HAS_N && nbulk) bulk_g2s(nrow[s], (s ? npattern : ntext) + row0 * np, nbulk, &bar);
        }
    }
    // ragged tails and rows past n (zero: valid codes, results are masked)
    for (int i = threadIdx.x; i < 2 * kPackPairs * dp; i += blockDim.x) {
        const int s = i / (kPackPairs * dp), off = i % (kPackPairs * dp);
        if (static_cast<uint32_t>(off) >= dbulk)
            dib[s][off] = static_cast<uint32_t>(off) < dbytes ? (s ? pattern : text)[row0 * dp + off] : 0;
    }
    if (HAS_N) {
        for (int i = threadIdx.x; i < 2 * kPackPairs * np; i += blockDim.x) {
            const int s = i / (kPackPairs * np), off = i % (kPackPairs * np);
            if (static_cast<uint32_t>(off) >= nbulk)
                nrow[s][off] =
                    static_cast<uint32_t>(off) < nbytes ? (s ? npattern : ntext)[row0 * np + off] : 0;
        }
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const int C = (m + CH - 1) / CH;
    const int Cfull = m / CH;
    for (int it = threadIdx.x; it < 2 * kPackGroups * C; it += blockDim.x) {
        const int c = it / (2 * kPackGroups);
        const int g = (it / 2) % kPackGroups;
        const int s = it % 2;
        uint32_t* dst = planes + plane_index(s, static_cast<long long>(blockIdx.x) * kPackGroups + g,
                                             c * CH, 0, nblocks, mc);
        const uint8_t* src = dib[s] + g * 32 * dp;
        const uint8_t* nsrc = nrow[s] + g * 32 * np;
        if (c < Cfull) {
            gather_chunk_dib<false, 4, HAS_N>(src, dp, nsrc, np, c * CH, m, dst, kPackGroups);
        } else {
            switch ((m - c * CH + 3) / 4) {
                case 1: gather_chunk_dib<true, 1, HAS_N>(src, dp, nsrc, np, c * CH, m, dst, kPackGroups); break;
                case 2: gather_chunk_dib<true, 2, HAS_N>(src, dp, nsrc, np, c * CH, m, dst, kPackGroups); break;
                case 3: gather_chunk_dib<true, 3, HAS_N>(src, dp, nsrc, np, c * CH, m, dst, kPackGroups); break;
                default: gather_chunk_dib<true, 4, HAS_N>(src, dp, nsrc, np, c * CH, m, dst, kPackGroups); break;
            }
        }
    }
}

}  // namespace

size_t dibit_pack_smem(int m) {
    return 2 * static_cast<size_t>(kPackPairs) * (dibit_pitch(m) + nplane_pitch(m));
}

bool dibit_pack_fits(int m) { return dibit_pack_smem(m) <= 200 * 1024; }

cudaError_t launch_pack_dibits(const uint8_t* text, const uint8_t* pattern, const uint8_t* ntext,
                               const uint8_t* npattern, long long n, int m, uint32_t* planes,
                               cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!dibit_pack_fits(m) || planes == nullptr) return cudaErrorInvalidValue;
    const size_t smem = dibit_pack_smem(m);
    const unsigned grid = static_cast<unsigned>((n + kPackPairs - 1) / kPackPairs);
    cudaError_t st;
    if (ntext != nullptr) {
        st = ensure_smem_attr<pack_dibit_kernel<true>>(200 * 1024);
        if (st == cudaSuccess)
            pack_dibit_kernel<true><<<grid, kPackNT, smem, s>>>(text, pattern, ntext, npattern, n,
                                                               m, planes);
    } else {
        st = ensure_smem_attr<pack_dibit_kernel<false>>(200 * 1024);
        if (st == cudaSuccess)
            pack_dibit_kernel<false><<<grid, kPackNT, smem, s>>>(text, pattern, nullptr, nullptr,
                                                                n, m, planes);
    }
    count_launch();
    return st != cudaSuccess ? st : cudaGetLastError();
}

}  // namespace sb
