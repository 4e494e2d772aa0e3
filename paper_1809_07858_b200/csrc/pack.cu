// Stage 1: ASCII records -> pair-sliced planes (see pack.cuh for the layout).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"

namespace sb {

namespace {

// One CTA of NT threads per tile of GROUPS x 32 pairs (pack_one_tile,
// pack_tile.cuh). NFLAG: also write the N-presence flags (pack.cuh) and skip
// N-free tiles' N planes. 128 registers: ptxas would otherwise take up to 180.
// ICH = 8 (lean): 8-column items, up to IPT per thread, 64 registers (8 CTAs
// of 128 threads fit the register file, so the pack's CTAs leave room for
// others on the SM).
template <int GROUPS, int NT, int PM, bool NIB, bool NFLAG = false, int ICH = CH, int IPT = 1>
__global__ void __launch_bounds__(NT, (ICH == CH ? 512 : 1024) / NT)
pack_tile_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                 size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ err_flag, uint32_t* __restrict__ nflags,
                 long long pf_groups) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t sflag[2];
    if (NFLAG && blockIdx.x == 0) {  // the all-zero N column image N-free groups read
        uint32_t* zero = nflags + nflag_words(n);
        for (int i = threadIdx.x; i < static_cast<int>(nzero_words(m)); i += NT) zero[i] = 0u;
    }
    // thread 0 initialises and arms the barrier inside pack_one_tile, before its
    // first __syncthreads (one barrier instead of two per CTA)
    const uint32_t err = pack_one_tile<PM, NT, NIB, NFLAG, ICH, IPT>(
        sm, &bar, 0, GROUPS, static_cast<long long>(blockIdx.x) * GROUPS, text, pattern, pitch, n, m,
        planes, nflags, sflag, pf_groups, true);
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
    uint32_t* dst = planes ? planes + lohi_index(s, g, c * CH, 0, nblocks, mc) : sink;
    uint32_t* ndst = planes ? planes + nplane_index(s, g, c * CH, nblocks, mc) : sink + 2 * CH;
    const int stride = planes ? kPackGroups : 1;
    const uint32_t err =
        produce_chunk(s == 0 ? text : pattern, pitch, g * 32, n, c, m, dst, ndst, stride);
    if (err) atomicOr(err_flag, 1u);
}

}  // namespace

// Tile geometry: `groups` record groups per CTA of `nt` threads, one
// (chunk, group, sequence) item per thread (2 * groups * ceil(m/16) <= nt),
// chosen so most threads hold an item and 3-4 CTAs' tiles fit one SM's shared
// memory (measured, tools/exp_stages.py with PF_PACK_GEOM): C = ceil(m/16) <= 8
// (m <= 128) 8 groups x 128 threads; C <= 12 4 x 96 (m=150: 1.16 ms per 16M
// pairs vs 1.33 for 4 x 128, 1.24 for 6 x 128, 1.29 for 8 x 160); otherwise
// 4 x 128 (m=250: 1.02 ms per 8M pairs vs 1.33 for 3 x 96 or 2 x 64).
// PF_PACK_GEOM="groups,threads" picks another compiled geometry (A/B runs).
struct TileGeom {
    int groups, nt;
};
static TileGeom tile_geom(size_t pitch, int m) {
    if (const char* e = std::getenv("PF_PACK_GEOM")) {
        int g = 0, t = 0;
        if (std::sscanf(e, "%d,%d", &g, &t) == 2 &&
            ((g == 8 && t == 128) || (g == 4 && t == 96) || (g == 4 && t == 128)))
            return {g, t};
    }
    const int C = (m + CH - 1) / CH;
    if (C <= 8 && tile_smem(pitch, 8) <= 110 * 1024) return {8, 128};
    if (C <= 12) return {4, 96};
    return {4, 128};
}

template <int GROUPS, int NT, int PM, bool NIB = false, bool NFLAG = false, int ICH = CH, int IPT = 1>
static cudaError_t launch_tile_f(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                                 long long n, int m, uint32_t* planes, uint32_t* err_flag,
                                 uint32_t* nflags, cudaStream_t s) {
    const cudaError_t st =
        ensure_smem_attr<pack_tile_kernel<GROUPS, NT, PM, NIB, NFLAG, ICH, IPT>>(110 * 1024);
    if (st != cudaSuccess) return st;
    const long long ngroups = (n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + GROUPS - 1) / GROUPS);
    // Each CTA also prefetches into L2 the records of the tile pf_tiles tiles
    // further on (cp.async.bulk.prefetch.L2), so that CTA's bulk copies wait on L2
    // rather than DRAM: shorter CTA lifetimes, more record bytes in flight per SM
    // for the same shared memory. Measured (tools/exp_stages.py, pack ms per 16M /
    // 16M / 8M pairs at m = 100 / 150 / 250): off 0.631 / 1.086 / 0.928, 100 tiles
    // 0.589 / 1.090 / 0.868, 200-450 tiles 0.573-0.578 / 1.062-1.065 / 0.853-0.855,
    // 1200 tiles 0.898 / 1.087 / 1.198 (the prefetched lines no longer survive in
    // L2). PF_PACK_L2PF overrides the distance (0: off).
    static const long long pf_tiles = [] {
        const char* e = std::getenv("PF_PACK_L2PF");
        return e ? std::atoll(e) : 320ll;
    }();
    pack_tile_kernel<GROUPS, NT, PM, NIB, NFLAG, ICH, IPT><<<grid, NT, tile_smem(pitch, GROUPS), s>>>(
        text, pattern, pitch, n, m, planes, err_flag, nflags, pf_tiles * GROUPS);
    return cudaGetLastError();
}

// The lean pack (4- or 8-column items, 64 registers) for the 8 x 128 geometry
// (m <= 128: at most 4 / 2 items per thread): PF_PACK_LEAN=4 or 8.
static int pack_lean() {
    static const int cols = [] {
        const char* e = std::getenv("PF_PACK_LEAN");
        const int v = e ? std::atoi(e) : 0;
        return v == 4 || v == 8 ? v : 0;
    }();
    return cols;
}

template <int PM, bool NIB = false, bool NFLAG = false>
static cudaError_t launch_tile_nt(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                                  long long n, int m, TileGeom tg, uint32_t* planes,
                                  uint32_t* err_flag, uint32_t* nflags, cudaStream_t s) {
    if (tg.groups == 8) {
        if constexpr (!NIB)
            if (pack_lean() && m <= 128)
                return pack_lean() == 4
                           ? launch_tile_f<8, 128, PM, false, NFLAG, 4, 4>(text, pattern, pitch, n, m,
                                                                         planes, err_flag, nflags, s)
                           : launch_tile_f<8, 128, PM, false, NFLAG, 8, 2>(text, pattern, pitch, n, m,
                                                                         planes, err_flag, nflags, s);
        return launch_tile_f<8, 128, PM, NIB, NFLAG>(text, pattern, pitch, n, m, planes, err_flag, nflags, s);
    }
    if (tg.nt == 96)
        return launch_tile_f<4, 96, PM, NIB, NFLAG>(text, pattern, pitch, n, m, planes, err_flag, nflags, s);
    return launch_tile_f<4, 128, PM, NIB, NFLAG>(text, pattern, pitch, n, m, planes, err_flag, nflags, s);
}

template <int PM, bool NIB = false>
static cudaError_t launch_tile(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                               long long n, int m, uint32_t* planes, uint32_t* err_flag,
                               uint32_t* nflags, cudaStream_t s) {
    const TileGeom tg = tile_geom(pitch, m);
    return nflags ? launch_tile_nt<PM, NIB, true>(text, pattern, pitch, n, m, tg, planes,
                                                  err_flag, nflags, s)
                  : launch_tile_nt<PM, NIB, false>(text, pattern, pitch, n, m, tg, planes,
                                                   err_flag, nullptr, s);
}

// The tile kernels can write N-presence flags when each thread owns at most
// one (chunk, group, sequence) item.
static bool tile_fits(size_t pitch, int m) {
    const TileGeom tg = tile_geom(pitch, m);
    return tile_smem(pitch, tg.groups) <= 110 * 1024;
}
static bool tile_nflags_fit(size_t pitch, int m) {
    const TileGeom tg = tile_geom(pitch, m);
    return tile_fits(pitch, m) && 2 * tg.groups * ((m + CH - 1) / CH) <= tg.nt;
}

bool pack_writes_nflags(const FilterArgs& a) {
    if (a.packed_text) return pack_planes_writes_nflags(a.packed_text, a.packed_pattern, a.m);
    if (a.dibits) return dibit_pack_fits(a.m);
    if (a.nibbles) return tile_nflags_fit(nibble_pitch(a.m), a.m);
    return a.pitch % 4 == 0 && tile_nflags_fit(a.pitch, a.m);
}

cudaError_t launch_pack(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                        int m, uint32_t* planes, uint32_t* err_flag, cudaStream_t s,
                        uint32_t* nflags) {
    if (n <= 0) return cudaSuccess;
    if (pitch % 4 != 0) return cudaErrorInvalidValue;
    if (nflags && (!planes || !tile_nflags_fit(pitch, m))) return cudaErrorInvalidValue;
    cudaError_t st;
    if (tile_fits(pitch, m)) {
        // row i of a group starts (i * pm) % 4 words past a 16-byte boundary
        switch ((pitch / 4) % 4) {
            case 0: st = launch_tile<0>(text, pattern, pitch, n, m, planes, err_flag, nflags, s); break;
            case 1: st = launch_tile<1>(text, pattern, pitch, n, m, planes, err_flag, nflags, s); break;
            case 2: st = launch_tile<2>(text, pattern, pitch, n, m, planes, err_flag, nflags, s); break;
            default: st = launch_tile<3>(text, pattern, pitch, n, m, planes, err_flag, nflags, s); break;
        }
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
    return tile_fits(np, m);
}

cudaError_t launch_pack_nibbles(const uint8_t* text, const uint8_t* pattern, long long n, int m,
                                uint32_t* planes, cudaStream_t s, uint32_t* nflags) {
    if (n <= 0) return cudaSuccess;
    if (!nibble_pack_fits(m) || planes == nullptr) return cudaErrorInvalidValue;
    const size_t np = nibble_pitch(m);
    if (nflags && !tile_nflags_fit(np, m)) return cudaErrorInvalidValue;
    const cudaError_t st = launch_tile<0, true>(text, pattern, np, n, m, planes, nullptr, nflags, s);
    count_launch();
    return st;
}

// ---- dibit records (host-packed upload format, pack.cuh) ---------------------------
namespace {

// One CTA per pair block (8 groups): a bulk copy per sequence brings the
// block's dibit rows (and, for chunks with N, its N-plane rows) into shared
// memory, then each thread gathers one (chunk, group, sequence) item.
// nflags (optional): N-presence flags — without N rows every group is N-free
// and its N planes are not stored; with N rows every group is flagged.
template <bool HAS_N, bool SKIP_N = false>
__global__ void __launch_bounds__(kPackNT)
pack_dibit_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                  const uint8_t* __restrict__ ntext, const uint8_t* __restrict__ npattern,
                  long long n, int m, uint32_t* __restrict__ planes,
                  uint32_t* __restrict__ nflags) {
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
    if (nflags && threadIdx.x < 2 * kPackGroups)
        nflags[nflag_index(threadIdx.x / kPackGroups,
                           static_cast<long long>(blockIdx.x) * kPackGroups + threadIdx.x % kPackGroups,
                           nblocks)] = HAS_N ? 1u : 0u;
    if (nflags && blockIdx.x == 0) {  // the all-zero N column image N-free groups read
        uint32_t* zero = nflags + nflag_words(n);
        for (int i = threadIdx.x; i < static_cast<int>(nzero_words(m)); i += blockDim.x) zero[i] = 0u;
    }
    for (int it = threadIdx.x; it < 2 * kPackGroups * C; it += blockDim.x) {
        const int c = it / (2 * kPackGroups);
        const int g = (it / 2) % kPackGroups;
        const int s = it % 2;
        const long long gg = static_cast<long long>(blockIdx.x) * kPackGroups + g;
        uint32_t* dst = planes + lohi_index(s, gg, c * CH, 0, nblocks, mc);
        uint32_t* ndst = planes + nplane_index(s, gg, c * CH, nblocks, mc);
        const uint8_t* src = dib[s] + g * 32 * dp;
        const uint8_t* nsrc = nrow[s] + g * 32 * np;
        if (c < Cfull) {
            gather_chunk_dib<false, 4, HAS_N, SKIP_N>(src, dp, nsrc, np, c * CH, m, dst, ndst, kPackGroups);
        } else {
            switch ((m - c * CH + 3) / 4) {
                case 1: gather_chunk_dib<true, 1, HAS_N, SKIP_N>(src, dp, nsrc, np, c * CH, m, dst, ndst, kPackGroups); break;
                case 2: gather_chunk_dib<true, 2, HAS_N, SKIP_N>(src, dp, nsrc, np, c * CH, m, dst, ndst, kPackGroups); break;
                case 3: gather_chunk_dib<true, 3, HAS_N, SKIP_N>(src, dp, nsrc, np, c * CH, m, dst, ndst, kPackGroups); break;
                default: gather_chunk_dib<true, 4, HAS_N, SKIP_N>(src, dp, nsrc, np, c * CH, m, dst, ndst, kPackGroups); break;
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
                               cudaStream_t s, uint32_t* nflags) {
    if (n <= 0) return cudaSuccess;
    if (!dibit_pack_fits(m) || planes == nullptr) return cudaErrorInvalidValue;
    const size_t smem = dibit_pack_smem(m);
    const unsigned grid = static_cast<unsigned>((n + kPackPairs - 1) / kPackPairs);
    cudaError_t st;
    if (ntext != nullptr) {
        st = ensure_smem_attr<pack_dibit_kernel<true>>(200 * 1024);
        if (st == cudaSuccess)
            pack_dibit_kernel<true><<<grid, kPackNT, smem, s>>>(text, pattern, ntext, npattern, n,
                                                               m, planes, nflags);
    } else if (nflags != nullptr) {
        st = ensure_smem_attr<pack_dibit_kernel<false, true>>(200 * 1024);
        if (st == cudaSuccess)
            pack_dibit_kernel<false, true><<<grid, kPackNT, smem, s>>>(text, pattern, nullptr,
                                                                      nullptr, n, m, planes, nflags);
    } else {
        st = ensure_smem_attr<pack_dibit_kernel<false>>(200 * 1024);
        if (st == cudaSuccess)
            pack_dibit_kernel<false><<<grid, kPackNT, smem, s>>>(text, pattern, nullptr, nullptr,
                                                                n, m, planes, nullptr);
    }
    count_launch();
    return st != cudaSuccess ? st : cudaGetLastError();
}

}  // namespace sb
