// Tile machinery of the pack kernels: TMA bulk
// copies of 32-record groups into bank-skewed shared memory, completion on an
// mbarrier, then the in-register gather of phase_a.cuh.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pack.cuh"
#include "phase_a.cuh"

namespace sb {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

// Shared-memory image of one tile: for each (sequence, group) the group's 32
// records, contiguous (one bulk copy each). Consecutive groups are offset by
// an extra 16 bytes (32 * pitch is a multiple of 128) and the pattern half
// starts 64 bytes past a 128-byte multiple of the text half, so the 8 lanes
// of a quarter-warp (2 sequences x 4 groups reading the same row/column
// offset) hit 8 distinct 16-byte bank groups in their LDS.128.
__host__ __device__ inline size_t group_stride(size_t pitch) { return 32 * pitch + 16; }
__host__ __device__ inline size_t seq_stride(size_t pitch, int groups) {
    return groups * group_stride(pitch) + 16 * ((4 - groups) & 7);
}
inline size_t tile_smem(size_t pitch, int groups) { return 2 * seq_stride(pitch, groups) + 128; }

template <bool EDGE, int PM, bool NIB = false, bool DEFER_N = false, int MAXNCG = 4>
__device__ __forceinline__ uint32_t gather_ncg(int ncg, const uint8_t* src, size_t pitch, int col0,
                                               int m, uint32_t* dst, uint32_t* ndst, int stride,
                                               uint32_t* nout = nullptr) {
    if constexpr (NIB) {
        switch (ncg) {
            case 1: gather_chunk_nib<EDGE, 1, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout); break;
            case 2: gather_chunk_nib<EDGE, 2, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout); break;
            case 3: gather_chunk_nib<EDGE, 3, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout); break;
            default: gather_chunk_nib<EDGE, 4, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout); break;
        }
        return 0u;
    }
    if constexpr (MAXNCG == 1) {
        return gather_chunk_smem<EDGE, 1, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
    } else if constexpr (MAXNCG == 2) {
        if (ncg == 1) return gather_chunk_smem<EDGE, 1, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
        return gather_chunk_smem<EDGE, 2, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
    } else {
        switch (ncg) {
            case 1: return gather_chunk_smem<EDGE, 1, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
            case 2: return gather_chunk_smem<EDGE, 2, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
            case 3: return gather_chunk_smem<EDGE, 3, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
            default: return gather_chunk_smem<EDGE, 4, PM, DEFER_N>(src, pitch, col0, m, dst, ndst, stride, nout);
        }
    }
}

// Pack one tile of GROUPS x 32 pairs starting at group g0 (all threads of the
// CTA call it; NT threads). sm: tile_smem() bytes of dynamic shared memory;
// bar: an initialised mbarrier; parity: its current phase (flipped on return
// by the caller). Returns nonzero on an illegal byte. NIB: the records are
// nibble records (pack.cuh; pitch = nibble_pitch(m)), validated by the host.
// NFLAG: write the tile's N-presence flags (pack.cuh) and store a sequence's
// N planes only when one of the tile's records of that sequence holds an N;
// needs one item per thread (2 * GROUPS * ceil(m/16) <= NT) and sflag, 2 words
// of shared memory.
// ICH: columns per item (16, or 8 for the lean form: half the accumulator
// registers per thread, up to IPT items per thread).
template <int PM, int NT, bool NIB = false, bool NFLAG = false, int ICH = CH, int IPT = 1>
__device__ __forceinline__ uint32_t pack_one_tile(uint8_t* sm, uint64_t* bar, uint32_t parity,
                                                  int GROUPS, long long g0,
                                                  const uint8_t* __restrict__ text,
                                                  const uint8_t* __restrict__ pattern, size_t pitch,
                                                  long long n, int m, uint32_t* __restrict__ planes,
                                                  uint32_t* __restrict__ nflags = nullptr,
                                                  uint32_t* sflag = nullptr,
                                                  long long pf_groups = 0,
                                                  bool init_bar = false) {
    const long long row0 = g0 * 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int rows = static_cast<int>(n - row0 < 32 * GROUPS ? n - row0 : 32 * GROUPS);
    const int mc = plane_cols(m);
    const int ipitch = static_cast<int>(pitch);
    const size_t gs = group_stride(pitch), ss = seq_stride(pitch, GROUPS);
    auto rec = [&](int sq, int g) { return sm + sq * ss + g * gs; };
    // bytes of group g moved by TMA (a multiple of 16; a ragged tail is copied below)
    auto tma_bytes = [&](int g) {
        const int r = rows - 32 * g;
        const int b = (r <= 0 ? 0 : (r < 32 ? r : 32)) * ipitch;
        return b & ~15;
    };
    if (threadIdx.x == 0) {
        if (init_bar) mbar_init(bar, 1);  // a one-tile CTA: init and arm under one barrier
        uint32_t total = 0;
        for (int g = 0; g < GROUPS; ++g) total += 2u * static_cast<uint32_t>(tma_bytes(g));
        mbar_expect_tx(bar, total);
    }
    if (NFLAG && threadIdx.x < 2) sflag[threadIdx.x] = 0u;
    __syncthreads();  // expect_tx before any complete_tx; previous tile's readers done
    if (threadIdx.x < 2 * GROUPS) {
        const int sq = threadIdx.x / GROUPS, g = threadIdx.x % GROUPS;
        const int b = tma_bytes(g);
        if (b > 0) {
            const uint8_t* src = (sq == 0 ? text : pattern) + (row0 + 32 * g) * pitch;
            bulk_g2s(rec(sq, g), src, static_cast<uint32_t>(b), bar);
        }
    } else if (pf_groups > 0 && threadIdx.x < 4 * GROUPS) {
        // L2 prefetch of the records a CTA pf_groups groups further on will load,
        // so its bulk copies wait on L2 instead of DRAM (PF_PACK_L2PF)
        const int t = threadIdx.x - 2 * GROUPS;
        const int sq = t / GROUPS, g = t % GROUPS;
        const long long row = row0 + 32 * (pf_groups + g);
        if (row + 32 <= n) {
            const uint8_t* src = (sq == 0 ? text : pattern) + row * pitch;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src),
                         "r"(static_cast<uint32_t>(32 * ipitch & ~15))
                         : "memory");
        }
    }
    mbar_wait(bar, parity);
    if (rows < 32 * GROUPS) {
        // last tile: copy the ragged tail of the last group byte-wise, then make
        // rows past n read as 'A' (valid; their results are masked)
        const int gl = (rows - 1) / 32;  // group holding the last row
        const int have = (rows - 32 * gl) * ipitch;
        const int tb = tma_bytes(gl);
        for (int i = threadIdx.x; i < 2 * (have - tb); i += NT) {
            const int sq = i / (have - tb), off = tb + i % (have - tb);
            rec(sq, gl)[off] = ((sq == 0 ? text : pattern) + (row0 + 32 * gl) * pitch)[off];
        }
        const int per_seq = (32 * GROUPS - rows) * ipitch;  // bytes to fill per sequence
        for (int i = threadIdx.x; i < 2 * per_seq; i += NT) {
            const int sq = i / per_seq;
            const int byte = rows * ipitch + i % per_seq;
            const int g = byte / (32 * ipitch);
            rec(sq, g)[byte - g * 32 * ipitch] = 'A';
        }
        __syncthreads();
    }
    // Items are (chunk, group, sequence) tiles of 32 pairs x ICH columns, the
    // sequence fastest. Full chunks come first and the one chunk straddling m
    // (if any) last, so no warp mixes the gather variants.
    static_assert(ICH == CH || ((ICH == 8 || ICH == 4) && !NIB), "lean items are 4 or 8 columns of ASCII records");
    const int C = (mc + ICH - 1) / ICH;
    const int Cfull = m / ICH;  // chunks entirely inside [0, m)
    uint32_t err = 0u;
    uint32_t sink[ICH * 3];
    uint32_t nw[IPT][ICH];  // NFLAG: this thread's items' N-plane words
    uint32_t* ndst[IPT];
    int nseq[IPT], ncols[IPT];
    const int items = 2 * GROUPS * C;
    // one item; nwk: its N-plane words (NFLAG), returns the N destination
    auto do_item = [&](int it, uint32_t* nwk, int& sq_out, int& ncols_out) -> uint32_t* {
        const int c = it / (2 * GROUPS);
        const int g = (it / 2) % GROUPS;
        const int sq = it % 2;
        uint32_t* dst = planes ? planes + lohi_index(sq, g0 + g, c * ICH, 0, nblocks, mc) : sink;
        uint32_t* nd = planes ? planes + nplane_index(sq, g0 + g, c * ICH, nblocks, mc) : sink + 2 * ICH;
        const int stride = planes ? kPackGroups : 1;
        if constexpr (NFLAG) {  // an edge chunk's gather fills only its first 4*ncg words
#pragma unroll
            for (int col = 0; col < ICH; ++col) nwk[col] = 0u;
        }
        if (c < Cfull) {
            if constexpr (NIB)
                gather_chunk_nib<false, 4, NFLAG>(rec(sq, g), pitch, c * ICH, m, dst, nd, stride, nwk);
            else
                err |= gather_chunk_smem<false, ICH / 4, PM, NFLAG>(rec(sq, g), pitch, c * ICH, m,
                                                                    dst, nd, stride, nwk);
        } else {
            err |= gather_ncg<true, PM, NIB, NFLAG, ICH / 4>((m - c * ICH + 3) / 4, rec(sq, g), pitch,
                                                       c * ICH, m, dst, nd, stride, nwk);
        }
        if constexpr (NFLAG) {
            uint32_t any = 0u;
#pragma unroll
            for (int col = 0; col < ICH; ++col) any |= nwk[col];
            if (any) sflag[sq] = 1u;
        }
        sq_out = sq;
        ncols_out = c < Cfull ? ICH : m - c * ICH;
        return nd;
    };
    if constexpr (NFLAG) {  // at most IPT items per thread (checked by the launcher)
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int it = threadIdx.x + k * NT;
            ndst[k] = it < items ? do_item(it, nw[k], nseq[k], ncols[k]) : nullptr;
        }
    } else {
        int sq_, nc_;
        for (int it = threadIdx.x; it < items; it += NT) do_item(it, nw[0], sq_, nc_);
    }
    if constexpr (NFLAG) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            if (ndst[k] != nullptr && sflag[nseq[k]]) {
#pragma unroll
                for (int col = 0; col < ICH; ++col)
                    if (col < ncols[k]) ndst[k][col * kNColWords] = nw[k][col];
            }
        }
        if (threadIdx.x < 2 * GROUPS) {
            const int sq = threadIdx.x / GROUPS, g = threadIdx.x % GROUPS;
            nflags[nflag_index(sq, g0 + g, nblocks)] = sflag[sq];
        }
    }
    return err;
}

}  // namespace sb
