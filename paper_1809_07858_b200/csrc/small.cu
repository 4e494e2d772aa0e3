// Latency form of the Shouji filter for small batches: a per-pair caller of
// shouji_filter (proj/src/shouji.cpp:41-58), or the few pairs the drop-in's
// coalescer gathers from concurrent callers. The throughput kernels slice 32
// pairs into every register word and sweep a pair's windows serially inside
// one thread (~50 µs for one group); here one CTA owns one pair and spreads
// its m windows over the threads instead:
//   * codes: the pair's bases from ASCII records (validated like
//     packed_sequence::from_string, packed_sequence.cpp:19-29; the first
//     illegal byte in pair order, text before pattern, is reported through the
//     same key as the locate kernel) or from packed_sequence planes;
//   * select_window (shouji.cpp:17-31): thread j scans d = -e..+e in reference
//     order over its own window with the reference's two-clause rule — more
//     zeros, or equal zeros with the incumbent's bit 0 set and the candidate's
//     clear; a mismatch cell is "codes differ", with N coded differently in
//     pattern and text and out-of-range columns coded apart from every base,
//     exactly neighborhood.cpp:67-76 and extract(pos, w, pad = 1);
//   * commit_window (shouji.cpp:33-39): the serial strict-improvement overwrite
//     over j, one thread, in shared memory; then the tally popcount and
//     accept = ones <= e (:56-57), e >= m accepting with estimate 0 (:48-49).
// Inputs and outputs may live in mapped pinned host memory (the host entry
// points pass device aliases of their staging buffers), so a call is one
// launch and one synchronisation; outputs are plain stores (one accept byte per
// pair, no atomics to host memory).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sb {

namespace {

__device__ __forceinline__ uint8_t code_ascii(uint8_t c, uint8_t ncode, bool* bad) {
    switch (c) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        case 'N': return ncode;
        default: *bad = true; return ncode;
    }
}

// The last CTA to finish publishes a.seq into *a.done (mapped host memory)
// after a system-scope fence, so the host can poll for completion instead of
// paying a stream synchronisation.
__device__ void finish(const SmallArgs& a) {
    if (a.done == nullptr) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(a.counter, 1u) == static_cast<unsigned>(a.n) - 1u) {
            *a.counter = 0u;
            __threadfence_system();
            *a.done = a.seq;
        }
    }
}

__global__ void shouji_small_kernel(SmallArgs a) {
    extern __shared__ uint8_t sm[];
    const int m = a.m, w = a.w, pair = blockIdx.x;
    const bool select = a.e < static_cast<uint32_t>(m) && w >= 3 && w <= 8;
    const int e = select ? static_cast<int>(a.e) : 0;
    uint8_t* pc = sm;                  // pattern codes at [e, e+m); 6 outside
    uint8_t* tc = pc + m + 2 * e + 16;  // text codes; 7 past m
    uint8_t* bs = tc + m + 16;          // best slice per window
    uint8_t* bz = bs + m + 16;          // its zero count
    uint8_t* bv = bz + m + 16;          // tally words (m + 16 bytes)
    __shared__ uint32_t ones_total;
    __shared__ int bad_here;
    if (threadIdx.x == 0) {
        ones_total = 0;
        bad_here = 0;
    }

    for (int i = threadIdx.x; i < m + 2 * e + 16; i += blockDim.x) pc[i] = 6;
    for (int i = threadIdx.x; i < m + 16; i += blockDim.x) tc[i] = 7;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        uint8_t p, t;
        if (a.text != nullptr) {
            bool bt = false, bp = false;
            t = code_ascii(a.text[static_cast<size_t>(pair) * a.stride + i], 5, &bt);
            p = code_ascii(a.pattern[static_cast<size_t>(pair) * a.stride + i], 4, &bp);
            // locate key ((pair*2 + field) << 24) | pos, as launch_locate writes it
            // (global atomics only on the error path: a.bad_key may be host memory)
            if (bt) {
                atomicMin(a.bad_key, ((static_cast<unsigned long long>(pair) * 2) << 24) | i);
                bad_here = 1;
            }
            if (bp) {
                atomicMin(a.bad_key, ((static_cast<unsigned long long>(pair) * 2 + 1) << 24) | i);
                bad_here = 1;
            }
        } else {
            const int W = (m + 63) / 64;
            const uint64_t* tp = a.tplanes + static_cast<size_t>(pair) * 3 * W;
            const uint64_t* pp = a.pplanes + static_cast<size_t>(pair) * 3 * W;
            const int wd = i >> 6, b = i & 63;
            t = ((tp[2 * W + wd] >> b) & 1u) ? 5
                                              : static_cast<uint8_t>(((tp[wd] >> b) & 1u) |
                                                                     (((tp[W + wd] >> b) & 1u) << 1));
            p = ((pp[2 * W + wd] >> b) & 1u) ? 4
                                              : static_cast<uint8_t>(((pp[wd] >> b) & 1u) |
                                                                     (((pp[W + wd] >> b) & 1u) << 1));
        }
        tc[i] = t;
        pc[e + i] = p;
    }
    __syncthreads();
    if (bad_here || (!select && (w < 3 || w > 8))) {
        finish(a);  // the host reports the illegal byte, or the width; no results
        return;
    }
    if (!select) {
        // e >= m: accept, estimate 0, all-zero tally (shouji.cpp:48-49)
        if (threadIdx.x == 0) {
            a.accept[pair] = 1;
            if (a.est) a.est[pair] = 0;
        }
        if (a.bits)
            for (int k = threadIdx.x; k < (m + 63) / 64; k += blockDim.x)
                a.bits[static_cast<size_t>(pair) * ((m + 63) / 64) + k] = 0;
        finish(a);
        return;
    }
    // select_window for every window j, diagonals in reference order
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        uint8_t best_s = 0, best_z = 0;
        for (int d = -e; d <= e; ++d) {
            const uint8_t* prow = pc + e + d + j;
            unsigned s = 0, ones = 0;
            for (int k = 0; k < w; ++k) {
                const unsigned x = prow[k] != tc[j + k];
                s |= x << k;
                ones += x;
            }
            const uint8_t z = static_cast<uint8_t>(w - ones);
            if (d == -e || z > best_z || (z == best_z && (best_s & 1u) && !(s & 1u))) {
                best_s = static_cast<uint8_t>(s);
                best_z = z;
            }
        }
        bs[j] = best_s;
        bz[j] = best_z;
    }
    __syncthreads();
    // commit_window, serially over j, as a (w-1)-bit state machine in registers
    // (SURVEY App. B2 for general w): when window j is examined, bv[j+w-1] is
    // still 1 (no earlier window reaches it), so the incumbent's zeros are those
    // of S = bv[j .. j+w-2] (bit i = column j+i; columns >= m read as 1, the
    // pad of extract(pos, w, pad = 1)). Strict improvement: commit iff
    // zeros(best) > (w-1) - popcount(S); the committed slice's overhang is
    // dropped (deposit, bitvector.hpp:97-100), i.e. read back as 1. Column j's
    // final bit is decided at step j. The best slices are read 16 windows at a
    // time ahead of the dependent chain; the tally bits go straight into words.
    // the tally words reuse bv's bytes (8-byte aligned: ceil(m/64)*8 <= m+9 bytes fit)
    uint64_t* tally = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bv) + 7) & ~uintptr_t(7));
    if (threadIdx.x == 0) {
        const unsigned full = (1u << (w - 1)) - 1u;
        unsigned S = full;  // bv starts all ones (shouji.cpp:52)
        uint64_t word = 0;
        uint32_t ones = 0;
        for (int j0 = 0; j0 < m; j0 += 16) {
            uint8_t zb[16], sb[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {  // bs / bz have 16 bytes of slack past m
                zb[k] = bz[j0 + k];
                sb[k] = bs[j0 + k];
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int j = j0 + k;
                if (j >= m) break;
                const unsigned z = zb[k], sl = sb[k];
                const bool commit = z + static_cast<unsigned>(__popc(S)) > static_cast<unsigned>(w - 1);
                const unsigned bit = commit ? (sl & 1u) : (S & 1u);
                S = commit ? (sl >> 1) : ((S >> 1) | (1u << (w - 2)));
                const int past = j + w - m;  // state columns past the end read as 1
                if (past > 0)
                    S |= (full << (w - 1 - (past < w - 1 ? past : w - 1))) & full;
                word |= static_cast<uint64_t>(bit) << (j & 63);
                ones += bit;
                if ((j & 63) == 63 || j == m - 1) {
                    tally[j >> 6] = word;
                    word = 0;
                }
            }
        }
        ones_total = ones;
    }
    __syncthreads();
    // tally bits (bitvector words)
    const int W = (m + 63) / 64;
    if (a.bits)
        for (int k = threadIdx.x; k < W; k += blockDim.x)
            a.bits[static_cast<size_t>(pair) * W + k] = tally[k];
    if (threadIdx.x == 0) {
        if (a.est) a.est[pair] = ones_total;
        a.accept[pair] = ones_total <= a.e ? 1 : 0;
    }
    finish(a);
}

}  // namespace

size_t small_smem_bytes(int m, uint32_t e) {
    const size_t ee = e < static_cast<uint32_t>(m) ? e : 0;
    return 5 * static_cast<size_t>(m) + 2 * ee + 80;
}

cudaError_t launch_small(const SmallArgs& a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    if (a.m < 1 || a.m > kSmallMaxM) return cudaErrorInvalidValue;
    const int threads = a.m <= 128 ? 128 : (a.m <= 256 ? 256 : 512);
    shouji_small_kernel<<<a.n, threads, small_smem_bytes(a.m, a.e), s>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
