// sm_100a kernels for the Shouji pre-alignment filter (arXiv 1809.07858).
//
// Reference hot path: prefilter::shouji_filter, proj/src/shouji.cpp:41-58,
// with neighborhood_map (proj/src/neighborhood.cpp:41-79), select_window
// (shouji.cpp:17-31), commit_window (shouji.cpp:33-39) and the codec
// packed_sequence::from_string (proj/src/packed_sequence.cpp:7-34).
//
// Design (DESIGN.md has the long form): PAIR-SLICED bit logic. One thread
// owns 32 consecutive pairs; every register word holds one bit of 32 pairs
// (bit b = pair 32*group + b). Nothing is ever serial per pair: the
// neighbourhood map, the window search, the commit step and the edit count
// are all 32-pair-wide LOP3 expressions. The reference's serial commit chain
// over columns becomes an 8-state machine (Appendix B2 of SURVEY.md) applied
// to 32 pairs per instruction.
//
//   stage 1 (pack.cu, pack_planes.cu): records -> planes[seq][pair block][col]
//            [plane][8 groups] in global memory. ASCII records arrive by TMA
//            bulk copy into shared memory and are bit-transposed in registers
//            (phase_a.cuh gather_chunk: FMA-pipe shifts, masked ORs, PRMT byte
//            insertion), validating every byte; host-packed dibit / nibble
//            records and packed_sequence planes have their own gathers.
//   stage 2 (fused.cuh for width 4 and E <= 31; shouji_generic below for
//            other widths, larger E and m > 255): per block of 4 windows the
//            2E+1 diagonals are scanned in reference order with the strict
//            first-argmin key 2*ones + bit0 (equivalent to shouji.cpp:26-28,
//            SURVEY App. B1); the chosen slices drive the commit FSM and a
//            bit-sliced counter; accept bits and estimates are written per group.
//
// This unit holds the generic search, the small helper kernels (illegal-byte
// locator, tally-bit transpose, e >= m short-circuit, repitch) and the launch
// dispatch.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "bitslice.cuh"
#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"
#include "phase_a.cuh"

#include <array>
#include <cstdlib>
#include <utility>

namespace sb {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count() { return g_launches.load(); }
void count_launch(int k) { g_launches.fetch_add(static_cast<uint64_t>(k)); }

// ---------------------------------------------------------------------------
// Generic path: any width 3..8, any e < m. Two kernels: pack (phase A into
// global planes [col][3][ngroups]) and a plain pair-sliced sweep reading them.
// ---------------------------------------------------------------------------
template <int W>
struct WCfg {
    static constexpr int NO = W >= 8 ? 4 : (W >= 4 ? 3 : 2);  // planes for ones in [0, W]
    static constexpr int NK = NO + 1;                          // key = 2*ones + bit0
    static constexpr int NS = W - 1 >= 4 ? 3 : (W - 1 >= 2 ? 2 : 1);  // planes for popcount(S)
};

template <int W, int NC>
__global__ void __launch_bounds__(128)
shouji_generic(const uint32_t* __restrict__ planes, long long n, int m, int e,
               uint32_t* __restrict__ accept, uint32_t* __restrict__ estimates,
               uint32_t* __restrict__ outplanes) {
    using Cfg = WCfg<W>;
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long ngroups = (n + 31) / 32;
    if (g >= ngroups) return;
    const long long row0 = g * 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const uint32_t* tb = planes + lohi_index(0, g, 0, 0, nblocks, mc);
    const uint32_t* pb = planes + lohi_index(1, g, 0, 0, nblocks, mc);
    const uint32_t* tnb = planes + nplane_index(0, g, 0, nblocks, mc);
    const uint32_t* pnb = planes + nplane_index(1, g, 0, nblocks, mc);
    auto tp = [&](int col, int k) {
        return k < 2 ? __ldg(tb + size_t(col) * kLhColWords + k * kPackGroups)
                     : __ldg(tnb + size_t(col) * kNColWords);
    };
    auto pp = [&](int col, int k) {
        return k < 2 ? __ldg(pb + size_t(col) * kLhColWords + k * kPackGroups)
                     : __ldg(pnb + size_t(col) * kNColWords);
    };

    uint32_t S[W - 1];
#pragma unroll
    for (int i = 0; i < W - 1; ++i) S[i] = ~0u;
    uint32_t cnt[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) cnt[i] = 0u;

    for (int j = 0; j < m; ++j) {
        uint32_t tw[W][3];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int col = j + k;
            if (col < m) {
                tw[k][0] = tp(col, 0);
                tw[k][1] = tp(col, 1);
                tw[k][2] = tp(col, 2);
            } else {
                tw[k][0] = tw[k][1] = 0u;
                tw[k][2] = ~0u;
            }
        }
        uint32_t bk[Cfg::NK], bsl[W];
        for (int d = -e; d <= e; ++d) {
            uint32_t sl[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int pc = j + k + d;
                uint32_t plo = 0u, phi = 0u, pn = ~0u;
                if (pc >= 0 && pc < m) {
                    plo = pp(pc, 0);
                    phi = pp(pc, 1);
                    pn = pp(pc, 2);
                }
                sl[k] = (plo ^ tw[k][0]) | (phi ^ tw[k][1]) | pn | tw[k][2];
            }
            uint32_t ones[Cfg::NO];
            bs_popcount<W>(sl, ones);
            uint32_t key[Cfg::NK];
            key[0] = sl[0];
#pragma unroll
            for (int i = 0; i < Cfg::NO; ++i) key[i + 1] = ones[i];
            if (d == -e) {
#pragma unroll
                for (int i = 0; i < Cfg::NK; ++i) bk[i] = key[i];
#pragma unroll
                for (int k = 0; k < W; ++k) bsl[k] = sl[k];
            } else {
                const uint32_t lt = bs_less(key, bk);
#pragma unroll
                for (int i = 0; i < Cfg::NK; ++i) bk[i] = bs_select(key[i], bk[i], lt);
#pragma unroll
                for (int k = 0; k < W; ++k) bsl[k] = bs_select(sl[k], bsl[k], lt);
            }
        }
        // commit: ones(best) <= popcount(S)  (general form of fsm_step4)
        uint32_t ps[Cfg::NS];
        bs_popcount<W - 1>(S, ps);
        uint32_t ones[Cfg::NO];
#pragma unroll
        for (int i = 0; i < Cfg::NO; ++i) ones[i] = bk[i + 1];
        const uint32_t commit = ~bs_less(ps, ones);
        const uint32_t out = (commit & bsl[0]) | (~commit & S[0]);
#pragma unroll
        for (int i = 0; i < W - 2; ++i) S[i] = (commit & bsl[i + 1]) | (~commit & S[i + 1]);
        S[W - 2] = bsl[W - 1] | ~commit;
        if (outplanes) outplanes[static_cast<long long>(j) * ngroups + g] = out;
        const uint32_t one[1] = {out};
        bs_add(cnt, one);
    }
    const long long valid = n - row0;
    const uint32_t vmask = valid >= 32 ? ~0u : ((1u << valid) - 1u);
    accept[g] = bs_le_const(cnt, static_cast<uint32_t>(e)) & vmask;
    if (estimates) {
        for (int b = 0; b < 32 && b < valid; ++b) {
            uint32_t est = 0;
#pragma unroll
            for (int i = 0; i < NC; ++i) est |= ((cnt[i] >> b) & 1u) << i;
            estimates[row0 + b] = est;
        }
    }
}

// ---------------------------------------------------------------------------
// Error location, tally transpose, short-circuit fill.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool valid_base(uint8_t c) {
    return c == 'A' || c == 'C' || c == 'G' || c == 'T' || c == 'N';
}

__global__ void locate_illegal(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                               size_t pitch, long long n, int m, unsigned long long* key) {
    const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    for (int field = 0; field < 2; ++field) {
        const uint8_t* s = (field == 0 ? text : pattern) + p * pitch;
        for (int i = 0; i < m; ++i) {
            if (!valid_base(s[i])) {
                const unsigned long long k =
                    (static_cast<unsigned long long>(p * 2 + field) << 24) | static_cast<unsigned>(i);
                atomicMin(key, k);
                return;
            }
        }
    }
}

__global__ void bits_transpose(const uint32_t* __restrict__ outplanes, long long n, int m,
                               uint64_t* __restrict__ bits) {
    const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const long long ngroups = (n + 31) / 32;
    const long long g = p / 32;
    const int b = static_cast<int>(p % 32);
    const int words = (m + 63) / 64;
    for (int w = 0; w < words; ++w) {
        uint64_t v = 0;
        for (int t = 0; t < 64; ++t) {
            const int j = 64 * w + t;
            if (j >= m) break;
            v |= static_cast<uint64_t>((outplanes[static_cast<long long>(j) * ngroups + g] >> b) & 1u) << t;
        }
        bits[p * words + w] = v;
    }
}

__global__ void accept_all(long long n, int m, uint32_t* accept, uint32_t* estimates, uint64_t* bits) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long ngroups = (n + 31) / 32;
    if (i < ngroups) {
        const long long valid = n - i * 32;
        accept[i] = valid >= 32 ? ~0u : ((1u << valid) - 1u);
    }
    if (i < n) {
        if (estimates) estimates[i] = 0u;
        if (bits) {
            const int words = (m + 63) / 64;
            for (int w = 0; w < words; ++w) bits[i * words + w] = 0ull;
        }
    }
}

// ---------------------------------------------------------------------------
// Launchers.
// ---------------------------------------------------------------------------
// Defined in fused.cuh, explicitly instantiated in fused_e*.cu (compiled in
// parallel: each E is its own fully unrolled kernel).
template <int E>
cudaError_t launch_search_e(const FilterArgs& a, cudaStream_t s);

using SearchFn = cudaError_t (*)(const FilterArgs&, cudaStream_t);
template <int... Es>
static constexpr std::array<SearchFn, sizeof...(Es)> make_search_table(std::integer_sequence<int, Es...>) {
    return {&launch_search_e<Es>...};
}
static constexpr auto kSearchTable =
    make_search_table(std::make_integer_sequence<int, kFusedMaxE + 1>{});

// Blocked any-width search (wsearch.cuh) instead of the per-column generic
// kernel: PF_WSEARCH=0 turns it off (A/B runs).
static bool wsearch_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("PF_WSEARCH");
        return !(e && e[0] == '0');
    }();
    return v;
}

// Prefetching search (fused.cuh shouji_search_w4_pf): PF_SEARCH_PF=0 turns it off.
bool search_prefetch_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("PF_SEARCH_PF");
        return !(e && e[0] == '0');
    }();
    return v;
}

template <int W, int NC>
static cudaError_t launch_generic_w(const FilterArgs& a, cudaStream_t s) {
    const long long ngroups = (a.n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + 127) / 128);
    shouji_generic<W, NC><<<grid, 128, 0, s>>>(a.planes, a.n, a.m, static_cast<int>(a.e), a.accept,
                                               a.estimates, a.outplanes);
    count_launch();
    return cudaGetLastError();
}

template <int NC>
static cudaError_t launch_generic(const FilterArgs& a, cudaStream_t s) {
    switch (a.width) {
        case 3: return launch_generic_w<3, NC>(a, s);
        case 4: return launch_generic_w<4, NC>(a, s);
        case 5: return launch_generic_w<5, NC>(a, s);
        case 6: return launch_generic_w<6, NC>(a, s);
        case 7: return launch_generic_w<7, NC>(a, s);
        case 8: return launch_generic_w<8, NC>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

size_t planes_scratch_words(long long n, int m) {
    return plane_words(n, m) + nflag_words(n) + nzero_words(m);
}

// The width-4 kernels count estimates in 12 bit planes (m <= 4095).
bool use_fused(uint32_t width, uint32_t e, int m) {
    return width == 4 && e <= static_cast<uint32_t>(kFusedMaxE) && m <= 4095;
}

// N-presence flags (pack.cuh): used when the pack kernel can write them and the
// search is the width-4 kernel (the other searches read every N plane; with
// flags the direct width-4 form replaces the prefetching one, which it matches
// or beats at 8 <= E <= 12 once N-free warps drop the N planes: m=100 E8 9.41
// vs 9.34, E10 8.37 vs 8.30, E12 7.37 vs 7.45 G pairs/s; m=150 E8 5.22 vs
// 5.09). PF_NFLAGS=0 turns them off (A/B runs).
static bool nflags_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("PF_NFLAGS");
        return !(e && e[0] == '0');
    }();
    return v;
}

static bool search_reads_nflags(const FilterArgs& a) {
    return use_fused(a.width, a.e, a.m) || (wsearch_enabled() && wsearch_applies(a));
}

// The N-presence flag region both stages agree on (or null).
static FilterArgs resolve_nflags(const FilterArgs& args) {
    FilterArgs a = args;
    a.nflags = nullptr;
    if (nflags_enabled() && args.planes_words >= planes_scratch_words(a.n, a.m) &&
        search_reads_nflags(a) && pack_writes_nflags(a))
        a.nflags = a.planes + plane_words(a.n, a.m);
    return a;
}

static cudaError_t launch_pack_of(const FilterArgs& a, cudaStream_t s) {
    return a.packed_text ? launch_pack_planes(a.packed_text, a.packed_pattern, a.n, a.m, a.planes, s,
                                              a.nflags)
           : a.dibits    ? launch_pack_dibits(a.text, a.pattern, a.ntext, a.npattern, a.n, a.m,
                                              a.planes, s, a.nflags)
           : a.nibbles   ? launch_pack_nibbles(a.text, a.pattern, a.n, a.m, a.planes, s, a.nflags)
                         : launch_pack(a.text, a.pattern, a.pitch, a.n, a.m, a.planes, a.err_flag, s,
                                       a.nflags);
}

static cudaError_t launch_search_of(const FilterArgs& a, cudaStream_t s) {
    if (use_fused(a.width, a.e, a.m)) return kSearchTable[a.e](a, s);
    if (wsearch_enabled() && wsearch_applies(a)) return launch_wsearch(a, s);
    return a.m <= 255 ? launch_generic<8>(a, s) : launch_generic<24>(a, s);
}

cudaError_t launch_filter_stage(const FilterArgs& args, cudaStream_t s, int stage) {
    if (args.n <= 0) return cudaSuccess;
    if (args.planes == nullptr || args.planes_words < plane_words(args.n, args.m))
        return cudaErrorInvalidValue;
    const FilterArgs a = resolve_nflags(args);
    return stage == 1 ? launch_pack_of(a, s) : launch_search_of(a, s);
}

cudaError_t launch_filter(const FilterArgs& args, cudaStream_t s) {
    if (args.n <= 0) return cudaSuccess;
    if (args.planes == nullptr || args.planes_words < plane_words(args.n, args.m))
        return cudaErrorInvalidValue;
    FilterArgs a = resolve_nflags(args);
    cudaError_t st =
        a.packed_text ? launch_pack_planes(a.packed_text, a.packed_pattern, a.n, a.m, a.planes, s,
                                           a.nflags)
        : a.dibits    ? launch_pack_dibits(a.text, a.pattern, a.ntext, a.npattern, a.n, a.m,
                                           a.planes, s, a.nflags)
        : a.nibbles   ? launch_pack_nibbles(a.text, a.pattern, a.n, a.m, a.planes, s, a.nflags)
                      : launch_pack(a.text, a.pattern, a.pitch, a.n, a.m, a.planes, a.err_flag, s,
                                    a.nflags);
    if (st != cudaSuccess) return st;
    if (a.stage_event != nullptr) {
        st = cudaEventRecord(a.stage_event, s);
        if (st != cudaSuccess) return st;
    }
    if (use_fused(a.width, a.e, a.m)) return kSearchTable[a.e](a, s);
    if (wsearch_enabled() && wsearch_applies(a)) return launch_wsearch(a, s);
    return a.m <= 255 ? launch_generic<8>(a, s) : launch_generic<24>(a, s);
}

cudaError_t launch_validate(const FilterArgs& a, cudaStream_t s) {
    return launch_pack(a.text, a.pattern, a.pitch, a.n, a.m, nullptr, a.err_flag, s);
}

cudaError_t launch_locate(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                          int m, unsigned long long* d_key, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    locate_illegal<<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, d_key);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_bits_transpose(const uint32_t* outplanes, long long n, int m, uint64_t* bits,
                                  cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    bits_transpose<<<grid, 128, 0, s>>>(outplanes, n, m, bits);
    count_launch();
    return cudaGetLastError();
}

// One thread per 4-byte output word; consecutive threads read consecutive
// source bytes, so the byte loads coalesce.
__global__ void repitch_kernel(const uint8_t* __restrict__ src, size_t src_stride,
                               uint8_t* __restrict__ dst, size_t dst_pitch, long long n, int m) {
    const int wpr = (m + 3) / 4;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * wpr) return;
    const long long row = i / wpr;
    const int c0 = static_cast<int>(i % wpr) * 4;
    const uint8_t* s = src + row * src_stride + c0;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (c0 + k < m) v |= static_cast<uint32_t>(__ldg(s + k)) << (8 * k);
    *reinterpret_cast<uint32_t*>(dst + row * dst_pitch + c0) = v;
}

cudaError_t launch_repitch(const uint8_t* src, size_t src_stride, uint8_t* dst, size_t dst_pitch,
                           long long n, int m, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const long long total = n * ((m + 3) / 4);
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    repitch_kernel<<<grid, 256, 0, s>>>(src, src_stride, dst, dst_pitch, n, m);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_accept_all(long long n, int m, uint32_t* accept, uint32_t* estimates,
                              uint64_t* bits, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    accept_all<<<grid, 128, 0, s>>>(n, m, accept, estimates, bits);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
