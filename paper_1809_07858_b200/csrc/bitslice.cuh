// Bit-sliced integer helpers for the pair-sliced Shouji kernels.
//
// Layout convention used everywhere in csrc/: a "plane word" is a uint32 whose
// bit b belongs to pair (32*group + b). A small unsigned integer that differs
// per pair (a window's zero count, an edit estimate, ...) is held as an array
// of plane words, plane i = bit i of the integer. Every operation below is
// therefore 32 pairs wide, and nvcc folds the expressions into LOP3.
#pragma once
#include <cstdint>

namespace sb {

__device__ __forceinline__ uint32_t rotl(uint32_t x, int s) {
    return __funnelshift_l(x, x, static_cast<unsigned>(s) & 31u);
}
__device__ __forceinline__ uint32_t rotr(uint32_t x, int s) {
    return __funnelshift_r(x, x, static_cast<unsigned>(s) & 31u);
}

// One LOP3 with an explicit truth table (imm = f(0xF0, 0xCC, 0xAA)). The asm
// is opaque to the optimizer, so a hand-counted expression stays that count
// (nvcc otherwise re-associates the compare/select chains into more LOP3s).
template <unsigned IMM>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(IMM));
    return d;
}

// Running "a < b" across planes 0..N-1 (LSB first): one LOP3 per plane.
template <int NA, int NB>
__device__ __forceinline__ uint32_t bs_less(const uint32_t (&a)[NA], const uint32_t (&b)[NB]) {
    constexpr int N = NA > NB ? NA : NB;
    uint32_t lt = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t ai = i < NA ? a[i] : 0u;
        const uint32_t bi = i < NB ? b[i] : 0u;
        lt = lop3<0x8E>(ai, bi, lt);  // (~ai & bi) | (~(ai ^ bi) & lt)
    }
    return lt;
}

// sel ? x : y, one LOP3.
__device__ __forceinline__ uint32_t bs_select(uint32_t x, uint32_t y, uint32_t sel) {
    return lop3<0xE4>(x, y, sel);
}

// counter += v (bit-sliced), truncating at NC planes.
template <int NC, int NV>
__device__ __forceinline__ void bs_add(uint32_t (&c)[NC], const uint32_t (&v)[NV]) {
    uint32_t carry = 0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        const uint32_t vi = i < NV ? v[i] : 0u;
        const uint32_t s = c[i] ^ vi ^ carry;
        carry = (c[i] & vi) | (carry & (c[i] ^ vi));
        c[i] = s;
    }
}

// Population count of N one-bit planes into NO planes (generic ripple form).
template <int N, int NO>
__device__ __forceinline__ void bs_popcount(const uint32_t* x, uint32_t (&o)[NO]) {
#pragma unroll
    for (int i = 0; i < NO; ++i) o[i] = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        uint32_t carry = x[k];
#pragma unroll
        for (int i = 0; i < NO; ++i) {
            const uint32_t t = o[i] & carry;
            o[i] ^= carry;
            carry = t;
        }
    }
}

// Mask of pairs whose counter value is <= the uniform constant e.
template <int NC>
__device__ __forceinline__ uint32_t bs_le_const(const uint32_t (&c)[NC], uint32_t e) {
    // c <= e  <=>  !(e < c)
    uint32_t lt = 0;  // running "e < c"
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        const uint32_t ei = ((e >> i) & 1u) ? ~0u : 0u;
        lt = (~ei & c[i]) | (~(ei ^ c[i]) & lt);
    }
    // bits of e above NC planes: if any set, every counter is below e.
    if (NC < 32 && (e >> NC) != 0u) return ~0u;
    return ~lt;
}

}  // namespace sb
