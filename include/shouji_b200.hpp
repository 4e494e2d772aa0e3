// shouji_b200.hpp — C++ host mirror of the reference's Shouji interface over the C ABI.
//
// Drop-in for the reference types a caller of the hot path touches
// (namespace prefilter -> shouji_b200):
//   packed_sequence      proj/include/prefilter/packed_sequence.hpp:17-61
//   bitvector            proj/include/prefilter/bitvector.hpp:16-129 (read side)
//   filter_decision      proj/include/prefilter/filter_decision.hpp:12-16
//   shouji_filter        proj/include/prefilter/shouji.hpp:57-59
//   magnet_filter        proj/include/prefilter/magnet.hpp:55-57
//   error hierarchy      proj/include/prefilter/errors.hpp:11-84
// plus a batch call (the fast path) that replaces run_filter + parallel_for_pairs
// (proj/src/evaluate.cpp:13-48). Every decision is computed on the GPU by
// libshouji_b200.so; this header only marshals arguments and maps status codes
// onto the reference's exception types.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "shouji_b200.h"

namespace shouji_b200 {

inline constexpr unsigned min_window_width = 3;
inline constexpr unsigned default_window_width = 4;
inline constexpr unsigned max_window_width = 8;

// ---- errors (errors.hpp:11-84) ------------------------------------------------
class error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class empty_sequence_error : public error {
public:
    empty_sequence_error() : error("empty sequence") {}
};
class illegal_character_error : public error {
public:
    illegal_character_error(std::size_t position, char byte, std::uint64_t pair = 0,
                            unsigned field = 0)
        : error("illegal character '" + std::string(1, byte) + "' at position " +
                std::to_string(position)),
          position_(position), byte_(byte), pair_(pair), field_(field) {}
    std::size_t position() const noexcept { return position_; }
    char byte() const noexcept { return byte_; }
    std::uint64_t pair() const noexcept { return pair_; }
    unsigned field() const noexcept { return field_; }  // 0 text, 1 pattern

private:
    std::size_t position_;
    char byte_;
    std::uint64_t pair_;
    unsigned field_;
};
class length_mismatch_error : public error {
public:
    using error::error;
};
class threshold_too_large_error : public error {
public:
    using error::error;
};
class out_of_band_error : public error {
public:
    using error::error;
};
class parse_error : public error {
public:
    using error::error;
};
class invalid_parameters_error : public error {
public:
    using error::error;
};
// Not a reference class: no usable device / CUDA failure.
class device_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void throw_status(int st, const pf_error& e) {
    switch (st) {
        case PF_OK: return;
        case PF_ERR_EMPTY_SEQUENCE: throw empty_sequence_error();
        case PF_ERR_ILLEGAL_CHARACTER:
            throw illegal_character_error(e.position, static_cast<char>(e.byte), e.pair, e.field);
        case PF_ERR_LENGTH_MISMATCH: throw length_mismatch_error(e.message);
        case PF_ERR_THRESHOLD_TOO_LARGE: throw threshold_too_large_error(e.message);
        case PF_ERR_OUT_OF_BAND: throw out_of_band_error(e.message);
        case PF_ERR_PARSE: throw parse_error(e.message);
        case PF_ERR_INVALID_PARAMETERS: throw invalid_parameters_error(e.message);
        default:
            throw device_error(std::string(pf_status_string(st)) + ": " + e.message);
    }
}

// ---- bitvector (read side of bitvector.hpp) ---------------------------------------
class bitvector {
public:
    bitvector() = default;
    explicit bitvector(std::size_t nbits, bool value = false)
        : nbits_(nbits), words_((nbits + 63) / 64, value ? ~std::uint64_t{0} : 0) {
        clear_tail();
    }
    static bitvector from_words(std::vector<std::uint64_t> words, std::size_t nbits) {
        bitvector bv;
        bv.nbits_ = nbits;
        bv.words_ = std::move(words);
        bv.words_.resize((nbits + 63) / 64, 0);
        bv.clear_tail();
        return bv;
    }
    std::size_t size() const { return nbits_; }
    bool get(std::size_t i) const { return (words_[i >> 6] >> (i & 63)) & 1u; }
    std::size_t count_ones() const {
        std::size_t n = 0;
        for (auto w : words_) n += static_cast<std::size_t>(__builtin_popcountll(w));
        return n;
    }
    std::size_t count_zeros() const { return nbits_ - count_ones(); }
    const std::vector<std::uint64_t>& words() const { return words_; }
    std::string to_string() const {
        std::string s(nbits_, '0');
        for (std::size_t i = 0; i < nbits_; ++i)
            if (get(i)) s[i] = '1';
        return s;
    }
    friend bool operator==(const bitvector&, const bitvector&) = default;

private:
    void clear_tail() {
        if (nbits_ & 63) words_.back() &= (std::uint64_t{1} << (nbits_ & 63)) - 1;
    }
    std::size_t nbits_ = 0;
    std::vector<std::uint64_t> words_;
};

struct filter_decision {
    bool accept = false;
    std::uint32_t edit_estimate = 0;
    bitvector bits;
};

// ---- packed_sequence (packed_sequence.hpp:17-61) ------------------------------------
// Holds the validated bases; the device packs them into planes.
class packed_sequence {
public:
    static packed_sequence from_string(std::string_view raw) {
        if (raw.empty()) throw empty_sequence_error();
        for (std::size_t i = 0; i < raw.size(); ++i) {
            const char c = raw[i];
            if (c != 'A' && c != 'C' && c != 'G' && c != 'T' && c != 'N')
                throw illegal_character_error(i, c);
        }
        packed_sequence s;
        s.bases_.assign(raw.begin(), raw.end());
        return s;
    }
    std::string to_string() const { return bases_; }
    std::size_t size() const { return bases_.size(); }
    bool is_n(std::size_t i) const { return bases_[i] == 'N'; }
    unsigned code(std::size_t i) const {
        switch (bases_[i]) {
            case 'C': return 1;
            case 'G': return 2;
            case 'T': return 3;
            default: return 0;
        }
    }
    char base_at(std::size_t i) const { return bases_[i]; }
    const char* data() const { return bases_.data(); }
    friend bool operator==(const packed_sequence&, const packed_sequence&) = default;

private:
    std::string bases_;
};

inline bool bases_match(const packed_sequence& a, std::size_t i, const packed_sequence& b,
                        std::size_t j) {
    return !a.is_n(i) && !b.is_n(j) && a.code(i) == b.code(j);
}

// ---- device context ------------------------------------------------------------
class context {
public:
    explicit context(const std::vector<int>& devices = {}) {
        const int st = pf_ctx_create(devices.empty() ? nullptr : devices.data(),
                                     static_cast<int>(devices.size()), &ctx_);
        if (st != PF_OK) {
            pf_error e{};
            throw_status(st, e);
        }
    }
    ~context() { pf_ctx_destroy(ctx_); }
    context(const context&) = delete;
    context& operator=(const context&) = delete;
    pf_ctx* get() const { return ctx_; }

    static context& default_context() {
        static context ctx;
        return ctx;
    }

private:
    pf_ctx* ctx_ = nullptr;
};

// ---- the hot path ----------------------------------------------------------------
// shouji_filter(pattern = read, text = reference segment, e, width) — shouji.hpp:57-59.
inline filter_decision shouji_filter(const packed_sequence& pattern, const packed_sequence& text,
                                     std::uint32_t e, unsigned width = default_window_width,
                                     context& ctx = context::default_context()) {
    pf_error err{};
    int accept = 0;
    std::uint32_t est = 0;
    std::vector<std::uint64_t> words((text.size() + 63) / 64 + 1, 0);
    const int st = pf_shouji_filter_one(ctx.get(), pattern.data(), pattern.size(), text.data(),
                                        text.size(), e, width, &accept, &est, words.data(), &err);
    throw_status(st, err);
    return {accept != 0, est, bitvector::from_words(std::move(words), text.size())};
}

// Batch result for n pairs.
struct batch_result {
    std::vector<std::uint32_t> accept_bitmap;  // LSB-first, ceil(n/32) words
    std::vector<std::uint32_t> estimates;      // empty unless requested
    bool accepted(std::size_t i) const { return (accept_bitmap[i / 32] >> (i % 32)) & 1u; }
};

// The fast path: n pairs of ASCII records (text[i] at text + i*stride, pattern[i] at
// pattern + i*stride, m bytes each), filtered on every device of ctx.
inline batch_result shouji_filter_batch(const std::uint8_t* text, const std::uint8_t* pattern,
                                        std::size_t stride, std::size_t n, std::uint32_t m,
                                        std::uint32_t e, unsigned width = default_window_width,
                                        bool estimates = false,
                                        context& ctx = context::default_context()) {
    batch_result r;
    r.accept_bitmap.assign((n + 31) / 32, 0);
    if (estimates) r.estimates.assign(n, 0);
    pf_error err{};
    const int st = pf_shouji_filter_batch(ctx.get(), text, pattern, stride, n, m, e, width,
                                          r.accept_bitmap.data(),
                                          estimates ? r.estimates.data() : nullptr, nullptr, &err);
    throw_status(st, err);
    return r;
}

// ---- MAGNET (proj/src/magnet.cpp) -------------------------------------------------
// magnet_filter(pattern = read, text = reference segment, e) — magnet.hpp:55-57.
inline filter_decision magnet_filter(const packed_sequence& pattern, const packed_sequence& text,
                                     std::uint32_t e, context& ctx = context::default_context()) {
    pf_error err{};
    int accept = 0;
    std::uint32_t est = 0;
    std::vector<std::uint64_t> words((text.size() + 63) / 64 + 1, 0);
    const int st = pf_magnet_filter_one(ctx.get(), pattern.data(), pattern.size(), text.data(),
                                        text.size(), e, &accept, &est, words.data(), &err);
    throw_status(st, err);
    return {accept != 0, est, bitvector::from_words(std::move(words), text.size())};
}

// filter_algo / run_filter (evaluate.hpp:11-19, evaluate.cpp:13-21).
enum class filter_algo { shouji, magnet };
inline filter_decision run_filter(filter_algo algo, const packed_sequence& pattern,
                                  const packed_sequence& text, std::uint32_t e,
                                  unsigned width = default_window_width,
                                  context& ctx = context::default_context()) {
    return algo == filter_algo::magnet ? magnet_filter(pattern, text, e, ctx)
                                       : shouji_filter(pattern, text, e, width, ctx);
}

// MAGNET over n pairs of ASCII records (layout as shouji_filter_batch).
inline batch_result magnet_filter_batch(const std::uint8_t* text, const std::uint8_t* pattern,
                                        std::size_t stride, std::size_t n, std::uint32_t m,
                                        std::uint32_t e, bool estimates = false,
                                        context& ctx = context::default_context()) {
    batch_result r;
    r.accept_bitmap.assign((n + 31) / 32, 0);
    if (estimates) r.estimates.assign(n, 0);
    pf_error err{};
    const int st = pf_magnet_filter_batch(ctx.get(), text, pattern, stride, n, m, e,
                                          r.accept_bitmap.data(),
                                          estimates ? r.estimates.data() : nullptr, nullptr, &err);
    throw_status(st, err);
    return r;
}

}  // namespace shouji_b200
