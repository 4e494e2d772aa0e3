// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library, whose sources are
// compiled where they lie under /root/reference/proj/src by oracle/Makefile.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
// `--impl reference` arm) may load the resulting oracle/_ref/libprefilter_ref.so.
//
// Every entry point calls the reference's own public API:
//   prefilter::generate_pairs        proj/src/dataset.cpp:71-126
//   prefilter::packed_sequence       proj/src/packed_sequence.cpp:7-34
//   prefilter::shouji_filter         proj/src/shouji.cpp:41-58
//   prefilter::parallel_for_pairs    proj/src/evaluate.cpp:23-48
//   prefilter::banded_edit_distance  proj/src/edit_distance.cpp:26-70
//   prefilter::magnet_filter         proj/src/magnet.cpp
// Errors are mapped onto the status codes of include/shouji_b200.h so the
// parity tests can compare error behaviour one to one.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "prefilter/dataset.hpp"
#include "prefilter/edit_distance.hpp"
#include "prefilter/errors.hpp"
#include "prefilter/evaluate.hpp"
#include "prefilter/magnet.hpp"
#include "prefilter/shouji.hpp"

namespace {

// Must agree with pf_status in include/shouji_b200.h.
enum : int {
    kOk = 0,
    kEmptySequence = 1,
    kIllegalCharacter = 2,
    kLengthMismatch = 3,
    kThresholdTooLarge = 4,
    kOutOfBand = 5,
    kParse = 6,
    kInvalidParameters = 7,
    kOther = 99,
};

struct ref_error {
    int code = kOk;
    std::uint64_t pair = 0;
    int field = 0;  // 0 = text, 1 = pattern
    std::uint64_t position = 0;
    int byte = 0;
};

int map_exception(const std::exception_ptr& ep, ref_error* err) {
    try {
        std::rethrow_exception(ep);
    } catch (const prefilter::illegal_character_error& e) {
        if (err) {
            err->code = kIllegalCharacter;
            err->position = e.position();
            err->byte = static_cast<unsigned char>(e.byte());
        }
        return kIllegalCharacter;
    } catch (const prefilter::empty_sequence_error&) {
        if (err) err->code = kEmptySequence;
        return kEmptySequence;
    } catch (const prefilter::length_mismatch_error&) {
        if (err) err->code = kLengthMismatch;
        return kLengthMismatch;
    } catch (const prefilter::threshold_too_large_error&) {
        if (err) err->code = kThresholdTooLarge;
        return kThresholdTooLarge;
    } catch (const prefilter::out_of_band_error&) {
        if (err) err->code = kOutOfBand;
        return kOutOfBand;
    } catch (const prefilter::parse_error&) {
        if (err) err->code = kParse;
        return kParse;
    } catch (const prefilter::invalid_parameters_error&) {
        if (err) err->code = kInvalidParameters;
        return kInvalidParameters;
    } catch (...) {
        if (err) err->code = kOther;
        return kOther;
    }
}

struct dataset_handle {
    std::vector<prefilter::packed_sequence> text;
    std::vector<prefilter::packed_sequence> pattern;
    std::size_t m = 0;
};

}  // namespace

extern "C" {

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// generate_pairs({seed, count, len, {lo, hi}}) exported as ASCII records:
// text[i] at text + i*stride, pattern[i] at pattern + i*stride (len bytes each).
int ref_generate_pairs(std::uint64_t seed, std::size_t count, std::size_t len,
                       std::uint32_t lo, std::uint32_t hi, char* text, char* pattern,
                       std::size_t stride) {
    try {
        const auto ds = prefilter::generate_pairs({seed, count, len, {lo, hi}});
        for (std::size_t i = 0; i < ds.pairs.size(); ++i) {
            const std::string t = ds.pairs[i].text.to_string();
            const std::string p = ds.pairs[i].pattern.to_string();
            std::memcpy(text + i * stride, t.data(), len);
            std::memcpy(pattern + i * stride, p.data(), len);
        }
        return kOk;
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
}

// Pack n ASCII pairs with packed_sequence::from_string, text before pattern
// for each pair in order (the order load_pairs uses, dataset.cpp:28-30), so
// the first error reported is the one the reference would throw first.
void* ref_pack(const char* text, const char* pattern, std::size_t stride, std::size_t n,
               std::size_t m, int* err_code, std::uint64_t* err_pair, int* err_field,
               std::uint64_t* err_pos, int* err_byte) {
    auto* h = new dataset_handle;
    h->m = m;
    h->text.reserve(n);
    h->pattern.reserve(n);
    *err_code = kOk;
    for (std::size_t i = 0; i < n; ++i) {
        for (int field = 0; field < 2; ++field) {
            const char* src = (field == 0 ? text : pattern) + i * stride;
            try {
                auto seq = prefilter::packed_sequence::from_string({src, m});
                (field == 0 ? h->text : h->pattern).push_back(std::move(seq));
            } catch (...) {
                ref_error e;
                map_exception(std::current_exception(), &e);
                *err_code = e.code;
                *err_pair = i;
                *err_field = field;
                *err_pos = e.position;
                *err_byte = e.byte;
                delete h;
                return nullptr;
            }
        }
    }
    return h;
}

void ref_free(void* handle) { delete static_cast<dataset_handle*>(handle); }

// shouji_filter(pattern, text, e, width) for every packed pair through the
// reference's own static-chunk thread pool. accept_bitmap: LSB-first,
// ceil(n/32) words. estimates / bits may be null; bits holds words_per_pair
// u64 words per pair (the decision's bitvector words).
int ref_shouji_run(void* handle, std::uint32_t e, unsigned width, unsigned threads,
                   std::uint32_t* accept_bitmap, std::uint32_t* estimates, std::uint64_t* bits,
                   std::size_t words_per_pair) {
    auto* h = static_cast<dataset_handle*>(handle);
    const std::size_t n = h->text.size();
    std::vector<unsigned char> acc(n, 0);
    try {
        prefilter::parallel_for_pairs(n, threads, [&](std::size_t i) {
            const auto d = prefilter::run_filter(prefilter::filter_algo::shouji, h->pattern[i],
                                                 h->text[i], e, width);
            acc[i] = d.accept ? 1 : 0;
            if (estimates) estimates[i] = d.edit_estimate;
            if (bits) {
                const auto& w = d.bits.words();
                for (std::size_t k = 0; k < words_per_pair; ++k)
                    bits[i * words_per_pair + k] = k < w.size() ? w[k] : 0;
            }
        });
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
    if (accept_bitmap) {
        std::memset(accept_bitmap, 0, ((n + 31) / 32) * sizeof(std::uint32_t));
        for (std::size_t i = 0; i < n; ++i)
            if (acc[i]) accept_bitmap[i / 32] |= 1u << (i % 32);
    }
    return kOk;
}

// Same through magnet_filter (run_filter's other branch, evaluate.cpp:13-21).
int ref_magnet_run(void* handle, std::uint32_t e, unsigned threads, std::uint32_t* accept_bitmap,
                   std::uint32_t* estimates) {
    auto* h = static_cast<dataset_handle*>(handle);
    const std::size_t n = h->text.size();
    std::vector<unsigned char> acc(n, 0);
    try {
        prefilter::parallel_for_pairs(n, threads, [&](std::size_t i) {
            const auto d = prefilter::run_filter(prefilter::filter_algo::magnet, h->pattern[i],
                                                 h->text[i], e, 4);
            acc[i] = d.accept ? 1 : 0;
            if (estimates) estimates[i] = d.edit_estimate;
        });
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
    if (accept_bitmap) {
        std::memset(accept_bitmap, 0, ((n + 31) / 32) * sizeof(std::uint32_t));
        for (std::size_t i = 0; i < n; ++i)
            if (acc[i]) accept_bitmap[i / 32] |= 1u << (i % 32);
    }
    return kOk;
}

// banded_edit_distance(pattern, text, e): out[i] = distance, or -1 when the
// pair lies outside the band (std::nullopt).
int ref_banded_run(void* handle, std::uint32_t e, unsigned threads, std::int32_t* out) {
    auto* h = static_cast<dataset_handle*>(handle);
    const std::size_t n = h->text.size();
    try {
        prefilter::parallel_for_pairs(n, threads, [&](std::size_t i) {
            const auto d = prefilter::banded_edit_distance(h->pattern[i], h->text[i], e);
            out[i] = d ? std::int32_t(*d) : -1;
        });
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
    return kOk;
}

// Single-pair entry with the reference's argument order, for error-path tests:
// packs both strings (pattern first, as a caller would write
// shouji_filter(seq(pattern), seq(text), ...)) and filters.
int ref_shouji_one(const char* pattern, std::size_t pattern_len, const char* text,
                   std::size_t text_len, std::uint32_t e, unsigned width, int* accept,
                   std::uint32_t* estimate, char* bits_string) {
    try {
        const auto p = prefilter::packed_sequence::from_string({pattern, pattern_len});
        const auto t = prefilter::packed_sequence::from_string({text, text_len});
        const auto d = prefilter::shouji_filter(p, t, e, width);
        *accept = d.accept ? 1 : 0;
        *estimate = d.edit_estimate;
        if (bits_string) {
            const std::string s = d.bits.to_string();
            std::memcpy(bits_string, s.data(), s.size());
            bits_string[s.size()] = '\0';
        }
        return kOk;
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
}

// load_pairs (proj/src/dataset.cpp:13-44) over an in-memory TSV; on failure
// returns the mapped status and copies e.what() into msg.
int ref_load_pairs_tsv(const char* data, std::size_t len, std::size_t* n, std::size_t* m,
                       char* msg, std::size_t msglen) {
    std::istringstream in(std::string(data, len));
    try {
        const auto ds = prefilter::load_pairs(in, "<stream>");
        *n = ds.pairs.size();
        *m = ds.length;
        return kOk;
    } catch (const std::exception& e) {
        if (msg && msglen) {
            std::strncpy(msg, e.what(), msglen - 1);
            msg[msglen - 1] = '\0';
        }
        return map_exception(std::current_exception(), nullptr);
    }
}

// magnet_filter (proj/src/magnet.cpp:77-87) for one pair, plus the extraction
// list of recover_subsequences(map, budget) (:70-75) when budget is given:
// ext receives (diagonal, start, len, lo, hi) per extraction (up to max_ext).
int ref_magnet_one(const char* pattern, std::size_t pattern_len, const char* text,
                   std::size_t text_len, std::uint32_t e, int* accept, std::uint32_t* estimate,
                   char* bits_string, std::int64_t budget, std::int64_t* ext, std::size_t max_ext,
                   std::size_t* n_ext, char* rec_bits_string) {
    try {
        const auto p = prefilter::packed_sequence::from_string({pattern, pattern_len});
        const auto t = prefilter::packed_sequence::from_string({text, text_len});
        const auto d = prefilter::magnet_filter(p, t, e);
        *accept = d.accept ? 1 : 0;
        *estimate = d.edit_estimate;
        if (bits_string) {
            const std::string s = d.bits.to_string();
            std::memcpy(bits_string, s.data(), s.size());
            bits_string[s.size()] = '\0';
        }
        if (budget >= 0 && n_ext) {
            const auto rec = prefilter::recover_subsequences(
                prefilter::neighborhood_map(p, t, e), static_cast<std::uint32_t>(budget));
            *n_ext = rec.extractions.size();
            for (std::size_t k = 0; k < rec.extractions.size() && k < max_ext; ++k) {
                const auto& x = rec.extractions[k];
                ext[5 * k + 0] = x.diagonal;
                ext[5 * k + 1] = static_cast<std::int64_t>(x.start);
                ext[5 * k + 2] = static_cast<std::int64_t>(x.len);
                ext[5 * k + 3] = static_cast<std::int64_t>(x.lo);
                ext[5 * k + 4] = static_cast<std::int64_t>(x.hi);
            }
            if (rec_bits_string) {
                const std::string s = rec.bits.to_string();
                std::memcpy(rec_bits_string, s.data(), s.size());
                rec_bits_string[s.size()] = '\0';
            }
        }
        return kOk;
    } catch (...) {
        return map_exception(std::current_exception(), nullptr);
    }
}

// The packed_sequence planes of a packed batch (packed_sequence.hpp:44-53):
// out[i][k][w], k = 0 low_plane, 1 high_plane, 2 n_plane, ceil(m/64) words.
void ref_export_planes(void* handle, std::uint64_t* text_out, std::uint64_t* pattern_out) {
    auto* h = static_cast<dataset_handle*>(handle);
    for (std::size_t i = 0; i < h->text.size(); ++i) {
        for (int f = 0; f < 2; ++f) {
            const auto& ps = f == 0 ? h->text[i] : h->pattern[i];
            std::uint64_t* out = (f == 0 ? text_out : pattern_out);
            const std::size_t w = ps.low_plane().size();
            std::uint64_t* dst = out + i * 3 * w;
            for (std::size_t k = 0; k < w; ++k) {
                dst[k] = ps.low_plane()[k];
                dst[w + k] = ps.high_plane()[k];
                dst[2 * w + k] = ps.n_plane()[k];
            }
        }
    }
}

// longest_zero_run (proj/src/magnet.cpp:9-22) on a '0'/'1' string.
void ref_longest_zero_run(const char* bits, std::size_t nbits, std::size_t lo, std::size_t hi,
                          std::size_t* start, std::size_t* len) {
    prefilter::bitvector bv(nbits);
    for (std::size_t i = 0; i < nbits; ++i) bv.set(i, bits[i] == '1');
    const auto r = prefilter::longest_zero_run(bv, lo, hi);
    *start = r.start;
    *len = r.len;
}

}  // extern "C"
