// The reference's Shouji unit tests (proj/tests/test_shouji.cpp), re-expressed
// against the C++ host mirror (include/shouji_b200.hpp): every decision below
// runs on the GPU through the C ABI. Exit code = number of failed checks.
#include <cstdio>
#include <random>
#include <string>

#include "shouji_b200.hpp"

using namespace shouji_b200;

static int failures = 0;
#define CHECK(x)                                                              \
    do {                                                                      \
        if (!(x)) {                                                           \
            std::fprintf(stderr, "%s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #x); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                              \
    do {                                                                      \
        bool ok_ = false;                                                     \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const T&) {                                                  \
            ok_ = true;                                                       \
        } catch (...) {                                                       \
        }                                                                     \
        if (!ok_) {                                                           \
            std::fprintf(stderr, "%s:%d %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static packed_sequence seq(const std::string& s) { return packed_sequence::from_string(s); }

static std::string random_dna(std::mt19937_64& rng, std::size_t len, bool with_n = false) {
    std::string s(len, 'A');
    for (auto& c : s) c = with_n ? "ACGTN"[rng() % 5] : "ACGT"[rng() % 4];
    return s;
}

static bool chars_match(char a, char b) { return a != 'N' && b != 'N' && a == b; }

int main() {
    const std::string golden_text = "GGTGCAGAGCTC", golden_pattern = "GGTGAGAGTTGT";
    {  // test_shouji.cpp:81-87
        const auto d = shouji_filter(seq(golden_pattern), seq(golden_text), 3);
        CHECK(d.accept);
        CHECK(d.edit_estimate == 3);
        CHECK(d.bits.to_string() == "000010000101");
        CHECK(d.bits.count_zeros() == 9);
    }
    {  // :89-93
        const auto d = shouji_filter(seq(golden_pattern), seq(golden_text), 2);
        CHECK(!d.accept);
        CHECK(d.edit_estimate > 2);
    }
    {  // :95-104 identical pairs always pass with estimate 0
        std::mt19937_64 rng(29);
        for (int it = 0; it < 30; ++it) {
            const auto s = random_dna(rng, 1 + rng() % 120);
            const auto e = std::uint32_t(rng() % 6);
            const auto d = shouji_filter(seq(s), seq(s), e);
            CHECK(d.accept && d.edit_estimate == 0);
        }
    }
    {  // :106-123 at threshold zero the estimate is the Hamming distance
        std::mt19937_64 rng(31);
        for (int it = 0; it < 200; ++it) {
            const std::size_t m = 1 + rng() % 50;
            const auto a = random_dna(rng, m, true);
            std::string b = a;
            const std::size_t muts = rng() % (m + 1);
            for (std::size_t k = 0; k < muts; ++k) b[rng() % m] = "ACGTN"[rng() % 5];
            std::uint32_t ham = 0;
            for (std::size_t i = 0; i < m; ++i) ham += !chars_match(a[i], b[i]);
            const auto d = shouji_filter(seq(b), seq(a), 0);
            CHECK(d.edit_estimate == ham);
            CHECK(d.accept == (ham == 0));
        }
    }
    {  // :125-137 accept agrees with the estimate against the threshold
        std::mt19937_64 rng(37);
        for (int it = 0; it < 200; ++it) {
            const std::size_t m = 1 + rng() % 100;
            const auto e = std::uint32_t(rng() % (m + 2));
            const auto d = shouji_filter(seq(random_dna(rng, m)), seq(random_dna(rng, m)), e);
            CHECK(d.accept == (d.edit_estimate <= e));
            CHECK(d.bits.size() == m);
            CHECK(d.edit_estimate == d.bits.count_ones());
        }
    }
    {  // :163-184 the estimate never exceeds the Hamming distance
        std::mt19937_64 rng(43);
        for (int it = 0; it < 300; ++it) {
            const std::size_t m = 4 + rng() % 120;
            const auto e = std::uint32_t(rng() % 8);
            if (e + 1 > m) continue;
            const auto a = random_dna(rng, m, true);
            auto b = a;
            const std::size_t muts = rng() % (m / 2 + 1);
            for (std::size_t k = 0; k < muts; ++k) b[rng() % m] = "ACGTN"[rng() % 5];
            std::uint32_t ham = 0;
            for (std::size_t i = 0; i < m; ++i) ham += !chars_match(a[i], b[i]);
            CHECK(shouji_filter(seq(b), seq(a), e).edit_estimate <= ham);
        }
    }
    {  // :186-205 compensating indels (frozen counterexample)
        const std::string text =
            "CACCATCCCAGAGCCACACGGTGCCGCAGTCGTAGTCAACGCGGACGTGTGCTATATAGTAACGTGAC"
            "AAATCAGGTTCACTGCGCTCTGCGCCATCGAT";
        const std::string pattern =
            "CACCATCCCAGAGCCACACGGTCGCCGCAGTCGTAGTCAACGCGGACGTGTGTATATAGTAACGTGAC"
            "AAATCAGGTTCACTGCGCTCTGCGCCATCGAT";
        const auto d = shouji_filter(seq(pattern), seq(text), 2);
        CHECK(!d.accept);
        CHECK(d.edit_estimate == 3);
        CHECK(shouji_filter(seq(pattern), seq(text), 3).accept);
    }
    {  // :207-226 short-circuit and validation
        const auto d = shouji_filter(seq("ACGT"), seq("TGCA"), 4);
        CHECK(d.accept && d.edit_estimate == 0 && d.bits.count_ones() == 0);
        CHECK_THROWS_AS(shouji_filter(seq("ACGT"), seq("ACG"), 1), length_mismatch_error);
        CHECK_THROWS_AS(shouji_filter(seq("ACGT"), seq("ACGT"), 1, 2), invalid_parameters_error);
        CHECK_THROWS_AS(shouji_filter(seq("ACGT"), seq("ACGT"), 1, 9), invalid_parameters_error);
        CHECK_THROWS_AS(shouji_filter(seq("ACGT"), seq("ACGT"), 99, 9), invalid_parameters_error);
        CHECK_THROWS_AS(seq(""), empty_sequence_error);
        CHECK_THROWS_AS(seq("acgt"), illegal_character_error);
    }
    {  // batch path: 4096 pairs, each compared with the per-pair call
        std::mt19937_64 rng(47);
        const std::size_t n = 4096, m = 100;
        std::string t(n * m, 'A'), p(n * m, 'A');
        for (std::size_t i = 0; i < n; ++i) {
            const auto a = random_dna(rng, m);
            auto b = a;
            for (int k = 0; k < 6; ++k) b[rng() % m] = "ACGT"[rng() % 4];
            t.replace(i * m, m, a);
            p.replace(i * m, m, b);
        }
        const auto r = shouji_filter_batch(reinterpret_cast<const std::uint8_t*>(t.data()),
                                           reinterpret_cast<const std::uint8_t*>(p.data()), m, n,
                                           m, 5, 4, true);
        for (std::size_t i = 0; i < n; i += 97) {
            const auto d = shouji_filter(seq(p.substr(i * m, m)), seq(t.substr(i * m, m)), 5);
            CHECK(d.accept == r.accepted(i));
            CHECK(d.edit_estimate == r.estimates[i]);
        }
        p[777 * m + 13] = 'x';
        CHECK_THROWS_AS(shouji_filter_batch(reinterpret_cast<const std::uint8_t*>(t.data()),
                                            reinterpret_cast<const std::uint8_t*>(p.data()), m, n,
                                            m, 5),
                        illegal_character_error);
    }
    {  // MAGNET through the same mirror (proj/tests/test_magnet.cpp:79-91,150-170)
        const auto d = magnet_filter(seq("GGTGAGAGTTGT"), seq("GGTGCAGAGCTC"), 3);
        CHECK(d.accept && d.edit_estimate == 3 && d.bits.count_zeros() == 9);
        CHECK(d.bits.to_string() == "000010000101");
        const auto big = magnet_filter(seq("ACGT"), seq("TGCA"), 7);
        CHECK(big.accept && big.edit_estimate == 0);
        CHECK_THROWS_AS(magnet_filter(seq("ACGT"), seq("ACG"), 1), length_mismatch_error);
        const auto via = run_filter(filter_algo::magnet, seq("GGTGAGAGTTGT"), seq("GGTGCAGAGCTC"), 3);
        CHECK(via.edit_estimate == 3);
        std::mt19937_64 rng(59);
        const std::size_t n = 2048, m = 150;
        std::string t(n * m, 'A'), p(n * m, 'A');
        for (std::size_t i = 0; i < n; ++i) {
            const auto a = random_dna(rng, m);
            auto b = a;
            for (int k = 0; k < 8; ++k) b[rng() % m] = "ACGT"[rng() % 4];
            t.replace(i * m, m, a);
            p.replace(i * m, m, b);
        }
        const auto r = magnet_filter_batch(reinterpret_cast<const std::uint8_t*>(t.data()),
                                           reinterpret_cast<const std::uint8_t*>(p.data()), m, n,
                                           m, 7, true);
        for (std::size_t i = 0; i < n; i += 61) {
            const auto one = magnet_filter(seq(p.substr(i * m, m)), seq(t.substr(i * m, m)), 7);
            CHECK(one.accept == r.accepted(i));
            CHECK(one.edit_estimate == r.estimates[i]);
            CHECK(one.edit_estimate == one.bits.count_ones());
        }
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures;
}
