"""Pin the CPU oracle (oracle/shouji_oracle.c) before trusting it as the checker.

1. The reference's own golden vectors and known-answer tests for this path
   (proj/tests/test_neighborhood.cpp, test_shouji.cpp, test_packed_sequence.cpp,
   acceptance_tests.cpp + proj/test_output.txt) — hard-coded below with citations.
2. The committed fixtures in tests/golden/, produced by the unmodified reference
   library (tests/golden/make_golden.py).
3. When oracle/_ref is built (this container): seeded random comparisons against
   the reference library itself.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle import OracleError

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDEN_TEXT = "GGTGCAGAGCTC"      # test_shouji.cpp:16, Fig. 1
GOLDEN_PATTERN = "GGTGAGAGTTGT"   # test_shouji.cpp:17


def bits_str(row):
    return "".join("1" if b else "0" for b in row)


def popcount_words(words):
    return sum(bin(int(w)).count("1") for w in np.asarray(words).ravel())


# --- reference known-answer tests ------------------------------------------------

def test_neighborhood_golden_pair(oracle):
    # test_neighborhood.cpp:20-31
    nm = oracle.neighborhood(GOLDEN_PATTERN, GOLDEN_TEXT, 3)
    expect = {-3: "111011000111", -2: "111011111101", -1: "101110000101", 0: "000011111111",
              1: "011110011101", 2: "101011110111", 3: "011111111111"}
    for d, s in expect.items():
        assert bits_str(nm[d + 3]) == s, d


def test_neighborhood_boundary_rule(oracle):
    # test_neighborhood.cpp:60-69
    nm = oracle.neighborhood("AAAAAA", "AAAAAA", 2)
    assert [bits_str(r) for r in nm] == ["110000", "100000", "000000", "000001", "000011"]


def test_neighborhood_matches_cell_definition(oracle):
    # test_neighborhood.cpp:43-58 and the cross-word case :103-117 (e=150)
    rng = np.random.default_rng(11)
    for m, e in [(80, 8), (37, 5), (200, 150), (5, 4)]:
        t = "".join(rng.choice(list("ACGTN"), m))
        p = "".join(rng.choice(list("ACGTN"), m))
        nm = oracle.neighborhood(p, t, e)
        for d in range(-e, e + 1):
            for j in range(m):
                i = j + d
                mis = True if (i < 0 or i >= m) else not (p[i] == t[j] and p[i] != "N")
                assert nm[d + e][j] == mis


def test_golden_decision(oracle):
    # test_shouji.cpp:81-93
    acc, est, bits = oracle.shouji_one(GOLDEN_PATTERN, GOLDEN_TEXT, 3)
    assert acc and est == 3 and bits == "000010000101" and bits.count("0") == 9
    acc, est, _ = oracle.shouji_one(GOLDEN_PATTERN, GOLDEN_TEXT, 2)
    assert not acc and est > 2


def test_tie_break_pair(oracle):
    # test_shouji.cpp:51-60: d=+1 slice 1010 wins the first window of AGTC/GACT
    nm = oracle.neighborhood("AGTC", "GACT", 1)
    s = {d: int("".join(str(b) for b in nm[d + 1][:4][::-1]), 2) for d in (-1, 0, 1)}
    assert s[1] == 0b1010 and bin(s[-1]).count("1") == 2


def test_compensating_indel_false_reject(oracle):
    # test_shouji.cpp:186-205 (frozen 100-base counterexample)
    text = ("CACCATCCCAGAGCCACACGGTGCCGCAGTCGTAGTCAACGCGGACGTGTGCTATATAGTAACGTGAC"
            "AAATCAGGTTCACTGCGCTCTGCGCCATCGAT")
    pattern = ("CACCATCCCAGAGCCACACGGTCGCCGCAGTCGTAGTCAACGCGGACGTGTGTATATAGTAACGTGAC"
               "AAATCAGGTTCACTGCGCTCTGCGCCATCGAT")
    acc, est, _ = oracle.shouji_one(pattern, text, 2)
    assert not acc and est == 3
    assert oracle.shouji_one(pattern, text, 3)[0]


def test_short_circuit_and_width_errors(oracle):
    # test_shouji.cpp:207-226
    acc, est, bits = oracle.shouji_one("ACGT", "TGCA", 4)
    assert acc and est == 0 and bits == "0000"
    with pytest.raises(OracleError) as ei:
        oracle.shouji_one("ACGT", "ACG", 1)
    assert ei.value.code == 3  # length_mismatch
    for w in (2, 9):
        with pytest.raises(OracleError) as ei:
            oracle.shouji_one("ACGT", "ACGT", 1, w)
        assert ei.value.code == 7  # invalid_parameters
    with pytest.raises(OracleError) as ei:  # width checked before the e >= m short-circuit
        oracle.shouji_one("ACGT", "ACGT", 99, 9)
    assert ei.value.code == 7


def test_hamming_at_e0_and_upper_bound(oracle):
    # test_shouji.cpp:106-123 (E=0 estimate == Hamming, N never matches) and :163-184
    rng = np.random.default_rng(31)
    for _ in range(200):
        m = int(rng.integers(1, 51))
        a = rng.choice(list("ACGTN"), m)
        b = a.copy()
        for _ in range(int(rng.integers(0, m + 1))):
            b[rng.integers(0, m)] = rng.choice(list("ACGTN"))
        ham = sum(1 for x, y in zip(a, b) if not (x == y and x != "N"))
        acc, est, _ = oracle.shouji_one("".join(b), "".join(a), 0)
        assert est == ham and acc == (ham == 0)
        e = int(rng.integers(0, 8))
        if e < m:
            assert oracle.shouji_one("".join(b), "".join(a), e)[1] <= ham


def test_illegal_bytes(oracle):
    # test_packed_sequence.cpp:37-49: position and byte of the first bad byte; lower case rejected
    t = np.frombuffer(b"ACGTACGT" * 4, np.uint8).reshape(4, 8).copy()
    p = t.copy()
    p[2, 5] = ord("a")
    t[3, 0] = ord("X")
    with pytest.raises(OracleError) as ei:
        oracle.shouji_batch(t, p, 1)
    assert (ei.value.code, ei.value.pair, ei.value.field, ei.value.position, ei.value.byte) == \
        (2, 2, 1, 5, ord("a"))


# --- fixtures from the reference library ----------------------------------------

def test_oracle_matches_edge_fixtures(oracle):
    z = np.load(os.path.join(GOLD, "edge_cases.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files})
    assert len(keys) > 300
    for k in keys:
        m, width, e = (int(x) for x in z[f"{k}_meta"])
        acc, est, bits = oracle.shouji_batch(z[f"{k}_text"], z[f"{k}_pattern"], e, width, bits=True)
        assert (acc == z[f"{k}_accept"]).all(), (k, m, width, e)
        assert (est == z[f"{k}_est"]).all(), (k, m, width, e)
        assert (bits == z[f"{k}_bits"]).all(), (k, m, width, e)


def test_oracle_generator_reproduces_config0(oracle):
    # generate_pairs restated (dataset.cpp:71-126): byte-identical 1M-pair config 0
    z = np.load(os.path.join(GOLD, "config0.npz"))
    t, p = oracle.generate_pairs(1809078580, 1_000_000, 100, 0, 10)
    assert hashlib.sha256(t.tobytes() + p.tobytes()).digest() == z["text_sha256"].tobytes()
    acc, est, _ = oracle.shouji_batch(t, p, 5)
    assert hashlib.sha256(acc.tobytes()).digest() == z["accept_sha256"].tobytes()
    assert int(est.astype(np.int64).sum()) == int(z["est_sum"])


@pytest.mark.parametrize("m,e,lost", [(100, 2, 583), (100, 5, 41), (150, 7, 7), (250, 15, 0)])
def test_acceptance_criterion2_counts(oracle, m, e, lost):
    # acceptance_tests.cpp:93-128; proj/test_output.txt:11 records 583/41/7/0
    z = np.load(os.path.join(GOLD, f"fr_m{m}_e{e}.npz"))
    t, p = oracle.generate_pairs(int(z["seed"]), 100_000, m, 0, e)
    acc, est, _ = oracle.shouji_batch(t, p, e)
    assert (acc == z["accept"]).all() and (est == z["est"]).all()
    a = np.unpackbits(acc.view(np.uint8), bitorder="little")[:100_000].astype(bool)
    assert int((z["similar"] & ~a).sum()) == lost


def _bools(acc, n):
    return np.unpackbits(np.ascontiguousarray(acc).view(np.uint8), bitorder="little")[:n].astype(bool)


def test_acceptance_criterion3_exact_at_zero(oracle):
    # acceptance_tests.cpp:132-146 (criterion 3): at e=0 the decision is equality;
    # SURVEY 8(c) records 3407/10000 identical pairs, 0 violations
    t, p = oracle.generate_pairs(3300, 10_000, 100, 0, 2)
    same = (t == p).all(axis=1)
    acc, _, _ = oracle.shouji_batch(t, p, 0)
    assert int(same.sum()) == 3407
    assert (_bools(acc, 10_000) == same).all()


def test_acceptance_criterion5_width_trend(oracle):
    # acceptance_tests.cpp:180-203 (criterion 5): over criterion 2's similar pairs,
    # width 4 loses 631 (= 583+41+7+0) and widths 5+6 lose 30,783 (proj/test_output.txt:19)
    lost4 = lost56 = 0
    for m, e in [(100, 2), (100, 5), (150, 7), (250, 15)]:
        z = np.load(os.path.join(GOLD, f"fr_m{m}_e{e}.npz"))
        t, p = oracle.generate_pairs(int(z["seed"]), 100_000, m, 0, e)
        for w in (4, 5, 6):
            acc, _, _ = oracle.shouji_batch(t, p, e, w, estimates=False)
            lost = int((z["similar"] & ~_bools(acc, 100_000)).sum())
            if w == 4:
                lost4 += lost
            else:
                lost56 += lost
    assert (lost4, lost56) == (631, 30_783)


@pytest.mark.parametrize("seed,e,subs_hi,fa_rate", [(7702, 2, 4, 0.257745), (7705, 5, 10, 0.643066)])
def test_acceptance_criterion7_rate_structure(oracle, seed, e, subs_hi, fa_rate):
    # acceptance_tests.cpp:246-310 (criterion 7): substitution-only pairs, evaluate()
    # (evaluate.cpp:50-79): fa_rate = false accepts / oracle rejects, printed with
    # std::to_string (6 decimals); Shouji never rejects a similar pair here
    t, p = oracle.substitution_pairs(seed, 20_000, 100, subs_hi)
    a = _bools(oracle.shouji_batch(t, p, e, estimates=False)[0], 20_000)
    within = np.array([oracle.banded_edit_distance(p[i].tobytes(), t[i].tobytes(), e) >= 0
                       for i in range(20_000)])
    assert round(float((a & ~within).sum()) / float((~within).sum()), 6) == fa_rate
    assert int((~a & within).sum()) == 0


# --- the reference library itself (build container only) -------------------------

def test_reference_unit_tests_pass_on_ref_build():
    # The reference's own unit tests (proj/tests/test_*.cpp except test_cli.cpp),
    # compiled unmodified against our doctest-compatible shim and linked with the
    # same objects as oracle/_ref: 80 cases, 175,923 checks, 0 failures
    import subprocess
    if not os.path.exists("/root/reference/proj/tests/test_shouji.cpp"):
        pytest.skip("reference tests absent (GPU box)")
    odir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")
    subprocess.run(["make", "-s", "-C", odir, "unit"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(odir, "_ref", "unit_tests")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split() == ["cases", "80", "checks", "175923", "failures", "0",
                                "failed_cases", "0"], r.stdout


def test_oracle_vs_reference_random(oracle, reference):
    rng = np.random.default_rng(7)
    for m, e, w in [(100, 5, 4), (150, 7, 4), (250, 25, 4), (64, 31, 4), (100, 5, 6), (33, 3, 3)]:
        t = np.frombuffer(b"ACGTN", np.uint8)[rng.integers(0, 5, size=(3000, m))]
        p = t.copy()
        mask = rng.random(p.shape) < 0.1
        p[mask] = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, size=int(mask.sum()))]
        a1, e1, b1 = oracle.shouji_batch(t, p, e, w, bits=True)
        a2, e2, b2 = reference.shouji_batch(t, p, e, w, bits=True)
        assert (a1 == a2).all() and (e1 == e2).all() and (b1 == b2).all()


def test_oracle_generator_vs_reference(oracle, reference):
    for seed, m, lo, hi in [(1, 100, 0, 10), (99, 37, 3, 3), (5, 250, 0, 50), (8, 1, 0, 1)]:
        t1, p1 = oracle.generate_pairs(seed, 5000, m, lo, hi)
        t2, p2 = reference.generate_pairs(seed, 5000, m, lo, hi)
        assert (t1 == t2).all() and (p1 == p2).all()


def test_estimate_can_exceed_hamming(oracle, reference):
    """The reference's comment "the estimate never exceeds the Hamming distance"
    (proj/tests/test_shouji.cpp:163-166) is not a theorem: this substitution-only
    pair (found in a 30M-pair config-1 run) has Hamming distance 2 and the
    reference library's estimate at E=5 is 3. Parity follows the implementation,
    so the oracle must agree with the library here, not with the comment."""
    t = ("AATTGCCAATATCGATAGTTTCAGCTGAGGATCCATCTCGGCGCTTAATGGGATGAGGCCGAATCCAGGACGACGTATCGG"
         "TCGGCGAGCAAGTTTACTG")
    p = ("AATTGCCAATATCGATAGTTTCAGCTGAGGATCCATCTCGGCGCTTAATGGGATGAGGCCGAATCCAGGACGACGTATCGG"
         "TCGGCGAGCACGGTTACTG")
    assert sum(a != b for a, b in zip(t, p)) == 2
    assert reference.shouji_one(p, t, 5)[1] == 3
    assert oracle.shouji_one(p, t, 5) == reference.shouji_one(p, t, 5)
