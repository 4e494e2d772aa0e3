"""Pin the MAGNET restatement (oracle/shouji_oracle.c so_magnet_*) before it
checks the GPU MAGNET kernel.

1. The reference's known answers for MAGNET (proj/tests/test_magnet.cpp):
   longest_zero_run cases, the golden pair's three extractions and decision,
   zero budget, and the fence / consistency / identity properties.
2. When oracle/_ref is built: seeded random comparisons of every extraction
   (diagonal, start, len, lo, hi), the recovered bits and the batch decisions
   against the unmodified reference library.
"""
import numpy as np
import pytest

from oracle.oracle import OracleError

GOLDEN_TEXT = "GGTGCAGAGCTC"      # test_magnet.cpp:15
GOLDEN_PATTERN = "GGTGAGAGTTGT"   # test_magnet.cpp:16


def rand_dna(rng, m, with_n=False):
    alphabet = "ACGTN" if with_n else "ACGT"
    return "".join(alphabet[i] for i in rng.integers(0, len(alphabet), size=m))


@pytest.mark.parametrize("bits,lo,hi,want", [
    ("11111", 0, 4, (0, 0)),          # no zero: len 0, start = lo
    ("1001101", 0, 6, (1, 2)),
    ("0011001100", 0, 9, (0, 2)),     # earliest of equal runs
    ("0011001100", 2, 9, (4, 2)),     # range hides the early run
    ("0000", 3, 1, (3, 0)),           # inverted range
    ("1100", 2, 400, (2, 2)),         # hi past the end is clipped
])
def test_longest_zero_run_known_answers(oracle, bits, lo, hi, want):
    # test_magnet.cpp:25-54
    assert oracle.longest_zero_run(bits, lo, hi) == want


def test_golden_pair_extractions(oracle):
    # test_magnet.cpp:56-77: budget 4, three extractions, in this order
    ext, bits = oracle.recover(GOLDEN_PATTERN, GOLDEN_TEXT, 3, 4)
    assert [x[:3] for x in ext] == [(0, 0, 4), (-1, 5, 4), (-1, 10, 1)]
    for d, start, ln, lo, hi in ext:
        assert lo <= start and start + ln - 1 <= hi
    assert bits == "000010000101" and bits.count("0") == 9


def test_golden_pair_decision_and_zero_budget(oracle):
    # test_magnet.cpp:79-91
    acc, est, bits = oracle.magnet_one(GOLDEN_PATTERN, GOLDEN_TEXT, 3)
    assert acc and est == 3 and bits.count("0") == 9
    ext, bits = oracle.recover(GOLDEN_PATTERN, GOLDEN_TEXT, 3, 0)
    assert ext == [] and bits.count("0") == 0


def test_extracted_runs_are_fenced(oracle):
    # test_magnet.cpp:93-121 (own seeds): runs never touch, bits count what was recovered
    rng = np.random.default_rng(43)
    for _ in range(300):
        m = int(2 + rng.integers(0, 90))
        e = int(rng.integers(0, min(m, 8)))
        t, p = rand_dna(rng, m, True), rand_dna(rng, m, True)
        ext, bits = oracle.recover(p, t, e, e + 1)
        assert len(ext) <= e + 1
        runs = sorted(ext, key=lambda x: x[1])
        for k, (d, start, ln, lo, hi) in enumerate(runs):
            assert lo <= start and start + ln - 1 <= hi and abs(d) <= e
            if k:
                assert runs[k - 1][1] + runs[k - 1][2] < start
        assert bits.count("0") == sum(x[2] for x in ext)


def test_decision_properties(oracle):
    # test_magnet.cpp:123-170
    rng = np.random.default_rng(47)
    for _ in range(200):
        m = int(1 + rng.integers(0, 80))
        e = int(rng.integers(0, m + 2))
        acc, est, bits = oracle.magnet_one(rand_dna(rng, m), rand_dna(rng, m), e)
        assert acc == (est <= e) and est == bits.count("1")
    for _ in range(200):  # threshold zero: only identical pairs pass
        m = int(1 + rng.integers(0, 40))
        a = rand_dna(rng, m)
        b = list(a)
        if rng.integers(0, 2):
            b[int(rng.integers(0, m))] = "ACGT"[int(rng.integers(0, 4))]
        b = "".join(b)
        assert oracle.magnet_one(b, a, 0)[0] == (a == b)
    for _ in range(50):  # identical pairs pass at any threshold
        s = rand_dna(rng, int(1 + rng.integers(0, 100)))
        acc, est, _ = oracle.magnet_one(s, s, int(rng.integers(0, 8)))
        assert acc and est == 0
    acc, est, bits = oracle.magnet_one("ACGT", "TGCA", 7)  # oversized threshold
    assert acc and est == 0 and bits == "0000"
    with pytest.raises(OracleError):
        oracle.magnet_one("ACGT", "ACG", 1)


def test_magnet_vs_reference_extractions(oracle, reference):
    rng = np.random.default_rng(2024)
    for _ in range(400):
        m = int(1 + rng.integers(0, 160))
        e = int(rng.integers(0, min(m, 30)))
        t = rand_dna(rng, m, True)
        if rng.integers(0, 2):  # related pair: a few edits
            p = list(t)
            for _ in range(int(rng.integers(0, 6))):
                i = int(rng.integers(0, m))
                p[i] = "ACGT"[int(rng.integers(0, 4))]
            p = "".join(p)
            sh = int(rng.integers(-2, 3))
            p = (p[sh:] + p[:sh]) if sh else p
        else:
            p = rand_dna(rng, m, True)
        budget = int(rng.integers(0, e + 3))
        (racc, rest, rbits), (rext, rrec) = reference.magnet_one(p, t, e, budget=budget)
        assert oracle.magnet_one(p, t, e) == (racc, rest, rbits), (p, t, e)
        ext, bits = oracle.recover(p, t, e, budget)
        assert [tuple(int(v) for v in x) for x in ext] == rext, (p, t, e, budget)
        assert bits == rrec


@pytest.mark.parametrize("m,lo,hi,e", [(100, 0, 10, 5), (150, 0, 15, 7), (250, 0, 25, 15)])
def test_magnet_batch_vs_reference(oracle, reference, m, lo, hi, e):
    t, p = reference.generate_pairs(1809 + m, 20_000, m, lo, hi)
    a1, e1, _ = oracle.magnet_batch(t, p, e)
    a2, e2 = reference.magnet_batch(t, p, e)
    assert (a1 == a2).all() and (e1 == e2).all()


def load_magnet_fixture():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "magnet.npz")
    return np.load(path)


def test_oracle_matches_magnet_fixture(oracle):
    """tests/golden/magnet.npz was produced by the reference library (make_golden_magnet.py)."""
    z = load_magnet_fixture()
    cases = sorted({k.split("_")[0] for k in z.files if k.startswith("c")})
    assert len(cases) > 250
    for c in cases:
        m, e = (int(v) for v in z[f"{c}_meta"])
        acc, est, bits = oracle.magnet_batch(z[f"{c}_text"], z[f"{c}_pattern"], e, bits=True)
        assert (acc == z[f"{c}_accept"]).all(), (c, m, e)
        assert (est == z[f"{c}_est"]).all(), (c, m, e)
        assert (bits == z[f"{c}_bits"]).all(), (c, m, e)
    for name in ("set_m100_e5", "set_m150_e7", "set_m250_e15"):
        e = int(name.split("_e")[1])
        acc, est, _ = oracle.magnet_batch(z[f"{name}_text"], z[f"{name}_pattern"], e)
        assert (acc == z[f"{name}_accept"]).all() and (est == z[f"{name}_est"]).all(), name
