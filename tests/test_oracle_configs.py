"""The full-size checker (oracle/config_oracle.c) pinned on CPU:

* its vectorisable shouji_filter restatement equals the plain restatement
  (oracle/shouji_oracle.c) and the unmodified reference library (oracle/_ref)
  on every BASELINE config's own data, across thresholds and widths 3..8;
* its generator mirror is self-consistent (any pair index on its own equals
  the same pair inside a range) and still produces the bytes the committed
  digests were computed from (tests/golden/fullsize_digests.json);
* the digest script's bitmap layout is the C ABI's (LSB-first u32 words).

The GPU side (tests/test_gpu_fullsize_digests.py) checks the device generator
against this mirror and the CUDA filter against the digests.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

import make_fullsize_digests as mfd  # noqa: E402

CASES = [(1, 100, e) for e in (0, 1, 5, 10)] + [(2, 150, e) for e in (0, 3, 7, 15)] + \
        [(3, 250, e) for e in (0, 1, 12, 25)] + [(4, 250, 25)]


@pytest.mark.parametrize("config,m,e", CASES)
def test_fast_restatement_equals_plain_oracle_and_reference(oracle, reference, config, m, e):
    seed = mfd.seed_of(config, e)
    n = 2000
    t, p = oracle.gen_config(config, seed, e, m, 0, n)
    a_slow, e_slow, _ = oracle.shouji_batch(t, p, e)
    a_ref, e_ref, _ = reference.shouji_batch(t, p, e)
    e_fast = oracle.shouji_fast_batch(t, p, e)
    e_gen = oracle.config_estimates(config, seed, e, m, e, 0, n)
    assert (e_slow == e_ref).all() and (a_slow == a_ref).all()
    assert (e_fast == e_ref).all()
    assert (e_gen == e_ref).all()
    assert (mfd.bitmap_words(e_gen, e) == a_ref).all()


@pytest.mark.parametrize("w", [3, 5, 6, 7, 8])
def test_fast_restatement_other_widths(oracle, reference, w):
    t, p = oracle.gen_config(3, 99, 9, 250, 0, 600)
    _, e_ref, _ = reference.shouji_batch(t, p, 9, width=w)
    assert (oracle.shouji_fast_batch(t, p, 9, width=w) == e_ref).all()


def test_fast_restatement_edge_shapes(oracle, reference):
    rng = np.random.default_rng(5)
    for m in (1, 2, 3, 4, 5, 7, 31, 63, 64, 65, 129):
        n = 300
        alpha = np.frombuffer(b"ACGTN", np.uint8)
        t = alpha[rng.choice(5, size=(n, m), p=[.24, .24, .24, .24, .04])]
        p = t.copy()
        flip = rng.random((n, m)) < 0.1
        p[flip] = alpha[rng.integers(0, 5, size=flip.sum())]
        for e in sorted({0, 1, m // 2, max(0, m - 1), m, m + 3}):
            _, e_ref, _ = reference.shouji_batch(t, p, e)
            assert (oracle.shouji_fast_batch(t, p, e) == e_ref).all(), (m, e)


def test_generator_rows_equal_ranges(oracle):
    for config, m, e in [(1, 100, 5), (2, 150, 7), (3, 250, 25), (4, 250, 25)]:
        t, p = oracle.gen_config(config, 17, e, m, 1000, 200)
        rows = np.array([1000, 1001, 1137, 1199])
        rt, rp = oracle.gen_config_rows(config, 17, e, m, rows)
        assert (rt == t[rows - 1000]).all() and (rp == p[rows - 1000]).all()
        assert set(np.unique(t)) <= set(b"ACGTN") and set(np.unique(p)) <= set(b"ACGTN")


def test_generator_config_properties(oracle):
    # config 3 at E=0 plants no edit; config 4 has N at ~0.1% of positions in both
    t, p = oracle.gen_config(3, 5, 0, 250, 0, 1000)
    assert (t == p).all()
    t, p = oracle.gen_config(4, 5, 25, 250, 0, 20000)
    for x in (t, p):
        rate = (x == ord("N")).mean()
        assert 0.0007 < rate < 0.0013, rate
    # config 1: half the pairs planted with k ~ U{0..2E}: 1/(2E+1) of those unedited
    t, p = oracle.gen_config(1, 5, 5, 100, 0, 20000)
    same = (t == p).all(axis=1).mean()
    assert 0.5 / 11 * 0.8 < same < 0.5 / 11 * 1.2, same


def test_digest_file_pins_the_generator_prefix(oracle):
    """Every committed set still matches the mirror's bytes (data_prefix_sha256)."""
    doc = json.load(open(mfd.OUT))
    assert len(doc["sets"]) == len(mfd.all_sets())
    for s in doc["sets"]:
        assert s["seed"] == mfd.seed_of(s["config"], s["E"])
        t, p = oracle.gen_config(s["config"], s["seed"], s["E"], s["m"], 0, mfd.PREFIX_PAIRS)
        h = hashlib.sha256(t.tobytes() + p.tobytes()).hexdigest()
        assert h == s["data_prefix_sha256"], (s["config"], s["E"])


@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_reference_library_reproduces_the_estimate_prefixes(oracle, reference, config):
    """The unmodified reference library recomputes the first 65536 pairs of every
    committed set of this config and hashes to the recorded estimate_prefix_sha256."""
    doc = json.load(open(mfd.OUT))
    sets = [s for s in doc["sets"] if s["config"] == config]
    if config == 3:  # the 26-threshold sweep: every fifth E on CPU (all of them on the GPU)
        sets = [s for s in sets if s["E"] % 5 == 0 or s["E"] == 25]
    for s in sets:
        t, p = oracle.gen_config(config, s["seed"], s["E"], s["m"], 0, mfd.ESTIMATE_PREFIX_PAIRS)
        _, est, _ = reference.shouji_batch(t, p, s["E"])
        h = hashlib.sha256(est.astype("<u4").tobytes()).hexdigest()
        assert h == s["estimate_prefix_sha256"], (config, s["E"])


def test_bitmap_layout_matches_the_c_abi(oracle):
    for n in (1, 31, 32, 33, 1000):
        t, p = oracle.gen_config(1, 3, 5, 100, 0, n)
        a, est, _ = oracle.shouji_batch(t, p, 5)
        assert (mfd.bitmap_words(est, 5) == a).all()
