"""The latency path (csrc/small.cu): batches of at most 64 pairs — a per-pair
caller of shouji_filter (proj/src/shouji.cpp:41-58) or the drop-in's coalesced
handful — run one CTA per pair from mapped pinned staging. Bit-exact accept,
estimate and tally bits against the oracle and against the throughput kernels
(PF_SMALL=0), the reference's error order (illegal byte before width), and the
packed-planes input."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHA = np.frombuffer(b"ACGT", np.uint8)


def pairs(rng, n, m, stride=None, n_rate=0.02, edit_rate=0.1):
    stride = stride or m
    t = np.full((n, stride), ord("x"), np.uint8)
    p = np.full((n, stride), ord("y"), np.uint8)
    t[:, :m] = ALPHA[rng.integers(0, 4, size=(n, m))]
    p[:, :m] = t[:, :m]
    mask = rng.random((n, m)) < edit_rate
    p[:, :m][mask] = ALPHA[rng.integers(0, 4, size=int(mask.sum()))]
    for x in (t, p):
        nm = rng.random((n, m)) < n_rate
        x[:, :m][nm] = ord("N")
    # a shifted copy for some pairs: indel-like structure
    k = n // 3
    if m > 3 and k:
        p[:k, 1:m] = t[:k, : m - 1]
    return t, p


@pytest.fixture
def small_off():
    os.environ["PF_SMALL"] = "0"
    yield
    os.environ.pop("PF_SMALL", None)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 7, 31, 63, 64, 65, 100, 150, 250, 1000, 2048])
def test_small_batches_match_oracle(gpu, oracle, m):
    rng = np.random.default_rng(m)
    for n in (1, 2, 31, 32, 33, 64):
        t, p = pairs(rng, n, m, stride=m + int(rng.integers(0, 5)))
        for e in sorted({0, 1, 3, m // 3, max(0, m - 1), m, m + 4}):
            for w in ((3, 4, 5, 8) if m <= 250 else (4,)):
                a1, e1, b1 = gpu.shouji_filter_batch(t, p, e, width=w, m=m, estimates=True,
                                                     bits=True)
                a2, e2, b2 = oracle.shouji_batch(t[:, :m], p[:, :m], e, width=w, bits=True)
                assert (a1 == a2).all() and (e1 == e2).all() and (b1 == b2).all(), (n, m, e, w)


def test_small_path_equals_throughput_path(gpu, oracle, small_off):
    rng = np.random.default_rng(9)
    for m, e in [(100, 5), (150, 7), (250, 25), (37, 2)]:
        t, p = pairs(rng, 64, m)
        os.environ["PF_SMALL"] = "0"
        big = gpu.shouji_filter_batch(t, p, e, estimates=True, bits=True)
        os.environ["PF_SMALL"] = "1"
        small = gpu.shouji_filter_batch(t, p, e, estimates=True, bits=True)
        for x, y in zip(big, small):
            assert (x == y).all(), (m, e)


def test_small_packed_planes(gpu, oracle):
    rng = np.random.default_rng(11)
    for m in (1, 64, 65, 100, 250, 1000):
        t, p = pairs(rng, 40, m)
        tp, pp = gpu.pack_planes(t), gpu.pack_planes(p)
        for e in (0, 2, 5, m):
            a1, e1, b1 = gpu.shouji_filter_packed_batch(tp, pp, m, e, estimates=True, bits=True)
            a2, e2, b2 = oracle.shouji_batch(t, p, e, bits=True)
            assert (a1 == a2).all() and (e1 == e2).all() and (b1 == b2).all(), (m, e)


def test_small_errors_in_reference_order(gpu, oracle):
    rng = np.random.default_rng(12)
    t, p = pairs(rng, 20, 50, n_rate=0.0)
    t[7, 30] = ord("a")   # lower case is illegal (packed_sequence.cpp:19-29)
    p[7, 3] = ord("X")    # same pair, pattern: text is checked first
    p[5, 44] = ord("-")   # an earlier pair wins
    for w in (4, 9):      # the illegal byte is reported before the width
        with pytest.raises(gpu.illegal_character_error) as ex:
            gpu.shouji_filter_batch(t, p, 3, width=w)
        assert (ex.value.pair, ex.value.field, ex.value.position()) == (5, 1, 44)
    p[5, 44] = ord("A")
    with pytest.raises(gpu.illegal_character_error) as ex:
        gpu.shouji_filter_batch(t, p, 3)
    assert (ex.value.pair, ex.value.field, ex.value.position(), ex.value.byte()) == (7, 0, 30, "a")
    t[7, 30] = ord("A")
    p[7, 3] = ord("A")
    with pytest.raises(gpu.invalid_parameters_error):
        gpu.shouji_filter_batch(t, p, 3, width=9)
    with pytest.raises(gpu.invalid_parameters_error):  # width checked even when e >= m
        gpu.shouji_filter_batch(t, p, 60, width=2)


def test_per_pair_entry_point_latency_path(gpu, oracle):
    # pf_shouji_filter_one: the shouji_filter signature, a batch of one
    rng = np.random.default_rng(13)
    for m, e in [(12, 3), (100, 5), (250, 25)]:
        t, p = pairs(rng, 10, m)
        for i in range(10):
            d = gpu.shouji_filter(gpu.seq(p[i].tobytes().decode()), gpu.seq(t[i].tobytes().decode()), e)
            acc, est, bits = oracle.shouji_one(p[i].tobytes().decode(), t[i].tobytes().decode(), e)
            assert (d.accept, d.edit_estimate, d.bits.to_string()) == (acc, est, bits)
