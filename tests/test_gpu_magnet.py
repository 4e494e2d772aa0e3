"""GPU parity of MAGNET (csrc/magnet.cu) through the C ABI,
against the oracle restatement (pinned by tests/test_oracle_magnet.py) and the
committed reference fixture tests/golden/magnet.npz.

Bar: bit-exact accept bitmap, estimates and tally bits."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDEN_TEXT = "GGTGCAGAGCTC"
GOLDEN_PATTERN = "GGTGAGAGTTGT"
ACGT = np.frombuffer(b"ACGT", np.uint8)
ACGTN = np.frombuffer(b"ACGTN", np.uint8)


def check(gpu, oracle, t, p, e, bits=True):
    a1, e1, b1 = gpu.magnet_filter_batch(t, p, e, estimates=True, bits=bits)
    a2, e2, b2 = oracle.magnet_batch(t, p, e, bits=bits)
    bad = np.nonzero(e1 != e2)[0]
    assert bad.size == 0, f"estimate differs at {bad[:8]}: gpu {e1[bad[:4]]} oracle {e2[bad[:4]]}"
    assert (a1 == a2).all()
    if bits:
        assert (b1 == b2).all()
    return a1, e1


def related(rng, n, m, rate=0.05, shifts=3, alphabet=ACGTN):
    t = alphabet[rng.integers(0, len(alphabet), size=(n, m))]
    p = t.copy()
    mask = rng.random(p.shape) < rate
    p[mask] = ACGT[rng.integers(0, 4, size=int(mask.sum()))]
    for i in range(n):
        for _ in range(int(rng.integers(0, shifts + 1))):
            pos = int(rng.integers(0, m))
            if rng.random() < 0.5:
                p[i, pos:] = np.concatenate([ACGT[rng.integers(0, 4, size=1)], p[i, pos:-1]])
            else:
                p[i, pos:] = np.concatenate([p[i, pos + 1:], ACGT[rng.integers(0, 4, size=1)]])
    return np.ascontiguousarray(t), np.ascontiguousarray(p)


def test_golden_pair(gpu):
    # test_magnet.cpp:79-84
    d = gpu.magnet_filter(gpu.seq(GOLDEN_PATTERN), gpu.seq(GOLDEN_TEXT), 3)
    assert d.accept and d.edit_estimate == 3 and d.bits.count_zeros() == 9
    assert d.bits.to_string() == "000010000101"


def test_per_pair_semantics(gpu):
    d = gpu.magnet_filter(gpu.seq("ACGT"), gpu.seq("TGCA"), 7)  # oversized threshold
    assert d.accept and d.edit_estimate == 0 and d.bits.count_ones() == 0
    with pytest.raises(gpu.length_mismatch_error):
        gpu.magnet_filter(gpu.seq("ACGT"), gpu.seq("ACG"), 1)
    assert gpu.run_filter("magnet", gpu.seq(GOLDEN_PATTERN), gpu.seq(GOLDEN_TEXT), 3).edit_estimate == 3
    rng = np.random.default_rng(59)
    for _ in range(20):  # identical pairs pass at any threshold
        s = "".join(rng.choice(list("ACGT"), int(1 + rng.integers(0, 100))))
        d = gpu.magnet_filter(gpu.seq(s), gpu.seq(s), int(rng.integers(0, 8)))
        assert d.accept and d.edit_estimate == 0


def test_reference_fixture(gpu):
    """Every case of tests/golden/magnet.npz (produced by the reference library)."""
    z = np.load(os.path.join(GOLD, "magnet.npz"))
    cases = sorted({k.split("_")[0] for k in z.files if k.startswith("c")})
    for c in cases:
        m, e = (int(v) for v in z[f"{c}_meta"])
        a, est, bits = gpu.magnet_filter_batch(z[f"{c}_text"], z[f"{c}_pattern"], e,
                                               estimates=True, bits=True)
        assert (a == z[f"{c}_accept"]).all(), (c, m, e)
        assert (est == z[f"{c}_est"]).all(), (c, m, e)
        assert (bits == z[f"{c}_bits"]).all(), (c, m, e)
    for name in ("set_m100_e5", "set_m150_e7", "set_m250_e15"):
        e = int(name.split("_e")[1])
        a, est, _ = gpu.magnet_filter_batch(z[f"{name}_text"], z[f"{name}_pattern"], e,
                                            estimates=True)
        assert (a == z[f"{name}_accept"]).all() and (est == z[f"{name}_est"]).all(), name


@pytest.mark.parametrize("m", [1, 2, 3, 7, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 150, 200,
                               250, 255, 256, 257, 300, 400, 512])
def test_lengths(gpu, oracle, m):
    rng = np.random.default_rng(1000 + m)
    n = 1500 if m <= 256 else 400
    t, p = related(rng, n, m)
    half = n // 2
    p[half:] = ACGTN[rng.integers(0, 5, size=(n - half, m))]  # unrelated half
    for e in sorted({0, 1, min(m - 1, 4), min(m - 1, 10), min(m - 1, 13), min(m - 1, 25),
                     min(m - 1, 31), m - 1, m, m + 3}):
        check(gpu, oracle, t, p, e)


def test_generated_configs(gpu, oracle):
    for m, lo, hi, e, seed in [(100, 0, 10, 5, 71), (150, 0, 15, 7, 72), (250, 0, 25, 25, 73),
                               (100, 0, 4, 2, 74)]:
        t, p = oracle.generate_pairs(seed, 20_000, m, lo, hi)
        check(gpu, oracle, t, p, e, bits=False)


def test_low_complexity(gpu, oracle):
    rng = np.random.default_rng(5)
    n, m = 3000, 150
    t = np.zeros((n, m), np.uint8)
    for i in range(n):
        unit = ACGT[rng.integers(0, 4, size=int(rng.integers(1, 5)))]
        t[i] = np.resize(unit, m)
    p = t.copy()
    for i in range(n):
        s = int(rng.integers(-3, 4))
        p[i] = np.roll(p[i], s)
    p[rng.random(p.shape) < 0.01] = ord("N")
    for e in (0, 3, 8, 20):
        check(gpu, oracle, t, p, e)


def test_ragged_and_strided(gpu, oracle):
    rng = np.random.default_rng(8)
    for n in (1, 31, 33, 4097):
        m, stride = 100, 113
        buf_t = np.full((n, stride), ord("x"), np.uint8)
        buf_p = np.full((n, stride), ord("y"), np.uint8)
        t, p = related(rng, n, m)
        buf_t[:, :m], buf_p[:, :m] = t, p
        a1, e1, b1 = gpu.magnet_filter_batch(buf_t, buf_p, 5, m=m, estimates=True, bits=True)
        a2, e2, b2 = oracle.magnet_batch(t, p, 5, bits=True)
        assert (a1 == a2).all() and (e1 == e2).all() and (b1 == b2).all()
        if n % 32:
            assert int(a1[-1]) >> (n % 32) == 0


def test_device_entry_point(gpu, oracle):
    import torch
    rng = np.random.default_rng(9)
    n, m = 5000, 150
    t, p = related(rng, n, m)
    pitch = gpu.device_pitch(m)
    bt = np.zeros((n, pitch), np.uint8)
    bp = np.zeros((n, pitch), np.uint8)
    bt[:, :m], bp[:, :m] = t, p
    tt, pt = torch.from_numpy(bt).cuda(), torch.from_numpy(bp).cuda()
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    bits = torch.zeros((n, (m + 63) // 64), dtype=torch.int64, device="cuda")
    gpu.magnet_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, 7, acc.data_ptr(),
                             d_estimates=est.data_ptr(), d_bits=bits.data_ptr())
    torch.cuda.synchronize()
    a2, e2, b2 = oracle.magnet_batch(t, p, 7, bits=True)
    assert (acc.cpu().numpy().view(np.uint32) == a2).all()
    assert (est.cpu().numpy().view(np.uint32) == e2).all()
    assert (bits.cpu().numpy().view(np.uint64) == b2).all()


def test_errors(gpu):
    rng = np.random.default_rng(10)
    n, m = 2000, 100
    t = np.ascontiguousarray(ACGT[rng.integers(0, 4, size=(n, m))])
    p = t.copy()
    p[1500, 7] = ord("a")
    t[1500, 9] = ord("-")  # text before pattern within a pair
    with pytest.raises(gpu.illegal_character_error) as ei:
        gpu.magnet_filter_batch(t, p, 5)
    assert (ei.value.pair, ei.value.field, ei.value.position()) == (1500, 0, 9)
    with pytest.raises(gpu.invalid_parameters_error):  # beyond the kernel's m limit
        big = np.full((2, 600), ord("A"), np.uint8)
        gpu.magnet_filter_batch(big, big, 5)
    # e >= m never reaches the kernel: accept all, even at m > 512
    big = np.full((2, 600), ord("A"), np.uint8)
    a, est, _ = gpu.magnet_filter_batch(big, big, 600, estimates=True)
    assert int(a[0]) == 3 and (est == 0).all()


def test_warp_and_thread_forms_agree(gpu, oracle):
    """E in [13, 31] runs the warp-cooperative kernel; both forms against the oracle
    around the switch-over and at the warp form's 2-diagonals-per-lane edge."""
    rng = np.random.default_rng(77)
    for m in (100, 250):
        t, p = related(rng, 1200, m, rate=0.1, shifts=4)
        for e in (12, 13, 15, 16, 31):
            check(gpu, oracle, t, p, e)
