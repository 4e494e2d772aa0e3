"""GPU parity of the packed-planes variant (pf_shouji_filter_packed_batch /
_device, csrc/pack_planes.cu): pairs in packed_sequence's own storage, re-sliced
on the device, filtered, compared with the oracle on the ASCII form of the same
pairs. Bit-exact accept, estimates and tally bits."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ACGT = np.frombuffer(b"ACGT", np.uint8)
ACGTN = np.frombuffer(b"ACGTN", np.uint8)


def pairs(rng, n, m, rate=0.06, alphabet=ACGTN):
    t = alphabet[rng.integers(0, len(alphabet), size=(n, m))]
    p = t.copy()
    mask = rng.random(p.shape) < rate
    p[mask] = ACGT[rng.integers(0, 4, size=int(mask.sum()))]
    for i in range(0, n, 5):
        p[i] = np.roll(p[i], int(rng.integers(-3, 4)))
    return np.ascontiguousarray(t), np.ascontiguousarray(p)


def check(gpu, oracle, t, p, e, width=4, bits=True):
    m = t.shape[1]
    a1, e1, b1 = gpu.shouji_filter_packed_batch(gpu.pack_planes(t), gpu.pack_planes(p), m, e,
                                                width, estimates=True, bits=bits)
    a2, e2, b2 = oracle.shouji_batch(t, p, e, width, bits=bits)
    assert (a1 == a2).all() and (e1 == e2).all(), (m, e, width)
    if bits:
        assert (b1 == b2).all(), (m, e, width)


@pytest.mark.parametrize("m", [1, 2, 5, 31, 32, 33, 63, 64, 65, 100, 128, 150, 250, 255, 256,
                               300])
def test_lengths(gpu, oracle, m):
    rng = np.random.default_rng(m)
    t, p = pairs(rng, 1500 + m, m)
    for e in sorted({0, min(m - 1, 3), min(m - 1, 5), min(m - 1, 17), m - 1, m}):
        check(gpu, oracle, t, p, e)


@pytest.mark.parametrize("width", [3, 5, 8])
def test_widths(gpu, oracle, width):
    rng = np.random.default_rng(width)
    t, p = pairs(rng, 3000, 100)
    for e in (2, 5, 40):
        check(gpu, oracle, t, p, e, width, bits=False)


def test_golden_fixture_configs(gpu, oracle):
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "config0.npz"))
    t, p = z["text_head"], z["pattern_head"]
    a, est, _ = gpu.shouji_filter_packed_batch(gpu.pack_planes(t), gpu.pack_planes(p), 100, 5,
                                               estimates=True)
    assert (a == z["accept_head"]).all() and (est == z["est_head"]).all()


def test_multi_chunk_pinned_and_pageable(gpu, oracle):
    import torch
    rng = np.random.default_rng(3)
    n, m = 2_300_001, 100
    t, p = pairs(rng, n, m, alphabet=ACGT)
    tp, pp = gpu.pack_planes(t), gpu.pack_planes(p)
    a_ref, e_ref, _ = oracle.shouji_batch(t, p, 5)
    a, e, _ = gpu.shouji_filter_packed_batch(tp, pp, m, 5, estimates=True)
    assert (a == a_ref).all() and (e == e_ref).all()
    tpin = torch.from_numpy(tp.reshape(n, -1)).pin_memory()
    ppin = torch.from_numpy(pp.reshape(n, -1)).pin_memory()
    h0, _ = gpu.transfer_bytes()
    a, e, _ = gpu.shouji_filter_packed_batch(tpin.numpy().reshape(tp.shape),
                                             ppin.numpy().reshape(pp.shape), m, 5, estimates=True)
    h1, _ = gpu.transfer_bytes()
    assert (a == a_ref).all() and (e == e_ref).all()
    assert h1 - h0 == 2 * n * gpu.packed_words(m) * 8


def test_errors_and_short_circuit(gpu):
    t = gpu.pack_planes(np.frombuffer(b"ACGTACGT", np.uint8)[None, :])
    with pytest.raises(gpu.invalid_parameters_error):  # width before e >= m (shouji.cpp:47-49)
        gpu.shouji_filter_packed_batch(t, t, 8, 9, width=2)
    a, est, bits = gpu.shouji_filter_packed_batch(t, t, 8, 8, estimates=True, bits=True)
    assert int(a[0]) == 1 and est[0] == 0 and int(bits[0, 0]) == 0
    with pytest.raises(gpu.length_mismatch_error):
        gpu.shouji_filter_packed_batch(t, t, 200, 3)


def test_device_entry_point(gpu, oracle):
    import torch
    rng = np.random.default_rng(4)
    n, m = 20_000, 150
    t, p = pairs(rng, n, m)
    dt = torch.from_numpy(gpu.pack_planes(t)).cuda()
    dp = torch.from_numpy(gpu.pack_planes(p)).cuda()
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    bits = torch.zeros((n, (m + 63) // 64), dtype=torch.int64, device="cuda")
    gpu.shouji_filter_packed_device(dt.data_ptr(), dp.data_ptr(), n, m, 7, acc.data_ptr(),
                                    d_estimates=est.data_ptr(), d_bits=bits.data_ptr())
    torch.cuda.synchronize()
    a2, e2, b2 = oracle.shouji_batch(t, p, 7, bits=True)
    assert (acc.cpu().numpy().view(np.uint32) == a2).all()
    assert (est.cpu().numpy().view(np.uint32) == e2).all()
    assert (bits.cpu().numpy().view(np.uint64) == b2).all()


def test_mixed_n_presence(gpu, oracle):
    """N-presence flags of the re-slice: most groups N-free (N planes neither stored nor read),
    a few holding an N in the text or the pattern (warps mixing both kinds), and blocks with
    no N at all (their N region is skipped)."""
    rng = np.random.default_rng(77)
    n, m = 40_000, 100
    t, p = pairs(rng, n, m, alphabet=ACGT)
    for i in rng.choice(n, size=300, replace=False):
        (t if rng.random() < 0.5 else p)[i, int(rng.integers(0, m))] = ord("N")
    for e in (0, 2, 5, 10, 13):
        check(gpu, oracle, t, p, e, bits=False)
    check(gpu, oracle, t[:5000], p[:5000], 5, bits=True)
