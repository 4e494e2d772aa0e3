"""Full BASELINE sizes (BASELINE.json configs 1, 3, 4 — up to 100M pairs on one
GPU) checked through size-independent properties, plus a bit-exact oracle
sample. The oracle itself only runs on samples (it finishes in seconds there);
the properties are the reference's own invariants:

* accept == (estimate <= E) for every pair (filter_decision.hpp:12-16);
* at E = 0 the estimate is the Hamming distance with N never matching
  (proj/tests/test_shouji.cpp:106-123). (The reference's other claim, that for
  any E the estimate never exceeds the Hamming distance, test_shouji.cpp:163-184,
  does not hold in general: the reference library itself exceeds it on ~1 pair
  in 10^5 here; tests/test_oracle.py pins one such pair. So it is not used.)
* the answer for a pair does not depend on the batch it arrives in (any split
  of the batch gives the same bitmap and estimates);
* the host entry point (host-pack upload path) equals the device entry point.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_CHAR = ord("N")


def device_batch(gpu, kind, seed, e, n, m):
    import torch
    pitch = gpu.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    gpu.generate_device(kind, seed, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    return tt, pt, pitch


def run_device(gpu, tt, pt, pitch, n, m, e, lo=0):
    import torch
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    gpu.shouji_filter_device(tt[lo:].data_ptr(), pt[lo:].data_ptr(), pitch, n, m, e,
                             acc.data_ptr(), d_estimates=est.data_ptr())
    torch.cuda.synchronize()
    return acc, est


def hamming(tt, pt, m, chunk=4_000_000):
    import torch
    out = []
    for lo in range(0, tt.shape[0], chunk):
        t = tt[lo:lo + chunk, :m]
        p = pt[lo:lo + chunk, :m]
        mis = (t != p) | (t == N_CHAR) | (p == N_CHAR)
        out.append(mis.sum(dim=1, dtype=torch.int32))
    return torch.cat(out)


def accept_bits(acc, n):
    import torch
    words = acc.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    shifts = torch.arange(32, device=acc.device, dtype=torch.int64)
    return ((words[:, None] >> shifts[None, :]) & 1).reshape(-1)[:n].to(torch.int32)


def check_properties(gpu, tt, pt, acc, est, n, m, e):
    bits = accept_bits(acc, n)
    assert bool(((est <= e).to(torch_int()) == bits).all()), "accept != (estimate <= E)"
    assert bool((est <= m).all())
    if e == 0:
        h = hamming(tt, pt, m)
        assert bool((est == h).all()), "E=0 estimate differs from the Hamming distance"


def torch_int():
    import torch
    return torch.int32


def sample_vs_oracle(oracle, tt, pt, acc, est, n, m, e, k=40_000, seed=0):
    rng = np.random.default_rng(seed)
    lo = int(rng.integers(0, max(1, n - k))) // 32 * 32
    t = tt[lo:lo + k, :m].cpu().numpy()
    p = pt[lo:lo + k, :m].cpu().numpy()
    a_ref, e_ref, _ = oracle.shouji_batch(t, p, e)
    assert (acc[lo // 32:(lo + k) // 32].cpu().numpy().view(np.uint32) == a_ref[: k // 32]).all()
    assert (est[lo:lo + k].cpu().numpy().view(np.uint32) == e_ref).all()


@pytest.mark.parametrize("e", [0, 5, 10])
def test_config1_full_30M(gpu, oracle, e):
    n, m = 30_000_000, 100
    tt, pt, pitch = device_batch(gpu, 1, 7000 + e, e, n, m)
    acc, est = run_device(gpu, tt, pt, pitch, n, m, e)
    check_properties(gpu, tt, pt, acc, est, n, m, e)
    sample_vs_oracle(oracle, tt, pt, acc, est, n, m, e, seed=e)
    if e == 5:
        # batch-split invariance at ragged split points
        import torch
        for cut in (12_345_679, 29_999_969):
            lo_n = cut // 32 * 32
            a1, e1 = run_device(gpu, tt, pt, pitch, lo_n, m, e)
            a2, e2 = run_device(gpu, tt, pt, pitch, n - lo_n, m, e, lo=lo_n)
            assert torch.equal(torch.cat([a1, a2]), acc) and torch.equal(torch.cat([e1, e2]), est)


def test_config1_host_path_equals_device_path(gpu):
    """30M pairs through pf_shouji_filter_batch (host-pack upload, 256Ki-pair chunks)
    against the device entry point on the same bytes."""
    import torch
    n, m, e = 30_000_000, 100, 5
    tt, pt, pitch = device_batch(gpu, 1, 7100, e, n, m)
    acc, est = run_device(gpu, tt, pt, pitch, n, m, e)
    ht = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
    hp = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
    ht.copy_(tt[:, :m])
    hp.copy_(pt[:, :m])
    a_h, e_h, _ = gpu.shouji_filter_batch(ht.numpy(), hp.numpy(), e, estimates=True)
    assert (a_h == acc.cpu().numpy().view(np.uint32)).all()
    assert (e_h == est.cpu().numpy().view(np.uint32)).all()


@pytest.mark.parametrize("e", [0, 25])
def test_config3_full_30M(gpu, oracle, e):
    n, m = 30_000_000, 250
    tt, pt, pitch = device_batch(gpu, 3, 7300 + e, e, n, m)
    acc, est = run_device(gpu, tt, pt, pitch, n, m, e)
    check_properties(gpu, tt, pt, acc, est, n, m, e)
    sample_vs_oracle(oracle, tt, pt, acc, est, n, m, e, k=20_000, seed=3 + e)


def test_config4_full_100M(gpu, oracle):
    """100M pairs of m=250 (25 GB per sequence array) in one device call: exercises
    64-bit indexing in every kernel (offsets beyond 2^31 bytes)."""
    n, m, e = 100_000_000, 250, 25
    tt, pt, pitch = device_batch(gpu, 4, 7400, e, n, m)
    acc, est = run_device(gpu, tt, pt, pitch, n, m, e)
    check_properties(gpu, tt, pt, acc, est, n, m, e)
    sample_vs_oracle(oracle, tt, pt, acc, est, n, m, e, k=10_000, seed=4)
    # the tail of the batch (offsets far beyond 2^32 bytes) against the oracle too
    k = 8192
    lo = n - k
    t = tt[lo:, :m].cpu().numpy()
    p = pt[lo:, :m].cpu().numpy()
    a_ref, e_ref, _ = oracle.shouji_batch(t, p, e)
    assert (acc[lo // 32:].cpu().numpy().view(np.uint32) == a_ref).all()
    assert (est[lo:].cpu().numpy().view(np.uint32) == e_ref).all()
