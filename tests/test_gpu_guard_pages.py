"""Device out-of-bounds checks with guard ranges (compute-sanitizer is closed on
this pool; tests/guard.py): every device input and output array of the device
entry points ends (or starts) at the edge of a CUDA virtual-memory mapping with
unmapped address space beyond it, so a kernel access past the array raises
cudaErrorIllegalAddress. Covered: the TMA tile pack and every search form
(width-4 carry/rebuild/prefetch, any-width), tally bits, the packed-planes
re-slice, dibit and nibble records (TMA), MAGNET (thread and warp forms).
Results must equal the oracle's. A run-to-run determinism stress of the
throughput path (shared-memory races would show as varying results) closes it.
"""
import hashlib

import numpy as np
import pytest

from guard import DeviceGuarded

pytestmark = pytest.mark.gpu

ALPHA = np.frombuffer(b"ACGTN", np.uint8)


def make(rng, n, m, n_rate=0.01):
    t = ALPHA[rng.choice(5, size=(n, m), p=[(1 - n_rate) / 4] * 4 + [n_rate])]
    p = t.copy()
    mask = rng.random((n, m)) < 0.08
    p[mask] = ALPHA[rng.integers(0, 4, size=int(mask.sum()))]
    k = n // 3
    if m > 2:
        p[:k, 1:] = t[:k, :-1]
    return t, p


def guarded_records(gpu, t, at_end):
    n, m = t.shape
    pitch = gpu.device_pitch(m)
    rec = np.full((n, pitch), ord("A"), np.uint8)
    rec[:, :m] = t
    g = DeviceGuarded(rec.nbytes, at_end=at_end)
    g.upload(rec)
    return g, pitch


def outputs(n, m, bits, at_end):
    acc = DeviceGuarded(((n + 31) // 32) * 4, at_end=at_end)
    est = DeviceGuarded(n * 4, at_end=at_end)
    bv = DeviceGuarded(n * ((m + 63) // 64) * 8, at_end=at_end) if bits else None
    return acc, est, bv


def fetch(acc, est, bv, n, m):
    import torch
    torch.cuda.synchronize()
    a = acc.download(np.uint32, ((n + 31) // 32,))
    e = est.download(np.uint32, (n,))
    b = bv.download(np.uint64, (n, (m + 63) // 64)) if bv else None
    return a, e, b


CASES = [(100, [0, 5, 10, 13]), (150, [7]), (250, [25]), (1, [0]), (31, [3]), (64, [6]),
         (65, [2]), (1000, [9])]


@pytest.mark.parametrize("at_end", [True, False])
@pytest.mark.parametrize("m,es", CASES)
def test_device_entry_stays_in_bounds(gpu, oracle, m, es, at_end):
    rng = np.random.default_rng(m)
    for n in (1, 33, 256, 4100, 70000 if m <= 150 else 9000):
        t, p = make(rng, n, m)
        gt, pitch = guarded_records(gpu, t, at_end)
        gp, _ = guarded_records(gpu, p, at_end)
        for e in es:
            for w in ((4, 3, 8) if e == es[0] else (4,)):
                acc, est, bv = outputs(n, m, True, at_end)
                gpu.shouji_filter_device(gt.ptr, gp.ptr, pitch, n, m, e, acc.ptr, width=w,
                                         d_estimates=est.ptr, d_bits=bv.ptr)
                a, v, b = fetch(acc, est, bv, n, m)
                a2, v2, b2 = oracle.shouji_batch(t, p, e, width=w, bits=True)
                assert (a == a2).all() and (v == v2).all() and (b == b2).all(), (n, m, e, w)
                for g in (acc, est, bv):
                    g.free()
        gt.free()
        gp.free()


@pytest.mark.parametrize("at_end", [True, False])
def test_packed_planes_dibits_nibbles_magnet_stay_in_bounds(gpu, oracle, at_end):
    rng = np.random.default_rng(2)
    for m, e, n in [(100, 5, 5000), (250, 20, 3000), (63, 4, 257)]:
        t, p = make(rng, n, m)
        a2, v2, _ = oracle.shouji_batch(t, p, e)
        # packed_sequence planes
        tp, pp = gpu.pack_planes(t), gpu.pack_planes(p)
        gtp, gpp = DeviceGuarded(tp.nbytes, at_end=at_end), DeviceGuarded(pp.nbytes, at_end=at_end)
        gtp.upload(tp)
        gpp.upload(pp)
        acc, est, _ = outputs(n, m, False, at_end)
        gpu.shouji_filter_packed_device(gtp.ptr, gpp.ptr, n, m, e, acc.ptr, d_estimates=est.ptr)
        a, v, _ = fetch(acc, est, None, n, m)
        assert (a == a2).all() and (v == v2).all(), ("planes", m)
        # dibit records (+ N planes): the host pack's output format
        dt, dq, nt, nq = gpu.host_pack_dibits(t, p)
        bufs = [DeviceGuarded(x.nbytes, at_end=at_end) for x in (dt, dq, nt, nq)]
        for g, x in zip(bufs, (dt, dq, nt, nq)):
            g.upload(x)
        acc2, est2, _ = outputs(n, m, False, at_end)
        gpu.shouji_filter_dibits_device(bufs[0].ptr, bufs[1].ptr, n, m, e, acc2.ptr,
                                        d_ntext=bufs[2].ptr, d_npattern=bufs[3].ptr,
                                        d_estimates=est2.ptr)
        a, v, _ = fetch(acc2, est2, None, n, m)
        assert (a == a2).all() and (v == v2).all(), ("dibits", m)
        # nibble records (N-free pairs: nibbles carry N in bit 3)
        ot, op = gpu.host_pack_nibbles(t, p)
        gnt, gnp = DeviceGuarded(ot.nbytes, at_end=at_end), DeviceGuarded(op.nbytes, at_end=at_end)
        gnt.upload(ot)
        gnp.upload(op)
        acc3, est3, _ = outputs(n, m, False, at_end)
        gpu.shouji_filter_nibbles_device(gnt.ptr, gnp.ptr, n, m, e, acc3.ptr, d_estimates=est3.ptr)
        a, v, _ = fetch(acc3, est3, None, n, m)
        assert (a == a2).all() and (v == v2).all(), ("nibbles", m)
        # MAGNET on guarded ASCII records
        gt, pitch = guarded_records(gpu, t, at_end)
        gp, _ = guarded_records(gpu, p, at_end)
        acc4, est4, bv4 = outputs(n, m, True, at_end)
        gpu.magnet_filter_device(gt.ptr, gp.ptr, pitch, n, m, e, acc4.ptr, d_estimates=est4.ptr,
                                 d_bits=bv4.ptr)
        a, v, b = fetch(acc4, est4, bv4, n, m)
        ma, mv, mb = oracle.magnet_batch(t, p, e, bits=True)
        assert (a == ma).all() and (v == mv).all() and (b == mb).all(), ("magnet", m)
        for g in [gtp, gpp, acc, est, acc2, est2, gnt, gnp, acc3, est3, gt, gp, acc4, est4, bv4] + bufs:
            g.free()


def test_throughput_path_is_deterministic(gpu):
    """30 repeats of the same 4M-pair batch (E=5 and E=10) with estimates: identical
    bitmaps and estimates every time (a shared-memory or cross-CTA race in the
    pack/search pair would show up as run-to-run differences)."""
    import torch
    n, m = 4_000_000, 100
    pitch = gpu.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    acc = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.empty(n, dtype=torch.int32, device="cuda")
    for e in (5, 10):
        gpu.generate_device(1, 99 + e, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
        seen = set()
        for _ in range(30):
            acc.fill_(-1)
            est.fill_(-1)
            gpu.shouji_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                     d_estimates=est.data_ptr())
            torch.cuda.synchronize()
            h = hashlib.sha256(acc.cpu().numpy().tobytes() + est.cpu().numpy().tobytes()).hexdigest()
            seen.add(h)
        assert len(seen) == 1, f"E={e}: {len(seen)} different results over 30 runs"
