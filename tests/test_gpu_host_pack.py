"""GPU parity of the host-pack upload path: records packed on the host's cores
(csrc/host_pack.cpp) into dibit records (+ N planes when a chunk has an N; the
default) or nibble records, filtered on the device from them (pack.cuh formats,
phase_a.cuh gather_chunk_dib / gather_chunk_nib) — against the oracle.

pf_shouji_filter_batch routes host batches of >= 65536 pairs through this path
(PF_HOST_PACK unset), so the large-batch tests below exercise it end to end,
including chunk boundaries (256Ki pairs per chunk) and error order across chunks.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ACGT = np.frombuffer(b"ACGT", np.uint8)
ACGTN = np.frombuffer(b"ACGTN", np.uint8)


def mutated(rng, n, m, rate=0.06, alphabet=ACGTN):
    t = alphabet[rng.integers(0, len(alphabet), size=(n, m))]
    p = t.copy()
    mask = rng.random(p.shape) < rate
    p[mask] = ACGT[rng.integers(0, 4, size=int(mask.sum()))]
    # some shifted patterns (indels) so the diagonals matter
    for i in range(0, n, 7):
        s = int(rng.integers(-3, 4))
        p[i] = np.roll(p[i], s)
    return np.ascontiguousarray(t), np.ascontiguousarray(p)


def run_nibbles(gpu, t, p, e, width=4):
    import torch
    n, m = t.shape
    nt, npat = gpu.host_pack_nibbles(t, p)
    dt = torch.from_numpy(nt).cuda()
    dp = torch.from_numpy(npat).cuda()
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    gpu.shouji_filter_nibbles_device(dt.data_ptr(), dp.data_ptr(), n, m, e, acc.data_ptr(),
                                     width=width, d_estimates=est.data_ptr())
    torch.cuda.synchronize()
    return acc.cpu().numpy().view(np.uint32), est.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("m", [1, 2, 5, 8, 9, 15, 16, 17, 31, 33, 64, 100, 127, 128, 129, 150,
                               250, 255, 256, 300, 512])
def test_nibble_device_path_lengths(gpu, oracle, m):
    rng = np.random.default_rng(m)
    n = 2000 + 3 * m + 5  # ragged last tile
    t, p = mutated(rng, n, m)
    for e in sorted({0, min(m - 1, 1), min(m - 1, 3), min(m - 1, 9), m - 1}):
        a1, e1 = run_nibbles(gpu, t, p, e)
        a2, e2, _ = oracle.shouji_batch(t, p, e)
        assert (a1 == a2).all(), (m, e)
        assert (e1 == e2).all(), (m, e)


@pytest.mark.parametrize("width", [3, 5, 6, 7, 8])
def test_nibble_device_path_widths(gpu, oracle, width):
    rng = np.random.default_rng(100 + width)
    t, p = mutated(rng, 3001, 100)
    for e in (2, 5, 12):
        a1, e1 = run_nibbles(gpu, t, p, e, width)
        a2, e2, _ = oracle.shouji_batch(t, p, e, width)
        assert (a1 == a2).all() and (e1 == e2).all(), (width, e)


def test_nibble_device_path_rejects_bad_parameters(gpu):
    import torch
    buf = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    acc = torch.zeros(4, dtype=torch.int32, device="cuda")
    for m, e, w in [(10, 10, 4), (10, 3, 2), (10, 3, 9), (0, 0, 4)]:
        with pytest.raises(gpu.invalid_parameters_error):
            gpu.shouji_filter_nibbles_device(buf.data_ptr(), buf.data_ptr(), 32, m, e,
                                             acc.data_ptr(), width=w)
    with pytest.raises(gpu.invalid_parameters_error):  # bulk copies need 16-byte aligned bases
        gpu.shouji_filter_nibbles_device(buf.data_ptr() + 4, buf.data_ptr(), 32, 10, 3,
                                         acc.data_ptr())


@pytest.mark.parametrize("n", [65536, 65536 + 31, 1_200_001])
def test_host_batch_uses_dibits_and_matches(gpu, oracle, n):
    rng = np.random.default_rng(n)
    t, p = mutated(rng, n, 100, alphabet=ACGT)
    before = gpu.launch_count()
    h0, _ = gpu.transfer_bytes()
    a1, e1, _ = gpu.shouji_filter_batch(t, p, 5, estimates=True)
    assert gpu.launch_count() > before
    h1, _ = gpu.transfer_bytes()
    assert h1 - h0 == 2 * n * gpu.dibit_pitch(100)  # dibit records (no N) crossed PCIe, not ASCII
    a2, e2, _ = oracle.shouji_batch(t, p, 5)
    assert (a1 == a2).all() and (e1 == e2).all()


def test_host_batch_pinned_and_strided(gpu, oracle):
    import torch
    rng = np.random.default_rng(5)
    n, m, stride = 300_000, 150, 157
    t, p = mutated(rng, n, m)
    bt = torch.full((n, stride), ord("q"), dtype=torch.uint8).pin_memory()
    bp = torch.full((n, stride), ord("q"), dtype=torch.uint8).pin_memory()
    bt.numpy()[:, :m] = t
    bp.numpy()[:, :m] = p
    a1, e1, _ = gpu.shouji_filter_batch(bt.numpy(), bp.numpy(), 7, m=m, estimates=True)
    a2, e2, _ = oracle.shouji_batch(t, p, 7)
    assert (a1 == a2).all() and (e1 == e2).all()


def test_host_batch_first_illegal_byte_across_chunks(gpu):
    rng = np.random.default_rng(11)
    n, m = 1_100_000, 100
    t = np.ascontiguousarray(ACGT[rng.integers(0, 4, size=(n, m))])
    p = t.copy()
    p[1_050_000, 5] = ord("x")   # third chunk
    t[700_000, 99] = ord("-")    # second chunk: reported first
    with pytest.raises(gpu.illegal_character_error) as ei:
        gpu.shouji_filter_batch(t, p, 5)
    err = ei.value
    assert (err.pair, err.field, err.position(), err.byte()) == (700_000, 0, 99, "-")
    t[700_000, 99] = ord("A")
    with pytest.raises(gpu.illegal_character_error) as ei:
        gpu.shouji_filter_batch(t, p, 5)
    assert (ei.value.pair, ei.value.field, ei.value.position()) == (1_050_000, 1, 5)
    p[1_050_000, 5] = ord("A")
    gpu.shouji_filter_batch(t, p, 5)  # and the context still works


def test_host_pack_with_device_shards(gpu, oracle):
    """A context over several devices runs one host-pack stream per shard (here the
    same device listed three times); results and first-error order are unchanged."""
    rng = np.random.default_rng(21)
    n = 600_001
    t, p = mutated(rng, n, 100, alphabet=ACGT)
    a_ref, e_ref, _ = oracle.shouji_batch(t, p, 5)
    ctx = gpu.Context([0, 0, 0])
    try:
        a, e, _ = gpu.shouji_filter_batch(t, p, 5, estimates=True, ctx=ctx)
        assert (a == a_ref).all() and (e == e_ref).all()
        p[450_000, 1] = ord("#")  # third shard
        t[250_000, 2] = ord("@")  # second shard: reported
        with pytest.raises(gpu.illegal_character_error) as ei:
            gpu.shouji_filter_batch(t, p, 5, ctx=ctx)
        assert (ei.value.pair, ei.value.field, ei.value.position()) == (250_000, 0, 2)
    finally:
        ctx.close()


def run_dibits(gpu, t, p, e, width=4):
    import torch
    n, m = t.shape
    dt, dq, nt, nq = gpu.host_pack_dibits(t, p)
    tens = [torch.from_numpy(a).cuda() if a is not None else None for a in (dt, dq, nt, nq)]
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    gpu.shouji_filter_dibits_device(tens[0].data_ptr(), tens[1].data_ptr(), n, m, e, acc.data_ptr(),
                                    d_ntext=tens[2].data_ptr() if nt is not None else None,
                                    d_npattern=tens[3].data_ptr() if nq is not None else None,
                                    width=width, d_estimates=est.data_ptr())
    torch.cuda.synchronize()
    return acc.cpu().numpy().view(np.uint32), est.cpu().numpy().view(np.uint32), nt is not None


@pytest.mark.parametrize("m", [1, 2, 5, 15, 16, 17, 31, 33, 64, 100, 127, 128, 150, 250, 256, 300])
@pytest.mark.parametrize("alphabet", ["ACGT", "ACGTN"])
def test_dibit_device_path(gpu, oracle, m, alphabet):
    rng = np.random.default_rng(m + len(alphabet))
    a = np.frombuffer(alphabet.encode(), np.uint8)
    t, p = mutated(rng, 1500 + 3 * m, m, alphabet=a)
    for e in sorted({0, min(m - 1, 2), min(m - 1, 5), min(m - 1, 17), m - 1}):
        a1, e1, had_n = run_dibits(gpu, t, p, e)
        assert had_n == (alphabet == "ACGTN")
        a2, e2, _ = oracle.shouji_batch(t, p, e)
        assert (a1 == a2).all() and (e1 == e2).all(), (m, e, alphabet)


def test_host_batch_chunks_with_and_without_n(gpu, oracle):
    """Chunks without N upload dibits only; a chunk with one N adds its N planes."""
    rng = np.random.default_rng(17)
    n = 700_000
    t, p = mutated(rng, n, 100, alphabet=ACGT)
    t[400_000, 50] = ord("N")  # second chunk only
    h0, _ = gpu.transfer_bytes()
    a1, e1, _ = gpu.shouji_filter_batch(t, p, 5, estimates=True)
    h1, _ = gpu.transfer_bytes()
    a2, e2, _ = oracle.shouji_batch(t, p, 5)
    assert (a1 == a2).all() and (e1 == e2).all()
    chunk = 1 << 18
    cn = min(chunk, n - chunk)
    assert h1 - h0 == 2 * n * gpu.dibit_pitch(100) + 2 * cn * gpu.nplane_pitch(100)


@pytest.mark.parametrize("m,e", [(100, 5), (100, 20), (17, 3), (250, 25), (512, 9)])
def test_magnet_host_batch_reads_dibits(gpu, oracle, m, e):
    """MAGNET host batches of >= 65536 pairs run straight from the dibit records
    (magnet.cu DibitSrc): two dibit rows per pair cross PCIe, and chunks with and
    without N (N planes uploaded only where present) match the oracle bit for bit."""
    rng = np.random.default_rng(m * 31 + e)
    n = 70_000 if m <= 100 else 66_000
    t, p = mutated(rng, n, m, alphabet=ACGT)
    t[n - 3, m // 2] = ord("N")  # one N in the only chunk
    h0, _ = gpu.transfer_bytes()
    a1, e1, b1 = gpu.magnet_filter_batch(t, p, e, estimates=True, bits=True)
    h1, _ = gpu.transfer_bytes()
    assert h1 - h0 == 2 * n * (gpu.dibit_pitch(m) + gpu.nplane_pitch(m))
    a2, e2, b2 = oracle.magnet_batch(t, p, e, bits=True)
    assert (e1 == e2).all() and (a1 == a2).all() and (b1 == b2).all()


def test_magnet_host_batch_chunks_and_errors(gpu, oracle):
    rng = np.random.default_rng(99)
    n, m = 600_000, 100  # three chunks; N only in the second
    t, p = mutated(rng, n, m, alphabet=ACGT)
    p[300_000:300_010, 3] = ord("N")
    a1, e1, _ = gpu.magnet_filter_batch(t, p, 6, estimates=True)
    a2, e2, _ = oracle.magnet_batch(t, p, 6)
    assert (e1 == e2).all() and (a1 == a2).all()
    p[590_000, 5] = ord("x")   # third chunk
    t[400_000, 99] = ord("-")  # second chunk: reported first
    with pytest.raises(gpu.illegal_character_error) as ei:
        gpu.magnet_filter_batch(t, p, 6)
    assert (ei.value.pair, ei.value.field, ei.value.position()) == (400_000, 0, 99)


@pytest.fixture
def hybrid_on():
    os.environ["PF_HYBRID"] = "1"
    yield
    os.environ.pop("PF_HYBRID", None)


def test_hybrid_upload_routes_match(gpu, oracle, hybrid_on):
    """PF_HYBRID=1: raw-ASCII chunks DMA'd from the pinned records run alongside the
    host-packed chunks (two routes taking chunks from one counter); the results must
    be the single-route results, and an illegal byte anywhere must still be the first
    one in pair order whichever route met it."""
    import torch
    n, m, e = 3_000_000, 100, 5
    t, p = oracle.gen_config(1, 5150, e, m, 0, n)
    ht = torch.from_numpy(t).pin_memory().numpy()
    hp = torch.from_numpy(p).pin_memory().numpy()
    a1, e1, _ = gpu.shouji_filter_batch(ht, hp, e, estimates=True)
    os.environ["PF_HYBRID"] = "0"
    a2, e2, _ = gpu.shouji_filter_batch(ht, hp, e, estimates=True)
    os.environ["PF_HYBRID"] = "1"
    assert (a1 == a2).all() and (e1 == e2).all()
    k = 20_000
    _, e3, _ = oracle.shouji_batch(t[-k:], p[-k:], e)
    assert (e1[-k:] == e3).all()
    for where in [(2_900_001, 1, 99), (262_145, 0, 0), (1_000_000, 1, 50)]:
        hq = hp.copy() if where[1] else hp
        hu = ht.copy() if not where[1] else ht
        hq = torch.from_numpy(hq).pin_memory().numpy()
        hu = torch.from_numpy(hu).pin_memory().numpy()
        tgt = hq if where[1] else hu
        tgt[where[0], where[2]] = ord("z")
        tgt[2_999_999, 3] = ord("y")  # a later one must not win
        with pytest.raises(gpu.illegal_character_error) as ex:
            gpu.shouji_filter_batch(hu, hq, e)
        assert (ex.value.pair, ex.value.field, ex.value.position()) == where
