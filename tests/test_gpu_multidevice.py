"""Multi-device host batches (proj/src/evaluate.cpp:23-48 is the
partition being mirrored): a context over several devices shards each batch —
one contiguous 32-aligned shard per device, or 1Mi-pair chunks dealt
round-robin (BASELINE config 4's streaming layout) — with no collective; the
results must be bit-identical to one device's.

The context uses every visible device; on a one-GPU box it lists device 0
twice, which still runs two independent device states (buffers, streams,
pinned staging) fed by two host threads — the multi-device code path, without
a second GPU's bandwidth.

config 4 in full: 100M pairs of m = 250 (50 GB of host records) streamed in
1Mi-pair chunks round-robin, through pf_shouji_filter_batch, hashed against the
committed oracle digests of the same set (tests/golden/fullsize_digests.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def devices(gpu):
    k = gpu.device_count()
    return list(range(k)) if k > 1 else [0, 0]


@pytest.mark.parametrize("chunk", [0, 65536, 1 << 20])
def test_every_visible_device_matches_one_device(gpu, oracle, chunk):
    n, m, e = 1_200_000, 100, 5
    t, p = oracle.gen_config(1, 4242, e, m, 0, n)
    one = gpu.Context([0])
    a1, e1, _ = gpu.shouji_filter_batch(t, p, e, estimates=True, ctx=one)
    multi = gpu.Context(devices(gpu))
    multi.set_shard_chunk(chunk)
    a2, e2, _ = gpu.shouji_filter_batch(t, p, e, estimates=True, ctx=multi)
    assert (a1 == a2).all() and (e1 == e2).all()
    k = 20_000
    a3, e3, _ = oracle.shouji_batch(t[-k:], p[-k:], e)
    assert (e2[-k:] == e3).all()
    # MAGNET shards the same way
    ma, me, _ = gpu.magnet_filter_batch(t[:200_000], p[:200_000], e, estimates=True, ctx=one)
    mb, mf, _ = gpu.magnet_filter_batch(t[:200_000], p[:200_000], e, estimates=True, ctx=multi)
    assert (ma == mb).all() and (me == mf).all()
    one.close()
    multi.close()


def test_illegal_byte_reported_from_the_right_shard(gpu, oracle):
    n, m = 300_000, 100
    t, p = oracle.gen_config(1, 4343, 5, m, 0, n)
    p[250_001, 7] = ord("q")
    t[260_000, 3] = ord("-")
    multi = gpu.Context(devices(gpu))
    multi.set_shard_chunk(65536)
    with pytest.raises(gpu.illegal_character_error) as ex:
        gpu.shouji_filter_batch(t, p, 5, ctx=multi)
    assert (ex.value.pair, ex.value.field, ex.value.position()) == (250_001, 1, 7)
    multi.close()


def test_config4_streamed_round_robin_100M(gpu):
    import torch
    sets = json.load(open(os.path.join(HERE, "golden", "fullsize_digests.json")))["sets"]
    s = [x for x in sets if x["config"] == 4][0]
    n, m, e = s["n"], s["m"], s["E"]
    pitch = gpu.device_pitch(m)
    # the set's ASCII records (one generator launch on the device, 50 GB), copied
    # out to pageable host memory in slices, then the device copy is freed
    ht = np.empty((n, m), np.uint8)
    hp = np.empty((n, m), np.uint8)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    gpu.generate_device(4, s["seed"], e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    torch.cuda.synchronize()
    step = 8_000_000
    for lo in range(0, n, step):
        ht[lo:lo + step] = tt[lo:lo + step, :m].cpu().numpy()
        hp[lo:lo + step] = pt[lo:lo + step, :m].cpu().numpy()
    del tt, pt
    torch.cuda.empty_cache()
    # streamed: 1Mi-pair chunks dealt round-robin over the devices, host-packed,
    # uploaded, filtered, bitmaps gathered at their word offsets
    ctx = gpu.Context(devices(gpu))
    ctx.set_shard_chunk(1 << 20)
    acc, est, _ = gpu.shouji_filter_batch(ht, hp, e, estimates=True, ctx=ctx)
    ctx.close()
    assert hashlib.sha256(acc.astype("<u4").tobytes()).hexdigest() == s["accept_sha256"]
    assert hashlib.sha256(est.astype("<u4").tobytes()).hexdigest() == s["estimate_sha256"]
