"""A reduced parity run that touches every kernel family and every host-side
ordering mechanism once, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

  compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_suite.py

Each step checks its result against the CPU oracle, so a run under a sanitizer
is also a parity run. Steps:
  pack_search      TMA tile pack (pack_tile_kernel) + width-4 search, E = 0, 5, 13
  search_pf        cp.async prefetching search (E = 8..12 with N-presence flags off)
  wsearch          any-width blocked search (widths 3, 5, 8)
  host_dibits      host-pack upload path, dibit records (pack_dibit_kernel, TMA), copy stream
  host_nibbles     nibble records (PF_HOST_FORMAT=nibble)
  packed_planes    packed_sequence planes input (pack_planes_kernel)
  bits             tally-bit output (bits_transpose)
  streams          device calls on two torch streams reusing the plane scratch
  illegal          illegal byte located (locate kernel, on-stream key reset)
  small            latency kernel, mapped staging, completion flag
  magnet           MAGNET thread and warp forms
  edit_distance    Myers banded edit distance
  split            green-context pack | search pipeline (PF_SPLIT)
python tools/sanitize_suite.py [--quick] [--only step,step]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1809_07858_b200 as pf  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="smaller batches (racecheck)")
ap.add_argument("--only", default="")
args = ap.parse_args()
o = Oracle()
Q = args.quick
ONLY = {x for x in args.only.split(",") if x}
ALPHA = np.frombuffer(b"ACGT", np.uint8)


def gen(kind, e, m, n, seed=5):
    return o.gen_config(kind, 1000 + seed, e, m, 0, n)


def check(t, p, e, width=4, **kw):
    a1, e1, _ = pf.shouji_filter_batch(t, p, e, width=width, estimates=True, **kw)
    a2, e2, _ = o.shouji_batch(t, p, e, width=width)
    assert (a1 == a2).all() and (e1 == e2).all()


def step(name):
    def deco(fn):
        if ONLY and name not in ONLY:
            return fn
        t0 = time.time()
        fn()
        torch.cuda.synchronize()
        print(f"{name}: ok ({time.time() - t0:.1f} s)", flush=True)
        return fn
    return deco


def device_run(t, p, e, m, stream=None, bits=False):
    n = t.shape[0]
    pitch = pf.device_pitch(m)
    tt = torch.zeros((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.zeros((n, pitch), dtype=torch.uint8, device="cuda")
    tt[:, :m] = torch.from_numpy(t).cuda()
    pt[:, :m] = torch.from_numpy(p).cuda()
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    bv = torch.zeros((n, (m + 63) // 64), dtype=torch.int64, device="cuda") if bits else None
    torch.cuda.synchronize()
    pf.shouji_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                            d_estimates=est.data_ptr(), d_bits=bv.data_ptr() if bits else None,
                            stream=stream)
    return tt, pt, acc, est, bv


@step("pack_search")
def _():
    for e, m in [(0, 100), (5, 100), (13, 150)]:
        n = 4096 if Q else 20000
        t, p = gen(1, e, m, n)
        _, _, acc, est, _ = device_run(t, p, e, m)
        torch.cuda.synchronize()
        a2, e2, _ = o.shouji_batch(t, p, e)
        assert (acc.cpu().numpy().view(np.uint32) == a2).all()
        assert (est.cpu().numpy().view(np.uint32) == e2).all()


@step("search_pf")
def _():
    os.environ["PF_NFLAGS"] = "0"
    try:
        for e in (8, 10):
            t, p = gen(1, e, 100, 4096 if Q else 10000)
            _, _, acc, est, _ = device_run(t, p, e, 100)
            torch.cuda.synchronize()
            _, e2, _ = o.shouji_batch(t, p, e)
            assert (est.cpu().numpy().view(np.uint32) == e2).all()
    finally:
        os.environ.pop("PF_NFLAGS", None)


@step("wsearch")
def _():
    t, p = gen(3, 6, 250, 2048 if Q else 6000)
    for w in (3, 5, 8):
        check(t, p, 6, width=w)


@step("host_dibits")
def _():
    os.environ["PF_HOST_PACK"] = "1"
    try:
        t, p = gen(4, 25, 250, 70_000 if not Q else 20_000)  # config 4: N planes too
        check(t, p, 25)
        t, p = gen(1, 5, 100, 300_000 if not Q else 20_000)
        check(t, p, 5)
    finally:
        os.environ.pop("PF_HOST_PACK", None)


@step("host_nibbles")
def _():
    os.environ["PF_HOST_PACK"] = "1"
    os.environ["PF_HOST_FORMAT"] = "nibble"
    try:
        t, p = gen(1, 5, 100, 70_000 if not Q else 20_000)
        check(t, p, 5)
    finally:
        os.environ.pop("PF_HOST_PACK", None)
        os.environ.pop("PF_HOST_FORMAT", None)


@step("packed_planes")
def _():
    t, p = gen(2, 7, 150, 8192 if Q else 40_000)
    a1, e1, _ = pf.shouji_filter_packed_batch(pf.pack_planes(t), pf.pack_planes(p), 150, 7,
                                              estimates=True)
    a2, e2, _ = o.shouji_batch(t, p, 7)
    assert (a1 == a2).all() and (e1 == e2).all()


@step("bits")
def _():
    t, p = gen(1, 5, 100, 2048 if Q else 10_000)
    a1, e1, b1 = pf.shouji_filter_batch(t, p, 5, estimates=True, bits=True)
    a2, e2, b2 = o.shouji_batch(t, p, 5, bits=True)
    assert (a1 == a2).all() and (e1 == e2).all() and (b1 == b2).all()


@step("streams")
def _():
    # two device calls with tally bits on two streams: the second must not
    # overwrite the shared plane / tally scratch while the first still reads it
    t1, p1 = gen(1, 5, 100, 4096 if Q else 20_000, seed=1)
    t2, p2 = gen(1, 5, 100, 4096 if Q else 20_000, seed=2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    r1 = device_run(t1, p1, 5, 100, stream=s1.cuda_stream, bits=True)
    r2 = device_run(t2, p2, 5, 100, stream=s2.cuda_stream, bits=True)
    torch.cuda.synchronize()
    for (t, p), r in (((t1, p1), r1), ((t2, p2), r2)):
        a2, e2, b2 = o.shouji_batch(t, p, 5, bits=True)
        assert (r[3].cpu().numpy().view(np.uint32) == e2).all()
        assert (r[4].cpu().numpy().view(np.uint64) == b2).all()


@step("illegal")
def _():
    t, p = gen(1, 5, 100, 3000)
    t[2222, 17] = ord("x")
    for fn in (lambda: pf.shouji_filter_batch(t, p, 5),
               lambda: device_run(t, p, 5, 100)):
        try:
            fn()
        except pf.illegal_character_error as ex:
            assert (ex.pair, ex.field, ex.position()) == (2222, 0, 17)
        else:
            raise AssertionError("illegal byte not reported")


@step("small")
def _():
    for m, e in [(100, 5), (250, 25), (31, 3)]:
        t, p = gen(1, e, m, 64)
        check(t, p, e)
        a, est, _ = pf.shouji_filter_batch(t[:1], p[:1], e, estimates=True)
        _, e2, _ = o.shouji_batch(t[:1], p[:1], e)
        assert (est == e2).all()


@step("magnet")
def _():
    for m, e in [(100, 5), (250, 20)]:
        t, p = gen(1, e, m, 1024 if Q else 4096)
        a1, e1, _ = pf.magnet_filter_batch(t, p, e, estimates=True)
        a2, e2, _ = o.magnet_batch(t, p, e)
        assert (a1 == a2).all() and (e1 == e2).all()


@step("edit_distance")
def _():
    t, p = gen(1, 5, 100, 2048 if Q else 8192)
    d = pf.banded_edit_distance_batch(t, p, 5)
    for i in range(0, len(d), 97):
        want = o.banded_edit_distance(p[i].tobytes(), t[i].tobytes(), 5)
        assert d[i] == want


@step("split")
def _():
    os.environ["PF_SPLIT"] = "72"
    os.environ["PF_SPLIT_CHUNK"] = str(1 << 15)
    try:
        t, p = gen(1, 5, 100, 1 << 17)
        pitch = pf.device_pitch(100)
        n = t.shape[0]
        tt = torch.from_numpy(t).cuda()
        pt = torch.from_numpy(p).cuda()
        acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        est = torch.zeros(n, dtype=torch.int32, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream()
        pf.shouji_filter_device_async(tt.data_ptr(), pt.data_ptr(), pitch, n, 100, 5,
                                      acc.data_ptr(), flag.data_ptr(), d_estimates=est.data_ptr(),
                                      stream=s.cuda_stream)
        torch.cuda.synchronize()
        a2, e2, _ = o.shouji_batch(t, p, 5)
        assert (est.cpu().numpy().view(np.uint32) == e2).all()
        assert (acc.cpu().numpy().view(np.uint32) == a2).all()
    finally:
        os.environ.pop("PF_SPLIT", None)
        os.environ.pop("PF_SPLIT_CHUNK", None)


print("sanitize suite: all steps ok", flush=True)
