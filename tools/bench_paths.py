"""Measurement of the §8(f) paths beside the headline (bench.py measures Shouji):
MAGNET, the exact banded edit distance (verification / eval oracle) and the
packed-planes Shouji variant. One JSON line per path on stdout:

  value  — device-resident pairs/s (CUDA events on the launching stream), where
           the path has a device entry point;
  e2e    — the host entry point from pinned host buffers (H2D + kernels + D2H +
           sync), pairs/s;
  cpu_baseline — the unmodified reference library (oracle/_ref) on all host
           threads over a bounded sample of the same pairs.

python tools/bench_paths.py > profiles/r1_secondary_paths.jsonl
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_07858_b200 as pf  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

REF = Reference() if Reference.available() else None


def gen(kind, m, e, n, seed):
    pitch = pf.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pf.generate_device(kind, seed, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    return tt, pt, pitch


def time_device(fn, reps=5):
    s = torch.cuda.current_stream()
    fn(s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(s)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def time_host(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def cpu_sample(fn, k):
    if REF is None:
        return None
    t0 = time.perf_counter()
    fn()
    dt = time.perf_counter() - t0
    return {"value": k / dt, "unit": "pairs/s", "cores": REF.hardware_concurrency(),
            "kind": "reference", "sample": f"first {k} pairs of the workload, pre-packed"}


def host_copy(tt, pt, m):
    n = tt.shape[0]
    ht = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
    hp = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
    ht.copy_(tt[:, :m])
    hp.copy_(pt[:, :m])
    return ht.numpy(), hp.numpy()


def magnet_line(kind, m, e, n):
    tt, pt, pitch = gen(kind, m, e, n, 900 + e)
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    dev = time_device(lambda s: pf.magnet_filter_device(
        tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(), stream=s.cuda_stream))
    ht, hp = host_copy(tt, pt, m)
    host = time_host(lambda: pf.magnet_filter_batch(ht, hp, e))
    k = 100_000 if e <= 10 else 20_000
    cpu = None
    if REF is not None:
        packed = REF.pack(ht[:k], hp[:k])
        cpu = cpu_sample(lambda: packed.magnet(e), k)
        packed.free()
    return {"path": "magnet_filter (magnet.cpp:77-87)", "metric": f"MAGNET pairs filtered/sec (m={m},E={e})",
            "value": n / dev, "unit": "pairs/s", "config": {"workload": f"config {kind}", "m": m, "E": e,
                                                          "pairs": n},
            "e2e": {"value": n / host, "unit": "pairs/s"}, "cpu_baseline": cpu}


def edit_distance_line(m, e, n):
    tt, pt, pitch = gen(1, m, e, n, 800 + e)
    ht, hp = host_copy(tt, pt, m)
    host = time_host(lambda: pf.banded_edit_distance_batch(ht, hp, e))
    k = 100_000
    cpu = None
    if REF is not None:
        packed = REF.pack(ht[:k], hp[:k])
        cpu = cpu_sample(lambda: packed.banded(e), k)
        packed.free()
    return {"path": "banded_edit_distance (edit_distance.cpp:26-70)",
            "metric": f"edit distances/sec (m={m},e={e})", "value": None, "unit": "pairs/s",
            "config": {"workload": "config 1", "m": m, "E": e, "pairs": n},
            "e2e": {"value": n / host, "unit": "pairs/s"}, "cpu_baseline": cpu}


def packed_line(m, e, n):
    tt, pt, pitch = gen(1, m, e, n, 700 + e)
    ht, hp = host_copy(tt, pt, m)
    tp, pp = pf.pack_planes(ht), pf.pack_planes(hp)
    dt, dp = torch.from_numpy(tp).cuda(), torch.from_numpy(pp).cuda()
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    dev = time_device(lambda s: pf.shouji_filter_packed_device(
        dt.data_ptr(), dp.data_ptr(), n, m, e, acc.data_ptr(), stream=s.cuda_stream))
    tpin = torch.from_numpy(tp.reshape(n, -1)).pin_memory().numpy().reshape(tp.shape)
    ppin = torch.from_numpy(pp.reshape(n, -1)).pin_memory().numpy().reshape(pp.shape)
    host = time_host(lambda: pf.shouji_filter_packed_batch(tpin, ppin, m, e))
    return {"path": "shouji_filter on pre-packed pairs (packed-planes variant, SURVEY 8(b))",
            "metric": f"Shouji pairs filtered/sec (m={m},E={e}, packed input)", "value": n / dev,
            "unit": "pairs/s", "config": {"workload": "config 1", "m": m, "E": e, "pairs": n},
            "e2e": {"value": n / host, "unit": "pairs/s",
                    "h2d_bytes_per_pair": 2 * pf.packed_words(m) * 8}}


def main():
    lines = [
        magnet_line(1, 100, 5, 8_000_000),
        magnet_line(3, 250, 25, 1_000_000),
        edit_distance_line(100, 5, 8_000_000),
        packed_line(100, 5, 8_000_000),
    ]
    for line in lines:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
