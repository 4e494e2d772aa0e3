"""MAGNET throughput: GPU (device-resident, validation + kernel) vs the
reference library on the host cores. One JSON line per (m, e)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

ref = Reference() if Reference.available() else None
for kind, m, e, n in [(1, 100, 2, 4_000_000), (1, 100, 5, 4_000_000), (1, 100, 10, 2_000_000),
                      (2, 150, 7, 2_000_000), (3, 250, 15, 1_000_000), (3, 250, 25, 1_000_000)]:
    pitch = pf.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pf.generate_device(kind, 11 + e, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.zeros(n, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    pf.magnet_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                            d_estimates=est.data_ptr(), stream=s.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        pf.magnet_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                d_estimates=est.data_ptr(), stream=s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    gpu = n / float(np.median(ts))
    line = {"m": m, "e": e, "config": kind, "gpu_pairs_per_s": gpu}
    if ref is not None:
        k = 200_000
        t = tt[:k, :m].cpu().numpy()
        p = pt[:k, :m].cpu().numpy()
        packed = ref.pack(t, p)
        t0 = time.perf_counter()
        ra, re_ = packed.magnet(e)
        cpu = k / (time.perf_counter() - t0)
        packed.free()
        ga = acc[: k // 32].cpu().numpy().view(np.uint32)
        ge = est[:k].cpu().numpy().view(np.uint32)
        line.update(cpu_pairs_per_s=cpu, cpu_threads=ref.hardware_concurrency(),
                    parity=bool((ga == ra).all() and (ge == re_).all()))
    print(json.dumps(line), flush=True)
    del tt, pt
