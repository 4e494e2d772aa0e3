"""Packed-planes variant throughput: device-resident (re-slice + search) and
host batch from pinned planes (H2D in chunks + kernels + D2H)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

n, m, e = 8_000_000, 100, 5
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(1, 5, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
t0 = time.time()
tp = pf.pack_planes(tt[:, :m].cpu().numpy())
pp = pf.pack_planes(pt[:, :m].cpu().numpy())
print("host pack_planes helper s", time.time() - t0, file=sys.stderr)
dt = torch.from_numpy(tp).cuda()
dp = torch.from_numpy(pp).cuda()
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
res = {}
for name, fn in [
    ("packed_device", lambda: pf.shouji_filter_packed_device(dt.data_ptr(), dp.data_ptr(), n, m, e,
                                                             acc.data_ptr(), stream=s.cuda_stream)),
    ("ascii_device", lambda: pf.shouji_filter_device_async(tt.data_ptr(), pt.data_ptr(), pitch, n, m,
                                                           e, acc.data_ptr(), flag.data_ptr(),
                                                           stream=s.cuda_stream)),
]:
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    res[name] = n / float(np.median(ts))
tpin = torch.from_numpy(tp.reshape(n, -1)).pin_memory().numpy().reshape(tp.shape)
ppin = torch.from_numpy(pp.reshape(n, -1)).pin_memory().numpy().reshape(pp.shape)
pf.shouji_filter_packed_batch(tpin, ppin, m, e)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    pf.shouji_filter_packed_batch(tpin, ppin, m, e)
    ts.append(time.perf_counter() - t0)
res["packed_host_pinned_e2e"] = n / float(np.median(ts))
ts = []
for _ in range(2):
    t0 = time.perf_counter()
    pf.shouji_filter_packed_batch(tp, pp, m, e)
    ts.append(time.perf_counter() - t0)
res["packed_host_pageable_e2e"] = n / float(np.median(ts))
print(json.dumps(res))
