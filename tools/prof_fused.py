"""Minimal driver for ncu: device-generated configs[1] workload, a few fused launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_07858_b200 as pf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=4_000_000)
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--e", type=int, default=5)
ap.add_argument("--kind", type=int, default=1)
ap.add_argument("--launches", type=int, default=3)
a = ap.parse_args()
n, m, e = a.pairs, a.m, a.e
pitch = pf.device_pitch(m)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
t = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
p = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(a.kind, 1809078581 + 1000 * e, e, t.data_ptr(), p.data_ptr(), pitch, n, m,
                   stream=s.cuda_stream)
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.launches):
    ev0.record(s)
    pf.shouji_filter_device_async(t.data_ptr(), p.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                  flag.data_ptr(), stream=s.cuda_stream)
    ev1.record(s)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"launch {i}: {ms:.3f} ms  {n / ms / 1e6:.3f} G pairs/s")
assert int(flag.item()) == 0
