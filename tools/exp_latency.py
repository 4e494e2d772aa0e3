"""Small-batch latency of the host and device entry points (n=1000, m=96)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402
from paper_1809_07858_b200 import _lib as L  # noqa: E402


def bench(fn, n=500):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


n, m, e = 1000, 96, 5
a = np.frombuffer(("GGTGCAGAGCTC" * 8).encode(), np.uint8)[None, :].repeat(n, 0).copy()
ctx = pf.default_context()
acc = np.zeros((n + 31) // 32, np.uint32)
err = L.PfError()
p = a.ctypes.data_as(C.c_void_p)
pacc = acc.ctypes.data_as(C.c_void_p)
print("raw C ABI batch (pageable in/out)", bench(lambda: L.lib.pf_shouji_filter_batch(
    ctx.handle, p, p, m, n, m, e, 4, pacc, None, None, C.byref(err))), "us")
pin = torch.from_numpy(a).pin_memory().numpy()
pacc_pin = torch.zeros(acc.size, dtype=torch.int32).pin_memory().numpy()
pp = pin.ctypes.data_as(C.c_void_p)
print("raw C ABI batch (pinned in/out)", bench(lambda: L.lib.pf_shouji_filter_batch(
    ctx.handle, pp, pp, m, n, m, e, 4, pacc_pin.ctypes.data_as(C.c_void_p), None, None,
    C.byref(err))), "us")
td = torch.from_numpy(a).cuda()
accd = torch.zeros(acc.size, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()


def dev():
    pf.shouji_filter_device_async(td.data_ptr(), td.data_ptr(), m, n, m, e, accd.data_ptr(),
                                  flag.data_ptr(), stream=s.cuda_stream)
    s.synchronize()


print("device async + sync", bench(dev), "us")
print("python per-pair API", bench(lambda: pf.shouji_filter(pf.seq("GGTGAGAGTTGT" * 8),
                                                            pf.seq("GGTGCAGAGCTC" * 8), 5)), "us")

# per-pair entry point (pf_shouji_filter_one -> latency kernel, csrc/small.cu), m = 100
one = b"GGTGCAGAGCTC" * 8 + b"ACGT"
est, ok = C.c_uint32(), C.c_int()
for small in ("1", "0"):
    os.environ["PF_SMALL"] = small
    print(f"pf_shouji_filter_one m=100 e=5 (PF_SMALL={small})", bench(lambda: L.lib.pf_shouji_filter_one(
        ctx.handle, one, len(one), one, len(one), 5, 4, C.byref(ok), C.byref(est), None,
        C.byref(err)), 2000), "us")
    for k in (16, 64):
        b = np.frombuffer(one, np.uint8)[None, :].repeat(k, 0).copy()
        acck = np.zeros((k + 31) // 32, np.uint32)
        print(f"  batch of {k}", bench(lambda: L.lib.pf_shouji_filter_batch(
            ctx.handle, b.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), 100, k, 100, 5,
            4, acck.ctypes.data_as(C.c_void_p), None, None, C.byref(err)), 1000), "us")
os.environ.pop("PF_SMALL", None)
