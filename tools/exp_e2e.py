"""e2e experiment: host batch throughput for the current PF_* environment.

python tools/exp_e2e.py [n] -> one JSON line: batch pairs/s, host-pack-only pairs/s.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
m, e = 100, 5
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(1, 7, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
ht = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
hp = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
ht.copy_(tt[:, :m])
hp.copy_(pt[:, :m])
del tt, pt
torch.cuda.empty_cache()
tn, pn = ht.numpy(), hp.numpy()
pf.shouji_filter_batch(tn, pn, e)
ts = []
for _ in range(4):
    t0 = time.perf_counter()
    pf.shouji_filter_batch(tn, pn, e)
    ts.append(time.perf_counter() - t0)
batch = n / float(np.median(ts))
# host pack alone into pinned buffers
np_ = pf.nibble_pitch(m)
ot = torch.empty((n, np_), dtype=torch.uint8, pin_memory=True).numpy()
op = torch.empty((n, np_), dtype=torch.uint8, pin_memory=True).numpy()
import ctypes as C  # noqa: E402
from paper_1809_07858_b200 import _lib as L  # noqa: E402
err = L.PfError()
hs = []
for _ in range(3):
    t0 = time.perf_counter()
    st = L.lib.pf_host_pack_nibbles(tn.ctypes.data_as(C.c_void_p), pn.ctypes.data_as(C.c_void_p), m, n, m,
                                    ot.ctypes.data_as(C.c_void_p), op.ctypes.data_as(C.c_void_p), 1,
                                    C.byref(err))
    hs.append(time.perf_counter() - t0)
    assert st == 0
# pure H2D of the nibble bytes
d = torch.empty((n, np_), dtype=torch.uint8, device="cuda")
src = torch.from_numpy(ot)
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(src, non_blocking=True)
torch.cuda.synchronize()
h2d = n * np_ / (time.perf_counter() - t0)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PF_")},
                  "batch_pairs_per_s": batch, "host_pack_pairs_per_s": n / float(np.median(hs)),
                  "h2d_GBps": h2d / 1e9}))
