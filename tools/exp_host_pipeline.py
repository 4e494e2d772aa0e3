"""Where the e2e (host records -> accept bitmap) time goes, on the bench workload:

* host_read  — the host cores stream-reading the pinned ASCII records (pf_host_read_bandwidth);
* pack_full  — the dibit host pack of all n pairs into one big pinned output (no DMA);
* pack_chunk — the same pack chunk by chunk (PF_HOST_CHUNK pairs) into two alternating
               pinned buffers, as the upload pipeline runs it, but with no DMA;
* batch      — pf_shouji_filter_batch end to end (pack + DMA + kernels + bitmap D2H).

python tools/exp_host_pipeline.py [n]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402
from paper_1809_07858_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
m, e = 100, 5
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(1, 1809078581 + 5000, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
ht = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
hp = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
ht.copy_(tt[:, :m])
hp.copy_(pt[:, :m])
del tt, pt
torch.cuda.empty_cache()
tn, pn = ht.numpy(), hp.numpy()
ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
out = {"n": n, "threads": int(os.environ.get("PF_HOST_THREADS", os.cpu_count() or 1)),
       "env": {k: v for k, v in os.environ.items() if k.startswith("PF_")}}
out["host_read_gbs"] = pf.host_read_bandwidth(tn, passes=2)
out["host_read_bound_pairs_per_s"] = out["host_read_gbs"] * 1e9 / (2 * m)

dp, npp = pf.dibit_pitch(m), pf.nplane_pitch(m)
err, has_n = L.PfError(), C.c_int()


def pack(t_src, p_src, k, ot, op, nt, nq):
    st = L.lib.pf_host_pack_dibits(ptr(t_src), ptr(p_src), m, k, m, ptr(ot), ptr(op), ptr(nt),
                                   ptr(nq), C.byref(has_n), 1, C.byref(err))
    assert st == 0


big_t = torch.empty((n, dp), dtype=torch.uint8, pin_memory=True).numpy()
big_p = torch.empty((n, dp), dtype=torch.uint8, pin_memory=True).numpy()
nt = np.zeros((n, npp), np.uint8)
nq = np.zeros((n, npp), np.uint8)
pack(tn, pn, n, big_t, big_p, nt, nq)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    pack(tn, pn, n, big_t, big_p, nt, nq)
    ts.append(time.perf_counter() - t0)
out["pack_full_pairs_per_s"] = n / min(ts)

chunk = int(os.environ.get("PF_HOST_CHUNK", 1 << 18))
bufs = [(torch.empty((chunk, dp), dtype=torch.uint8, pin_memory=True).numpy(),
         torch.empty((chunk, dp), dtype=torch.uint8, pin_memory=True).numpy()) for _ in range(2)]
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    for i, lo in enumerate(range(0, n, chunk)):
        k = min(chunk, n - lo)
        bt, bp = bufs[i & 1]
        pack(tn[lo:], pn[lo:], k, bt, bp, nt, nq)
    ts.append(time.perf_counter() - t0)
out["pack_chunk_pairs_per_s"] = n / min(ts)
out["chunk"] = chunk

pf.shouji_filter_batch(tn, pn, e)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    pf.shouji_filter_batch(tn, pn, e)
    ts.append(time.perf_counter() - t0)
out["batch_pairs_per_s"] = n / float(np.median(ts))
out["batch_best_pairs_per_s"] = n / min(ts)
print(json.dumps(out))
