"""Host dibit-pack throughput at PF_HOST_THREADS threads (8M random m=100 pairs):
for t in 1 2 4 8 16; do PF_HOST_THREADS=$t python tools/exp_host_threads.py; done"""
import os, sys, time, json, ctypes as C
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1809_07858_b200 as pf
from paper_1809_07858_b200 import _lib as L
n, m = 8_000_000, 100
rng = np.random.default_rng(1)
tn = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, size=(n, m), dtype=np.uint8)]
pn = tn.copy()
dp = pf.dibit_pitch(m)
ot = np.zeros((n, dp), np.uint8); op = np.zeros_like(ot)
nt_ = np.zeros((n, pf.nplane_pitch(m)), np.uint8); nq_ = np.zeros_like(nt_)
has_n = C.c_int(); err = L.PfError()
ptr = lambda a: a.ctypes.data_as(C.c_void_p)
def hp_():
    L.lib.pf_host_pack_dibits(ptr(tn), ptr(pn), m, n, m, ptr(ot), ptr(op), ptr(nt_), ptr(nq_), C.byref(has_n), 1, C.byref(err))
hp_(); ts=[]
for _ in range(3):
    t0=time.perf_counter(); hp_(); ts.append(time.perf_counter()-t0)
print(os.environ.get("PF_HOST_THREADS"), round(n/min(ts)/1e6,1), "M pairs/s", round(2*n*m/min(ts)/1e9,1), "GB/s ASCII read")
