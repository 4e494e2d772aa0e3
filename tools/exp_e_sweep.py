"""Device-resident throughput per threshold (config 1, m=100 unless given): pack +
search, CUDA events on the launching stream. python tools/exp_e_sweep.py [m] [E,E,...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
es = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 2, 5, 7, 10]
width = int(sys.argv[3]) if len(sys.argv) > 3 else 4
n = 16_000_000 if m <= 150 else 8_000_000
kind = {100: 1, 150: 2, 250: 3}.get(m, 1)
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
out = {"m": m, "pairs": n, "width": width}
for e in es:
    pf.generate_device(kind, 100 + e, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    run = lambda: pf.shouji_filter_device_async(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e,  # noqa
                                                acc.data_ptr(), flag.data_ptr(), width=width,
                                                stream=s.cuda_stream)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    out[f"E{e}"] = round(n / float(np.median(ts)) / 1e9, 3)
print(json.dumps(out))
