"""Edit-distance (Myers bit-vector, edit_distance.cu) on config 1 pairs for ncu:
python tools/prof_edit.py [m] [e] [pairs]. Pairs are generated on the device and
copied to host records, then run through pf_banded_edit_distance_batch twice."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
e = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4_000_000
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device({100: 1, 150: 2, 250: 3}.get(m, 1), 5, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
t = tt[:, :m].cpu().numpy().copy()
p = pt[:, :m].cpu().numpy().copy()
for _ in range(2):
    t0 = time.perf_counter()
    d = pf.banded_edit_distance_batch(t, p, e)
    print(f"{n / (time.perf_counter() - t0) / 1e6:.1f} M pairs/s (host batch), within e: {(d >= 0).mean():.3f}")
