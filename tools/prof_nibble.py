"""One host-pack batch (2Mi pairs, m=100, E=5) for ncu: nibble pack + search kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

n, m, e = 1 << 21, 100, 5
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(1, 5, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
ht = tt[:, :m].cpu().pin_memory().numpy()
hp = pt[:, :m].cpu().pin_memory().numpy()
for _ in range(2):
    pf.shouji_filter_batch(ht, hp, e)
print("ok")
