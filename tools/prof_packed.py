"""One packed-planes device call on 2M pairs (m=100, E=5) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

n, m, e = 2_000_000, 100, 5
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device(1, 5, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
dt = torch.from_numpy(pf.pack_planes(tt[:, :m].cpu().numpy())).cuda()
dp = torch.from_numpy(pf.pack_planes(pt[:, :m].cpu().numpy())).cuda()
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
for _ in range(2):
    pf.shouji_filter_packed_device(dt.data_ptr(), dp.data_ptr(), n, m, e, acc.data_ptr())
torch.cuda.synchronize()
print("ok")
