"""One MAGNET device call (config 1, m=100, E=5, 2M pairs) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
e = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 2_000_000
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pf.generate_device({100: 1, 150: 2, 250: 3}.get(m, 1), 5, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
for _ in range(2):
    pf.magnet_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr())
torch.cuda.synchronize()
print("ok")
