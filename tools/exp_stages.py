"""Pack / search split of the device path per threshold (CUDA events between the
two launches, pf_shouji_profile_stages). python tools/exp_stages.py [m] [E,E,...] [kind]
Env switches (PF_NFLAGS, PF_SEARCH_PF, ...) select the variants being compared."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100
es = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5]
kind = int(sys.argv[3]) if len(sys.argv) > 3 else {100: 1, 150: 2, 250: 3}.get(m, 1)
n = 16_000_000 if m <= 150 else 8_000_000
pitch = pf.device_pitch(m)
tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
out = {"m": m, "kind": kind, "pairs": n, "env": {k: v for k, v in os.environ.items() if k.startswith("PF_")}}
for e in es:
    pf.generate_device(kind, 100 + e, e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    pf.profile_stages(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                      flag.data_ptr(), reps=1)  # warm-up: scratch allocation, smem attributes
    pk, se = pf.profile_stages(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                               flag.data_ptr(), reps=10)
    out[f"E{e}"] = {"pack_ms": round(pk, 4), "search_ms": round(se, 4),
                    "Gpairs_s": round(n / ((pk + se) * 1e-3) / 1e9, 3)}
print(json.dumps(out))
