"""SM-split pack | search pipeline sweep (csrc/split.cpp): pack-partition SMs x chunk
size against the serial pack + search, device-resident configs[1] records, with the
bitmap and estimates checked against the serial run.

python tools/exp_split.py [--m 100 --e 5 --pairs 30000000] [--sms 48,56,64] [--chunks 2,3,4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_07858_b200 as pf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=30_000_000)
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--e", type=str, default="5")
ap.add_argument("--kind", type=int, default=1)
ap.add_argument("--sms", default="40,48,56,64,72")
ap.add_argument("--chunks", default="1,2,3,4,6", help="Mi pairs")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

n, m = a.pairs, a.m
pitch = pf.device_pitch(m)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
sh = s.cuda_stream
t = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
p = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
est = torch.zeros(n, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")


def run(reps):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        pf.shouji_filter_device_async(t.data_ptr(), p.data_ptr(), pitch, n, m, E, acc.data_ptr(),
                                      flag.data_ptr(), stream=sh, d_estimates=est.data_ptr())
    ev0.record(s)
    for _ in range(reps):
        pf.shouji_filter_device_async(t.data_ptr(), p.data_ptr(), pitch, n, m, E, acc.data_ptr(),
                                      flag.data_ptr(), stream=sh, d_estimates=est.data_ptr())
    ev1.record(s)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / reps


rows = []
for E in [int(x) for x in a.e.split(",")]:
    pf.generate_device(a.kind, 1809078581 + 1000 * E, E, t.data_ptr(), p.data_ptr(), pitch, n, m,
                       stream=sh)
    torch.cuda.synchronize()
    os.environ["PF_SPLIT"] = "0"
    base = run(a.reps)
    ref_acc, ref_est = acc.clone(), est.clone()
    print(f"E={E} serial: {base:.3f} ms  {n / base / 1e6:.2f} G pairs/s", flush=True)
    rows.append({"E": E, "m": m, "sms": 0, "chunk": 0, "ms": base})
    for sms in [int(x) for x in a.sms.split(",")]:
        for ch in [float(x) for x in a.chunks.split(",")]:
            os.environ["PF_SPLIT"] = str(sms)
            os.environ["PF_SPLIT_CHUNK"] = str(int(ch * (1 << 20)))
            acc.zero_()
            est.zero_()
            ms = run(a.reps)
            ok = torch.equal(acc, ref_acc) and torch.equal(est, ref_est) and int(flag.item()) == 0
            print(f"E={E} pack SMs {sms:3d} chunk {ch:4.1f} Mi: {ms:.3f} ms  "
                  f"{n / ms / 1e6:.2f} G pairs/s  x{base / ms:.3f}  {'ok' if ok else 'MISMATCH'}",
                  flush=True)
            rows.append({"E": E, "m": m, "sms": sms, "chunk": ch, "ms": ms, "ok": ok})
os.environ["PF_SPLIT"] = "0"
print(json.dumps(rows))
