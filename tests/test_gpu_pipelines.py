"""The A/B pipelines kept behind switches stay bit-exact with the serial pack + search:
the SM-partitioned chunk pipeline (PF_SPLIT > 0, green contexts), the shared-SM chunk pipeline
with priority streams (PF_SPLIT = -1) and the 64-register lean pack (PF_PACK_LEAN = 4 / 8).
PF_PACK_LEAN is read once per process, so each configuration runs in its own interpreter."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import hashlib, json, os, sys
sys.path.insert(0, %(root)r)
import torch
import paper_1809_07858_b200 as pf
n, m = 3_000_000, 100
pitch = pf.device_pitch(m)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
t = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
p = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
est = torch.zeros(n, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
out = {}
for e in (5, 10):
    pf.generate_device(1, 1809078581 + 77 * e, e, t.data_ptr(), p.data_ptr(), pitch, n, m,
                       stream=s.cuda_stream)
    for split in ("0", "64", "-1"):
        os.environ["PF_SPLIT"] = split
        os.environ["PF_SPLIT_CHUNK"] = str(1 << 20)
        acc.zero_(); est.zero_()
        pf.shouji_filter_device_async(t.data_ptr(), p.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                      flag.data_ptr(), stream=s.cuda_stream,
                                      d_estimates=est.data_ptr())
        torch.cuda.synchronize()
        h = hashlib.sha256(acc.cpu().numpy().tobytes() + est.cpu().numpy().tobytes()).hexdigest()
        out[f"E{e}/split{split}"] = h
    assert int(flag.item()) == 0
print(json.dumps(out))
"""


def _digests(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_chunk_pipelines_and_lean_pack_match_serial():
    base = _digests({"PF_PACK_LEAN": "0"})
    for e in (5, 10):
        ref = base[f"E{e}/split0"]
        assert base[f"E{e}/split64"] == ref, "green-context split differs"
        assert base[f"E{e}/split-1"] == ref, "shared-SM pipeline differs"
    for lean in ("4", "8"):
        got = _digests({"PF_PACK_LEAN": lean})
        assert got == base, f"lean pack ({lean}-column items) differs"
