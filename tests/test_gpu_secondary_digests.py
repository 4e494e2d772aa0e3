"""The path's neighbours at full size against the reference library itself:
MAGNET (csrc/magnet.cu) and the banded edit distance (csrc/edit_distance.cu) over
30M-pair BASELINE config sets, hashed against digests the unmodified reference
library computed for every pair (tests/golden/secondary_digests.json, made by
tests/golden/make_secondary_digests.py): accept bitmap + estimates for MAGNET
(proj/src/magnet.cpp:77-87), the distance within the band or -1 for
banded_edit_distance (proj/src/edit_distance.cpp:26-70)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _sets():
    with open(os.path.join(HERE, "golden", "secondary_digests.json")) as f:
        return json.load(f)["sets"]


def _ids():
    try:
        return [f"{s['algo']}-c{s['config']}-e{s['E']}" for s in _sets()]
    except FileNotFoundError:
        return []


@pytest.mark.parametrize("idx", range(len(_ids())), ids=_ids())
def test_secondary_set_matches_reference_digest(gpu, idx):
    import torch
    s = _sets()[idx]
    n, m, e = s["n"], s["m"], s["E"]
    pitch = gpu.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    gpu.generate_device(s["config"], s["seed"], e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
    torch.cuda.synchronize()
    if s["algo"] == "magnet":
        acc = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        est = torch.zeros(n, dtype=torch.int32, device="cuda")
        gpu.magnet_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                 d_estimates=est.data_ptr())
        torch.cuda.synchronize()
        a = acc.cpu().numpy().view(np.uint32)
        v = est.cpu().numpy().view(np.uint32)
        assert int((v <= e).sum()) == s["accepted"]
        assert hashlib.sha256(a.tobytes()).hexdigest() == s["accept_sha256"]
        assert hashlib.sha256(v.tobytes()).hexdigest() == s["estimate_sha256"]
    else:
        ht = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
        hp = torch.empty((n, m), dtype=torch.uint8, pin_memory=True)
        ht.copy_(tt[:, :m])
        hp.copy_(pt[:, :m])
        del tt, pt
        d = gpu.banded_edit_distance_batch(ht.numpy(), hp.numpy(), e)
        assert int((d >= 0).sum()) == s["within"]
        assert hashlib.sha256(d.astype("<i4").tobytes()).hexdigest() == s["distance_sha256"]
