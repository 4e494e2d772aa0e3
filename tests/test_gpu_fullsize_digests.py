"""Bit-exact parity at the full BASELINE sizes: every (config, E) set of
BASELINE.json configs 1-4 — 30M pairs per set (100M for config 4), config 1 at
E = 0..10, config 2 at E in {0, 3, 7, 15}, config 3 at E = 0..25, config 4 at
E = 25 — is generated on the device and filtered by the CUDA path through the
C ABI (pf_shouji_filter_device); the GPU's accept bitmap and per-pair estimates
must hash to the digests the CPU oracle computed for every pair of the same set
(tests/golden/fullsize_digests.json, made by tests/golden/make_fullsize_digests.py;
the oracle restates proj/src/shouji.cpp:41-58 and is pinned to the reference
library, which also recomputed the leading pairs of every set).

The sets' bytes come from csrc/datagen.cu; the oracle regenerated them with its
byte-identical CPU mirror (oracle/config_oracle.c), which is checked here
against the device bytes on sampled rows of every set (first, last and random
pair indices) and on a 4096-pair prefix.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = os.path.join(HERE, "golden", "fullsize_digests.json")


def _sets():
    with open(DIGESTS) as f:
        return json.load(f)["sets"]


def _by_config():
    out = {}
    for s in _sets():
        out.setdefault(s["config"], []).append(s)
    return out


EXPECTED_E = {1: list(range(11)), 2: [0, 3, 7, 15], 3: list(range(26)), 4: [25]}
EXPECTED_N = {1: 30_000_000, 2: 30_000_000, 3: 30_000_000, 4: 100_000_000}


def test_digest_file_covers_every_baseline_set():
    by = _by_config()
    for c, es in EXPECTED_E.items():
        got = sorted(s["E"] for s in by.get(c, []) if "estimate_sha256" in s)
        assert got == es, f"config {c}: digests for E={got}, expected {es}"
        assert all(s["n"] == EXPECTED_N[c] for s in by[c])


def _check_rows(oracle, s, tt, pt, m, rng):
    n = s["n"]
    rows = np.unique(np.concatenate([[0, 1, 31, 32, n // 2, n - 2, n - 1],
                                     rng.integers(0, n, size=57)])).astype(np.int64)
    idx = __import__("torch").as_tensor(rows, device=tt.device)
    dt = tt.index_select(0, idx)[:, :m].cpu().numpy()
    dp = pt.index_select(0, idx)[:, :m].cpu().numpy()
    ht, hp = oracle.gen_config_rows(s["config"], s["seed"], s["E"], m, rows)
    assert (dt == ht).all(), f"config {s['config']} E={s['E']}: device text rows != CPU mirror"
    assert (dp == hp).all(), f"config {s['config']} E={s['E']}: device pattern rows != CPU mirror"
    k = 4096
    ht, hp = oracle.gen_config(s["config"], s["seed"], s["E"], m, 0, k)
    assert (tt[:k, :m].cpu().numpy() == ht).all() and (pt[:k, :m].cpu().numpy() == hp).all()


@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_fullsize_sets_match_oracle_digests(gpu, oracle, config):
    import torch
    sets = sorted(_by_config()[config], key=lambda s: s["E"])
    assert [s["E"] for s in sets] == EXPECTED_E[config]
    n = max(s["n"] for s in sets)
    m = sets[0]["m"]
    pitch = gpu.device_pitch(m)
    tt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    pt = torch.empty((n, pitch), dtype=torch.uint8, device="cuda")
    acc = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    est = torch.empty(n, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(config)
    failures = []
    for s in sets:
        assert s["m"] == m and s["n"] == n
        e = s["E"]
        gpu.generate_device(config, s["seed"], e, tt.data_ptr(), pt.data_ptr(), pitch, n, m)
        acc.fill_(-1)
        est.fill_(-1)
        gpu.shouji_filter_device(tt.data_ptr(), pt.data_ptr(), pitch, n, m, e, acc.data_ptr(),
                                 d_estimates=est.data_ptr())
        torch.cuda.synchronize()
        _check_rows(oracle, s, tt, pt, m, rng)
        a = acc.cpu().numpy().view(np.uint32)
        v = est.cpu().numpy().view(np.uint32)
        ha = hashlib.sha256(a.tobytes()).hexdigest()
        hv = hashlib.sha256(v.tobytes()).hexdigest()
        if ha != s["accept_sha256"] or hv != s["estimate_sha256"]:
            hist = np.bincount(v, minlength=m + 1)
            want = np.zeros(m + 1, np.int64)
            for k, c in s["estimate_hist"].items():
                want[int(k)] = c
            failures.append(f"E={e}: accepted {int((v <= e).sum())} vs {s['accepted']}, "
                            f"histogram diff at {np.nonzero(hist != want)[0][:8].tolist()}")
    assert not failures, f"config {config}: " + "; ".join(failures)
