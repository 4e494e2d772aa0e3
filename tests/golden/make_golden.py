"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py

Every expected value in the fixtures comes from oracle/_ref/libprefilter_ref.so,
i.e. the reference's own shouji_filter / generate_pairs / banded_edit_distance
compiled from /root/reference/proj/src. The GPU box has no /root/reference, so
the parity tests there read these committed fixtures (plus the C restatement in
oracle/, itself pinned against these fixtures by tests/test_oracle.py).
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402


def rnd_dna(rng, n, m, with_n=False):
    alpha = np.frombuffer(b"ACGTN" if with_n else b"ACGT", np.uint8)
    return alpha[rng.integers(0, len(alpha), size=(n, m))]


def tandem(rng, n, m):
    out = np.zeros((n, m), np.uint8)
    alpha = np.frombuffer(b"ACGT", np.uint8)
    for i in range(n):
        p = int(rng.integers(1, 7))
        unit = alpha[rng.integers(0, 4, size=p)]
        out[i] = np.resize(unit, m)
    return out


def mutate(rng, t, rate, with_n=False):
    p = t.copy()
    alpha = np.frombuffer(b"ACGTN" if with_n else b"ACGT", np.uint8)
    mask = rng.random(t.shape) < rate
    p[mask] = alpha[rng.integers(0, len(alpha), size=int(mask.sum()))]
    # a few shifts (indels) per row
    for i in range(t.shape[0]):
        k = int(rng.integers(0, 3))
        for _ in range(k):
            pos = int(rng.integers(0, t.shape[1]))
            if rng.random() < 0.5:
                p[i, pos:] = np.concatenate([alpha[rng.integers(0, 4, size=1)], p[i, pos:-1]])
            else:
                p[i, pos:] = np.concatenate([p[i, pos + 1:], alpha[rng.integers(0, 4, size=1)]])
    return p


def main():
    ref = Reference()
    out = {}

    # 1. Config 0 (BASELINE.json configs[0]): generate_pairs({1809078580, 1M, 100, {0,10}}), E=5.
    t, p = ref.generate_pairs(1809078580, 1_000_000, 100, 0, 10)
    acc, est, _ = ref.shouji_batch(t, p, 5)
    out["config0"] = dict(
        text_head=t[:4096], pattern_head=p[:4096], accept_head=acc[:128], est_head=est[:4096],
        accept_sha256=np.frombuffer(hashlib.sha256(acc.tobytes()).digest(), np.uint8),
        text_sha256=np.frombuffer(hashlib.sha256(t.tobytes() + p.tobytes()).digest(), np.uint8),
        accepted=np.int64(sum(bin(int(w)).count("1") for w in acc)),
        est_sum=np.int64(est.astype(np.int64).sum()),
        est_hist=np.bincount(est, minlength=101).astype(np.int64),
    )

    # 2. Acceptance criterion 2 suite (acceptance_tests.cpp:93-128): seeded 100k sets.
    for m, e, seed in [(100, 2, 1102), (100, 5, 1105), (150, 7, 1157), (250, 15, 1265)]:
        t, p = ref.generate_pairs(seed, 100_000, m, 0, e)
        packed = ref.pack(t, p)
        acc, est, _ = packed.shouji(e)
        dist = packed.banded(e)
        packed.free()
        out[f"fr_m{m}_e{e}"] = dict(accept=acc, est=est.astype(np.uint16), similar=(dist >= 0),
                                    seed=np.int64(seed))

    # 3. Edge sets: lengths 1..300 incl. word boundaries, E up to 40 and >= m,
    #    widths 3..8, N-heavy, tandem repeats; bits recorded for every pair.
    rng = np.random.default_rng(20240601)
    cases = []
    lengths = [1, 2, 3, 4, 5, 12, 31, 32, 33, 63, 64, 65, 100, 129, 150, 250, 255, 256, 300]
    kinds = ("rand", "mut", "mutN", "tandem")
    for li, m in enumerate(lengths):
        for wi, width in enumerate((3, 4, 5, 8)):
            for kind in (kinds[(li + wi) % 4], kinds[(li + wi + 1) % 4]):
                es = sorted({0, 2, 5, min(m - 1, 16), min(m - 1, 25), m})
                for e in es:
                    if e < 0:
                        continue
                    n = 24 if width == 4 else 12
                    if kind == "rand":
                        t = rnd_dna(rng, n, m, True)
                        p = rnd_dna(rng, n, m, True)
                    elif kind == "tandem":
                        t = tandem(rng, n, m)
                        p = mutate(rng, t, 0.05)
                    else:
                        t = rnd_dna(rng, n, m, kind == "mutN")
                        p = mutate(rng, t, 0.08, kind == "mutN")
                    cases.append((m, width, e, t, p))
    recs = {}
    for idx, (m, width, e, t, p) in enumerate(cases):
        acc, est, bits = ref.shouji_batch(t, p, e, width, bits=True)
        recs[f"c{idx}"] = (m, width, e, t, p, acc, est, bits)
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"),
                        **{f"{k}_meta": np.array(v[:3], np.int64) for k, v in recs.items()},
                        **{f"{k}_text": v[3] for k, v in recs.items()},
                        **{f"{k}_pattern": v[4] for k, v in recs.items()},
                        **{f"{k}_accept": v[5] for k, v in recs.items()},
                        **{f"{k}_est": v[6] for k, v in recs.items()},
                        **{f"{k}_bits": v[7] for k, v in recs.items()})
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
