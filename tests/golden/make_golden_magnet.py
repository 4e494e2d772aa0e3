"""Generate tests/golden/magnet.npz from the UNMODIFIED reference library.

Run in the build container (/root/reference present, oracle/_ref built):
    python tests/golden/make_golden_magnet.py

Expected values come from oracle/_ref/libprefilter_ref.so: magnet_filter
(proj/src/magnet.cpp:77-87) through run_filter for the batch sets, and per pair
for the bit vectors (bitvector::to_string of the decision's bits).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402
from make_golden import mutate, rnd_dna, tandem  # noqa: E402


def main():
    ref = Reference()
    rng = np.random.default_rng(1809_07858)
    out = {}
    # 1. per-pair bits on edge lengths / thresholds / content kinds
    k = 0
    for m in (1, 2, 5, 12, 31, 32, 33, 64, 65, 100, 150, 250, 300):
        for kind in ("rand", "mut", "mutN", "tandem"):
            for e in sorted({0, 1, 3, min(m - 1, 5), min(m - 1, 12), min(m - 1, 25), m}):
                n = 8
                if kind == "rand":
                    t, p = rnd_dna(rng, n, m, True), rnd_dna(rng, n, m, True)
                elif kind == "tandem":
                    t = tandem(rng, n, m)
                    p = mutate(rng, t, 0.05)
                else:
                    t = rnd_dna(rng, n, m, kind == "mutN")
                    p = mutate(rng, t, 0.06, kind == "mutN")
                t, p = np.ascontiguousarray(t), np.ascontiguousarray(p)
                bits = np.zeros((n, (m + 63) // 64), np.uint64)
                acc = np.zeros((n + 31) // 32, np.uint32)
                est = np.zeros(n, np.uint32)
                for i in range(n):
                    a, s, b = ref.magnet_one(p[i].tobytes().decode(), t[i].tobytes().decode(), e)
                    if a:
                        acc[i // 32] |= np.uint32(1 << (i % 32))
                    est[i] = s
                    for j, ch in enumerate(b):
                        if ch == "1":
                            bits[i, j // 64] |= np.uint64(1 << (j % 64))
                out[f"c{k}_meta"] = np.array([m, e], np.int64)
                out[f"c{k}_text"], out[f"c{k}_pattern"] = t, p
                out[f"c{k}_accept"], out[f"c{k}_est"], out[f"c{k}_bits"] = acc, est, bits
                k += 1
    # 2. batch decisions on generate_pairs sets (run_filter(magnet), parallel_for_pairs)
    for m, lo, hi, e, seed in [(100, 0, 10, 5, 4100), (150, 0, 15, 7, 4150), (250, 0, 25, 15, 4250)]:
        t, p = ref.generate_pairs(seed, 2000, m, lo, hi)
        acc, est = ref.magnet_batch(t, p, e)
        out[f"set_m{m}_e{e}_text"], out[f"set_m{m}_e{e}_pattern"] = t, p
        out[f"set_m{m}_e{e}_accept"], out[f"set_m{m}_e{e}_est"] = acc, est.astype(np.uint16)
    np.savez_compressed(os.path.join(HERE, "magnet.npz"), **out)


if __name__ == "__main__":
    main()
