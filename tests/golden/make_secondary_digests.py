#!/usr/bin/env python
"""Full-size digests of the path's SURVEY §8(f) neighbours, computed by the
UNMODIFIED reference library (oracle/_ref) itself on BASELINE config sets:

* MAGNET (magnet_filter, proj/src/magnet.cpp:77-87): accept bitmap (C ABI word
  layout) and u32 estimates, per set;
* the exact banded edit distance (banded_edit_distance,
  proj/src/edit_distance.cpp:26-70): i32 distance per pair, -1 when beyond e
  (the C ABI's pf_banded_edit_distance_batch convention).

Data: the same config generators as make_fullsize_digests.py (csrc/datagen.cu,
regenerated on the CPU by its mirror oracle/config_oracle.c), 30M pairs per set.
tests/test_gpu_secondary_digests.py compares the CUDA kernels against these.

python tests/golden/make_secondary_digests.py [--threads T]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_fullsize_digests import bitmap_words, seed_of  # noqa: E402

OUT = os.path.join(HERE, "secondary_digests.json")
CHUNK = 1 << 21
N = 30_000_000
SETS = [("magnet", 1, 100, 2), ("magnet", 1, 100, 5), ("magnet", 1, 100, 10),
        ("magnet", 2, 150, 7), ("magnet", 3, 250, 15),
        ("edit_distance", 1, 100, 5), ("edit_distance", 2, 150, 7),
        ("edit_distance", 3, 250, 15)]


def run(algo, config, m, e, threads):
    from oracle.oracle import Oracle, Reference
    o, ref = Oracle(), Reference()
    seed = seed_of(config, e)
    h1, h2 = hashlib.sha256(), hashlib.sha256()
    summary = 0
    for lo in range(0, N, CHUNK):
        k = min(CHUNK, N - lo)
        t, p = o.gen_config(config, seed, e, m, lo, k)
        pk = ref.pack(t, p)
        try:
            if algo == "magnet":
                acc, est = pk.magnet(e, threads=threads)
                est = est.astype("<u4")
                h1.update(bitmap_words(est, e).tobytes())
                h2.update(est.tobytes())
                summary += int((est <= e).sum())
            else:
                d = pk.banded(e, threads=threads).astype("<i4")
                h1.update(d.tobytes())
                summary += int((d >= 0).sum())
        finally:
            pk.free()
    rec = {"algo": algo, "config": config, "m": m, "E": e, "seed": seed, "n": N}
    if algo == "magnet":
        rec.update(accept_sha256=h1.hexdigest(), estimate_sha256=h2.hexdigest(), accepted=summary)
    else:
        rec.update(distance_sha256=h1.hexdigest(), within=summary)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out = []
    for algo, config, m, e in SETS:
        t0 = time.time()
        out.append(run(algo, config, m, e, args.threads))
        print(algo, config, m, e, f"{time.time() - t0:.0f} s", flush=True)
        doc = {"what": "Reference-library digests of MAGNET and the banded edit distance on "
                       "BASELINE config sets (tests/golden/make_secondary_digests.py)",
               "sets": out}
        with open(OUT + ".tmp", "w") as f:
            json.dump(doc, f, indent=1)
        os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main()
