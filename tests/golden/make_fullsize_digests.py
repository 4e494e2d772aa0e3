#!/usr/bin/env python
"""Full-size parity digests for BASELINE.json configs 1-4 (test fixture generator).

For every (config, E) set below — the full BASELINE sizes, 30M pairs (100M for
config 4) — the CPU oracle computes every pair's Shouji estimate
(``so_config_estimates``: the generator mirror of csrc/datagen.cu feeding the
vectorisable restatement of proj/src/shouji.cpp:41-58, both in
oracle/config_oracle.c), and this script records

* ``accept_sha256``   — sha256 of the accept bitmap as the C ABI writes it
  (LSB-first u32 words, little endian, ceil(n/32) words, tail bits zero);
  accept = estimate <= E (filter_decision.hpp:12-16);
* ``estimate_sha256`` — sha256 of the estimates as u32 little endian, one per pair;
* ``accepted`` and ``estimate_hist`` (readable summaries of the same data);
* ``data_prefix_sha256`` — sha256 of the set's first 4096 pairs' bytes (the
  generator mirror's output; text rows then pattern rows);
* ``estimate_prefix_sha256`` — sha256 of the first 65536 pairs' estimates, which
  the CPU suite recomputes with the reference library itself
  (tests/test_oracle_configs.py).

tests/test_gpu_fullsize_digests.py regenerates each set on the device and
compares the GPU's own bitmap and estimates against these digests.

Cross-checks by the unmodified reference library (oracle/_ref, the reference
compiled from its sources): ``--ref-prefix K`` recomputes the first K pairs of
every set with the reference and requires identical estimates (recorded as
``ref_checked_pairs``); ``--ref-full`` recomputes whole sets with the reference
and records ``ref_estimate_sha256`` (hours of CPU; run in the background).

Usage:  python tests/golden/make_fullsize_digests.py [--threads T] [--only 1,3]
        python tests/golden/make_fullsize_digests.py --ref-prefix 1000000
        python tests/golden/make_fullsize_digests.py --ref-full --only 1
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

OUT = os.path.join(HERE, "fullsize_digests.json")
CHUNK = 1 << 21  # pairs per oracle call (a multiple of 32: bitmap words never straddle chunks)
SEED0 = 1809078581  # bench.py's configs[1] seed at rank 0 is SEED0 + 1000 * E


def seed_of(config: int, e: int) -> int:
    return SEED0 + 100_000 * (config - 1) + 1000 * e


def all_sets():
    """BASELINE.json configs 1-4 with their E sweeps, at full size."""
    sets = []
    for e in range(0, 11):
        sets.append((1, 100, e, 30_000_000))
    for e in (0, 3, 7, 15):
        sets.append((2, 150, e, 30_000_000))
    for e in range(0, 26):
        sets.append((3, 250, e, 30_000_000))
    sets.append((4, 250, 25, 100_000_000))
    return [{"config": c, "m": m, "E": e, "seed": seed_of(c, e), "n": n} for c, m, e, n in sets]


def bitmap_words(est: np.ndarray, e: int) -> np.ndarray:
    acc = (est <= e).astype(np.uint8)
    pad = (-acc.size) % 32
    if pad:
        acc = np.concatenate([acc, np.zeros(pad, np.uint8)])
    return np.packbits(acc, bitorder="little").view("<u4")


class Digest:
    def __init__(self, e: int, m: int):
        self.e, self.m = e, m
        self.h_acc = hashlib.sha256()
        self.h_est = hashlib.sha256()
        self.hist = np.zeros(m + 1, np.int64)
        self.accepted = 0

    def update(self, est: np.ndarray):
        est = np.ascontiguousarray(est, dtype="<u4")
        self.h_est.update(est.tobytes())
        self.h_acc.update(bitmap_words(est, self.e).tobytes())
        self.hist += np.bincount(est, minlength=self.m + 1)[: self.m + 1]
        self.accepted += int((est <= self.e).sum())

    def result(self):
        nz = np.nonzero(self.hist)[0]
        return {"accept_sha256": self.h_acc.hexdigest(), "estimate_sha256": self.h_est.hexdigest(),
                "accepted": self.accepted,
                "estimate_hist": {int(k): int(self.hist[k]) for k in nz}}


def run_oracle(s, o, threads):
    d = Digest(s["E"], s["m"])
    for lo in range(0, s["n"], CHUNK):
        k = min(CHUNK, s["n"] - lo)
        d.update(o.config_estimates(s["config"], s["seed"], s["E"], s["m"], s["E"], lo, k,
                                    threads=threads))
    return d.result()


def run_reference(s, o, ref, threads, limit=None):
    """The reference library over the set's first `limit` pairs (all when None)."""
    n = s["n"] if limit is None else min(limit, s["n"])
    d = Digest(s["E"], s["m"])
    for lo in range(0, n, CHUNK):
        k = min(CHUNK, n - lo)
        t, p = o.gen_config(s["config"], s["seed"], s["E"], s["m"], lo, k)
        _, est, _ = ref.shouji_batch(t, p, s["E"], threads=threads)
        mine = o.config_estimates(s["config"], s["seed"], s["E"], s["m"], s["E"], lo, k,
                                  threads=threads)
        bad = np.nonzero(est != mine)[0]
        if bad.size:
            raise SystemExit(f"oracle != reference at config {s['config']} E={s['E']} "
                             f"pair {lo + int(bad[0])}: {mine[bad[0]]} vs {est[bad[0]]}")
        d.update(est)
    return n, d.result()


PREFIX_PAIRS = 4096
ESTIMATE_PREFIX_PAIRS = 1 << 16


def data_prefix(s, o, k=PREFIX_PAIRS):
    """sha256 of the set's first k pairs (text rows then pattern rows, m bytes each)."""
    t, p = o.gen_config(s["config"], s["seed"], s["E"], s["m"], 0, k)
    return hashlib.sha256(t.tobytes() + p.tobytes()).hexdigest()


def estimate_prefix(s, o, k=ESTIMATE_PREFIX_PAIRS, threads=None):
    """sha256 of the estimates (u32 LE) of the set's first k pairs."""
    est = o.config_estimates(s["config"], s["seed"], s["E"], s["m"], s["E"], 0, k, threads=threads)
    return hashlib.sha256(est.astype("<u4").tobytes()).hexdigest()


def key(s):
    return (s["config"], s["E"], s["seed"], s["n"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--only", default="", help="comma-separated config numbers")
    ap.add_argument("--e-list", default="", help="comma-separated thresholds (default: all)")
    ap.add_argument("--ref-prefix", type=int, default=0)
    ap.add_argument("--ref-full", action="store_true")
    ap.add_argument("--data-prefix-only", action="store_true",
                    help="only (re)compute data_prefix_sha256 of every set")
    args = ap.parse_args()
    from oracle.oracle import Oracle, Reference
    o = Oracle()
    only = {int(x) for x in args.only.split(",") if x}
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    have = {key(s): s for s in doc.get("sets", [])}
    for s in all_sets():
        if only and s["config"] not in only:
            continue
        if args.e_list and s["E"] not in {int(x) for x in args.e_list.split(",")}:
            continue
        rec = dict(have.get(key(s), s))
        t0 = time.time()
        rec["data_prefix_sha256"] = data_prefix(s, o)
        rec["estimate_prefix_sha256"] = estimate_prefix(s, o, threads=args.threads)
        if args.data_prefix_only:
            pass
        elif args.ref_prefix or args.ref_full:
            ref = Reference()
            n, r = run_reference(s, o, ref, args.threads, None if args.ref_full else args.ref_prefix)
            if "estimate_sha256" in rec and n == s["n"]:
                assert r["estimate_sha256"] == rec["estimate_sha256"], s
            if n == s["n"]:
                rec["ref_estimate_sha256"] = r["estimate_sha256"]
            rec["ref_checked_pairs"] = max(n, rec.get("ref_checked_pairs", 0))
        else:
            rec.update(run_oracle(s, o, args.threads))
        print(f"config {s['config']} m={s['m']} E={s['E']:2d} n={s['n']}: "
              f"accepted {rec.get('accepted')}  ref_checked {rec.get('ref_checked_pairs', 0)}  "
              f"({time.time() - t0:.1f} s)", flush=True)
        have[key(s)] = rec
        doc = {
            "what": "Full-size parity digests of BASELINE.json configs 1-4 (tests/golden/"
                    "make_fullsize_digests.py). Data: csrc/datagen.cu, mirrored byte for byte "
                    "by oracle/config_oracle.c (so_gen_config). Estimates: so_config_estimates "
                    "(oracle/config_oracle.c), a restatement of proj/src/shouji.cpp:41-58 pinned "
                    "to the reference library; ref_checked_pairs = leading pairs of the set "
                    "recomputed by the unmodified reference library (oracle/_ref) with identical "
                    "estimates; ref_estimate_sha256 = the reference library's own digest of the "
                    "whole set.",
            "chunk_pairs": CHUNK,
            "sets": sorted(have.values(), key=lambda r: (r["config"], r["E"])),
        }
        with open(OUT + ".tmp", "w") as f:
            json.dump(doc, f, indent=1)
        os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main()
