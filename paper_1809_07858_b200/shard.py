"""Multi-process (one rank per GPU) sharding of a pair batch.

Pairs are independent, so a batch is split into contiguous, 32-pair-aligned
ranges — the static chunking of the reference's parallel_for_pairs
(proj/src/evaluate.cpp:36-37, begin = n*t/T) rounded to whole bitmap words so no
accept word straddles two ranks. Each rank filters its range on its own GPU; the
only communication is the final gather of accept-bitmap words (no collective on
the data path). The same split is used by pf_ctx_create contexts over several
devices inside one process (csrc/capi.cpp).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, parts: int) -> list[int]:
    """parts+1 boundaries; shard t is [b[t], b[t+1]), every boundary a multiple of 32 (or n)."""
    groups = (n + 31) // 32
    return [min(n, (groups * t // parts) * 32) for t in range(parts + 1)]


def gather_bitmaps(local: np.ndarray, bounds: list[int], rank: int, world: int, group=None) -> np.ndarray:
    """All-gather per-rank accept-bitmap words into the full bitmap (host side).

    ``local`` holds ceil((b[r+1]-b[r])/32) words for this rank's shard. Works with
    any torch.distributed backend (gloo on CPU, nccl on GPU via a CPU copy)."""
    import torch
    import torch.distributed as dist

    words = [(bounds[t + 1] - bounds[t] + 31) // 32 for t in range(world)]
    width = max(words) if words else 0
    buf = torch.zeros(width, dtype=torch.int64)
    buf[: words[rank]] = torch.from_numpy(local.astype(np.int64))
    out = [torch.zeros(width, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    full = np.concatenate([out[t][: words[t]].numpy() for t in range(world)]).astype(np.uint32)
    return full


def filter_sharded(text, pattern, e, rank, world, filter_fn, width=4, group=None):
    """Filter this rank's shard with ``filter_fn(text, pattern, e, width) -> bitmap``
    and return the full accept bitmap on every rank."""
    n = text.shape[0]
    b = shard_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    local = filter_fn(text[lo:hi], pattern[lo:hi], e, width) if hi > lo else np.zeros(0, np.uint32)
    return gather_bitmaps(np.asarray(local, np.uint32), b, rank, world, group)
