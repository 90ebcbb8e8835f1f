"""TEST INFRASTRUCTURE ONLY.  KVStore round and the key sharding rule.

The reference has one level-2 server holding whole keys (kvstore.py:368-404),
so the sharding rule is this build's own contract, restated
here independently of the product so tests can check it bit-exactly:

  * keys are laid out in init order, each padded to a multiple of 64
    elements;
  * walking the keys in push order (last key first), consecutive keys form
    a bucket until it holds >= bucket_bytes, and a key of >= bucket_bytes
    starts its own bucket;
  * a bucket of L elements is split among N owners at
    floor((r*L/N) / 32) * 32, the last owner ending at L.

A round (kvstore.py:190-241, 301-404) = two-level tree merge of every
worker's gradient, then the updater on the stored value; all replicas read
the same result.
"""

from __future__ import annotations

from typing import List, Tuple

import numpy as np

from . import numerics as nm


def arena_layout(numels: List[int], bucket_bytes: int):
    """Offsets in init order; buckets packed from the LAST key backwards
    (push order) and listed in arena order; bucket index of every key."""
    offsets = []
    pos = 0
    for n in numels:
        offsets.append(pos)
        pos += ((n + 63) // 64) * 64
    rev = []
    end, start = pos, pos
    for n, off in zip(reversed(numels), reversed(offsets)):
        if end != start and (4 * (end - start) >= bucket_bytes or 4 * n >= bucket_bytes):
            rev.append((start, end))
            end = start
        start = off
    if end != start or not rev:
        rev.append((start, end))
    buckets = list(reversed(rev))
    owner_bucket = [next(b for b, (lo, hi) in enumerate(buckets) if lo <= off < hi)
                    if any(lo <= off < hi for lo, hi in buckets) else len(buckets) - 1
                    for off in offsets]
    return offsets, buckets, owner_bucket


def owner_shards(length: int, owners: int) -> List[Tuple[int, int]]:
    cuts = [((r * length) // owners) // 32 * 32 for r in range(owners)] + [length]
    return list(zip(cuts[:-1], cuts[1:]))


def sgd_round(weights: np.ndarray, velocity: np.ndarray, grads: List[np.ndarray], eta: float,
              momentum: float, weight_decay: float, machines: int = 1):
    """One sequential-mode round with make_sgd_updater(cfg, scale=M*W)."""
    total = nm.kv_merge(grads, machines)
    return nm.kv_updater(weights, total, velocity, eta, momentum, weight_decay, len(grads))


def add_round(weights: np.ndarray, grads: List[np.ndarray], machines: int = 1):
    """One round with the default add updater (kvstore.py:47-49)."""
    return (weights + nm.kv_merge(grads, machines)).astype(np.float32)
