"""Input side of the training step: record files and batch order.

Reads the reference's example record files (recordio.py:1-198: magic
0x4D585245, [len u32][crc32 u32][payload], ``.idx`` of u64 offsets, record 0
= feature dimension, then label u32 + D float32 per example) and reproduces
its batch order (dataiter.py:28-46: splitmix64-driven Fisher-Yates, partial
batch dropped, seed+1 per epoch), so a device run sees exactly the
reference's batches.  Batches are assembled on the host and handed to the
step as pinned tensors (one H2D copy per step).
"""

from __future__ import annotations

import struct
import zlib
from typing import Iterator, List, Tuple

import numpy as np

from .errors import ArgumentError, CorruptRecordError, RecordParseError

MAGIC = 0x4D585245
VERSION = 1
_M64 = (1 << 64) - 1


def splitmix64(seed: int) -> Iterator[int]:
    state = seed & _M64
    while True:
        state = (state + 0x9E3779B97F4A7C15) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        yield z ^ (z >> 31)


def shuffled_order(n: int, seed: int) -> List[int]:
    """Fisher-Yates permutation of range(n) (dataiter.py:39-46)."""
    order = list(range(n))
    rng = splitmix64(seed)
    for i in range(n - 1, 0, -1):
        j = next(rng) % (i + 1)
        order[i], order[j] = order[j], order[i]
    return order


def read_examples(path: str) -> Tuple[np.ndarray, np.ndarray]:
    """All examples of a record file as (features [N, D] f32, labels [N] f32)."""
    raw = open(path, "rb").read()
    if len(raw) < 8:
        raise RecordParseError(f"{path}: truncated file header")
    magic, version = struct.unpack_from("<II", raw, 0)
    if magic != MAGIC:
        raise RecordParseError(f"{path}: bad magic {magic:#x}")
    if version != VERSION:
        raise RecordParseError(f"{path}: unsupported version {version}")
    try:
        idx = open(path + ".idx", "rb").read()
    except OSError as exc:
        raise RecordParseError(f"{path}: missing index file") from exc
    if len(idx) % 8:
        raise RecordParseError(f"{path}: index size not a multiple of 8")
    offsets = struct.unpack(f"<{len(idx) // 8}Q", idx)

    def record(i: int) -> bytes:
        off = offsets[i]
        if off + 8 > len(raw):
            raise RecordParseError(f"{path}: truncated record {i} header")
        length, crc = struct.unpack_from("<II", raw, off)
        payload = raw[off + 8: off + 8 + length]
        if len(payload) < length:
            raise RecordParseError(f"{path}: truncated record {i} payload")
        if zlib.crc32(payload) != crc:
            raise CorruptRecordError(f"{path}: crc mismatch at record {i}")
        return payload

    if not offsets:
        raise RecordParseError(f"{path}: missing metadata record")
    (dim,) = struct.unpack("<I", record(0))
    n = len(offsets) - 1
    feats = np.empty((n, dim), np.float32)
    labels = np.empty((n,), np.float32)
    for i in range(n):
        p = record(i + 1)
        if len(p) != 4 + 4 * dim:
            raise RecordParseError(f"example record {i}: {len(p)} bytes, expected {4 + 4 * dim}")
        labels[i] = struct.unpack_from("<I", p)[0]
        feats[i] = np.frombuffer(p, dtype="<f4", offset=4)
    return feats, labels


class BatchOrder:
    """Epoch-by-epoch batches of (features, labels) in the reference order
    (BatchIterator, dataiter.py:49-155, without the prefetch thread)."""

    def __init__(self, feats: np.ndarray, labels: np.ndarray, batch: int, seed: int = 0,
                 shuffle: bool = True):
        if batch < 1:
            raise ArgumentError("batch size must be >= 1")
        self.feats, self.labels = feats, labels
        self.batch, self.seed, self.shuffle = batch, seed, shuffle
        self.batches_per_epoch = len(feats) // batch

    def epoch(self, e: int) -> Iterator[Tuple[np.ndarray, np.ndarray]]:
        n = len(self.feats)
        order = shuffled_order(n, self.seed + e) if self.shuffle else list(range(n))
        idx = np.asarray(order, np.int64)
        for b in range(self.batches_per_epoch):
            rows = idx[b * self.batch:(b + 1) * self.batch]
            yield self.feats[rows], self.labels[rows]
