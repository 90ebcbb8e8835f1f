"""Input side of the training step: record files and batch order.

Reads the reference's example record files (recordio.py:1-198: magic
0x4D585245, [len u32][crc32 u32][payload], ``.idx`` of u64 offsets, record 0
= feature dimension, then label u32 + D float32 per example) and reproduces
its batch order (dataiter.py:28-46: splitmix64-driven Fisher-Yates, partial
batch dropped, seed+1 per epoch), so a device run sees exactly the
reference's batches.

``BatchIterator`` is the reference's prefetching iterator (dataiter.py:49-155:
bounded queue, producer thread, partial batch dropped, ``reset`` advances
the seed).  B200 layout: the file is decoded once into one contiguous
[N, D] float32 array, a batch is a single vectorised row gather, and the
producer writes each batch into a ring of PINNED host buffers (depth + 3),
so handing a batch to the device is one DMA with no staging copy
(``DataParallelStep.stage`` / ``tensor.load_host`` take pinned tensors
directly).
"""

from __future__ import annotations

import queue
import struct
import threading
import zlib
from typing import Iterator, List, Optional, Tuple

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


class BatchIterator:
    """Yields (features [B, D] float32, labels [B] float32) batches of a
    record file (or of in-memory (features, labels) arrays) in the
    reference's order (dataiter.py:49-155).

    ``prefetch`` > 0: a producer thread assembles batches ahead into a ring
    of ``prefetch + 3`` pinned buffer pairs, handed over through a bounded
    queue of depth ``prefetch``; a yielded batch stays valid until two
    further batches have been taken (enough for an asynchronous H2D copy
    started when it was taken and waited on one step later; copy it to keep
    it longer).  ``prefetch`` = 0 assembles synchronously.  Batch contents
    depend only on (data, batch size, seed), never on prefetch depth."""

    def __init__(self, source, batch_size: int, seed: int = 0, prefetch: int = 2,
                 shuffle: bool = True, affine: Optional[Tuple[np.ndarray, np.ndarray]] = None,
                 engine=None, pinned: bool = True):
        if batch_size < 1:
            raise ArgumentError("batch size must be >= 1")
        if prefetch < 0:
            raise ArgumentError("prefetch depth must be >= 0")
        if isinstance(source, str):
            self.path = source
            feats, labels = read_examples(source)
        else:
            self.path = None
            feats, labels = (np.ascontiguousarray(a, np.float32) for a in source)
        self._feats, self._labels = feats, labels
        self.batch_size, self.seed, self.prefetch = batch_size, seed, prefetch
        self.shuffle, self.engine = shuffle, engine
        self.affine = None if affine is None else tuple(np.asarray(a, np.float32) for a in affine)
        self.num_examples, self.dim = feats.shape
        self.batches_per_epoch = self.num_examples // batch_size
        self._ring = [self._buffers(pinned) for _ in range(prefetch + 3 if prefetch else 1)]
        self._start_epoch()

    def _buffers(self, pinned: bool):
        if pinned:
            try:
                import torch
                if torch.cuda.is_available():
                    x = torch.empty((self.batch_size, self.dim), dtype=torch.float32,
                                    pin_memory=True)
                    y = torch.empty((self.batch_size,), dtype=torch.float32, pin_memory=True)
                    return x.numpy(), y.numpy(), x, y
            except Exception:  # noqa: BLE001 - no pinned memory: plain host arrays
                pass
        x = np.empty((self.batch_size, self.dim), np.float32)
        y = np.empty((self.batch_size,), np.float32)
        return x, y, None, None

    # ------------------------------------------------------------ epochs

    def _start_epoch(self) -> None:
        n = self.num_examples
        order = shuffled_order(n, self.seed) if self.shuffle else range(n)
        self._order = np.fromiter(order, np.int64, count=n)
        self._served = 0
        self._exhausted = False
        self._queue: Optional[queue.Queue] = None
        self._thread: Optional[threading.Thread] = None
        self._error: Optional[BaseException] = None
        if self.prefetch > 0:
            self._queue = queue.Queue(maxsize=self.prefetch)
            self._thread = threading.Thread(target=self._produce, daemon=True,
                                            name="mgx-prefetch")
            self._thread.start()

    def _assemble(self, b: int, slot: int) -> Tuple[np.ndarray, np.ndarray]:
        x, y, _tx, _ty = self._ring[slot]
        rows = self._order[b * self.batch_size:(b + 1) * self.batch_size]
        np.take(self._feats, rows, axis=0, out=x)
        np.take(self._labels, rows, out=y)
        if self.affine is not None:
            shift, scale = self.affine
            np.multiply(x + shift, scale, out=x)
        return x, y

    def _produce(self) -> None:
        try:
            for b in range(self.batches_per_epoch):
                self._queue.put((b, self._assemble(b, b % len(self._ring))))
        except BaseException as exc:  # noqa: BLE001 - re-raised in the consumer
            self._error = exc
        self._queue.put(None)

    def __iter__(self):
        return self

    def __next__(self) -> Tuple[np.ndarray, np.ndarray]:
        if self._queue is not None:
            item = self._queue.get()
            if item is None:
                self._exhausted = True
                if self._error is not None:
                    raise self._error
                raise StopIteration
            return item[1]
        if self._served >= self.batches_per_epoch:
            raise StopIteration
        batch = self._assemble(self._served, 0)
        self._served += 1
        return batch

    def pinned(self, batch: Tuple[np.ndarray, np.ndarray]):
        """The pinned torch tensors behind a yielded batch (for a direct H2D
        copy), or None when the buffers are not pinned."""
        for x, y, tx, ty in self._ring:
            if x is batch[0]:
                return (tx, ty) if tx is not None else None
        return None

    def next_batch(self):
        """Next batch as device tensors; raises StopIteration at epoch end."""
        from . import tensor as tmod
        feats, labels = next(self)
        pin = self.pinned((feats, labels))
        x = tmod.Tensor(feats.shape, engine=self.engine)
        y = tmod.Tensor(labels.shape, engine=self.engine)
        tmod.load_host(x, pin[0] if pin else feats)
        tmod.load_host(y, pin[1] if pin else labels)
        return x, y

    def _drain(self) -> None:
        if self._thread is None:
            return
        if not self._exhausted:
            while self._queue.get() is not None:
                pass
        self._thread.join()
        self._thread = None

    def reset(self) -> None:
        """Begin the next epoch; the shuffle seed advances by one."""
        self._drain()
        self.seed += 1
        self._start_epoch()

    def close(self) -> None:
        self._drain()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
