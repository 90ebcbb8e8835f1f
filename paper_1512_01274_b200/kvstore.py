"""Device key-value store for data-parallel training.

Drop-in for the reference KVStore (kvstore.py:84-409): ``KVStore(machines,
workers, mode, etype, engine, tcp)`` with ``init / set_updater / push /
pull / round_barrier / quiesce / stats / close``.  Instead of level-1 and
level-2 server threads exchanging copies through queues, one fused kernel
per flush (csrc/kv.cu) does, for every pushed key:

    level-1 tree over each machine's W workers (ascending worker id)
    -> level-2 tree over the M machine aggregates (ascending machine id)
    -> updater (fused momentum SGD, add, or a plugin callable)
    -> the new value stored into every worker's replica (the pull source)

Bit-exactness with the reference's per-element float sequence is kept for
every sharding, so the placement rule below is a free choice:

* keys are laid out in init order in a flat arena, each key starting on a
  256-byte boundary and padded to 64 elements (padding stays zero);
* consecutive keys are grouped, in push order (the reverse of init order),
  into buckets of at least ``bucket_bytes`` (4 MB default; a key of that
  size or more is a bucket of its own);
* each bucket range of L elements is split into ``M*W`` contiguous owner
  shards: owner r gets [floor32(r*L/N), floor32((r+1)*L/N)), the last owner
  ending at L (``shard_ranges``); the owner keeps the momentum state for
  its shard only.

Two placements of the workers:

* single process (the reference's own model, kvstore.py:84-135): every
  worker's gradient buffer and weight replica live on this engine's device;
  one kernel reduces all of them;
* ``distributed=True`` (one process per GPU under torch.distributed, world
  size == machines*workers, worker id == rank): replicas are exchanged once
  as CUDA IPC mappings; each rank's kernel reads its shard from every peer
  over NVLink, updates it, and stores it into every peer's replica, with a
  device-side flag barrier at both ends of the kernel (no NCCL on the data
  path).

Consistency (kvstore.py:8-17): "sequential" = a key is reduced when every
worker of this process has pushed it for the round; a pull of a key whose
round is complete but not yet reduced flushes all pending keys in one launch.
"eventual" = every push is applied at once (single process only).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from . import _lib as L
from . import tensor as tmod
from .engine import Engine, default_engine
from .errors import ArgumentError, KVStoreError, StateError
from .tensor import Tensor

MODES = ("sequential", "eventual")
KEY_ALIGN = 64            # elements (256 bytes)
SHARD_ALIGN = 32          # elements (128 bytes)
DEFAULT_BUCKET_BYTES = 4 << 20


def add_updater(key: int, stored, incoming) -> None:
    """Default updater (kvstore.py:47-49): stored += incoming, on device."""
    stored.add_(incoming)


def padded(n: int) -> int:
    return -(-n // KEY_ALIGN) * KEY_ALIGN


def shard_ranges(length: int, owners: int) -> List[Tuple[int, int]]:
    """Owner shards of a bucket of ``length`` elements (the sharding rule)."""
    bounds = [(r * length // owners) // SHARD_ALIGN * SHARD_ALIGN for r in range(owners)]
    bounds.append(length)
    return [(bounds[r], bounds[r + 1]) for r in range(owners)]


def plan_buckets(numels: List[int], bucket_bytes: int = DEFAULT_BUCKET_BYTES
                 ) -> Tuple[List[int], List[Tuple[int, int]], List[int]]:
    """Arena layout for keys in init order: (key offsets, bucket ranges in
    arena order, bucket of each key).  Offsets/lengths in elements.

    Buckets are packed in PUSH order -- gradient-ready order, the reverse of
    init order for a feed-forward net: walking the keys from
    the last, consecutive keys join the open bucket until it holds
    ``bucket_bytes``; a key of ``bucket_bytes`` or more closes it and starts
    its own.  Each bucket is still a contiguous arena range, so its round is
    one launch that can start as soon as its last gradient is produced."""
    offs, pos = [], 0
    for n in numels:
        offs.append(pos)
        pos += padded(n)
    spans: List[Tuple[int, int]] = []
    hi = lo = pos
    for i in range(len(numels) - 1, -1, -1):
        if hi > lo and ((hi - lo) * 4 >= bucket_bytes or numels[i] * 4 >= bucket_bytes):
            spans.append((lo, hi))
            hi = lo
        lo = offs[i]
    if hi > lo or not spans:
        spans.append((lo, hi))
    buckets = spans[::-1]
    key_bucket, b = [], 0
    for off in offs:
        while buckets[b][1] <= off and b + 1 < len(buckets):
            b += 1
        key_bucket.append(b)
    return offs, buckets, key_bucket


def compact_velocity_layout(buckets: List[Tuple[int, int]], owners: int, owner: int
                            ) -> Tuple[Dict[int, int], int]:
    """Momentum layout of one owner: its shard of every bucket, packed in
    bucket order.  Returns (bucket -> offset, total length)."""
    offs, pos = {}, 0
    for b, (lo, hi) in enumerate(buckets):
        s0, s1 = shard_ranges(hi - lo, owners)[owner]
        offs[b] = pos
        pos += s1 - s0
    return offs, pos


def owner_segments(keys: List[Tuple[int, int, int]], buckets: List[Tuple[int, int]],
                   owners: int, owner: int, vbase: Optional[Dict[int, int]] = None
                   ) -> List[Tuple[int, int, int]]:
    """Element ranges ``owner`` reduces for the given keys.

    keys: (arena offset, padded length, bucket) per key, any order.
    Returns (arena offset, length, momentum offset) segments in arena order;
    momentum offsets use the compact layout ``vbase`` (bucket -> offset) or,
    when None, the full layout (momentum offset == arena offset).
    """
    segs = []
    for off, plen, b in sorted(keys):
        blo, bhi = buckets[b]
        s0, s1 = shard_ranges(bhi - blo, owners)[owner]
        lo, hi = max(off, blo + s0), min(off + plen, blo + s1)
        if lo < hi:
            voff = lo if vbase is None else vbase[b] + (lo - blo - s0)
            segs.append((lo, hi - lo, voff))
    return segs


def launches_for(segment_counts: List[int], max_segs: int) -> int:
    """Kernel launches a flush needs so every rank launches the same number
    (their device barriers pair up launch by launch)."""
    return -(-max(max(segment_counts), 1) // max_segs)


@dataclass
class _Key:
    key: int
    shape: tuple
    numel: int
    init: object                      # host float32 array until materialised
    off: int = -1
    bucket: int = -1
    arena: int = -1


@dataclass
class _Arena:
    """One materialised group of keys (keys inited after the first push or
    pull go into a new arena)."""
    keys: List[int]
    length: int
    buckets: List[Tuple[int, int]]
    weights: List[int] = field(default_factory=list)   # per-worker device pointers
    grads: List[int] = field(default_factory=list)
    flags: List[int] = field(default_factory=list)
    velocity: int = 0
    vlen: int = 0
    voff: Dict[Tuple[int, int], int] = field(default_factory=dict)  # (bucket, owner)
    agg: int = 0
    epoch_ctr: int = 0
    stage: List[int] = field(default_factory=list)    # push-mode staging buffers, per worker
    stage_slot: int = 0                                 # elements per slot of this rank's stage
    owned_local: List[int] = field(default_factory=list)  # pointers this process allocated
    opened: List[int] = field(default_factory=list)       # IPC-mapped pointers
    torch_views: Dict[Tuple[str, int], object] = field(default_factory=dict)


class _RawBuffer:
    """__cuda_array_interface__ over a device pointer so torch can view it."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class KVStore:
    def __init__(self, machines: int = 1, workers: int = 1, mode: str = "sequential",
                 etype: str = "float32", engine: Optional[Engine] = None,
                 tcp: Optional[str] = None, distributed: bool = False,
                 bucket_bytes: int = DEFAULT_BUCKET_BYTES, timeout: float = 120.0,
                 bucket_flush: bool = True):
        # bucket_flush: launch a bucket's round as soon as all its keys are
        # pushed (default); False defers every round to the next pull /
        # barrier / explicit flush, so a whole step's keys reduce in one
        # launch (one pair of cross-GPU barriers instead of one per bucket)
        self.bucket_flush = bucket_flush
        # push_mode: distributed rounds move every NVLink byte as a remote
        # store (gradients scattered to their owners' staging buffers, a
        # barrier, then weights broadcast).  Off by default: the one-phase
        # pull round (owners load peer gradients while storing weights, both
        # link directions busy at once) measured faster (N=2, 256 MB: 621 vs
        # 583 GB/s busbw).  MGX_KV_PUSH=1 turns it on.
        import os as _os
        self.push_mode = _os.environ.get("MGX_KV_PUSH", "0") == "1"
        if machines < 1 or workers < 1:
            raise ArgumentError("topology needs machines >= 1 and workers >= 1")
        if mode not in MODES:
            raise ArgumentError(f"unknown consistency mode {mode!r}")
        if etype != "float32":
            raise ArgumentError(f"unsupported etype {etype!r} (the device store is fp32)")
        if tcp is not None:
            raise ArgumentError("the TCP level-1/level-2 link is out of scope on one box "
                                "(kvstore.py:139-158); all workers share NVLink")
        self.machines, self.workers, self.mode, self.etype = machines, workers, mode, etype
        self.nw = machines * workers
        self.engine = engine or default_engine()
        self.distributed = distributed
        self.bucket_bytes = int(bucket_bytes)
        self.timeout = timeout
        if distributed:
            import torch.distributed as dist
            if not dist.is_initialized():
                raise ArgumentError("distributed KVStore needs torch.distributed initialised")
            if dist.get_world_size() != self.nw:
                raise ArgumentError(f"world size {dist.get_world_size()} != machines*workers "
                                    f"{self.nw}")
            if mode != "sequential":
                raise ArgumentError("eventual mode is single-process only")
            self.rank = dist.get_rank()
            self.local_workers = [self.rank]
        else:
            self.rank = 0
            self.local_workers = list(range(self.nw))
        self._lock = threading.RLock()
        self._cv = threading.Condition(self._lock)
        self._keys: Dict[int, _Key] = {}
        self._order: List[int] = []          # init order
        self._arenas: List[_Arena] = []
        self._rounds: Dict[Tuple[int, int], int] = {}
        self._pushed: Dict[int, set] = {}    # key -> local workers pushed this round
        self._pending: List[int] = []        # keys whose round is complete, not reduced
        self._stats = {"level2_messages": 0, "level2_updates": 0, "level1_aggregates": 0,
                       "pushes": 0, "pulls": 0, "flushes": 0, "launches": 0}
        self._updater: Callable = add_updater
        self._native = L.KV_ADD
        self._sgd = None                      # (eta, momentum, wd, scale)
        self._epoch = 0
        self._err = None
        self._failed = ""
        self._embedded: List = []       # round args placed inside executors
        # blocks per round when it runs inside the backward (fewer SMs taken
        # from the overlapped compute; env MGX_KV_OVERLAP_BLOCKS, 0 = all;
        # 32 measured best at N=2: AlexNet 2.588 -> 2.464 ms, Inception-BN
        # 5.887 -> 5.794 ms vs every SM, profiles/r02_overlap_sweep_n2.txt)
        self.overlap_blocks = int(_os.environ.get("MGX_KV_OVERLAP_BLOCKS", "32"))
        self._launch_count = 0          # kernels launched by rounds so far
        self.launches_per_flush = 0     # ... by the latest flush
        self._closed = False
        self._grid_cap = None

    # ------------------------------------------------------------ public API

    def init(self, key: int, value) -> None:
        """Register ``key`` with its initial value (kvstore.py:162-181)."""
        if not isinstance(key, (int, np.integer)) or key < 0:
            raise ArgumentError("keys are non-negative integers")
        key = int(key)
        if isinstance(value, Tensor):
            arr = tmod.to_numpy(value)
        else:
            import torch
            if isinstance(value, torch.Tensor):
                arr = value.detach().float().cpu().numpy()
            else:
                arr = np.array(value, dtype=np.float32)
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        with self._lock:
            if key in self._keys:
                raise KVStoreError(f"double init of key {key}")
            self._keys[key] = _Key(key, tuple(arr.shape), int(arr.size), arr.ravel().copy())
            self._order.append(key)

    def set_updater(self, fn: Callable) -> None:
        """Install the level-2 merge function (kvstore.py:183-188).  The
        momentum-SGD updater from ``optim.make_sgd_updater`` and the default
        add run fused in the reduce kernel; any other callable runs on
        device tensors after an aggregate-only reduction."""
        with self._lock:
            self._flush_locked()
            sgd = getattr(fn, "_mgx_sgd", None)
            if sgd is not None:
                cfg, scale = sgd
                self._native = L.KV_SGD
                self._sgd = (float(np.float32(cfg.eta)), float(np.float32(cfg.momentum)),
                             float(np.float32(cfg.weight_decay)),
                             float(np.float32(1.0 / scale)))
            elif fn is add_updater:
                self._native = L.KV_ADD
            else:
                if self._embedded:
                    raise KVStoreError("a plugin updater cannot run inside a bound step's "
                                       "backward (embedded rounds); set it before binding")
                self._native = L.KV_AGG
            self._updater = fn
            for a in self._embedded:
                self._set_updater_fields(a)

    def push(self, key: int, value: Tensor, worker: int) -> None:
        """Join this worker's next round for ``key`` (kvstore.py:190-211)."""
        self._check_worker(worker)
        k = self._key(key)
        if value.shape != k.shape:
            raise KVStoreError(f"push shape {value.shape} != init shape {k.shape}")
        if value.engine is not self.engine:
            raise ArgumentError("pushed tensor is on another engine")
        with self._lock:
            ar = self._materialize_locked(k)
            r = self._rounds.get((worker, key), 0) + 1
            self._rounds[(worker, key)] = r
            self._stats["pushes"] += 1
            dst = ar.grads[self._slot(worker)] + 4 * k.off
            if value.ptr != dst:
                self.engine.push(lambda: L.call("mgx_copy", value.ptr, dst, k.numel,
                                                self.engine.stream_handle),
                                 reads=[value.tag], label=f"kv-push:{key}")
            if self.mode == "eventual":
                self._launch_locked([key], single_worker=self._slot(worker))
                return
            done = self._pushed.setdefault(key, set())
            if worker in done:
                raise StateError(f"worker {worker} pushed key {key} twice in one round")
            done.add(worker)
            if len(done) == len(self.local_workers):
                self._pushed[key] = set()
                self._pending.append(key)
                self._cv.notify_all()
                if self.bucket_flush and self._bucket_complete_locked(k):
                    self._flush_locked()

    def pull(self, key: int, out: Tensor, worker: int) -> None:
        """Copy this worker's round value of ``key`` into ``out``
        (kvstore.py:213-241)."""
        self._check_worker(worker)
        k = self._key(key)
        if out.shape != k.shape:
            raise KVStoreError(f"pull shape {out.shape} != init shape {k.shape}")
        if out.engine is not self.engine:
            raise ArgumentError("pulled tensor is on another engine")
        with self._lock:
            ar = self._materialize_locked(k)
            self._stats["pulls"] += 1
            if self.mode == "sequential":
                want = self._rounds.get((worker, key), 0)
                self._wait_round_locked(key, want)
                if key in self._pending:
                    self._flush_locked()
            src = ar.weights[self._slot(worker)] + 4 * k.off
            if out.ptr != src:
                self.engine.push(lambda: L.call("mgx_copy", src, out.ptr, k.numel,
                                                self.engine.stream_handle),
                                 writes=[out.tag], label=f"kv-pull:{key}")

    def round_barrier(self) -> None:
        """Reduce everything pushed so far and wait for the device."""
        with self._lock:
            self._flush_locked()
        self.engine.wait_all()
        self._check_error()

    def quiesce(self) -> None:
        self.round_barrier()

    def stats(self) -> Dict[str, int]:
        with self._lock:
            return dict(self._stats)

    def close(self) -> None:
        if self._closed:
            return
        with self._lock:
            self._flush_locked()
        try:
            self.engine.synchronize()
        except Exception:  # noqa: BLE001
            pass
        if self.distributed:
            import torch.distributed as dist
            dist.barrier()
        for ar in self._arenas:
            for p in ar.opened:
                L.lib().mgx_ipc_close_handle(p)
            for p in ar.owned_local:
                L.lib().mgx_free(p)
        if self._err is not None:
            try:
                self.engine._checks.remove(self._check_error)
            except ValueError:
                pass
            L.lib().mgx_host_free(self._err)
            self._err = None
        self._arenas = []
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -------------------------------------------------- zero-copy endpoints

    def weight_tensor(self, key: int, worker: int) -> Tensor:
        """The replica ``pull`` reads for ``worker``, as a bindable Tensor
        (binding it as the executor argument makes pull a no-op)."""
        return self._view("w", key, worker)

    def grad_tensor(self, key: int, worker: int) -> Tensor:
        """The buffer ``push`` reduces from for ``worker``; binding it as the
        executor's gradient makes push copy-free."""
        return self._view("g", key, worker)

    def _view(self, kind: str, key: int, worker: int) -> Tensor:
        self._check_worker(worker)
        k = self._key(key)
        with self._lock:
            ar = self._materialize_locked(k)
            base = (ar.weights if kind == "w" else ar.grads)[self._slot(worker)]
            import torch
            full = ar.torch_views.get((kind, worker))
            if full is None:
                full = torch.as_tensor(_RawBuffer(base, ar.length), device=f"cuda:{self.engine.device}")
                ar.torch_views[(kind, worker)] = full
            return Tensor(k.shape, "float32", engine=self.engine,
                          _storage=full[k.off: k.off + k.numel].view(k.shape))

    # --------------------------------------------------------------- helpers

    def _check_worker(self, worker: int) -> None:
        if not 0 <= worker < self.nw:
            raise ArgumentError(f"no worker {worker} in this topology")
        if worker not in self.local_workers:
            raise ArgumentError(f"worker {worker} belongs to another process (rank {worker})")

    def _key(self, key: int) -> _Key:
        k = self._keys.get(key)
        if k is None:
            raise KVStoreError(f"key {key} used before init")
        return k

    def _slot(self, worker: int) -> int:
        return worker  # replica / gradient pointer index == worker id

    def _wait_round_locked(self, key: int, want: int) -> None:
        """Sequential mode: block until every local worker reached round
        ``want`` for key (other threads may still be pushing)."""
        def ready():
            return all(self._rounds.get((w, key), 0) >= want for w in self.local_workers)
        if not self._cv.wait_for(ready, timeout=self.timeout):
            raise KVStoreError(f"timed out waiting for round {want} of key {key}")

    def _bucket_complete_locked(self, k: _Key) -> bool:
        ar = self._arenas[k.arena]
        members = [kk for kk in ar.keys if self._keys[kk].bucket == k.bucket]
        return all(m in self._pending for m in members)

    # ------------------------------------------------------------ materialise

    def _materialize_locked(self, k: _Key) -> _Arena:
        if k.arena >= 0:
            return self._arenas[k.arena]
        new = [kk for kk in self._order if self._keys[kk].arena < 0]
        numels = [self._keys[kk].numel for kk in new]
        offs, buckets, kb = plan_buckets(numels, self.bucket_bytes)
        length = sum(padded(n) for n in numels)
        ar = _Arena(keys=new, length=length, buckets=buckets)
        aid = len(self._arenas)
        for kk, off, b in zip(new, offs, kb):
            self._keys[kk].off, self._keys[kk].bucket, self._keys[kk].arena = off, b, aid
        self.engine.activate()
        nbytes = 4 * length
        st = self.engine.stream_handle

        def alloc(n):
            p = ctypes.c_void_p()
            L.call("mgx_malloc", n, ctypes.byref(p))
            ar.owned_local.append(p.value)
            L.call("mgx_memset_async", p.value, 0, n, st)
            return p.value

        if self._err is None:
            p = ctypes.c_void_p()
            L.call("mgx_host_alloc", 64, ctypes.byref(p))
            ctypes.memset(p.value, 0, 64)
            self._err = p.value
            # every engine sync point (wait_for / wait_all / to_numpy) raises
            # once a device barrier has timed out
            self.engine.add_check(self._check_error)
        if self.distributed:
            self._materialize_distributed(ar, alloc, nbytes)
        else:
            ar.weights = [alloc(nbytes) for _ in range(self.nw)]
            ar.grads = [alloc(nbytes) for _ in range(self.nw)]
            ar.velocity = alloc(nbytes)
            ar.vlen = length
            for b, (lo, _hi) in enumerate(buckets):
                for r in range(self.nw):
                    ar.voff[(b, r)] = lo  # full layout: velocity offset == arena offset
            for kk in new:
                key = self._keys[kk]
                host = key.init
                for w in range(self.nw):
                    dst = ar.weights[w] + 4 * key.off
                    L.call("mgx_memcpy_async", dst, host.ctypes.data, 4 * key.numel, st)
            L.call("mgx_stream_sync", st)
        for kk in new:
            self._keys[kk].init = None
        self._arenas.append(ar)
        return ar

    def _materialize_distributed(self, ar: _Arena, alloc, nbytes: int) -> None:
        import torch.distributed as dist
        st = self.engine.stream_handle
        own_w = alloc(nbytes)
        own_g = alloc(nbytes)
        flag_bytes = 4 * L.KV_FLAG_WORDS_PER_WORKER * self.nw
        own_f = alloc(flag_bytes)
        ar.epoch_ctr = alloc(256)
        # compact momentum layout: this rank's shard of every bucket
        vb, vpos = compact_velocity_layout(ar.buckets, self.nw, self.rank)
        for b, off in vb.items():
            ar.voff[(b, self.rank)] = off
        ar.vlen = vpos
        ar.velocity = alloc(max(4 * vpos, 256))
        # push-mode staging: one slot per worker, laid out like the momentum
        # shard (every worker stores its gradient values for this shard there)
        ar.stage_slot = -(-max(vpos, 1) // KEY_ALIGN) * KEY_ALIGN
        own_s = alloc(4 * ar.stage_slot * self.nw)
        for kk in ar.keys:
            key = self._keys[kk]
            L.call("mgx_memcpy_async", own_w + 4 * key.off, key.init.ctypes.data,
                   4 * key.numel, st)
        L.call("mgx_stream_sync", st)

        def handle(p):
            buf = ctypes.create_string_buffer(L.IPC_HANDLE_BYTES)
            L.call("mgx_ipc_get_handle", p, buf)
            return buf.raw

        mine = (handle(own_w), handle(own_g), handle(own_f), handle(own_s))
        everyone: List = [None] * self.nw
        dist.all_gather_object(everyone, mine)

        def open_(h, own):
            if h in mine:
                return own
            p = ctypes.c_void_p()
            L.call("mgx_ipc_open_handle", ctypes.create_string_buffer(h, L.IPC_HANDLE_BYTES),
                   ctypes.byref(p))
            ar.opened.append(p.value)
            return p.value

        for r in range(self.nw):
            hw, hg, hf, hs = everyone[r]
            ar.weights.append(own_w if r == self.rank else open_(hw, own_w))
            ar.grads.append(own_g if r == self.rank else open_(hg, own_g))
            ar.flags.append(own_f if r == self.rank else open_(hf, own_f))
            ar.stage.append(own_s if r == self.rank else open_(hs, own_s))
        dist.barrier()
        # every replica starts from worker 0's init value (kvstore init
        # broadcasts one value, kvstore.py:177-181)
        if self.rank != 0:
            L.call("mgx_memcpy_async", own_w, ar.weights[0], nbytes, st)
            L.call("mgx_stream_sync", st)
        dist.barrier()

    # -------------------------------------------------------------- reduce

    def _flush_locked(self) -> None:
        if not self._pending:
            return
        pending, self._pending = self._pending, []
        before = self._launch_count
        by_arena: Dict[int, List[int]] = {}
        for key in pending:
            by_arena.setdefault(self._keys[key].arena, []).append(key)
        for aid in sorted(by_arena):
            self._launch_locked(by_arena[aid])
        self._stats["flushes"] += 1
        self.launches_per_flush = self._launch_count - before
        for key in pending:
            self._stats["level1_aggregates"] += self.machines
            self._stats["level2_messages"] += self.machines
            self._stats["level2_updates"] += 1

    def _segments(self, ar: _Arena, keys: List[int], owners: List[int],
                  whole_keys: bool = False) -> List[Tuple[int, int, int]]:
        spans = [(self._keys[kk].off, padded(self._keys[kk].numel), self._keys[kk].bucket)
                 for kk in keys]
        if whole_keys:
            return [(off, plen, off) for off, plen, _b in sorted(spans)]
        segs = []
        for r in owners:
            vbase = ({b: ar.voff[(b, r)] for b in range(len(ar.buckets))}
                     if self.distributed else None)
            segs += owner_segments(spans, ar.buckets, self.nw, r, vbase)
        return sorted(segs)

    def _grid_locked(self, total_elems: int) -> int:
        if self._grid_cap is None:
            cap, thr, unr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
            L.call("mgx_kv_config", self.machines, self.workers, ctypes.byref(cap),
                   ctypes.byref(thr), ctypes.byref(unr))
            self._grid_cap, self._per_block = cap.value, thr.value * unr.value
        # identical on every rank: derived from the flush size only
        per_rank4 = -(-total_elems // (4 * self.nw))
        want = -(-per_rank4 // self._per_block)
        return max(1, min(self._grid_cap, want))

    def _launch_locked(self, keys: List[int], single_worker: Optional[int] = None) -> None:
        if self._failed:
            raise KVStoreError(f"store failed earlier: {self._failed}")
        ar = self._arenas[self._keys[keys[0]].arena]
        updater = self._native
        custom = updater == L.KV_AGG
        if custom and ar.agg == 0:
            p = ctypes.c_void_p()
            L.call("mgx_malloc", 4 * ar.length, ctypes.byref(p))
            ar.owned_local.append(p.value)
            ar.agg = p.value
        if single_worker is not None:
            # eventual mode: apply this worker's push alone
            segs = self._segments(ar, keys, [], whole_keys=True)
            machines, workers = 1, 1
            grads = [ar.grads[single_worker]]
            weights = list(ar.weights)
        else:
            owners = self.local_workers if self.distributed else list(range(self.nw))
            segs = self._segments(ar, keys, owners, whole_keys=custom)
            machines, workers = self.machines, self.workers
            grads, weights = ar.grads, ar.weights
        total = sum(padded(self._keys[kk].numel) for kk in keys)
        barrier = self.distributed and single_worker is None
        nchunks = -(-max(len(segs), 1) // L.KV_MAX_SEGS)
        if barrier and not custom:
            # every rank must launch the same number of kernels so the
            # device barrier epochs line up: use the largest owner's count
            spans = [(self._keys[kk].off, padded(self._keys[kk].numel), self._keys[kk].bucket)
                     for kk in keys]
            counts = [len(owner_segments(spans, ar.buckets, self.nw, r)) for r in range(self.nw)]
            nchunks = launches_for(counts, L.KV_MAX_SEGS)
        scatter = None
        if barrier and not custom and self.push_mode and nchunks == 1:
            scatter = self._scatter_segments(ar, keys)
            if len(scatter) > L.KV_MAX_SEGS:
                scatter = None
        for c in range(nchunks):
            chunk = segs[c * L.KV_MAX_SEGS: (c + 1) * L.KV_MAX_SEGS]
            self._launch_one(ar, chunk, machines, workers, grads, weights, updater, total,
                             barrier=barrier, scatter=scatter)
        if custom:
            self._run_custom_updater(ar, keys)

    def _scatter_segments(self, ar: _Arena, keys: List[int]) -> List[Tuple[int, int, int, int]]:
        """Push mode, phase 1: for every owner (ascending), that owner's
        segments in its own order, with the element offset of this rank's
        slot in the owner's staging buffer: (arena off, len, stage off, owner)."""
        spans = [(self._keys[kk].off, padded(self._keys[kk].numel), self._keys[kk].bucket)
                 for kk in keys]
        out = []
        for o in range(self.nw):
            vb, vlen = compact_velocity_layout(ar.buckets, self.nw, o)
            slot = -(-max(vlen, 1) // KEY_ALIGN) * KEY_ALIGN
            for off, ln, voff in owner_segments(spans, ar.buckets, self.nw, o, vb):
                out.append((off, ln, self.rank * slot + voff, o))
        return out

    def _launch_one(self, ar, segs, machines, workers, grads, weights, updater, total,
                    barrier: bool, scatter=None) -> None:
        a, _keep = self._round_args(ar, segs, machines, workers, grads, weights, updater, total,
                                    barrier, scatter)
        nw = machines * workers
        # an eventual-mode push reduces one source; the kernel stores into
        # that many replicas, the rest are refreshed by a copy below
        broadcast_rest = nw == 1 and len(weights) > 1
        self._launch_count += 1 + (len(segs) * (len(weights) - 1) if broadcast_rest else 0)
        self.engine.activate()
        L.call("mgx_kv_round", ctypes.byref(a), self.engine.stream_handle)
        self._stats["launches"] += 1
        if broadcast_rest and updater != L.KV_AGG:
            for off, ln, _ in segs:
                for w in weights[1:]:
                    L.call("mgx_copy", weights[0] + 4 * off, w + 4 * off, ln,
                           self.engine.stream_handle)

    def _round_args(self, ar, segs, machines, workers, grads, weights, updater, total,
                    barrier: bool, scatter=None, grid_cap: Optional[int] = None):
        """mgx_kv_round_args for one launch, plus the host arrays it points
        to (the caller keeps them alive as long as the args are used)."""
        nw = machines * workers
        a = L.KvRoundArgs()
        seg_arr = (L.KvSeg * max(len(segs), 1))()
        for i, (off, ln, voff) in enumerate(segs):
            seg_arr[i].off, seg_arr[i].len, seg_arr[i].voff = off, ln, voff
        g_arr = (ctypes.c_void_p * nw)(*grads[:nw])
        w_arr = (ctypes.c_void_p * len(weights))(*weights)
        a.segs = seg_arr
        a.nseg = len(segs)
        a.machines, a.workers = machines, workers
        a.grads = ctypes.cast(g_arr, ctypes.POINTER(ctypes.c_void_p))
        a.weights = ctypes.cast(w_arr, ctypes.POINTER(ctypes.c_void_p))
        a.self_replica = self.rank if self.distributed else 0
        a.velocity = ar.velocity
        a.agg_out = ar.agg or None
        a.updater = updater
        self._set_updater_fields(a, updater)
        f_arr = None
        if barrier:
            self._epoch += 1
            f_arr = (ctypes.c_void_p * nw)(*ar.flags)
            a.flags = ctypes.cast(f_arr, ctypes.POINTER(ctypes.c_void_p))
            a.rank = self.rank
            a.epoch_ctr = ar.epoch_ctr
            a.error_word = self._err
            a.grid = self._grid_locked(total)
            if grid_cap:
                a.grid = max(1, min(a.grid, grid_cap))
        else:
            a.flags = None
            a.grid = 0
        a.nscatter = 0
        if scatter:
            sc_arr = (L.KvSeg * len(scatter))()
            own_arr = (ctypes.c_int32 * len(scatter))()
            for q, (off, ln, soff, o) in enumerate(scatter):
                sc_arr[q].off, sc_arr[q].len, sc_arr[q].voff = off, ln, soff
                own_arr[q] = o
            st_arr = (ctypes.c_void_p * nw)(*ar.stage)
            a.scatter = sc_arr
            a.scatter_owner = own_arr
            a.nscatter = len(scatter)
            a.stage = ctypes.cast(st_arr, ctypes.POINTER(ctypes.c_void_p))
            a.stage_slot = ar.stage_slot
        keep = [seg_arr, g_arr, w_arr, f_arr]
        if scatter:
            keep += [sc_arr, own_arr, st_arr]
        return a, keep

    def _set_updater_fields(self, a, updater: Optional[int] = None) -> None:
        a.updater = self._native if updater is None else updater
        if self._sgd is not None:
            eta, mom, wd, rescale = self._sgd
            a.rescale, a.neg_eta, a.momentum, a.weight_decay = rescale, -eta, mom, wd

    # ------------------------------------------- rounds inside the backward

    def embedded_rounds(self, worker: int) -> List[dict]:
        """Per-bucket round launches for a step in which ``worker`` (this
        process's only worker) pushes every key, in push order (last bucket
        first), for the executor to place INSIDE its backward program: each
        round then starts as soon as its bucket's last gradient is written
        and overlaps the rest of the backward (the
        reference pushes after the backward, kvstore.py:116-120,
        train.py:210-223).  Each dict: ``args`` (mgx_kv_round_args, kept
        alive with ``keep``), ``reads`` (this worker's gradient ranges of the
        bucket's keys), ``writes`` (its weight ranges), ``keys``.  Only for
        the fused native updaters in sequential mode with one local worker;
        returns [] otherwise (the step then flushes after the backward)."""
        if (self.mode != "sequential" or self._native == L.KV_AGG
                or self.local_workers != [worker] or not self._order):
            return []
        rounds = []
        with self._lock:
            for key in self._order:
                self._materialize_locked(self._keys[key])
            for aid, ar in enumerate(self._arenas):
                by_bucket: Dict[int, List[int]] = {}
                for kk in ar.keys:
                    by_bucket.setdefault(self._keys[kk].bucket, []).append(kk)
                for b in sorted(by_bucket, reverse=True):
                    keys = by_bucket[b]
                    rounds += self._bucket_rounds(ar, keys, worker)
        return rounds

    def _bucket_rounds(self, ar: _Arena, keys: List[int], worker: int) -> List[dict]:
        owners = self.local_workers if self.distributed else list(range(self.nw))
        segs = self._segments(ar, keys, owners)
        total = sum(padded(self._keys[kk].numel) for kk in keys)
        barrier = self.distributed
        nchunks = -(-max(len(segs), 1) // L.KV_MAX_SEGS)
        if barrier:
            spans = [(self._keys[kk].off, padded(self._keys[kk].numel), self._keys[kk].bucket)
                     for kk in keys]
            counts = [len(owner_segments(spans, ar.buckets, self.nw, r)) for r in range(self.nw)]
            nchunks = launches_for(counts, L.KV_MAX_SEGS)
        slot = self._slot(worker)
        reads = [(ar.grads[slot] + 4 * self._keys[kk].off,
                  ar.grads[slot] + 4 * (self._keys[kk].off + self._keys[kk].numel)) for kk in keys]
        writes = [(ar.weights[slot] + 4 * self._keys[kk].off,
                   ar.weights[slot] + 4 * (self._keys[kk].off + self._keys[kk].numel))
                  for kk in keys]
        out = []
        for c in range(nchunks):
            chunk = segs[c * L.KV_MAX_SEGS: (c + 1) * L.KV_MAX_SEGS]
            a, keep = self._round_args(ar, chunk, self.machines, self.workers, ar.grads,
                                       ar.weights, self._native, total, barrier,
                                       grid_cap=self.overlap_blocks)
            out.append({"args": a, "keep": keep, "reads": reads, "writes": writes,
                        "keys": list(keys), "bytes": 4 * total})
            # set_updater refreshes these in place (the program captures the
            # struct's values at launch / graph-capture time)
            self._embedded.append(a)
        return out

    def note_embedded_round(self, worker: int) -> None:
        """Book-keeping for a step whose rounds ran inside the executor's
        backward: every key's round counter advances as if pushed and
        reduced (pulls and round_barrier stay consistent)."""
        with self._lock:
            for key in self._order:
                self._rounds[(worker, key)] = self._rounds.get((worker, key), 0) + 1
            self._stats["pushes"] += len(self._order)
            self._stats["level1_aggregates"] += self.machines * len(self._order)
            self._stats["level2_messages"] += self.machines * len(self._order)
            self._stats["level2_updates"] += len(self._order)
            self._cv.notify_all()

    def _run_custom_updater(self, ar: _Arena, keys: List[int]) -> None:
        import torch
        dev = f"cuda:{self.engine.device}"
        own = self.rank if self.distributed else 0
        stored_full = torch.as_tensor(_RawBuffer(ar.weights[own], ar.length), device=dev)
        agg_full = torch.as_tensor(_RawBuffer(ar.agg, ar.length), device=dev)
        with torch.cuda.stream(self.engine.stream):
            for key in keys:
                k = self._keys[key]
                stored = stored_full[k.off: k.off + k.numel].view(k.shape)
                incoming = agg_full[k.off: k.off + k.numel].view(k.shape)
                self._updater(key, stored, incoming)
                if not self.distributed:
                    for w in range(1, self.nw):
                        L.call("mgx_copy", ar.weights[0] + 4 * k.off, ar.weights[w] + 4 * k.off,
                               k.numel, self.engine.stream_handle)

    def _check_error(self) -> None:
        if self._failed:
            raise KVStoreError(self._failed)
        if self._err is not None and ctypes.c_uint32.from_address(self._err).value:
            # the timed-out blocks skipped their reduce and closing barrier:
            # replicas and barrier epochs are no longer consistent
            self._failed = ("a peer did not reach the device barrier within the kernel's 30 s "
                            "limit; replicas may have diverged, the store refuses further rounds")
            raise KVStoreError(self._failed)
