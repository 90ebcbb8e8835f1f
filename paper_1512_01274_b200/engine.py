"""Stream-ordered engine: the B200 replacement for the reference's
read/write-tag thread pool (engine.py:65-264).

The reference lets host closures run concurrently unless their tags
conflict, and serialises conflicting ones in push order.  On the GPU every
closure only *enqueues* device work, and all of an engine's work goes onto
one CUDA stream, so push order is execution order — a strictly stronger
guarantee than per-tag FIFO, with no host threads involved.  The API keeps
the reference's surface: tags, ``push``/``push_delete``, ``wait_for``/
``wait_all`` as synchronisation points, poisoning of a failed closure's
written tags surfaced as ``OperationFailed``, and the rule that closures
must not call ``wait_*`` (engine.py:217-219).
"""

from __future__ import annotations

import itertools
import threading
from typing import Callable, Iterable, List, Optional

from . import _lib as L
from .errors import LifecycleError, OperationFailed, StateError

_ctx = threading.local()


def _stack() -> List["Engine"]:
    st = getattr(_ctx, "stack", None)
    if st is None:
        st = _ctx.stack = []
    return st


def current_engine() -> "Engine":
    st = _stack()
    return st[-1] if st else default_engine()


def current_stream() -> int:
    return current_engine().stream_handle


def current_device() -> int:
    return current_engine().device


class ResourceTag:
    """Identity of one mutable resource (engine.py:27-50)."""

    __slots__ = ("id", "label", "engine", "_poison", "_dying", "_dead", "_pending")

    def __init__(self, tag_id: int, label: str, engine: "Engine"):
        self.id = tag_id
        self.label = label
        self.engine = engine
        self._poison: Optional[BaseException] = None
        self._dying = False
        self._dead = False
        self._pending = 0

    def __repr__(self):
        return f"ResourceTag({self.id}, {self.label!r})"


class Engine:
    """One CUDA stream on one device; closures run at push time and enqueue
    their kernels on that stream."""

    def __init__(self, threads: Optional[int] = None, device: Optional[int] = None):
        import torch
        if not torch.cuda.is_available():
            raise StateError("the device engine needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.num_threads = threads or 1
        with torch.cuda.device(self.device):
            L.call("mgx_set_device", self.device)
            self.stream = torch.cuda.Stream(device=self.device)
        self.stream_handle = int(self.stream.cuda_stream)
        self._ids = itertools.count(1)
        self._lock = threading.Lock()
        self._executed = 0
        self._since_sync = 0
        self._closed = False
        self._checks: List[Callable[[], None]] = []

    # -------------------------------------------------------------- tags

    def new_tag(self, label: str = "") -> ResourceTag:
        return ResourceTag(next(self._ids), label, self)

    # ------------------------------------------------------------ context

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def activate(self) -> "Engine":
        """Make this engine's device current for native calls (cheap)."""
        if getattr(_ctx, "device", None) != self.device:
            import torch
            torch.cuda.set_device(self.device)
            L.call("mgx_set_device", self.device)
            _ctx.device = self.device
        return self

    # --------------------------------------------------------------- push

    def push(self, closure: Callable[[], None], reads: Iterable[ResourceTag] = (),
             writes: Iterable[ResourceTag] = (), label: str = "") -> None:
        """Run ``closure`` now; it enqueues device work on this stream.  A
        raising closure poisons its written tags (engine.py:181-196)."""
        writes = tuple(dict.fromkeys(writes))
        reads = tuple(t for t in dict.fromkeys(reads) if t not in set(writes))
        if self._closed:
            raise StateError("engine is closed")
        for t in reads + writes:
            if t._dying or t._dead:
                raise LifecycleError(f"push on deleted tag {t!r}")
        if getattr(_ctx, "in_closure", False):
            self._run(closure, writes)
            return
        _ctx.in_closure = True
        try:
            self.activate()
            _stack().append(self)
            try:
                self._run(closure, writes)
            finally:
                _stack().pop()
        finally:
            _ctx.in_closure = False

    def _run(self, closure, writes):
        try:
            closure()
        except BaseException as exc:  # noqa: BLE001 - surfaced at wait_for
            for t in writes:
                if t._poison is None:
                    t._poison = exc
        with self._lock:
            self._executed += 1
            self._since_sync += 1

    def push_delete(self, tag: ResourceTag,
                    on_delete: Optional[Callable[[], None]] = None) -> None:
        if tag._dying or tag._dead:
            raise LifecycleError(f"double delete of tag {tag!r}")
        tag._dying = True

        def _delete():
            if on_delete is not None:
                on_delete()
            tag._dead = True

        # deletion must wait for enqueued work that still reads the buffer
        self.synchronize()
        self.push(_delete, writes=(), label=f"delete:{tag.label}")

    # --------------------------------------------------------------- sync

    def add_check(self, fn: Callable[[], None]) -> None:
        """Register a post-sync check (e.g. a device error word)."""
        self._checks.append(fn)

    def synchronize(self) -> None:
        L.call("mgx_stream_sync", self.stream_handle)
        with self._lock:
            self._since_sync = 0

    def wait_for(self, tag: ResourceTag) -> None:
        """Synchronisation point: all enqueued work done; re-raise the tag's
        captured failure as OperationFailed (engine.py:200-209)."""
        self._check_waitable()
        try:
            self.synchronize()
            for fn in self._checks:
                fn()
        except Exception as exc:  # noqa: BLE001
            raise OperationFailed(f"device work failed: {exc}") from exc
        if tag._poison is not None:
            raise OperationFailed(
                f"operation on tag {tag.label!r} failed: {tag._poison!r}") from tag._poison

    def wait_all(self) -> None:
        self._check_waitable()
        try:
            self.synchronize()
            for fn in self._checks:
                fn()
        except Exception as exc:  # noqa: BLE001
            raise OperationFailed(f"device work failed: {exc}") from exc

    def _check_waitable(self):
        if getattr(_ctx, "in_closure", False):
            raise StateError("engine closures must not call wait_* (deadlock rule)")

    @property
    def pending(self) -> int:
        """Closures pushed since the stream was last seen idle whose device
        work may still be in flight (0 once the stream has drained)."""
        with self._lock:
            if self._since_sync and self.stream.query():
                self._since_sync = 0
            return self._since_sync

    @property
    def executed(self) -> int:
        with self._lock:
            return self._executed

    def dump(self) -> str:
        return (f"engine: device {self.device} stream 0x{self.stream_handle:x}, "
                f"{self._executed} executed")

    def close(self) -> None:
        if not self._closed:
            self.synchronize()
            self._closed = True

    def __del__(self):
        pass


_default: Optional[Engine] = None
_default_lock = threading.Lock()


def default_engine() -> Engine:
    global _default
    with _default_lock:
        if _default is None or _default._closed:
            _default = Engine()
        return _default


def set_default_engine(engine: Engine) -> None:
    global _default
    with _default_lock:
        _default = engine


def configure_default_engine(threads: int) -> Engine:
    global _default
    with _default_lock:
        if _default is not None and not _default._closed:
            _default.close()
        _default = Engine(threads=threads)
        return _default
