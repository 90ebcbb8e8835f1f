"""Training drivers: the data-parallel step over the device KVStore.

Mirrors the reference's train.py (mlp/param_names/init_params/TrainReport,
train_local, train_distributed; train.py:57-270) with the per-worker step

    pull every key -> load the worker's row shard -> forward -> backward
    -> push every key -> read the outputs

Worker g takes rows [g*B/N, (g+1)*B/N) of every global batch and every
worker walks the same shuffled batch order (train.py:166-168, 195, 206).
Executors are bound zero-copy to the store: a worker's parameter arguments
ARE its KVStore replica and its gradient outputs ARE its KVStore gradient
buffer, so push/pull move no bytes and the only data-path kernels are the
graph's and the store's fused reduce+update+broadcast.

``DataParallelStep`` is the reusable core; it can also capture one whole
step (forward, backward, store round) into a single CUDA graph.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from . import symbol
from . import tensor as tmod
from .data import BatchOrder, read_examples
from .engine import Engine, default_engine
from .errors import ArgumentError
from .executor import bind
from .kvstore import KVStore
from .optim import SGDConfig, make_sgd_updater, sgd_step
from .symbol import SymbolGraph, infer_shape

RESERVED_ARGS = ("data", "label")
CSV_HEADER = "epoch,loss,acc,seconds,planner_bytes,engine_ops"


@dataclass
class TrainReport:
    rows: List[tuple] = field(default_factory=list)

    def append(self, epoch, loss, acc, seconds, planner_bytes, engine_ops) -> None:
        self.rows.append((epoch, loss, acc, seconds, planner_bytes, engine_ops))

    def to_csv(self) -> str:
        out = [CSV_HEADER]
        for e, loss, acc, sec, pb, ops in self.rows:
            out.append(f"{e},{loss!r},{acc!r},{sec:.3f},{pb},{ops}")
        return "\n".join(out) + "\n"

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.to_csv())


def mlp(hidden: Sequence[int], classes: int) -> SymbolGraph:
    """relu MLP ending in a softmax loss head (train.py:57-67)."""
    net = symbol.variable("data")
    for i, h in enumerate(hidden, 1):
        net = symbol.apply("FullyConnected", {"num_hidden": int(h)}, [net], name=f"fc{i}")
        net = symbol.apply("Activation", {"act_type": "relu"}, [net], name=f"act{i}")
    net = symbol.apply("FullyConnected", {"num_hidden": int(classes)}, [net], name="out")
    return symbol.apply("SoftmaxOutput", {}, [net], name="softmax")


AUX_SUFFIXES = ("_moving_mean", "_moving_var")


def param_names(g: SymbolGraph) -> List[str]:
    """Trainable arguments in list_arguments order (the KVStore keys)."""
    return [n for n in g.list_arguments()
            if n not in RESERVED_ARGS and not n.endswith(AUX_SUFFIXES)]


def aux_names(g: SymbolGraph) -> List[str]:
    """BatchNorm moving statistics: per-worker state, never pushed."""
    return [n for n in g.list_arguments() if n.endswith(AUX_SUFFIXES)]


def init_params(g: SymbolGraph, arg_shapes: Dict[str, tuple], seed: int) -> Dict[str, np.ndarray]:
    """randn*0.1 weights in parameter order, zero biases (train.py:74-85);
    BatchNorm gamma ones and beta zeros (no RNG draw, like the biases)."""
    rs = np.random.RandomState(seed)
    out = {}
    for name in param_names(g):
        shape = arg_shapes[name]
        if name.endswith(("_bias", "_beta")):
            out[name] = np.zeros(shape, dtype=np.float32)
        elif name.endswith("_gamma"):
            out[name] = np.ones(shape, dtype=np.float32)
        else:
            out[name] = (rs.randn(*shape) * 0.1).astype(np.float32)
    return out


def init_aux(g: SymbolGraph, arg_shapes: Dict[str, tuple]) -> Dict[str, np.ndarray]:
    """moving_mean zeros, moving_var ones (MXNet's aux initialisation)."""
    return {n: (np.zeros if n.endswith("_moving_mean") else np.ones)(arg_shapes[n], np.float32)
            for n in aux_names(g)}


def cross_entropy_mean(probs: np.ndarray, labels: np.ndarray, eps: float = 1e-12) -> float:
    """Host-side metric only (kernels.py:86-89)."""
    idx = labels.astype(np.int64)
    picked = probs[np.arange(idx.shape[0]), idx]
    return float(np.mean(-np.log(np.maximum(picked, eps))))


def _check_graph(g: SymbolGraph):
    args = g.list_arguments()
    for need in RESERVED_ARGS:
        if need not in args:
            raise ArgumentError(f"training graph needs a {need!r} argument")


def _load(data) -> Tuple[np.ndarray, np.ndarray]:
    if isinstance(data, str):
        return read_examples(data)
    feats, labels = data
    return np.asarray(feats, np.float32), np.asarray(labels, np.float32)


class DataParallelStep:
    """One data-parallel training step over a device KVStore.

    Binds one executor per local worker (all workers in a single-process
    store, the rank's own worker in a distributed one) against the store's
    replicas and gradient buffers.

    Push/backward overlap (``overlap=True``): when this
    process drives exactly one worker (one rank per GPU, or a 1-worker
    store) and the updater is a fused native one, the store's per-bucket
    rounds are placed INSIDE the executor's backward program on their own
    stream: bucket b's fused reduce + update + broadcast starts as soon as
    its last gradient is written and overlaps the rest of the backward
    (buckets are packed in push order, KVStore.plan_buckets).  Otherwise --
    several workers in one process, a plugin updater -- every key is pushed
    after the backward and reduced in one flush (the reference's order,
    kvstore.py:116-120, train.py:210-223).  Executors bind lazily, at the
    first step / capture / ``execs`` access, so ``set_updater`` may come
    after construction.
    """

    def __init__(self, g: SymbolGraph, kv: KVStore, shard_shapes: Dict[str, tuple],
                 params0: Dict[str, np.ndarray], strategy: str = "both",
                 engine: Optional[Engine] = None, use_graph: bool = True, dense: str = "fp32",
                 overlap: Optional[bool] = None, split_target: int = 0,
                 hoist_wgrad: Optional[bool] = None):
        _check_graph(g)
        if overlap is None:  # env MGX_OVERLAP=0 turns it off (A/B measurements)
            import os
            overlap = os.environ.get("MGX_OVERLAP", "1") != "0"
        self.g, self.kv = g, kv
        # the step pushes every key back to back after the backward: reduce
        # them in one flush (the next pull, capture() or round_barrier)
        kv.bucket_flush = False
        self.engine = engine or kv.engine
        self.names = param_names(g)
        self.aux = aux_names(g)
        self._shard_shapes = dict(shard_shapes)
        arg_shapes, _ = infer_shape(g, shard_shapes)
        aux0 = init_aux(g, arg_shapes)
        for i, n in enumerate(self.names):
            kv.init(i, params0[n])
        self.workers = list(kv.local_workers)
        self.args: Dict[int, Dict[str, tmod.Tensor]] = {}
        self.grads: Dict[int, Dict[str, tmod.Tensor]] = {}
        self._execs: Dict[int, object] = {}
        for w in self.workers:
            args = {"data": tmod.zeros(shard_shapes["data"], engine=self.engine),
                    "label": tmod.zeros(shard_shapes["label"], engine=self.engine)}
            grads = {}
            for i, n in enumerate(self.names):
                args[n] = kv.weight_tensor(i, w)
                grads[n] = kv.grad_tensor(i, w)
            for n in self.aux:
                args[n] = tmod.from_host(arg_shapes[n], "float32", aux0[n], engine=self.engine)
            self.args[w], self.grads[w] = args, grads
        self._bind_opts = dict(strategy=strategy, use_graph=use_graph, dense=dense,
                               split_target=split_target)
        self._hoist = hoist_wgrad
        self._overlap = overlap
        self.embedded = False
        self._graph_exec = None

    def _ensure_bound(self) -> None:
        if self._execs:
            return
        kv = self.kv
        embed = (self._overlap and len(self.workers) == 1 and kv.mode == "sequential"
                 and kv._native != L.KV_AGG)
        for w in self.workers:
            rounds = kv.embedded_rounds(w) if embed else []
            # rounds that exchange over NVLink (several workers): issue the
            # weight gradients early so the rounds overlap the backward
            # (hoist_wgrad=True/False forces it: a chain-shaped net like
            # AlexNet gains on one GPU too, 2.42 -> 2.27 ms; Inception-BN
            # loses there, 4.68 -> 4.82 ms)
            cross = (bool(rounds) and kv.machines * kv.workers > 1
                     if self._hoist is None else bool(self._hoist))
            self._execs[w] = bind(self.g, self.args[w], {n: "write" for n in self.names},
                                  self.grads[w], engine=self.engine, rounds=rounds,
                                  hoist_wgrad=cross, **self._bind_opts)
            self.embedded = bool(rounds)
            if os.environ.get("MGX_PGO", "1") == "1":
                # schedule the lanes on measured instruction times
                self._execs[w].reschedule_from_profile(
                    keep=[self.args[w][n] for n in self.aux])

    @property
    def execs(self) -> Dict[int, object]:
        self._ensure_bound()
        return self._execs

    @property
    def plan_bytes(self) -> int:
        return self.execs[self.workers[0]].plan.total_internal_bytes

    # host-staged step (the reference's per-step sequence)
    def load(self, w: int, feats, labels) -> None:
        tmod.load_host(self.args[w]["data"], feats)
        tmod.load_host(self.args[w]["label"], labels)

    # ---------------------------------------------- prefetching input pipe

    def stage(self, w: int, feats, labels) -> None:
        """Start the host->device copy of worker w's NEXT batch (pinned torch
        tensors) on a copy stream, into a staging buffer, so it overlaps the
        step in flight (the input-pipeline prefetch).
        ``step(staged=True)`` consumes it."""
        import torch
        if not hasattr(self, "_stage"):
            self._copy_stream = torch.cuda.Stream(device=self.engine.device)
            self._stage = {}
        if w not in self._stage:
            dev = f"cuda:{self.engine.device}"
            self._stage[w] = (torch.empty(self.args[w]["data"].size, device=dev),
                              torch.empty(self.args[w]["label"].size, device=dev),
                              torch.cuda.Event())
        xs, ys, ev = self._stage[w]
        # the staging buffers are free once the previous step consumed them
        done = getattr(self, "_stage_done", {}).get(w)
        if done is not None:
            self._copy_stream.wait_event(done)
        with torch.cuda.stream(self._copy_stream):
            xs.copy_(feats.reshape(-1), non_blocking=True)
            ys.copy_(labels.reshape(-1), non_blocking=True)
            ev.record(self._copy_stream)

    def _consume_stage(self, w: int) -> None:
        import torch
        xs, ys, ev = self._stage[w]
        eng = self.engine
        data, label = self.args[w]["data"], self.args[w]["label"]

        def go():
            torch.cuda.ExternalStream(eng.stream_handle).wait_event(ev)
            L.call("mgx_copy", xs.data_ptr(), data.ptr, data.size, eng.stream_handle)
            L.call("mgx_copy", ys.data_ptr(), label.ptr, label.size, eng.stream_handle)
            done = torch.cuda.Event()
            done.record(torch.cuda.ExternalStream(eng.stream_handle))
            if not hasattr(self, "_stage_done"):
                self._stage_done = {}
            self._stage_done[w] = done

        eng.push(go, writes=[data.tag, label.tag], label="stage-consume")

    def run_worker(self, w: int, pull: bool = True) -> None:
        kv, ex = self.kv, self.execs[w]
        if pull:
            for i, n in enumerate(self.names):
                kv.pull(i, self.args[w][n], w)
        ex.forward()
        ex.backward()
        self._push(w)

    def _push(self, w: int) -> None:
        if self.embedded:
            # the rounds ran inside the backward program
            self.kv.note_embedded_round(w)
            return
        for i, n in enumerate(self.names):
            self.kv.push(i, self.grads[w][n], w)

    def step(self, shards: Optional[Dict[int, Tuple[np.ndarray, np.ndarray]]] = None,
             staged: bool = False) -> None:
        """pull -> (load) -> forward -> backward -> push, for every local
        worker.  staged=True takes the batch started by ``stage``."""
        self._ensure_bound()
        for w in self.workers:
            if not self.embedded:
                for i, n in enumerate(self.names):
                    self.kv.pull(i, self.args[w][n], w)
            # (rounds inside the backward: the executor's arguments ARE the
            # replicas the previous step's rounds wrote, in stream order --
            # the per-key pulls would be no-ops)
            if shards is not None:
                self.load(w, *shards[w])
            elif staged:
                self._consume_stage(w)
            ex = self._execs[w]
            ex.forward()
            ex.backward()
            self._push(w)
        # one fused reduce + update + broadcast round for all the step's keys
        # (nothing pending when the rounds ran inside the backward)
        with self.kv._lock:
            self.kv._flush_locked()

    def outputs(self, w: int) -> np.ndarray:
        return tmod.to_numpy(self.execs[w].outputs[0])

    # ---------------------------------------------------- whole-step graph

    def capture(self) -> None:
        """Capture one device-resident step (all workers) as a CUDA graph,
        instantiated natively with per-node priorities (the critical lane's
        kernels keep their stream priority).  Executors run eagerly inside
        the capture; the store's launches use a device-side barrier epoch,
        so replays stay correct."""
        self._ensure_bound()
        for ex in self.execs.values():
            ex._use_graph = False
        self.engine.activate()
        self.engine.synchronize()
        st = self.engine.stream_handle
        L.call("mgx_capture_begin", st)
        try:
            self.step()
            with self.kv._lock:
                self.kv._flush_locked()
        finally:
            h = ctypes.c_uint64()
            rc = L.lib().mgx_capture_end(st, ctypes.byref(h))
        L.check(rc, "mgx_capture_end")
        if self._graph_exec is not None:
            L.lib().mgx_graph_destroy(self._graph_exec)
        self._graph_exec = h.value

    def replay(self) -> None:
        if self._graph_exec is None:
            raise ArgumentError("capture() first")
        self.engine.activate()
        L.call("mgx_graph_launch", self._graph_exec, self.engine.stream_handle)

    def __del__(self):
        g = getattr(self, "_graph_exec", None)
        if g:
            try:
                L.lib().mgx_graph_destroy(g)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass


# ----------------------------------------------------------------- drivers

def train_local(g: SymbolGraph, data, cfg: SGDConfig, epochs: int, batch: int,
                strategy: str = "both", param_seed: int = 0, shuffle_seed: int = 0,
                prefetch: int = 2, engine: Optional[Engine] = None
                ) -> Tuple[TrainReport, Dict[str, np.ndarray]]:
    """Single-device SGD (train.py:97-153): forward, backward, then one
    fused SGD kernel per parameter."""
    _check_graph(g)
    engine = engine or default_engine()
    feats, labels = _load(data)
    it = BatchOrder(feats, labels, batch, seed=shuffle_seed)
    if it.batches_per_epoch < 1:
        raise ArgumentError("batch size exceeds the dataset")
    given = {"data": (batch,) + tuple(feats.shape[1:]), "label": (batch,)}
    arg_shapes, _ = infer_shape(g, given)
    params0 = init_params(g, arg_shapes, param_seed)
    names = param_names(g)
    args = {"data": tmod.zeros(given["data"], engine=engine),
            "label": tmod.zeros(given["label"], engine=engine)}
    for n in names:
        args[n] = tmod.from_host(arg_shapes[n], "float32", params0[n], engine=engine)
    for n, v in init_aux(g, arg_shapes).items():
        args[n] = tmod.from_host(arg_shapes[n], "float32", v, engine=engine)
    grads = {n: tmod.zeros(arg_shapes[n], engine=engine) for n in names}
    vel = {n: tmod.zeros(arg_shapes[n], engine=engine) for n in names}
    ex = bind(g, args, {n: "write" for n in names}, grads, strategy=strategy, engine=engine)
    report = TrainReport()
    last = engine.executed
    for epoch in range(epochs):
        t0 = time.perf_counter()
        losses, correct, seen = [], 0, 0
        for fb, lb in it.epoch(epoch):
            tmod.load_host(args["data"], fb)
            tmod.load_host(args["label"], lb)
            ex.forward()
            ex.backward()
            for n in names:
                sgd_step(args[n], grads[n], vel[n], vel[n], cfg)
            probs = tmod.to_numpy(ex.outputs[0]).astype(np.float64).reshape(batch, -1)
            losses.append(cross_entropy_mean(probs, lb))
            correct += int((probs.argmax(axis=1) == lb).sum())
            seen += batch
        engine.wait_all()
        report.append(epoch, float(np.mean(losses)), correct / seen, time.perf_counter() - t0,
                      ex.plan.total_internal_bytes, engine.executed - last)
        last = engine.executed
    params = {n: tmod.to_numpy(args[n]) for n in names}
    return report, params


def train_distributed(g: SymbolGraph, data, cfg: SGDConfig, epochs: int, batch: int,
                      machines: int = 1, workers: int = 1, mode: str = "sequential",
                      strategy: str = "both", param_seed: int = 0, shuffle_seed: int = 0,
                      tcp: Optional[str] = None, distributed: bool = False,
                      engine: Optional[Engine] = None, dense: str = "fp32"
                      ) -> Tuple[TrainReport, Dict[str, np.ndarray]]:
    """Data-parallel SGD through the device KVStore (train.py:158-270).

    ``distributed=False``: all M*W workers in this process on one device (the
    reference's threading model).  ``distributed=True``: one worker per
    torch.distributed rank (launch with torchrun, world size M*W).
    ``dense="bf16"`` runs the FC contractions on the tcgen05 tensor cores
    (bf16 operands, fp32 accumulation; tolerance-matched, not exact order)."""
    _check_graph(g)
    nworkers = machines * workers
    if batch % nworkers:
        raise ArgumentError(f"batch {batch} not divisible by {nworkers} workers")
    shard = batch // nworkers
    feats, labels = _load(data)
    it = BatchOrder(feats, labels, batch, seed=shuffle_seed)
    if it.batches_per_epoch < 1:
        raise ArgumentError("batch size exceeds the dataset")
    given = {"data": (shard,) + tuple(feats.shape[1:]), "label": (shard,)}
    arg_shapes, _ = infer_shape(g, given)
    params0 = init_params(g, arg_shapes, param_seed)
    engine = engine or default_engine()
    kv = KVStore(machines, workers, mode, engine=engine, tcp=tcp, distributed=distributed)
    try:
        step = DataParallelStep(g, kv, given, params0, strategy=strategy, engine=engine,
                                dense=dense)
        kv.set_updater(make_sgd_updater(cfg, scale=nworkers))
        report = TrainReport()
        last = engine.executed
        for epoch in range(epochs):
            t0 = time.perf_counter()
            losses, correct, seen = [], 0, 0
            for fb, lb in it.epoch(epoch):
                shards = {w: (fb[w * shard:(w + 1) * shard], lb[w * shard:(w + 1) * shard])
                          for w in step.workers}
                step.step(shards)
                for w in step.workers:
                    probs = step.outputs(w).astype(np.float64).reshape(shard, -1)
                    lw = shards[w][1]
                    losses.append(cross_entropy_mean(probs, lw))
                    correct += int((probs.argmax(axis=1) == lw).sum())
                    seen += shard
            kv.round_barrier()
            report.append(epoch, float(np.mean(losses)), correct / seen,
                          time.perf_counter() - t0, step.plan_bytes, engine.executed - last)
            last = engine.executed
        w0 = step.workers[0]
        params = {n: tmod.to_numpy(step.args[w0][n]) for n in step.names}
    finally:
        kv.close()
    return report, params
