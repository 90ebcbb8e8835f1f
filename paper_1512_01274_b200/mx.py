"""MXNet-style aliases over the reference-shaped API.

    from paper_1512_01274_b200 import mx
    net = mx.sym.Variable("data")
    net = mx.sym.FullyConnected(data=net, num_hidden=128, name="fc1")
    net = mx.sym.Activation(data=net, act_type="relu", name="act1")
    net = mx.sym.SoftmaxOutput(data=mx.sym.FullyConnected(data=net, num_hidden=10, name="out"),
                               name="softmax")
    ex = net.simple_bind(mx.gpu(0), grad_req="write", data=(100, 784))
    kv = mx.kv.create("device", num_devices=2)
    kv.set_optimizer(mx.optimizer.SGD(learning_rate=0.05, momentum=0.9, wd=1e-4,
                                      rescale_grad=1.0 / 2))

Every alias is a thin mapping onto symbol.apply / bind / KVStore /
make_sgd_updater; nothing here computes.  Operators: Variable,
FullyConnected, Convolution, Activation, BatchNorm, Pooling, Concat,
Flatten, SoftmaxOutput, Group; keyword attributes are MXNet's names.

``mx.kv.create('device')`` placement: the store's
workers are data-parallel replicas.
* Under torch.distributed with world size > 1 (torchrun, one process per
  GPU -- the B200 layout): one worker per rank, each on its own GPU; the
  fused reduce + update + broadcast runs over NVLink peer memory.  Same as
  ``'dist_device_sync'``.
* In a single process: ``num_devices`` workers share the process's GPU (the
  reference's threading model, train.py:182-243: W workers in one process);
  pass ``ctx`` contexts that are all the same GPU, or none.  One process
  never drives several GPUs: a list of contexts on different GPUs raises.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

from . import symbol as _sym
from . import tensor as _t
from .engine import Engine, default_engine
from .errors import ArgumentError
from .executor import bind as _bind
from .kvstore import KVStore
from .optim import SGDConfig, make_sgd_updater

AUX_SUFFIXES = ("_moving_mean", "_moving_var")


class Context:
    def __init__(self, device_type: str, device_id: int = 0):
        self.device_type, self.device_id = device_type, device_id

    def __repr__(self):
        return f"{self.device_type}({self.device_id})"


def gpu(device_id: int = 0) -> Context:
    return Context("gpu", device_id)


class Symbol:
    """Wraps a SymbolGraph with MXNet's method names."""

    def __init__(self, graph: _sym.SymbolGraph):
        self.graph = graph

    def list_arguments(self) -> List[str]:
        return self.graph.list_arguments()

    def infer_shape(self, **shapes):
        args, named = _sym.infer_shape(self.graph, shapes)
        outs = [named[n.name] for n, _ in self.graph.outputs]
        return [args[a] for a in self.list_arguments()], outs, []

    def list_auxiliary_states(self) -> List[str]:
        """BatchNorm moving statistics (arguments here, never gradients)."""
        return [n for n in self.list_arguments() if n.endswith(AUX_SUFFIXES)]

    def simple_bind(self, ctx: Optional[Context] = None, grad_req="write", engine=None,
                    dense: str = "fp32", **shapes):
        """Infer shapes, allocate argument/gradient tensors on the device,
        and bind (symbol.infer_shape + tensor.zeros + executor.bind).  The
        inputs named in ``shapes`` and the auxiliary states get no gradient;
        moving variances start at one (MXNet's aux initialisation)."""
        engine = engine or _engine_for(ctx)
        args_shapes, _ = _sym.infer_shape(self.graph, shapes)
        names = self.list_arguments()
        aux = set(self.list_auxiliary_states())
        arg_dict = {n: (_t.ones if n.endswith("_moving_var") else _t.zeros)(args_shapes[n],
                                                                             engine=engine)
                    for n in names}
        if isinstance(grad_req, str):
            reqs = {n: (grad_req if n not in shapes and n not in aux else "null") for n in names}
        else:
            reqs = dict(grad_req)
        reqs = {n: ("none" if r == "null" else r) for n, r in reqs.items()}
        grad_dict = {n: _t.zeros(args_shapes[n], engine=engine)
                     for n, r in reqs.items() if r != "none"}
        ex = _bind(self.graph, arg_dict, reqs, grad_dict, engine=engine, dense=dense)
        return _MXExecutor(ex, arg_dict, grad_dict, aux)

    def __repr__(self):
        return f"<Symbol {self.graph!r}>"


class _MXExecutor:
    def __init__(self, ex, arg_dict, grad_dict, aux=()):
        self._ex = ex
        self.arg_dict = arg_dict
        self.grad_dict = grad_dict
        self.aux_dict = {n: arg_dict[n] for n in arg_dict if n in aux}
        self.arg_arrays = list(arg_dict.values())
        self.grad_arrays = list(grad_dict.values())

    @property
    def outputs(self):
        return self._ex.outputs

    def forward(self, is_train: bool = True, **feed):
        for k, v in feed.items():
            _t.load_host(self.arg_dict[k], v)
        return self._ex.forward()

    def backward(self):
        self._ex.backward()


_engines: Dict[int, Engine] = {}


def _engine_for(ctx: Optional[Context]) -> Engine:
    if ctx is None:
        return default_engine()
    if ctx.device_type != "gpu":
        raise ArgumentError("only gpu contexts exist (no CPU fallback)")
    if ctx.device_id not in _engines:
        _engines[ctx.device_id] = Engine(device=ctx.device_id)
    return _engines[ctx.device_id]


def _apply(op: str, data, name, attrs, extra: Sequence = ()):
    ins = [data.graph] + [e.graph for e in extra if e is not None]
    return Symbol(_sym.apply(op, attrs, ins, name=name))


def _attrs(**kw):
    """MXNet keyword attributes (None = not given)."""
    return {k: (tuple(v) if isinstance(v, list) else v) for k, v in kw.items() if v is not None}


class sym:  # noqa: N801 - mirrors mx.sym
    @staticmethod
    def Variable(name: str, **attrs) -> Symbol:  # noqa: N802
        return Symbol(_sym.variable(name, **attrs))

    @staticmethod
    def FullyConnected(data: Symbol, num_hidden: int, name: Optional[str] = None,  # noqa: N802
                       weight: Optional[Symbol] = None, bias: Optional[Symbol] = None) -> Symbol:
        return _apply("FullyConnected", data, name, {"num_hidden": int(num_hidden)}, (weight, bias))

    @staticmethod
    def Activation(data: Symbol, act_type: str, name: Optional[str] = None) -> Symbol:  # noqa: N802
        return _apply("Activation", data, name, {"act_type": act_type})

    @staticmethod
    def SoftmaxOutput(data: Symbol, name: Optional[str] = None,  # noqa: N802
                      label: Optional[Symbol] = None) -> Symbol:
        return _apply("SoftmaxOutput", data, name, {}, (label,))

    @staticmethod
    def Flatten(data: Symbol, name: Optional[str] = None) -> Symbol:  # noqa: N802
        return _apply("Flatten", data, name, {})

    @staticmethod
    def Convolution(data: Symbol, kernel, num_filter: int, stride=None, pad=None,  # noqa: N802
                    no_bias: Optional[bool] = None, name: Optional[str] = None,
                    weight: Optional[Symbol] = None, bias: Optional[Symbol] = None,
                    **kw) -> Symbol:
        """Channels-last convolution (data (B,H,W,C), weight (F,kh,kw,C))."""
        attrs = _attrs(kernel=kernel, num_filter=int(num_filter), stride=stride, pad=pad,
                       no_bias=no_bias, **kw)
        return _apply("Convolution", data, name, attrs, (weight, bias))

    @staticmethod
    def BatchNorm(data: Symbol, eps: Optional[float] = None,  # noqa: N802
                  momentum: Optional[float] = None, fix_gamma: Optional[bool] = None,
                  name: Optional[str] = None, gamma: Optional[Symbol] = None,
                  beta: Optional[Symbol] = None, **kw) -> Symbol:
        """Training-mode BatchNorm; moving statistics are the auxiliary
        inputs ``<name>_moving_mean`` / ``<name>_moving_var``."""
        attrs = _attrs(eps=eps, momentum=momentum, fix_gamma=fix_gamma, **kw)
        return _apply("BatchNorm", data, name, attrs, (gamma, beta))

    @staticmethod
    def Pooling(data: Symbol, kernel=None, pool_type: Optional[str] = None,  # noqa: N802
                stride=None, pad=None, global_pool: Optional[bool] = None,
                pooling_convention: Optional[str] = None, name: Optional[str] = None) -> Symbol:
        attrs = _attrs(kernel=kernel, pool_type=pool_type, stride=stride, pad=pad,
                       global_pool=global_pool, pooling_convention=pooling_convention)
        return _apply("Pooling", data, name, attrs)

    @staticmethod
    def Concat(*data: Symbol, dim: Optional[int] = None, name: Optional[str] = None,  # noqa: N802
               num_args: Optional[int] = None) -> Symbol:
        attrs = _attrs(dim=dim, num_args=num_args if num_args is not None else len(data))
        return Symbol(_sym.apply("Concat", attrs, [d.graph for d in data], name=name))

    @staticmethod
    def Group(*symbols: Symbol) -> Symbol:  # noqa: N802
        return Symbol(_sym.group(*[s.graph for s in symbols]))


class optimizer:  # noqa: N801
    class SGD:
        def __init__(self, learning_rate: float = 0.01, momentum: float = 0.0, wd: float = 0.0,
                     rescale_grad: float = 1.0):
            self.learning_rate, self.momentum, self.wd = learning_rate, momentum, wd
            self.rescale_grad = rescale_grad


class _MXKVStore:
    """mx.kv store: one worker per device list entry (single process) or
    one per rank (dist_device_sync)."""

    def __init__(self, kind: str, num_devices: int, engine: Optional[Engine]):
        import torch.distributed as dist
        multi_rank = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        # 'device' under a multi-rank process group is the one-GPU-per-rank
        # store; in a single process its workers share the process's GPU
        distributed = kind.startswith("dist") or (kind == "device" and multi_rank)
        if distributed:
            num_devices = dist.get_world_size()
        self.type = kind
        self._kv = KVStore(1, num_devices, engine=engine, distributed=distributed)
        self.num_workers = num_devices
        self.rank = self._kv.rank

    def init(self, key, value):
        keys, vals = _as_lists(key, value)
        for k, v in zip(keys, vals):
            self._kv.init(k, v[0] if isinstance(v, (list, tuple)) else v)

    def push(self, key, value):
        keys, vals = _as_lists(key, value)
        for k, v in zip(keys, vals):
            grads = v if isinstance(v, (list, tuple)) else [v]
            workers = self._kv.local_workers
            for w, gr in zip(workers, grads):
                self._kv.push(k, gr, w)

    def pull(self, key, out):
        keys, outs = _as_lists(key, out)
        for k, o in zip(keys, outs):
            targets = o if isinstance(o, (list, tuple)) else [o]
            for w, t in zip(self._kv.local_workers, targets):
                self._kv.pull(k, t, w)

    def set_optimizer(self, opt: "optimizer.SGD"):
        scale = round(1.0 / opt.rescale_grad) if opt.rescale_grad else 1
        cfg = SGDConfig(eta=opt.learning_rate, momentum=opt.momentum, weight_decay=opt.wd)
        self._kv.set_updater(make_sgd_updater(cfg, scale=max(1, scale)))

    def set_updater(self, fn):
        self._kv.set_updater(fn)

    def close(self):
        self._kv.close()


def _as_lists(key, value):
    if isinstance(key, (list, tuple)):
        return list(key), list(value)
    return [key], [value]


class kv:  # noqa: N801
    @staticmethod
    def create(name: str = "local", num_devices: int = 1, engine: Optional[Engine] = None,
               ctx: Optional[Sequence[Context]] = None) -> _MXKVStore:
        if name not in ("local", "device", "dist_sync", "dist_device_sync"):
            raise ArgumentError(f"unknown kvstore type {name!r}")
        if ctx:
            if len({c.device_id for c in ctx}) > 1:
                raise ArgumentError("one process drives one GPU: launch one rank per GPU "
                                    "(torchrun) for a multi-GPU store")
            num_devices = len(ctx)
            engine = engine or _engine_for(ctx[0])
        return _MXKVStore(name, num_devices, engine)
