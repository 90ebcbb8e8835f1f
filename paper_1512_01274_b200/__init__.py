"""B200-native data-parallel training step (arXiv 1512.01274 / minigraph).

Drop-in for the reference's hot path: symbolic graphs, the static memory
planner, executors (forward/backward) and the two-level KVStore, running
hand-written sm_100a kernels through the C-ABI in ``libmgx.so``
(include/mgx.h).  Host-side graph construction and planning mirror the
reference API; all numeric work is on the GPU (no CPU fallback).

Importing the package does not touch CUDA; device objects (engines,
tensors, executors, stores) need a GPU and the built library.
"""

from . import errors, ops, symbol
from .errors import (ArgumentError, CorruptRecordError, GraphParseError, InferenceError,
                     KVStoreError, LifecycleError, MinigraphError, OperationFailed, PlanError,
                     RecordParseError, StateError)
from .symbol import (SymbolGraph, apply, gradient, group, infer_shape, load, reset_names, save,
                     to_dot, variable)

__version__ = "0.1.0"


def __getattr__(name):
    # device-facing modules load lazily so `import paper_1512_01274_b200`
    # works on a CPU-only host (graph building, planning, tests)
    import importlib
    lazy = {
        "planner": "planner", "tensor": "tensor", "engine": "engine", "executor": "executor",
        "kvstore": "kvstore", "optim": "optim", "train": "train", "mx": "mx", "data": "data",
    }
    if name in lazy:
        return importlib.import_module(f".{lazy[name]}", __name__)
    attrs = {
        "plan_memory": ("planner", "plan_memory"), "prune": ("planner", "prune"),
        "Engine": ("engine", "Engine"), "Tensor": ("tensor", "Tensor"),
        "Executor": ("executor", "Executor"), "bind": ("executor", "bind"),
        "KVStore": ("kvstore", "KVStore"), "SGDConfig": ("optim", "SGDConfig"),
        "sgd_step": ("optim", "sgd_step"), "make_sgd_updater": ("optim", "make_sgd_updater"),
        "train_local": ("train", "train_local"), "train_distributed": ("train", "train_distributed"),
        "TrainReport": ("train", "TrainReport"),
    }
    if name in attrs:
        mod, attr = attrs[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)
