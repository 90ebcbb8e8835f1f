"""Shared fixtures.  `-m "not gpu"` runs on a CPU-only host; `-m gpu` tests
need a B200 and the built libmgx.so (they fail loudly without it)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libmgx.so")


@pytest.fixture(autouse=True)
def _fresh_names():
    from paper_1512_01274_b200 import symbol
    symbol.reset_names()
    yield


@pytest.fixture(scope="session")
def ops_golden():
    return np.load(os.path.join(GOLDEN, "ops_golden.npz"))


@pytest.fixture(scope="session")
def kv_golden():
    return np.load(os.path.join(GOLDEN, "kv_golden.npz"))


@pytest.fixture(scope="session")
def train_golden():
    return np.load(os.path.join(GOLDEN, "train_golden.npz"))


@pytest.fixture(scope="session")
def plans_golden():
    with open(os.path.join(GOLDEN, "plans_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test on a host without CUDA")
    from paper_1512_01274_b200 import _lib
    _lib.lib()  # loud failure if the native library is missing
    return torch


@pytest.fixture()
def engine(cuda):
    from paper_1512_01274_b200.engine import Engine
    eng = Engine(device=0)
    yield eng
    eng.close()


def random_dag(seed: int, max_ops: int = 12):
    """Restatement of the reference's test generator (tests/conftest.py:37-85)
    over this package's API: shape-preserving random graphs on (4, 4)."""
    from paper_1512_01274_b200 import symbol
    rng = np.random.RandomState(seed)
    pool, feed = [], {}
    for v in range(rng.randint(1, 4)):
        pool.append(symbol.variable(f"x{v}"))
        feed[f"x{v}"] = rng.randn(4, 4).astype(np.float32)
    for _ in range(rng.randint(1, max_ops + 1)):
        kind = rng.randint(0, 6)
        if kind in (0, 1, 5):
            a, b = pool[rng.randint(len(pool))], pool[rng.randint(len(pool))]
            op = {0: "ElementwiseAdd", 1: "ElementwiseMul", 5: "MatMul"}[kind]
            pool.append(symbol.apply(op, {}, [a, b]))
        elif kind in (2, 3):
            a = pool[rng.randint(len(pool))]
            op = "ScalarAdd" if kind == 2 else "ScalarMul"
            pool.append(symbol.apply(op, {"value": float(rng.randn())}, [a]))
        else:
            a = pool[rng.randint(len(pool))]
            act = "relu" if rng.randint(2) else "sigmoid"
            pool.append(symbol.apply("Activation", {"act_type": act}, [a]))
    used = set()
    for g in pool:
        for node in g.topo_nodes():
            for src, _ in node.inputs:
                used.add(id(src))
    outs = [g for g in pool if not g.outputs[0][0].is_variable and id(g.outputs[0][0]) not in used]
    extra = [g for g in pool if not g.outputs[0][0].is_variable]
    if extra:
        outs.append(extra[rng.randint(len(extra))])
    graph = symbol.group(*outs)
    return graph, {k: v for k, v in feed.items() if k in graph.list_arguments()}
