"""TEST INFRASTRUCTURE ONLY.  The data-parallel training step, restated.

A plain-numpy restatement of ``train_distributed`` for relu MLPs ending in
SoftmaxOutput (train.py:57-85, 158-270 with executor.py's node order): every
worker takes a contiguous row shard of each global batch, computes
forward/backward with the reference's reduction orders (oracle.numerics),
and each key is merged with the two-level tree and updated by the KV
updater.  Also restates the seeded batch order (dataiter.py:28-46) and
parameter init (train.py:74-85).
"""

from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import numerics as nm

F32 = np.float32
_M64 = (1 << 64) - 1


def splitmix64(seed: int):
    """dataiter.py:28-36"""
    s = seed & _M64
    while True:
        s = (s + 0x9E3779B97F4A7C15) & _M64
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        yield z ^ (z >> 31)


def shuffled_order(n: int, seed: int) -> List[int]:
    """dataiter.py:39-46: Fisher-Yates driven by splitmix64."""
    perm = list(range(n))
    rng = splitmix64(seed)
    for i in range(n - 1, 0, -1):
        j = next(rng) % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def mlp_param_names(hidden: Sequence[int]) -> List[str]:
    names = []
    for i in range(1, len(hidden) + 1):
        names += [f"fc{i}_weight", f"fc{i}_bias"]
    return names + ["out_weight", "out_bias"]


def mlp_param_shapes(hidden: Sequence[int], classes: int, dim: int) -> Dict[str, tuple]:
    shapes, prev = {}, dim
    for i, h in enumerate(hidden, 1):
        shapes[f"fc{i}_weight"], shapes[f"fc{i}_bias"] = (h, prev), (h,)
        prev = h
    shapes["out_weight"], shapes["out_bias"] = (classes, prev), (classes,)
    return shapes


def init_params(hidden, classes, dim, seed) -> Dict[str, np.ndarray]:
    """train.py:74-85: randn*0.1 weights in parameter order, zero biases."""
    rs = np.random.RandomState(seed)
    shapes = mlp_param_shapes(hidden, classes, dim)
    out = {}
    for n in mlp_param_names(hidden):
        if n.endswith("_bias"):
            out[n] = np.zeros(shapes[n], F32)
        else:
            out[n] = (rs.randn(*shapes[n]) * 0.1).astype(F32)
    return out


def mlp_forward_backward(params: Dict[str, np.ndarray], hidden: Sequence[int], x: np.ndarray,
                         label: np.ndarray) -> Tuple[np.ndarray, Dict[str, np.ndarray]]:
    """One worker's forward + backward; returns (softmax output, grads)."""
    layers = [f"fc{i}" for i in range(1, len(hidden) + 1)] + ["out"]
    inputs, outs = [], []
    h = x.astype(F32)
    for li, name in enumerate(layers):
        inputs.append(h)
        z = nm.fc_forward(h, params[f"{name}_weight"], params[f"{name}_bias"])
        h = nm.relu(z) if li < len(layers) - 1 else z
        outs.append(h)
    p = nm.softmax_rows(h)
    grads = {}
    d = nm.softmax_backward(p, label)
    for li in range(len(layers) - 1, -1, -1):
        name = layers[li]
        grads[f"{name}_weight"] = nm.tree_outer(d, inputs[li])
        grads[f"{name}_bias"] = nm.tree_sum(d)
        if li > 0:  # the data gradient is never requested (pruned)
            dx = nm.seq_matmul(d, params[f"{name}_weight"])
            d = nm.relu_backward(outs[li - 1], dx)
    return p, grads


def train_distributed(hidden: Sequence[int], classes: int, feats: np.ndarray,
                      labels: np.ndarray, eta: float, momentum: float, weight_decay: float,
                      epochs: int, batch: int, machines: int = 1, workers: int = 1,
                      param_seed: int = 0, shuffle_seed: int = 0, max_steps: int = None
                      ) -> Tuple[Dict[str, np.ndarray], List[np.ndarray]]:
    """Restatement of train_distributed (sequential mode).  Returns the final
    parameters and every step's worker-0 softmax output."""
    nw = machines * workers
    shard = batch // nw
    params = init_params(hidden, classes, feats.shape[1], param_seed)
    names = mlp_param_names(hidden)
    vel = {n: np.zeros_like(params[n]) for n in names}
    probs0 = []
    steps = 0
    for epoch in range(epochs):
        order = np.asarray(shuffled_order(len(feats), shuffle_seed + epoch), np.int64)
        for b in range(len(feats) // batch):
            if max_steps is not None and steps >= max_steps:
                return params, probs0
            rows = order[b * batch:(b + 1) * batch]
            per_worker = []
            for w in range(nw):
                r = rows[w * shard:(w + 1) * shard]
                p, g = mlp_forward_backward(params, hidden, feats[r], labels[r])
                per_worker.append(g)
                if w == 0:
                    probs0.append(p)
            for n in names:
                total = nm.kv_merge([g[n] for g in per_worker], machines)
                params[n], vel[n] = nm.kv_updater(params[n], total, vel[n], eta, momentum,
                                                  weight_decay, nw)
            steps += 1
    return params, probs0


def train_local(hidden, classes, feats, labels, eta, momentum, weight_decay, epochs, batch,
                param_seed=0, shuffle_seed=0, max_steps=None):
    """Restatement of train_local (train.py:97-153): sgd_step per parameter."""
    params = init_params(hidden, classes, feats.shape[1], param_seed)
    names = mlp_param_names(hidden)
    vel = {n: np.zeros_like(params[n]) for n in names}
    steps = 0
    for epoch in range(epochs):
        order = np.asarray(shuffled_order(len(feats), shuffle_seed + epoch), np.int64)
        for b in range(len(feats) // batch):
            if max_steps is not None and steps >= max_steps:
                return params
            r = order[b * batch:(b + 1) * batch]
            _p, g = mlp_forward_backward(params, hidden, feats[r], labels[r])
            for n in names:
                params[n], vel[n] = nm.sgd_update(params[n], g[n], vel[n], eta, momentum,
                                                  weight_decay)
            steps += 1
    return params


# ------------------------------------------------------------- synthetic data

def cfg1_data(n: int, seed: int = 0, dim: int = 784, classes: int = 10):
    """BASELINE.md §2 config-1 inputs: features RandomState(seed).rand(N, 784)
    float32, labels randint(0, 10) from the same stream."""
    rs = np.random.RandomState(seed)
    feats = rs.rand(n, dim).astype(F32)
    labels = rs.randint(0, classes, n).astype(F32)
    return feats, labels
