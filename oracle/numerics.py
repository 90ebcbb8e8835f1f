"""TEST INFRASTRUCTURE ONLY.  Numeric kernels of the reference, restated.

Reduction orders (pinned against the reference by tests/test_oracle_golden.py):
  * FC forward   det_matmul(x, w.T)  -> numpy pairwise over K      (kernels.py:20-29, ops.py:102-106)
  * FC dX        det_matmul(og, w)   -> sequential over H          (ops.py:111-112)
  * FC dW, db    tree over the batch                              (kernels.py:32-47, ops.py:113-116)
  * softmax      exp(x - max) / pairwise row sum                  (kernels.py:68-76)
  * KV merge     tree over workers (ascending id), then machines  (kvstore.py:335, :400)
  * SGD updater  g*f32(1/scale); tmp=g+w*wd; v=v*mom; v=v+tmp*(-eta); w=w+v*1  (optim.py:53-78)
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


# ------------------------------------------------------ numpy pairwise sum
# numpy's pairwise_sum (the order np.add.reduce uses over a contiguous axis),
# restated literally for pinning; `pairwise_rows` is the vectorised form.

def pairwise_sum(a: np.ndarray) -> np.float32:
    """Literal restatement for one 1-D float32 vector."""
    n = a.shape[0]
    if n < 8:
        res = F32(0.0)
        for i in range(n):
            res = F32(res + a[i])
        return res
    if n <= 128:
        r = [F32(a[j]) for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] = F32(r[j] + a[i + j])
            i += 8
        res = F32(F32(F32(r[0] + r[1]) + F32(r[2] + r[3])) +
                  F32(F32(r[4] + r[5]) + F32(r[6] + r[7])))
        while i < n:
            res = F32(res + a[i])
            i += 1
        return res
    half = n // 2
    half -= half % 8
    return F32(pairwise_sum(a[:half]) + pairwise_sum(a[half:]))


def pairwise_rows(prod: np.ndarray) -> np.ndarray:
    """Pairwise sum along the last (contiguous) axis of a float32 array,
    vectorised over the leading axes (same algorithm as pairwise_sum)."""
    prod = np.ascontiguousarray(prod, dtype=F32)
    n = prod.shape[-1]
    if n < 8:
        res = np.zeros(prod.shape[:-1], F32)
        for i in range(n):
            res = (res + prod[..., i]).astype(F32)
        return res
    if n <= 128:
        r = [prod[..., j].copy() for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] = (r[j] + prod[..., i + j]).astype(F32)
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        res = res.astype(F32)
        while i < n:
            res = (res + prod[..., i]).astype(F32)
            i += 1
        return res
    half = n // 2
    half -= half % 8
    return (pairwise_rows(prod[..., :half]) + pairwise_rows(prod[..., half:])).astype(F32)


# -------------------------------------------------------------- contractions

def fc_forward(x2: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """pairwise_k(x2[m,k]*w[n,k]) then + b, separately rounded (ops.py:102-106)."""
    prod = (x2[:, None, :] * w[None, :, :]).astype(F32)       # (M, N, K), K contiguous
    return (pairwise_rows(prod) + b).astype(F32)


def seq_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """sequential_k(a[m,k]*b[k,n]) from the first product (kernels.py:20-29
    with contiguous b: the reduced axis is not innermost)."""
    acc = (a[:, 0:1] * b[0:1, :]).astype(F32)
    for k in range(1, a.shape[1]):
        acc = (acc + (a[:, k:k + 1] * b[k:k + 1, :]).astype(F32)).astype(F32)
    return acc


def tree_sum(a: np.ndarray) -> np.ndarray:
    """Balanced power-of-two tree along axis 0 (kernels.py:32-42)."""
    n = a.shape[0]
    if n == 1:
        return a[0].astype(F32).copy()
    half = 1 << ((n - 1).bit_length() - 1)
    return (tree_sum(a[:half]) + tree_sum(a[half:])).astype(F32)


def tree_outer(dy: np.ndarray, x: np.ndarray) -> np.ndarray:
    """tree_b(dy[b,:,None]*x[b,None,:]) (kernels.py:45-47)."""
    return tree_sum((dy[:, :, None] * x[:, None, :]).astype(F32))


# --------------------------------------------------------------- activations

def relu(x):
    return np.maximum(x, F32(0))


def relu_backward(y, og):
    """og * (y > 0) (ops.py:140)."""
    return (og * (y > 0)).astype(F32)


def sigmoid(x):
    return (F32(1.0) / (F32(1.0) + np.exp(-x))).astype(F32)


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """e = exp(x - rowmax); e / pairwise_rowsum(e) (kernels.py:68-76)."""
    e = np.exp((x - np.max(x, axis=1, keepdims=True)).astype(F32)).astype(F32)
    return (e / pairwise_rows(e)[:, None]).astype(F32)


def softmax_backward(p: np.ndarray, label: np.ndarray) -> np.ndarray:
    """(p - onehot(int64(label))) / f32(B) (ops.py:188-196)."""
    bsz, classes = p.shape
    oh = np.zeros_like(p)
    oh[np.arange(bsz), label.astype(np.int64)] = 1
    return np.true_divide((p - oh).astype(F32), F32(bsz)).astype(F32)


# ------------------------------------------------------------------- update

def axpy(alpha, x, y):
    """y + x*alpha, two roundings (kernels.py:50-53)."""
    return (y + (x * F32(alpha)).astype(F32)).astype(F32)


def sgd_update(w, g, v, eta, momentum, weight_decay):
    """sgd_arrays (optim.py:53-61): returns new (w, v)."""
    tmp = axpy(weight_decay, w, g.astype(F32))
    v = (v * F32(momentum)).astype(F32)
    v = axpy(-eta, tmp, v)
    w = axpy(1.0, v, w)
    return w, v


def kv_updater(w, incoming, v, eta, momentum, weight_decay, scale):
    """make_sgd_updater (optim.py:64-78): g = incoming * f32(1/scale)."""
    g = (incoming * F32(1.0 / scale)).astype(F32)
    return sgd_update(w, g, v, eta, momentum, weight_decay)


def kv_merge(grads, machines: int = 1):
    """Level-1 tree over each machine's workers (ascending worker id), then
    level-2 tree over machine aggregates (kvstore.py:335, :400)."""
    grads = [np.asarray(g, F32) for g in grads]
    w = len(grads) // machines
    aggs = [tree_sum(np.stack(grads[m * w:(m + 1) * w])) for m in range(machines)]
    return tree_sum(np.stack(aggs))
