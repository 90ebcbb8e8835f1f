"""TEST INFRASTRUCTURE ONLY.  Convolution-net oracle (configs 3-5).

PARITY UNPINNED BY REFERENCE: the reference (minigraph) has no Convolution,
Pooling, BatchNorm or Concat (SURVEY.md §0 fact 7, §8c "Ops with no
oracle").  This module restates MXNet's operator semantics in
float64 PyTorch-CPU (a different implementation from the device kernels) so
the sm_100a path can be checked against an independent computation:

* Convolution: channels-last data (B,H,W,C), weight (F,kh,kw,C), bias (F,);
* BatchNorm (training): batch mean and biased variance over all non-channel
  axes, y = (x-mean)/sqrt(var+eps)*gamma + beta, fix_gamma pins gamma to 1;
  moving = moving*momentum + batch*(1-momentum);
* Pooling: max ignores padding (first maximum gets the gradient), avg
  divides by the window area clipped to the padded extent
  (count_include_pad); global_pool averages the whole map;
* Concat along channels; Flatten of NHWC rows; FullyConnected x.W^T + b;
  SoftmaxOutput with gradient (p - onehot)/B (mean cross-entropy).

``run_graph`` interprets a bound symbol graph node by node and returns the
outputs and, through autograd, the parameter gradients.  ``bf16`` rounds a
tensor to bfloat16 (round-to-nearest-even) for emulating the tensor-core
operand rounding.  Nothing here is imported by the product.
"""

from __future__ import annotations

from typing import Dict, Tuple

import numpy as np


def _torch():
    import torch
    return torch


def bf16(t):
    """Round to bfloat16 and back to float64."""
    torch = _torch()
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def _pair(v):
    return (v, v) if isinstance(v, int) else (int(v[0]), int(v[1]))


def conv2d_nhwc(x, w, b, stride, pad):
    """x (B,H,W,C), w (F,kh,kw,C) -> (B,Ho,Wo,F)."""
    import torch.nn.functional as F
    y = F.conv2d(x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, stride=stride, padding=pad)
    return y.permute(0, 2, 3, 1)


class _Bf16Conv:
    """Convolution whose three contractions see bf16-rounded operands, like
    the device: forward bf16(x)*bf16(w); dX = bf16(dY) (*) bf16(w);
    dW = bf16(x) (*) bf16(dY) (float64 accumulation)."""

    @staticmethod
    def apply(x, w, b, stride, pad):
        torch = _torch()

        class F(torch.autograd.Function):
            @staticmethod
            def forward(ctx, x, w):
                xr, wr = bf16(x), bf16(w)
                ctx.save_for_backward(xr, wr)
                return conv2d_nhwc(xr, wr, None, stride, pad)

            @staticmethod
            def backward(ctx, dy):
                from torch.nn.grad import conv2d_input, conv2d_weight
                xr, wr = ctx.saved_tensors
                dyr = bf16(dy).permute(0, 3, 1, 2)
                xn, wn = xr.permute(0, 3, 1, 2), wr.permute(0, 3, 1, 2)
                dx = conv2d_input(xn.shape, wn, dyr, stride=stride, padding=pad)
                dw = conv2d_weight(xn, wn.shape, dyr, stride=stride, padding=pad)
                return dx.permute(0, 2, 3, 1), dw.permute(0, 2, 3, 1)

        y = F.apply(x, w)
        return y + b if b is not None else y


def batchnorm(x, gamma, beta, eps, fix_gamma):
    dims = tuple(range(x.dim() - 1))
    mean = x.mean(dim=dims)
    var = ((x - mean) ** 2).mean(dim=dims)
    g = 1.0 if fix_gamma else gamma
    return (x - mean) / (var + eps).sqrt() * g + beta, mean, var


def pool_nhwc(x, attrs):
    import torch.nn.functional as F
    torch = _torch()
    if attrs.get("global_pool", False):
        return x.mean(dim=(1, 2), keepdim=True)
    k = _pair(attrs["kernel"])
    s = _pair(attrs.get("stride", 1))
    p = _pair(attrs.get("pad", 0))
    ceil = attrs.get("pooling_convention", "valid") == "full"
    xn = x.permute(0, 3, 1, 2)
    if attrs.get("pool_type", "max") == "max":
        y = F.max_pool2d(xn, k, s, p, ceil_mode=ceil)
    else:
        y = F.avg_pool2d(xn, k, s, p, ceil_mode=ceil, count_include_pad=True)
    del torch
    return y.permute(0, 2, 3, 1)


class _Bf16FC:
    """FullyConnected whose three contractions see bf16-rounded operands like
    the device's bf16 dense mode (executor dense="bf16"): y = bf16(x)
    bf16(W)^T + b; dX = bf16(dY) bf16(W); dW = bf16(dY)^T bf16(x)."""

    @staticmethod
    def apply(x2, w, b):
        torch = _torch()

        class F(torch.autograd.Function):
            @staticmethod
            def forward(ctx, x2, w):
                xr, wr = bf16(x2), bf16(w)
                ctx.save_for_backward(xr, wr)
                return xr @ wr.T

            @staticmethod
            def backward(ctx, dy):
                xr, wr = ctx.saved_tensors
                dyr = bf16(dy)
                return dyr @ wr, dyr.T @ xr

        return F.apply(x2, w) + b


def run_graph(g, values: Dict[str, np.ndarray], wrt=(), bf16_operands: bool = False,
              bf16_fc: bool = False, dtype: str = "float64"
              ) -> Tuple[Dict[str, np.ndarray], Dict[str, np.ndarray], Dict[str, np.ndarray]]:
    """Forward (and, for a SoftmaxOutput head, backward) of ``g`` in float64.

    Returns (node outputs by name, gradients of ``wrt`` by name, updated
    BatchNorm moving statistics by name).  ``bf16_operands`` rounds every
    operand of the Convolution contractions (forward, data and weight
    gradients) to bf16 like the device does; ``bf16_fc`` does the same for
    FullyConnected (the device's dense="bf16" mode).  ``dtype="float32"``
    runs the same restatement in fp32 (bench.py's CPU baseline timing only;
    parity uses float64)."""
    torch = _torch()
    tdt = getattr(torch, dtype)
    env = {}
    leaves = {}
    aux_out = {}
    for name, v in values.items():
        t = torch.tensor(np.asarray(v), dtype=tdt)
        if name in wrt:
            t.requires_grad_(True)
        leaves[name] = t
    loss = None
    for n in g.topo_nodes():
        if n.is_variable:
            env[id(n)] = leaves[n.name]
            continue
        ins = [env[id(src)] for src, _ in n.inputs]
        a = n.attrs
        if n.op == "Convolution" and bf16_operands:
            y = _Bf16Conv.apply(ins[0], ins[1], ins[2] if len(ins) > 2 else None,
                                _pair(a.get("stride", 1)), _pair(a.get("pad", 0)))
        elif n.op == "Convolution":
            y = conv2d_nhwc(ins[0], ins[1], ins[2] if len(ins) > 2 else None,
                            _pair(a.get("stride", 1)), _pair(a.get("pad", 0)))
        elif n.op == "FullyConnected" and bf16_fc:
            y = _Bf16FC.apply(ins[0].reshape(ins[0].shape[0], -1), ins[1], ins[2])
        elif n.op == "FullyConnected":
            x2 = ins[0].reshape(ins[0].shape[0], -1)
            y = x2 @ ins[1].T + ins[2]
        elif n.op == "BatchNorm":
            y, mean, var = batchnorm(ins[0], ins[1], ins[2], float(a.get("eps", 1e-3)),
                                     a.get("fix_gamma", True))
            mom = float(a.get("momentum", 0.9))
            mm, mv = n.inputs[3][0].name, n.inputs[4][0].name
            aux_out[mm] = (ins[3] * mom + mean.detach() * (1 - mom)).numpy()
            aux_out[mv] = (ins[4] * mom + var.detach() * (1 - mom)).numpy()
        elif n.op == "Activation":
            y = {"relu": torch.relu, "tanh": torch.tanh, "sigmoid": torch.sigmoid}[a["act_type"]](ins[0])
        elif n.op == "Pooling":
            y = pool_nhwc(ins[0], a)
        elif n.op == "Concat":
            y = torch.cat(ins, dim=-1)
        elif n.op == "Flatten":
            y = ins[0].reshape(ins[0].shape[0], -1)
        elif n.op == "SoftmaxOutput":
            logits = ins[0]
            y = torch.softmax(logits, dim=1)
            lab = ins[1].detach().long()
            loss = torch.nn.functional.cross_entropy(logits, lab, reduction="mean")
        else:
            raise NotImplementedError(n.op)
        env[id(n)] = y
    outs = {n.name: env[id(n)].detach().numpy() for n in g.topo_nodes() if not n.is_variable}
    grads = {}
    if wrt and loss is not None:
        loss.backward()
        torch_zeros = torch.zeros_like
        grads = {k: (leaves[k].grad if leaves[k].grad is not None else torch_zeros(leaves[k]))
                 .detach().numpy() for k in wrt}
    return outs, grads, aux_out
