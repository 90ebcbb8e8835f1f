"""Convolution-net operators: Convolution, Pooling, BatchNorm, Concat.

The reference registers no such operators (ops.py:127-527),
so these follow MXNet's operator semantics (arXiv 1512.01274 §2, the paper's
Inception-BN/AlexNet experiments) behind the reference's plugin surface
(``OperatorDef``, ops.py:23-41): shape inference, ``forward``/``backward``,
``backward_uses`` roles, plus native lowerings to ``mgx_instr`` records.

Layout is channels-last (MXNet's ``layout='NHWC'``): data (B, H, W, C),
convolution weight (num_filter, kh, kw, C), per-channel parameters (C,).
Every 4-D activation is therefore an [B*H*W, C] row-major matrix, which is
what the tensor-core GEMMs and the per-channel reductions want.

Convolutions always run on the tcgen05 tensor cores with bf16 operand copies
and fp32 accumulation (tolerance path; there is no exact-order reference to
match).  The bf16 copies a backward pass needs (im2col of the input, the
weight, the output gradient) are made once per step and shared between the
forward and the sibling backward nodes through the lowering context memo.
"""

from __future__ import annotations

import os

from math import prod
from typing import Optional

from . import _lib as L
from .errors import ArgumentError, InferenceError
from .ops import OperatorDef, View, _fill, _native_backward, _native_forward, _need, current_ctx
from .ops import instr, register


def _pair(v, what: str) -> tuple:
    if isinstance(v, int):
        return (v, v)
    if isinstance(v, (tuple, list)) and len(v) == 2 and all(isinstance(x, int) for x in v):
        return (int(v[0]), int(v[1]))
    raise InferenceError(f"{what} must be an int or a pair of ints, got {v!r}")


def _pad8(n: int) -> int:
    return -(-int(n) // 8) * 8


def _check_layout(attrs, op):
    lay = attrs.get("layout", "NHWC")
    if lay != "NHWC":
        raise InferenceError(f"{op}: only layout='NHWC' is implemented (channels-last), got {lay!r}")


def _geom(shape, kernel, stride, pad) -> list:
    b, h, w, c = shape
    return [b, h, w, c, (kernel[0] << 16) | kernel[1], (stride[0] << 16) | stride[1],
            (pad[0] << 16) | pad[1]]


_PAIR = ((int, tuple, list), False)

# ------------------------------------------------------------- Convolution


def _conv_params(attrs):
    k = _pair(attrs["kernel"], "kernel")
    s = _pair(attrs.get("stride", 1), "stride")
    p = _pair(attrs.get("pad", 0), "pad")
    if attrs.get("num_group", 1) != 1:
        raise InferenceError("Convolution: num_group != 1 is not implemented")
    if _pair(attrs.get("dilate", 1), "dilate") != (1, 1):
        raise InferenceError("Convolution: dilation is not implemented")
    return k, s, p


def _conv_out(h, w, k, s, p):
    ho, wo = (h + 2 * p[0] - k[0]) // s[0] + 1, (w + 2 * p[1] - k[1]) // s[1] + 1
    if ho <= 0 or wo <= 0:
        raise InferenceError(f"Convolution: window {k} larger than padded input {(h, w)}")
    return ho, wo


def _conv_infer(shapes, attrs):
    _check_layout(attrs, "Convolution")
    data = _need(shapes[0], "Convolution", "data")
    if len(data) != 4:
        raise InferenceError("Convolution: data must be (batch, height, width, channels)")
    b, h, w, c = data
    k, s, p = _conv_params(attrs)
    f = attrs["num_filter"]
    ho, wo = _conv_out(h, w, k, s, p)
    filled = [tuple(data), _fill(shapes[1], (f, k[0], k[1], c), "weight")]
    if not attrs.get("no_bias", False):
        filled.append(_fill(shapes[2], (f,), "bias"))
    return filled, [(b, ho, wo, f)]


def _conv_inputs(attrs):
    return ("data", "weight") if attrs.get("no_bias", False) else ("data", "weight", "bias")


def _cast_rows(src: View, rows: int, cols: int, dst: int, ld: int):
    return instr(L.OP_CAST_BF16, [src.ptr, dst], [rows, cols, cols, rows, ld, 0])


def _gemm(a: int, lda: int, a_mn: bool, b: int, ldb: int, b_mn: bool, c: int, ldc: int,
          m: int, n: int, k: int, bias: Optional[int] = None, act: int = 0, splits: int = 1,
          ws: Optional[int] = None):
    flags = (1 if a_mn else 0) | (2 if b_mn else 0)
    return instr(L.OP_GEMM_TC_EX, [a, b, bias, c, ws], [m, n, k, lda, ldb, ldc, flags, splits],
                 act=act)


def _auto_split(m: int, n: int, k: int, ctx):
    """(splits, workspace) for a GEMM with fewer output tiles than the
    bind's CTA target (``ctx.split_target``, 0: the library default):
    split-K over the K loop (deterministic in-order reduce); (1, None) when
    the tiles already suffice.  The count is fixed here, at lowering."""
    return split_plan(m, n, k, ctx)


def split_plan(m: int, n: int, k: int, ctx):
    import ctypes
    sp, nws = ctypes.c_int32(), ctypes.c_int64()
    L.call("mgx_gemm_split_plan", m, n, k, int(getattr(ctx, "split_target", 0) or 0),
           ctypes.byref(sp), ctypes.byref(nws))
    if sp.value <= 1:
        return 1, None
    return sp.value, ctx.scratch(4 * nws.value)


def _weights_bf16(w: View, ctx, code: list):
    """wb[F, ldk] bf16 (zero K padding) of a convolution weight; once per
    step (memo on the weight node)."""
    f = w.shape[0]
    kk = prod(w.shape[1:])
    ldk = _pad8(kk)
    key = ("wb", id(ctx.input_node("in1")), w.ptr)
    wb = ctx.memo.get(key)
    if wb is None:
        wb = ctx.prep(key, 2 * f * ldk, lambda dst: [_cast_rows(w, f, kk, dst, ldk)],
                      (w.ptr, w.ptr + 4 * w.size))
    return wb, ldk


def _conv_operands(x: View, w: View, attrs, ctx, code: list):
    """Explicit-GEMM operands (C % 8 != 0): col = im2col(x) [M, ldk] and the
    bf16 weight, shared by the forward and the backward."""
    k, s, p = _conv_params(attrs)
    b, h, wd, c = x.shape
    ho, wo = _conv_out(h, wd, k, s, p)
    m, kk = b * ho * wo, k[0] * k[1] * c
    ldk = _pad8(kk)
    f = w.shape[0]
    xn = ctx.input_node("in0")
    key_c = ("col", id(xn), x.ptr, tuple(k), tuple(s), tuple(p))
    col = ctx.memo.get(key_c)
    if col is None:
        col = ctx.persistent(2 * m * ldk)
        ctx.memo[key_c] = col
        code.append(instr(L.OP_IM2COL, [x.ptr, col], _geom(x.shape, k, s, p) + [ldk]))
    wb, _ = _weights_bf16(w, ctx, code)
    return col, wb, (m, kk, ldk, f, k, s, p, ho, wo)


def _pointwise(k, s, p) -> bool:
    return tuple(k) == (1, 1) and tuple(s) == (1, 1) and tuple(p) == (0, 0)


def _implicit_ok(c: int) -> bool:
    return c % 8 == 0


def _shadow(v: View, node, ctx, code: list) -> int:
    """Compact bf16 NHWC copy of ``v`` for the implicit GEMM: the producer's
    (written in its own pass) or a cast made here once per step."""
    sh = ctx.shadow_of(node)
    if sh is None:
        n = v.size
        key = ("shadow", id(node) if node is not None else v.ptr)
        sh = ctx.persistent(2 * n)
        ctx.memo[key] = sh
        c = v.shape[-1]
        code.append(_cast_rows(v, n // c, c, sh, c))
    return sh


def _pack_geom(shape, k, s, p) -> tuple:
    b, h, w, c = shape
    assert max(b, h, w, c) < (1 << 16) and max(*k, *s, *p) < (1 << 8)
    return ((b << 48) | (h << 32) | (w << 16) | c,
            (k[0] << 40) | (k[1] << 32) | (s[0] << 24) | (s[1] << 16) | (p[0] << 8) | p[1])


def _gemm_conv(mode: int, src: int, shape, k, s, p, op: int, ldop: int, out: int, ldc: int,
               m: int, n: int, kdim: int, bias=None, act: int = 0, splits: int = 1, ws=None,
               colstats=None):
    g1, g2 = _pack_geom(shape, k, s, p)
    return instr(L.OP_GEMM_CONV, [src, op, bias, out, ws, colstats],
                 [m, n, kdim, ldop, ldc, mode | (splits << 8), g1, g2], act=act)


def _conv_lower_fwd(ins, out, attrs):
    return conv_forward_instrs(ins, out, attrs)


def conv_forward_instrs(ins, out, attrs, colstats: Optional[int] = None) -> list:
    """Convolution forward; colstats: buffer for the epilogue's per-32-row
    (mean, M2) column statistics (a BatchNorm follows, executor fusion)."""
    ctx = current_ctx()
    code = []
    x, w = ins[0], ins[1]
    bias = ins[2].ptr if len(ins) > 2 else None
    k, s, p = _conv_params(attrs)
    f = w.shape[0]
    if _implicit_ok(x.shape[3]):
        # implicit GEMM: the A operand gathered from x's bf16 copy in-kernel
        sh = _shadow(x, ctx.input_node("in0"), ctx, code)
        wb, ldk = _weights_bf16(w, ctx, code)
        b, h, wd, c = x.shape
        ho, wo = _conv_out(h, wd, k, s, p)
        kk = k[0] * k[1] * c
        sp, ws = (1, None) if colstats else _auto_split(b * ho * wo, f, kk, ctx)
        if _pointwise(k, s, p):
            # 1x1 / stride 1: the bf16 copy IS the A operand -- both operands
            # by TMA, no gather warps
            g = _gemm(sh, c, False, wb, ldk, False, out.ptr, f, b * h * wd, f, c, bias=bias,
                      splits=sp, ws=ws)
            g.ptr[5] = colstats or None
            code.append(g)
            return code
        code.append(_gemm_conv(1, sh, x.shape, k, s, p, wb, ldk, out.ptr, f, b * ho * wo, f, kk,
                               bias=bias, colstats=colstats, splits=sp, ws=ws))
        return code
    col, wb, (m, kk, ldk, f, *_r) = _conv_operands(x, w, attrs, ctx, code)
    sp, ws = (1, None) if colstats else _auto_split(m, f, kk, ctx)
    g = _gemm(col, ldk, False, wb, ldk, False, out.ptr, f, m, f, kk, bias=bias, splits=sp, ws=ws)
    g.ptr[5] = colstats or None
    code.append(g)
    return code


def _conv_dy(og: View, f: int, ctx, code: list):
    """bf16 output gradient [M, ld]: the producer's compact copy (ld = F)
    when there is one, else a padded cast made once per step."""
    node = ctx.input_node("og")
    if f % 8 == 0:
        return _shadow(og, node, ctx, code), f
    m = prod(og.shape[:-1])
    ldf = _pad8(f)
    key = ("dyb", id(node), og.ptr)
    dyb = ctx.memo.get(key)
    if dyb is None:
        dyb = ctx.persistent(2 * m * ldf)
        ctx.memo[key] = dyb
        code.append(_cast_rows(og, m, f, dyb, ldf))
    return dyb, ldf


def _conv_lower_bwd(slot, env, out, attrs):
    ctx = current_ctx()
    og = env["og"]
    code = []
    if slot == 2:
        m, f = prod(og.shape[:-1]), og.shape[-1]
        ws = ctx.scratch(_reduce_ws(m, f))
        return [instr(L.OP_COLSUM, [og.ptr, ws, out.ptr], [m, f])]
    x, w = env["in0"], env["in1"]
    k, s, p = _conv_params(attrs)
    b, h, wd, c = x.shape
    ho, wo = _conv_out(h, wd, k, s, p)
    m, kk, f = b * ho * wo, k[0] * k[1] * c, w.shape[0]
    implicit = _implicit_ok(c)
    if slot == 1:
        # dW[f, kk] = sum_m dY[m, f] col[m, kk]: both operands MN-major, split-K
        dyb, ldf = _conv_dy(og, f, ctx, code)
        sp, ws = _auto_split(f, kk, m, ctx)
        if implicit:
            sh = _shadow(x, ctx.input_node("in0"), ctx, code)
            if _pointwise(k, s, p):  # dW = dY^T x over the bf16 copies, both by TMA
                code.append(_gemm(dyb, ldf, True, sh, c, True, out.ptr, kk, f, kk, m,
                                  splits=sp, ws=ws))
                return code
            code.append(_gemm_conv(2, sh, x.shape, k, s, p, dyb, ldf, out.ptr, kk, f, kk, m,
                                   splits=sp, ws=ws))
            return code
        col, _wb, (m, kk, ldk, *_r) = _conv_operands(x, w, attrs, ctx, code)
        code.append(_gemm(dyb, ldf, True, col, ldk, True, out.ptr, kk, f, kk, m,
                          splits=sp, ws=ws))
        return code
    # dX
    dyb, ldf = _conv_dy(og, f, ctx, code)
    wb, ldk = _weights_bf16(w, ctx, code)
    if k == (1, 1) and s == (1, 1) and p == (0, 0):
        sp, ws = _auto_split(m, c, f, ctx)
        code.append(_gemm(dyb, ldf, False, wb, ldk, True, out.ptr, c, m, c, f, splits=sp, ws=ws))
        return code
    if s == (1, 1) and p[0] < k[0] and p[1] < k[1]:
        # stride 1: dX = conv(dY, flipped W, pad k-1-p): implicit GEMM over
        # dY's bf16 copy when F % 8 == 0, else explicit im2col(dY)
        kf = k[0] * k[1] * f
        ldkf = _pad8(kf)
        key = ("wflip", id(ctx.input_node("in1")), w.ptr)
        wfl = ctx.memo.get(key)
        if wfl is None:
            wfl = ctx.prep(key, 2 * c * ldkf,
                           lambda dst: [instr(L.OP_WFLIP, [w.ptr, dst], [f, k[0], k[1], c, ldkf])],
                           (w.ptr, w.ptr + 4 * w.size))
        pf = (k[0] - 1 - p[0], k[1] - 1 - p[1])
        sp, ws = _auto_split(b * h * wd, c, kf, ctx)
        if f % 8 == 0:
            code.append(_gemm_conv(1, dyb, og.shape, k, (1, 1), pf, wfl, ldkf, out.ptr, c,
                                   b * h * wd, c, kf, splits=sp, ws=ws))
            return code
        dcolt = ctx.scratch(2 * b * h * wd * ldkf)
        code.append(instr(L.OP_IM2COL, [og.ptr, dcolt], _geom(og.shape, k, (1, 1), pf) + [ldkf]))
        code.append(_gemm(dcolt, ldkf, False, wfl, ldkf, False, out.ptr, c, b * h * wd, c, kf,
                          splits=sp, ws=ws))
        return code
    if (s == (2, 2) and p[0] < k[0] and p[1] < k[1] and f % 8 == 0
            and os.environ.get("MGX_S2_DX", "col2im") == "mode3"):
        # stride 2: dX = the stride-1 transposed convolution of dY read
        # dilated by 2 (gather mode 3) with the flipped weights -- no column
        # matrix, no col2im
        kf = k[0] * k[1] * f
        ldkf = _pad8(kf)
        key = ("wflip", id(ctx.input_node("in1")), w.ptr)
        wfl = ctx.memo.get(key)
        if wfl is None:
            wfl = ctx.prep(key, 2 * c * ldkf,
                           lambda dst: [instr(L.OP_WFLIP, [w.ptr, dst], [f, k[0], k[1], c, ldkf])],
                           (w.ptr, w.ptr + 4 * w.size))
        sp, ws = _auto_split(b * h * wd, c, kf, ctx)
        code.append(_gemm_conv(3, dyb, x.shape, k, s, p, wfl, ldkf, out.ptr, c, b * h * wd, c, kf,
                               splits=sp, ws=ws))
        return code
    dcol = ctx.scratch(4 * m * kk)
    sp, ws = _auto_split(m, kk, f, ctx)
    code.append(_gemm(dyb, ldf, False, wb, ldk, True, dcol, kk, m, kk, f, splits=sp, ws=ws))
    code.append(instr(L.OP_COL2IM, [dcol, out.ptr], _geom(x.shape, k, s, p) + [kk]))
    return code


def _conv_uses(slot, nin):
    return {0: (("og", "in0", "in1"), "in0"),
            1: (("og", "in0", "in1"), "in1"),
            2: (("og", "in2"), "in2")}[slot]


register(OperatorDef(
    name="Convolution", prefix="conv", input_names=("data", "weight", "bias"),
    attr_schema={"kernel": ((int, tuple, list), True), "num_filter": (int, True),
                 "stride": _PAIR, "pad": _PAIR, "dilate": _PAIR, "no_bias": (bool, False),
                 "num_group": (int, False), "layout": (str, False), "workspace": (int, False)},
    infer_shape=_conv_infer, forward=_native_forward(_conv_lower_fwd),
    backward=_native_backward("Convolution"), backward_uses=_conv_uses,
    lower_forward=_conv_lower_fwd, lower_backward=_conv_lower_bwd, inputs_for=_conv_inputs,
))


# ---------------------------------------------------------------- BatchNorm
# MXNet BatchNorm over the channel axis: training normalises with the batch
# mean and biased variance and updates moving_mean/moving_var with
# `momentum`; inference (no gradients requested, or use_global_stats) uses
# the moving averages.  fix_gamma=True (MXNet's default) pins gamma to 1 and
# its gradient to 0.  Inputs 3/4 are the auxiliary moving statistics.

def _reduce_ws(m: int, c: int) -> int:
    import ctypes
    out = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", max(m, 1), max(c, 1), ctypes.byref(out))
    return out.value


def _bn_infer(shapes, attrs):
    data = _need(shapes[0], "BatchNorm", "data")
    if len(data) < 2:
        raise InferenceError("BatchNorm: data must have rank >= 2")
    c = data[-1]
    return ([tuple(data)] + [_fill(shapes[i], (c,), n) for i, n in
                             ((1, "gamma"), (2, "beta"), (3, "moving_mean"), (4, "moving_var"))],
            [tuple(data)])


_FUSED_OK = {}


def bn_fused_kind(m: int, c: int, backward: bool) -> int:
    """How the cluster-fused BatchNorm kernels (bn_fused.cu) take this
    (rows, channels) shape: 0 not at all, 1 rows staged on-chip, 2 rows
    streamed twice through L2."""
    key = (m, c, bool(backward))
    if key not in _FUSED_OK:
        import ctypes
        ok = ctypes.c_int(0)
        L.call("mgx_bn_fused_ok", m, c, 1 if backward else 0, ctypes.byref(ok))
        _FUSED_OK[key] = int(ok.value)
    return _FUSED_OK[key]


def bn_fused_ok(m: int, c: int, backward: bool) -> bool:
    """Whether the cluster-fused BatchNorm kernels take this shape: one
    launch per pass instead of 2-4."""
    return bn_fused_kind(m, c, backward) != 0


def _bn_train_fused(attrs, ctx, m, c) -> bool:
    return (ctx.training and not attrs.get("use_global_stats", False)
            and bn_fused_ok(m, c, False))


def _bn_stats(x: View, attrs, ctx, code: list, update: bool, mm=None, mv=None,
              xnode=None, tiles: Optional[int] = None) -> int:
    m, c = prod(x.shape[:-1]), x.shape[-1]
    eps = float(attrs.get("eps", 1e-3))
    key = ("bnstats", id(xnode if xnode is not None else ctx.input_node("in0")), x.ptr, eps)
    st = ctx.memo.get(key)
    if st is None:
        st = ctx.persistent(8 * c)
        ctx.memo[key] = st
        use_global = (not ctx.training) or bool(attrs.get("use_global_stats", False))
        mmp = mm.ptr if (update or use_global) and mm else None
        mvp = mv.ptr if (update or use_global) and mv else None
        if tiles is not None and not use_global:
            # from the convolution epilogue's per-tile statistics (no re-read)
            code.append(instr(L.OP_BN_STATS, [x.ptr, tiles, st, mmp, mvp], [m, c, 0, 1],
                              [eps, float(attrs.get("momentum", 0.9))]))
        else:
            ws = ctx.scratch(_reduce_ws(m, c))
            code.append(instr(L.OP_BN_STATS, [x.ptr, ws, st, mmp, mvp],
                              [m, c, 1 if use_global else 0, 0],
                              [eps, float(attrs.get("momentum", 0.9))]))
    return st


def bn_forward_instrs(ins, out: View, attrs, act: int = 0, tiles: Optional[int] = None,
                      xnode=None, y_fp32: bool = True, cat: Optional[tuple] = None) -> list:
    """BatchNorm (+ activation) forward: statistics, then one apply pass
    writing the fp32 output and, when a convolution consumes it, its bf16
    copy; ``y_fp32=False`` (the executor proved every consumer reads the
    copy) drops the fp32 write."""
    ctx = current_ctx()
    x = ins[0]
    m, c = prod(x.shape[:-1]), x.shape[-1]
    code = []
    gamma = None if attrs.get("fix_gamma", True) else ins[1].ptr
    y16 = ctx.shadow_out(out.size) if c % 8 == 0 else None
    yp = out.ptr if (y_fp32 or y16 is None) else None
    ldo = 0
    if cat is not None:
        # the output is a channel slice of a Concat written in place
        yp, y16, ldo = cat
    eps = float(attrs.get("eps", 1e-3))
    key = ("bnstats", id(xnode if xnode is not None else ctx.input_node("in0")), x.ptr, eps)
    if tiles is None and key not in ctx.memo and _bn_train_fused(attrs, ctx, m, c):
        # statistics + moving averages + apply in one cluster kernel
        st = ctx.persistent(8 * c)
        ctx.memo[key] = st
        code.append(instr(L.OP_BN_FWD_FUSED, [x.ptr, st, gamma, ins[2].ptr, yp, y16],
                          [m, c, ins[3].ptr if ins[3] else 0, ins[4].ptr if ins[4] else 0, ldo],
                          [eps, float(attrs.get("momentum", 0.9))], act=act))
        return code
    st = _bn_stats(x, attrs, ctx, code, update=True, mm=ins[3], mv=ins[4], xnode=xnode,
                   tiles=tiles)
    code.append(instr(L.OP_BN_APPLY, [x.ptr, st, gamma, ins[2].ptr, yp, y16], [m, c, ldo], act=act))
    return code


def _bn_lower_fwd(ins, out, attrs):
    return bn_forward_instrs(ins, out, attrs)


def _bn_lower_bwd(slot, env, out, attrs):
    ctx = current_ctx()
    if slot >= 3:
        return [instr(L.OP_FILL, [out.ptr], [out.size], [0.0])]
    og, x = env["og"], env["in0"]
    m, c = prod(x.shape[:-1]), x.shape[-1]
    code = []
    st = _bn_stats(x, attrs, ctx, code, update=False)
    key = ("bnsums", id(ctx.input_node("og")), id(ctx.input_node("in0")), og.ptr, x.ptr)
    sums = ctx.memo.get(key)
    if sums is None:
        sums = ctx.persistent(8 * c)
        ctx.memo[key] = sums
        ws = ctx.scratch(_reduce_ws(m, c))
        code.append(instr(L.OP_BN_BWD_REDUCE, [og.ptr, x.ptr, st, ws, sums, None],
                          [m, c, 0, 0, 0, 0]))
    fix = attrs.get("fix_gamma", True)
    if slot == 0:
        gamma = None if fix else env["in1"].ptr
        ws = ctx.scratch(_reduce_ws(m, c))
        code.append(instr(L.OP_BN_BWD_DX, [og.ptr, x.ptr, st, sums, gamma, out.ptr],
                          [m, c, 0, 0, ws, 0]))
    elif slot == 1:
        code.append(instr(L.OP_FILL, [out.ptr], [c], [0.0]) if fix else
                    instr(L.OP_COPY, [sums + 4 * c, out.ptr], [c]))
    else:
        code.append(instr(L.OP_COPY, [sums, out.ptr], [c]))
    return code


def bn_backward_group(og: View, relu: bool, x: View, gamma: View, beta: View, attrs,
                      xnode, dx: Optional[View], dgamma: Optional[View],
                      dbeta: Optional[View], dbias_conv: Optional[View] = None,
                      dx_node=None, dx_fp32: bool = True, pool=None,
                      og_slice: Optional[tuple] = None) -> list:
    """All requested BatchNorm gradients of one node in one pass pair (the
    executor's fusion of the sibling Backward nodes, optionally with the
    ReLU backward in front of them): one reduction that also writes dbeta /
    dgamma, then dx.  relu: og is the ReLU's output gradient; its mask is
    recomputed from x, gamma and beta (never read back)."""
    ctx = current_ctx()
    m, c = prod(x.shape[:-1]), x.shape[-1]
    code = []
    st = _bn_stats(x, attrs, ctx, code, update=False, xnode=xnode)
    fix = attrs.get("fix_gamma", True)
    if pool is not None:
        # og = the max pooling's input gradient, gathered from its output
        # gradient and argmax inside both passes (stem fusion; executor)
        dyp, pnode, pattrs, pshape = pool
        k, s, p, full = _pool_params(pattrs, pshape)
        arg = _pool_argmax(pnode, pshape, dyp.size, k, 0, ctx)
        g1, g2 = _pack_geom(pshape, k, s, p)
        g2 |= int(full) << 48
        g = None if fix else gamma.ptr
        sums = ctx.persistent(8 * c)
        ws = ctx.scratch(_reduce_ws(m, c))
        code.append(instr(L.OP_BN_BWD_REDUCE_POOL, [dyp.ptr, x.ptr, st, ws, sums, arg],
                          [m, c, dbeta.ptr if dbeta else 0, dgamma.ptr if dgamma else 0,
                           (g or 0) if relu else 0, beta.ptr if relu else 0, g1, g2],
                          act=1 if fix else 0))
        dx16 = ctx.shadow_out(dx.size, dx_node)
        assert dx16 is not None and not dx_fp32, "pooled BatchNorm dx writes the bf16 copy only"
        dws = ctx.scratch(_reduce_ws(m, c))
        code.append(instr(L.OP_BN_BWD_DX_POOL, [dyp.ptr, x.ptr, st, sums, g, arg],
                          [m, c, beta.ptr if relu else 0,
                           dbias_conv.ptr if dbias_conv is not None else 0, dws, dx16, g1, g2]))
        return code
    if dx is not None and bn_fused_ok(m, c, True):
        # reductions + dx (+ conv bias gradient) in one cluster kernel;
        # og_slice = (pointer, row stride): the output gradient read in
        # place from a channel slice of a Concat's gradient (executor)
        g = None if fix else gamma.ptr
        dx16 = ctx.shadow_out(dx.size, dx_node) if (c % 8 == 0 and dx_node is not None) else None
        dxp = dx.ptr if (dx_fp32 or dx16 is None) else None
        ogp, ldd = og_slice if og_slice is not None else (og.ptr, 0)
        code.append(instr(L.OP_BN_BWD_FUSED, [ogp, x.ptr, st, g, dxp, dx16],
                          [m, c, (g or 0) if relu else 0, beta.ptr if relu else 0,
                           dbeta.ptr if dbeta else 0, dgamma.ptr if dgamma else 0,
                           (1 if fix else 0) | (ldd << 8),
                           dbias_conv.ptr if dbias_conv is not None else 0]))
        return code
    assert og_slice is None, "an in-place gradient slice needs the cluster BatchNorm kernel"
    sums = ctx.persistent(8 * c)
    ws = ctx.scratch(_reduce_ws(m, c))
    g = None if fix else gamma.ptr
    rb = beta.ptr if relu else None
    code.append(instr(L.OP_BN_BWD_REDUCE, [og.ptr, x.ptr, st, ws, sums, rb],
                      [m, c, dbeta.ptr if dbeta else 0, dgamma.ptr if dgamma else 0,
                       1 if fix else 0, (g or 0) if relu else 0]))
    if dx is not None:
        dws = ctx.scratch(_reduce_ws(m, c))
        dx16 = ctx.shadow_out(dx.size, dx_node) if (c % 8 == 0 and dx_node is not None) else None
        # dx_fp32=False: every consumer of dx reads its bf16 copy (the
        # convolution's implicit GEMMs) -- the fp32 tensor is never stored
        dxp = dx.ptr if (dx_fp32 or dx16 is None) else None
        code.append(instr(L.OP_BN_BWD_DX, [og.ptr, x.ptr, st, sums, g, dxp],
                          [m, c, rb or 0, dbias_conv.ptr if dbias_conv is not None else 0, dws,
                           (g or 0) if relu else 0, dx16 or 0]))
    return code


def _bn_uses(slot, nin):
    if slot >= 3:
        return ((f"in{slot}",), f"in{slot}")
    return (("og", "in0", "in1", "in2"), f"in{slot}")


register(OperatorDef(
    name="BatchNorm", prefix="bn",
    input_names=("data", "gamma", "beta", "moving_mean", "moving_var"),
    attr_schema={"eps": ((int, float), False), "momentum": ((int, float), False),
                 "fix_gamma": (bool, False), "use_global_stats": (bool, False),
                 "axis": (int, False), "output_mean_var": (bool, False)},
    infer_shape=_bn_infer, forward=_native_forward(_bn_lower_fwd),
    backward=_native_backward("BatchNorm"), backward_uses=_bn_uses,
    lower_forward=_bn_lower_fwd, lower_backward=_bn_lower_bwd,
))

AUX_SUFFIXES = ("_moving_mean", "_moving_var")


def conv_bn_instrs(cins, cout: View, cattrs, bins, bout: View, battrs, act: int, conv_node,
                   y_fp32: bool = True, cat: Optional[tuple] = None):
    """Convolution -> BatchNorm (-> activation) forward: the GEMM epilogue
    produces the BatchNorm statistics of its output (per 32-row (mean, M2)
    pairs), so the BatchNorm never re-reads the convolution output for its
    statistics (executor fusion)."""
    ctx = current_ctx()
    m, f = prod(cout.shape[:-1]), cout.shape[-1]
    if _bn_train_fused(battrs, ctx, m, f):
        # the cluster-fused BatchNorm computes its own statistics from one
        # on-chip pass: no epilogue statistics needed
        code = conv_forward_instrs(cins, cout, cattrs)
        return code + bn_forward_instrs(bins, bout, battrs, act=act, xnode=conv_node,
                                        y_fp32=y_fp32, cat=cat)
    tiles = ctx.scratch(8 * (-(-m // 32)) * f)
    code = conv_forward_instrs(cins, cout, cattrs, colstats=tiles)
    code += bn_forward_instrs(bins, bout, battrs, act=act, tiles=tiles, xnode=conv_node,
                              y_fp32=y_fp32, cat=cat)
    return code


def conv_bn_pool_instrs(cins, cout: View, cattrs, bins, battrs, act: int, conv_node,
                        pool_node, pattrs, pout: View, y_fp32: bool = True):
    """Convolution -> BatchNorm -> activation -> max pooling (the stem):
    statistics from the GEMM epilogue, then ONE pass normalising, activating
    and pooling with the argmax -- the activation tensor is never written
    (its backward recomputes the mask from x; the pooling backward reads the
    argmax).  Executor fusion."""
    ctx = current_ctx()
    m, f = prod(cout.shape[:-1]), cout.shape[-1]
    tiles = ctx.scratch(8 * (-(-m // 32)) * f)
    code = conv_forward_instrs(cins, cout, cattrs, colstats=tiles)
    x = bins[0]
    st = _bn_stats(x, battrs, ctx, code, update=True, mm=bins[3], mv=bins[4], xnode=conv_node,
                   tiles=tiles)
    gamma = None if battrs.get("fix_gamma", True) else bins[1].ptr
    k, s, p, full = _pool_params(pattrs, x.shape)
    arg = _pool_argmax(pool_node, x.shape, pout.size, k, 0, ctx)
    ctx.memo[("argmax_fwd", id(pool_node))] = True
    y16 = ctx.shadow_out(pout.size, pool_node) if f % 8 == 0 else None
    yp = None if (not y_fp32 and y16 is not None) else pout.ptr
    geom = _geom(x.shape, k, s, p)
    geom[6] |= int(full) << 40
    code.append(instr(L.OP_BN_ACT_POOL, [x.ptr, st, gamma, bins[2].ptr, yp, y16], geom + [arg],
                      act=act))
    return code


# ------------------------------------------------------------------ Pooling

_POOL_TYPES = {"max": 0, "avg": 1}


def _pool_params(attrs, shape):
    _check_layout(attrs, "Pooling")
    if attrs.get("pool_type", "max") not in _POOL_TYPES:
        raise InferenceError(f"Pooling: pool_type must be max or avg, got {attrs.get('pool_type')!r}")
    conv = attrs.get("pooling_convention", "valid")
    if conv not in ("valid", "full"):
        raise InferenceError(f"Pooling: unknown pooling_convention {conv!r}")
    if attrs.get("global_pool", False):
        return (shape[1], shape[2]), (1, 1), (0, 0), False
    k = _pair(attrs["kernel"], "kernel")
    s = _pair(attrs.get("stride", 1), "stride")
    p = _pair(attrs.get("pad", 0), "pad")
    return k, s, p, conv == "full"


def _pool_out(h, w, k, s, p, full):
    def one(n, kk, ss, pp):
        span = n + 2 * pp - kk
        return (-(-span // ss) if full else span // ss) + 1
    return one(h, k[0], s[0], p[0]), one(w, k[1], s[1], p[1])


def _pool_infer(shapes, attrs):
    data = _need(shapes[0], "Pooling", "data")
    if len(data) != 4:
        raise InferenceError("Pooling: data must be (batch, height, width, channels)")
    if not attrs.get("global_pool", False) and "kernel" not in attrs:
        raise InferenceError("Pooling: kernel is required unless global_pool")
    k, s, p, full = _pool_params(attrs, data)
    ho, wo = _pool_out(data[1], data[2], k, s, p, full)
    if ho <= 0 or wo <= 0:
        raise InferenceError("Pooling: window larger than the padded input")
    return [tuple(data)], [(data[0], ho, wo, data[3])]


def _pool_argmax(node, x_shape, out_size, k, kind, ctx) -> Optional[int]:
    """uint8 argmax side buffer of a max-pooling node (forward writes it,
    backward reads it); None when the vectorised kernels do not apply."""
    if kind != 0 or x_shape[-1] % 4 or k[0] * k[1] > 255 or node is None:
        return None
    key = ("argmax", id(node))
    ptr = ctx.memo.get(key)
    if ptr is None:
        ptr = ctx.persistent(out_size)
        ctx.memo[key] = ptr
    return ptr


def _pool_lower_fwd(ins, out, attrs):
    ctx = current_ctx()
    x = ins[0]
    k, s, p, full = _pool_params(attrs, x.shape)
    kind = _POOL_TYPES[attrs.get("pool_type", "max")]
    arg = _pool_argmax(ctx.node, x.shape, out.size, k, kind, ctx) if ctx.training else None
    if arg is not None:
        ctx.memo[("argmax_fwd", id(ctx.node))] = True
    y16 = ctx.shadow_out(out.size) if (x.shape[-1] % 8 == 0 and k[0] * k[1] <= 255) else None
    yp = None if (ctx.fp32_dead and y16 is not None) else out.ptr
    return [instr(L.OP_POOL_FWD, [x.ptr, yp, arg, y16], _geom(x.shape, k, s, p) + [int(full)],
                  act=kind)]


def _pool_lower_bwd(slot, env, out, attrs):
    ctx = current_ctx()
    x = env["in0"]
    k, s, p, full = _pool_params(attrs, x.shape)
    kind = _POOL_TYPES[attrs.get("pool_type", "max")]
    node = ctx.input_node("out")
    arg = None
    if node is not None and ctx.memo.get(("argmax_fwd", id(node))):
        arg = _pool_argmax(node, x.shape, env["out"].size, k, kind, ctx)
    # arg None: no forward recorded the argmax (eager call) -> rescan x
    return [instr(L.OP_POOL_BWD, [x.ptr, env["out"].ptr, env["og"].ptr, out.ptr, arg],
                  _geom(x.shape, k, s, p) + [int(full)], act=kind)]


register(OperatorDef(
    name="Pooling", prefix="pool", input_names=("data",),
    attr_schema={"kernel": ((int, tuple, list), False), "pool_type": (str, False),
                 "stride": _PAIR, "pad": _PAIR, "global_pool": (bool, False),
                 "pooling_convention": (str, False), "layout": (str, False)},
    infer_shape=_pool_infer, forward=_native_forward(_pool_lower_fwd),
    backward=_native_backward("Pooling"),
    backward_uses=lambda slot, nin: (("og", "in0", "out"), "in0"),
    lower_forward=_pool_lower_fwd, lower_backward=_pool_lower_bwd,
))


# ------------------------------------------------------------------- Concat
# Concatenation along the channel (last) axis: one channel-offset copy per
# input; the backward slices the output gradient.

def _concat_axis(attrs, rank):
    d = attrs.get("dim", -1)
    if d not in (-1, rank - 1):
        raise InferenceError(f"Concat: only the channel (last) axis is implemented, got dim={d}")


def _concat_infer(shapes, attrs):
    known = [s for s in shapes if s is not None]
    if len(known) != len(shapes) or not known:
        raise InferenceError("Concat: every input shape must be known")
    rank = len(known[0])
    _concat_axis(attrs, rank)
    lead = tuple(known[0][:-1])
    for s in known:
        if len(s) != rank or tuple(s[:-1]) != lead:
            raise InferenceError(f"Concat: incompatible shapes {known}")
    return [tuple(s) for s in shapes], [lead + (sum(s[-1] for s in shapes),)]


def _concat_lower_fwd(ins, out, attrs):
    rows, tot = prod(out.shape[:-1]), out.shape[-1]
    ok16 = tot % 8 == 0 and all(x.shape[-1] % 4 == 0 for x in ins)
    o16 = current_ctx().shadow_out(out.size) if ok16 else None
    if ok16 and len(ins) <= 4:
        # one pass over the output (and its bf16 copy)
        chans = [x.shape[-1] for x in ins] + [0] * (4 - len(ins))
        return [instr(L.OP_CONCAT, [x.ptr for x in ins] + [None] * (4 - len(ins)) + [out.ptr, o16],
                      [rows, len(ins)] + chans)]
    code, off = [], 0
    for x in ins:
        c = x.shape[-1]
        code.append(instr(L.OP_CHAN_COPY, [x.ptr, out.ptr, o16], [rows, c, c, 0, tot, off]))
        off += c
    return code


def _concat_lower_bwd(slot, env, out, attrs):
    og = env["og"]
    rows, tot = prod(og.shape[:-1]), og.shape[-1]
    off = sum(env[f"in{i}"].shape[-1] for i in range(slot))
    c = out.shape[-1]
    return [instr(L.OP_CHAN_COPY, [og.ptr, out.ptr], [rows, c, tot, off, c, 0])]


register(OperatorDef(
    name="Concat", prefix="concat", input_names=(),
    attr_schema={"dim": (int, False), "num_args": (int, False)},
    infer_shape=_concat_infer, forward=_native_forward(_concat_lower_fwd),
    backward=_native_backward("Concat"), variadic=True,
    backward_uses=lambda slot, nin: (("og",) + tuple(f"in{i}" for i in range(nin)), f"in{slot}"),
    lower_forward=_concat_lower_fwd, lower_backward=_concat_lower_bwd,
))


def validate_concat_inputs(n: int) -> None:
    if n < 1:
        raise ArgumentError("Concat needs at least one input")
