"""Operator registry: shape inference plus native lowerings.

Same plugin surface as the reference (ops.py:23-55): an ``OperatorDef`` with
``infer_shape``, ``forward(ins, out, attrs)``, ``backward(ins, out, og,
grads, attrs)``, ``inplace_identity``, ``is_loss``, ``variadic`` and
``backward_uses``.  Arrays handed to ``forward``/``backward`` are CUDA
``torch.Tensor`` views (device memory), not numpy arrays; built-in operators
enqueue hand-written sm_100a kernels through the C-ABI on the engine's
current stream.  A user plugin may supply plain ``forward``/``backward``
callables written against torch tensors and the executor runs them in
order on the same stream.

Built-in operators additionally carry ``lower_forward`` /
``lower_backward``: they turn a node into ``mgx_instr`` records (see
include/mgx.h) so a bound graph becomes one native program that can be
replayed or captured as a CUDA graph.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod
from typing import Callable, Dict, List, Optional, Sequence

from . import _lib as L
from .errors import ArgumentError, InferenceError


@dataclass(frozen=True)
class OperatorDef:
    name: str
    prefix: str
    input_names: tuple
    attr_schema: dict
    infer_shape: Callable
    forward: Optional[Callable]
    backward: Optional[Callable]
    inplace_identity: tuple = ()
    is_loss: bool = False
    variadic: bool = False
    backward_uses: Optional[Callable] = None
    # native lowering: (ins: [View], out: View, attrs) -> [Instr]
    lower_forward: Optional[Callable] = None
    # (slot, env: {role: View}, out: View, attrs) -> [Instr]
    lower_backward: Optional[Callable] = None
    # attrs -> input names when they depend on attributes (no_bias)
    inputs_for: Optional[Callable] = None

    def input_names_for(self, attrs: dict) -> tuple:
        return self.inputs_for(attrs) if self.inputs_for is not None else self.input_names

    @property
    def num_inputs(self) -> int:
        return len(self.input_names)


OPS: Dict[str, OperatorDef] = {}


def register(op: OperatorDef) -> OperatorDef:
    OPS[op.name] = op
    return op


def get_op(name: str) -> OperatorDef:
    try:
        return OPS[name]
    except KeyError:
        raise ArgumentError(f"unknown operator {name!r}") from None


def validate_attrs(op: OperatorDef, attrs: dict) -> None:
    if op.variadic:
        return
    for key in attrs:
        if key not in op.attr_schema:
            raise ArgumentError(f"{op.name}: unknown attr {key!r}")
    for key, (typ, required) in op.attr_schema.items():
        if key in attrs:
            if not isinstance(attrs[key], typ):
                raise ArgumentError(f"{op.name}: attr {key!r} must be {typ}")
        elif required:
            raise ArgumentError(f"{op.name}: missing required attr {key!r}")


# ------------------------------------------------------------ device views

class View:
    """A device buffer as the lowering sees it: address + shape (fp32)."""

    __slots__ = ("ptr", "shape")

    def __init__(self, ptr: int, shape: Sequence[int]):
        self.ptr = int(ptr)
        self.shape = tuple(int(d) for d in shape)

    @property
    def size(self) -> int:
        return prod(self.shape)

    @classmethod
    def of(cls, t) -> "View":
        return cls(t.data_ptr(), tuple(t.shape))


def instr(op: int, ptrs: Sequence[Optional[int]] = (), dims: Sequence[int] = (),
          fattr: Sequence[float] = (), act: int = 0) -> L.Instr:
    ins = L.Instr()
    ins.op = op
    ins.act = act
    for i, d in enumerate(dims):
        ins.dims[i] = int(d)
    for i, f in enumerate(fattr):
        ins.fattr[i] = float(f)
    for i, p in enumerate(ptrs):
        ins.ptr[i] = p or None
    return ins


def instr_cost(ins: L.Instr) -> tuple:
    """(algorithmic bytes, flops) of one instruction: every operand read once
    and every result written once (the roofline numerator)."""
    d, op = ins.dims, ins.op
    has = [bool(ins.ptr[i]) for i in range(6)]
    if op == L.OP_GEMM_PW:
        m, n, k = d[0], d[1], d[2]
        return 4 * (m * k + n * k + m * n + (n if has[2] else 0)), 2 * m * n * k
    if op == L.OP_GEMM_SEQ:
        m, n, k = d[0], d[1], d[2]
        return 4 * (m * k + k * n + m * n + (m * n if has[3] else 0)), 2 * m * n * k
    if op == L.OP_DW_DB:
        b, h, f = d[0], d[1], d[2]
        byt = 4 * (b * h + ((b * f + h * f) if has[2] else 0) + (h if has[3] else 0))
        return byt, (2 * b * h * f if has[2] else 0) + (b * h if has[3] else 0)
    if op == L.OP_GEMM_TC:
        m, n, k = d[0], d[1], d[2]
        return 2 * (m * k + n * k) + 4 * m * n + (4 * n if has[2] else 0), 2 * m * n * k
    if op == L.OP_GEMM_TC_EX:
        m, n, k = d[0], d[1], d[2]
        return 2 * (m * k + n * k) + 4 * m * n + (4 * n if has[2] else 0), 2 * m * n * k
    if op == L.OP_GEMM_CONV:  # implicit GEMM: the gathered source counted once
        m, n, k = d[0], d[1], d[2]
        a, w = d[6], d[7]
        src = 2 * ((a >> 48) & 0xFFFF) * ((a >> 32) & 0xFFFF) * ((a >> 16) & 0xFFFF) * (a & 0xFFFF)
        mode = d[5] & 0xFF
        opb = 2 * (n * k if mode in (1, 3) else m * k)
        # mode 3 (stride-2 data gradient over the dilated dY): 3 of 4 taps
        # multiply inserted zeros -- the algorithmic work is a quarter
        flops = 2 * m * n * k // (4 if mode == 3 else 1)
        return src + opb + 4 * m * n + (4 * n if has[2] else 0), flops
    if op == L.OP_IM2COL:  # reads the input once, writes the bf16 col matrix
        b, h, w, c = d[0], d[1], d[2], d[3]
        kh, kw, sh, sw, ph, pw = d[4] >> 16, d[4] & 0xFFFF, d[5] >> 16, d[5] & 0xFFFF, d[6] >> 16, d[6] & 0xFFFF
        ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        return 4 * b * h * w * c + 2 * b * ho * wo * d[7], 0
    if op == L.OP_COL2IM:
        b, h, w, c = d[0], d[1], d[2], d[3]
        kh, kw, sh, sw, ph, pw = d[4] >> 16, d[4] & 0xFFFF, d[5] >> 16, d[5] & 0xFFFF, d[6] >> 16, d[6] & 0xFFFF
        ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        return 4 * b * ho * wo * d[7] + 4 * b * h * w * c, b * ho * wo * d[7]
    if op == L.OP_BN_STATS:
        return (0 if d[2] else 4 * d[0] * d[1]) + 8 * d[1], 2 * d[0] * d[1]
    if op == L.OP_BN_APPLY:
        return 8 * d[0] * d[1], 4 * d[0] * d[1]
    if op == L.OP_BN_BWD_REDUCE:
        return 8 * d[0] * d[1], 4 * d[0] * d[1]
    if op == L.OP_BN_BWD_DX:
        return 12 * d[0] * d[1], 6 * d[0] * d[1]
    if op == L.OP_BN_ACT_POOL:  # x read once (taps from L1/L2), pooled y16/y + argmax
        n_in = d[0] * d[1] * d[2] * d[3]
        return 4 * n_in + (n_in // 4) * (3 + (4 if has[4] else 0)), 6 * n_in
    if op == L.OP_BN_BWD_REDUCE_POOL:  # windows: pooled gradient + argmax + x at the argmax
        return 9 * d[0] * d[1] // 4, 4 * d[0] * d[1]
    if op == L.OP_BN_BWD_DX_POOL:  # x + pooled gradient + argmax read, dx16 written
        return 4 * d[0] * d[1] + 5 * d[0] * d[1] // 4 + 2 * d[0] * d[1], 10 * d[0] * d[1]
    if op == L.OP_BN_FWD_FUSED:  # read x once, write y and/or y16
        return (4 + (4 if has[4] else 0) + (2 if has[5] else 0)) * d[0] * d[1], 6 * d[0] * d[1]
    if op == L.OP_BN_BWD_FUSED:  # read dy and x once, write dx and/or dx16
        return (8 + (4 if has[4] else 0) + (2 if has[5] else 0)) * d[0] * d[1], 10 * d[0] * d[1]
    if op in (L.OP_POOL_FWD, L.OP_POOL_BWD):
        b, h, w, c = d[0], d[1], d[2], d[3]
        kh, kw, sh, sw, ph, pw = d[4] >> 16, d[4] & 0xFFFF, d[5] >> 16, d[5] & 0xFFFF, d[6] >> 16, d[6] & 0xFFFF
        span_h, span_w = h + 2 * ph - kh, w + 2 * pw - kw
        ho = (-(-span_h // sh) if d[7] else span_h // sh) + 1
        wo = (-(-span_w // sw) if d[7] else span_w // sw) + 1
        n_in, n_out = b * h * w * c, b * ho * wo * c
        if op == L.OP_POOL_FWD:
            return 4 * (n_in + n_out), n_out * kh * kw
        return 4 * (2 * n_in + 2 * n_out), n_out * kh * kw
    if op == L.OP_SUM_N:
        return 4 * d[0] * (d[1] + 1), d[0] * (d[1] - 1)
    if op == L.OP_CONCAT:
        return 8 * d[0] * sum(d[2:2 + d[1]]), 0
    if op == L.OP_CHAN_COPY:
        return 8 * d[0] * d[1], 0
    if op == L.OP_COLSUM:
        return 4 * d[0] * d[1], d[0] * d[1]
    if op == L.OP_CAST_BF16:
        return 4 * d[0] * d[1] + 2 * d[3] * d[4], d[3] * d[4]
    if op == L.OP_SOFTMAX_FWD:
        return 4 * 2 * d[0] * d[1], 4 * d[0] * d[1]
    if op == L.OP_SOFTMAX_BWD:
        return 4 * (2 * d[0] * d[1] + d[0]), 2 * d[0] * d[1]
    streams = {L.OP_FILL: 1, L.OP_COPY: 2, L.OP_EW: 3, L.OP_SCALAR: 2, L.OP_ACT_FWD: 2,
               L.OP_ACT_BWD: 3, L.OP_AXPY: 3}.get(op, 0)
    return 4 * streams * d[0], d[0]


# ------------------------------------------------------- lowering context

class LowerCtx:
    """Device scratch and cross-node memo for lowering one bound graph.

    ``scratch(n)`` is op-local memory (reused by the next node's lowering:
    instructions run in program order on one stream); ``persistent(n)``
    lives as long as the program (bf16 operand copies a node's backward
    reuses from its forward, BatchNorm statistics).  The executor lowers
    twice: a measuring pass against a fake base, then the real pass against
    two allocations of the measured sizes.  ``node`` is the graph node being
    lowered, ``training`` whether the bind requested gradients."""

    ALIGN = 256
    FAKE_BASE = 1 << 44

    def __init__(self, training: bool, scratch_base: Optional[int] = None,
                 persist_base: Optional[int] = None, device: int = 0,
                 unique_scratch: bool = False):
        self.training = training
        self.device = device
        self.measuring = scratch_base is None
        self._sbase = self.FAKE_BASE if scratch_base is None else scratch_base
        self._pbase = self.FAKE_BASE * 2 if persist_base is None else persist_base
        self._op_off = 0
        self._p_off = 0
        self.scratch_peak = 0
        # unique_scratch: no scratch reuse between nodes (nodes may then run
        # concurrently on different lanes of a multi-stream schedule)
        self.unique_scratch = unique_scratch
        self._sizes: Dict[int, int] = {}
        self.reads: List[tuple] = []    # persistent buffers read by the current node
        self.writes: List[tuple] = []   # ... and written by it
        self.memo = _Memo(self)
        self.node = None
        # set by the executor: the fp32 output of the node being lowered has
        # no reader (every consumer gathers from its bf16 copy)
        self.fp32_dead = False
        # implicit-GEMM operands: ids of nodes whose outputs feed a
        # convolution (set by the executor); out_node = the node whose
        # output the current lowering writes
        self.want_shadow: set = set()
        self.out_node = None
        self.pre: list = []
        # split-K CTA target of this bind's GEMMs (0: the library default)
        self.split_target = 0

    def begin_op(self, node) -> None:
        self.node = node
        self.out_node = node
        self._op_off = 0
        self.reads, self.writes = [], []
        self.pre = []

    def prep(self, key, nbytes: int, instrs, src_range) -> int:
        """Independent preparation work of the current node (a weight cast):
        allocates the persistent result under memo ``key`` and queues the
        instructions as their own group (their only input is ``src_range``),
        so a multi-lane schedule can run them off the node's critical path.
        The node itself records a read of the result."""
        ptr = self.persistent(nbytes)
        dict.__setitem__(self.memo, key, ptr)
        rng = (ptr, ptr + self._sizes[ptr])
        self.pre.append((instrs(ptr), [src_range], [rng]))
        self.reads.append(rng)
        return ptr

    def shadow_out(self, elems: int, node=None) -> Optional[int]:
        """A compact bf16 copy of the output of ``node`` (default: the node
        being lowered) when a convolution consumes it: the producer writes
        it in the same pass, the convolution gathers from it."""
        node = node if node is not None else self.out_node
        if node is None or id(node) not in self.want_shadow:
            return None
        key = ("shadow", id(node))
        ptr = self.memo.get(key)
        if ptr is None:
            ptr = self.persistent(2 * elems)
            self.memo[key] = ptr
        return ptr

    def shadow_of(self, node) -> Optional[int]:
        if node is None:
            return None
        return self.memo.get(("shadow", id(node)))

    def _al(self, n: int) -> int:
        return -(-max(int(n), 1) // self.ALIGN) * self.ALIGN

    def scratch(self, nbytes: int) -> int:
        if self.unique_scratch:
            return self.persistent(nbytes)
        ptr = self._sbase + self._op_off
        self._op_off += self._al(nbytes)
        self.scratch_peak = max(self.scratch_peak, self._op_off)
        return ptr

    def persistent(self, nbytes: int) -> int:
        ptr = self._pbase + self._p_off
        self._p_off += self._al(nbytes)
        self._sizes[ptr] = self._al(nbytes)
        return ptr

    @property
    def persistent_bytes(self) -> int:
        return self._p_off

    def input_node(self, role: str):
        """Source node of ``role`` ('in0', 'og', ...) of the node being
        lowered (a Backward node's roles name its inputs)."""
        n = self.node
        if n is None:
            return None
        if n.op == "Backward":
            roles = n.attrs["roles"]
            if role not in roles:
                return None
            return n.inputs[roles.index(role)][0]
        if role.startswith("in"):
            return n.inputs[int(role[2:])][0]
        return None


class _Memo(dict):
    """The lowering memo; records which persistent buffers the current
    node creates (writes) and reuses (reads), for the hazard analysis of the
    multi-lane schedule."""

    def __init__(self, ctx: "LowerCtx"):
        super().__init__()
        self._ctx = ctx

    def _note(self, value, into: list) -> None:
        if isinstance(value, int) and not isinstance(value, bool) and value in self._ctx._sizes:
            into.append((value, value + self._ctx._sizes[value]))

    def get(self, key, default=None):
        if key is None:
            return default
        value = super().get(key, default)
        if key in self:
            self._note(value, self._ctx.reads)
        return value

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._note(value, self._ctx.writes)


class _EagerCtx(LowerCtx):
    """Context for plugin-style eager calls: real allocations per request,
    kept alive with the context object's owner list."""

    _keep: list = []

    def __init__(self, device: int):
        super().__init__(training=True, scratch_base=0, persist_base=0, device=device)

    def _alloc(self, nbytes: int) -> int:
        import torch
        t = torch.empty(self._al(nbytes), dtype=torch.uint8, device=f"cuda:{self.device}")
        keep = _EagerCtx._keep
        if len(keep) >= 512:
            # the oldest allocations may still be read by queued kernels:
            # drain the device before handing them back to the allocator
            torch.cuda.synchronize(self.device)
            del keep[:-256]
        keep.append(t)
        return t.data_ptr()

    def scratch(self, nbytes: int) -> int:
        return self._alloc(nbytes)

    def persistent(self, nbytes: int) -> int:
        return self._alloc(nbytes)

    def prep(self, key, nbytes: int, instrs, src_range) -> int:
        """Eager: the preparation runs right away on the current stream."""
        ptr = self._alloc(nbytes)
        dict.__setitem__(self.memo, key, ptr)
        run_instrs(instrs(ptr), _current_stream())
        return ptr


_CTX: List[LowerCtx] = []


def current_ctx() -> LowerCtx:
    """The lowering context of the bind in progress (or an eager one)."""
    if _CTX:
        return _CTX[-1]
    from .engine import current_device
    return _EagerCtx(current_device())


class lowering:
    """``with lowering(ctx): ...`` makes ``ctx`` current."""

    def __init__(self, ctx: LowerCtx):
        self.ctx = ctx

    def __enter__(self):
        _CTX.append(self.ctx)
        return self.ctx

    def __exit__(self, *exc):
        _CTX.pop()


def run_instrs(instrs: List[L.Instr], stream: int) -> None:
    if not instrs:
        return
    arr = (L.Instr * len(instrs))(*instrs)
    L.call("mgx_instr_run", arr, len(instrs), stream)


def _current_stream() -> int:
    from .engine import current_stream
    return current_stream()


def _native_forward(lower):
    def forward(ins, out, attrs):
        run_instrs(lower([View.of(t) for t in ins], View.of(out), attrs), _current_stream())
    return forward


def _native_backward(op_name: str):
    def backward(ins, out, og, grads, attrs):
        op = OPS[op_name]
        env = {f"in{i}": View.of(t) for i, t in enumerate(ins) if t is not None}
        if out is not None:
            env["out"] = View.of(out)
        if og is not None:
            env["og"] = View.of(og)
        code = []
        for slot, g in enumerate(grads):
            if g is not None:
                code += op.lower_backward(slot, env, View.of(g), attrs)
        run_instrs(code, _current_stream())
    return backward


# -------------------------------------------------------- shape utilities

def _need(shape, node, what):
    if shape is None:
        raise InferenceError(f"cannot infer {what} shape for node {node}")
    return shape


def _fill(slot_shape, new_shape, what):
    if slot_shape is not None and tuple(slot_shape) != tuple(new_shape):
        raise InferenceError(f"inconsistent {what} shape: {slot_shape} vs {new_shape}")
    return tuple(new_shape)


def _flat2(shape):
    return (shape[0], prod(shape[1:]))


# ---------------------------------------------------------- FullyConnected
# ops.py:91-133.  forward: pairwise_k(x2 . w^T) then + b; backward slot 0:
# sequential_h(og . w); slot 1: tree_outer(og, x2); slot 2: tree_sum(og).

def _fc_infer(shapes, attrs):
    h = attrs["num_hidden"]
    data = _need(shapes[0], "FullyConnected", "data")
    if len(data) < 2:
        raise InferenceError("FullyConnected: data must have rank >= 2")
    b, f = _flat2(data)
    return ([tuple(data), _fill(shapes[1], (h, f), "weight"), _fill(shapes[2], (h,), "bias")],
            [(b, h)])


def fc_forward_instr(x: View, w: View, b: Optional[View], out: View, act: int = 0):
    bsz, f = _flat2(x.shape)
    h = w.shape[0]
    return instr(L.OP_GEMM_PW, [x.ptr, w.ptr, b.ptr if b else None, out.ptr],
                 [bsz, h, f, f, f, h], act=act)


# ---- bf16 tensor-core lowering (executor dense="bf16"): tolerance path.
# Operands are cast (and transposed where the contraction needs K-major
# operands) into bf16 scratch with K padded to a multiple of 8, then one
# tcgen05 GEMM with fp32 accumulation in TMEM (csrc/tc_gemm.cu).

def _pad8(n: int) -> int:
    return -(-n // 8) * 8


def _cast(src: View, rows_in: int, cols_in: int, dst: int, rows_out: int, ld_out: int,
          transpose: bool):
    return instr(L.OP_CAST_BF16, [src.ptr, dst],
                 [rows_in, cols_in, cols_in, rows_out, ld_out, 1 if transpose else 0])


def _bf16_copy(kind: str, role: str, src: View, rows: int, cols: int, code: list) -> tuple:
    """bf16 copy [rows, pad8(cols)] of ``src`` (zero K padding), made once
    per step and shared by the forward and backward contractions that read
    it (memo keyed on the source node of ``role``)."""
    ctx = current_ctx()
    ld = _pad8(cols)
    node = ctx.input_node(role)
    key = (kind, id(node), src.ptr) if node is not None else None
    ptr = ctx.memo.get(key) if key is not None else None
    if ptr is None:
        ptr = ctx.persistent(2 * rows * ld)
        if key is not None:
            ctx.memo[key] = ptr
        code.append(_cast(src, rows, cols, ptr, rows, ld, False))
    return ptr, ld


def _gemm_ex(a, lda, a_mn, b, ldb, b_mn, c, ldc, m, n, k, bias=None, act=0, splits=1, ws=None):
    flags = (1 if a_mn else 0) | (2 if b_mn else 0)
    return instr(L.OP_GEMM_TC_EX, [a, b, bias, c, ws], [m, n, k, lda, ldb, ldc, flags, splits],
                 act=act)


def fc_forward_tc(x: View, w: View, b: Optional[View], out: View, act: int, alloc=None) -> list:
    """y[B,H] = x[B,F] . W[H,F]^T (+b, act): both operands K-major."""
    bsz, f = _flat2(x.shape)
    h = w.shape[0]
    code = []
    xb, ldx = _bf16_copy("fcx", "in0", x, bsz, f, code)
    wb, ldw = _bf16_copy("fcw", "in1", w, h, f, code)
    code.append(_gemm_ex(xb, ldx, False, wb, ldw, False, out.ptr, h, bsz, h, f,
                         bias=b.ptr if b else None, act=act))
    return code


def fc_dx_tc(og: View, w: View, dx: View, alloc=None) -> list:
    """dX[B,F] = og[B,H] . W[H,F]: og K-major, W MN-major (its own layout)."""
    bsz, h = og.shape
    f = w.shape[1]
    code = []
    ogb, ldo = _bf16_copy("fcog", "og", og, bsz, h, code)
    wb, ldw = _bf16_copy("fcw", "in1", w, h, f, code)
    code.append(_gemm_ex(ogb, ldo, False, wb, ldw, True, dx.ptr, f, bsz, f, h))
    return code


def fc_dw_tc(og: View, x: View, dw: View, alloc=None) -> list:
    """dW[H,F] = og[B,H]^T . x[B,F]: both MN-major (batch is the contraction)."""
    bsz, h = og.shape
    f = _flat2(x.shape)[1]
    code = []
    ogb, ldo = _bf16_copy("fcog", "og", og, bsz, h, code)
    xb, ldx = _bf16_copy("fcx", "in0", x, bsz, f, code)
    from .conv_ops import split_plan
    sp, ws = split_plan(h, f, bsz, current_ctx())
    code.append(_gemm_ex(ogb, ldo, True, xb, ldx, True, dw.ptr, f, h, f, bsz,
                         splits=sp, ws=ws))
    return code


def _fc_lower_fwd(ins, out, attrs):
    return [fc_forward_instr(ins[0], ins[1], ins[2], out)]


def fc_dx_instr(og: View, w: View, dx: View, y: Optional[View] = None, act: int = 0):
    bsz, h = og.shape
    f = w.shape[1]
    return instr(L.OP_GEMM_SEQ, [og.ptr, w.ptr, dx.ptr, y.ptr if y else None],
                 [bsz, f, h, h, 1, f, 1, f], act=act)


def fc_dw_db_instr(og: View, x: Optional[View], dw: Optional[View], db: Optional[View]):
    bsz, h = og.shape
    f = _flat2(x.shape)[1] if x is not None else 1
    return instr(L.OP_DW_DB, [og.ptr, x.ptr if x else None, dw.ptr if dw else None,
                              db.ptr if db else None], [bsz, h, f])


def _fc_lower_bwd(slot, env, out, attrs):
    og = env["og"]
    if slot == 0:
        return [fc_dx_instr(og, env["in1"], out)]
    if slot == 1:
        return [fc_dw_db_instr(og, env["in0"], out, None)]
    return [fc_dw_db_instr(og, None, None, out)]


def _fc_uses(slot, nin):
    # in1/in2 feed slots 1/2 only as shape sources; they are argument
    # variables with dedicated storage (ops.py:119-124).
    return {0: (("og", "in0", "in1"), "in0"),
            1: (("og", "in0", "in1"), "in1"),
            2: (("og", "in2"), "in2")}[slot]


register(OperatorDef(
    name="FullyConnected", prefix="fc", input_names=("data", "weight", "bias"),
    attr_schema={"num_hidden": (int, True)}, infer_shape=_fc_infer,
    forward=_native_forward(_fc_lower_fwd), backward=_native_backward("FullyConnected"),
    backward_uses=_fc_uses, lower_forward=_fc_lower_fwd, lower_backward=_fc_lower_bwd,
))


# -------------------------------------------------------------- Activation

def _act_infer(shapes, attrs):
    if attrs["act_type"] not in L.ACT_CODES:
        raise InferenceError(f"unknown act_type {attrs['act_type']!r}")
    s = _need(shapes[0], "Activation", "data")
    return [tuple(s)], [tuple(s)]


def _act_lower_fwd(ins, out, attrs):
    return [instr(L.OP_ACT_FWD, [ins[0].ptr, out.ptr], [out.size],
                  act=L.ACT_CODES[attrs["act_type"]])]


def _act_lower_bwd(slot, env, out, attrs):
    # derivative through the forward output only (ops.py:140-147)
    return [instr(L.OP_ACT_BWD, [env["out"].ptr, env["og"].ptr, out.ptr], [out.size],
                  act=L.ACT_CODES[attrs["act_type"]])]


register(OperatorDef(
    name="Activation", prefix="act", input_names=("data",),
    attr_schema={"act_type": (str, True)}, infer_shape=_act_infer,
    forward=_native_forward(_act_lower_fwd), backward=_native_backward("Activation"),
    inplace_identity=((0, 0),), backward_uses=lambda slot, nin: (("og", "out"), "out"),
    lower_forward=_act_lower_fwd, lower_backward=_act_lower_bwd,
))


# ----------------------------------------------------------- SoftmaxOutput

def _softmax_infer(shapes, attrs):
    data = _need(shapes[0], "SoftmaxOutput", "data")
    if len(data) != 2:
        raise InferenceError("SoftmaxOutput: data must be (batch, classes)")
    return [tuple(data), _fill(shapes[1], (data[0],), "label")], [tuple(data)]


def _softmax_lower_fwd(ins, out, attrs):
    bsz, classes = out.shape
    return [instr(L.OP_SOFTMAX_FWD, [ins[0].ptr, out.ptr], [bsz, classes])]


def _softmax_lower_bwd(slot, env, out, attrs):
    if slot == 1:
        return [instr(L.OP_FILL, [out.ptr], [out.size], [0.0])]
    bsz, classes = env["out"].shape
    return [instr(L.OP_SOFTMAX_BWD, [env["out"].ptr, env["in1"].ptr, out.ptr], [bsz, classes])]


register(OperatorDef(
    name="SoftmaxOutput", prefix="softmax", input_names=("data", "label"),
    attr_schema={}, infer_shape=_softmax_infer,
    forward=_native_forward(_softmax_lower_fwd), backward=_native_backward("SoftmaxOutput"),
    is_loss=True,
    backward_uses=lambda slot, nin: {0: (("in1", "out"), "out"), 1: (("in1",), "in1")}[slot],
    lower_forward=_softmax_lower_fwd, lower_backward=_softmax_lower_bwd,
))


# ------------------------------------------------- elementwise and scalar

def _same_shape_infer(shapes, attrs):
    known = [s for s in shapes if s is not None]
    if not known:
        raise InferenceError("elementwise: no input shape known")
    s = tuple(known[0])
    return [_fill(x, s, "operand") for x in shapes], [s]


def _ew_lower(code):
    def lower(ins, out, attrs):
        return [instr(L.OP_EW, [ins[0].ptr, ins[1].ptr, out.ptr], [out.size, code])]
    return lower


def _copy_instr(src: View, dst: View):
    return instr(L.OP_COPY, [src.ptr, dst.ptr], [dst.size])


def _ew_add_lower_bwd(slot, env, out, attrs):
    return [_copy_instr(env["og"], out)]


def _ew_mul_lower_bwd(slot, env, out, attrs):
    other = env["in1"] if slot == 0 else env["in0"]
    return [instr(L.OP_EW, [env["og"].ptr, other.ptr, out.ptr], [out.size, 2])]


register(OperatorDef(
    name="ElementwiseAdd", prefix="add", input_names=("lhs", "rhs"), attr_schema={},
    infer_shape=_same_shape_infer, forward=_native_forward(_ew_lower(0)),
    backward=_native_backward("ElementwiseAdd"), inplace_identity=((0, 0), (1, 0)),
    backward_uses=lambda slot, nin: (("og",), "og"),
    lower_forward=_ew_lower(0), lower_backward=_ew_add_lower_bwd,
))

register(OperatorDef(
    name="ElementwiseMul", prefix="mul", input_names=("lhs", "rhs"), attr_schema={},
    infer_shape=_same_shape_infer, forward=_native_forward(_ew_lower(2)),
    backward=_native_backward("ElementwiseMul"), inplace_identity=((0, 0), (1, 0)),
    backward_uses=lambda slot, nin: {0: (("og", "in1"), "og"), 1: (("og", "in0"), "og")}[slot],
    lower_forward=_ew_lower(2), lower_backward=_ew_mul_lower_bwd,
))


def _scalar_infer(shapes, attrs):
    s = _need(shapes[0], "scalar op", "data")
    return [tuple(s)], [tuple(s)]


def _scalar_lower(code):
    def lower(ins, out, attrs):
        return [instr(L.OP_SCALAR, [ins[0].ptr, out.ptr], [out.size, code], [attrs["value"]])]
    return lower


def _sadd_lower_bwd(slot, env, out, attrs):
    return [_copy_instr(env["og"], out)]


def _smul_lower_bwd(slot, env, out, attrs):
    return [instr(L.OP_SCALAR, [env["og"].ptr, out.ptr], [out.size, 1], [attrs["value"]])]


register(OperatorDef(
    name="ScalarAdd", prefix="sadd", input_names=("data",),
    attr_schema={"value": ((int, float), True)}, infer_shape=_scalar_infer,
    forward=_native_forward(_scalar_lower(0)), backward=_native_backward("ScalarAdd"),
    inplace_identity=((0, 0),), backward_uses=lambda slot, nin: (("og",), "og"),
    lower_forward=_scalar_lower(0), lower_backward=_sadd_lower_bwd,
))

register(OperatorDef(
    name="ScalarMul", prefix="smul", input_names=("data",),
    attr_schema={"value": ((int, float), True)}, infer_shape=_scalar_infer,
    forward=_native_forward(_scalar_lower(1)), backward=_native_backward("ScalarMul"),
    inplace_identity=((0, 0),), backward_uses=lambda slot, nin: (("og",), "og"),
    lower_forward=_scalar_lower(1), lower_backward=_smul_lower_bwd,
))


# ------------------------------------------------------------------ MatMul
# forward det_matmul(a, b): b contiguous -> sequential over K.  backward
# slot 0 det_matmul(og, b^T): pairwise over N; slot 1 det_matmul(a^T, og):
# sequential over M (orders pinned by probe against kernels.det_matmul).

def _matmul_infer(shapes, attrs):
    a = _need(shapes[0], "MatMul", "lhs")
    b = _need(shapes[1], "MatMul", "rhs")
    if len(a) != 2 or len(b) != 2 or a[1] != b[0]:
        raise InferenceError(f"MatMul: incompatible shapes {a} @ {b}")
    return [tuple(a), tuple(b)], [(a[0], b[1])]


def _matmul_lower_fwd(ins, out, attrs):
    (m, k), (_, n) = ins[0].shape, ins[1].shape
    return [instr(L.OP_GEMM_SEQ, [ins[0].ptr, ins[1].ptr, out.ptr, None],
                  [m, n, k, k, 1, n, 1, n])]


def _matmul_lower_bwd(slot, env, out, attrs):
    a, b, og = env["in0"], env["in1"], env["og"]
    (m, k), (_, n) = a.shape, b.shape
    if slot == 0:
        # ga[m, kk] = pairwise_n(og[m, n] * b[kk, n])
        return [instr(L.OP_GEMM_PW, [og.ptr, b.ptr, None, out.ptr], [m, k, n, n, n, k])]
    # gb[kk, n] = sequential_m(a[m, kk] * og[m, n])
    return [instr(L.OP_GEMM_SEQ, [a.ptr, og.ptr, out.ptr, None], [k, n, m, 1, k, n, 1, n])]


register(OperatorDef(
    name="MatMul", prefix="matmul", input_names=("lhs", "rhs"), attr_schema={},
    infer_shape=_matmul_infer, forward=_native_forward(_matmul_lower_fwd),
    backward=_native_backward("MatMul"),
    backward_uses=lambda slot, nin: {0: (("og", "in0", "in1"), "in0"),
                                     1: (("og", "in0", "in1"), "in1")}[slot],
    lower_forward=_matmul_lower_fwd, lower_backward=_matmul_lower_bwd,
))


# ----------------------------------------------------------------- Flatten

def _flatten_infer(shapes, attrs):
    s = _need(shapes[0], "Flatten", "data")
    if len(s) < 2:
        raise InferenceError("Flatten: data must have rank >= 2")
    return [tuple(s)], [_flat2(s)]


def _flatten_lower_fwd(ins, out, attrs):
    return [_copy_instr(ins[0], out)]


def _flatten_lower_bwd(slot, env, out, attrs):
    return [_copy_instr(env["og"], out)]


register(OperatorDef(
    name="Flatten", prefix="flatten", input_names=("data",), attr_schema={},
    infer_shape=_flatten_infer, forward=_native_forward(_flatten_lower_fwd),
    backward=_native_backward("Flatten"), inplace_identity=((0, 0),),
    backward_uses=lambda slot, nin: (("og", "in0"), "in0"),
    lower_forward=_flatten_lower_fwd, lower_backward=_flatten_lower_bwd,
))


# --------------------------------------------------------------- ZerosLike

def _zeros_lower_fwd(ins, out, attrs):
    return [instr(L.OP_FILL, [out.ptr], [out.size], [0.0])]


def _zeros_lower_bwd(slot, env, out, attrs):
    return [instr(L.OP_FILL, [out.ptr], [out.size], [0.0])]


register(OperatorDef(
    name="ZerosLike", prefix="zeros", input_names=("data",), attr_schema={},
    infer_shape=_scalar_infer, forward=_native_forward(_zeros_lower_fwd),
    backward=_native_backward("ZerosLike"), backward_uses=lambda slot, nin: (("in0",), "in0"),
    lower_forward=_zeros_lower_fwd, lower_backward=_zeros_lower_bwd,
))


# ---------------------------------------------------------------- Backward
# attrs {of, nin, slot, roles, shape_role, of_attrs} (ops.py:465-527).

def backward_roles(op: OperatorDef, slot: int, nin: int) -> tuple:
    """(roles read, role giving the gradient shape) for ``slot``."""
    if op.backward_uses is not None:
        return op.backward_uses(slot, nin)
    roles = () if op.is_loss else ("og",)
    roles += tuple(f"in{i}" for i in range(nin)) + ("out",)
    return roles, f"in{slot}"


def _backward_infer(shapes, attrs):
    roles = attrs["roles"]
    what = f"{attrs['of']}.backward"
    filled = [_need(s, what, r) for r, s in zip(roles, shapes)]
    return [tuple(s) for s in filled], [tuple(filled[roles.index(attrs["shape_role"])])]


def _backward_lower(ins, out, attrs):
    of = get_op(attrs["of"])
    if of.lower_backward is None:
        raise ArgumentError(f"operator {of.name} has no native backward")
    env = dict(zip(attrs["roles"], ins))
    return of.lower_backward(attrs["slot"], env, out, attrs.get("of_attrs", {}))


def _backward_forward(ins, out, attrs):
    of = get_op(attrs["of"])
    env = dict(zip(attrs["roles"], ins))
    fwd_in = [env.get(f"in{i}") for i in range(attrs["nin"])]
    grads = [None] * attrs["nin"]
    grads[attrs["slot"]] = out
    of.backward(fwd_in, env.get("out"), env.get("og"), grads, attrs.get("of_attrs", {}))


def backward_inplace_pairs(of_name: str, slot: int) -> tuple:
    """Backward nodes whose gradient is og times a mask/constant may write
    over og (ops.py:509-517); og is always input position 0 for these."""
    if slot == 0 and of_name in ("Activation", "ScalarAdd", "ScalarMul", "Flatten",
                                 "ElementwiseAdd"):
        return ((0, 0),)
    return ()


register(OperatorDef(
    name="Backward", prefix="bwd", input_names=(),
    attr_schema={"of": (str, True), "nin": (int, True), "slot": (int, True),
                 "roles": (list, True), "shape_role": (str, True),
                 "of_attrs": (dict, False)},
    infer_shape=_backward_infer, forward=_backward_forward, backward=None, variadic=True,
    lower_forward=_backward_lower,
))


def node_lowering(op_name: str, attrs: dict) -> Optional[Callable]:
    """Native lowering of a node, or None when the op is a Python plugin."""
    op = get_op(op_name)
    if op_name == "Backward":
        of = get_op(attrs["of"])
        return _backward_lower if of.lower_backward is not None else None
    return op.lower_forward


# convolution-net operators register themselves into OPS
from . import conv_ops  # noqa: E402,F401
