"""ctypes binding of libmgx.so, the C-ABI declared in include/mgx.h.

This is the only place Python touches the native library.  Loading fails
loudly when the shared object is missing: there is no CPU fallback for any
device operation (build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_1512_01274_b200/csrc``).

Status handling mirrors the reference's flat boundary (capi.py:26-29,
102-116): 0 ok, 1 bad handle, 2 bad argument, 3 internal; the message comes
from ``mgx_last_error_message``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ArgumentError, MinigraphError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmgx.so")

OK, BAD_HANDLE, BAD_ARGUMENT, INTERNAL = 0, 1, 2, 3

ACT_CODES = {"relu": 1, "sigmoid": 2, "tanh": 3}

# instruction opcodes (include/mgx.h MGX_OP_*)
OP_FILL, OP_COPY, OP_EW, OP_SCALAR, OP_GEMM_PW, OP_GEMM_SEQ, OP_DW_DB = 1, 2, 3, 4, 5, 6, 7
OP_ACT_FWD, OP_ACT_BWD, OP_SOFTMAX_FWD, OP_SOFTMAX_BWD, OP_AXPY = 8, 9, 10, 11, 12
OP_CAST_BF16, OP_GEMM_TC = 13, 14
OP_IM2COL, OP_COL2IM, OP_BN_STATS, OP_BN_APPLY, OP_BN_BWD_REDUCE, OP_BN_BWD_DX = 15, 16, 17, 18, 19, 20
OP_POOL_FWD, OP_POOL_BWD, OP_CHAN_COPY, OP_COLSUM, OP_GEMM_TC_EX = 21, 22, 23, 24, 25
OP_WFLIP, OP_GEMM_CONV, OP_SUM_N, OP_CONCAT = 26, 27, 28, 29
OP_BN_FWD_FUSED, OP_BN_BWD_FUSED = 30, 31
OP_BN_ACT_POOL, OP_BN_BWD_REDUCE_POOL, OP_BN_BWD_DX_POOL = 32, 33, 34
OP_PREP_BATCH = 35
OP_KV_ROUND = 36

KV_ADD, KV_SGD, KV_AGG = 0, 1, 2
KV_MAX_SEGS = 256
KV_FLAG_WORDS_PER_WORKER = 2048
IPC_HANDLE_BYTES = 64


class NativeError(MinigraphError):
    """A C-ABI call returned a non-zero status (INTERNAL / BAD_HANDLE)."""


c_i32, c_i64, c_u32, c_u64, c_f32 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_float)
c_vp, c_up, c_sz = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t
c_uptr = ctypes.c_size_t  # uintptr_t


class Instr(ctypes.Structure):
    """mgx_instr (include/mgx.h)."""
    _fields_ = [("op", c_i32), ("act", c_i32), ("dims", c_i64 * 8),
                ("fattr", c_f32 * 4), ("ptr", c_vp * 6)]


class KvSeg(ctypes.Structure):
    """mgx_kv_seg: element offset in the key arena, length, momentum offset."""
    _fields_ = [("off", c_i64), ("len", c_i64), ("voff", c_i64)]


class KvRoundArgs(ctypes.Structure):
    """mgx_kv_round_args (include/mgx.h)."""
    _fields_ = [
        ("segs", ctypes.POINTER(KvSeg)), ("nseg", c_i32),
        ("machines", c_i32), ("workers", c_i32),
        ("grads", ctypes.POINTER(c_vp)), ("weights", ctypes.POINTER(c_vp)),
        ("self_replica", c_i32), ("velocity", c_vp), ("agg_out", c_vp),
        ("updater", c_i32), ("rescale", c_f32), ("neg_eta", c_f32),
        ("momentum", c_f32), ("weight_decay", c_f32),
        ("flags", ctypes.POINTER(c_vp)), ("rank", c_i32), ("epoch_ctr", c_vp),
        ("error_word", c_vp), ("grid", c_i32),
        ("scatter", ctypes.POINTER(KvSeg)), ("scatter_owner", ctypes.POINTER(c_i32)),
        ("nscatter", c_i32), ("stage", ctypes.POINTER(c_vp)), ("stage_slot", c_i64),
    ]


_SIGNATURES = {
    "mgx_last_error_message": ([], ctypes.c_char_p),
    "mgx_abi_version": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgx_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgx_set_device": ([ctypes.c_int], ctypes.c_int),
    "mgx_malloc": ([c_sz, ctypes.POINTER(c_vp)], ctypes.c_int),
    "mgx_free": ([c_vp], ctypes.c_int),
    "mgx_host_alloc": ([c_sz, ctypes.POINTER(c_vp)], ctypes.c_int),
    "mgx_host_free": ([c_vp], ctypes.c_int),
    "mgx_stream_create": ([ctypes.POINTER(c_uptr)], ctypes.c_int),
    "mgx_stream_destroy": ([c_uptr], ctypes.c_int),
    "mgx_stream_sync": ([c_uptr], ctypes.c_int),
    "mgx_memcpy_async": ([c_vp, c_vp, c_sz, c_uptr], ctypes.c_int),
    "mgx_memset_async": ([c_vp, ctypes.c_int, c_sz, c_uptr], ctypes.c_int),
    "mgx_event_create": ([ctypes.POINTER(c_uptr)], ctypes.c_int),
    "mgx_event_destroy": ([c_uptr], ctypes.c_int),
    "mgx_event_record": ([c_uptr, c_uptr], ctypes.c_int),
    "mgx_event_elapsed_ms": ([c_uptr, c_uptr, ctypes.POINTER(c_f32)], ctypes.c_int),
    "mgx_stream_wait_event": ([c_uptr, c_uptr], ctypes.c_int),
    "mgx_ipc_get_handle": ([c_vp, c_vp], ctypes.c_int),
    "mgx_ipc_open_handle": ([c_vp, ctypes.POINTER(c_vp)], ctypes.c_int),
    "mgx_ipc_close_handle": ([c_vp], ctypes.c_int),
    "mgx_fill": ([c_vp, c_i64, c_f32, c_uptr], ctypes.c_int),
    "mgx_copy": ([c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_axpy": ([c_f32, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_elementwise": ([ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_scalar_op": ([ctypes.c_int, c_vp, c_f32, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_gemm_pairwise": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
                           ctypes.c_int, c_uptr], ctypes.c_int),
    "mgx_gemm_sequential": ([c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp,
                             ctypes.c_int, c_i64, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_fc_dw_db": ([c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_tree_sum_rows": ([c_vp, c_vp, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_act_forward": ([ctypes.c_int, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_act_backward": ([ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_softmax_forward": ([c_vp, c_vp, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_softmax_backward": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_gemm_bf16_tc": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
                          ctypes.c_int, c_uptr], ctypes.c_int),
    "mgx_cast_f32_bf16": ([c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_cast_bf16_2d": ([c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, ctypes.c_int, c_uptr],
                         ctypes.c_int),
    "mgx_sgd_step": ([c_vp, c_vp, c_vp, c_i64, c_f32, c_f32, c_f32, c_uptr], ctypes.c_int),
    "mgx_plan_memory": ([c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32,
                         c_vp, c_vp, c_vp, ctypes.POINTER(c_i32), c_vp, c_i32,
                         ctypes.POINTER(c_i32), ctypes.POINTER(c_i64),
                         ctypes.POINTER(c_i64)], ctypes.c_int),
    "mgx_py_set_order": ([c_vp, c_i32, c_vp, ctypes.POINTER(c_i32)], ctypes.c_int),
    "mgx_grad_build": ([c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp,
                        c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_i32),
                        ctypes.POINTER(c_i32)], ctypes.c_int),
    "mgx_push_order": ([c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(c_i32)],
                       ctypes.c_int),
    "mgx_instr_run": ([ctypes.POINTER(Instr), c_i32, c_uptr], ctypes.c_int),
    "mgx_prog_create": ([ctypes.POINTER(Instr), c_i32, ctypes.POINTER(c_u64)], ctypes.c_int),
    "mgx_prog_run": ([c_u64, c_i32, c_i32, c_uptr, c_i32], ctypes.c_int),
    "mgx_prog_profile": ([c_u64, c_i32, c_i32, c_uptr, ctypes.POINTER(c_f32)], ctypes.c_int),
    "mgx_prog_destroy": ([c_u64], ctypes.c_int),
    "mgx_capture_begin": ([c_uptr], ctypes.c_int),
    "mgx_capture_end": ([c_uptr, ctypes.POINTER(c_u64)], ctypes.c_int),
    "mgx_graph_launch": ([c_u64, c_uptr], ctypes.c_int),
    "mgx_graph_destroy": ([c_u64], ctypes.c_int),
    "mgx_prog_set_schedule": ([c_u64, c_i32, c_vp, c_vp, c_vp], ctypes.c_int),
    "mgx_prog_kernel_count": ([c_u64, c_i32, c_i32, c_uptr, ctypes.POINTER(c_i64)], ctypes.c_int),
    "mgx_kv_round": ([ctypes.POINTER(KvRoundArgs), c_uptr], ctypes.c_int),
    "mgx_gemm_bf16_tc_ex": ([c_vp, c_i64, ctypes.c_int, c_vp, c_i64, ctypes.c_int, c_vp, c_vp,
                             c_i64, c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_vp, c_vp,
                             c_uptr], ctypes.c_int),
    "mgx_gemm_bf16_conv": ([ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64,
                            c_i64, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_bn_stats_from_tiles": ([c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_f32, c_f32, c_uptr],
                                ctypes.c_int),
    "mgx_gemm_splitk_workspace": ([c_i64, c_i64, c_i64, ctypes.POINTER(c_i64)], ctypes.c_int),
    "mgx_gemm_split_plan": ([c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_i32),
                             ctypes.POINTER(c_i64)], ctypes.c_int),
    "mgx_im2col_bf16": ([c_vp, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_col2im": ([c_vp, c_i64, c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_weight_flip_bf16": ([c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_reduce_workspace_bytes": ([c_i64, c_i64, ctypes.POINTER(c_i64)], ctypes.c_int),
    "mgx_bn_stats": ([c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_f32, c_f32, ctypes.c_int,
                      c_uptr], ctypes.c_int),
    "mgx_bn_apply_ld": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, ctypes.c_int, c_vp, c_i64,
                         c_uptr], ctypes.c_int),
    "mgx_bn_fwd_fused_ld": ([c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_f32, c_f32, c_vp, c_vp, c_vp,
                             c_vp, ctypes.c_int, c_i64, c_uptr], ctypes.c_int),
    "mgx_bn_apply": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, ctypes.c_int, c_vp, c_uptr],
                     ctypes.c_int),
    "mgx_bn_bwd_reduce": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, ctypes.c_int,
                           c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_bn_bwd_dx": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                       c_vp, c_uptr], ctypes.c_int),
    "mgx_bn_fused_ok": ([c_i64, c_i64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgx_bn_fwd_fused": ([c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_f32, c_f32, c_vp, c_vp, c_vp,
                          c_vp, ctypes.c_int, c_uptr], ctypes.c_int),
    "mgx_bn_bwd_fused": ([c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                          ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_bn_act_pool_fwd": ([c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_vp, c_vp,
                             c_vp, c_uptr], ctypes.c_int),
    "mgx_bn_bwd_reduce_pooled": ([c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_i64, c_i64, c_vp,
                                  c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_uptr],
                                 ctypes.c_int),
    "mgx_bn_bwd_dx_pooled": ([c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                              c_vp, c_vp, c_vp, c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_prep_batch": ([c_vp, c_i64, c_i64, c_uptr], ctypes.c_int),
    "mgx_colsum": ([c_vp, c_i64, c_i64, c_vp, c_vp, c_uptr], ctypes.c_int),
    "mgx_pool_forward": ([c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_uptr],
                         ctypes.c_int),
    "mgx_pool_backward": ([c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_uptr],
                          ctypes.c_int),
    "mgx_sum_n": ([c_vp, c_i32, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_concat": ([c_vp, c_vp, c_i32, c_vp, c_vp, c_i64, c_uptr], ctypes.c_int),
    "mgx_chan_copy": ([c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_uptr],
                      ctypes.c_int),
    "mgx_kv_max_grid": ([c_i32, c_i32, ctypes.POINTER(c_i32)], ctypes.c_int),
    "mgx_kv_config": ([c_i32, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                       ctypes.POINTER(c_i32)], ctypes.c_int),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"native library {LIB_PATH} is missing; build it with "
                    "`make -C paper_1512_01274_b200/csrc` (no CPU fallback exists)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (argtypes, restype) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().mgx_last_error_message()
    return msg.decode(errors="replace") if msg else ""


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    msg = last_error()
    where = f"{what}: " if what else ""
    if status == BAD_ARGUMENT:
        raise ArgumentError(f"{where}{msg}")
    raise NativeError(f"{where}status {status}: {msg}")


def np_ptr(a) -> ctypes.c_void_p:
    """Host pointer of a contiguous numpy array (index arrays for the native
    graph builder and planner)."""
    return a.ctypes.data_as(ctypes.c_void_p)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
