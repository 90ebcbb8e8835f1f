"""The C-ABI library loads on a CPU host and exports exactly what
include/mgx.h declares; status/error conventions follow capi.py.  CPU."""

import ctypes
import os
import re

import numpy as np

from conftest import ROOT
from paper_1512_01274_b200 import _lib as L


def declared_functions():
    text = open(os.path.join(ROOT, "include", "mgx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(mgx_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(L.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_status_and_last_error_without_gpu():
    lib = L.lib()
    v = ctypes.c_int()
    assert lib.mgx_abi_version(ctypes.byref(v)) == L.OK and v.value == 1
    assert lib.mgx_abi_version(None) == L.BAD_ARGUMENT
    assert "null" in L.last_error()
    assert lib.mgx_prog_run(12345, 0, 0, 0, 0) == L.BAD_HANDLE
    assert lib.mgx_kv_round(None, 0) == L.BAD_ARGUMENT


def test_planner_core_runs_without_gpu():
    # a 3-node chain x -> a -> b through the C-ABI directly
    n = 3
    is_var = np.array([1, 0, 0], np.uint8)
    nbytes = np.array([16, 16, 16], np.int64)
    ded = np.array([1, 0, 1], np.uint8)
    in_ptr = np.array([0, 0, 1, 2], np.int32)
    in_idx = np.array([0, 1], np.int32)
    ip_ptr = np.array([0, 0, 1, 2], np.int32)
    ip_pos = np.array([0, 0], np.int32)
    phase = np.zeros(3, np.int32)
    slot_of = np.zeros(3, np.int32)
    sb = np.zeros(3, np.int64)
    sd = np.zeros(3, np.uint8)
    edges = np.zeros(8, np.int32)
    ns, ne = ctypes.c_int32(), ctypes.c_int32()
    tot, vis = ctypes.c_int64(), ctypes.c_int64()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.lib().mgx_plan_memory(n, p(is_var), p(nbytes), p(ded), p(in_ptr), p(in_idx), p(ip_ptr),
                                 p(ip_pos), p(phase), 3, p(slot_of), p(sb), p(sd),
                                 ctypes.byref(ns), p(edges), 4, ctypes.byref(ne),
                                 ctypes.byref(tot), ctypes.byref(vis))
    assert st == L.OK
    assert ns.value == 3 and tot.value == 16 and list(slot_of) == [0, 1, 2]


def test_split_plan_without_gpu():
    """mgx_gemm_split_plan: about `target` CTAs per GEMM, at least 16 and at
    most 128 k-blocks per split (the fp32 accumulation-run bound), the
    default target (0) = 128; the count never depends on anything but
    (M, N, K, target) -- the lowering fixes it (tc_gemm.cu auto_splits)."""
    def plan(m, n, k, target):
        sp, ws = ctypes.c_int32(), ctypes.c_int64()
        assert L.lib().mgx_gemm_split_plan(m, n, k, target, ctypes.byref(sp),
                                           ctypes.byref(ws)) == L.OK
        return sp.value, ws.value
    # many tiles: no split
    assert plan(50176, 256, 1152, 32) == (1, 0)
    # the 14x14 weight gradient [192, 1728, 12544]: 2 x 9 tiles, 196 k-blocks
    s32, ws32 = plan(192, 1728, 12544, 32)
    s128, _ = plan(192, 1728, 12544, 0)
    assert s32 < s128 and ws32 == s32 * 192 * 1728
    nk = -(-12544 // 64)
    for s in (s32, s128):
        assert -(-nk // s) <= 128 and -(-nk // s) >= 16
    # the stem weight gradient [64, 147, 802816]: one tile, 12544 k-blocks --
    # the accumulation bound wins over any target
    s, _ = plan(64, 147, 802816, 32)
    assert -(-12544 // s) <= 128
    assert L.lib().mgx_gemm_split_plan(0, 1, 1, 0, None, None) == L.BAD_ARGUMENT
