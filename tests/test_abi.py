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
