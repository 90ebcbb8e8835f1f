"""Bandwidth micro-benchmark of the non-GEMM convnet kernels at the
Inception-BN (batch 64) shapes: pooling forward/backward and the BatchNorm
statistics / apply / backward passes, each timed alone with CUDA events
(inputs larger than or comparable to L2; 20 launches after 3 warm-up).

    python tools/kbench.py [pool|bn|all]

Prints one line per case: microseconds per launch and the algorithmic
bytes (reads + writes of distinct tensor elements) per microsecond."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _geom(shape, k, s, p):
    b, h, w, c = shape
    return np.array([b, h, w, c, (k[0] << 16) | k[1], (s[0] << 16) | s[1], (p[0] << 16) | p[1]],
                    np.int64)


def _time(torch, fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


POOLS = [  # (input shape, kernel, stride, pad, type)
    ((64, 112, 112, 64), 3, 2, 0, "max"),
    ((64, 55, 55, 192), 3, 2, 0, "max"),
    ((64, 27, 27, 192), 3, 1, 1, "avg"),
    ((64, 27, 27, 320), 3, 2, 0, "max"),
    ((64, 14, 14, 576), 3, 1, 1, "avg"),
    ((64, 14, 14, 576), 3, 2, 0, "max"),
    ((64, 7, 7, 1024), 7, 1, 0, "avg"),
]


def bench_pool(torch, L):
    for shape, k, s, p, kind in POOLS:
        b, h, w, c = shape
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        x = torch.randn(*shape, device="cuda")
        y = torch.empty(b, ho, wo, c, device="cuda")
        y16 = torch.empty(b, ho, wo, c, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty_like(x)
        t = 0 if kind == "max" else 1
        arg = torch.empty(y.numel(), dtype=torch.uint8, device="cuda") if t == 0 else None
        argp = arg.data_ptr() if arg is not None else None
        geom = _geom(shape, (k, k), (s, s), (p, p))
        gp = geom.ctypes.data_as(ctypes.c_void_p)

        def fwd():
            L.call("mgx_pool_forward", x.data_ptr(), y.data_ptr(), gp, 0, t, argp,
                   y16.data_ptr(), 0)

        def bwd():
            L.call("mgx_pool_backward", x.data_ptr(), y.data_ptr(), y.data_ptr(), dx.data_ptr(),
                   gp, 0, t, argp, 0)
        fwd()
        us_f, us_b = _time(torch, fwd), _time(torch, bwd)
        nx, ny = x.numel(), y.numel()
        abytes = ny if t == 0 else 0
        bf = 4 * nx + 6 * ny + abytes
        bb = 4 * ny + abytes + 4 * nx
        print(f"pool_fwd {kind} {shape} k{k}s{s}: {us_f:8.1f} us  {bf / us_f / 1e3:7.0f} GB/s")
        print(f"pool_bwd {kind} {shape} k{k}s{s}: {us_b:8.1f} us  {bb / us_b / 1e3:7.0f} GB/s")


BNS = [(802816, 64), (193600, 192), (193600, 64), (46656, 32), (46656, 64), (46656, 96),
       (46656, 256), (12544, 576), (3136, 1024)]


def bench_bn(torch, L):
    for m, c in BNS:
        x = torch.randn(m, c, device="cuda")
        dy = torch.randn(m, c, device="cuda")
        y = torch.empty_like(x)
        y16 = torch.empty(m, c, device="cuda", dtype=torch.bfloat16)
        st = torch.empty(2 * c, device="cuda")
        sums = torch.empty(2 * c, device="cuda")
        gam = torch.ones(c, device="cuda")
        bet = torch.zeros(c, device="cuda")
        wsb = ctypes.c_int64()
        L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
        ws = torch.empty(max(wsb.value, 8) // 4 + 1024, device="cuda")

        def stats():
            L.call("mgx_bn_stats", x.data_ptr(), m, c, ws.data_ptr(), st.data_ptr(), None, None,
                   1e-5, 0.9, 0, 0)

        def apply():
            L.call("mgx_bn_apply", x.data_ptr(), st.data_ptr(), gam.data_ptr(), bet.data_ptr(),
                   y.data_ptr(), m, c, 1, y16.data_ptr(), 0)

        def red():
            L.call("mgx_bn_bwd_reduce", dy.data_ptr(), x.data_ptr(), st.data_ptr(), m, c,
                   ws.data_ptr(), sums.data_ptr(), None, None, 0, gam.data_ptr(),
                   bet.data_ptr(), 0)

        def dxk():
            L.call("mgx_bn_bwd_dx", dy.data_ptr(), x.data_ptr(), st.data_ptr(), sums.data_ptr(),
                   gam.data_ptr(), None, m, c, gam.data_ptr(), bet.data_ptr(), None,
                   ws.data_ptr(), y16.data_ptr(), 0)
        stats()
        n = m * c
        for name, fn, nb in (("bn_stats", stats, 4 * n), ("bn_apply", apply, 10 * n),
                             ("bn_bwd_reduce", red, 8 * n), ("bn_bwd_dx", dxk, 10 * n)):
            us = _time(torch, fn)
            print(f"{name:14s} ({m}, {c}): {us:8.1f} us  {nb / us / 1e3:7.0f} GB/s")


BNF = [(12544, 160), (12544, 576), (193600, 64), (46656, 32), (46656, 64), (46656, 96),
       (46656, 256), (3136, 352), (3136, 1024)]


def bench_bn_fused(torch, L):
    for m, c in BNF:
        ok = ctypes.c_int()
        L.call("mgx_bn_fused_ok", m, c, 1, ctypes.byref(ok))
        if not ok.value:
            print(f"bn_fused       ({m}, {c}): no cluster shape")
            continue
        x = torch.randn(m, c, device="cuda")
        dy = torch.randn(m, c, device="cuda")
        y16 = torch.empty(m, c, device="cuda", dtype=torch.bfloat16)
        st = torch.empty(2 * c, device="cuda")
        gam = torch.ones(c, device="cuda")
        bet = torch.zeros(c, device="cuda")
        mm, mv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda")
        db, dg, ds = (torch.empty(c, device="cuda") for _ in range(3))

        def fwd():
            L.call("mgx_bn_fwd_fused", x.data_ptr(), m, c, st.data_ptr(), mm.data_ptr(),
                   mv.data_ptr(), 1e-3, 0.9, gam.data_ptr(), bet.data_ptr(), None,
                   y16.data_ptr(), 1, 0)

        def bwd():
            L.call("mgx_bn_bwd_fused", dy.data_ptr(), c, x.data_ptr(), st.data_ptr(), gam.data_ptr(),
                   m, c, gam.data_ptr(), bet.data_ptr(), db.data_ptr(), dg.data_ptr(), 0, None,
                   None, y16.data_ptr(), ds.data_ptr(), 0)
        fwd()
        n = m * c
        for name, fn, nb in (("bn_fwd_fused", fwd, 6 * n), ("bn_bwd_fused", bwd, 10 * n)):
            us = _time(torch, fn)
            print(f"{name:14s} ({m}, {c}): {us:8.1f} us  {nb / us / 1e3:7.0f} GB/s")


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    import torch
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.engine import Engine
    Engine(device=0)
    if what in ("pool", "all"):
        bench_pool(torch, L)
    if what in ("bn", "all"):
        bench_bn(torch, L)
    if what in ("bnf", "all"):
        bench_bn_fused(torch, L)


if __name__ == "__main__":
    main()
