"""The stem-fusion kernels at the Inception-BN stem shapes (conv_1 /
conv_2 outputs, batch 64), for ncu: BN+ReLU+maxpool forward, pooled BN
reduce, pooled BN dx.

    python tools/stem_bench.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.engine import Engine
    Engine(device=0)
    for b, h, w, c in ((64, 112, 112, 64), (64, 55, 55, 192)):
        m = b * h * w
        ho, wo = (h - 3) // 2 + 1, (w - 3) // 2 + 1
        n_out = b * ho * wo * c
        geom = np.array([b, h, w, c, (3 << 16) | 3, (2 << 16) | 2, 0], np.int64)
        gp = geom.ctypes.data_as(ctypes.c_void_p)
        x = torch.randn(m, c, device="cuda")
        st = torch.cat([torch.zeros(c), torch.ones(c)]).cuda()
        beta = torch.zeros(c, device="cuda")
        y16 = torch.empty(n_out, dtype=torch.bfloat16, device="cuda")
        arg = torch.empty(n_out, dtype=torch.uint8, device="cuda")
        dyp = torch.randn(n_out, device="cuda")
        wsb = ctypes.c_int64()
        L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
        ws = torch.empty(wsb.value // 4 + 1, device="cuda")
        sums = torch.empty(2 * c, device="cuda")
        dx16 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
        ds = torch.empty(c, device="cuda")

        def fwd():
            L.call("mgx_bn_act_pool_fwd", x.data_ptr(), st.data_ptr(), None, beta.data_ptr(), 1,
                   gp, 0, None, y16.data_ptr(), arg.data_ptr(), 0)

        def red():
            L.call("mgx_bn_bwd_reduce_pooled", dyp.data_ptr(), arg.data_ptr(), gp, 0, x.data_ptr(),
                   st.data_ptr(), m, c, ws.data_ptr(), sums.data_ptr(), None, None, 1, None,
                   beta.data_ptr(), 0)

        def dxp():
            L.call("mgx_bn_bwd_dx_pooled", dyp.data_ptr(), arg.data_ptr(), gp, 0, x.data_ptr(),
                   st.data_ptr(), sums.data_ptr(), None, m, c, beta.data_ptr(), ds.data_ptr(),
                   ws.data_ptr(), None, dx16.data_ptr(), 0)
        for name, fn in (("bn_act_pool_fwd", fwd), ("bn_bwd_reduce_pooled", red),
                         ("bn_bwd_dx_pooled", dxp)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"{name:22s} {(b, h, w, c)}: {e0.elapsed_time(e1) * 100:7.1f} us")
    print("ok")


if __name__ == "__main__":
    main()
