"""Implicit-GEMM convolution forward (mgx_gemm_bf16_conv mode 1) at the
Inception-BN shapes, timed as 20 launches captured in one CUDA graph (no
host overhead in the number): us per launch and TFLOP/s.

    python tools/conv_gemm_bench.py [splits]      (splits 1 = none, 0 = auto)
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [  # (B, H, W, C, F, k, s, p)
    (64, 27, 27, 96, 96, 3, 1, 1),     # 3a double_3x3_1 [46656, 96, 864]
    (64, 27, 27, 64, 96, 3, 1, 1),     # 3a 3x3 [46656, 96, 576]
    (64, 14, 14, 192, 256, 3, 1, 1),   # 4e double_3x3_0 [12544, 256, 1728]
    (64, 14, 14, 128, 192, 3, 1, 1),   # 4d 3x3 [12544, 192, 1152]
    (64, 7, 7, 192, 320, 3, 1, 1),     # 5a 3x3 [3136, 320, 1728]
    (64, 14, 14, 576, 128, 1, 1, 0),   # 4x 1x1 reduce [12544, 128, 576]
    (64, 55, 55, 64, 192, 3, 1, 1),    # conv_2 [193600, 192, 576]
]


def main():
    import torch
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.engine import Engine
    Engine(device=0)
    splits = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    for b, h, w, c, f, k, s, p in SHAPES:
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        m, kk = b * ho * wo, k * k * c
        ldk = -(-kk // 8) * 8
        x = torch.randn(b, h, w, c, device="cuda").to(torch.bfloat16)
        wt = torch.randn(f, ldk, device="cuda").to(torch.bfloat16)
        out = torch.empty(m, f, device="cuda")
        ws = torch.empty(148 * m * f + 1, device="cuda") if splits != 1 else None
        geom = np.array([b, h, w, c, (k << 16) | k, (s << 16) | s, (p << 16) | p], np.int64)
        gp = geom.ctypes.data_as(ctypes.c_void_p)
        st = torch.cuda.Stream()

        def launch(stream):
            L.call("mgx_gemm_bf16_conv", 1, x.data_ptr(), gp, wt.data_ptr(), ldk, None,
                   out.data_ptr(), f, m, f, kk, 0, splits,
                   ws.data_ptr() if ws is not None else None, None, stream)
        with torch.cuda.stream(st):
            for _ in range(3):
                launch(st.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20):
                launch(st.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        tf = 2 * m * f * kk / us / 1e6
        print(f"conv [{m}, {f}, {kk}] C={c} k={k}: {us:7.1f} us  {tf:6.1f} TFLOP/s")


if __name__ == "__main__":
    main()
