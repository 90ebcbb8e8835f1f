"""Time mgx_gemm_bf16_tc_ex on conv-net shapes (CUDA events, warm L2
flushed): ms, TFLOP/s, output GB/s.  Diagnostics for the GEMM kernel.

    python tools/gemm_bench.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [  # (M, N, K, a_mn, b_mn, splits)
    (193600, 64, 64, 0, 0, 1),      # conv_2_red forward
    (46656, 192, 64, 0, 1, 1),      # 1x1 dgrad
    (193600, 576, 192, 0, 1, 1),    # 3x3 dgrad (dcol)
    (193600, 192, 576, 0, 0, 1),    # conv_2 forward
    (46656, 96, 864, 0, 0, 1),      # 3x3 forward
    (192, 576, 193600, 1, 1, 0),    # wgrad split-K
    (12544, 192, 1728, 0, 0, 1),    # 14x14 3x3 forward (one tile per CTA)
    (3136, 224, 2016, 0, 0, 0),     # 7x7 3x3 forward (split-K)
    (8192, 8192, 8192, 0, 0, 1),    # big square
]


def main():
    import torch
    from paper_1512_01274_b200 import _lib as L
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    flush = torch.empty(64 << 20, device="cuda")
    for m, n, k, amn, bmn, sp in SHAPES:
        pad = lambda v: -(-v // 8) * 8  # noqa: E731
        lda = pad(m) if amn else pad(k)
        ldb = pad(n) if bmn else pad(k)
        a = torch.randn((k if amn else m) * lda, device="cuda").to(torch.bfloat16)
        b = torch.randn((k if bmn else n) * ldb, device="cuda").to(torch.bfloat16)
        c = torch.empty(m * n, device="cuda")
        ws = torch.empty(200 * m * n if sp == 0 else 1, device="cuda")
        args = (a.data_ptr(), lda, amn, b.data_ptr(), ldb, bmn, None, c.data_ptr(), n, m, n, k, 0,
                sp, ws.data_ptr(), None, 0)
        for _ in range(3):
            L.call("mgx_gemm_bf16_tc_ex", *args)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.call("mgx_gemm_bf16_tc_ex", *args)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / reps
        byt = 2 * (m * k + n * k) + 4 * m * n
        # cuBLAS (torch.matmul, bf16 in / bf16 out) on the same shape, for context
        ta = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        tb = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            torch.matmul(ta, tb)
        torch.cuda.synchronize()
        cb = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(ta, tb)
            e1.record()
            torch.cuda.synchronize()
            cb += e0.elapsed_time(e1)
        cb /= reps
        print(f"M={m:7d} N={n:5d} K={k:7d} amn={amn} bmn={bmn}: {ms * 1e3:9.1f} us "
              f"{2 * m * n * k / ms / 1e9:8.1f} TF/s  {byt / ms / 1e6:8.1f} GB/s   "
              f"| cuBLAS {cb * 1e3:8.1f} us {2 * m * n * k / cb / 1e9:8.1f} TF/s", flush=True)
    # write-bandwidth reference: fill of the largest output
    c = torch.empty(193600 * 576, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.call("mgx_fill", c.data_ptr(), c.numel(), 0.0, 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"fill {c.numel() * 4 / 1e6:.0f} MB: {ms * 1e3:.1f} us {c.numel() * 4 / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
