"""Dependent-launch overhead inside a CUDA graph: N tiny kernels in one
stream, captured and replayed (diagnostics for the many-small-kernel
Inception-BN step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1512_01274_b200 import _lib as L
    st = torch.cuda.Stream()
    x = torch.empty(1 << 20, device="cuda")
    for n_el in (256, 1 << 16, 1 << 20):
        for count in (100, 1000):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                L.call("mgx_fill", x.data_ptr(), n_el, 1.0, st.cuda_stream)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(count):
                        L.call("mgx_fill", x.data_ptr(), n_el, 1.0, st.cuda_stream)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(5):
                    g.replay()
                e1.record(st)
                torch.cuda.synchronize()
            print(f"fill {n_el:8d} floats x {count:5d} in a graph: "
                  f"{1000 * e0.elapsed_time(e1) / 5 / count:.2f} us per kernel")


if __name__ == "__main__":
    main()
