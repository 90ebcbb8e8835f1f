"""One training pass (forward + backward) of a configuration between
cudaProfilerStart/Stop, for `ncu --profile-from-start off` captures of the
step's kernels (DRAM traffic per kernel family, full sections of one GEMM).

    ncu --profile-from-start off --metrics ... python tools/ncu_step.py [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "inception_bn"
    import torch
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.executor import bind
    from paper_1512_01274_b200.train import aux_names, init_aux, init_params, param_names
    cfg = bench.CONFIGS[name]
    eng = Engine(device=0)
    g = bench.build_graph(name)
    b = cfg["batch"]
    given = {"data": (b,) + cfg["image"], "label": (b,)}
    shapes, _ = symbol.infer_shape(g, given)
    x, y = bench.synthetic(name, b, 0)
    p0, a0 = init_params(g, shapes, 0), init_aux(g, shapes)
    names = param_names(g)
    args = {"data": tmod.from_host(given["data"], "float32", x, engine=eng),
            "label": tmod.from_host((b,), "float32", y, engine=eng)}
    for n in names:
        args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=eng)
    for n in aux_names(g):
        args[n] = tmod.from_host(shapes[n], "float32", a0[n], engine=eng)
    grads = {n: tmod.zeros(shapes[n], engine=eng) for n in names}
    ex = bind(g, args, {n: "write" for n in names}, grads, engine=eng, dense=cfg["dense"],
              use_graph=False, strategy=cfg.get("strategy", "both"),
              split_target=cfg.get("split_target", 0))
    for _ in range(2):
        ex.forward()
        ex.backward()
    eng.wait_all()
    torch.cuda.cudart().cudaProfilerStart()
    ex.forward()
    ex.backward()
    eng.wait_all()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"{name}: one pass profiled, {ex.num_instructions} instructions")


if __name__ == "__main__":
    main()
