"""Which groups each embedded KVStore round waits for (hazard dependencies
of the executor's backward program), for bench.py's configuration at N=1.

    python tools/kv_deps.py [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "inception_bn"
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params
    eng = Engine(device=0)
    cfg = bench.CONFIGS[name]
    per = cfg["batch"]
    kv = KVStore(1, 1, engine=eng)
    g = bench.build_graph(name)
    given = {"data": (per,) + cfg["image"], "label": (per,)}
    shapes, _ = symbol.infer_shape(g, given)
    step = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng,
                            dense=cfg["dense"], strategy=cfg.get("strategy", "both"),
                            split_target=cfg.get("split_target", 0),
                            hoist_wgrad=cfg.get("hoist_wgrad"))
    kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=1))
    ex = step.execs[0]
    groups = ex._groups[1]
    deps = ex._group_deps(groups)
    base = ex._n_fwd
    lab = ex.instr_labels
    ops = ex.instr_ops
    for gi, gr in enumerate(groups):
        if ops[base + gr[0]] != L.OP_KV_ROUND:
            continue
        ds = sorted(deps[gi])
        print(f"group {gi} {lab[base + gr[0]]}: {len(ds)} deps, latest:",
              [(d, lab[base + groups[d][0]]) for d in ds[-4:]])
    print("backward groups:", len(groups))
    kv.close()


if __name__ == "__main__":
    main()
