"""Debug: train_distributed (W=2, batch 100) step by step, program kernel on
and off, reporting the first NaN and the executors' fused state."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import step as ostep
from paper_1512_01274_b200 import symbol, tensor as tmod
from paper_1512_01274_b200.engine import Engine
from paper_1512_01274_b200.kvstore import KVStore
from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
from paper_1512_01274_b200.train import DataParallelStep, init_params, mlp

feats, labels = ostep.cfg1_data(500)
res = {}
for fused in (False, True):
    eng = Engine(device=0)
    symbol.reset_names()
    g = mlp([128, 64], 10)
    given = {"data": (50, 784), "label": (50,)}
    shapes, _ = symbol.infer_shape(g, given)
    kv = KVStore(1, 2, engine=eng)
    st = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng)
    for ex in st.execs.values():
        ex._fused = None if fused else False
    kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=2))
    hist = []
    for s in range(5):
        rows = slice(s * 100, s * 100 + 100)
        f, l = feats[rows], labels[rows]
        st.step({0: (f[:50], l[:50]), 1: (f[50:], l[50:])})
        outs = [st.outputs(w) for w in (0, 1)]
        grads = {n: tmod.to_numpy(st.grads[0][n]) for n in st.names}
        w = {n: tmod.to_numpy(st.args[0][n]) for n in st.names}
        hist.append((outs, grads, w))
        print("fused", fused, "step", s, "nan out", [int(np.isnan(o).sum()) for o in outs],
              "nan grads", {n: int(np.isnan(v).sum()) for n, v in grads.items()},
              "nan w", {n: int(np.isnan(v).sum()) for n, v in w.items()},
              "uses", [e.uses_program_kernel for e in st.execs.values()],
              [getattr(e, "fused_fallback_reason", "") for e in st.execs.values()])
    res[fused] = hist
    kv.close()
for s in range(5):
    a, b = res[False][s], res[True][s]
    print("step", s, "outs equal", [np.array_equal(x, y) for x, y in zip(a[0], b[0])],
          "grads equal", all(np.array_equal(a[1][n], b[1][n]) for n in a[1]),
          "w equal", all(np.array_equal(a[2][n], b[2][n]) for n in a[2]))
