"""Time the config-1 MLP forward+backward in each program mode, plus the
program kernel's per-level completion times."""
import sys, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import step as ostep
from paper_1512_01274_b200 import symbol, tensor as tmod, _lib as L
from paper_1512_01274_b200.engine import Engine
from paper_1512_01274_b200.executor import bind
from paper_1512_01274_b200.train import init_params, mlp, param_names
B = int(sys.argv[1]) if len(sys.argv) > 1 else 100
eng = Engine(device=0)
feats, labels = ostep.cfg1_data(B)
g = mlp([128, 64], 10)
shapes, _ = symbol.infer_shape(g, {"data": (B, 784), "label": (B,)})
p0 = init_params(g, shapes, 0); names = param_names(g)
args = {"data": tmod.from_host((B, 784), "float32", feats, engine=eng),
        "label": tmod.from_host((B,), "float32", labels, engine=eng)}
for n in names: args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=eng)
grads = {n: tmod.zeros(shapes[n], engine=eng) for n in names}
ex = bind(g, args, {n: "write" for n in names}, grads, engine=eng)
s = eng.stream_handle
for mode in (0, 1, 2, 3):
    for _ in range(20):
        L.lib().mgx_prog_run(ex._prog, 0, ex._n_fwd, s, mode); L.lib().mgx_prog_run(ex._prog, ex._n_fwd, ex._n_all, s, mode)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    for _ in range(200):
        L.lib().mgx_prog_run(ex._prog, 0, ex._n_fwd, s, mode); L.lib().mgx_prog_run(ex._prog, ex._n_fwd, ex._n_all, s, mode)
    b.record(eng.stream); torch.cuda.synchronize()
    print(f"B={B} mode {mode}: {a.elapsed_time(b) / 200 * 1000:.1f} us per fwd+bwd")
for name, (lo, hi) in (("fwd", (0, ex._n_fwd)), ("bwd", (ex._n_fwd, ex._n_all))):
    nl, grid, lv = ex.levels("forward" if name == "fwd" else "backward")
    ns = (ctypes.c_double * nl)()
    for _ in range(3):
        L.call("mgx_prog_time_levels", ex._prog, lo, hi, s, ns)
    print(name, "grid", grid, "levels", lv, "level done at (us):", [round(x / 1000, 2) for x in ns])
prof = ex.profile()
print("per-instruction (graph w/ event nodes, us):", [(l, round(m * 1000, 1)) for l, m in prof])
