"""Debug: does the cooperative program kernel run eagerly, in its own
graph, and inside an outer torch graph capture?"""
import sys, traceback
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import step as ostep
from paper_1512_01274_b200 import symbol, tensor as tmod, _lib as L
from paper_1512_01274_b200.engine import Engine
from paper_1512_01274_b200.executor import bind
from paper_1512_01274_b200.train import init_params, mlp, param_names
eng = Engine(device=0)
feats, labels = ostep.cfg1_data(100)
g = mlp([128, 64], 10)
shapes, _ = symbol.infer_shape(g, {"data": (100, 784), "label": (100,)})
p0 = init_params(g, shapes, 0); names = param_names(g)
args = {"data": tmod.from_host((100, 784), "float32", feats, engine=eng),
        "label": tmod.from_host((100,), "float32", labels, engine=eng)}
for n in names: args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=eng)
grads = {n: tmod.zeros(shapes[n], engine=eng) for n in names}
ex = bind(g, args, {n: "write" for n in names}, grads, engine=eng)
print("levels fwd", ex.levels("forward"), "bwd", ex.levels("backward"))
for mode in (2, 3):
    st = L.lib().mgx_prog_run(ex._prog, 0, ex._n_fwd, eng.stream_handle, mode)
    print("mode", mode, "status", st, L.last_error())
    st = L.lib().mgx_stream_sync(eng.stream_handle); print(" sync", st, L.last_error())
gr = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(gr, stream=eng.stream, capture_error_mode="thread_local"):
        st = L.lib().mgx_prog_run(ex._prog, 0, ex._n_fwd, eng.stream_handle, 2)
        print("in torch capture mode 2 status", st, L.last_error())
        st = L.lib().mgx_prog_run(ex._prog, ex._n_fwd, ex._n_all, eng.stream_handle, 2)
        print("in torch capture mode 2 bwd status", st, L.last_error())
    print("torch capture ok")
except Exception:
    traceback.print_exc()
