"""Debug: program kernel vs per-instruction kernels, instruction by
instruction and for whole passes (compares the arena and outputs)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import step as ostep
from paper_1512_01274_b200 import symbol, tensor as tmod, _lib as L
from paper_1512_01274_b200.engine import Engine
from paper_1512_01274_b200.executor import bind
from paper_1512_01274_b200.train import init_params, mlp, param_names

eng = Engine(device=0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 100
feats, labels = ostep.cfg1_data(B)
g = mlp([128, 64], 10)
shapes, _ = symbol.infer_shape(g, {"data": (B, 784), "label": (B,)})
p0 = init_params(g, shapes, 0); names = param_names(g)
args = {"data": tmod.from_host((B, 784), "float32", feats, engine=eng),
        "label": tmod.from_host((B,), "float32", labels, engine=eng)}
for n in names: args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=eng)
grads = {n: tmod.zeros(shapes[n], engine=eng) for n in names}
ex = bind(g, args, {n: "write" for n in names}, grads, engine=eng)
print(ex.instr_labels)


def snap():
    torch.cuda.synchronize()
    return [ex._arena.clone(), ex.outputs[0].arr.clone()] + [grads[n].arr.clone() for n in names]


def run(b, e, mode):
    st = L.lib().mgx_prog_run(ex._prog, b, e, eng.stream_handle, mode)
    assert st == 0, L.last_error()


def reset():
    ex._arena.fill_(float("nan"))
    ex.outputs[0].arr.fill_(float("nan"))
    for n in names: grads[n].arr.fill_(float("nan"))
    torch.cuda.synchronize()


n = ex._n_all
for mode in (2, 3):
    # per instruction: state from eager prefix, then instruction i in mode
    for i in range(n):
        reset(); run(0, i, 0); run(i, i + 1, 0); want = snap()
        reset(); run(0, i, 0); run(i, i + 1, mode); got = snap()
        bad = [k for k, (a, b) in enumerate(zip(want, got)) if not torch.equal(torch.nan_to_num(a, 7.0), torch.nan_to_num(b, 7.0))]
        print("instr", i, ex.instr_labels[i], "mismatch buffers" if bad else "ok", bad)
    reset(); run(0, ex._n_fwd, 0); run(ex._n_fwd, n, 0); want = snap()
    reset(); run(0, ex._n_fwd, mode); run(ex._n_fwd, n, mode); got = snap()
    for k, (a, b) in enumerate(zip(want, got)):
        print("whole", k, torch.equal(torch.nan_to_num(a, 7.0), torch.nan_to_num(b, 7.0)),
              int(torch.isnan(b).sum()))
print("err word", L.lib().mgx_prog_error)

# two executors on one engine, alternating, mode 3 vs mode 0
ex2 = bind(g, {k: (tmod.from_host(v.shape, "float32", tmod.to_numpy(v), engine=eng)) for k, v in args.items()},
           {n: "write" for n in names}, {n: tmod.zeros(shapes[n], engine=eng) for n in names}, engine=eng)
for mode in (0, 3):
    outs = []
    for e in (ex, ex2):
        e.engine.synchronize()
    for _ in range(3):
        for e in (ex, ex2):
            L.lib().mgx_prog_run(e._prog, 0, e._n_fwd, eng.stream_handle, mode)
            L.lib().mgx_prog_run(e._prog, e._n_fwd, e._n_all, eng.stream_handle, mode)
    torch.cuda.synchronize()
    print("two executors mode", mode, [float(e.outputs[0].arr.sum()) for e in (ex, ex2)])
