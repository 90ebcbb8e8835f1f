"""bf16 tensor-core dense path (executor dense="bf16"): FC forward, dX and
dW run as tcgen05 GEMMs on bf16 operand copies with fp32 accumulation.

Stated tolerances (probed on the reference): after 1 step
rtol 1e-2 / atol 1e-3; after 5 steps rtol 5e-2 / atol 5e-3."""

import numpy as np
import pytest

from oracle import step as ostep

pytestmark = pytest.mark.gpu


def test_bf16_executor_uses_tensor_core_program(engine):
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.executor import bind
    from paper_1512_01274_b200.train import init_params, mlp, param_names
    feats, labels = ostep.cfg1_data(100)
    g = mlp([128, 64], 10)
    shapes, _ = symbol.infer_shape(g, {"data": (100, 784), "label": (100,)})
    p0 = init_params(g, shapes, 0)
    names = param_names(g)
    args = {"data": tmod.from_host((100, 784), "float32", feats, engine=engine),
            "label": tmod.from_host((100,), "float32", labels, engine=engine)}
    for n in names:
        args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=engine)
    grads = {n: tmod.zeros(shapes[n], engine=engine) for n in names}
    ex = bind(g, args, {n: "write" for n in names}, grads, engine=engine, dense="bf16")
    ops = [lbl for lbl, cost in zip(ex.instr_labels, ex.instr_costs)]
    assert len(ops) > 10
    ex.forward()
    ex.backward()
    p_want, g_want = bf16_emulated_step(p0, [128, 64], feats, labels)
    np.testing.assert_allclose(tmod.to_numpy(ex.outputs[0]), p_want, rtol=1e-3, atol=1e-5)
    for n in names:
        # same bf16-rounded operands, fp32 tensor-core accumulation vs fp64:
        # differences come from accumulation order and from a bf16 operand
        # that rounds the other way after an fp32 ulp difference upstream
        scale = float(np.abs(g_want[n]).max())
        np.testing.assert_allclose(tmod.to_numpy(grads[n]), g_want[n], rtol=1e-2,
                                   atol=2e-3 * scale, err_msg=n)


def bf16(x):
    """Round fp32 to bf16 (nearest even), returned as fp32 (the value the
    cast kernel stores)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def bf16_emulated_step(params, hidden, x, label):
    """The dense="bf16" lowering restated in numpy: every tensor-core GEMM
    operand rounded to bf16, products accumulated in fp64, results fp32;
    bias/db/softmax/relu as the fp32 path computes them."""
    layers = [f"fc{i}" for i in range(1, len(hidden) + 1)] + ["out"]
    f32 = np.float32
    ins, outs = [], []
    h = x.astype(f32)
    for li, name in enumerate(layers):
        ins.append(h)
        z = (bf16(h).astype(np.float64) @ bf16(params[f"{name}_weight"]).astype(np.float64).T)
        z = (z.astype(f32) + params[f"{name}_bias"]).astype(f32)
        h = np.maximum(z, 0).astype(f32) if li < len(layers) - 1 else z
        outs.append(h)
    e = np.exp(h.astype(np.float64) - h.max(axis=1, keepdims=True))
    p = (e / e.sum(axis=1, keepdims=True)).astype(f32)
    onehot = np.eye(p.shape[1], dtype=f32)[label.astype(np.int64)]
    d = ((p - onehot) / f32(p.shape[0])).astype(f32)
    grads = {}
    for li in range(len(layers) - 1, -1, -1):
        name = layers[li]
        grads[f"{name}_weight"] = (bf16(d).astype(np.float64).T
                                   @ bf16(ins[li]).astype(np.float64)).astype(f32)
        grads[f"{name}_bias"] = d.astype(np.float64).sum(axis=0).astype(f32)
        if li > 0:
            dx = (bf16(d).astype(np.float64)
                  @ bf16(params[f"{name}_weight"]).astype(np.float64)).astype(f32)
            d = np.where(outs[li - 1] > 0, dx, f32(0)).astype(f32)
    return p, grads


@pytest.mark.parametrize("n,rtol,atol", [(100, 1e-2, 1e-3), (500, 5e-2, 5e-3)])
def test_bf16_training_within_stated_tolerance(engine, train_golden, n, rtol, atol):
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200.optim import SGDConfig
    from paper_1512_01274_b200.train import mlp, train_distributed
    symbol.reset_names()
    feats, labels = ostep.cfg1_data(500)
    _rep, params = train_distributed(mlp([128, 64], 10), (feats[:n], labels[:n]),
                                     SGDConfig(0.05, 0.9, 1e-4), epochs=1, batch=100, machines=1,
                                     workers=2, engine=engine, dense="bf16")
    want, _ = ostep.train_distributed([128, 64], 10, feats[:n], labels[:n], 0.05, 0.9, 1e-4,
                                      epochs=1, batch=100, machines=1, workers=2)
    for k, v in want.items():
        np.testing.assert_allclose(params[k], v, rtol=rtol, atol=atol, err_msg=k)
