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
    p_want, g_want = ostep.mlp_forward_backward(p0, [128, 64], feats, labels)
    np.testing.assert_allclose(tmod.to_numpy(ex.outputs[0]), p_want, rtol=1e-2, atol=1e-3)
    for n in names:
        # gradients: bf16 operand rounding relative to the gradient's scale
        scale = float(np.abs(g_want[n]).max())
        np.testing.assert_allclose(tmod.to_numpy(grads[n]), g_want[n], rtol=2e-2,
                                   atol=2e-2 * scale, err_msg=n)


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
