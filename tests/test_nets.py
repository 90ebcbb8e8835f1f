"""Convolution-net symbols on CPU: shape inference, parameter counts,
gradient graph construction and memory plans (configs 3-5)."""

from math import prod

import pytest

from paper_1512_01274_b200 import nets, symbol
from paper_1512_01274_b200.errors import InferenceError
from paper_1512_01274_b200.planner import plan_memory
from paper_1512_01274_b200.symbol import build_gradient
from paper_1512_01274_b200.train import aux_names, param_names

CASES = [("lenet", (128, 28, 28, 1), 431_080, 4.586e6),
         ("alexnet", (128, 224, 224, 3), 62_378_344, 2.2705e9),
         ("inception_bn", (64, 224, 224, 3), 11_295_240, 3.9744e9)]


@pytest.mark.parametrize("name,shape,nparams,fwd_flops", CASES)
def test_net_shapes_params_flops(name, shape, nparams, fwd_flops):
    g = nets.NETS[name]()
    given = {"data": shape, "label": (shape[0],)}
    args, named = symbol.infer_shape(g, given)
    assert named["softmax"] == (shape[0], 10 if name == "lenet" else 1000)
    assert sum(prod(args[n]) for n in param_names(g)) == nparams
    assert abs(nets.forward_flops(g, given) / shape[0] - fwd_flops) / fwd_flops < 1e-3


def test_inception_bn_structure():
    g = nets.inception_bn()
    ops = [n.op for n in g.topo_nodes() if not n.is_variable]
    assert ops.count("Convolution") == 69 and ops.count("BatchNorm") == 69
    assert ops.count("Concat") == 10
    aux = aux_names(g)
    assert len(aux) == 2 * 69 and all(a not in param_names(g) for a in aux)
    args, named = symbol.infer_shape(g, {"data": (2, 224, 224, 3), "label": (2,)})
    assert named["global_pool"] == (2, 1, 1, 1024)


@pytest.mark.parametrize("strategy", ["none", "inplace", "coshare", "both"])
def test_convnet_gradient_graph_plans(strategy):
    g = nets.inception_bn()
    wrt = param_names(g)
    eps, _heads = build_gradient(g, wrt)
    combined = symbol.SymbolGraph(tuple(g.outputs) + tuple(eps))
    given = {"data": (2, 224, 224, 3), "label": (2,)}
    fwd = {id(n) for n in g.topo_nodes()}
    phases = [0 if (n.is_variable or id(n) in fwd) else 1 for n in combined.topo_nodes()]
    plan = plan_memory(combined, given, strategy, phases=phases)
    none = plan_memory(combined, given, "none", phases=phases)
    assert plan.total_internal_bytes <= none.total_internal_bytes


def test_conv_attribute_errors():
    data = symbol.variable("data")
    with pytest.raises(InferenceError):
        g = symbol.apply("Convolution", {"kernel": (3, 3), "num_filter": 4, "layout": "NCHW"},
                         [data])
        symbol.infer_shape(g, {"data": (1, 8, 8, 3)})
    g = symbol.apply("Convolution", {"kernel": (3, 3), "num_filter": 4, "no_bias": True}, [data],
                     name="c")
    assert g.list_arguments() == ["data", "c_weight"]
    with pytest.raises(InferenceError):
        symbol.infer_shape(symbol.apply("Concat", {"dim": 1}, [data, data]),
                           {"data": (1, 4, 4, 2)})
