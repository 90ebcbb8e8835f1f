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


def test_weight_gradient_hoisting_keeps_a_topological_order():
    """executor._hoist_weight_grads (DataParallelStep's hoist_wgrad): every
    weight / bias gradient moves up to one node after its last input, the
    result is still a topological order of the combined graph, and nothing
    else changes order."""
    from paper_1512_01274_b200.executor import (_gradient_request, _hoist_weight_grads,
                                                launch_order, prune)
    symbol.reset_names()
    g = nets.inception_bn(1000)
    given = {"data": (8, 224, 224, 3), "label": (8,)}
    shapes, _ = symbol.infer_shape(g, given)
    fg = prune(g, None)
    names = param_names(fg)
    wrt, grad_eps, head_pairs, combined = _gradient_request(fg, {n: "write" for n in names})
    fnamed = symbol.infer_shape(fg, given)[1]
    given2 = {a: shapes[a] for a in fg.list_arguments()}
    given2.update((hv.name, fnamed[nd.name]) for hv, (nd, _s) in head_pairs)
    topo = combined.topo_nodes()
    index = {id(nd): i for i, nd in enumerate(topo)}
    fids = {id(nd) for nd in fg.topo_nodes()}
    phase = [int(nd.op is not None and id(nd) not in fids) for nd in topo]
    plan = plan_memory(combined, given2, "inplace", phases=phase)
    order = launch_order(topo, index, phase, plan.extra_dep_edges)
    new = _hoist_weight_grads(order, topo, index, phase)
    assert sorted(new) == sorted(order)
    pos = {n: q for q, n in enumerate(new)}
    for i in new:
        for src, _ in topo[i].inputs:
            if src.op is not None:
                assert pos[index[id(src)]] < pos[i], (topo[i].name, src.name)
    wg = [i for i in order if topo[i].op == "Backward"
          and topo[i].attrs["of"] in ("Convolution", "FullyConnected")
          and topo[i].attrs["slot"] in (1, 2)]
    old = {n: q for q, n in enumerate(order)}
    assert sum(pos[i] < old[i] for i in wg) > len(wg) // 2  # most move up
    rest = [i for i in new if i not in set(wg)]
    assert rest == [i for i in order if i not in set(wg)]
