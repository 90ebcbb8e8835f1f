"""mx.* alias layer on the CPU: graph structure and argument checks
(no device work)."""

import pytest

from test_mx_gpu import _mx_block, _mx_lenet, _mx_mlp


def test_mx_lenet_is_the_config3_graph():
    from paper_1512_01274_b200 import mx, nets, symbol
    assert symbol.save(_mx_lenet(mx).graph) == symbol.save(nets.lenet(10))



def test_mx_mlp_is_the_config1_graph():
    from paper_1512_01274_b200 import mx, symbol
    from paper_1512_01274_b200.train import mlp
    text = symbol.save(_mx_mlp(mx).graph)
    symbol.reset_names()
    assert text == symbol.save(mlp([128, 64], 10))


def test_mx_aux_states_and_shapes():
    from paper_1512_01274_b200 import mx
    net = _mx_block(mx)
    args, outs, _aux = net.infer_shape(data=(8, 12, 12, 8), label=(8,))
    assert outs == [(8, 10)]
    assert all(n in net.list_arguments() for n in net.list_auxiliary_states())
    assert len(args) == len(net.list_arguments())


def test_kv_create_rejects_multi_gpu_contexts_in_one_process():
    from paper_1512_01274_b200 import mx
    from paper_1512_01274_b200.errors import ArgumentError
    with pytest.raises(ArgumentError):
        mx.kv.create("device", ctx=[mx.gpu(0), mx.gpu(1)])
