"""The north-star drop-in surface (SURVEY.md §8b "North-star aliases"):
mx.sym -> simple_bind -> forward/backward -> mx.kv.create('device') with
init/push/pull/set_optimizer, on the device, against the reference.

* config 1 through mx.*: reproduces the reference's train_distributed
  weights (train_golden ``w2b100``, 2 workers, batch 100, 500 samples) within
  the north-star tolerance rtol 1e-5 / atol 1e-6;
* LeNet (config 3) built with mx.sym.Convolution/Pooling: one data-parallel
  step's gradients and post-SGD weights vs oracle/convnet.py (bf16 operands;
  tolerances of test_convnet_gpu.py);
* an Inception-style block built with mx.sym.BatchNorm/Concat binds to the
  same graph text as nets.py's builder and trains.
"""

import numpy as np
import pytest

from oracle import convnet as oc
from oracle import step as ostep

pytestmark = pytest.mark.gpu


def _mx_mlp(mx):
    net = mx.sym.Variable("data")
    net = mx.sym.FullyConnected(data=net, num_hidden=128, name="fc1")
    net = mx.sym.Activation(data=net, act_type="relu", name="act1")
    net = mx.sym.FullyConnected(data=net, num_hidden=64, name="fc2")
    net = mx.sym.Activation(data=net, act_type="relu", name="act2")
    net = mx.sym.FullyConnected(data=net, num_hidden=10, name="out")
    return mx.sym.SoftmaxOutput(data=net, name="softmax")


def _train_mx(mx, engine, net, feats, labels, batch, workers, params0, names, epochs=1,
              dense="fp32"):
    from paper_1512_01274_b200.data import BatchOrder
    shard = batch // workers
    dshape = (shard,) + feats.shape[1:]
    exes = [net.simple_bind(mx.gpu(0), grad_req="write", engine=engine, dense=dense,
                            data=dshape, label=(shard,)) for _ in range(workers)]
    kv = mx.kv.create("device", num_devices=workers, engine=engine)
    for i, n in enumerate(names):
        kv.init(i, params0[n])
    kv.set_optimizer(mx.optimizer.SGD(learning_rate=0.05, momentum=0.9, wd=1e-4,
                                      rescale_grad=1.0 / workers))
    for i, n in enumerate(names):
        kv.pull(i, out=[ex.arg_dict[n] for ex in exes])
    order = BatchOrder(feats, labels, batch, seed=0)
    for e in range(epochs):
        for fb, lb in order.epoch(e):
            for w, ex in enumerate(exes):
                ex.forward(is_train=True, data=fb[w * shard:(w + 1) * shard],
                           label=lb[w * shard:(w + 1) * shard])
                ex.backward()
            for i, n in enumerate(names):
                kv.push(i, [ex.grad_dict[n] for ex in exes])
            for i, n in enumerate(names):
                kv.pull(i, out=[ex.arg_dict[n] for ex in exes])
    return exes, kv


def test_config1_through_mx_matches_reference(engine, train_golden):
    from paper_1512_01274_b200 import mx
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.train import init_params, param_names
    net = _mx_mlp(mx)
    feats, labels = ostep.cfg1_data(500)
    shapes, _ = __import__("paper_1512_01274_b200.symbol", fromlist=["x"]).infer_shape(
        net.graph, {"data": (50, 784), "label": (50,)})
    names = param_names(net.graph)
    assert names == ["fc1_weight", "fc1_bias", "fc2_weight", "fc2_bias", "out_weight", "out_bias"]
    exes, kv = _train_mx(mx, engine, net, feats, labels, 100, 2,
                         init_params(net.graph, shapes, 0), names)
    for n in names:
        for ex in exes:
            np.testing.assert_allclose(tmod.to_numpy(ex.arg_dict[n]),
                                       train_golden[f"dist_w2b100_n500_{n}"], rtol=1e-5,
                                       atol=1e-6, err_msg=n)
    kv.close()


def _mx_lenet(mx):
    net = mx.sym.Variable("data")
    net = mx.sym.Convolution(data=net, kernel=(5, 5), num_filter=20, name="conv1")
    net = mx.sym.Activation(data=net, act_type="tanh", name="tanh1")
    net = mx.sym.Pooling(data=net, kernel=(2, 2), stride=(2, 2), pool_type="max", name="pool1")
    net = mx.sym.Convolution(data=net, kernel=(5, 5), num_filter=50, name="conv2")
    net = mx.sym.Activation(data=net, act_type="tanh", name="tanh2")
    net = mx.sym.Pooling(data=net, kernel=(2, 2), stride=(2, 2), pool_type="max", name="pool2")
    net = mx.sym.Flatten(data=net, name="flatten")
    net = mx.sym.FullyConnected(data=net, num_hidden=500, name="fc1")
    net = mx.sym.Activation(data=net, act_type="tanh", name="tanh3")
    net = mx.sym.FullyConnected(data=net, num_hidden=10, name="fc2")
    return mx.sym.SoftmaxOutput(data=net, name="softmax")


def test_lenet_through_mx_matches_oracle(engine):
    from paper_1512_01274_b200 import mx, symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.train import init_aux, init_params, param_names
    net = _mx_lenet(mx)
    rs = np.random.RandomState(7)
    feats = rs.randn(32, 28, 28, 1).astype(np.float32)
    labels = rs.randint(0, 10, 32).astype(np.float32)
    shapes, _ = symbol.infer_shape(net.graph, {"data": (16, 28, 28, 1), "label": (16,)})
    names = param_names(net.graph)
    p0 = init_params(net.graph, shapes, 3)
    exes, kv = _train_mx(mx, engine, net, feats, labels, 32, 2, p0, names)
    # the one step's batch, as BatchOrder(seed 0) gave it
    from paper_1512_01274_b200.data import BatchOrder
    fb, lb = next(BatchOrder(feats, labels, 32, seed=0).epoch(0))
    total = {}
    for w in range(2):
        vals = {"data": fb[16 * w:16 * (w + 1)], "label": lb[16 * w:16 * (w + 1)], **p0,
                **init_aux(net.graph, shapes)}
        _o, gw, _a = oc.run_graph(net.graph, vals, wrt=names, bf16_operands=True)
        for n in names:
            total[n] = total.get(n, 0) + gw[n]
        for n in names:
            scale = float(np.abs(gw[n]).max())
            np.testing.assert_allclose(tmod.to_numpy(exes[w].grad_dict[n]), gw[n], rtol=2e-2,
                                       atol=2e-2 * scale + 1e-6, err_msg=n)
    for n in names:
        gmean = total[n] / 2
        want = p0[n] - 0.05 * (gmean + 1e-4 * p0[n])  # first step: v = -eta*(g + wd*w)
        scale = 0.05 * (float(np.abs(gmean).max()) or 1.0)
        for ex in exes:
            np.testing.assert_allclose(tmod.to_numpy(ex.arg_dict[n]), want, rtol=1e-3,
                                       atol=3e-2 * scale, err_msg=n)
    kv.close()


def _mx_block(mx, classes=10):
    def factory(x, f, k, name, s=(1, 1), p=(0, 0)):
        x = mx.sym.Convolution(data=x, kernel=k, num_filter=f, stride=s, pad=p,
                               name=f"conv_{name}")
        x = mx.sym.BatchNorm(data=x, fix_gamma=False, name=f"bn_{name}")
        return mx.sym.Activation(data=x, act_type="relu", name=f"relu_{name}")

    data = mx.sym.Variable("data")
    a = factory(data, 8, (1, 1), "a")
    b = factory(factory(data, 8, (1, 1), "b_red"), 16, (3, 3), "b", p=(1, 1))
    c = mx.sym.Pooling(data=data, kernel=(3, 3), stride=(1, 1), pad=(1, 1), pool_type="avg",
                       name="c_pool")
    net = mx.sym.Concat(a, b, c, name="concat")
    net = mx.sym.Pooling(data=net, kernel=(1, 1), pool_type="avg", global_pool=True,
                         name="global_pool")
    net = mx.sym.Flatten(data=net, name="flatten")
    net = mx.sym.FullyConnected(data=net, num_hidden=classes, name="fc")
    return mx.sym.SoftmaxOutput(data=net, name="softmax")


def test_mx_batchnorm_concat_block_trains(engine):
    """BatchNorm aux states start at (0, 1) and move; gradients match the
    oracle; loss decreases under the mx.kv SGD store."""
    from paper_1512_01274_b200 import mx, symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.train import init_aux, init_params, param_names
    net = _mx_block(mx)
    assert net.list_auxiliary_states() == ["bn_a_moving_mean", "bn_a_moving_var",
                                           "bn_b_red_moving_mean", "bn_b_red_moving_var",
                                           "bn_b_moving_mean", "bn_b_moving_var"]
    shapes, _ = symbol.infer_shape(net.graph, {"data": (8, 12, 12, 8), "label": (8,)})
    names = param_names(net.graph)
    p0 = init_params(net.graph, shapes, 1)
    ex = net.simple_bind(mx.gpu(0), engine=engine, data=(8, 12, 12, 8), label=(8,))
    assert set(ex.grad_dict) == set(names)
    for n in names:
        tmod.load_host(ex.arg_dict[n], p0[n])
    rs = np.random.RandomState(2)
    x = rs.randn(8, 12, 12, 8).astype(np.float32)
    y = rs.randint(0, 10, 8).astype(np.float32)
    ex.forward(data=x, label=y)
    ex.backward()
    aux0 = init_aux(net.graph, shapes)
    _o, want, aux_want = oc.run_graph(net.graph, {"data": x, "label": y, **p0, **aux0},
                                      wrt=names, bf16_operands=True)
    for n in names:
        scale = float(np.abs(want[n]).max())
        np.testing.assert_allclose(tmod.to_numpy(ex.grad_dict[n]), want[n], rtol=2e-2,
                                   atol=2e-2 * scale + 1e-6, err_msg=n)
    for n in net.list_auxiliary_states():
        np.testing.assert_allclose(tmod.to_numpy(ex.aux_dict[n]), aux_want[n], rtol=1e-4,
                                   atol=1e-5, err_msg=n)
