"""Symbol builders for the convolution-net configurations (BASELINE.json
configs 3-5), in the style of the reference's ``mlp`` builder
(train.py:57-67) and MXNet's example symbols the paper trains (arXiv
1512.01274 §4: Inception-BN / GoogLeNet-BN on ILSVRC12).

All three are channels-last (data (batch, height, width, channels)).

* ``lenet``: conv5x5x20-tanh-maxpool2, conv5x5x50-tanh-maxpool2, fc500-tanh,
  fc(classes), SoftmaxOutput (MXNet's LeNet example).
* ``alexnet``: the AlexNet layer stack (conv11x11/4 96, conv5x5 256,
  3 x conv3x3, fc 4096 x 2 -- 61M parameters, fc6 = 4096 x 9216) without LRN
  and dropout (neither is a reference or north-star operator).
* ``inception_bn``: MXNet's Inception-BN (ConvFactory = Conv-BN-ReLU,
  InceptionFactoryA/B), 1000 classes by default.
"""

from __future__ import annotations

from . import symbol
from .symbol import SymbolGraph


def _apply(op, attrs, ins, name):
    return symbol.apply(op, attrs, ins, name=name)


def lenet(classes: int = 10) -> SymbolGraph:
    net = symbol.variable("data")
    net = _apply("Convolution", {"kernel": (5, 5), "num_filter": 20}, [net], "conv1")
    net = _apply("Activation", {"act_type": "tanh"}, [net], "tanh1")
    net = _apply("Pooling", {"kernel": (2, 2), "stride": (2, 2), "pool_type": "max"}, [net], "pool1")
    net = _apply("Convolution", {"kernel": (5, 5), "num_filter": 50}, [net], "conv2")
    net = _apply("Activation", {"act_type": "tanh"}, [net], "tanh2")
    net = _apply("Pooling", {"kernel": (2, 2), "stride": (2, 2), "pool_type": "max"}, [net], "pool2")
    net = _apply("Flatten", {}, [net], "flatten")
    net = _apply("FullyConnected", {"num_hidden": 500}, [net], "fc1")
    net = _apply("Activation", {"act_type": "tanh"}, [net], "tanh3")
    net = _apply("FullyConnected", {"num_hidden": classes}, [net], "fc2")
    return _apply("SoftmaxOutput", {}, [net], "softmax")


def alexnet(classes: int = 1000) -> SymbolGraph:
    net = symbol.variable("data")

    def conv(x, name, f, k, s=1, p=0):
        x = _apply("Convolution", {"kernel": (k, k), "num_filter": f, "stride": (s, s),
                                   "pad": (p, p)}, [x], name)
        return _apply("Activation", {"act_type": "relu"}, [x], f"relu_{name}")

    def pool(x, name):
        return _apply("Pooling", {"kernel": (3, 3), "stride": (2, 2), "pool_type": "max"}, [x], name)

    net = pool(conv(net, "conv1", 96, 11, 4, 2), "pool1")
    net = pool(conv(net, "conv2", 256, 5, 1, 2), "pool2")
    net = conv(net, "conv3", 384, 3, 1, 1)
    net = conv(net, "conv4", 384, 3, 1, 1)
    net = pool(conv(net, "conv5", 256, 3, 1, 1), "pool5")
    net = _apply("Flatten", {}, [net], "flatten")
    for i in (6, 7):
        net = _apply("FullyConnected", {"num_hidden": 4096}, [net], f"fc{i}")
        net = _apply("Activation", {"act_type": "relu"}, [net], f"relu{i}")
    net = _apply("FullyConnected", {"num_hidden": classes}, [net], "fc8")
    return _apply("SoftmaxOutput", {}, [net], "softmax")


def _conv_factory(x, f, k, name, s=(1, 1), p=(0, 0)):
    x = _apply("Convolution", {"kernel": k, "num_filter": f, "stride": s, "pad": p}, [x],
               f"conv_{name}")
    x = _apply("BatchNorm", {}, [x], f"bn_{name}")
    return _apply("Activation", {"act_type": "relu"}, [x], f"relu_{name}")


def _inception_a(x, n1, n3r, n3, nd3r, nd3, pool, proj, name):
    c1 = _conv_factory(x, n1, (1, 1), f"{name}_1x1")
    c3r = _conv_factory(x, n3r, (1, 1), f"{name}_3x3_reduce")
    c3 = _conv_factory(c3r, n3, (3, 3), f"{name}_3x3", p=(1, 1))
    cd3r = _conv_factory(x, nd3r, (1, 1), f"{name}_double_3x3_reduce")
    cd3 = _conv_factory(cd3r, nd3, (3, 3), f"{name}_double_3x3_0", p=(1, 1))
    cd3 = _conv_factory(cd3, nd3, (3, 3), f"{name}_double_3x3_1", p=(1, 1))
    pl = _apply("Pooling", {"kernel": (3, 3), "stride": (1, 1), "pad": (1, 1), "pool_type": pool},
                [x], f"{pool}_pool_{name}_pool")
    cp = _conv_factory(pl, proj, (1, 1), f"{name}_proj")
    return _apply("Concat", {"num_args": 4}, [c1, c3, cd3, cp], f"ch_concat_{name}_chconcat")


def _inception_b(x, n3r, n3, nd3r, nd3, name):
    c3r = _conv_factory(x, n3r, (1, 1), f"{name}_3x3_reduce")
    c3 = _conv_factory(c3r, n3, (3, 3), f"{name}_3x3", s=(2, 2), p=(1, 1))
    cd3r = _conv_factory(x, nd3r, (1, 1), f"{name}_double_3x3_reduce")
    cd3 = _conv_factory(cd3r, nd3, (3, 3), f"{name}_double_3x3_0", p=(1, 1))
    cd3 = _conv_factory(cd3, nd3, (3, 3), f"{name}_double_3x3_1", s=(2, 2), p=(1, 1))
    pl = _apply("Pooling", {"kernel": (3, 3), "stride": (2, 2), "pad": (1, 1), "pool_type": "max"},
                [x], f"max_pool_{name}_pool")
    return _apply("Concat", {"num_args": 3}, [c3, cd3, pl], f"ch_concat_{name}_chconcat")


def inception_bn(classes: int = 1000) -> SymbolGraph:
    net = symbol.variable("data")
    net = _conv_factory(net, 64, (7, 7), "1", s=(2, 2), p=(3, 3))
    net = _apply("Pooling", {"kernel": (3, 3), "stride": (2, 2), "pool_type": "max"}, [net], "pool_1")
    net = _conv_factory(net, 64, (1, 1), "2_red")
    net = _conv_factory(net, 192, (3, 3), "2", p=(1, 1))
    net = _apply("Pooling", {"kernel": (3, 3), "stride": (2, 2), "pool_type": "max"}, [net], "pool_2")
    net = _inception_a(net, 64, 64, 64, 64, 96, "avg", 32, "3a")
    net = _inception_a(net, 64, 64, 96, 64, 96, "avg", 64, "3b")
    net = _inception_b(net, 128, 160, 64, 96, "3c")
    net = _inception_a(net, 224, 64, 96, 96, 128, "avg", 128, "4a")
    net = _inception_a(net, 192, 96, 128, 96, 128, "avg", 128, "4b")
    net = _inception_a(net, 160, 128, 160, 128, 160, "avg", 128, "4c")
    net = _inception_a(net, 96, 128, 192, 160, 192, "avg", 128, "4d")
    net = _inception_b(net, 128, 192, 192, 256, "4e")
    net = _inception_a(net, 352, 192, 320, 160, 224, "avg", 128, "5a")
    net = _inception_a(net, 352, 192, 320, 192, 224, "max", 128, "5b")
    net = _apply("Pooling", {"kernel": (7, 7), "stride": (1, 1), "pool_type": "avg",
                             "global_pool": True}, [net], "global_pool")
    net = _apply("Flatten", {}, [net], "flatten")
    net = _apply("FullyConnected", {"num_hidden": classes}, [net], "fc1")
    return _apply("SoftmaxOutput", {}, [net], "softmax")


NETS = {"lenet": lenet, "alexnet": alexnet, "inception_bn": inception_bn}


def forward_flops(g: SymbolGraph, shapes_given) -> int:
    """Multiply-add FLOPs (x2) of the Convolution and FullyConnected nodes of
    one forward pass (the roofline numerator of a training step is ~3x)."""
    from math import prod
    _args, named = symbol.infer_shape(g, shapes_given)
    total = 0
    for n in g.topo_nodes():
        if n.op == "Convolution":
            out = named[n.name]
            w = named[n.inputs[1][0].name]
            total += 2 * prod(out) * prod(w[1:])
        elif n.op == "FullyConnected":
            out = named[n.name]
            w = named[n.inputs[1][0].name]
            total += 2 * out[0] * prod(w)
    return total
