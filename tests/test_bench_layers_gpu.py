"""Every convolution geometry of the benchmarked Inception-BN, at the bench
batch (64), checked on its own against a float64 reference.

The whole-net comparison (test_bench_config_gpu.py) can only be as tight as
the bf16-rounding noise floor of a 63-convolution-deep net.  Here each
distinct (H, W, C, F, kernel, stride, pad) of ``nets.inception_bn(1000)`` at
batch 64 is bound alone through the executor in the production mode
(``dense="bf16"``, default lanes), so the shape-dependent kernel variant the
bench runs for that layer -- TMA-im2col or gathered implicit GEMM, plain TMA
GEMM for 1x1, the stem's column-matrix path for C=3, stride-2 data gradients
as transposed convolutions, the auto split-K count for (M, N, K) -- runs on
exactly the bench's shapes, and forward, dX, dW and db are checked tightly.

Reference: torch float64 convolutions on the GPU over the same bf16-rounded
operands (x, w, dY), i.e. exactly the rounding the device applies; what is
left is fp32 (device) vs fp64 accumulation order.  Tolerance: rtol 1e-4,
atol = max(1e-4 * max(1, sqrt(K)/8), 1e-5 * max|ref|) (K = the contraction
length of each product; the second term is fp32 accumulation over the
longest contractions, e.g. conv_2's weight gradient sums K = 193,600
products of magnitude ~1 into values of ~2e3).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PER = 64


def _geometries():
    from paper_1512_01274_b200 import nets, symbol
    symbol.reset_names()
    g = nets.inception_bn(1000)
    _a, named = symbol.infer_shape(g, {"data": (PER, 224, 224, 3), "label": (PER,)})
    seen = {}
    for n in g.topo_nodes():
        if n.op != "Convolution":
            continue
        src = n.inputs[0][0]
        b, h, w, c = named[src.name]
        a = n.attrs
        pair = lambda v: (v, v) if isinstance(v, int) else tuple(v)  # noqa: E731
        key = (h, w, c, int(a["num_filter"]), pair(a["kernel"]), pair(a.get("stride", 1)),
               pair(a.get("pad", 0)))
        seen.setdefault(key, n.name)
    return [(v,) + k for k, v in seen.items()]


GEOMS = _geometries()


@pytest.mark.parametrize("geom", GEOMS, ids=[g[0] for g in GEOMS])
def test_bench_conv_geometry(engine, geom):
    import torch
    from torch.nn.grad import conv2d_input, conv2d_weight
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.executor import bind
    name, h, w, c, f, k, s, p = geom
    symbol.reset_names()
    net = symbol.apply("Convolution", {"kernel": k, "num_filter": f, "stride": s, "pad": p},
                       [symbol.variable("data")], name="conv")
    shapes, named = symbol.infer_shape(net, {"data": (PER, h, w, c)})
    oshape = named["conv"]
    gen = torch.Generator(device="cuda").manual_seed(h * 7919 + c * 31 + f + k[0] * 3 + s[0])
    dev = "cuda:0"
    x = torch.randn(PER, h, w, c, device=dev, generator=gen)
    wt = torch.randn(f, k[0], k[1], c, device=dev, generator=gen) * 0.2
    bias = torch.randn(f, device=dev, generator=gen)
    og = torch.randn(*oshape, device=dev, generator=gen)
    args = {"data": tmod.Tensor.wrap(x.clone(), engine), "conv_weight": tmod.Tensor.wrap(wt.clone(), engine),
            "conv_bias": tmod.Tensor.wrap(bias.clone(), engine),
            "conv_head_grad": tmod.Tensor.wrap(og.clone(), engine)}
    grads = {n: tmod.zeros(tuple(shapes[n]), engine=engine) for n in ("data", "conv_weight", "conv_bias")}
    torch.cuda.synchronize()
    ex = bind(net, args, {n: "write" for n in grads}, grads, engine=engine, dense="bf16",
              split_target=20)  # bench.CONFIGS["inception_bn"]["split_target"]
    ex.forward()
    ex.backward()
    engine.wait_all()
    y = ex.outputs[0].arr.double()
    r16 = lambda t: t.to(torch.bfloat16).double().permute(0, 3, 1, 2)  # noqa: E731
    xr, wr, ogr = r16(x), r16(wt), r16(og)
    y_ref = torch.nn.functional.conv2d(xr, wr, bias.double(), stride=s, padding=p).permute(0, 2, 3, 1)
    dx_ref = conv2d_input(xr.shape, wr, ogr, stride=s, padding=p).permute(0, 2, 3, 1)
    dw_ref = conv2d_weight(xr, wr.shape, ogr, stride=s, padding=p).permute(0, 2, 3, 1)
    db_ref = og.double().sum(dim=(0, 1, 2))
    def close(got, ref, kk):
        atol = max(1e-4 * max(1.0, kk ** 0.5 / 8), 1e-5 * float(ref.abs().max()))
        torch.testing.assert_close(got, ref, rtol=1e-4, atol=atol)

    close(y, y_ref, k[0] * k[1] * c)
    close(grads["data"].arr.double(), dx_ref, k[0] * k[1] * f)
    close(grads["conv_weight"].arr.double(), dw_ref, PER * oshape[1] * oshape[2])
    torch.testing.assert_close(grads["conv_bias"].arr.double(), db_ref, rtol=1e-5,
                               atol=1e-4 * max(1.0, (PER * oshape[1] * oshape[2]) ** 0.5 / 8))
