"""Convolution-net kernels through the C-ABI (configs 3-5).

No reference oracle exists for these operators (parity
unpinned by reference); they are checked against oracle/convnet.py's
float64 restatement of MXNet's semantics.  Tolerances:
  * tensor-core GEMM/conv: operands rounded to bf16 exactly like the kernel,
    fp32 accumulation vs fp64: rtol 1e-4, atol 1e-4 * sqrt(K)/8 * max|term|;
  * BatchNorm / pooling / concat / col2im (fp32 arithmetic, fixed order):
    rtol 1e-5 / atol 1e-5 (max pooling and concat: exact).
"""

import numpy as np
import pytest

from oracle import convnet as oc

pytestmark = pytest.mark.gpu


def _geom(shape, k, s, p):
    b, h, w, c = shape
    return np.array([b, h, w, c, (k[0] << 16) | k[1], (s[0] << 16) | s[1], (p[0] << 16) | p[1]],
                    np.int64)


def _ptr(a):
    import ctypes
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (200, 72, 40), (64, 300, 1000), (20, 576, 6400)])
def test_gemm_operand_majors(cuda, a_mn, b_mn, m, n, k):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(m + 7 * n + 13 * k + a_mn + 2 * b_mn)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    pad = lambda v: -(-v // 8) * 8  # noqa: E731
    # store A as [m, lda] (K-major) or [k, lda] (MN-major), same for B
    if a_mn:
        lda = pad(m)
        abuf = torch.zeros(k, lda, dtype=torch.bfloat16, device="cuda")
        abuf[:, :m] = a.T
    else:
        lda = pad(k)
        abuf = torch.zeros(m, lda, dtype=torch.bfloat16, device="cuda")
        abuf[:, :k] = a
    if b_mn:
        ldb = pad(n)
        bbuf = torch.zeros(k, ldb, dtype=torch.bfloat16, device="cuda")
        bbuf[:, :n] = b.T
    else:
        ldb = pad(k)
        bbuf = torch.zeros(n, ldb, dtype=torch.bfloat16, device="cuda")
        bbuf[:, :k] = b
    c = torch.full((m, n), float("nan"), device="cuda")
    ws = torch.empty(64 * m * n + 1, device="cuda")
    L.call("mgx_gemm_bf16_tc_ex", abuf.data_ptr(), lda, a_mn, bbuf.data_ptr(), ldb, b_mn, None,
           c.data_ptr(), n, m, n, k, 0, 0, ws.data_ptr(), None, 0)
    torch.cuda.synchronize()
    ref = a.double() @ b.double().T
    torch.testing.assert_close(c.double(), ref, rtol=1e-4, atol=1e-3 * max(1.0, (k / 64) ** 0.5))


CONV_CASES = [
    # (B, H, W, C, F, k, s, p)
    (2, 8, 8, 16, 24, (1, 1), (1, 1), (0, 0)),
    (2, 9, 7, 8, 16, (3, 3), (1, 1), (1, 1)),
    (3, 12, 12, 1, 20, (5, 5), (1, 1), (0, 0)),
    (2, 15, 15, 3, 8, (7, 7), (2, 2), (3, 3)),
    (1, 23, 23, 3, 12, (11, 11), (4, 4), (2, 2)),
    (2, 9, 9, 12, 20, (3, 3), (2, 2), (1, 1)),
    # stride-2 data gradient as a transposed convolution over dY read dilated
    # (gather mode 3): exact and ragged (14 -> 7) output extents
    (2, 14, 14, 16, 24, (3, 3), (2, 2), (1, 1)),
    (2, 27, 27, 32, 16, (3, 3), (2, 2), (0, 0)),
    (2, 10, 11, 8, 16, (3, 3), (2, 2), (1, 1)),
    # C % 64 == 0: forward A and weight-gradient B by TMA im2col (ragged
    # pixel counts: the last 64-pixel k-block is partial)
    (2, 9, 9, 64, 24, (3, 3), (1, 1), (1, 1)),
    (2, 14, 13, 128, 80, (3, 3), (2, 2), (1, 1)),
    (1, 7, 7, 64, 64, (1, 7), (1, 1), (0, 3)),
    # few filters: the weight gradient computed transposed (GEMM mode 6)
    (2, 10, 10, 64, 160, (3, 3), (1, 1), (1, 1)),
    (2, 10, 10, 32, 160, (3, 3), (1, 1), (1, 1)),  # ... its A operand gathered (mode 7)
]


def _conv_case(torch, case, seed):
    b, h, w, c, f, k, s, p = case
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(b, h, w, c, generator=g, dtype=torch.float64)
    wt = torch.randn(f, k[0], k[1], c, generator=g, dtype=torch.float64) * 0.2
    bias = torch.randn(f, generator=g, dtype=torch.float64)
    return x, wt, bias


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_executor_forward_backward(cuda, engine, case):
    """Convolution node bound through the executor: forward, dX, dW, db
    against the float64 oracle on bf16-rounded operands."""
    torch = cuda
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.executor import bind
    b, h, wd, c, f, k, s, p = case
    x, wt, bias = _conv_case(torch, case, sum(case[:5]))
    net = symbol.apply("Convolution", {"kernel": k, "num_filter": f, "stride": s, "pad": p},
                       [symbol.variable("data")], name="conv")
    shapes, named = symbol.infer_shape(net, {"data": tuple(x.shape)})
    oshape = named["conv"]
    og = torch.randn(*oshape, generator=torch.Generator().manual_seed(5), dtype=torch.float64)
    head = net.head_grad_names() if hasattr(net, "head_grad_names") else []
    args = {"data": tmod.from_host(x.shape, "float32", x.float().numpy(), engine=engine),
            "conv_weight": tmod.from_host(wt.shape, "float32", wt.float().numpy(), engine=engine),
            "conv_bias": tmod.from_host(bias.shape, "float32", bias.float().numpy(), engine=engine)}
    grads = {n: tmod.zeros(tuple(t.shape), engine=engine) for n, t in
             (("data", x), ("conv_weight", wt), ("conv_bias", bias))}
    args["conv_head_grad"] = tmod.from_host(oshape, "float32", og.float().numpy(), engine=engine)
    del head
    ex = bind(net, args, {n: "write" for n in grads}, grads, engine=engine)
    ex.forward()
    ex.backward()
    y = tmod.to_numpy(ex.outputs[0])
    # oracle on the same bf16-rounded operands
    xr, wr = oc.bf16(x).requires_grad_(True), oc.bf16(wt).requires_grad_(True)
    br = bias.clone().requires_grad_(True)
    yr = oc.conv2d_nhwc(xr, wr, br, s, p)
    ogr = oc.bf16(og.float().double())
    (yr * ogr).sum().backward()
    kk = k[0] * k[1] * c
    tol = 1e-4 * max(1.0, kk ** 0.5 / 8)
    np.testing.assert_allclose(y, yr.detach().numpy(), rtol=1e-4, atol=tol)
    np.testing.assert_allclose(tmod.to_numpy(grads["data"]), xr.grad.numpy(), rtol=1e-4,
                               atol=1e-4 * max(1.0, (f * k[0] * k[1]) ** 0.5 / 8))
    np.testing.assert_allclose(tmod.to_numpy(grads["conv_weight"]), wr.grad.numpy(), rtol=1e-4,
                               atol=1e-4 * max(1.0, (b * oshape[1] * oshape[2]) ** 0.5 / 8))
    np.testing.assert_allclose(tmod.to_numpy(grads["conv_bias"]), og.sum(dim=(0, 1, 2)).numpy(),
                               rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("m,c", [(1000, 16), (4096, 64), (333, 200), (64 * 49, 1024), (50, 3)])
@pytest.mark.parametrize("fix_gamma", [True, False])
def test_batchnorm_kernels(cuda, m, c, fix_gamma):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    g = torch.Generator().manual_seed(m + c)
    x = torch.randn(m, c, generator=g, dtype=torch.float64) * 3 + 1
    gamma = torch.rand(c, generator=g, dtype=torch.float64) + 0.5
    beta = torch.randn(c, generator=g, dtype=torch.float64)
    dy = torch.randn(m, c, generator=g, dtype=torch.float64)
    xd, gd, bd, dyd = (t.float().cuda() for t in (x, gamma, beta, dy))
    mm = torch.zeros(c, device="cuda")
    mv = torch.ones(c, device="cuda")
    wsb = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    st = torch.empty(2 * c, device="cuda")
    y = torch.empty(m, c, device="cuda")
    sums = torch.empty(2 * c, device="cuda")
    dx = torch.empty(m, c, device="cuda")
    gp = None if fix_gamma else gd.data_ptr()
    L.call("mgx_bn_stats", xd.data_ptr(), m, c, ws.data_ptr(), st.data_ptr(), mm.data_ptr(),
           mv.data_ptr(), 1e-3, 0.9, 0, 0)
    y16 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda") if c % 4 == 0 else None
    L.call("mgx_bn_apply", xd.data_ptr(), st.data_ptr(), gp, bd.data_ptr(), y.data_ptr(), m, c, 0,
           y16.data_ptr() if y16 is not None else None, 0)
    L.call("mgx_bn_bwd_reduce", dyd.data_ptr(), xd.data_ptr(), st.data_ptr(), m, c, ws.data_ptr(),
           sums.data_ptr(), None, None, 0, None, None, 0)
    L.call("mgx_bn_bwd_dx", dyd.data_ptr(), xd.data_ptr(), st.data_ptr(), sums.data_ptr(), gp,
           dx.data_ptr(), m, c, None, None, None, ws.data_ptr(), None, 0)
    torch.cuda.synchronize()
    if c % 4 == 0:  # fused dx + per-channel sum of dx
        dx2 = torch.empty(m, c, device="cuda")
        dsum = torch.empty(c, device="cuda")
        dx16 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
        L.call("mgx_bn_bwd_dx", dyd.data_ptr(), xd.data_ptr(), st.data_ptr(), sums.data_ptr(), gp,
               dx2.data_ptr(), m, c, None, None, dsum.data_ptr(), ws.data_ptr(), dx16.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(dx2, dx)
        assert torch.equal(dx16, dx.to(torch.bfloat16))
        # sum_rows(dx) cancels to ~0: compare against the summed magnitude
        mag = float(dx.double().abs().sum(0).max())
        np.testing.assert_allclose(dsum.cpu().numpy(), dx.double().sum(0).cpu().numpy(),
                                   rtol=1e-4, atol=2e-7 * mag)
    xr = xd.double().cpu().requires_grad_(True)
    gr = gd.double().cpu().requires_grad_(True)
    br = bd.double().cpu().requires_grad_(True)
    yr, mean, var = oc.batchnorm(xr, gr, br, 1e-3, fix_gamma)
    (yr * dyd.double().cpu()).sum().backward()
    np.testing.assert_allclose(y.cpu().numpy(), yr.detach().numpy(), rtol=1e-5, atol=2e-5)
    if y16 is not None:  # the bf16 copy written in the same pass
        assert torch.equal(y16, y.to(torch.bfloat16))
    np.testing.assert_allclose(dx.cpu().numpy(), xr.grad.numpy(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(sums[:c].cpu().numpy(), br.grad.numpy(), rtol=1e-5, atol=1e-4)
    if not fix_gamma:
        np.testing.assert_allclose(sums[c:].cpu().numpy(), gr.grad.numpy(), rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(mm.cpu().numpy(), (0.1 * mean).detach().numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(mv.cpu().numpy(), (0.9 + 0.1 * var).detach().numpy(), rtol=1e-5, atol=1e-6)


POOL_CASES = [
    # (shape, kernel, stride, pad, type)
    ((2, 12, 12, 8), (2, 2), (2, 2), (0, 0), "max"),
    ((2, 13, 13, 16), (3, 3), (2, 2), (0, 0), "max"),
    ((2, 14, 14, 8), (3, 3), (1, 1), (1, 1), "max"),
    ((2, 14, 14, 8), (3, 3), (1, 1), (1, 1), "avg"),
    ((2, 27, 27, 4), (3, 3), (2, 2), (1, 1), "max"),
    ((1, 7, 7, 32), (7, 7), (1, 1), (0, 0), "avg"),
    ((2, 11, 11, 6), (3, 3), (2, 2), (1, 1), "max"),
    ((2, 11, 11, 6), (3, 3), (1, 1), (1, 1), "avg"),
]


@pytest.mark.parametrize("case", POOL_CASES)
@pytest.mark.parametrize("ties", [False, True])
@pytest.mark.parametrize("use_argmax", [False, True])
def test_pooling_kernels(cuda, case, ties, use_argmax):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    shape, k, s, p, kind = case
    if use_argmax and (shape[3] % 4 or kind != "max"):
        pytest.skip("argmax side buffer: max pooling with C % 4 == 0 only")
    g = torch.Generator().manual_seed(sum(shape))
    x = torch.randn(*shape, generator=g, dtype=torch.float64)
    if ties:  # post-ReLU maps: many equal zeros in a window
        x = torch.relu(x - 0.5).float().double()
    x = x.float().double()
    xr = x.clone().requires_grad_(True)
    yr = oc.pool_nhwc(xr, {"kernel": k, "stride": s, "pad": p, "pool_type": kind})
    dy = torch.randn(*yr.shape, generator=g, dtype=torch.float64).float().double()
    (yr * dy).sum().backward()
    geom = _geom(shape, k, s, p)
    xd, dyd = x.float().cuda(), dy.float().cuda()
    y = torch.empty(*yr.shape, device="cuda")
    dx = torch.empty(*shape, device="cuda")
    t = 0 if kind == "max" else 1
    arg = torch.zeros(y.numel(), dtype=torch.uint8, device="cuda") if use_argmax else None
    argp = arg.data_ptr() if arg is not None else None
    y16 = torch.empty(*yr.shape, dtype=torch.bfloat16, device="cuda") if shape[3] % 4 == 0 else None
    L.call("mgx_pool_forward", xd.data_ptr(), y.data_ptr(), _ptr(geom), 0, t, argp,
           y16.data_ptr() if y16 is not None else None, 0)
    L.call("mgx_pool_backward", xd.data_ptr(), y.data_ptr(), dyd.data_ptr(), dx.data_ptr(),
           _ptr(geom), 0, t, argp, 0)
    torch.cuda.synchronize()
    if y16 is not None:
        assert torch.equal(y16, y.to(torch.bfloat16))
    if kind == "max":
        np.testing.assert_array_equal(y.cpu().numpy(), yr.detach().float().numpy())
    else:
        np.testing.assert_allclose(y.cpu().numpy(), yr.detach().numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dx.cpu().numpy(), xr.grad.numpy(), rtol=1e-5, atol=1e-6)


def test_chan_copy_and_colsum(cuda):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    a = torch.randn(37, 12, device="cuda")
    b = torch.randn(37, 5, device="cuda")
    out = torch.zeros(37, 17, device="cuda")
    L.call("mgx_chan_copy", a.data_ptr(), 12, 0, out.data_ptr(), 17, 0, 37, 12, None, 0)
    L.call("mgx_chan_copy", b.data_ptr(), 5, 0, out.data_ptr(), 17, 12, 37, 5, None, 0)
    torch.cuda.synchronize()
    assert torch.equal(out, torch.cat([a, b], dim=1))
    # channel-aligned concat with its bf16 copy
    a2, b2 = torch.randn(37, 16, device="cuda"), torch.randn(37, 24, device="cuda")
    o2 = torch.zeros(37, 40, device="cuda")
    o16 = torch.zeros(37, 40, dtype=torch.bfloat16, device="cuda")
    L.call("mgx_chan_copy", a2.data_ptr(), 16, 0, o2.data_ptr(), 40, 0, 37, 16, o16.data_ptr(), 0)
    L.call("mgx_chan_copy", b2.data_ptr(), 24, 0, o2.data_ptr(), 40, 16, 37, 24, o16.data_ptr(), 0)
    torch.cuda.synchronize()
    assert torch.equal(o2, torch.cat([a2, b2], dim=1))
    assert torch.equal(o16, o2.to(torch.bfloat16))
    x = torch.randn(5000, 24, device="cuda")
    wsb = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", 5000, 24, ctypes.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    s = torch.empty(24, device="cuda")
    L.call("mgx_colsum", x.data_ptr(), 5000, 24, ws.data_ptr(), s.data_ptr(), 0)
    torch.cuda.synchronize()
    np.testing.assert_allclose(s.cpu().numpy(), x.double().sum(0).cpu().numpy(), rtol=1e-6,
                               atol=1e-5)


@pytest.mark.parametrize("m,c", [(3000, 64), (777, 12), (500, 6)])
@pytest.mark.parametrize("fix_gamma", [True, False])
def test_batchnorm_backward_with_fused_relu(cuda, m, c, fix_gamma):
    """ReLU(BatchNorm(x)) backward in one pass pair: the ReLU mask is
    recomputed from x, gamma and beta; dbeta/dgamma land in their buffers;
    the dx pass also reduces sum_rows(dx) (conv bias gradient)."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    g = torch.Generator().manual_seed(m * 7 + c)
    x = (torch.randn(m, c, generator=g, dtype=torch.float64) * 2 + 0.3).float().cuda()
    gamma = (torch.rand(c, generator=g, dtype=torch.float64) + 0.5).float().cuda()
    beta = torch.randn(c, generator=g, dtype=torch.float64).float().cuda()
    og = torch.randn(m, c, generator=g, dtype=torch.float64).float().cuda()
    wsb = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    st = torch.empty(2 * c, device="cuda")
    sums = torch.empty(2 * c, device="cuda")
    dbeta = torch.full((c,), float("nan"), device="cuda")
    dgamma = torch.full((c,), float("nan"), device="cuda")
    dx = torch.empty(m, c, device="cuda")
    dsum = torch.empty(c, device="cuda")
    gp = None if fix_gamma else gamma.data_ptr()
    L.call("mgx_bn_stats", x.data_ptr(), m, c, ws.data_ptr(), st.data_ptr(), None, None, 1e-3,
           0.9, 0, 0)
    L.call("mgx_bn_bwd_reduce", og.data_ptr(), x.data_ptr(), st.data_ptr(), m, c, ws.data_ptr(),
           sums.data_ptr(), dbeta.data_ptr(), dgamma.data_ptr(), 1 if fix_gamma else 0, gp,
           beta.data_ptr(), 0)
    L.call("mgx_bn_bwd_dx", og.data_ptr(), x.data_ptr(), st.data_ptr(), sums.data_ptr(), gp,
           dx.data_ptr(), m, c, gp, beta.data_ptr(), dsum.data_ptr() if c % 4 == 0 else None,
           ws.data_ptr(), None, 0)
    torch.cuda.synchronize()
    xr = x.double().cpu().requires_grad_(True)
    gr = gamma.double().cpu().requires_grad_(True)
    br = beta.double().cpu().requires_grad_(True)
    yr, _mean, _var = oc.batchnorm(xr, gr, br, 1e-3, fix_gamma)
    (torch.relu(yr) * og.double().cpu()).sum().backward()
    np.testing.assert_allclose(dx.cpu().numpy(), xr.grad.numpy(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(dbeta.cpu().numpy(), br.grad.numpy(), rtol=1e-5, atol=1e-4)
    if fix_gamma:
        assert torch.count_nonzero(dgamma).item() == 0
    else:
        np.testing.assert_allclose(dgamma.cpu().numpy(), gr.grad.numpy(), rtol=1e-5, atol=1e-4)
    if c % 4 == 0:
        mag = float(dx.double().abs().sum(0).max())
        np.testing.assert_allclose(dsum.cpu().numpy(), dx.double().sum(0).cpu().numpy(),
                                   rtol=1e-4, atol=2e-7 * mag)


@pytest.mark.parametrize("m,c", [(12544, 96), (3136, 1024), (23328, 64), (1001, 48), (97, 16),
                                 (12544, 576),
                                 # streaming variant (rows read twice from
                                 # global memory): 4- and 2-vector slices,
                                 # clusters of 16 and 8, ragged row split
                                 (46656, 64), (46656, 96), (40001, 136), (32768, 32)])
@pytest.mark.parametrize("fix_gamma,relu", [(True, True), (False, False), (False, True)])
def test_batchnorm_cluster_fused(cuda, m, c, fix_gamma, relu):
    """The cluster-fused BatchNorm passes (one kernel per pass, rows staged
    on-chip or -- from 32768 rows -- streamed twice through L2, DSMEM
    reduction) against the float64 oracle, and against the
    unfused statistics kernel for the values the backward consumes."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    ok = ctypes.c_int()
    L.call("mgx_bn_fused_ok", m, c, 1, ctypes.byref(ok))
    assert ok.value == (2 if m >= 32768 else 1)  # 2: the streaming variant
    L.call("mgx_bn_fused_ok", m, 12, 1, ctypes.byref(ok))
    assert ok.value == 0  # C % 8 != 0: the unfused kernels
    g = torch.Generator().manual_seed(m + 3 * c)
    x = (torch.randn(m, c, generator=g, dtype=torch.float64) * 2 + 0.7).float().cuda()
    gamma = (torch.rand(c, generator=g, dtype=torch.float64) + 0.5).float().cuda()
    beta = torch.randn(c, generator=g, dtype=torch.float64).float().cuda()
    og = torch.randn(m, c, generator=g, dtype=torch.float64).float().cuda()
    gp = None if fix_gamma else gamma.data_ptr()
    act = 1 if relu else 0  # MGX_ACT_RELU
    st = torch.empty(2 * c, device="cuda")
    mm, mv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda")
    y = torch.empty(m, c, device="cuda")
    y16 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
    L.call("mgx_bn_fwd_fused", x.data_ptr(), m, c, st.data_ptr(), mm.data_ptr(), mv.data_ptr(),
           1e-3, 0.9, gp, beta.data_ptr(), y.data_ptr(), y16.data_ptr(), act, 0)
    dx = torch.empty(m, c, device="cuda")
    dx16 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
    dbeta = torch.full((c,), float("nan"), device="cuda")
    dgamma = torch.full((c,), float("nan"), device="cuda")
    sums = torch.empty(2 * c, device="cuda")
    dsum = torch.empty(c, device="cuda")
    L.call("mgx_bn_bwd_fused", og.data_ptr(), c, x.data_ptr(), st.data_ptr(), gp, m, c,
           gp if relu else None, beta.data_ptr() if relu else None, dbeta.data_ptr(),
           dgamma.data_ptr(), 1 if fix_gamma else 0, sums.data_ptr(), dx.data_ptr(),
           dx16.data_ptr(), dsum.data_ptr(), 0)
    # the unfused statistics for comparison
    wsb = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    st2 = torch.empty(2 * c, device="cuda")
    L.call("mgx_bn_stats", x.data_ptr(), m, c, ws.data_ptr(), st2.data_ptr(), None, None, 1e-3,
           0.9, 0, 0)
    torch.cuda.synchronize()
    np.testing.assert_allclose(st.cpu().numpy(), st2.cpu().numpy(), rtol=2e-6, atol=1e-6)
    assert torch.equal(y16, y.to(torch.bfloat16))
    assert torch.equal(dx16, dx.to(torch.bfloat16))
    assert torch.equal(sums[:c], dbeta)
    xr = x.double().cpu().requires_grad_(True)
    gr = gamma.double().cpu().requires_grad_(True)
    br = beta.double().cpu().requires_grad_(True)
    yr, mean, var = oc.batchnorm(xr, gr, br, 1e-3, fix_gamma)
    if relu:
        yr = torch.relu(yr)
    (yr * og.double().cpu()).sum().backward()
    np.testing.assert_allclose(y.cpu().numpy(), yr.detach().numpy(), rtol=1e-5, atol=2e-5)
    np.testing.assert_allclose(mm.cpu().numpy(), (0.1 * mean).detach().numpy(), rtol=1e-5,
                               atol=1e-6)
    np.testing.assert_allclose(mv.cpu().numpy(), (0.9 + 0.1 * var).detach().numpy(), rtol=1e-5,
                               atol=1e-6)
    np.testing.assert_allclose(dx.cpu().numpy(), xr.grad.numpy(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(dbeta.cpu().numpy(), br.grad.numpy(), rtol=1e-5, atol=1e-4)
    if fix_gamma:
        assert torch.count_nonzero(dgamma).item() == 0
    else:
        np.testing.assert_allclose(dgamma.cpu().numpy(), gr.grad.numpy(), rtol=1e-5, atol=1e-4)
    mag = float(dx.double().abs().sum(0).max())
    np.testing.assert_allclose(dsum.cpu().numpy(), dx.double().sum(0).cpu().numpy(),
                               rtol=1e-4, atol=2e-7 * mag)
    # deterministic: a second run is bitwise identical
    dx_b = torch.empty_like(dx)
    L.call("mgx_bn_bwd_fused", og.data_ptr(), c, x.data_ptr(), st.data_ptr(), gp, m, c,
           gp if relu else None, beta.data_ptr() if relu else None, None, None, 0, None,
           dx_b.data_ptr(), None, None, 0)
    torch.cuda.synchronize()
    assert torch.equal(dx_b, dx)
    # the output gradient read in place from a channel slice of a wider
    # tensor (a Concat's gradient): row stride ldd = c + 16, offset 8
    wide = torch.zeros(m, c + 16, device="cuda")
    wide[:, 8:8 + c] = og
    dx_w = torch.empty_like(dx)
    L.call("mgx_bn_bwd_fused", wide.data_ptr() + 8 * 4, c + 16, x.data_ptr(), st.data_ptr(), gp,
           m, c, gp if relu else None, beta.data_ptr() if relu else None, None, None, 0, None,
           dx_w.data_ptr(), None, None, 0)
    torch.cuda.synchronize()
    assert torch.equal(dx_w, dx)


@pytest.mark.parametrize("shape,k,s,p", [((2, 18, 18, 16), 3, 2, 0), ((2, 13, 11, 8), 3, 2, 1),
                                         ((3, 10, 10, 24), 2, 2, 0)])
@pytest.mark.parametrize("fix_gamma", [True, False])
def test_bn_act_pool_stem_fusion(cuda, shape, k, s, p, fix_gamma):
    """BatchNorm + ReLU + max pooling in one pass (bitwise equal to apply ->
    pool), and the BatchNorm backward reading its gradient through the
    pooling (reductions over the windows' argmax pixels, dx from the
    covering windows) against the unfused chain (pool backward -> reduce ->
    dx): the sums differ only in summation order."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    b, h, w, c = shape
    m = b * h * w
    g = torch.Generator().manual_seed(m + c + k)
    x = (torch.randn(m, c, generator=g, dtype=torch.float64) * 2 + 0.3).float().cuda()
    gamma = (torch.rand(c, generator=g, dtype=torch.float64) + 0.5).float().cuda()
    beta = torch.randn(c, generator=g, dtype=torch.float64).float().cuda()
    gp = None if fix_gamma else gamma.data_ptr()
    geom = _geom(shape, (k, k), (s, s), (p, p))
    ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    n_out = b * ho * wo * c
    wsb = ctypes.c_int64()
    L.call("mgx_reduce_workspace_bytes", m, c, ctypes.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    st = torch.empty(2 * c, device="cuda")
    L.call("mgx_bn_stats", x.data_ptr(), m, c, ws.data_ptr(), st.data_ptr(), None, None, 1e-3,
           0.9, 0, 0)
    # unfused chain
    z = torch.empty(m, c, device="cuda")
    L.call("mgx_bn_apply", x.data_ptr(), st.data_ptr(), gp, beta.data_ptr(), z.data_ptr(), m, c, 1,
           None, 0)
    y1 = torch.empty(n_out, device="cuda")
    a1 = torch.empty(n_out, dtype=torch.uint8, device="cuda")
    L.call("mgx_pool_forward", z.data_ptr(), y1.data_ptr(), _ptr(geom), 0, 0, a1.data_ptr(), None, 0)
    dyp = torch.randn(n_out, generator=g, dtype=torch.float64).float().cuda()
    og = torch.empty(m, c, device="cuda")
    L.call("mgx_pool_backward", None, None, dyp.data_ptr(), og.data_ptr(), _ptr(geom), 0, 0,
           a1.data_ptr(), 0)
    sums1 = torch.empty(2 * c, device="cuda")
    L.call("mgx_bn_bwd_reduce", og.data_ptr(), x.data_ptr(), st.data_ptr(), m, c, ws.data_ptr(),
           sums1.data_ptr(), None, None, 1 if fix_gamma else 0, gp, beta.data_ptr(), 0)
    dx1 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
    ds1 = torch.empty(c, device="cuda")
    L.call("mgx_bn_bwd_dx", og.data_ptr(), x.data_ptr(), st.data_ptr(), sums1.data_ptr(), gp, None,
           m, c, gp, beta.data_ptr(), ds1.data_ptr(), ws.data_ptr(), dx1.data_ptr(), 0)
    # fused
    y2 = torch.empty(n_out, device="cuda")
    y16 = torch.empty(n_out, dtype=torch.bfloat16, device="cuda")
    a2 = torch.empty(n_out, dtype=torch.uint8, device="cuda")
    L.call("mgx_bn_act_pool_fwd", x.data_ptr(), st.data_ptr(), gp, beta.data_ptr(), 1, _ptr(geom),
           0, y2.data_ptr(), y16.data_ptr(), a2.data_ptr(), 0)
    sums2 = torch.empty(2 * c, device="cuda")
    db2, dg2 = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    L.call("mgx_bn_bwd_reduce_pooled", dyp.data_ptr(), a2.data_ptr(), _ptr(geom), 0, x.data_ptr(),
           st.data_ptr(), m, c, ws.data_ptr(), sums2.data_ptr(), db2.data_ptr(), dg2.data_ptr(),
           1 if fix_gamma else 0, gp, beta.data_ptr(), 0)
    dx2 = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
    ds2 = torch.empty(c, device="cuda")
    L.call("mgx_bn_bwd_dx_pooled", dyp.data_ptr(), a2.data_ptr(), _ptr(geom), 0, x.data_ptr(),
           st.data_ptr(), sums2.data_ptr(), gp, m, c, beta.data_ptr(), ds2.data_ptr(),
           ws.data_ptr(), None, dx2.data_ptr(), 0)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(y16, y2.to(torch.bfloat16))
    assert torch.equal(a1, a2)
    mag = float(og.abs().sum()) / c
    np.testing.assert_allclose(sums2.cpu().numpy(), sums1.cpu().numpy(), rtol=1e-5,
                               atol=1e-6 * mag)
    assert torch.equal(db2, sums2[:c])
    # dx: 1-ulp bf16 flips where the sums' last bits differ
    np.testing.assert_allclose(dx2.float().cpu().numpy(), dx1.float().cpu().numpy(), rtol=8e-3,
                               atol=1e-6 * mag)
    dmag = float(dx1.float().abs().sum(0).max())
    np.testing.assert_allclose(ds2.cpu().numpy(), ds1.cpu().numpy(), rtol=1e-3, atol=1e-5 * dmag)


IMPLICIT_CASES = [
    # (B, H, W, C, F, k, s, p)
    (2, 9, 7, 16, 24, (3, 3), (1, 1), (1, 1)),
    (2, 8, 8, 64, 72, (1, 1), (1, 1), (0, 0)),
    (3, 13, 11, 8, 40, (5, 5), (1, 1), (2, 2)),
    (2, 15, 15, 24, 136, (3, 3), (2, 2), (1, 1)),
    (1, 23, 23, 8, 16, (7, 7), (2, 2), (3, 3)),
    (4, 27, 27, 96, 192, (3, 3), (1, 1), (1, 1)),
    # C % 64 == 0: the A tile by TMA im2col loads (gather mode 3 of the kernel)
    (2, 14, 14, 64, 96, (3, 3), (1, 1), (1, 1)),
    (2, 15, 15, 128, 64, (3, 3), (2, 2), (1, 1)),
    (1, 9, 11, 64, 40, (5, 5), (1, 1), (2, 2)),
    (3, 7, 7, 192, 128, (3, 3), (1, 1), (1, 1)),
]


@pytest.mark.parametrize("case", IMPLICIT_CASES)
def test_implicit_gemm_convolution(cuda, case):
    """mgx_gemm_bf16_conv: the operand gathered by cp.async producer warps
    inside the tcgen05 GEMM equals the explicit im2col contraction (mode 1:
    forward; mode 2: weight gradient) against float64 on bf16 operands."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    b, h, w, c, f, k, s, p = case
    g = torch.Generator().manual_seed(sum(case[:5]))
    x = torch.randn(b, h, w, c, generator=g, dtype=torch.float64).to(torch.bfloat16)
    wt = (torch.randn(f, k[0], k[1], c, generator=g, dtype=torch.float64) * 0.2).to(torch.bfloat16)
    geom = _geom((b, h, w, c), k, s, p)
    ho, wo = (h + 2 * p[0] - k[0]) // s[0] + 1, (w + 2 * p[1] - k[1]) // s[1] + 1
    m, kk = b * ho * wo, k[0] * k[1] * c
    xd, wd = x.cuda(), wt.reshape(f, kk).contiguous().cuda()
    ldw = -(-kk // 8) * 8
    wpad = torch.zeros(f, ldw, dtype=torch.bfloat16, device="cuda")
    wpad[:, :kk] = wd
    out = torch.full((m, f), float("nan"), device="cuda")
    # forward with the epilogue's per-32-row column statistics (BatchNorm input)
    cs = torch.full((-(-m // 32), f, 2), float("nan"), device="cuda") if f % 4 == 0 else None
    L.call("mgx_gemm_bf16_conv", 1, xd.data_ptr(), _ptr(geom), wpad.data_ptr(), ldw, None,
           out.data_ptr(), f, m, f, kk, 0, 1, None, cs.data_ptr() if cs is not None else None, 0)
    # weight gradient: dW[f, kk] = sum_m dY[m, f] gather(x)[m, kk]
    dy = torch.randn(m, f, generator=g, dtype=torch.float64).to(torch.bfloat16)
    ldf = -(-f // 8) * 8
    dyd = torch.zeros(m, ldf, dtype=torch.bfloat16, device="cuda")
    dyd[:, :f] = dy.cuda()
    dw = torch.full((f, kk), float("nan"), device="cuda")
    ws = torch.empty(max(64 * f * kk, 148 * m * f) + 1, device="cuda")
    L.call("mgx_gemm_bf16_conv", 2, xd.data_ptr(), _ptr(geom), dyd.data_ptr(), ldf, None,
           dw.data_ptr(), kk, f, kk, m, 0, 0, ws.data_ptr(), None, 0)
    torch.cuda.synchronize()
    if cs is not None:
        # BatchNorm statistics merged from the tiles == mgx_bn_stats over the output
        import ctypes
        st1, st2 = torch.empty(2 * f, device="cuda"), torch.empty(2 * f, device="cuda")
        mm1, mv1 = torch.zeros(f, device="cuda"), torch.ones(f, device="cuda")
        mm2, mv2 = torch.zeros(f, device="cuda"), torch.ones(f, device="cuda")
        L.call("mgx_bn_stats_from_tiles", cs.data_ptr(), m, f, st1.data_ptr(), mm1.data_ptr(),
               mv1.data_ptr(), 1e-3, 0.9, 0)
        wsb = ctypes.c_int64()
        L.call("mgx_reduce_workspace_bytes", m, f, ctypes.byref(wsb))
        rws = torch.empty(wsb.value // 4 + 1, device="cuda")
        L.call("mgx_bn_stats", out.data_ptr(), m, f, rws.data_ptr(), st2.data_ptr(), mm2.data_ptr(),
               mv2.data_ptr(), 1e-3, 0.9, 0, 0)
        torch.cuda.synchronize()
        torch.testing.assert_close(st1, st2, rtol=1e-5, atol=1e-6)
        torch.testing.assert_close(mv1, mv2, rtol=1e-5, atol=1e-6)
    ref = oc.conv2d_nhwc(x.double(), wt.double(), None, s, p).reshape(m, f)
    torch.testing.assert_close(out.double().cpu(), ref, rtol=1e-4, atol=1e-3 * max(1, kk / 64) ** 0.5)
    # split-K forward (auto split count, in-order reduce) with a bias: the
    # same contraction, bias added once after the split sum
    bias = torch.randn(f, generator=g, dtype=torch.float64).float().cuda()
    out2 = torch.full((m, f), float("nan"), device="cuda")
    L.call("mgx_gemm_bf16_conv", 1, xd.data_ptr(), _ptr(geom), wpad.data_ptr(), ldw,
           bias.data_ptr(), out2.data_ptr(), f, m, f, kk, 0, 0, ws.data_ptr(), None, 0)
    torch.cuda.synchronize()
    torch.testing.assert_close(out2.double().cpu(), ref + bias.double().cpu(), rtol=1e-4,
                               atol=1e-3 * max(1, kk / 64) ** 0.5)
    xr = x.double().permute(0, 3, 1, 2)
    from torch.nn.grad import conv2d_weight
    dwr = conv2d_weight(xr, (f, c, k[0], k[1]), dy.double().reshape(b, ho, wo, f).permute(0, 3, 1, 2),
                        stride=s, padding=p).permute(0, 2, 3, 1).reshape(f, kk)
    torch.testing.assert_close(dw.double().cpu(), dwr, rtol=1e-4, atol=1e-3 * max(1, m / 64) ** 0.5)


def test_sum_n_and_concat_kernels(cuda):
    """One-pass ElementwiseAdd chains (same left-to-right rounding: bitwise)
    and one-pass channel concat with its bf16 copy (exact)."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    import ctypes
    xs = [torch.randn(4096 * 3, device="cuda") for _ in range(4)]
    out = torch.empty_like(xs[0])
    arr = (ctypes.c_void_p * 4)(*[x.data_ptr() for x in xs])
    L.call("mgx_sum_n", arr, 4, out.data_ptr(), out.numel(), 0)
    torch.cuda.synchronize()
    assert torch.equal(out, ((xs[0] + xs[1]) + xs[2]) + xs[3])
    ins = [torch.randn(123, c, device="cuda") for c in (32, 64, 96, 8)]
    cat = torch.empty(123, 200, device="cuda")
    c16 = torch.empty(123, 200, dtype=torch.bfloat16, device="cuda")
    arr = (ctypes.c_void_p * 4)(*[x.data_ptr() for x in ins])
    ch = (ctypes.c_int64 * 4)(32, 64, 96, 8)
    L.call("mgx_concat", arr, ch, 4, cat.data_ptr(), c16.data_ptr(), 123, 0)
    torch.cuda.synchronize()
    assert torch.equal(cat, torch.cat(ins, dim=1))
    assert torch.equal(c16, cat.to(torch.bfloat16))


@pytest.mark.parametrize("case", [(2, 15, 15, 3, 8, (7, 7), (2, 2), (3, 3)),
                                  (2, 9, 7, 8, 16, (3, 3), (1, 1), (1, 1))])
def test_conv_eager_forward(cuda, engine, case):
    """Plugin-style eager call of the Convolution operator (no executor):
    its preparation work (weight casts, the stem's column matrix) runs
    right away on the current stream."""
    torch = cuda
    from paper_1512_01274_b200 import ops
    b, h, wd, c, f, k, s, p = case
    x, wt, bias = _conv_case(torch, case, 3 + sum(case[:5]))
    xd, wd_, bd = (t.float().cuda() for t in (x, wt, bias))
    ho, wo = (h + 2 * p[0] - k[0]) // s[0] + 1, (wd + 2 * p[1] - k[1]) // s[1] + 1
    y = torch.full((b, ho, wo, f), float("nan"), device="cuda")
    ops.get_op("Convolution").forward([xd, wd_, bd], y, {"kernel": k, "num_filter": f,
                                                         "stride": s, "pad": p})
    torch.cuda.synchronize()
    r16 = lambda t: t.float().to(torch.bfloat16).double()  # noqa: E731
    ref = oc.conv2d_nhwc(r16(x), r16(wt), bias, s, p)
    kk = k[0] * k[1] * c
    torch.testing.assert_close(y.double().cpu(), ref, rtol=1e-4,
                               atol=1e-4 * max(1.0, (kk / 64) ** 0.5) * 8)


@pytest.mark.parametrize("m,c", [(65536 + 7, 40), (200704, 64), (1000, 24)])
def test_bn_stats_from_tiles(cuda, m, c):
    """BatchNorm statistics merged from per-32-row (mean, M2) pairs -- the
    cluster kernel from 65536 rows (coalesced 32-channel rows, 16 CTAs per
    channel group; ragged channel groups and row blocks), the per-channel
    block below -- against float64 over the rows, moving averages too."""
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    g = torch.Generator().manual_seed(m + c)
    x = (torch.randn(m, c, generator=g, dtype=torch.float64) * 3 + 1.5)
    nb = -(-m // 32)
    pad = torch.zeros(nb * 32, c, dtype=torch.float64)
    pad[:m] = x
    blocks = pad.reshape(nb, 32, c)
    cnt = torch.full((nb, 1), 32.0, dtype=torch.float64)
    cnt[-1] = m - (nb - 1) * 32
    mean_b = blocks.sum(1) / cnt
    dev = blocks - mean_b[:, None, :]
    mask = (torch.arange(32)[None, :, None] < cnt[:, :, None])
    m2_b = (dev * dev * mask).sum(1)
    part = torch.stack([mean_b, m2_b], dim=-1).float().cuda().contiguous()
    st = torch.empty(2 * c, device="cuda")
    mm, mv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda")
    L.call("mgx_bn_stats_from_tiles", part.data_ptr(), m, c, st.data_ptr(), mm.data_ptr(),
           mv.data_ptr(), 1e-3, 0.9, 0)
    torch.cuda.synchronize()
    mean, var = x.mean(0), x.var(0, unbiased=False)
    np.testing.assert_allclose(st[:c].cpu().numpy(), mean.numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(st[c:].cpu().numpy(), (1 / (var + 1e-3).sqrt()).numpy(),
                               rtol=1e-5)
    np.testing.assert_allclose(mv.cpu().numpy(), (0.9 + 0.1 * var).numpy(), rtol=1e-5)
