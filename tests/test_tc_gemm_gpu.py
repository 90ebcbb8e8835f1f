"""tcgen05/TMA bf16 GEMM (the tolerance dense path) vs an fp32 reference of
the same bf16-rounded operands.  Stated tolerance: fp32 accumulation in
tensor-core order, rtol 1e-4 / atol 1e-3 * sqrt(K/64) on N(0,1) data."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (100, 128, 784), (256, 384, 1024),
                                   (77, 200, 136), (128, 4096, 9216), (300, 10, 64)])
@pytest.mark.parametrize("act", [0, 1])
def test_tc_gemm_matches_fp32_reference(cuda, m, n, k, act):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(m * 131 + n * 7 + k)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    bias = torch.randn(n, device="cuda", generator=g)
    c = torch.full((m, n), float("nan"), device="cuda")
    L.call("mgx_gemm_bf16_tc", a.data_ptr(), k, b.data_ptr(), k, bias.data_ptr(), c.data_ptr(), n,
           m, n, k, act, 0)
    torch.cuda.synchronize()
    ref = a.double() @ b.double().T + bias.double()
    if act == 1:
        ref = ref.clamp_min(0)
    tol = 1e-3 * max(1.0, (k / 64) ** 0.5)
    torch.testing.assert_close(c.double(), ref, rtol=1e-4, atol=tol)


def test_cast_f32_bf16_rounds_to_nearest_even(cuda):
    torch = cuda
    from paper_1512_01274_b200 import _lib as L
    x = torch.randn(10007, device="cuda") * 100
    y = torch.empty(10007, dtype=torch.bfloat16, device="cuda")
    L.call("mgx_cast_f32_bf16", x.data_ptr(), y.data_ptr(), x.numel(), 0)
    torch.cuda.synchronize()
    assert torch.equal(y, x.to(torch.bfloat16))
