"""sm_100a operator kernels vs the oracle and the reference's golden outputs.
Bitwise wherever the reference order is reproducible; softmax/sigmoid/tanh
(numpy SIMD exp/tanh) within stated tolerances."""

import numpy as np
import pytest

from oracle import numerics as nm

pytestmark = pytest.mark.gpu
F32 = np.float32
FC_SHAPES = [(50, 784, 128), (50, 128, 64), (50, 64, 10)]
PW_K = [1, 3, 7, 8, 9, 15, 16, 17, 64, 100, 127, 128, 129, 200, 784, 1000, 4096, 9216]


def fc_inputs(seed, b, f, h):
    rs = np.random.RandomState(seed)
    return (rs.rand(b, f).astype(F32), (rs.randn(h, f) * 0.1).astype(F32),
            (rs.randn(h) * 0.1).astype(F32), (rs.randn(b, h) * 0.01).astype(F32))


def dev(cuda, a):
    return cuda.from_numpy(np.ascontiguousarray(a, dtype=F32)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def L():
    from paper_1512_01274_b200 import _lib
    return _lib


@pytest.mark.parametrize("i", range(3))
def test_fc_kernels_bitwise(cuda, ops_golden, i):
    b, f, h = FC_SHAPES[i]
    x, w, bias, og = fc_inputs(100 + i, b, f, h)
    X, Wt, Bt, OG = dev(cuda, x), dev(cuda, w), dev(cuda, bias), dev(cuda, og)
    Y = cuda.empty(b, h, device="cuda")
    L().call("mgx_gemm_pairwise", X.data_ptr(), f, Wt.data_ptr(), f, Bt.data_ptr(), Y.data_ptr(),
             h, b, h, f, 0, 0)
    assert np.array_equal(host(Y), ops_golden[f"fc{i}_y"])
    DX = cuda.empty(b, f, device="cuda")
    L().call("mgx_gemm_sequential", OG.data_ptr(), h, 1, Wt.data_ptr(), f, 1, DX.data_ptr(), f,
             None, 0, b, f, h, 0)
    assert np.array_equal(host(DX), ops_golden[f"fc{i}_dx"])
    DW = cuda.empty(h, f, device="cuda")
    DB = cuda.empty(h, device="cuda")
    L().call("mgx_fc_dw_db", OG.data_ptr(), X.data_ptr(), DW.data_ptr(), DB.data_ptr(), b, h, f, 0)
    assert np.array_equal(host(DW), ops_golden[f"fc{i}_dw"])
    assert np.array_equal(host(DB), ops_golden[f"fc{i}_db"])
    # fused FC + relu epilogue == relu(FC)
    R = cuda.empty(b, h, device="cuda")
    L().call("mgx_gemm_pairwise", X.data_ptr(), f, Wt.data_ptr(), f, Bt.data_ptr(), R.data_ptr(),
             h, b, h, f, 1, 0)
    assert np.array_equal(host(R), ops_golden[f"fc{i}_relu"])
    G = cuda.empty(b, h, device="cuda")
    L().call("mgx_act_backward", 1, R.data_ptr(), OG.data_ptr(), G.data_ptr(), b * h, 0)
    assert np.array_equal(host(G), ops_golden[f"fc{i}_relu_bwd"])


@pytest.mark.parametrize("k", PW_K)
def test_pairwise_and_sequential_all_lengths(cuda, ops_golden, k):
    rs = np.random.RandomState(7000 + k)
    a = rs.randn(3, k).astype(F32)
    bm = rs.randn(5, k).astype(F32)
    A, B = dev(cuda, a), dev(cuda, bm)
    C = cuda.empty(3, 5, device="cuda")
    L().call("mgx_gemm_pairwise", A.data_ptr(), k, B.data_ptr(), k, None, C.data_ptr(), 5,
             3, 5, k, 0, 0)
    assert np.array_equal(host(C), ops_golden[f"pw{k}"])
    BT = dev(cuda, np.ascontiguousarray(bm.T))
    S = cuda.empty(3, 5, device="cuda")
    L().call("mgx_gemm_sequential", A.data_ptr(), k, 1, BT.data_ptr(), 5, 1, S.data_ptr(), 5,
             None, 0, 3, 5, k, 0)
    assert np.array_equal(host(S), ops_golden[f"seq{k}"])


def test_batch_tree_all_lengths(cuda, ops_golden):
    for n in list(range(1, 70)) + [100, 128, 1000, 4099]:
        rs = np.random.RandomState(8000 + n)
        a = rs.randn(n, 7).astype(F32)
        A = dev(cuda, a)
        O = cuda.empty(7, device="cuda")
        L().call("mgx_tree_sum_rows", A.data_ptr(), O.data_ptr(), n, 7, 0)
        want = ops_golden[f"tree{n}"] if n < 70 else nm.tree_sum(a)
        assert np.array_equal(host(O), want), n


def test_dw_large_batch_and_odd_shapes(cuda):
    for (b, h, f) in [(1, 3, 5), (7, 33, 65), (300, 17, 130), (2049, 5, 40)]:
        rs = np.random.RandomState(b)
        og, x = rs.randn(b, h).astype(F32), rs.randn(b, f).astype(F32)
        OG, X = dev(cuda, og), dev(cuda, x)
        DW, DB = cuda.empty(h, f, device="cuda"), cuda.empty(h, device="cuda")
        L().call("mgx_fc_dw_db", OG.data_ptr(), X.data_ptr(), DW.data_ptr(), DB.data_ptr(),
                 b, h, f, 0)
        assert np.array_equal(host(DW), nm.tree_outer(og, x)), (b, h, f)
        assert np.array_equal(host(DB), nm.tree_sum(og)), (b, h, f)


def test_softmax_within_ulps(cuda, ops_golden):
    rs = np.random.RandomState(9000)
    for j, (bsz, c) in enumerate([(50, 10), (7, 3), (33, 130), (4, 1000)]):
        x = (rs.randn(bsz, c) * 3).astype(F32)
        lab = rs.randint(0, c, bsz).astype(F32)
        X, LB = dev(cuda, x), dev(cuda, lab)
        P, G = cuda.empty(bsz, c, device="cuda"), cuda.empty(bsz, c, device="cuda")
        L().call("mgx_softmax_forward", X.data_ptr(), P.data_ptr(), bsz, c, 0)
        L().call("mgx_softmax_backward", P.data_ptr(), LB.data_ptr(), G.data_ptr(), bsz, c, 0)
        # exp differs from numpy's SIMD float32 exp by <= 1 ulp per element
        np.testing.assert_allclose(host(P), ops_golden[f"softmax{j}_p"], rtol=4e-7, atol=1e-9)
        np.testing.assert_allclose(host(G), ops_golden[f"softmax{j}_g"], rtol=4e-7, atol=1e-9)


def test_matmul_op_orders(cuda, ops_golden):
    for j, (m, k, n) in enumerate([(6, 20, 9), (30, 17, 12), (3, 200, 5)]):
        rs = np.random.RandomState(9100 + j)
        a, b, og = rs.randn(m, k).astype(F32), rs.randn(k, n).astype(F32), rs.randn(m, n).astype(F32)
        A, B, OG = dev(cuda, a), dev(cuda, b), dev(cuda, og)
        Y = cuda.empty(m, n, device="cuda")
        L().call("mgx_gemm_sequential", A.data_ptr(), k, 1, B.data_ptr(), n, 1, Y.data_ptr(), n,
                 None, 0, m, n, k, 0)
        GA = cuda.empty(m, k, device="cuda")
        L().call("mgx_gemm_pairwise", OG.data_ptr(), n, B.data_ptr(), n, None, GA.data_ptr(), k,
                 m, k, n, 0, 0)
        GB = cuda.empty(k, n, device="cuda")
        L().call("mgx_gemm_sequential", A.data_ptr(), 1, k, OG.data_ptr(), n, 1, GB.data_ptr(), n,
                 None, 0, k, n, m, 0)
        assert np.array_equal(host(Y), ops_golden[f"mm{j}_y"])
        assert np.array_equal(host(GA), ops_golden[f"mm{j}_ga"])
        assert np.array_equal(host(GB), ops_golden[f"mm{j}_gb"])


def test_pointwise_and_sgd_bitwise(cuda):
    rs = np.random.RandomState(5)
    n = 1003
    a, b = rs.randn(n).astype(F32), rs.randn(n).astype(F32)
    A, B, O = dev(cuda, a), dev(cuda, b), cuda.empty(n, device="cuda")
    for code, fn in enumerate([np.add, np.subtract, np.multiply, np.true_divide]):
        L().call("mgx_elementwise", code, A.data_ptr(), B.data_ptr(), O.data_ptr(), n, 0)
        assert np.array_equal(host(O), fn(a, b).astype(F32))
    L().call("mgx_scalar_op", 1, A.data_ptr(), float(F32(-1.5)), O.data_ptr(), n, 0)
    assert np.array_equal(host(O), (a * F32(-1.5)).astype(F32))
    Y = dev(cuda, b)
    L().call("mgx_axpy", float(F32(0.3)), A.data_ptr(), Y.data_ptr(), n, 0)
    assert np.array_equal(host(Y), nm.axpy(0.3, a, b))
    w, g, v = rs.randn(n).astype(F32), rs.randn(n).astype(F32), rs.randn(n).astype(F32)
    W, Gt, V = dev(cuda, w), dev(cuda, g), dev(cuda, v)
    for _ in range(3):
        L().call("mgx_sgd_step", W.data_ptr(), Gt.data_ptr(), V.data_ptr(), n, 0.05, 0.9, 1e-4, 0)
        w, v = nm.sgd_update(w, g, v, 0.05, 0.9, 1e-4)
    assert np.array_equal(host(W), w) and np.array_equal(host(V), v)
    # activations: relu exact, sigmoid/tanh to the ulp
    x = (rs.randn(n) * 4).astype(F32)
    X, Y2 = dev(cuda, x), cuda.empty(n, device="cuda")
    L().call("mgx_act_forward", 1, X.data_ptr(), Y2.data_ptr(), n, 0)
    assert np.array_equal(host(Y2), nm.relu(x))
    L().call("mgx_act_forward", 2, X.data_ptr(), Y2.data_ptr(), n, 0)
    np.testing.assert_allclose(host(Y2), nm.sigmoid(x), rtol=5e-7, atol=0)
    L().call("mgx_act_forward", 3, X.data_ptr(), Y2.data_ptr(), n, 0)
    np.testing.assert_allclose(host(Y2), np.tanh(x), rtol=5e-7, atol=1e-30)


def test_unaligned_views_take_scalar_path(cuda):
    a = np.arange(37, dtype=F32)
    A = dev(cuda, a)
    O = cuda.zeros(40, device="cuda")
    L().call("mgx_copy", A.data_ptr() + 4, O.data_ptr() + 4, 30, 0)
    out = host(O)
    assert np.array_equal(out[1:31], a[1:31]) and out[0] == 0 and out[31] == 0
