"""Pin the CPU oracle against golden outputs of the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import kv as okv
from oracle import numerics as nm
from oracle import plan as oplan
from oracle import step as ostep

F32 = np.float32
FC_SHAPES = [(50, 784, 128), (50, 128, 64), (50, 64, 10)]
PW_K = [1, 3, 7, 8, 9, 15, 16, 17, 64, 100, 127, 128, 129, 200, 784, 1000, 4096, 9216]


def fc_inputs(seed, b, f, h):
    rs = np.random.RandomState(seed)
    x = rs.rand(b, f).astype(F32)
    w = (rs.randn(h, f) * 0.1).astype(F32)
    bias = (rs.randn(h) * 0.1).astype(F32)
    og = (rs.randn(b, h) * 0.01).astype(F32)
    return x, w, bias, og


@pytest.mark.parametrize("i", range(3))
def test_fc_orders_bitwise(ops_golden, i):
    b, f, h = FC_SHAPES[i]
    x, w, bias, og = fc_inputs(100 + i, b, f, h)
    y = nm.fc_forward(x, w, bias)
    assert np.array_equal(y, ops_golden[f"fc{i}_y"])
    assert np.array_equal(nm.seq_matmul(og, w), ops_golden[f"fc{i}_dx"])
    assert np.array_equal(nm.tree_outer(og, x), ops_golden[f"fc{i}_dw"])
    assert np.array_equal(nm.tree_sum(og), ops_golden[f"fc{i}_db"])
    assert np.array_equal(nm.relu(y), ops_golden[f"fc{i}_relu"])
    assert np.array_equal(nm.relu_backward(nm.relu(y), og), ops_golden[f"fc{i}_relu_bwd"])


@pytest.mark.parametrize("k", PW_K)
def test_pairwise_and_sequential_orders(ops_golden, k):
    rs = np.random.RandomState(7000 + k)
    a = rs.randn(3, k).astype(F32)
    bm = rs.randn(5, k).astype(F32)
    got = nm.pairwise_rows((a[:, None, :] * bm[None, :, :]).astype(F32))
    assert np.array_equal(got, ops_golden[f"pw{k}"])
    if k <= 200:  # literal restatement agrees with the vectorised one
        lit = np.array([[nm.pairwise_sum((a[i] * bm[j]).astype(F32)) for j in range(5)]
                        for i in range(3)], F32)
        assert np.array_equal(lit, ops_golden[f"pw{k}"])
    assert np.array_equal(nm.seq_matmul(a, np.ascontiguousarray(bm.T)), ops_golden[f"seq{k}"])


def test_tree_sum_all_lengths(ops_golden):
    for n in range(1, 70):
        rs = np.random.RandomState(8000 + n)
        assert np.array_equal(nm.tree_sum(rs.randn(n, 7).astype(F32)), ops_golden[f"tree{n}"]), n


def test_softmax_forward_backward(ops_golden):
    rs = np.random.RandomState(9000)
    for j, (bsz, c) in enumerate([(50, 10), (7, 3), (33, 130), (4, 1000)]):
        x = (rs.randn(bsz, c) * 3).astype(F32)
        lab = rs.randint(0, c, bsz).astype(F32)
        p = nm.softmax_rows(x)
        # same numpy exp on the same host: bitwise
        assert np.array_equal(p, ops_golden[f"softmax{j}_p"])
        assert np.array_equal(nm.softmax_backward(p, lab), ops_golden[f"softmax{j}_g"])


def test_matmul_orders(ops_golden):
    for j, (m, k, n) in enumerate([(6, 20, 9), (30, 17, 12), (3, 200, 5)]):
        rs = np.random.RandomState(9100 + j)
        a, b, og = rs.randn(m, k).astype(F32), rs.randn(k, n).astype(F32), rs.randn(m, n).astype(F32)
        assert np.array_equal(nm.seq_matmul(a, b), ops_golden[f"mm{j}_y"])
        ga = nm.pairwise_rows((og[:, None, :] * b[None, :, :]).astype(F32))
        assert np.array_equal(ga, ops_golden[f"mm{j}_ga"])
        assert np.array_equal(nm.seq_matmul(np.ascontiguousarray(a.T), og), ops_golden[f"mm{j}_gb"])


@pytest.mark.parametrize("machines,workers", [(1, 2), (1, 4), (1, 8), (2, 2)])
def test_kv_rounds(kv_golden, machines, workers):
    nw = machines * workers
    for key, n in enumerate([1000, 10, 5003]):
        w0 = (np.random.RandomState(key).randn(n) * 0.1).astype(F32)
        ws, wa, v = w0.copy(), w0.copy(), np.zeros(n, F32)
        for r in range(3):
            grads = [np.random.RandomState(1000 + w + 100 * r + 10000 * key).randn(n).astype(F32)
                     for w in range(nw)]
            ws, v = okv.sgd_round(ws, v, grads, 0.05, 0.9, 1e-4, machines)
            wa = okv.add_round(wa, grads, machines)
        assert np.array_equal(ws, kv_golden[f"m{machines}w{workers}_sgd_k{key}"])
        assert np.array_equal(wa, kv_golden[f"m{machines}w{workers}_add_k{key}"])


def _flat_view(text, given):
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200.planner import FlatGraph
    return FlatGraph.of(symbol.load(text), given, "float32")


def test_plan_oracle_matches_reference_plans(plans_golden):
    for rec in plans_golden["mlp"]:
        b, f = rec["given"]
        view = _flat_view(rec["comb_text"], {"data": (b, f), "label": (b,)})
        for s, want in rec["plans"].items():
            slot_of, slot_bytes, ded, edges, total = oplan.plan(
                view.is_var, view.nbytes, view.dedicated, view.inputs, view.inplace_positions,
                s, rec["phases"])
            assert [slot_of[i] for i in range(view.n)] == want["slot_of"]
            assert [slot_bytes[i] for i in range(len(slot_bytes))] == want["slot_bytes"]
            assert sorted(ded) == want["dedicated"]
            assert [list(e) for e in edges] == want["edges"]
            assert total == want["total"]
    for rec in plans_golden["dags"][:100]:
        view = _flat_view(rec["text"], {k: tuple(v) for k, v in rec["shapes"].items()})
        for s, want in rec["plans"].items():
            slot_of, _sb, _d, edges, total = oplan.plan(
                view.is_var, view.nbytes, view.dedicated, view.inputs, view.inplace_positions, s)
            assert [slot_of[i] for i in range(view.n)] == want["slot_of"], (rec["seed"], s)
            assert [list(e) for e in edges] == want["edges"]
            assert total == want["total"]


def test_config1_golden_plan_numbers(plans_golden):
    # config-1 (B=50) internal bytes per strategy
    rec = plans_golden["mlp"][0]
    totals = {s: p["total"] for s, p in rec["plans"].items()}
    assert totals == {"none": 157600, "inplace": 78800, "coshare": 117200, "both": 78800}


def test_sharding_rule_restatement():
    from paper_1512_01274_b200.kvstore import plan_buckets, shard_ranges
    rs = np.random.RandomState(0)
    for _ in range(300):
        numels = list(rs.randint(1, 300000, rs.randint(1, 20)))
        bb = int(rs.choice([1 << 12, 1 << 16, 4 << 20]))
        assert plan_buckets(numels, bb) == okv.arena_layout(numels, bb)
        for length in (64, 640, 100352, 1 << 20):
            for owners in (1, 2, 3, 4, 8, 16):
                assert shard_ranges(length, owners) == okv.owner_shards(length, owners)


@pytest.mark.parametrize("tag,batch,machines,workers,n", [
    ("w2b100", 100, 1, 2, 500), ("w8b128", 128, 1, 8, 500), ("m2w2b128", 128, 2, 2, 500)])
def test_train_distributed_oracle_bitwise(train_golden, tag, batch, machines, workers, n):
    feats, labels = ostep.cfg1_data(n)
    params, _ = ostep.train_distributed([128, 64], 10, feats, labels, 0.05, 0.9, 1e-4, epochs=1,
                                        batch=batch, machines=machines, workers=workers)
    for k, v in params.items():
        assert np.array_equal(v, train_golden[f"dist_{tag}_n{n}_{k}"]), k


def test_train_local_oracle_bitwise(train_golden):
    feats, labels = ostep.cfg1_data(500)
    params = ostep.train_local([128, 64], 10, feats, labels, 0.05, 0.9, 1e-4, epochs=1, batch=100)
    for k, v in params.items():
        assert np.array_equal(v, train_golden[f"local_b100_n500_{k}"]), k
