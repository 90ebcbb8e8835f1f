"""Generate the golden fixtures from the reference implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Inputs are regenerated from numpy RandomState seeds by the tests, so only
reference OUTPUTS are stored:
  ops_golden.npz    operator kernels at config-1 shapes + order probes
  kv_golden.npz     KVStore rounds (SGD and add updaters, W=2/4/8, M=2xW=2)
  plans_golden.json memory plans: config-1 MLP, 8x64 MLP, 200 random DAGs
  train_golden.npz  train_distributed / train_local weights on config-1 data
  blobs130.rec(+.idx), data_golden.npz
                    a record file packed by the reference's recordio.pack and
                    the batches its BatchIterator yields (seeds 0/1, two
                    epochs, shuffle on/off, affine)
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from minigraph import kernels, ops, symbol  # noqa: E402
from minigraph.engine import Engine  # noqa: E402
from minigraph import tensor as tmod  # noqa: E402
from minigraph.kvstore import KVStore  # noqa: E402
from minigraph.optim import SGDConfig, make_sgd_updater  # noqa: E402
from minigraph.planner import plan_memory, STRATEGIES  # noqa: E402
from minigraph.recordio import Example, pack  # noqa: E402
from minigraph.symbol import SymbolGraph  # noqa: E402
from minigraph.train import mlp, train_distributed, train_local  # noqa: E402
from conftest import random_dag, ref_forward  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32

# shared with the tests: seeds and shapes
FC_SHAPES = [(50, 784, 128), (50, 128, 64), (50, 64, 10)]
PW_K = [1, 3, 7, 8, 9, 15, 16, 17, 64, 100, 127, 128, 129, 200, 784, 1000, 4096, 9216]
MATMUL_SHAPES = [(6, 20, 9), (30, 17, 12), (3, 200, 5)]
KV_CASES = [(1, 2), (1, 4), (1, 8), (2, 2)]
KV_NUMELS = [1000, 10, 5003]


def fc_inputs(seed, b, f, h):
    rs = np.random.RandomState(seed)
    x = rs.rand(b, f).astype(F32)
    w = (rs.randn(h, f) * 0.1).astype(F32)
    bias = (rs.randn(h) * 0.1).astype(F32)
    og = (rs.randn(b, h) * 0.01).astype(F32)
    return x, w, bias, og


def make_ops():
    out = {}
    for i, (b, f, h) in enumerate(FC_SHAPES):
        x, w, bias, og = fc_inputs(100 + i, b, f, h)
        op = ops.get_op("FullyConnected")
        y = np.empty((b, h), F32)
        op.forward([x, w, bias], y, {"num_hidden": h})
        grads = [np.empty_like(x), np.empty_like(w), np.empty_like(bias)]
        op.backward([x, w, bias], y, og, grads, {"num_hidden": h})
        out[f"fc{i}_y"], out[f"fc{i}_dx"], out[f"fc{i}_dw"], out[f"fc{i}_db"] = y, *grads
        act = ops.get_op("Activation")
        r = np.empty_like(y)
        act.forward([y], r, {"act_type": "relu"})
        g = np.empty_like(y)
        act.backward([y], r, og, [g], {"act_type": "relu"})
        out[f"fc{i}_relu"], out[f"fc{i}_relu_bwd"] = r, g
    for k in PW_K:
        rs = np.random.RandomState(7000 + k)
        a = rs.randn(3, k).astype(F32)
        bm = rs.randn(5, k).astype(F32)
        out[f"pw{k}"] = kernels.det_matmul(a, bm.T)
        out[f"seq{k}"] = kernels.det_matmul(a, np.ascontiguousarray(bm.T))
    for n in range(1, 70):
        rs = np.random.RandomState(8000 + n)
        out[f"tree{n}"] = kernels.tree_sum(rs.randn(n, 7).astype(F32))
    rs = np.random.RandomState(9000)
    for j, (bsz, c) in enumerate([(50, 10), (7, 3), (33, 130), (4, 1000)]):
        x = (rs.randn(bsz, c) * 3).astype(F32)
        lab = rs.randint(0, c, bsz).astype(F32)
        sm = ops.get_op("SoftmaxOutput")
        p = np.empty_like(x)
        sm.forward([x, lab], p, {})
        g = np.empty_like(x)
        sm.backward([x, lab], p, None, [g, None], {})
        out[f"softmax{j}_p"], out[f"softmax{j}_g"] = p, g
    for j, (m, k, n) in enumerate(MATMUL_SHAPES):
        rs = np.random.RandomState(9100 + j)
        a, bm, og = rs.randn(m, k).astype(F32), rs.randn(k, n).astype(F32), rs.randn(m, n).astype(F32)
        mm = ops.get_op("MatMul")
        y = np.empty((m, n), F32)
        mm.forward([a, bm], y, {})
        ga, gb = np.empty_like(a), np.empty_like(bm)
        mm.backward([a, bm], y, og, [ga, gb], {})
        out[f"mm{j}_y"], out[f"mm{j}_ga"], out[f"mm{j}_gb"] = y, ga, gb
    np.savez_compressed(os.path.join(HERE, "ops_golden.npz"), **out)


def kv_grads(nw, rounds):
    return [[np.random.RandomState(1000 + w + 100 * r) for w in range(nw)] for r in range(rounds)]


def make_kv():
    out = {}
    cfg = SGDConfig(eta=0.05, momentum=0.9, weight_decay=1e-4)
    for machines, workers in KV_CASES:
        nw = machines * workers
        for upd in ("sgd", "add"):
            eng = Engine(threads=2 * nw + 6)
            kv = KVStore(machines, workers, engine=eng)
            for key, n in enumerate(KV_NUMELS):
                kv.init(key, (np.random.RandomState(key).randn(n) * 0.1).astype(F32))
            if upd == "sgd":
                kv.set_updater(make_sgd_updater(cfg, scale=nw))
            for r in range(3):
                for key, n in enumerate(KV_NUMELS):
                    for w in range(nw):
                        g = np.random.RandomState(1000 + w + 100 * r + 10000 * key).randn(n)
                        kv.push(key, tmod.from_host((n,), "float32", g.astype(F32), engine=eng), w)
            for key, n in enumerate(KV_NUMELS):
                o = tmod.zeros((n,), engine=eng)
                kv.pull(key, o, 0)
                out[f"m{machines}w{workers}_{upd}_k{key}"] = np.asarray(tmod.to_host(o), F32)
            kv.close()
            eng.close()
    np.savez_compressed(os.path.join(HERE, "kv_golden.npz"), **out)


def plan_record(p):
    n = len(p.node_names)
    return {"slot_of": [p.slot_of[i] for i in range(n)],
            "slot_bytes": [p.slot_bytes[s] for s in range(len(p.slot_bytes))],
            "dedicated": sorted(p.dedicated_slots), "edges": [list(e) for e in p.extra_dep_edges],
            "total": p.total_internal_bytes, "visits": p.visits}


def combined_graph(g):
    wrt = [n for n in g.list_arguments() if n not in ("data", "label")]
    ends, _ = symbol.build_gradient(g, wrt)
    comb = SymbolGraph(list(g.outputs) + ends)
    fwd = {id(n) for n in g.topo_nodes()}
    phases = [0 if (n.is_variable or id(n) in fwd) else 1 for n in comb.topo_nodes()]
    return comb, phases


def make_plans():
    out = {"mlp": [], "dags": []}
    for hidden, classes, b, f in [([128, 64], 10, 50, 784), ([64] * 8, 10, 64, 64),
                                  ([16], 3, 32, 6)]:
        symbol.reset_names()
        g = mlp(hidden, classes)
        fwd_text = symbol.save(g)
        comb, phases = combined_graph(g)
        given = {"data": (b, f), "label": (b,)}
        rec = {"hidden": hidden, "classes": classes, "given": [b, f], "fwd_text": fwd_text,
               "comb_text": symbol.save(comb), "phases": phases, "plans": {}, "fwd_plans": {}}
        for s in STRATEGIES:
            rec["plans"][s] = plan_record(plan_memory(comb, given, s, phases=phases))
            rec["fwd_plans"][s] = plan_record(plan_memory(g, given, s))
        out["mlp"].append(rec)
    for seed in range(200):
        symbol.reset_names()
        g, feed = random_dag(seed, max_ops=12)
        shapes = {k: list(v.shape) for k, v in feed.items()}
        rec = {"seed": seed, "text": symbol.save(g), "shapes": shapes, "plans": {}}
        for s in STRATEGIES:
            rec["plans"][s] = plan_record(plan_memory(g, shapes, s))
        if seed < 30:
            rec["forward"] = [o.astype(float).ravel().tolist()
                              for o in ref_forward(g, feed)]
            rec["feed"] = {k: v.astype(float).ravel().tolist() for k, v in feed.items()}
        out["dags"].append(rec)
    with open(os.path.join(HERE, "plans_golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


def cfg1_data(n, seed=0):
    rs = np.random.RandomState(seed)
    return rs.rand(n, 784).astype(F32), rs.randint(0, 10, n).astype(F32)


def make_train():
    out = {}
    cfg = SGDConfig(eta=0.05, momentum=0.9, weight_decay=1e-4)
    with tempfile.TemporaryDirectory() as tmp:
        for n in (500, 2000):
            feats, labels = cfg1_data(n)
            path = os.path.join(tmp, f"cfg1_{n}.rec")
            pack((Example(int(l), f) for f, l in zip(feats, labels)), path)
            runs = [("w2b100", dict(batch=100, machines=1, workers=2))]
            if n == 500:
                runs += [("w8b128", dict(batch=128, machines=1, workers=8)),
                         ("m2w2b128", dict(batch=128, machines=2, workers=2))]
            for tag, kw in runs:
                symbol.reset_names()
                rep, params = train_distributed(mlp([128, 64], 10), path, cfg, epochs=1, **kw)
                for k, v in params.items():
                    out[f"dist_{tag}_n{n}_{k}"] = v
                out[f"dist_{tag}_n{n}_loss"] = np.array([r[1] for r in rep.rows])
            if n == 500:
                symbol.reset_names()
                eng = Engine(threads=4)
                rep, params = train_local(mlp([128, 64], 10), path, cfg, epochs=1, batch=100,
                                          engine=eng)
                eng.close()
                for k, v in params.items():
                    out[f"local_b100_n{n}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "train_golden.npz"), **out)


def make_data():
    from minigraph.dataiter import BatchIterator
    from minigraph.datasets import pack_blobs
    path = os.path.join(HERE, "blobs130.rec")
    pack_blobs(path, 130, classes=3, dim=4, seed=0)
    out = {}
    for tag, kw in (("s0", dict(seed=0)), ("s1", dict(seed=1)), ("noshuf", dict(shuffle=False)),
                    ("affine", dict(seed=0, affine=(np.array([1.0, -1.0, 0.5, 0.0], F32),
                                                    np.array([0.5, 2.0, 1.0, 3.0], F32))))):
        with BatchIterator(path, 16, prefetch=2, **kw) as it:
            for epoch in range(2):
                for b, (f, l) in enumerate(it):
                    out[f"{tag}_e{epoch}_b{b}_x"] = f
                    out[f"{tag}_e{epoch}_b{b}_y"] = l
                it.reset()
    np.savez_compressed(os.path.join(HERE, "data_golden.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["data"]:
        make_data()
        sys.exit(0)
    make_data()
    make_ops()
    make_kv()
    make_plans()
    make_train()
    print("golden fixtures written to", HERE)
