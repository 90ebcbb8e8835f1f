"""Device KVStore: the reference's KVStore suite (tests/test_kvstore.py) plus
bit-exact rounds against the oracle and the reference's golden rounds."""

import numpy as np
import pytest

from oracle import kv as okv

pytestmark = pytest.mark.gpu
F32 = np.float32


def mods():
    from paper_1512_01274_b200 import kvstore, optim
    from paper_1512_01274_b200 import tensor as tmod
    return kvstore, optim, tmod


def push_pull_sum(kv, engine, nworkers, rounds=1):
    _, _, tmod = mods()
    kv.init(0, np.zeros(4, F32))
    outs = [tmod.zeros((4,), engine=engine) for _ in range(nworkers)]
    for _ in range(rounds):
        for w in range(nworkers):
            kv.push(0, tmod.from_host((4,), "float32", np.full(4, w + 1, F32), engine=engine), w)
        for w in range(nworkers):
            kv.pull(0, outs[w], w)
    return [tmod.to_numpy(o) for o in outs]


def test_sequential_sum_single_and_two_machines(engine):
    kvstore, _, _ = mods()
    kv = kvstore.KVStore(1, 4, engine=engine)
    for g in push_pull_sum(kv, engine, 4):
        assert np.array_equal(g, np.full(4, 10, F32))
    kv.close()
    kv = kvstore.KVStore(2, 2, engine=engine)
    got = push_pull_sum(kv, engine, 4, rounds=2)
    for g in got:
        assert np.array_equal(g, np.full(4, 20, F32))
    for other in got[1:]:
        assert np.array_equal(got[0], other)
    kv.close()


def test_level2_traffic_stats(engine):
    kvstore, _, _ = mods()
    kv = kvstore.KVStore(2, 2, engine=engine)
    push_pull_sum(kv, engine, 4, rounds=3)
    st = kv.stats()
    assert st["level2_messages"] == 6 and st["level1_aggregates"] == 6 and st["pushes"] == 12
    kv.close()


def test_eventual_mode(engine):
    kvstore, _, tmod = mods()
    kv = kvstore.KVStore(1, 4, mode="eventual", engine=engine)
    kv.init(0, np.zeros(4, F32))
    for w in range(4):
        kv.push(0, tmod.from_host((4,), "float32", np.full(4, w + 1, F32), engine=engine), w)
    kv.quiesce()
    out = tmod.zeros((4,), engine=engine)
    kv.pull(0, out, 0)
    assert np.array_equal(tmod.to_numpy(out), np.full(4, 10, F32))
    kv.close()


def test_custom_updater_runs_on_device(engine):
    kvstore, _, tmod = mods()
    kv = kvstore.KVStore(1, 2, engine=engine)
    kv.init(0, np.ones(3, F32))

    def maxer(key, stored, incoming):
        import torch
        torch.maximum(stored, incoming, out=stored)

    kv.set_updater(maxer)
    for w, v in ((0, 5.0), (1, 2.0)):
        kv.push(0, tmod.from_host((3,), "float32", np.full(3, v, F32), engine=engine), w)
    out = tmod.zeros((3,), engine=engine)
    kv.pull(0, out, 1)
    assert np.array_equal(tmod.to_numpy(out), np.full(3, 7, F32))
    kv.close()


def test_errors(engine):
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.errors import ArgumentError, KVStoreError
    kvstore, _, tmod = mods()
    kv = kvstore.KVStore(1, 2, engine=engine)
    kv.init(0, np.zeros(2, F32))
    with pytest.raises(KVStoreError):
        kv.init(0, np.zeros(2, F32))
    with pytest.raises(KVStoreError):
        kv.push(0, tmod.zeros((3,), engine=engine), 0)
    with pytest.raises(KVStoreError):
        kv.push(99, tmod.zeros((2,), engine=engine), 0)
    with pytest.raises(ArgumentError):
        kv.push(0, tmod.zeros((2,), engine=engine), 7)
    with pytest.raises(ArgumentError):
        kv.init(-1, np.zeros(2, F32))
    other = Engine(device=0)
    with pytest.raises(ArgumentError):
        kv.push(0, tmod.zeros((2,), engine=other), 0)
    kv.close()


def test_many_keys_round_trip(engine):
    kvstore, _, tmod = mods()
    kv = kvstore.KVStore(1, 2, engine=engine)
    for k in range(6):
        kv.init(k, np.full(2, k, F32))
    for k in range(6):
        for w in range(2):
            kv.push(k, tmod.from_host((2,), "float32", [1, 1], engine=engine), w)
    for k in range(6):
        out = tmod.zeros((2,), engine=engine)
        kv.pull(k, out, 0)
        assert np.array_equal(tmod.to_numpy(out), np.full(2, k + 2, F32))
    kv.close()


@pytest.mark.parametrize("machines,workers", [(1, 2), (1, 4), (1, 8), (2, 2)])
@pytest.mark.parametrize("bucket_bytes", [4 << 20, 4096])
def test_rounds_match_reference_golden(engine, kv_golden, machines, workers, bucket_bytes):
    """Same inputs as tests/golden/make_golden.py: 3 rounds over keys of
    1000/10/5003 elements; every sharding gives the reference's bits."""
    kvstore, optim, tmod = mods()
    nw = machines * workers
    numels = [1000, 10, 5003]
    for upd in ("sgd", "add"):
        kv = kvstore.KVStore(machines, workers, engine=engine, bucket_bytes=bucket_bytes)
        for key, n in enumerate(numels):
            kv.init(key, (np.random.RandomState(key).randn(n) * 0.1).astype(F32))
        if upd == "sgd":
            kv.set_updater(optim.make_sgd_updater(optim.SGDConfig(0.05, 0.9, 1e-4), scale=nw))
        for r in range(3):
            for key, n in enumerate(numels):
                for w in range(nw):
                    g = np.random.RandomState(1000 + w + 100 * r + 10000 * key).randn(n)
                    kv.push(key, tmod.from_host((n,), "float32", g.astype(F32), engine=engine), w)
        for key, n in enumerate(numels):
            for w in range(nw):
                o = tmod.zeros((n,), engine=engine)
                kv.pull(key, o, w)
                assert np.array_equal(tmod.to_numpy(o),
                                      kv_golden[f"m{machines}w{workers}_{upd}_k{key}"]), (upd, key, w)
        kv.close()


def test_large_key_matches_oracle(engine):
    """A 64 MB key (config-2 size) reduced over 8 emulated workers."""
    kvstore, optim, tmod = mods()
    n = 16 << 20
    nw = 8
    rs = np.random.RandomState(0)
    w0 = (rs.randn(n) * 0.1).astype(F32)
    kv = kvstore.KVStore(1, nw, engine=engine)
    kv.init(0, w0)
    kv.set_updater(optim.make_sgd_updater(optim.SGDConfig(0.05, 0.9, 1e-4), scale=nw))
    grads = [np.random.RandomState(1000 + w).randn(n).astype(F32) for w in range(nw)]
    for w in range(nw):
        kv.push(0, tmod.from_host((n,), "float32", grads[w], engine=engine), w)
    out = tmod.zeros((n,), engine=engine)
    kv.pull(0, out, 3)
    want, _ = okv.sgd_round(w0, np.zeros(n, F32), grads, 0.05, 0.9, 1e-4)
    assert np.array_equal(tmod.to_numpy(out), want)
    kv.close()


def test_zero_copy_endpoints(engine):
    kvstore, optim, tmod = mods()
    kv = kvstore.KVStore(1, 2, engine=engine)
    kv.init(0, np.arange(10, dtype=F32))
    w0, g0 = kv.weight_tensor(0, 0), kv.grad_tensor(0, 0)
    w1, g1 = kv.weight_tensor(0, 1), kv.grad_tensor(0, 1)
    assert np.array_equal(tmod.to_numpy(w1), np.arange(10, dtype=F32))
    tmod.load_host(g0, np.ones(10, F32))
    tmod.load_host(g1, np.full(10, 2, F32))
    kv.push(0, g0, 0)
    kv.push(0, g1, 1)
    kv.pull(0, w0, 0)   # no-op copy: the replica is the bound tensor
    assert np.array_equal(tmod.to_numpy(w0), np.arange(10, dtype=F32) + 3)
    assert kv.stats()["launches"] == 1
    kv.close()
