"""One rank of the multi-GPU KVStore checks (launched by test_kv_dist_gpu.py
under torchrun; one process per GPU, worker id == rank)."""

import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
F32 = np.float32


def check_kv_golden(eng, world, rank, failures):
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    golden = np.load(os.path.join(ROOT, "tests", "golden", "kv_golden.npz"))
    numels = [1000, 10, 5003]
    for bucket, push in ((4 << 20, False), (4096, False), (4 << 20, True), (4096, True)):
        for upd in ("sgd", "add"):
            kv = KVStore(1, world, engine=eng, distributed=True, bucket_bytes=bucket)
            kv.push_mode = push  # all-remote-store rounds: same tree order, bitwise
            for key, n in enumerate(numels):
                kv.init(key, (np.random.RandomState(key).randn(n) * 0.1).astype(F32))
            if upd == "sgd":
                kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=world))
            for r in range(3):
                for key, n in enumerate(numels):
                    g = np.random.RandomState(1000 + rank + 100 * r + 10000 * key).randn(n)
                    kv.push(key, tmod.from_host((n,), "float32", g.astype(F32), engine=eng), rank)
            for key, n in enumerate(numels):
                o = tmod.zeros((n,), engine=eng)
                kv.pull(key, o, rank)
                got = tmod.to_numpy(o)
                want = golden[f"m1w{world}_{upd}_k{key}"]
                if not np.array_equal(got, want):
                    failures.append(f"kv {upd} bucket={bucket} push={push} key={key}: "
                                    f"max diff {np.abs(got - want).max()}")
            kv.round_barrier()
            kv.close()


def check_training(eng, world, rank, failures):
    from oracle import step as ostep
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200.optim import SGDConfig
    from paper_1512_01274_b200.train import mlp, train_distributed
    batch = 100 if 100 % world == 0 else 128
    feats, labels = ostep.cfg1_data(5 * batch)
    symbol.reset_names()
    _rep, params = train_distributed(mlp([128, 64], 10), (feats, labels),
                                     SGDConfig(0.05, 0.9, 1e-4), epochs=1, batch=batch,
                                     machines=1, workers=world, distributed=True, engine=eng)
    want, _ = ostep.train_distributed([128, 64], 10, feats, labels, 0.05, 0.9, 1e-4, epochs=1,
                                      batch=batch, machines=1, workers=world)
    for k, v in want.items():
        if not np.allclose(params[k], v, rtol=1e-5, atol=1e-6):
            failures.append(f"train {k}: max diff {np.abs(params[k] - v).max()}")


def check_capture(eng, world, rank, failures):
    import torch
    from oracle import step as ostep
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params, mlp
    feats, labels = ostep.cfg1_data(100 * world)
    outs = []
    for captured in (False, True):
        symbol.reset_names()
        g = mlp([128, 64], 10)
        given = {"data": (100, 784), "label": (100,)}
        shapes, _ = symbol.infer_shape(g, given)
        kv = KVStore(1, world, engine=eng, distributed=True)
        st = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng)
        kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=world))
        st.load(rank, feats[rank * 100:(rank + 1) * 100], labels[rank * 100:(rank + 1) * 100])
        if captured:
            st.step()
            st.capture()
            for _ in range(9):
                st.replay()
        else:
            for _ in range(10):
                st.step()
        kv.round_barrier()
        outs.append({n: tmod.to_numpy(st.args[rank][n]) for n in st.names})
        kv.close()
    for n in outs[0]:
        if not np.array_equal(outs[0][n], outs[1][n]):
            failures.append(f"capture {n} differs from eager")


def check_convnet(eng, world, rank, failures):
    """LeNet (bf16 tensor-core convs, config 3) trained 3 steps with one
    rank per GPU == the same step with all `world` workers in one process
    (bitwise: identical kernels, identical tree order in the store).  The
    distributed runs cover the store's rounds inside the backward program
    (push/backward overlap, eager and captured) and after it."""
    from paper_1512_01274_b200 import nets, symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params
    rs = np.random.RandomState(7)
    xs = rs.randn(3, 16 * world, 28, 28, 1).astype(F32)
    ls = rs.randint(0, 10, (3, 16 * world)).astype(F32)
    given = {"data": (16, 28, 28, 1), "label": (16,)}
    results = []
    variants = ((True, True, False), (False, True, False), (True, False, False),
                (True, True, True))
    for distributed, overlap, captured in variants:
        symbol.reset_names()
        g = nets.lenet(10)
        shapes, _ = symbol.infer_shape(g, given)
        # small buckets so the step has several rounds inside the backward
        kv = KVStore(1, world, engine=eng, distributed=distributed, bucket_bytes=1 << 16)
        st = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng, dense="bf16",
                              overlap=overlap)
        kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=world))
        for s in range(3):
            shard = {w: (xs[s, 16 * w:16 * (w + 1)], ls[s, 16 * w:16 * (w + 1)])
                     for w in st.workers}
            if captured and s > 0:
                for w in st.workers:
                    st.load(w, *shard[w])
                if s == 1:
                    st.capture()
                st.replay()
            else:
                st.step(shard)
        kv.round_barrier()
        if distributed and overlap and not st.embedded:
            failures.append("distributed 1-worker step did not embed its rounds")
        w0 = st.workers[0]
        results.append({n: tmod.to_numpy(st.args[w0][n]) for n in st.names})
        kv.close()
    for v, other in zip(variants[1:], results[1:]):
        for n in results[0]:
            if not np.array_equal(results[0][n], other[n]):
                failures.append(f"convnet {n}: variant {v} != distributed overlapped "
                                f"(max diff {np.abs(results[0][n] - other[n]).max()})")


def main():
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1512_01274_b200.engine import Engine
    eng = Engine(device=local)
    failures = []
    for check in (check_kv_golden, check_training, check_capture, check_convnet):
        try:
            check(eng, world, rank, failures)
        except Exception:  # noqa: BLE001
            failures.append(f"{check.__name__} raised:\n{traceback.format_exc()}")
        dist.barrier()
    out = os.environ.get("DIST_RESULT_DIR", ".")
    with open(os.path.join(out, f"rank{rank}.txt"), "w") as f:
        f.write("\n".join(failures) if failures else "OK")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
