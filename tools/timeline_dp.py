"""GPU timeline of the data-parallel step (bench.py's configuration, the
whole step replayed from its CUDA graph) under torchrun: where the KVStore
rounds run relative to the backward (push/backward overlap evidence).

    torchrun --nproc-per-node N tools/timeline_dp.py [config] [--trace out.json]

Rank 0 prints: step span, the backward's kernel span, each kv_round kernel's
start/end relative to the step start, and how much of the KV time overlapped
other kernels."""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "alexnet"
    import torch
    import torch.distributed as dist
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params
    world, rank, local = bench.dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    eng = Engine(device=local)
    cfg = bench.CONFIGS[name]
    per = cfg["batch"]
    kv = KVStore(1, world, engine=eng, distributed=world > 1)
    g = bench.build_graph(name)
    given = {"data": (per,) + cfg["image"], "label": (per,)}
    shapes, _ = symbol.infer_shape(g, given)
    step = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng,
                            dense=cfg["dense"], strategy=cfg.get("strategy", "both"),
                            split_target=cfg.get("split_target", 0),
                            hoist_wgrad=cfg.get("hoist_wgrad"))
    kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=world))
    x, y = bench.synthetic(name, per, rank)
    step.load(step.workers[0], x, y)
    for _ in range(3):
        step.step()
    step.capture()
    for _ in range(3):
        step.replay()
    eng.wait_all()
    bench.barrier(world)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            step.replay()
        eng.wait_all()
    bench.barrier(world)
    if rank == 0:
        path = (sys.argv[sys.argv.index("--trace") + 1] if "--trace" in sys.argv
                else os.path.join(tempfile.gettempdir(), "mgx_timeline_dp.json"))
        prof.export_chrome_trace(path)
        ks = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
        ks.sort(key=lambda e: e["ts"])
        n = len(ks) // 3
        ks = ks[-n:]
        t0 = ks[0]["ts"]
        end = max(e["ts"] + e["dur"] for e in ks)
        kvk = [e for e in ks if "kv_round" in e["name"]]
        other = [e for e in ks if "kv_round" not in e["name"]]
        print(f"{name} N={world}: step span {(end - t0) / 1e3:.3f} ms, {len(ks)} kernels, "
              f"embedded rounds: {step.embedded}")
        last_other = max(e["ts"] + e["dur"] for e in other)
        print(f"  last non-KV kernel ends at {(last_other - t0) / 1e3:.3f} ms")
        ov_total, kv_total = 0.0, 0.0
        for e in kvk:
            s, f = e["ts"], e["ts"] + e["dur"]
            # time of this KV kernel during which another kernel was running
            ivs = sorted((max(s, o["ts"]), min(f, o["ts"] + o["dur"])) for o in other
                         if o["ts"] < f and o["ts"] + o["dur"] > s)
            cov, cur = 0.0, s
            for a, b in ivs:
                if b > cur:
                    cov += b - max(a, cur)
                    cur = max(cur, b)
            ov_total += cov
            kv_total += f - s
            print(f"  kv_round {(s - t0) / 1e3:7.3f} -> {(f - t0) / 1e3:7.3f} ms "
                  f"({e['dur']:.1f} us, overlapped {cov:.1f} us)")
        print(f"  KV kernels {kv_total / 1e3:.3f} ms, overlapped with compute "
              f"{ov_total / 1e3:.3f} ms ({100 * ov_total / max(kv_total, 1):.0f} %)")
    kv.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
