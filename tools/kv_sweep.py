"""KVStore push+pull+SGD round bandwidth under torchrun (one rank per GPU).

    torchrun --nproc-per-node N tools/kv_sweep.py --mb 64 256 [--rounds 20]

Prints one JSON line per key size on rank 0: ms per round (max over ranks),
algbw = S/t and busbw = algbw * 2(N-1)/N.  The launch shape can be varied
with MGX_KV_VARIANT="<unroll>,<threads>".
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, nargs="+", default=[64, 256])
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--nccl", action="store_true",
                    help="also time NCCL all_reduce (fp32, sum) on the same sizes: the "
                         "library baseline for the collective part alone")
    args = ap.parse_args()
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    eng = Engine(device=local)
    for mb in args.mb:
        n = (mb << 20) // 4
        kv = KVStore(1, world, engine=eng, distributed=True)
        kv.init(0, np.zeros(n, np.float32))
        kv.set_updater(make_sgd_updater(SGDConfig(0.05, 0.9, 1e-4), scale=world))
        g, w = kv.grad_tensor(0, rank), kv.weight_tensor(0, rank)
        for _ in range(3):
            kv.push(0, g, rank)
            kv.pull(0, w, rank)
        eng.wait_all()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        for _ in range(args.rounds):
            kv.push(0, g, rank)
            kv.pull(0, w, rank)
        b.record(eng.stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.rounds], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kv.close()
        ms = float(t.item())
        S = 4 * n
        algbw = S / (ms * 1e-3) / 1e9
        if rank == 0:
            print(json.dumps({"n": world, "variant": os.environ.get("MGX_KV_VARIANT", "default"),
                              "key_mb": mb, "ms": ms, "algbw": algbw,
                              "busbw": algbw * 2 * (world - 1) / world}), flush=True)
        if args.nccl:
            x = torch.ones(n, dtype=torch.float32, device=f"cuda:{local}")
            for _ in range(3):
                dist.all_reduce(x)
            torch.cuda.synchronize()
            dist.barrier()
            a.record()
            for _ in range(args.rounds):
                dist.all_reduce(x)
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / args.rounds], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nms = float(t.item())
            nalg = S / (nms * 1e-3) / 1e9
            if rank == 0:
                print(json.dumps({"n": world, "variant": "nccl_all_reduce", "key_mb": mb, "ms": nms,
                                  "algbw": nalg, "busbw": nalg * 2 * (world - 1) / world}),
                      flush=True)
            del x
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
