"""Per-direction NVLink bandwidth of the access patterns the KV round uses,
through the store's own CUDA IPC mappings (torchrun, one rank per GPU).

Each rank moves S/N bytes to/from every peer in a rotating schedule:
  read   : copy peer[(r+k)%N] slice -> local        (remote loads)
  write  : copy local -> peer[(r+k)%N] slice        (remote stores)
  mixed  : one read kernel and one write kernel per step, same stream
Reports per-direction GB/s = (N-1)/N * S / t per rank (max time over ranks).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    eng = Engine(device=local)
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    n = (mb << 20) // 4
    kv = KVStore(1, world, engine=eng, distributed=True)
    kv.init(0, np.zeros(n, np.float32))
    kv.weight_tensor(0, rank)  # materialise
    ar = kv._arenas[0]
    part = n // world
    scratch = torch.empty(n, dtype=torch.float32, device=f"cuda:{local}")
    st = eng.stream_handle

    side = [torch.cuda.Stream(device=f"cuda:{local}") for _ in range(2 * world)]

    def run_ce(kind):
        # copy engines: one cudaMemcpyAsync per peer, each on its own stream
        # (forked from / joined back into the engine stream)
        ev0 = torch.cuda.Event()
        ev0.record(eng.stream)
        for k in range(1, world):
            peer = (rank + k) % world
            for j, what in enumerate(("read", "write")):
                if kind not in ("ce_" + what, "ce_mixed"):
                    continue
                s_ = side[2 * k + j]
                s_.wait_event(ev0)
                if what == "read":
                    L.call("mgx_memcpy_async", scratch.data_ptr() + 4 * k * part,
                           ar.grads[peer] + 4 * rank * part, 4 * part, s_.cuda_stream)
                else:
                    L.call("mgx_memcpy_async", ar.weights[peer] + 4 * rank * part,
                           scratch.data_ptr() + 4 * k * part, 4 * part, s_.cuda_stream)
                e = torch.cuda.Event()
                e.record(s_)
                eng.stream.wait_event(e)

    def run(kind):
        if kind.startswith("ce_"):
            return run_ce(kind)
        for k in range(1, world):
            peer = (rank + k) % world
            if kind in ("read", "mixed"):
                L.call("mgx_copy", ar.grads[peer] + 4 * rank * part,
                       scratch.data_ptr() + 4 * k * part, part, st)
            if kind in ("write", "mixed"):
                L.call("mgx_copy", scratch.data_ptr() + 4 * k * part,
                       ar.weights[peer] + 4 * rank * part, part, st)

    out = {"n": world, "key_mb": mb}
    for kind in ("read", "write", "mixed", "ce_read", "ce_write", "ce_mixed"):
        for _ in range(2):
            run(kind)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        reps = 10
        for _ in range(reps):
            run(kind)
        b.record(eng.stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # per direction per rank: (N-1)/N*S each way; mixed carries both
        bytes_dir = (world - 1) * part * 4
        if kind in ("mixed",):
            bytes_dir *= 2  # one stream carries both directions' bytes in sequence
        out[kind + "_GBps_per_dir"] = bytes_dir / (float(t.item()) * 1e-3) / 1e9
    dist.barrier()
    kv.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
