"""Multi-process host logic of the distributed KVStore, world_size 2 over
gloo on CPU: every rank plans its flushes independently, the plans agree on
launch counts, the owner segments tile every key exactly once, and a
rank-sharded round (numpy arithmetic, compact momentum layout, 3 rounds)
reproduces the whole-key oracle bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kv as okv
        from oracle import numerics as nm
        from paper_1512_01274_b200.kvstore import (compact_velocity_layout, launches_for,
                                                   owner_segments, padded, plan_buckets)
        rs = np.random.RandomState(11)
        failures = []
        for trial in range(20):
            numels = [int(x) for x in rs.randint(1, 40000, rs.randint(1, 30))]
            bucket_bytes = int(rs.choice([4096, 65536, 4 << 20]))
            offs, buckets, kb = plan_buckets(numels, bucket_bytes)
            spans = [(o, padded(n), b) for o, n, b in zip(offs, numels, kb)]
            vb, vlen = compact_velocity_layout(buckets, world, rank)
            mine = owner_segments(spans, buckets, world, rank, vb)
            counts = [len(owner_segments(spans, buckets, world, r)) for r in range(world)]
            launches = launches_for(counts, 256)
            everyone = [None] * world
            dist.all_gather_object(everyone, (mine, launches, vlen))
            # identical launch counts on every rank
            if len({e[1] for e in everyone}) != 1:
                failures.append(f"trial {trial}: launch counts differ")
            # segments tile the padded keys exactly once
            cover = np.zeros(offs[-1] + padded(numels[-1]), np.int32)
            for segs, _l, _v in everyone:
                for off, ln, _vo in segs:
                    cover[off:off + ln] += 1
            want = np.zeros_like(cover)
            for o, n in zip(offs, numels):
                want[o:o + padded(n)] = 1
            if not np.array_equal(cover, want):
                failures.append(f"trial {trial}: segments do not tile the keys")
            # this rank's momentum offsets stay inside its compact buffer, disjoint
            used = np.zeros(max(vlen, 1), np.int32)
            for _off, ln, vo in mine:
                if vo < 0 or vo + ln > vlen:
                    failures.append(f"trial {trial}: momentum offset out of range")
                    break
                used[vo:vo + ln] += 1
            if used.max(initial=0) > 1:
                failures.append(f"trial {trial}: momentum ranges overlap")

            # rank-sharded SGD rounds == whole-key oracle, bitwise
            total = offs[-1] + padded(numels[-1])
            w = np.zeros(total, np.float32)
            for o, n in zip(offs, numels):
                w[o:o + n] = (np.random.RandomState(o).randn(n) * 0.1).astype(np.float32)
            w_ref, v_ref = w.copy(), np.zeros(total, np.float32)
            v_mine = np.zeros(max(vlen, 1), np.float32)
            for r in range(3):
                g_local = np.zeros(total, np.float32)
                for o, n in zip(offs, numels):
                    g_local[o:o + n] = np.random.RandomState(1000 + rank + 100 * r + o).randn(n)
                grads = [None] * world
                dist.all_gather_object(grads, g_local)           # stands in for IPC reads
                new_w = w.copy()
                for off, ln, vo in mine:
                    sl = slice(off, off + ln)
                    nw_, nv = okv.sgd_round(w[sl], v_mine[vo:vo + ln], [g[sl] for g in grads],
                                            0.05, 0.9, 1e-4)
                    new_w[sl], v_mine[vo:vo + ln] = nw_, nv
                pieces = [None] * world
                dist.all_gather_object(pieces, [(off, new_w[off:off + ln]) for off, ln, _ in mine])
                for plist in pieces:                             # stands in for remote stores
                    for off, arr in plist:
                        w[off:off + len(arr)] = arr
                w_ref, v_ref = okv.sgd_round(w_ref, v_ref, grads, 0.05, 0.9, 1e-4)
            if not np.array_equal(w, w_ref):
                failures.append(f"trial {trial}: sharded rounds differ from the oracle")
        with open(os.path.join(result_dir, f"rank{rank}.txt"), "w") as f:
            f.write("\n".join(failures) if failures else "OK")
    finally:
        dist.destroy_process_group()


def test_distributed_kv_host_logic_world2(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"rank{r}.txt").read_text() == "OK"
