"""Benchmark: data-parallel training step (config-1 MLP) over the device
KVStore, plus the KVStore push+pull bus bandwidth sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by the driver under torchrun (one rank per GPU, NCCL only
for host-side barriers and max-over-ranks; the KVStore data path is the
fused P2P kernel).  Prints ONE JSON line on rank 0.

A step = every GPU runs forward + backward of the config-1 MLP
(784-128-64-10, SoftmaxOutput) on its batch of 100, then one KVStore round
(tree-reduce gradients over all GPUs, momentum SGD on the owner shard,
broadcast weights).  Weak scaling: 100 images per GPU per step.

value : device-resident step (whole step captured as one CUDA graph),
        timed with CUDA events per step, L2 flushed between steps
e2e   : the public API per step -- load_host of the batch from pinned host
        memory, DataParallelStep.step(), D2H of the softmax output
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PER_GPU_BATCH = 100
HIDDEN, CLASSES, DIM = [128, 64], 10, 784
ETA, MOM, WD = 0.05, 0.9, 1e-4
METRIC = "train images/sec"
WORKLOAD = ("config-1 MLP 784-128-64-10 SoftmaxOutput, batch 100 per GPU, momentum SGD "
            "(lr 0.05, mom 0.9, wd 1e-4), kvstore device (fused P2P reduce+SGD+broadcast)")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and throttle reasons every 50 ms through NVML while
    the timed region runs (the nvidia-smi query fields of the profiling
    recipe, read via nvidia-ml-py)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.smax = None
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            return self
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, rs))
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(0.05)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": ["unsampled"]}
        reasons = sorted({name for _sm, rs in self.samples
                          for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.smax, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ dist

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------- reference arm

def cpu_step_sample(nworkers: int, seconds: float, steps: int = None):
    """The oracle port of the reference step (oracle/step.py) on host cores:
    nworkers shards of 100 images, forward/backward per shard, tree merge and
    the SGD updater per key.  Returns (images/s, steps, seconds)."""
    from oracle import numerics as nm
    from oracle import step as ostep
    feats, labels = ostep.cfg1_data(PER_GPU_BATCH * nworkers, seed=0)
    params = ostep.init_params(HIDDEN, CLASSES, DIM, 0)
    vel = {k: np.zeros_like(v) for k, v in params.items()}
    done, t0 = 0, time.perf_counter()
    while True:
        grads = []
        for w in range(nworkers):
            sl = slice(w * PER_GPU_BATCH, (w + 1) * PER_GPU_BATCH)
            grads.append(ostep.mlp_forward_backward(params, HIDDEN, feats[sl], labels[sl])[1])
        for k in params:
            total = nm.kv_merge([g[k] for g in grads])
            params[k], vel[k] = nm.kv_updater(params[k], total, vel[k], ETA, MOM, WD, nworkers)
        done += 1
        el = time.perf_counter() - t0
        if (steps is not None and done >= steps) or (steps is None and el >= seconds and done >= 3):
            return done * PER_GPU_BATCH * nworkers / el, done, el


def run_reference(args, world, rank):
    if rank != 0:
        return
    n = args.gpus
    for _ in range(args.warmup):
        cpu_step_sample(n, 0, steps=1)
    value, steps, el = cpu_step_sample(n, 0, steps=args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (RandomState(0).rand features, randint labels)",
        "config": {"workload": WORKLOAD, "global_batch": PER_GPU_BATCH * n,
                   "per_gpu_batch": PER_GPU_BATCH, "parallelism": f"dp{n}"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": 1, "kind": "port",
                         "sample": f"{steps} steps x {n} worker shards of 100 images, "
                                   "oracle/step.py restatement (numpy, single thread)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- our arm

def algorithmic(label: str, ex_shapes) -> tuple:
    """(bytes, flops) a program instruction must move/compute, from its label."""
    return ex_shapes.get(label, (0, 0))


def run_ours(args, world, rank, local):
    import torch
    from oracle import step as ostep
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params, mlp

    torch.cuda.set_device(local)
    eng = Engine(device=local)
    distributed = world > 1
    kv = KVStore(1, world, engine=eng, distributed=distributed)
    symbol.reset_names()
    g = mlp(HIDDEN, CLASSES)
    given = {"data": (PER_GPU_BATCH, DIM), "label": (PER_GPU_BATCH,)}
    shapes, _ = symbol.infer_shape(g, given)
    step = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng)
    kv.set_updater(make_sgd_updater(SGDConfig(ETA, MOM, WD), scale=world))
    w = step.workers[0]
    feats, labels = ostep.cfg1_data(PER_GPU_BATCH * world, seed=0)
    sl = slice(w * PER_GPU_BATCH, (w + 1) * PER_GPU_BATCH)
    pin_x = torch.from_numpy(feats[sl].copy()).pin_memory()
    pin_y = torch.from_numpy(labels[sl].copy()).pin_memory()
    step.load(w, pin_x, pin_y)
    eng.wait_all()

    # ---- device-resident step: warm up eagerly, then capture the whole step
    for _ in range(max(args.warmup, 3)):
        step.step()
    eng.wait_all()
    step.capture()
    for _ in range(3):
        step.replay()
    eng.wait_all()
    barrier(world)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches_per_step = step.execs[w].num_instructions + 1
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        align = torch.zeros(1, device=f"cuda:{local}") if world > 1 else None
        for i in range(args.steps):
            L.call("mgx_fill", flush.data_ptr(), flush.numel(), float(i), eng.stream_handle)
            if align is not None:
                # untimed: re-align the ranks on-device after their independent
                # L2 flushes, so the step's in-kernel barrier does not charge
                # flush skew to the timed region
                with torch.cuda.stream(eng.stream):
                    torch.distributed.all_reduce(align)
            starts[i].record(eng.stream)
            step.replay()
            ends[i].record(eng.stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_local = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_total = max_over_ranks(ms_local, world)
    ms_per_step = ms_total / args.steps
    value = PER_GPU_BATCH * world * args.steps / (ms_total / 1e3)

    # ---- e2e through the public API: host batch in, softmax output out
    for ex in step.execs.values():
        ex._use_graph = True
    h2d = pin_x.numel() * 4 + pin_y.numel() * 4
    d2h = PER_GPU_BATCH * CLASSES * 4
    out_pin = torch.empty(PER_GPU_BATCH, CLASSES, dtype=torch.float32, pin_memory=True)
    y = step.execs[w].outputs[0]

    def e2e_step():
        step.step({w: (pin_x, pin_y)})
        eng.push(lambda: L.call("mgx_memcpy_async", out_pin.data_ptr(), y.ptr, d2h,
                                eng.stream_handle), reads=[y.tag])
        eng.wait_for(y.tag)

    for _ in range(max(args.warmup, 3)):
        e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_value = PER_GPU_BATCH * world * args.steps / (e2e_ms / 1e3)
    barrier(world)

    # ---- roofline: per-kernel device time of the step's instructions (eager,
    # events on the launching stream), averaged over K profiled steps
    ex = step.execs[w]
    prof = {}
    for _ in range(args.steps):
        for lbl, ms in ex.profile():
            prof.setdefault(lbl, []).append(ms)
    kv_ms = []
    ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        for i in range(len(step.names)):
            kv.push(i, step.grads[w][step.names[i]], w)
        ka.record(eng.stream)
        with kv._lock:
            kv._flush_locked()
        kb.record(eng.stream)
        torch.cuda.synchronize()
        kv_ms.append(ka.elapsed_time(kb))
    avg = {k: sum(v) / len(v) for k, v in prof.items()}
    avg["kv_round"] = sum(kv_ms) / len(kv_ms)
    hbm, _bf16, src = peaks()
    traffic = {lbl: cost[0] for lbl, cost in zip(ex.instr_labels, ex.instr_costs)}
    key_elems = sum(int(np.prod(shapes[n])) for n in step.names)
    # per rank and round: read the W gradient shards, w and v of its shard;
    # write v and W replicas of the new weights
    shard = key_elems / world
    traffic["kv_round"] = int(4 * shard * (2 * world + 3))
    dom = max(avg, key=avg.get)
    dom_bytes = traffic.get(dom)
    achieved = dom_bytes / (avg[dom] * 1e-3) / 1e9 if dom_bytes else None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                "peak_source": src, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None,
                "traffic": None, "kernel_ms": avg[dom],
                "step_share": avg[dom] / sum(avg.values()),
                "per_kernel_ms": avg}

    # ---- KVStore sweep: push+pull+update rounds on big keys (busbw)
    kvres = kv_sweep(args, eng, world, rank, distributed)

    # ---- CPU baseline (rank 0, N=1 only): oracle port, bounded sample
    cpu = None
    if rank == 0 and world == 1:
        v, nsteps, el = cpu_step_sample(1, args.cpu_seconds)
        cpu = {"value": v, "unit": "images/s", "cores": 1, "kind": "port",
               "sample": f"{nsteps} steps of 100 images ({el:.1f} s), oracle/step.py "
                         "restatement of the reference step (numpy, single thread)"}
    kv.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (RandomState(0).rand features, randint labels; resident batch)",
            "config": {"workload": WORKLOAD, "global_batch": PER_GPU_BATCH * world,
                       "per_gpu_batch": PER_GPU_BATCH, "parallelism": f"dp{world}",
                       "l2": "flushed between timed steps (256 MB device write, untimed)",
                       "step": "forward+backward+KVStore round captured as one CUDA graph",
                       "program_kernel": step.execs[w].uses_program_kernel},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "DataParallelStep.step(host pinned batch) + D2H softmax output + sync"},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "kvstore": kvres,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


def kv_sweep(args, eng, world, rank, distributed):
    import torch
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    out = []
    hbm, _b, _s = peaks()
    for mb in args.kv_mb:
        n = (mb << 20) // 4
        kv = KVStore(1, world, engine=eng, distributed=distributed)
        kv.init(0, np.zeros(n, np.float32))
        kv.set_updater(make_sgd_updater(SGDConfig(ETA, MOM, WD), scale=world))
        w = kv.local_workers[0]
        gt, wt = kv.grad_tensor(0, w), kv.weight_tensor(0, w)
        rounds = max(3, min(args.steps, 20))
        for _ in range(3):
            kv.push(0, gt, w)
            kv.pull(0, wt, w)
        eng.wait_all()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        for _ in range(rounds):
            kv.push(0, gt, w)
            kv.pull(0, wt, w)
        b.record(eng.stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(a.elapsed_time(b), world) / rounds
        kv.close()
        S = 4 * n
        algbw = S / (ms * 1e-3) / 1e9
        rec = {"key_bytes": S, "ms_per_round": ms, "algbw_GBps": algbw}
        if world > 1:
            busbw = algbw * 2 * (world - 1) / world
            rec.update({"busbw_GBps": busbw, "nvlink_frac_of_900": busbw / 900.0,
                        "nvlink_frac_of_measured_770": busbw / 770.0})
        else:
            # one worker: read g, w, v; write v, w -> 5 S bytes of HBM
            rec.update({"hbm_GBps": 5 * S / (ms * 1e-3) / 1e9,
                        "hbm_frac": 5 * S / (ms * 1e-3) / 1e9 / hbm})
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--kv-mb", type=int, nargs="*", default=[64, 256])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        # CPU reference arm: rank 0 alone times the oracle port; the other
        # ranks have no work and exit immediately
        run_reference(args, world, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
