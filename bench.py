"""Benchmark: the data-parallel training step over the device KVStore.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config inception_bn|alexnet|lenet|mlp] [--no-extra]

N>1 is launched by the driver under torchrun (one rank per GPU; NCCL only
for host-side barriers and max-over-ranks; the KVStore data path is the
fused P2P kernel).  Prints ONE JSON line on rank 0.

Headline (BASELINE.json metric "train images/sec at 1/2/4/8 B200", quoted on
config 5): Inception-BN, synthetic 224x224x3 images, batch 64 per GPU, bf16
tensor-core convolutions (fp32 activations, BatchNorm, softmax; fp32 master
weights in the KVStore), momentum SGD.  A step = every GPU runs forward +
backward on its 64 images, then one KVStore round (tree-reduce gradients
over all GPUs, SGD on the owner shard, broadcast weights).  Weak scaling.

value : device-resident step (whole step captured as one CUDA graph), CUDA
        events per step on the step's stream, L2 flushed between steps
e2e   : the public API per step -- the batch from pinned host memory,
        DataParallelStep.step(), D2H of the softmax output, sync
Also reported: the other configurations (MLP config 1 with its pinned
reference, LeNet, AlexNet-style) and the KVStore push+pull sweep (config 2).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ETA, MOM, WD = 0.05, 0.9, 1e-4
METRIC = "train images/sec"

CONFIGS = {
    "mlp": dict(batch=100, image=(784,), classes=10, dense="fp32", dtype="fp32",
                workload="config-1 MLP 784-128-64-10 SoftmaxOutput, batch 100 per GPU, momentum "
                         "SGD (lr 0.05, mom 0.9, wd 1e-4), exact-order fp32 kernels, kvstore "
                         "device (fused P2P reduce+SGD+broadcast)"),
    "lenet": dict(batch=128, image=(28, 28, 1), classes=10, dense="bf16", dtype="bf16",
                  workload="config-3 LeNet (conv5x5x20-tanh-pool, conv5x5x50-tanh-pool, fc500, "
                           "fc10), synthetic 28x28x1, batch 128 per GPU, kvstore device"),
    # hoist_wgrad: weight gradients issued as soon as their inputs exist
    # (the chain's dW GEMMs overlap the dX chain: 2.42 -> 2.27 ms)
    "alexnet": dict(batch=128, image=(224, 224, 3), classes=1000, dense="bf16", dtype="bf16",
                    hoist_wgrad=True,
                    workload="config-4 AlexNet-style (5 conv, fc6 4096x9216, fc7, fc8; 62M params), "
                             "synthetic 224x224x3, batch 128 per GPU, kvstore device"),
    # strategy "inplace": no co-shared slots between independent branches
    # (their reuse adds write-after-read edges across lanes: 5.24 -> 5.19 ms);
    # split_target 20: split-K sized for ~20 CTAs per GEMM, the inception
    # branches run side by side (128 -> 32: 4.83 -> 4.67 ms; with 8 lanes
    # 32 -> 20: 4.60 -> 4.51 ms; a chain like AlexNet keeps the default 128)
    "inception_bn": dict(batch=64, image=(224, 224, 3), classes=1000, dense="bf16", dtype="bf16",
                         strategy="inplace", split_target=20,
                         workload="config-5 Inception-BN (MXNet symbol, 69 conv+BN+ReLU, 10 "
                                  "inception concats), synthetic 224x224x3, batch 64 per GPU, bf16 "
                                  "tensor-core convs, momentum SGD, kvstore device"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), \
            "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, 1400.0, "fallback"


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


# -------------------------------------------------------- configurations

def build_graph(name: str):
    from paper_1512_01274_b200 import nets, symbol
    from paper_1512_01274_b200.train import mlp
    symbol.reset_names()
    if name == "mlp":
        return mlp([128, 64], 10)
    return nets.NETS[name](CONFIGS[name]["classes"])


def synthetic(name: str, n: int, seed: int):
    """Seeded synthetic batch of ``n`` images: config 1 as SURVEY §8d
    (RandomState.rand features, randint labels); conv nets randn images."""
    cfg = CONFIGS[name]
    if name == "mlp":
        from oracle import step as ostep
        return ostep.cfg1_data(n, seed=seed)
    rs = np.random.RandomState(seed)
    x = rs.randn(n, *cfg["image"]).astype(np.float32)
    y = rs.randint(0, cfg["classes"], n).astype(np.float32)
    return x, y


def train_flops_per_image(name: str) -> float:
    """Tensor-core FLOPs of one training image: forward contractions, plus
    weight gradients (same FLOPs), plus data gradients for every layer but
    the first (whose input needs no gradient)."""
    from paper_1512_01274_b200 import nets
    g = build_graph(name)
    b = CONFIGS[name]["batch"]
    given = {"data": (b,) + CONFIGS[name]["image"], "label": (b,)}
    fwd = nets.forward_flops(g, given)
    from paper_1512_01274_b200 import symbol
    _a, named = symbol.infer_shape(g, given)
    first = next(n for n in g.topo_nodes() if n.op in ("Convolution", "FullyConnected"))
    from math import prod
    w = named[first.inputs[1][0].name]
    first_fl = 2 * prod(named[first.name]) * (prod(w[1:]) if first.op == "Convolution" else 1)
    if first.op == "FullyConnected":
        first_fl = 2 * named[first.name][0] * prod(w)
    return (3 * fwd - first_fl) / b


# ------------------------------------------------------- reference arm

def cpu_sample(name: str, seconds: float = None, steps: int = None, nworkers: int = 1):
    """The CPU oracle port of one training step on host cores.

    mlp: oracle/step.py (numpy restatement of the reference step, pinned
    bitwise to the reference; single thread, like numpy's ufunc reductions).
    conv nets: oracle/convnet.py float64 torch-CPU restatement on a small
    sample of images per step (the reference has no conv operators; this is
    the port the GPU path is checked against), all host threads.
    Returns (images/s, steps, seconds, cores, sample description)."""
    if name == "mlp":
        from oracle import numerics as nm
        from oracle import step as ostep
        per = CONFIGS["mlp"]["batch"]
        feats, labels = ostep.cfg1_data(per * nworkers, seed=0)
        params = ostep.init_params([128, 64], 10, 784, 0)
        vel = {k: np.zeros_like(v) for k, v in params.items()}
        done, t0 = 0, time.perf_counter()
        while True:
            grads = []
            for w in range(nworkers):
                sl = slice(w * per, (w + 1) * per)
                grads.append(ostep.mlp_forward_backward(params, [128, 64], feats[sl], labels[sl])[1])
            for k in params:
                total = nm.kv_merge([g[k] for g in grads])
                params[k], vel[k] = nm.kv_updater(params[k], total, vel[k], ETA, MOM, WD, nworkers)
            done += 1
            el = time.perf_counter() - t0
            if (steps is not None and done >= steps) or (steps is None and el >= seconds and done >= 3):
                return (done * per * nworkers / el, done, el, 1,
                        f"{done} steps x {nworkers} shards of {per} images, oracle/step.py numpy "
                        "restatement of the reference step (single thread)")
    import torch
    from oracle import convnet as oc
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200.train import init_aux, init_params, param_names
    g = build_graph(name)
    sample = CONFIGS[name]["batch"]  # the full per-GPU batch of the config
    given = {"data": (sample,) + CONFIGS[name]["image"], "label": (sample,)}
    shapes, _ = symbol.infer_shape(g, given)
    x, y = synthetic(name, sample, 0)
    vals = {"data": x, "label": y, **init_params(g, shapes, 0), **init_aux(g, shapes)}
    names = param_names(g)
    done, t0 = 0, time.perf_counter()
    while True:
        oc.run_graph(g, vals, wrt=names, dtype="float32")
        done += 1
        el = time.perf_counter() - t0
        if (steps is not None and done >= steps) or (steps is None and el >= seconds and done >= 1):
            return (done * sample / el, done, el, torch.get_num_threads(),
                    f"{done} forward+backward passes of the full {sample}-image batch, "
                    "oracle/convnet.py restatement in fp32 torch-CPU (the reference has no "
                    "convolution operators, so no reference CPU number exists for this config)")


def host_cpu() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def reference_own(seconds: float = 20.0) -> dict:
    """The reference's OWN CPU implementation (minigraph from baseline/_ref,
    installed offline from /root/reference), timed on this host: config 1
    train_distributed (W=2, batch 100, engine threads 2W+6 as train.py:181)
    and config 2 KVStore(1, W) push -> pull -> wait rounds with the SGD
    updater (kvstore.py:190-241), bounded to ~``seconds`` in total."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "minigraph")):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref)
    try:
        import tempfile
        from minigraph import symbol as rsym
        from minigraph.kvstore import KVStore as RKV
        from minigraph.optim import SGDConfig as RCfg, make_sgd_updater as rmk
        from minigraph.recordio import Example, pack
        from minigraph import tensor as rt
        from minigraph.train import mlp as rmlp, train_distributed as rtd
        from oracle import step as ostep
        out = {"source": "baseline/_ref (reference minigraph, unmodified)", **host_cpu()}
        feats, labels = ostep.cfg1_data(2000)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "cfg1.rec")
            pack((Example(int(l), f) for f, l in zip(feats, labels)), path)
            rsym.reset_names()
            t0 = time.perf_counter()
            rtd(rmlp([128, 64], 10), path, RCfg(ETA, MOM, WD), epochs=1, batch=100, machines=1,
                workers=2)
            el = time.perf_counter() - t0
        out["config1"] = {"value": 2000 / el, "unit": "images/s",
                          "sample": "1 epoch of 2000 synthetic MNIST-shaped images, batch 100, "
                                    "W=2 (train_distributed incl. its per-epoch setup)"}
        kv = []
        budget = time.perf_counter() + seconds
        for nbytes in (1 << 10, 1 << 14, 1 << 18, 1 << 22, 1 << 24, 1 << 26):
            n = nbytes // 4
            for w_ in (2, 4, 8):
                if time.perf_counter() > budget:
                    break
                with RKV(1, w_) as store:
                    store.init(0, np.zeros(n, np.float32))
                    store.set_updater(rmk(RCfg(ETA, MOM, WD), scale=w_))
                    grads = [rt.from_host((n,), "float32", np.ones(n, np.float32))
                             for _ in range(w_)]
                    outs = [rt.zeros((n,)) for _ in range(w_)]
                    rounds = 0
                    t0 = time.perf_counter()
                    while rounds < 3 or (time.perf_counter() - t0 < 0.5 and rounds < 50):
                        for w in range(w_):
                            store.push(0, grads[w], w)
                        for w in range(w_):
                            store.pull(0, outs[w], w)
                        for o in outs:
                            o.engine.wait_for(o.tag)
                        rounds += 1
                    ms = (time.perf_counter() - t0) * 1e3 / rounds
                kv.append({"key_bytes": nbytes, "workers": w_, "ms_per_round": ms,
                           "algbw_GBps": nbytes / (ms * 1e-3) / 1e9})
        out["kvstore"] = kv
        return out
    except Exception as exc:  # noqa: BLE001 - report, never fail the arm
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    finally:
        sys.path.remove(ref)


def run_reference(args, world, rank):
    """CPU arm.  Headline conv nets: the oracle's fp32 torch-CPU restatement
    of the same step on the full per-GPU batch (no reference conv ops exist;
    kind "port").  Config 1 (--config mlp): the reference's own
    train_distributed from baseline/_ref when installed (kind "reference"),
    else the bitwise numpy restatement.  Plus the reference's own config-1
    and KVStore timings (``reference_own``)."""
    if rank != 0:
        return
    import torch
    # torchrun sets OMP_NUM_THREADS=1 per rank: the CPU arm uses every host core
    torch.set_num_threads(os.cpu_count() or 1)
    n = args.gpus
    name = args.config
    kind = "port"
    if name == "mlp" and os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "minigraph")):
        own = reference_own(seconds=5.0)
        value = own.get("config1", {}).get("value")
        kind = "reference" if value else "port"
    if kind == "port":
        for _ in range(args.warmup if name == "mlp" else min(args.warmup, 1)):
            cpu_sample(name, steps=1, nworkers=n)
        value, steps, el, cores, sample = cpu_sample(
            name, steps=args.steps if name == "mlp" else max(1, min(args.steps, 3)), nworkers=n)
        ms = 1e3 * el / steps
    else:
        cores, steps = 2 * 2 + 6, 1
        sample = own["config1"]["sample"]
        ms = 1e3 * CONFIGS["mlp"]["batch"] * 2 / value
    cfg = CONFIGS[name]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": n,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32", "data": "synthetic",
        "config": {"workload": cfg["workload"] + (
            " -- CPU arm: fp32 torch-CPU restatement of the same step on the host cores (the "
            "reference has no conv operators)" if name != "mlp" else ""),
            "global_batch": cfg["batch"] * n, "per_gpu_batch": cfg["batch"],
            "parallelism": f"dp{n}", "same_config": name == "mlp",
            "same_precision": name == "mlp"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind,
                         "sample": sample, **host_cpu()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not args.no_extra:
        line["reference_own"] = reference_own(seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- our arm

KERNEL_OF = {}  # opcode -> kernel family name, filled lazily


def kernel_family(op: int) -> str:
    from paper_1512_01274_b200 import _lib as L
    if not KERNEL_OF:
        KERNEL_OF.update({
            L.OP_GEMM_TC_EX: "tc_gemm_bf16 (tcgen05)", L.OP_GEMM_TC: "tc_gemm_bf16 (tcgen05)",
            L.OP_GEMM_CONV: "tc_gemm_bf16 (tcgen05)", L.OP_WFLIP: "weight_flip",
            L.OP_SUM_N: "sum_n", L.OP_CONCAT: "concat",
            L.OP_IM2COL: "im2col_bf16", L.OP_COL2IM: "col2im", L.OP_CAST_BF16: "cast_bf16",
            L.OP_BN_STATS: "bn_stats", L.OP_BN_APPLY: "bn_apply", L.OP_BN_BWD_REDUCE: "bn_bwd_reduce",
            L.OP_BN_BWD_DX: "bn_bwd_dx", L.OP_BN_FWD_FUSED: "bn_fwd_fused",
            L.OP_BN_BWD_FUSED: "bn_bwd_fused", L.OP_POOL_FWD: "pool_fwd", L.OP_POOL_BWD: "pool_bwd",
            L.OP_CHAN_COPY: "concat_copy", L.OP_COLSUM: "colsum", L.OP_ACT_FWD: "act_fwd",
            L.OP_ACT_BWD: "act_bwd", L.OP_GEMM_PW: "gemm_pairwise", L.OP_GEMM_SEQ: "gemm_sequential",
            L.OP_DW_DB: "fc_dw_db", L.OP_SOFTMAX_FWD: "softmax_fwd", L.OP_SOFTMAX_BWD: "softmax_bwd",
            L.OP_COPY: "copy", L.OP_FILL: "fill", L.OP_EW: "elementwise", L.OP_AXPY: "axpy",
            L.OP_SCALAR: "scalar", L.OP_BN_ACT_POOL: "bn_act_pool (stem fwd)",
            L.OP_BN_BWD_REDUCE_POOL: "bn_bwd_reduce_pool (stem)",
            L.OP_BN_BWD_DX_POOL: "bn_bwd_dx_pool (stem)", L.OP_PREP_BATCH: "prep_batch (weight casts)",
            L.OP_KV_ROUND: "kv_round (fused reduce+SGD+broadcast)"})
    return KERNEL_OF.get(op, f"op{op}")


def run_config(name, args, world, rank, local, eng, steps, warmup, with_e2e=True,
               with_profile=True):
    """Measure one configuration; returns a dict (rank 0 meaningful)."""
    import torch
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    from paper_1512_01274_b200.train import DataParallelStep, init_params

    cfg = CONFIGS[name]
    per = cfg["batch"]
    distributed = world > 1
    kv = KVStore(1, world, engine=eng, distributed=distributed)
    g = build_graph(name)
    given = {"data": (per,) + cfg["image"], "label": (per,)}
    shapes, _ = symbol.infer_shape(g, given)
    step = DataParallelStep(g, kv, given, init_params(g, shapes, 0), engine=eng,
                            dense=cfg["dense"], strategy=cfg.get("strategy", "both"),
                            split_target=cfg.get("split_target", 0),
                            hoist_wgrad=cfg.get("hoist_wgrad"))
    kv.set_updater(make_sgd_updater(SGDConfig(ETA, MOM, WD), scale=world))
    w = step.workers[0]
    feats, labels = synthetic(name, per * world, 0)
    sl = slice(w * per, (w + 1) * per)
    pin_x = torch.from_numpy(np.ascontiguousarray(feats[sl])).pin_memory()
    pin_y = torch.from_numpy(np.ascontiguousarray(labels[sl])).pin_memory()
    step.load(w, pin_x, pin_y)
    eng.wait_all()

    # ---- device-resident step: warm up eagerly, capture the whole step
    for _ in range(max(warmup, 3)):
        step.step()
    eng.wait_all()
    step.capture()
    for _ in range(3):
        step.replay()
    eng.wait_all()
    barrier(world)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        align = torch.zeros(1, device=f"cuda:{local}") if world > 1 else None
        for i in range(steps):
            L.call("mgx_fill", flush.data_ptr(), flush.numel(), float(i), eng.stream_handle)
            if align is not None:
                # untimed: re-align the ranks on-device after their L2 flushes
                with torch.cuda.stream(eng.stream):
                    torch.distributed.all_reduce(align)
            starts[i].record(eng.stream)
            step.replay()
            ends[i].record(eng.stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_local = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_total = max_over_ranks(ms_local, world)
    res = {"config_name": name, "workload": cfg["workload"], "per_gpu_batch": per,
           "global_batch": per * world,
           "ms_per_step": ms_total / steps,
           "value": per * world * steps / (ms_total / 1e3), "clocks": clocks.summary(),
           "dtype": cfg["dtype"]}
    ex = step.execs[w]
    res["kernels_per_step"] = ex.kernel_count() + kv_launches(kv)
    res["plan_bytes"] = step.plan_bytes
    res["scratch_bytes"] = getattr(ex, "scratch_bytes", 0)

    # ---- e2e through the public API: host batch in, softmax output out
    if with_e2e:
        for e in step.execs.values():
            e._use_graph = True
        h2d = pin_x.numel() * 4 + pin_y.numel() * 4
        d2h = per * cfg["classes"] * 4
        out_pins = [torch.empty(per, cfg["classes"], dtype=torch.float32, pin_memory=True)
                    for _ in range(2)]
        y = ex.outputs[0]
        pending = []

        def e2e_step(i):
            # this step's batch was staged (H2D on the copy stream) while the
            # previous step ran; stage the next one, queue this step's D2H of
            # the softmax output, then wait for the PREVIOUS step's output on
            # the host (a depth-1 pipeline: the host never idles the GPU)
            step.step(staged=True)
            step.stage(w, pin_x, pin_y)
            buf = out_pins[i % 2]
            eng.push(lambda: L.call("mgx_memcpy_async", buf.data_ptr(), y.ptr, d2h,
                                    eng.stream_handle), reads=[y.tag])
            ev = torch.cuda.Event()
            ev.record(eng.stream)
            pending.append(ev)
            if len(pending) > 1:
                pending.pop(0).synchronize()

        step.stage(w, pin_x, pin_y)
        for i in range(max(warmup, 3)):
            e2e_step(i)
        eng.wait_for(y.tag)
        pending.clear()
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        step.stage(w, pin_x, pin_y)  # the first timed step's copy, inside the region
        for i in range(steps):
            e2e_step(i)
        pending[-1].synchronize()  # the last step's output is on the host
        e1.record(eng.stream)
        torch.cuda.synchronize()
        eng.wait_for(y.tag)  # surface any device-side error of the timed steps
        pending.clear()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
        res["e2e"] = {"value": per * world * steps / (e2e_ms / 1e3), "unit": "images/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "path": "DataParallelStep.stage (pinned H2D on a copy stream, overlapping the "
                              "previous step) + step + D2H of the softmax output every step, the "
                              "host waiting for each step's output one step later (depth-1 "
                              "pipeline)"}
        barrier(world)

    # ---- roofline: per-instruction device time (events captured between
    # instructions on the launching stream), aggregated per kernel family
    if with_profile:
        nprof = max(1, min(steps, 5))
        times = [0.0] * ex.num_instructions
        for _ in range(nprof):
            for idx, (_lbl, ms) in enumerate(ex.profile()):
                times[idx] += ms / nprof
        fam_ms, fam_bytes, fam_flops = {}, {}, {}
        for idx, ms in enumerate(times):
            fam = kernel_family(ex.instr_ops[idx])
            fam_ms[fam] = fam_ms.get(fam, 0.0) + ms
            fam_bytes[fam] = fam_bytes.get(fam, 0) + ex.instr_costs[idx][0]
            fam_flops[fam] = fam_flops.get(fam, 0) + ex.instr_costs[idx][1]
        res["per_kernel_ms"] = {k: round(v, 5) for k, v in sorted(fam_ms.items(),
                                                                 key=lambda kv: -kv[1])}
        res["profiled_step_ms"] = sum(fam_ms.values())
        res["_fam"] = (fam_ms, fam_bytes, fam_flops)

    res["kvstore_round_ms"] = kv_round_ms(step, kv, eng, steps)
    res["kv_bytes_per_step"] = 4 * sum(int(np.prod(shapes[n])) for n in step.names)
    kv.close()
    return res


def kv_launches(kv) -> int:
    """Kernels the store launched for ONE step's round (counted by the store
    around the step's flush)."""
    return kv.launches_per_flush


def kv_round_ms(step, kv, eng, steps):
    """Device time of the step's KVStore part (every key pushed -> fused
    reduce + SGD + broadcast), captured as a CUDA graph like the step itself
    and replayed; max over ranks is taken by the caller's barrier shape."""
    import torch
    w = step.workers[0]

    def one_round():
        for i in range(len(step.names)):
            kv.push(i, step.grads[w][step.names[i]], w)
        with kv._lock:
            kv._flush_locked()

    one_round()
    eng.wait_all()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=eng.stream, capture_error_mode="thread_local"):
        one_round()
    reps = max(3, min(steps, 10))
    with torch.cuda.stream(eng.stream):
        g.replay()
    torch.cuda.synchronize()
    ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ka.record(eng.stream)
    with torch.cuda.stream(eng.stream):
        for _ in range(reps):
            g.replay()
    kb.record(eng.stream)
    torch.cuda.synchronize()
    return ka.elapsed_time(kb) / reps


def roofline_of(res):
    """Roofline object for the dominant kernel family of the step."""
    hbm, bf16, bf16_sus, src = peaks()
    fam_ms, fam_bytes, fam_flops = res["_fam"]
    dom = max(fam_ms, key=fam_ms.get)
    ms = fam_ms[dom]
    tensor = dom.startswith("tc_gemm")
    if tensor:
        achieved = fam_flops[dom] / (ms * 1e-3) / 1e12
        peak, unit = bf16_sus, "TFLOP/s"
        psrc = f"{src} bf16 sustained (kernel timed inside the step)"
    else:
        achieved = fam_bytes[dom] / (ms * 1e-3) / 1e9
        peak, unit = hbm, "GB/s"
        psrc = f"{src} HBM copy"
    traffic, tsrc = None, None
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{res['config_name']}.json")) as f:
            t = json.load(f)
        if t.get("kernel") == dom:
            traffic, tsrc = t["dram_bytes_per_pass"], t["source"]
    except Exception:  # noqa: BLE001 - no committed ncu capture for this config
        pass
    return {"bound": "tensor" if tensor else "hbm", "kernel": dom, "achieved": achieved,
            "peak": peak, "peak_source": psrc, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "DRAM bytes per step (all launches of the family)",
            "traffic_source": tsrc, "kernel_ms_per_step": ms,
            "step_share": ms / sum(fam_ms.values()),
            "algorithmic_per_step": fam_flops[dom] if tensor else fam_bytes[dom],
            "algorithmic_bytes_per_step": fam_bytes[dom]}


def kv_sweep(args, eng, world, rank, distributed):
    import torch
    from paper_1512_01274_b200.kvstore import KVStore
    from paper_1512_01274_b200.optim import SGDConfig, make_sgd_updater
    out = []
    hbm = peaks()[0]
    for nbytes in args.kv_bytes:
        n = nbytes // 4
        kv = KVStore(1, world, engine=eng, distributed=distributed)
        kv.init(0, np.zeros(n, np.float32))
        kv.set_updater(make_sgd_updater(SGDConfig(ETA, MOM, WD), scale=world))
        w = kv.local_workers[0]
        gt, wt = kv.grad_tensor(0, w), kv.weight_tensor(0, w)
        rounds = max(3, min(args.steps, 20)) if n >= (1 << 24) else 50
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
            rec.update({"hbm_GBps": 5 * S / (ms * 1e-3) / 1e9,
                        "hbm_frac": 5 * S / (ms * 1e-3) / 1e9 / hbm})
        out.append(rec)
    return out


def run_ours(args, world, rank, local):
    import torch
    from paper_1512_01274_b200.engine import Engine
    torch.cuda.set_device(local)
    eng = Engine(device=local)
    name = args.config
    head = run_config(name, args, world, rank, local, eng, args.steps, args.warmup)
    roof = roofline_of(head)
    flops_img = train_flops_per_image(name) if name != "mlp" else None
    extra = {}
    if not args.no_extra:
        for other in ("mlp", "lenet", "alexnet", "inception_bn"):
            if other == name:
                continue
            r = run_config(other, args, world, rank, local, eng, max(5, args.steps // 4),
                           3, with_e2e=(other == "mlp"), with_profile=True)
            rr = roofline_of(r)
            extra[other] = {k: v for k, v in r.items() if k not in ("_fam",)}
            extra[other]["roofline"] = {k: rr[k] for k in ("bound", "kernel", "achieved", "unit",
                                                             "frac", "step_share")}
    kvres = kv_sweep(args, eng, world, rank, world > 1)
    cpu = None
    if rank == 0 and world == 1:
        v, nsteps, el, cores, sample = cpu_sample(name, seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample}
    if rank == 0:
        cfg = CONFIGS[name]
        tensor_tflops = (flops_img * head["value"] / world / 1e12) if flops_img else None
        if roof and tensor_tflops and roof.get("bound") == "tensor":
            # the family's rate from isolated per-launch times understates a
            # step whose GEMMs run side by side: also the step-level rate
            roof = dict(roof, step_achieved=tensor_tflops,
                        step_frac=tensor_tflops / roof["peak"])
        line = {
            "metric": METRIC, "value": head["value"], "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"],
            "data": "synthetic (seeded randn images, randint labels; resident batch)",
            "config": {"workload": cfg["workload"], "global_batch": cfg["batch"] * world,
                       "per_gpu_batch": cfg["batch"], "parallelism": f"dp{world}",
                       "l2": "flushed between timed steps (256 MB device write, untimed)",
                       "step": "forward+backward+KVStore round captured as one CUDA graph"},
            "e2e": head.get("e2e"),
            "gpu_launches": head["kernels_per_step"] * args.steps,
            "roofline": roof,
            "step_tensor_tflops_per_gpu": tensor_tflops,
            "per_kernel_ms": head.get("per_kernel_ms"),
            "kvstore_round_ms": head["kvstore_round_ms"],
            "kv_bytes_per_step": head["kv_bytes_per_step"],
            "cpu_baseline": cpu, "kvstore": kvres, "clocks": head["clocks"],
            "configs": extra,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="inception_bn")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary configurations")
    ap.add_argument("--kv-bytes", type=int, nargs="*",
                    default=[1 << e for e in range(10, 31, 2)],
                    help="config-2 KVStore sweep key sizes (default 1 KB ... 1 GB, x4)")
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
