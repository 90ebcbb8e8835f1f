"""Per-instruction device profile of one training pass of a configuration:
label, kernel family, shape, ms, achieved TFLOP/s or GB/s (diagnostics).

    python tools/profile_net.py [inception_bn|alexnet|lenet|mlp] [--top N]
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "inception_bn"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 60
    import torch
    from paper_1512_01274_b200 import symbol
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.executor import bind
    from paper_1512_01274_b200.train import aux_names, init_aux, init_params, param_names
    cfg = bench.CONFIGS[name]
    eng = Engine(device=0)
    g = bench.build_graph(name)
    b = cfg["batch"]
    given = {"data": (b,) + cfg["image"], "label": (b,)}
    shapes, _ = symbol.infer_shape(g, given)
    x, y = bench.synthetic(name, b, 0)
    p0, a0 = init_params(g, shapes, 0), init_aux(g, shapes)
    names = param_names(g)
    args = {"data": tmod.from_host(given["data"], "float32", x, engine=eng),
            "label": tmod.from_host((b,), "float32", y, engine=eng)}
    for n in names:
        args[n] = tmod.from_host(shapes[n], "float32", p0[n], engine=eng)
    for n in aux_names(g):
        args[n] = tmod.from_host(shapes[n], "float32", a0[n], engine=eng)
    grads = {n: tmod.zeros(shapes[n], engine=eng) for n in names}
    ex = bind(g, args, {n: "write" for n in names}, grads, engine=eng, dense=cfg["dense"],
              strategy=cfg.get("strategy", "both"), split_target=cfg.get("split_target", 0))
    for _ in range(3):
        ex.forward()
        ex.backward()
    eng.wait_all()
    reps = 5
    t = np.zeros(ex.num_instructions)
    for _ in range(reps):
        t += np.array([ms for _l, ms in ex.profile()]) / reps
    rows = []
    for i, ms in enumerate(t):
        op = ex.instr_ops[i]
        byt, fl = ex.instr_costs[i]
        fam = bench.kernel_family(op)
        rate = (f"{fl / ms / 1e9:8.1f} TF/s" if fam.startswith("tc_gemm")
                else f"{byt / ms / 1e6:8.1f} GB/s")
        d = list(ex._prog_dims[i]) if hasattr(ex, "_prog_dims") else []
        d = d + ["ptrs:" + "".join("1" if p else "0" for p in ex._prog_ptrs[i])]
        rows.append((ms, i, ex.instr_labels[i], fam, rate, d))
    total = t.sum()
    # critical path of the multi-lane schedule with these durations (each
    # lane in order, cross-lane event waits; forward and backward joined)
    if getattr(ex, "schedule", None) is not None:
        lane, ptr, idx = ex.schedule
        for over in (0.0, 0.002):
            fin = [0.0] * len(t)
            lane_end, start, cp_total, lane_busy = {}, 0.0, 0.0, {}
            for i in range(len(t)):
                if i == ex._n_fwd:  # join before the backward range
                    start = max(fin[:i]) if i else 0.0
                    lane_end = {}
                d = max(t[i] - over, 0.0005)
                s0 = max([lane_end.get(lane[i], start)] + [fin[j] for j in idx[ptr[i]:ptr[i + 1]]])
                fin[i] = s0 + d
                lane_end[lane[i]] = fin[i]
                lane_busy[lane[i]] = lane_busy.get(lane[i], 0.0) + d
            print(f"modeled multi-lane pass (per-instruction overhead {over * 1e3:.0f} us "
                  f"removed): {max(fin):.3f} ms; lane busy ms: "
                  + ", ".join(f"{k}:{v:.2f}" for k, v in sorted(lane_busy.items())))
        # critical path backtrace (overhead-removed durations)
        fin = [0.0] * len(t)
        pred = [-1] * len(t)
        lane_last, start_i = {}, -1
        for i in range(len(t)):
            if i == ex._n_fwd:
                start_i = max(range(i), key=lambda q: fin[q]) if i else -1
                lane_last = {}
            d = max(t[i] - 0.002, 0.0005)
            cands = [lane_last.get(lane[i], start_i)] + list(idx[ptr[i]:ptr[i + 1]])
            best = max(cands, key=lambda q: fin[q] if q >= 0 else 0.0)
            fin[i] = (fin[best] if best >= 0 else 0.0) + d
            pred[i] = best
            lane_last[lane[i]] = i
        cur = max(range(len(t)), key=lambda q: fin[q])
        path = []
        while cur >= 0:
            path.append(cur)
            cur = pred[cur]
        fams_cp = {}
        for i in path:
            f = bench.kernel_family(ex.instr_ops[i])
            fams_cp[f] = fams_cp.get(f, 0.0) + max(t[i] - 0.002, 0.0005)
        print(f"critical path: {len(path)} instructions, "
              + ", ".join(f"{k} {v:.3f}" for k, v in sorted(fams_cp.items(), key=lambda kv: -kv[1])))
        if "--path" in sys.argv:
            for i in reversed(path):
                print(f"  cp #{i:4d} lane {lane[i]} {t[i] * 1e3:7.1f} us  "
                      f"{bench.kernel_family(ex.instr_ops[i]):22s} {ex.instr_labels[i]}")
    print(f"{name}: {ex.num_instructions} instructions, {total:.3f} ms profiled pass, "
          f"kernels {ex.kernel_count()}, lanes {ex.lanes_used}")
    fams = {}
    for ms, i, lbl, fam, rate, d in rows:
        fams[fam] = fams.get(fam, 0) + ms
    for fam, ms in sorted(fams.items(), key=lambda kv: -kv[1]):
        print(f"  {fam:28s} {ms:8.3f} ms {100 * ms / total:5.1f}%")
    for ms, i, lbl, fam, rate, d in sorted(rows, reverse=True)[:top]:
        print(f"{ms:8.4f} ms  #{i:4d} {fam:24s} {rate}  {lbl}  {d}")


if __name__ == "__main__":
    main()
