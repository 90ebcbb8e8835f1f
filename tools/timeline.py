"""GPU timeline of the captured Inception-BN forward+backward (CUDA graph,
4 lanes) from CUPTI kernel records (torch.profiler): span, busy time (at
least one kernel running), idle gaps, mean concurrency, and the kernel
families by summed / exclusive time -- what the multi-lane schedule actually
achieves, as opposed to the per-instruction serial profile.

    python tools/timeline.py [config] [--trace out.json]
"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "inception_bn"
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
              use_graph=True)
    for _ in range(5):
        ex.forward()
        ex.backward()
    eng.wait_all()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            ex.forward()
            ex.backward()
        eng.wait_all()
    path = (sys.argv[sys.argv.index("--trace") + 1] if "--trace" in sys.argv
            else os.path.join(tempfile.gettempdir(), "mgx_timeline.json"))
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    # the last of the 3 passes: split on the largest idle gap structure --
    # take kernels after the 2nd-to-last forward start = last third by count
    n = len(ks) // 3
    ks = ks[-n:]
    t0 = ks[0]["ts"]
    span = max(e["ts"] + e["dur"] for e in ks) - t0
    # busy time and concurrency
    pts = []
    for e in ks:
        pts.append((e["ts"], 1))
        pts.append((e["ts"] + e["dur"], -1))
    pts.sort()
    busy, conc_area, cur, last = 0.0, 0.0, 0, pts[0][0]
    gaps = []
    for tt, d in pts:
        if cur > 0:
            busy += tt - last
            conc_area += cur * (tt - last)
        elif tt > last:
            gaps.append(tt - last)
        cur += d
        last = tt
    total = sum(e["dur"] for e in ks)
    print(f"{name}: {len(ks)} kernels in one fwd+bwd, span {span / 1e3:.3f} ms, busy "
          f"{busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms in {len(gaps)} gaps "
          f"(largest {max(gaps, default=0):.1f} us), summed kernel time {total / 1e3:.3f} ms, "
          f"mean concurrency {conc_area / max(busy, 1):.2f}")
    fam = {}
    for e in ks:
        k = e["name"].split("(")[0].split("<")[0].replace("void ", "")
        f = fam.setdefault(k, [0, 0.0])
        f[0] += 1
        f[1] += e["dur"]
    for k, (c, d) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"  {k:45s} n={c:4d} {d / 1e3:8.3f} ms")


if __name__ == "__main__":
    main()
