"""Summaries of raw ncu CSV logs for profiles/ (and bench.py's roofline
`traffic`):

    python tools/ncu_summarize.py step RAW.csv OUT.csv [config]
        raw = `ncu --profile-from-start off --metrics dram__bytes_read.sum,
        dram__bytes_write.sum,gpu__time_duration.sum --csv` of
        tools/ncu_step.py: per kernel family launches, DRAM GB, ms; also
        writes profiles/traffic_<config>.json for the GEMM family
    python tools/ncu_summarize.py launches RAW.csv OUT.csv
        raw = `ncu --metrics gpu__time_duration.sum --csv` of a bench run:
        per family launches, total us, share
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rows(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    return list(csv.DictReader(lines))


def _family(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").strip()
    base = base.split("<")[0]
    return base.split("::")[-1]


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def step(raw, out, config="inception_bn"):
    per = defaultdict(lambda: {"n": 0, "bytes": 0.0, "ns": 0.0})
    launches = {}
    for r in _rows(raw):
        key = (r["ID"], r["Kernel Name"])
        launches[key] = r["Kernel Name"]
        f = per[_family(r["Kernel Name"])]
        m, v, unit = r["Metric Name"], _num(r["Metric Value"]), r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1,
                 "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        if m.startswith("dram__bytes"):
            f["bytes"] += v * scale
        elif m == "gpu__time_duration.sum":
            f["ns"] += v * scale
            f["n"] += 1
    tot_b = sum(f["bytes"] for f in per.values())
    tot_ms = sum(f["ns"] for f in per.values()) / 1e6
    tot_n = sum(f["n"] for f in per.values())
    with open(out, "w") as fh:
        fh.write("# ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
                 f" over ONE {config} forward+backward\n# (tools/ncu_step.py, --clock-control none;"
                 " serialised cold launches)\n")
        fh.write(f"# total: {tot_n} launches, {tot_ms:.3f} ms, DRAM {tot_b / 1e9:.2f} GB\n")
        fh.write("family,launches,dram_GB,kernel_ms,dram_GBps\n")
        for k, f in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
            ms = f["ns"] / 1e6
            fh.write(f"{k},{f['n']},{f['bytes'] / 1e9:.3f},{ms:.3f},"
                     f"{f['bytes'] / 1e9 / (ms / 1e3) if ms else 0:.0f}\n")
    g = per.get("tc_gemm_bf16_kernel")
    if g:
        rel = os.path.relpath(out, ROOT)
        with open(os.path.join(ROOT, "profiles", f"traffic_{config}.json"), "w") as fh:
            json.dump({"config": config, "kernel": "tc_gemm_bf16 (tcgen05)",
                       "launches_per_pass": g["n"], "dram_bytes_per_pass": g["bytes"],
                       "kernel_ms_ncu": g["ns"] / 1e6,
                       "source": f"{rel} (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                                 "over one fwd+bwd pass)"}, fh, indent=1)


def launches(raw, out):
    per = defaultdict(lambda: [0, 0.0])
    for r in _rows(raw):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "nsecond")
        us = _num(r["Metric Value"]) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(unit, 1e-3)
        f = per[_family(r["Kernel Name"])]
        f[0] += 1
        f[1] += us
    tot = sum(v[1] for v in per.values())
    with open(out, "w") as fh:
        fh.write("# ncu launch list of `python bench.py --no-extra --steps 2 --warmup 3 --kv-bytes 1048576` (tools/ncu_round.sh) "
                 "(Inception-BN, 1 B200)\n# gpu__time_duration.sum, --clock-control none; "
                 "cold-cache serialised launches: compare shares\n")
        fh.write(f"# total kernel time {tot / 1e3:.3f} ms over {sum(v[0] for v in per.values())}"
                 " launches\nfamily,launches,total_us,share\n")
        for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k},{n},{us:.1f},{us / tot:.4f}\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "step":
        step(sys.argv[2], sys.argv[3], *(sys.argv[4:5]))
    else:
        launches(sys.argv[2], sys.argv[3])
