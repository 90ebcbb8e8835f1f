"""Diagnostic: device vs oracle at the bench configuration, next to the
oracle's own sensitivity (oracle vs oracle on inputs perturbed by one fp32
ulp), per tensor.  Prints one line per tensor: max |d| / max|ref|."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import convnet as oc  # noqa: E402
from paper_1512_01274_b200 import nets, symbol  # noqa: E402
from paper_1512_01274_b200.engine import Engine  # noqa: E402
from paper_1512_01274_b200.train import init_aux, init_params, param_names  # noqa: E402
import test_bench_config_gpu as tb  # noqa: E402

eng = Engine(device=0)
_g, shapes, p0, kv, step = tb._make_step(eng)
step.step()
kv.round_barrier()
got = tb._state(step, eng)
symbol.reset_names()
g = nets.inception_bn(1000)
x, y = tb._synthetic()
vals = {"data": x, "label": y, **init_params(g, shapes, 0), **init_aux(g, shapes)}
names = param_names(g)
o1, g1, a1 = oc.run_graph(g, vals, wrt=names, bf16_operands=True, bf16_fc=True)
xp = np.nextafter(x, np.float32(np.inf))
o2, g2, a2 = oc.run_graph(g, {**vals, "data": xp}, wrt=names, bf16_operands=True, bf16_fc=True)


def rel(a, b):
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-30))


rows = [("softmax", rel(got["__softmax"], o1["softmax"]), rel(o2["softmax"], o1["softmax"]))]
for n in names:
    rows.append((n, rel(got["d_" + n], g1[n]), rel(g2[n], g1[n])))
for n in step.aux:
    rows.append((n, rel(got[n], a1[n]), rel(a2[n], a1[n])))
worst = 0
for n, dev, floor in rows:
    print(f"{n:40s} device {dev:.3e}  oracle-floor {floor:.3e}  ratio {dev / max(floor, 1e-30):.2f}")
    worst = max(worst, dev)
print("worst device", worst, "worst floor", max(r[2] for r in rows))
