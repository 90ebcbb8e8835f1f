"""Native memory planner vs the reference's plans (bit-exact), plus the
reference planner suite's properties (tests/test_planner.py there).  CPU."""

import random

import numpy as np
import pytest

from conftest import random_dag
from oracle import plan as oplan
from paper_1512_01274_b200 import symbol
from paper_1512_01274_b200.errors import ArgumentError
from oracle.plan import validate_plan
from paper_1512_01274_b200.planner import STRATEGIES, FlatGraph, plan_memory, prune, py_set_order
from paper_1512_01274_b200.symbol import SymbolGraph
from paper_1512_01274_b200.train import mlp


def as_record(p):
    n = len(p.node_names)
    return {"slot_of": [p.slot_of[i] for i in range(n)],
            "slot_bytes": [p.slot_bytes[s] for s in range(len(p.slot_bytes))],
            "dedicated": sorted(p.dedicated_slots), "edges": [list(e) for e in p.extra_dep_edges],
            "total": p.total_internal_bytes, "visits": p.visits}


def combined(g):
    wrt = [n for n in g.list_arguments() if n not in ("data", "label")]
    ends, _ = symbol.build_gradient(g, wrt)
    comb = SymbolGraph(list(g.outputs) + ends)
    fwd = {id(n) for n in g.topo_nodes()}
    return comb, [0 if (n.is_variable or id(n) in fwd) else 1 for n in comb.topo_nodes()]


def test_mlp_plans_bit_exact(plans_golden):
    for rec in plans_golden["mlp"]:
        symbol.reset_names()
        g = mlp(rec["hidden"], rec["classes"])
        # the graph this package builds is the reference's, node for node
        assert symbol.save(g) == rec["fwd_text"]
        comb, phases = combined(g)
        assert symbol.save(comb) == rec["comb_text"]
        assert phases == rec["phases"]
        b, f = rec["given"]
        given = {"data": (b, f), "label": (b,)}
        for s in STRATEGIES:
            assert as_record(plan_memory(comb, given, s, phases=phases)) == rec["plans"][s], s
            assert as_record(plan_memory(g, given, s)) == rec["fwd_plans"][s], s


def test_random_dag_plans_bit_exact(plans_golden):
    for rec in plans_golden["dags"]:
        g = symbol.load(rec["text"])
        shapes = {k: tuple(v) for k, v in rec["shapes"].items()}
        for s in STRATEGIES:
            assert as_record(plan_memory(g, shapes, s)) == rec["plans"][s], (rec["seed"], s)


def test_random_dag_generator_matches_reference(plans_golden):
    for rec in plans_golden["dags"][:60]:
        symbol.reset_names()
        g, _feed = random_dag(rec["seed"])
        assert symbol.save(g) == rec["text"], rec["seed"]


def test_native_planner_equals_oracle_on_fresh_dags():
    for seed in range(200, 400):
        symbol.reset_names()
        g, feed = random_dag(seed, max_ops=16)
        shapes = {k: v.shape for k, v in feed.items()}
        view = FlatGraph.of(g, shapes, "float32")
        for s in STRATEGIES:
            p = plan_memory(g, shapes, s)
            slot_of, _sb, ded, edges, total = oplan.plan(
                view.is_var, view.nbytes, view.dedicated, view.inputs, view.inplace_positions, s)
            assert [p.slot_of[i] for i in range(view.n)] == [slot_of[i] for i in range(view.n)]
            assert p.extra_dep_edges == edges and p.total_internal_bytes == total


def test_python_set_order_emulation():
    rng = random.Random(3)
    for _ in range(5000):
        keys = [rng.randrange(rng.choice([8, 64, 4096, 1 << 40])) for _ in range(rng.randrange(50))]
        assert py_set_order(keys) == list(set(keys)), keys


def chain(n):
    g = symbol.variable("x")
    for i in range(n):
        g = symbol.apply("ScalarAdd", {"value": float(i)}, [g])
    return g


def test_none_strategy_slots():
    plan = plan_memory(chain(5), {"x": (4,)}, "none")
    internal = [s for s in plan.slot_bytes if s not in plan.dedicated_slots]
    assert len(internal) == 4 and plan.total_internal_bytes == 64


def test_inplace_collapses_chain():
    assert plan_memory(chain(8), {"x": (4,)}, "inplace").total_internal_bytes == 16


def test_unknown_strategy_and_duplicate_names():
    with pytest.raises(ArgumentError):
        plan_memory(chain(2), {"x": (4,)}, "optimal")
    a = symbol.variable("x")
    g1 = symbol.apply("ScalarAdd", {"value": 1.0}, [a], name="n")
    g2 = symbol.apply("ScalarMul", {"value": 2.0}, [a], name="n")
    with pytest.raises(ArgumentError):
        plan_memory(symbol.group(g1, g2), {"x": (2,)}, "none")


def test_validate_random_plans_and_negative_control():
    for seed in range(40):
        symbol.reset_names()
        g, feed = random_dag(seed)
        shapes = {k: v.shape for k, v in feed.items()}
        for s in STRATEGIES:
            assert validate_plan(g, plan_memory(g, shapes, s), shapes) == [], (seed, s)
    a = symbol.variable("x")
    s1 = symbol.apply("ScalarAdd", {"value": 1.0}, [a])
    s2 = symbol.apply("ScalarAdd", {"value": 2.0}, [a])
    merged = symbol.apply("ElementwiseAdd", {}, [s1, s2])
    plan = plan_memory(merged, {"x": (4,)}, "none")
    names = [n.name for n in merged.topo_nodes()]
    plan.slot_of[names.index(s2.outputs[0][0].name)] = plan.slot_of[names.index(s1.outputs[0][0].name)]
    assert validate_plan(merged, plan, {"x": (4,)})


def test_memory_ratios_acceptance():
    # reference acceptance (tests/test_acceptance.py:40-60): fwd+bwd <= 0.5, fwd <= 0.25
    g = mlp([64] * 8, 10)
    given = {"data": (64, 64), "label": (64,)}
    comb, phases = combined(g)
    full = (plan_memory(comb, given, "both", phases=phases).total_internal_bytes /
            plan_memory(comb, given, "none", phases=phases).total_internal_bytes)
    fwd = (plan_memory(g, given, "both").total_internal_bytes /
           plan_memory(g, given, "none").total_internal_bytes)
    assert full <= 0.5 and fwd <= 0.25
    assert abs(full - 0.283) < 0.01 and abs(fwd - 0.133) < 0.01


def test_visits_linear():
    v = []
    for n in (40, 80):
        symbol.reset_names()
        v.append(plan_memory(chain(n), {"x": (4,)}, "both").visits)
    assert v[1] <= 2 * v[0] + 50


def test_prune_structure():
    a = symbol.variable("x")
    keep = symbol.apply("ScalarAdd", {"value": 1.0}, [a])
    drop = symbol.apply("ScalarMul", {"value": 2.0}, [a])
    assert len(prune(symbol.group(keep, drop), [0]).topo_nodes()) == 2
    with pytest.raises(ArgumentError):
        prune(symbol.group(keep, drop), [5])
