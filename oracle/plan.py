"""TEST INFRASTRUCTURE ONLY.  The static memory planner, restated.

Restates planner.py:221-348 (_plan_view with its co-share order) over the
flat index view of a graph.  Inputs per topo node: is_var, nbytes,
dedicated, inputs (with repeats), in-place candidate positions, phase.
Output: (slot_of, slot_bytes, dedicated_slots, sorted extra edges, internal
bytes).  Freed inputs go back to the pools in CPython ``set`` iteration
order, exactly as the reference's ``for u in set(inputs)`` (planner.py:298).
"""

from __future__ import annotations

import heapq
from typing import Dict, List, Sequence, Tuple


def _coshare_order(n, is_var, inputs, consumers, phase) -> List[int]:
    """planner.py:317-348: ready nodes by (phase, depth to sink, index)."""
    ops_ = [i for i in range(n) if not is_var[i]]
    isop = set(ops_)
    depth = {i: 1 for i in ops_}
    for i in reversed(ops_):
        for c in consumers[i]:
            if c in isop and phase[c] == phase[i]:
                depth[i] = max(depth[i], depth[c] + 1)
    pending = {i: sum(1 for u in inputs[i] if u in isop) for i in ops_}
    ready = [(phase[i], depth[i], i) for i in ops_ if pending[i] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        cur = heapq.heappop(ready)[2]
        order.append(cur)
        for c in consumers[cur]:
            if c in isop:
                pending[c] -= 1
                if pending[c] == 0:
                    heapq.heappush(ready, (phase[c], depth[c], c))
    return order


def plan(is_var: Sequence[bool], nbytes: Sequence[int], dedicated: Sequence[bool],
         inputs: Sequence[Sequence[int]], inplace_positions: Sequence[Sequence[int]],
         strategy: str, phase: Sequence[int] = None):
    n = len(is_var)
    phase = list(phase) if phase is not None else [0] * n
    consumers: List[List[int]] = [[] for _ in range(n)]
    for i in range(n):
        for u in inputs[i]:
            consumers[u].append(i)
    if strategy in ("coshare", "both"):
        order = _coshare_order(n, is_var, inputs, consumers, phase)
    else:
        order = sorted((i for i in range(n) if not is_var[i]), key=lambda i: (phase[i], i))
    claims = strategy in ("inplace", "both")
    pooled = strategy != "none"

    slot_of: Dict[int, int] = {}
    slot_bytes: Dict[int, int] = {}
    ded_slots = set()

    def new_slot(i, ded):
        s = len(slot_bytes)
        slot_of[i] = s
        slot_bytes[s] = nbytes[i]
        if ded:
            ded_slots.add(s)

    for i in range(n):
        if is_var[i]:
            new_slot(i, True)
    remaining = [len(consumers[i]) for i in range(n)]
    free: Dict[int, List[Tuple[int, int]]] = {}
    moved = set()
    edges = set()
    for v in order:
        ins = list(inputs[v])
        if dedicated[v]:
            new_slot(v, True)
        else:
            done = False
            if claims:
                for pos in inplace_positions[v]:
                    u = ins[pos]
                    if (not dedicated[u] and not is_var[u] and remaining[u] == 1
                            and ins.count(u) == 1 and nbytes[u] == nbytes[v]):
                        slot_of[v] = slot_of[u]
                        moved.add(u)
                        edges.update((c, v) for c in consumers[u] if c != v and c not in ins)
                        done = True
                        break
            if not done and pooled and free.get(nbytes[v]):
                s, owner = free[nbytes[v]].pop()
                slot_of[v] = s
                if consumers[owner]:
                    edges.update((c, v) for c in set(consumers[owner]) if c != v and c not in ins)
                elif owner not in ins:
                    edges.add((owner, v))
                done = True
            if not done:
                new_slot(v, False)
        for u in set(ins):                     # CPython set order matters here
            if dedicated[u]:
                continue
            remaining[u] -= ins.count(u)
            if remaining[u] == 0 and u not in moved:
                free.setdefault(nbytes[u], []).append((slot_of[u], u))
    total = sum(b for s, b in slot_bytes.items() if s not in ded_slots)
    return slot_of, slot_bytes, ded_slots, sorted(edges), total


# ------------------------------------------------------------ plan checker
#
# Restates the reference's plan replay checker (planner.py:378-474): a plan
# is valid if, for every topological order of the operator nodes under the
# graph edges plus the plan's extra edges, no internal slot is overwritten
# while the value in it still has consumers to run.  Small graphs are checked
# over all orders (capped), larger ones over random orders.

def _op_successors(fg, extra_edges):
    ops_ = [i for i in range(fg.n) if not fg.is_var[i]]
    is_op = set(ops_)
    succ = {i: [] for i in ops_}
    indeg = {i: 0 for i in ops_}
    edges = [(u, v) for v in ops_ for u in fg.inputs[v] if u in is_op]
    edges += [(a, b) for a, b in extra_edges if a in is_op and b in is_op]
    for a, b in edges:
        succ[a].append(b)
        indeg[b] += 1
    return ops_, succ, indeg


def _kahn_ok(ops_, succ, indeg) -> bool:
    left = dict(indeg)
    ready = [i for i in ops_ if left[i] == 0]
    count = 0
    while ready:
        x = ready.pop()
        count += 1
        for y in succ[x]:
            left[y] -= 1
            if left[y] == 0:
                ready.append(y)
    return count == len(ops_)


def _all_orders(ops_, succ, indeg, cap):
    """Every topological order (lexicographic over ready sets), at most cap."""
    left = dict(indeg)
    order: List[int] = []
    produced = [0]

    def rec(ready):
        if produced[0] >= cap:
            return
        if len(order) == len(ops_):
            produced[0] += 1
            yield list(order)
            return
        for r in sorted(ready):
            freed = []
            for c in succ[r]:
                left[c] -= 1
                if left[c] == 0:
                    freed.append(c)
            order.append(r)
            yield from rec([x for x in ready if x != r] + freed)
            order.pop()
            for c in succ[r]:
                left[c] += 1

    yield from rec([i for i in ops_ if left[i] == 0])


def _random_orders(ops_, succ, indeg, samples, seed):
    import random
    rng = random.Random(seed)
    for _ in range(samples):
        left = dict(indeg)
        ready = [i for i in ops_ if left[i] == 0]
        order = []
        while ready:
            x = ready.pop(rng.randrange(len(ready)))
            order.append(x)
            for y in succ[x]:
                left[y] -= 1
                if left[y] == 0:
                    ready.append(y)
        yield order


def _replay(fg, slot_of, order):
    owner: Dict[int, List[int]] = {}   # slot -> [node holding it, consumers left]
    for v in order:
        for u in fg.inputs[v]:
            if fg.dedicated[u]:
                continue
            held = owner.get(slot_of[u])
            if held is None or held[0] != u:
                who = fg.names[held[0]] if held else "<gone>"
                return (f"value of {fg.names[u]} overwritten by {who} before its consumer "
                        f"{fg.names[v]} ran")
            held[1] -= 1
        if fg.dedicated[v]:
            continue
        held = owner.get(slot_of[v])
        if held is not None and held[0] != v and held[1] > 0:
            return f"slot collision: {fg.names[v]} overwrites live value of {fg.names[held[0]]}"
        owner[slot_of[v]] = [v, len(fg.consumers[v])]
    return None


def validate_plan(g, plan, given_shapes, etype="float32", outputs=None, exhaustive_nodes=10,
                  samples=10000, order_cap=300000, seed=0) -> List[str]:
    """[] when ``plan`` is safe for every admissible execution order, else
    the first violation found."""
    from paper_1512_01274_b200.planner import FlatGraph
    fg = FlatGraph.of(g, given_shapes, etype, outputs)
    ops_, succ, indeg = _op_successors(fg, plan.extra_dep_edges)
    if not _kahn_ok(ops_, succ, indeg):
        return ["cycle in graph plus extra_dep_edges"]
    sources = []
    if len(ops_) <= exhaustive_nodes:
        sources.append(_all_orders(ops_, succ, indeg, order_cap))
    sources.append(_random_orders(ops_, succ, indeg, samples, seed))
    for i, orders in enumerate(sources):
        seen = 0
        for order in orders:
            seen += 1
            msg = _replay(fg, plan.slot_of, order)
            if msg:
                return [msg]
        if i == 0 and seen < order_cap:
            return []  # every order enumerated
    return []
