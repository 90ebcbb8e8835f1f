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
