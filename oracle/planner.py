"""Oracle: shared-arc detection and weld-schedule planning (restates
`partition.py:149-324`). TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

`greedy_schedule` is the reference planner (longest arc first, ties on
(ca, cb, chain[0]), `partition.py:254-266`). `pair_schedule` builds the same
WeldStep records for an explicit merge order (used for the documented
"rows -> strips, then pairwise tree" deviation on 8x8 blocks).
"""

from dataclasses import dataclass

import numpy as np

from .surface import OraclePartitionError


@dataclass
class Step:
    comp_a: int
    comp_b: int
    a_cycle: np.ndarray
    b_cycle: np.ndarray
    k: int
    closed: bool
    merged_cycle: np.ndarray


def cyclic_runs(c1, c2):
    """Maximal runs of consecutive c1 vertices that are consecutive and
    reversed in c2 (`partition.py:149-179`). Returns a list of int lists,
    or "full" when the whole cycle matches."""
    c1 = np.asarray(c1, dtype=np.int64)
    c2 = np.asarray(c2, dtype=np.int64)
    n1, n2 = len(c1), len(c2)
    order = np.argsort(c2)
    srt = c2[order]
    loc = np.searchsorted(srt, c1)
    loc = np.minimum(loc, max(n2 - 1, 0))
    present = (n2 > 0) & (srt[loc] == c1) if n2 else np.zeros(n1, bool)
    pos = np.where(present, order[loc], -1)
    pos_next = np.roll(pos, -1)
    ok = present & np.roll(present, -1) & ((pos_next + 1) % max(n2, 1) == pos)
    if ok.all():
        if n1 != n2:
            raise OraclePartitionError("inconsistent full-cycle correspondence")
        return "full"
    if not ok.any():
        return []
    runs = []
    first_bad = int(np.flatnonzero(~ok)[0])
    for step in range(1, n1 + 1):
        i = (first_bad + step) % n1
        if ok[i] and not ok[i - 1]:
            j = i
            chain = [int(c1[j])]
            while ok[j % n1]:
                chain.append(int(c1[(j + 1) % n1]))
                j += 1
            runs.append(chain)
    return runs


def _rotate(cycle, v):
    cyc = [int(x) for x in cycle]
    at = cyc.index(int(v))
    return cyc[at:] + cyc[:at]


def _glue(cycles, ca, cb, chain):
    """One WeldStep gluing `chain` between components ca < cb
    (`partition.py:271-289`)."""
    left = (set(cycles[ca]) & set(cycles[cb])) - set(chain)
    if left:
        raise OraclePartitionError(
            f"components {ca} and {cb} share vertices beyond one contiguous arc; "
            "this cut layout needs multi-arc gluing, which is unsupported")
    a_cyc = _rotate(cycles[ca], chain[0])
    b_cyc = _rotate(list(reversed(cycles[cb])), chain[0])
    k = len(chain) - 1
    if a_cyc[:k + 1] != chain or b_cyc[:k + 1] != chain:
        raise OraclePartitionError("arc is not a prefix of both component cycles")
    merged = [chain[-1]] + a_cyc[k + 1:] + [chain[0]] + list(reversed(b_cyc[k + 1:]))
    step = Step(ca, cb, np.array(a_cyc), np.array(b_cyc), k, False, np.array(merged))
    del cycles[cb]
    cycles[ca] = merged
    return step


def _sphere_close(cycles, steps):
    ca, cb = sorted(cycles)
    c1, c2 = cycles[ca], cycles[cb]
    if set(c1) != set(c2) or len(c1) != len(c2):
        raise OraclePartitionError("final two components do not share their full boundary")
    if cyclic_runs(c1, c2) != "full":
        raise OraclePartitionError("final boundaries are not a reversed cyclic match")
    s = min(c1)
    a_cyc = _rotate(c1, s)
    b_cyc = _rotate(list(reversed(c2)), s)
    steps.append(Step(ca, cb, np.array(a_cyc), np.array(b_cyc), len(a_cyc) - 1, True,
                      np.array([], dtype=np.int64)))


def _check_cover(steps, cuts):
    """Every cut edge glued exactly once (`partition.py:307-323`)."""
    glued = set()
    for st in steps:
        arc = [int(x) for x in st.a_cycle[:st.k + 1]]
        pairs = list(zip(arc[:-1], arc[1:]))
        if st.closed:
            pairs.append((arc[-1], arc[0]))
        for u, v in pairs:
            e = (min(u, v), max(u, v))
            if e in glued:
                raise OraclePartitionError(f"edge {e} glued twice in the schedule")
            glued.add(e)
    want = {(int(a), int(b)) for a, b in np.asarray(cuts).reshape(-1, 2)}
    if glued != want:
        raise OraclePartitionError(
            f"schedule does not cover all cut edges ({len(want - glued)} missing)")


def greedy_schedule(boundary_cycles, cuts, mode="free"):
    """Reference planner `plan_weld_schedule` (`partition.py:236-324`)."""
    K = len(boundary_cycles)
    if mode == "sphere" and K < 2:
        raise OraclePartitionError("sphere mode needs at least 2 submeshes")
    target = 2 if mode == "sphere" else 1
    cycles = {i: [int(x) for x in boundary_cycles[i]] for i in range(K)}
    steps = []
    while len(cycles) > target:
        # only component pairs sharing a vertex can have a run
        owner = {}
        for c, cyc in cycles.items():
            for v in cyc:
                owner.setdefault(v, set()).add(c)
        pairs = set()
        for cs in owner.values():
            if len(cs) > 1:
                cs = sorted(cs)
                for x in range(len(cs)):
                    for y in range(x + 1, len(cs)):
                        pairs.add((cs[x], cs[y]))
        best = None
        for ca, cb in sorted(pairs):
            runs = cyclic_runs(cycles[ca], cycles[cb])
            if runs == "full":
                continue
            for chain in runs:
                key = (-len(chain), ca, cb, chain[0])
                if best is None or key < best[0]:
                    best = (key, ca, cb, chain)
        if best is None:
            raise OraclePartitionError(
                "no contiguous shared arc between any two components; "
                "multi-arc gluing in one step is unsupported")
        steps.append(_glue(cycles, best[1], best[2], best[3]))
    if mode == "sphere":
        _sphere_close(cycles, steps)
    _check_cover(steps, cuts)
    return steps


def pair_schedule(boundary_cycles, cuts, pairs, mode="free"):
    """WeldSteps for an explicit (rep_a, rep_b) merge order. The glued arc of
    each pair is its longest shared run (ties on chain[0])."""
    K = len(boundary_cycles)
    cycles = {i: [int(x) for x in boundary_cycles[i]] for i in range(K)}
    steps = []
    for ca, cb in pairs:
        ca, cb = (ca, cb) if ca < cb else (cb, ca)
        if ca not in cycles or cb not in cycles:
            raise OraclePartitionError(f"pair ({ca}, {cb}) is not two live components")
        runs = cyclic_runs(cycles[ca], cycles[cb])
        if runs == "full" or not runs:
            raise OraclePartitionError(f"components {ca} and {cb} share no open arc")
        chain = min(runs, key=lambda ch: (-len(ch), ch[0]))
        steps.append(_glue(cycles, ca, cb, chain))
    target = 2 if mode == "sphere" else 1
    if len(cycles) != target:
        raise OraclePartitionError("merge order leaves more than the target components")
    if mode == "sphere":
        _sphere_close(cycles, steps)
    _check_cover(steps, cuts)
    return steps
