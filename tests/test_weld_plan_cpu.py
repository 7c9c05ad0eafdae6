"""The native weld plan (planner.cpp pgcp_weld_plan) against a plain numpy
statement of the same bookkeeping (the per-component dicts of the
reference's weld loop, pipeline.py:172-213, flattened to boundary slots)."""

import numpy as np
import pytest

from conftest import case_pairs, load_golden, unpack

from paper_1903_12359_b200 import generators as gen

CYC_A, CYC_B, SIDE_B = 1 << 25, 1 << 26, 1 << 31


def _numpy_plan(cycles, steps, n_parent):
    K = len(cycles)
    nb = np.array([len(c) for c in cycles], dtype=np.int64)
    loop_off = np.zeros(K + 1, dtype=np.int64)
    loop_off[1:] = np.cumsum(nb)
    slot_parent = np.concatenate(cycles).astype(np.int64)
    members = {i: [i] for i in range(K)}
    table = np.full(n_parent, -1, dtype=np.int64)
    arcpos = np.zeros(n_parent, dtype=np.int64)
    cyc = np.zeros(n_parent, dtype=np.int64)
    info, src, wb, wb_off, ext = [], [], [], [0], None
    for st in steps:
        A, B = members[st.comp_a], members[st.comp_b]
        sa = np.concatenate([np.arange(loop_off[i], loop_off[i + 1]) for i in A])
        sb = np.concatenate([np.arange(loop_off[i], loop_off[i + 1]) for i in B])
        for s in sa:  # last slot of a parent wins
            table[slot_parent[s]] = s
        a_src = table[st.a_cycle]
        table[slot_parent[sa]] = -1
        for s in sb:
            table[slot_parent[s]] = s
        b_src = table[st.b_cycle]
        table[slot_parent[sb]] = -1
        k = int(st.k)
        arcpos[st.a_cycle[:k + 1]] = np.arange(1, k + 2)
        cyc[st.a_cycle] |= CYC_A
        cyc[st.b_cycle] |= CYC_B
        pa, pb = slot_parent[sa], slot_parent[sb]
        ca = arcpos[pa] | cyc[pa]
        cb = (arcpos[pb] | cyc[pb]) | SIDE_B
        arcpos[st.a_cycle[:k + 1]] = 0
        cyc[st.a_cycle] = 0
        cyc[st.b_cycle] = 0
        wb.append(np.stack([sa, ca], 1))
        wb.append(np.stack([sb, cb], 1))
        wb_off.append(wb_off[-1] + len(sa) + len(sb))
        src += [a_src, b_src]
        info.append([k, int(st.closed), len(st.a_cycle), len(st.b_cycle), st.comp_a, st.comp_b])
        if st.closed:
            ext = (sorted(A), sorted(B))
        members[st.comp_a] = A + B
        del members[st.comp_b]
    wbv = (np.concatenate(wb).astype(np.int64) & 0xffffffff).astype(np.uint32).view(np.int32).reshape(-1, 2)
    return (np.array(info, dtype=np.int32), np.concatenate(src).astype(np.int32), np.array(wb_off), wbv, ext)


class _P:
    pass


@pytest.mark.parametrize("case", ["cfg1", "strips4", "blocks3x3", "disk2x2", "flat2x2", "sphere2", "sphere4",
                                  "tree4x4", "ptree4x4", "qtree4x4"])
def test_native_weld_plan_matches_numpy(case):
    from paper_1903_12359_b200.partition import plan_weld_schedule
    from paper_1903_12359_b200.pipeline import WeldPlan
    z = load_golden(case)
    p = _P()
    p.boundary_cycles = unpack(z, "cycles")
    p.cuts = np.sort(z["cuts"], axis=1) if len(z["cuts"]) else np.zeros((0, 2), np.int64)
    pairs = case_pairs(case)
    steps = plan_weld_schedule(p, str(z["mode"]), pairs=pairs)
    n_parent = len(z["V"])
    plan = WeldPlan(p.boundary_cycles, steps, n_parent)
    info, src, wb_off, wb, ext = _numpy_plan(p.boundary_cycles, steps, n_parent)
    assert np.array_equal(plan.info, info)
    assert np.array_equal(plan.src, src)
    assert np.array_equal(plan.wb_off, wb_off)
    assert np.array_equal(plan.wb, wb)
    if ext is not None:
        assert tuple(sorted(x) for x in plan.exterior_candidates) == ext
