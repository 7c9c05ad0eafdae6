"""CPU tests: the C-ABI library loads and exports every declared symbol,
the native planner matches the reference schedules, generators match the
SURVEY fingerprints."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, case_pairs, load_golden, unpack

import oracle
from paper_1903_12359_b200 import generators as gen

HEADER = os.path.join(ROOT, "include", "pgcp_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PGCP_API\s+(?:int|const char\*)\s+(pgcp_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1903_12359_b200 import _native, build
    build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.pgcp_abi_version() == 2


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1903_12359_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def _part(case):
    z = load_golden(case)

    class P:
        pass
    p = P()
    p.boundary_cycles = unpack(z, "cycles")
    p.cuts = np.sort(z["cuts"], axis=1) if len(z["cuts"]) else np.zeros((0, 2), np.int64)
    return z, p


@pytest.mark.parametrize("case", ["cfg1", "strips4", "blocks3x3", "disk2x2", "flat2x2",
                                  "sphere2", "sphere4", "tree4x4", "ptree4x4", "qtree4x4"])
def test_native_planner_matches_reference(case):
    from paper_1903_12359_b200.partition import plan_weld_schedule
    z, p = _part(case)
    pairs = case_pairs(case)
    steps = plan_weld_schedule(p, str(z["mode"]), pairs=pairs)
    A, B, M = unpack(z, "step_a"), unpack(z, "step_b"), unpack(z, "step_merged")
    assert len(steps) == len(A)
    for s, a, b, m, meta in zip(steps, A, B, M, z["step_meta"]):
        assert np.array_equal(s.a_cycle, a) and np.array_equal(s.b_cycle, b)
        assert np.array_equal(s.merged_cycle, m)
        assert [s.comp_a, s.comp_b, s.k, int(s.closed)] == list(meta)


@pytest.mark.parametrize("n,k", [(65, 8), (129, 16)])
def test_native_planner_matches_oracle_large(n, k):
    from paper_1903_12359_b200.partition import plan_weld_schedule
    V, F, c = gen.height_field_case(n, k)
    sp = oracle.split_mesh(V, F, c)

    class P:
        pass
    p = P()
    p.boundary_cycles, p.cuts = sp.boundary_cycles, sp.cuts
    steps = plan_weld_schedule(p)
    ref = oracle.greedy_schedule(sp.boundary_cycles, sp.cuts)
    assert len(steps) == len(ref) == k * k - 1
    for s, o in zip(steps, ref):
        assert (s.comp_a, s.comp_b, s.k) == (o.comp_a, o.comp_b, o.k)
        assert np.array_equal(s.a_cycle, o.a_cycle) and np.array_equal(s.b_cycle, o.b_cycle)


def test_planner_rejects_corner_only_contact():
    from paper_1903_12359_b200.errors import PartitionError
    from paper_1903_12359_b200.partition import plan_weld_schedule

    class P:
        pass
    p = P()
    p.boundary_cycles = [np.array([0, 1, 2]), np.array([2, 3, 4])]
    p.cuts = np.zeros((0, 2), np.int64)
    with pytest.raises(PartitionError):
        plan_weld_schedule(p)


def test_generator_fingerprints():
    V, F, cuts = gen.cfg1(0)
    h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    assert h(V) == "c09f242d3e13faad"
    assert h(F) == "38e046bed638756d"
    assert len(cuts) == 198 and h(cuts) == "86338b0a7b75d7bb"
    assert V[:, 2].min() == -0.18727264361230875


def test_row_tree_order_covers_blocks():
    order = gen.row_tree_schedule_order(8, 8)
    assert len(order) == 63
    assert order[:2] == [(0, 1), (0, 2)] and order[-1] == (0, 32)


def test_cfg3_cfg4_generators_shape():
    """The irregular BASELINE meshes at test size: a disk whose boundary is
    the 256-gon on the unit circle (cfg 3), a closed genus-0 surface (cfg 4);
    both split into disk-type components by their k-means cuts."""
    V, F, cuts = gen.cfg3(seed=0, n_points=20000, n_clusters=16)
    chi, nl, cls = oracle.topology_class(len(V), F.astype(np.int64))
    assert cls == "disk_type"
    loop = oracle.boundary_loop_list(F.astype(np.int64))[0]
    assert len(loop) == 256 and np.allclose(np.hypot(V[loop, 0], V[loop, 1]), 1.0)
    sp = oracle.split_mesh(V, F, cuts)
    assert sp.n_sub == 16
    V, F, cuts = gen.cfg4(seed=0, subdiv=4, n_clusters=8)
    chi, nl, cls = oracle.topology_class(len(V), F.astype(np.int64))
    assert cls == "sphere_type"
    r = np.linalg.norm(V, axis=1)
    assert 0.69 <= r.min() and r.max() <= 1.31
    assert oracle.split_mesh(V, F, cuts).n_sub == 8


def test_cyclic_runs_matches_oracle():
    """partition._cyclic_runs (vectorised) equals the oracle's run finder
    (oracle/planner.py, pinned to partition.py:149-179) on the goldens'
    boundary-cycle pairs and on random cycles."""
    import oracle.planner as op
    from paper_1903_12359_b200.partition import _cyclic_runs
    pairs = []
    for case in ("cfg1", "blocks3x3", "strips4", "sphere4", "qtree4x4"):
        cyc = unpack(load_golden(case), "cycles")
        pairs += [(cyc[i], cyc[j]) for i in range(len(cyc)) for j in range(len(cyc)) if i != j]
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(3, 40))
        c1 = rng.permutation(60)[:n]
        c2 = list(rng.permutation(60)[:int(rng.integers(3, 40))])
        if rng.random() < 0.7:  # splice a reversed arc of c1 into c2
            s, ln = int(rng.integers(0, n)), int(rng.integers(2, n + 1))
            arc = [int(c1[(s + t) % n]) for t in range(ln)][::-1]
            c2 = arc + [v for v in c2 if v not in arc]
        pairs.append((c1, np.array(c2)))
    pairs.append((np.arange(6), np.arange(6)[::-1].copy()))
    for a, b in pairs:
        assert _cyclic_runs(a, b) == op.cyclic_runs(list(map(int, a)), list(map(int, b)))


def test_cut_file_round_trip(tmp_path):
    from paper_1903_12359_b200 import PartitionError
    from paper_1903_12359_b200.partition import read_cut_edges, write_cut_edges
    cuts = np.array([[0, 5], [3, 9], [12, 2]])
    p = tmp_path / "c.cuts"
    write_cut_edges(p, cuts)
    assert np.array_equal(read_cut_edges(p), cuts)
    p.write_text("# header\n1 2\n\n3 4\n")
    assert np.array_equal(read_cut_edges(p), [[0, 1], [2, 3]])
    p.write_text("1 2\n0 4\n")
    with pytest.raises(PartitionError, match=":2: vertex ids are 1-based"):
        read_cut_edges(p)
    p.write_text("1 2 3\n")
    with pytest.raises(PartitionError, match="expected two vertex ids"):
        read_cut_edges(p)


def test_validate_cuts_normalises_and_rejects_duplicates():
    """partition.py:48-59: every pair sorted, order kept, duplicates (in either
    orientation) rejected with the reference's message; empty input allowed."""
    from paper_1903_12359_b200.errors import PartitionError
    from paper_1903_12359_b200.partition import validate_cuts
    rng = np.random.default_rng(3)
    a = rng.permutation(5000)[:2000].reshape(-1, 2).astype(np.int64)
    norm = validate_cuts(None, a)
    assert np.array_equal(norm, np.sort(a, axis=1))
    assert norm.dtype == np.int64 and norm.flags.c_contiguous
    assert validate_cuts(None, np.zeros((0, 2), np.int64)).shape == (0, 2)
    assert np.array_equal(validate_cuts(None, [[7, 3]]), [[3, 7]])
    dup = np.vstack([a, a[17][::-1]])
    with pytest.raises(PartitionError, match="duplicate cut edges"):
        validate_cuts(None, dup)
