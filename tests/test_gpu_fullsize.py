"""Stage-wise parity at the BASELINE sizes of cfg 3, cfg 4 and cfg 5.

The reference cannot weld these layouts end to end (ragged k-means cuts for
cfg 3/4; 16x16 blocks exceed the zipper's FP64 reach for cfg 5, SURVEY
§8(c)), so as in SURVEY the contract is stage-wise, checked here against the
oracle (pinned bitwise to the reference):

  * partition integers of EVERY subdomain bit for bit (`partition.py:94-137`):
    face labels, sorted vertex maps, boundary cycles, local loops;
  * the DNCP flatten (`flatten.py:125-188`) and the Dirichlet solve with the
    flattened boundary values (`assemble.py:23-50`) of 16 subdomains spread
    over the batch, <= 1e-6 x the subdomain diameter, from one batched
    launch per stage over all subdomains;
  * the solve-kernel times are printed (-s) and gathered in
    profiles/r2_fullsize_stagewise.log.

cfg 3: 500K-point Delaunay disk, 128 k-means subdomains; cfg 4: icosphere
subdivided 9 times (2.6M vertices), 256 subdomains; cfg 5: 4096^2 height
field, 64 bumps, 16x16 = 256 subdomains of ~66K vertices. Generation and the
oracle split take ~1-2 min per config on the host (slow marker).
"""

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NSAMPLE = 16


def _make(name):
    from paper_1903_12359_b200 import generators as gen
    if name == "cfg3":
        return gen.cfg3(seed=0)
    if name == "cfg4":
        return gen.cfg4(seed=0)
    return gen.height_field_case(4096, 16, n_bumps=64, seed=0)


@pytest.fixture(scope="module", params=["cfg3", "cfg4", "cfg5"])
def full(request, cuda):
    import oracle
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    V, F, cuts = _make(request.param)
    part = partition_mesh(TriMesh(V, F), cuts)
    sp = oracle.split_mesh(V, F, cuts)
    yield request.param, part, sp
    part.batch.close()


def test_partition_bit_exact_every_subdomain(full):
    name, part, sp = full
    assert part.n_submeshes == sp.n_sub
    assert np.array_equal(part.face_assignment, sp.face_assignment)
    for c, (a, b) in enumerate(zip(part.vertex_maps, sp.vertex_maps)):
        assert np.array_equal(a, b), (name, c)
    for c, (a, b) in enumerate(zip(part.boundary_cycles, sp.boundary_cycles)):
        assert np.array_equal(a, b), (name, c)
    for c, (a, b) in enumerate(zip(part.local_loops, sp.loops)):
        assert np.array_equal(a, b), (name, c)


def _pool(n):
    # one BLAS thread per worker process (SuperLU's dense kernels otherwise
    # oversubscribe the host: 16 workers x 16 OpenBLAS threads)
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    return ProcessPoolExecutor(max_workers=max(1, min(n, mp.cpu_count())), mp_context=mp.get_context("spawn"))


def test_sampled_solves_match_oracle(full):
    import torch
    from oracle.pipeline import _dirichlet_job, _flatten_job
    from paper_1903_12359_b200 import _native as nat
    name, part, sp = full
    b = part.batch
    z, st = b.flatten()
    assert all(s["status"] == 0 for s in st)
    fl = b.last_solve(0)
    z = z.cpu().numpy()
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
    zh, sth = b.harmonic(gid, z[gid])
    assert all(s["status"] == 0 for s in sth)
    hm = b.last_solve(1)
    zh = zh.cpu().numpy()
    sample = sorted(set(np.linspace(0, b.K - 1, NSAMPLE).round().astype(int).tolist()))
    with _pool(len(sample)) as ex:
        ref_f = list(ex.map(_flatten_job, [(sp.sub_V[c], sp.sub_F[c], sp.loops[c]) for c in sample]))
        ref_h = list(ex.map(_dirichlet_job, [(sp.sub_V[c], sp.sub_F[c], sp.loops[c], z[voff[c] + sp.loops[c]])
                                             for c in sample]))
    worst_f = worst_h = 0.0
    for c, rf, rh in zip(sample, ref_f, ref_h):
        got = z[voff[c]:voff[c + 1]]
        ef = np.max(np.abs(got - rf)) / (2 * np.max(np.abs(rf - rf.mean())))
        got_h = zh[voff[c]:voff[c + 1]]
        eh = np.max(np.abs(got_h - rh)) / (2 * np.max(np.abs(rh - rh.mean())))
        worst_f, worst_h = max(worst_f, ef), max(worst_h, eh)
        assert ef <= 1e-6, (name, c, ef)
        assert eh <= 1e-6, (name, c, eh)
    its = sorted(s["iters"] for s in st)
    print(f"\n[{name}] K={b.K} sampled {len(sample)}: flatten err/diam {worst_f:.2e}, harmonic {worst_h:.2e}; "
          f"flatten kernel {fl['kernel_ms']:.1f} ms (cluster {fl['cluster']}, iters min/med/max "
          f"{its[0]}/{its[len(its) // 2]}/{its[-1]}), harmonic kernel {hm['kernel_ms']:.1f} ms")
