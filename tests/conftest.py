import os
import sys

# the oracle's SuperLU solves run in worker processes in several tests: one
# BLAS thread each (unset, every worker spins up a thread per core)
for _var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_var, "1")

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PIPELINE_CASES = ["cfg1", "strips4", "blocks3x3", "disk2x2", "k1free", "k1disk", "flat2x2",
                  "sphere2", "sphere4", "tree4x4", "ptree4x4", "qtree4x4"]
REPAIR_CASES = ["repair_k1disk", "repair_strips3", "repair_disk2"]


def case_pairs(case):
    """Explicit weld order of a golden case (None: the reference's greedy plan)."""
    from paper_1903_12359_b200 import generators as gen
    if case == "tree4x4":
        return gen.row_tree_schedule_order(4, 4)
    if case == "ptree4x4":
        return gen.pairwise_tree_schedule_order(4, 4)
    if case == "qtree4x4":
        return gen.quadtree_schedule_order(4, 4)
    return None


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: larger sizes")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


def unpack(z, name):
    off = z[name + "_off"]
    d = z[name]
    return [d[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def unpack_csr(z, name, values=True):
    from scipy import sparse
    ip = unpack(z, name + "_indptr")
    ix = unpack(z, name + "_indices")
    dv = unpack(z, name + "_data") if values else [np.zeros(len(a)) for a in ix]
    out = []
    for a, b, c in zip(ip, ix, dv):
        n = len(a) - 1
        out.append(sparse.csr_matrix((c, b, a), shape=(n, n)))
    return out


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1903_12359_b200  # noqa: F401
    return torch.device("cuda", 0)
