"""The reference-side binding of INTEGRATION.md §2, executed as written.

The two ```python blocks of INTEGRATION.md §2 (`flatten_all`, which replaces
`_run_tasks(_dncp_task, ...)`, and `harmonic_and_repair`, which replaces
`_run_tasks(_harmonic_task, ...)`; reference `pipeline.py:105-109`, called at
`:159-161` and `:246-257`) are extracted from the document and exec'd with
raw ctypes on libpgcp_b200.so and torch only: nothing from the package is
imported into their namespace. The only edit is the library path, made
absolute. Their per-submesh outputs are compared with the reference's
`_run_tasks` outputs stored in the goldens (flatten and harmonic within
1e-6 of the subdomain's diameter; repair info equal)."""

import os
import re
import types

import numpy as np
import pytest

from conftest import ROOT, load_golden, unpack


def _section2_blocks():
    with open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8") as fh:
        text = fh.read()
    sec = text[text.index("## 2."):text.index("## 3.")]
    blocks = re.findall(r"```python\n(.*?)```", sec, flags=re.S)
    assert len(blocks) == 2, "INTEGRATION.md §2 should hold the two binding blocks"
    return blocks


def _binding():
    lib = os.path.join(ROOT, "paper_1903_12359_b200", "libpgcp_b200.so")
    assert os.path.exists(lib)
    ns = {"__name__": "pgcp_b200_binding"}
    for src in _section2_blocks():
        src = src.replace('ctypes.CDLL("libpgcp_b200.so")', f"ctypes.CDLL({lib!r})")
        exec(compile(src, "INTEGRATION.md", "exec"), ns)
    return ns


def test_blocks_are_package_free():
    for src in _section2_blocks():
        assert "paper_1903_12359_b200" not in src.replace("paper_1903_12359_b200/_native.py", "")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1", "blocks3x3", "strips4", "repair_strips3"])
def test_integration_binding_matches_reference(cuda, case):
    ns = _binding()
    z = load_golden(case)
    mesh = types.SimpleNamespace(vertices=z["V"], faces=z["F"])
    b, flat = ns["flatten_all"](mesh, z["cuts"])
    try:
        ref_flat = unpack(z, "flat")
        assert len(flat) == len(ref_flat)
        for c, (got, ref) in enumerate(zip(flat, ref_flat)):
            diam = 2 * np.max(np.abs(ref - ref.mean()))
            assert got.shape == ref.shape
            assert np.max(np.abs(got - ref)) <= 1e-6 * diam, (case, c)
        # the reference's welded boundary values, as _harmonic_task received them
        res = ns["harmonic_and_repair"](b, unpack(z, "harm_g"))
        ref_h = unpack(z, "harm")
        for c, ((got, info), ref) in enumerate(zip(res, ref_h)):
            diam = 2 * np.max(np.abs(ref - ref.mean()))
            assert np.max(np.abs(got - ref)) <= 1e-6 * diam, (case, c)
            assert info["flips_before"] == int(z["flips_before"][c])
    finally:
        ns["L"].pgcp_batch_destroy(b)
