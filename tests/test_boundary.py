"""CPU-side checks of the drop-in boundary (no GPU needed).

* libgpuim.so loads and exports every symbol include/gpuim.h declares;
* the Python binding table covers exactly those symbols;
* the drop-in keeps the reference signature, and `install()` rebinds the
  entry point at every reference import site (when the reference is present).
"""
from __future__ import annotations

import inspect
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "gpuim.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(gim_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    from paper_2510_12196_b200 import _lib
    lib = _lib.load()  # loading needs no GPU
    syms = header_symbols()
    assert syms, "no symbols parsed from gpuim.h"
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gim_[a-z0-9_]+)", out))
    assert syms <= exported
    assert set(_lib.SIGNATURES) == syms


def test_version_without_gpu():
    from paper_2510_12196_b200 import _lib
    assert _lib.load().gim_version() == 1


def test_dropin_signature_matches_reference():
    from paper_2510_12196_b200 import integrated_map
    sig = inspect.signature(integrated_map)
    names = list(sig.parameters)
    assert names[:4] == ["g", "t", "eps", "seed"]
    expected = dict(coarsest_factor=128, phi=0.999, rho=2, filter_mode="nonneg",
                    jet_filter_c=0.25, sigma_coarse=0.065, sigma_fine=0.005, iw_max_finest=10)
    for k, v in expected.items():
        assert sig.parameters[k].default == v
        assert sig.parameters[k].kind == inspect.Parameter.KEYWORD_ONLY


def test_gpu_hm_signature_matches_reference():
    from paper_2510_12196_b200 import hierarchical_multisection
    names = list(inspect.signature(hierarchical_multisection).parameters)
    assert names == ["g", "t", "eps", "partitioner", "seed", "trace"]


def test_dropin_rejects_like_reference():
    from paper_2510_12196_b200 import integrated_map
    from paper_2510_12196_b200.generators import HostGraph, gen_grid
    import numpy as np

    class T:
        hierarchy = (2,)
        distances = (1,)
    empty = HostGraph(np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64),
                      np.zeros(0, np.int64))
    with pytest.raises(ValueError, match="empty"):
        integrated_map(empty, T(), 0.03)
    with pytest.raises(ValueError):
        integrated_map(gen_grid(3, 3), T(), 0.03, filter_mode="bogus")
    with pytest.raises(ValueError):
        integrated_map(gen_grid(3, 3), T(), 0.03, phi=0.0)


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference package not present")
def test_install_rebinds_every_import_site():
    code = f"""
import sys
sys.path.insert(0, {str(REF)!r}); sys.path.insert(0, {str(ROOT)!r})
import promap, promap.pipelines, promap.estimators, promap.cli, promap.bench, promap.graph
import paper_2510_12196_b200 as P
patched = P.install()
assert set(patched) == {{'promap.pipelines','promap.estimators','promap.cli','promap.bench','promap','promap.graph'}}, patched
for m in (promap.graph, promap.cli, promap.bench):
    assert m.load_metis is P.load_metis
for m in (promap, promap.pipelines, promap.estimators, promap.cli, promap.bench):
    assert m.integrated_map is P.integrated_map
    assert m.hierarchical_multisection is P.hierarchical_multisection
P.uninstall()
assert promap.pipelines.integrated_map is not P.integrated_map
assert promap.pipelines.hierarchical_multisection is not P.hierarchical_multisection
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "ok" in r.stdout
