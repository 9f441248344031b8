"""The reference package's own harness running on the GPU path (SURVEY §8(f)
row 4): with the unmodified reference installed in baseline/_ref (pip
install --no-deps of /root/reference/pkg; it travels to the GPU box),
`install()` rebinds `integrated_map` / `hierarchical_multisection` /
`load_metis` at every import site and then

* `promap.bench.run_once` (bench.py:73-95) produces the same RunRecord J and
  balance flag as the reference CPU run recorded in the golden fixtures;
* `promap map --algo im|hm` (cli.py:141-198) writes the reference's mapping
  file and stats for a METIS input;
* `IntegratedMapper` (estimators.py:99-106) maps through the drop-in.

Skipped when the reference is not installed (it is not product code)."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_npz

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def promap():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (REF / "promap").is_dir():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    import promap as P  # noqa: N813

    from paper_2510_12196_b200 import install, uninstall
    patched = install()
    assert "promap.bench" in patched and "promap.cli" in patched
    yield P
    uninstall()


def test_bench_run_once_on_gpu(promap):
    """run_once on config 1 (grid 128x128, H=4:8:2) equals the reference's
    recorded mappings for seeds 0-4 (tests/golden, made by the reference)."""
    from promap import bench
    from promap.graph import gen_grid
    from promap.topology import Topology
    z = load_npz("im_cfg1")
    g = gen_grid(128, 128)
    t = Topology((4, 8, 2), (1, 10, 100))
    for seed in range(5):
        rec = bench.run_once("grid_128x128", g, t, 0.03, "im", seed)
        assert rec.balanced
        assert rec.j == int(z[f"{seed}/j"])
    # the GPU path really ran: the module-level name is ours
    from paper_2510_12196_b200 import integrated_map
    assert bench.integrated_map is integrated_map


def test_cli_map_metis_on_gpu(promap, tmp_path):
    from promap import cli
    from promap.graph import gen_grid, write_metis
    g = gen_grid(32, 32)
    path = tmp_path / "g.metis"
    write_metis(g, str(path))
    for algo in ("im", "hm"):
        out, stats = tmp_path / f"{algo}.map", tmp_path / f"{algo}.json"
        rc = cli.main(["map", "--graph", str(path), "--algo", algo, "--hierarchy", "2:2:2",
                       "--distance", "1:10:100", "--coarsest-factor", "16", "--seed", "1",
                       "--out", str(out), "--stats", str(stats)])
        assert rc == 0
        a = np.loadtxt(out, dtype=np.int64)
        st = json.loads(stats.read_text())
        assert len(a) == g.n and st["balanced"]
        # same mapping as the reference's own CPU code on the same input
        from paper_2510_12196_b200 import install, uninstall
        from promap import pipelines
        t = promap.topology.Topology((2, 2, 2), (1, 10, 100))
        uninstall()
        try:
            cpu = (pipelines.integrated_map(g, t, 0.03, seed=1, coarsest_factor=16)
                   if algo == "im" else pipelines.hierarchical_multisection(g, t, 0.03, seed=1))
        finally:
            install()
        assert np.array_equal(a, cpu.assignment)


def test_estimator_through_dropin(promap):
    from promap.estimators import IntegratedMapper
    from promap.graph import gen_grid
    g = gen_grid(24, 24)
    est = IntegratedMapper(hierarchy="2:2:2", distances="1:10:100", epsilon=0.03,
                           coarsest_factor=16)
    est.fit(g)
    assert est.balanced_
    assert len(est.labels_) == g.n
    from promap import estimators
    from paper_2510_12196_b200 import integrated_map
    assert estimators.integrated_map is integrated_map
