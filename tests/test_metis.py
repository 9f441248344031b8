"""Native METIS reader (libgpuim.so, host C++) vs the reference's
promap.graph.load_metis (graph.py:185-294): identical CSR on valid files,
identical MetisFormatError messages on malformed ones.  Golden vectors:
scripts/make_golden_metis.py (the reference run in the build container)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN


def _cases():
    z = np.load(GOLDEN / "metis.npz")
    for i in range(int(z["count"])):
        yield i, z


@pytest.mark.parametrize("i", range(int(np.load(GOLDEN / "metis.npz")["count"])))
def test_metis_matches_reference(i, tmp_path):
    from paper_2510_12196_b200.metis import load_metis
    z = np.load(GOLDEN / "metis.npz")
    p = tmp_path / "g.metis"
    p.write_bytes(z[f"{i}/text"].tobytes())
    err = str(z[f"{i}/error"])
    if err:
        with pytest.raises(ValueError) as ei:
            load_metis(str(p))
        assert str(ei.value) == err
        assert type(ei.value).__name__ == "MetisFormatError"
    else:
        g = load_metis(str(p))
        assert np.array_equal(g.offsets, z[f"{i}/offsets"])
        assert np.array_equal(g.edge_targets, z[f"{i}/targets"])
        assert np.array_equal(g.edge_weights, z[f"{i}/weights"])
        assert np.array_equal(g.vertex_weights, z[f"{i}/vweights"])


def test_metis_roundtrip_large(tmp_path):
    """A multi-thread-sized file: write the rgg generator's graph in the
    reference's METIS layout, read it back natively."""
    from paper_2510_12196_b200.generators import gen_rgg
    from paper_2510_12196_b200.metis import load_metis
    g = gen_rgg(1 << 14, 0.55, 2)
    p = tmp_path / "rgg.metis"
    with open(p, "w") as fh:
        fh.write(f"{g.n} {g.m} 11\n")
        for v in range(g.n):
            b, e = g.offsets[v], g.offsets[v + 1]
            row = [str(int(g.vertex_weights[v]))]
            for u, w in zip(g.edge_targets[b:e], g.edge_weights[b:e]):
                row += [str(int(u) + 1), str(int(w))]
            fh.write(" ".join(row) + "\n")
    h = load_metis(str(p))
    assert np.array_equal(h.offsets, g.offsets)
    assert np.array_equal(h.edge_targets, g.edge_targets)
    assert np.array_equal(h.edge_weights, g.edge_weights)


def test_metis_missing_file():
    from paper_2510_12196_b200.metis import load_metis
    with pytest.raises(FileNotFoundError):
        load_metis("/nonexistent/graph.metis")
