"""Golden vectors for the native METIS reader: each case is a file text,
parsed by the REFERENCE's promap.graph.load_metis (graph.py:185-294) in this
container; stored: the text, and either the CSR arrays or the exact error
message.  Writes tests/golden/metis.npz (run from the repo root with the
reference on PYTHONPATH)."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from promap.graph import MetisFormatError, gen_grid, gen_rgg, load_metis, write_metis  # noqa: E402

CASES = {
    "triangle": "3 3\n2 3\n1 3\n1 2\n",
    "weighted_011": "3 2 011\n5 2 7\n1 1 7 3 4\n2 3 4\n",
    "vweights_010": "% comment\n3 2 10\n4 2\n1 1 3\n1 2\n",
    "comments_blank": "% a\n% b\n4 2\n2\n\n% inner\n4\n3\n\n\n",
    "no_trailing_newline": "2 1\n2\n1",
    "isolated_only": "3 0\n\n\n\n",
    "crlf": "2 1\r\n2\r\n1\r\n",
    "tabs": "2 1 001\n2\t5\n1 \t 5\n",
    "underscore_ints": "2 1\n2\n1_0\n",
    "empty_file": "",
    "only_comments": "% x\n% y\n",
    "bad_header_len": "3\n",
    "malformed_header": "3 x\n",
    "negative_header": "-1 0\n",
    "unsupported_fmt": "2 1 100\n2\n1\n",
    "fmt_4digits": "2 1 0001\n2\n1\n",
    "too_few_lines": "3 1\n2\n1\n",
    "too_many_lines": "1 0\n\n2\n",
    "missing_vweight": "2 1 010\n\n1 1\n",
    "bad_vweight": "2 1 010\nx 2\n1 1\n",
    "nonpos_vweight": "2 1 010\n0 2\n1 1\n",
    "dangling": "2 1 001\n2\n1 1\n",
    "bad_edge_token": "2 1\n2.0\n1\n",
    "out_of_range": "2 1\n3\n1\n",
    "self_loop": "2 1\n1\n1\n",
    "nonpos_eweight": "2 1 001\n2 0\n1 0\n",
    "duplicate": "3 2\n2 2\n1 1\n\n",
    "no_reverse": "3 2\n2 3\n1\n\n",
    "weight_mismatch": "2 1 001\n2 3\n1 4\n",
    "edge_count": "3 3\n2\n1 3\n2\n",
    "dup_before_bad": "3 2\n2 2\n1 x\n1\n",
}


def main():
    texts, arrays = {}, {}
    for name, text in CASES.items():
        texts[name] = text
    # real graphs through the reference writer (with explicit weights) and
    # hand-rolled unweighted files
    g = gen_grid(7, 9)
    r = gen_rgg(300, 0.55, 3)
    with tempfile.TemporaryDirectory() as d:
        for name, graph in (("grid7x9", g), ("rgg300", r)):
            p = os.path.join(d, name)
            write_metis(graph, p)
            texts[name] = open(p).read()
        out = {"count": np.int64(len(texts))}
        for i, (name, text) in enumerate(texts.items()):
            p = os.path.join(d, f"c{i}")
            with open(p, "w", newline="") as fh:
                fh.write(text)
            out[f"{i}/name"] = np.array(name)
            out[f"{i}/text"] = np.frombuffer(text.encode(), dtype=np.uint8)
            try:
                gr = load_metis(p)
                out[f"{i}/error"] = np.array("")
                out[f"{i}/offsets"] = gr.offsets
                out[f"{i}/targets"] = gr.edge_targets
                out[f"{i}/weights"] = gr.edge_weights
                out[f"{i}/vweights"] = gr.vertex_weights
            except MetisFormatError as e:
                out[f"{i}/error"] = np.array(str(e))
    np.savez_compressed("tests/golden/metis.npz", **out)
    print("cases", len(texts))


if __name__ == "__main__":
    main()
