"""Golden graph files and the adjacency the REAL reference reads from them.

Run in the build container (where /root/reference is mounted):

    python tests/golden/make_golden_graph_io.py

Writes small Matrix Market and JSON edge-list files under
tests/golden/graph_io/, loads each with the reference's
`qwalk.graph_io.load_graph_file` (graph_io.py:65-76; imported read-only from
/root/reference/pkg/src) and records its adjacency CSR, or the exception class
and message for the malformed ones, in expected.json.
"""

from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "graph_io")


def _write(name, text):
    with open(os.path.join(OUT, name), "w", encoding="utf-8") as f:
        f.write(text)


def make_files():
    rng = np.random.default_rng(41)
    # a random symmetric pattern graph (symmetric storage: lower triangle only)
    n = 30
    edges = sorted({(int(max(a, b)), int(min(a, b))) for a, b in rng.integers(0, n, (70, 2)) if a != b})
    body = "".join(f"{i + 1} {j + 1}\n" for i, j in edges)
    _write("sym_pattern.mtx", f"%%MatrixMarket matrix coordinate pattern symmetric\n{n} {n} {len(edges)}\n{body}")
    # the same graph stored general / real with unit weights
    both = sorted(edges + [(j, i) for i, j in edges])
    body = "".join(f"{i + 1} {j + 1} 1.0\n" for i, j in both)
    _write("general_real.mtx", f"%%MatrixMarket matrix coordinate real general\n{n} {n} {len(both)}\n{body}")
    # no extension: sniffed as Matrix Market
    shutil.copy(os.path.join(OUT, "sym_pattern.mtx"), os.path.join(OUT, "noext"))
    # edge lists: plain, with duplicate edges (merged by summation -> weight 2 -> rejected)
    e = [[int(a), int(b)] for a, b in edges]
    _write("edges.json", json.dumps({"n": n, "edges": e}))
    _write("edges_dup.json", json.dumps({"n": n, "edges": e + [e[0]]}))
    _write("edges_isolated.json", json.dumps({"n": n + 3, "edges": e}))
    # malformed inputs
    _write("bad_keys.json", json.dumps({"n": 3, "edges": [], "x": 1}))
    _write("bad_n.json", json.dumps({"n": 0, "edges": []}))
    _write("bad_edge.json", json.dumps({"n": 3, "edges": [[0, 1, 2]]}))
    _write("bad_json.json", "{not json")
    _write("self_loop.json", json.dumps({"n": 3, "edges": [[0, 0]]}))
    _write("out_of_range.json", json.dumps({"n": 3, "edges": [[0, 5]]}))
    _write("nonsquare.mtx", "%%MatrixMarket matrix coordinate pattern general\n3 4 1\n1 2\n")
    _write("asym.mtx", "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\n")
    _write("weighted.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n2 1 2.5\n")
    _write("garbage.mtx", "this is not matrix market\n")
    _write("graph.txt", "")


CASES = ["sym_pattern.mtx", "general_real.mtx", "noext", "edges.json", "edges_dup.json",
         "edges_isolated.json", "bad_keys.json", "bad_n.json", "bad_edge.json", "bad_json.json",
         "self_loop.json", "out_of_range.json", "nonsquare.mtx", "asym.mtx", "weighted.mtx",
         "garbage.mtx", "graph.txt"]


def main():
    sys.path.insert(0, REF_SRC)
    from qwalk import graph_io  # reference package

    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    make_files()
    expected = {}
    for name in CASES:
        try:
            g = graph_io.load_graph_file(os.path.join(OUT, name))
        except Exception as exc:   # noqa: BLE001 (recording the reference's behaviour)
            msg = str(exc).replace(OUT, "<dir>")
            expected[name] = {"error": type(exc).__name__, "message": msg}
            continue
        a = g.adjacency
        expected[name] = {"n": int(g.n), "offsets": a.row_offsets.tolist(), "cols": a.col_indices.tolist()}
    with open(os.path.join(OUT, "expected.json"), "w", encoding="utf-8") as f:
        json.dump(expected, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
