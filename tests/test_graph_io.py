"""Graph files (reference graph_io.py:26-76) vs what the reference itself read
from the same files (tests/golden/graph_io/, made by
tests/golden/make_golden_graph_io.py): adjacency CSR, or exception class and
message."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2406_08186_b200 import graph_io

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "graph_io")
with open(os.path.join(GOLD, "expected.json"), encoding="utf-8") as _f:
    EXPECTED = json.load(_f)


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_graph_file_matches_reference(name):
    exp = EXPECTED[name]
    path = os.path.join(GOLD, name)
    if "error" in exp:
        with pytest.raises(Exception) as ei:
            graph_io.load_graph_file(path)
        assert type(ei.value).__name__ == exp["error"]
        assert str(ei.value).replace(GOLD, "<dir>") == exp["message"]
        return
    g = graph_io.load_graph_file(path)
    assert g.n == exp["n"]
    np.testing.assert_array_equal(g.adjacency.row_offsets, exp["offsets"])
    np.testing.assert_array_equal(g.adjacency.col_indices, exp["cols"])


def test_explicit_format_and_unknown_format():
    g = graph_io.load_graph_file(os.path.join(GOLD, "noext"), fmt="mtx")
    assert g.n == EXPECTED["noext"]["n"]
    with pytest.raises(Exception, match="unknown graph file format"):
        graph_io.load_graph_file(os.path.join(GOLD, "edges.json"), fmt="xml")
