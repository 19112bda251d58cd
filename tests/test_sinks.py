"""Distribution sinks (reference cli.py:398-431) vs files written by the
reference itself (tests/golden/sinks/, made by tests/golden/make_golden_sinks.py).

Host-only: the formatter lives in libqwb200.so but needs no GPU."""

from __future__ import annotations

import csv
import importlib.util
import io
import json
import os

import numpy as np
import pytest

from paper_2406_08186_b200 import sinks

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "sinks")
_spec = importlib.util.spec_from_file_location("make_golden_sinks", os.path.join(HERE, "golden", "make_golden_sinks.py"))
_mk = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mk)
GRAPH_COINED, GRAPH_CTQW, golden_records = _mk.GRAPH_COINED, _mk.GRAPH_CTQW, _mk.golden_records


def _read(path) -> bytes:
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", ["coined", "ctqw"])
@pytest.mark.parametrize("chunk", [1 << 22, 7])
def test_sinks_match_reference_files(tmp_path, monkeypatch, name, chunk):
    monkeypatch.setattr(sinks, "_CHUNK", chunk)   # 7: records cross chunk boundaries
    coined, ctqw = golden_records()
    recs = [sinks.DistributionRecord(k, t, p) for k, t, p in (coined if name == "coined" else ctqw)]
    desc = GRAPH_COINED if name == "coined" else GRAPH_CTQW
    sinks.write_json_sink(tmp_path / "out.json", name, desc, recs)
    sinks.write_csv_sink(tmp_path / "out.csv", recs)
    sinks.write_frames_sink(tmp_path / "frames", recs)
    assert _read(tmp_path / "out.json") == _read(os.path.join(GOLD, f"{name}.json"))
    assert _read(tmp_path / "out.csv") == _read(os.path.join(GOLD, f"{name}.csv"))
    gold_frames = sorted(os.listdir(os.path.join(GOLD, f"{name}_frames")))
    assert sorted(os.listdir(tmp_path / "frames")) == gold_frames
    for fn in gold_frames:
        assert _read(tmp_path / "frames" / fn) == _read(os.path.join(GOLD, f"{name}_frames", fn))


def test_float_repr_random_bit_patterns():
    rng = np.random.default_rng(7)
    x = rng.integers(0, 2 ** 64, size=20000, dtype=np.uint64).view(np.float64)
    x = np.concatenate([x, rng.random(5000), rng.random(5000) ** 12, 10.0 ** rng.uniform(-8, 20, 5000)])
    for v in x:
        v = float(v)
        assert sinks.format_float(v) == str(v)
        assert sinks.format_float(v, json_style=True) == json.dumps(v)


def test_threaded_record_matches_python_writers(tmp_path):
    # large enough for the multi-threaded formatter (>= 2^17 values)
    p = np.random.default_rng(3).random(300_001) ** 3
    recs = [sinks.DistributionRecord(4, 0.4, p)]
    sinks.write_json_sink(tmp_path / "a.json", "ctqw", {"family": "cycle", "n": p.size}, recs)
    doc = {"schema": 1, "model": "ctqw", "graph": {"family": "cycle", "n": p.size},
           "snapshots": [{"k": 4, "t": 0.4, "p": [float(v) for v in p]}]}
    assert _read(tmp_path / "a.json") == (json.dumps(doc, separators=(",", ":")) + "\n").encode()
    sinks.write_csv_sink(tmp_path / "a.csv", recs)
    s = io.StringIO()
    w = csv.writer(s, lineterminator="\n")
    w.writerow(["snapshot", "t", "vertex", "probability"])
    for v, pv in enumerate(p):
        w.writerow([4, 0.4, v, float(pv)])
    assert _read(tmp_path / "a.csv") == s.getvalue().encode()


def test_records_pairing_and_device_free_inputs():
    from paper_2406_08186_b200.state import SimRange
    recs = sinks.records(SimRange(0, 6, 2), [np.zeros(3)] * 3, times=[0.0, 0.5, 1.0])
    assert [(r.k, r.t) for r in recs] == [(0, 0.0), (2, 0.5), (4, 1.0)]
    with pytest.raises(ValueError):
        sinks._host_f64(np.zeros((2, 2)))
