"""Golden files of the distribution sinks, written by the REAL reference.

Run in the build container (where /root/reference is mounted):

    python tests/golden/make_golden_sinks.py

It imports the reference's `qwalk.cli` from /root/reference/pkg/src
(read-only; nothing is copied) and calls its JSON, CSV and frames sink
writers (cli.py:398-431) on seeded records: a coined walk's distributions
(integer times) and a CTQW run's (times k * delta_t), plus values that
exercise every branch of Python's float repr (fixed / exponent boundaries,
subnormals, whole numbers, -0.0, non-finite).  Output: tests/golden/sinks/.
"""

from __future__ import annotations

import os
import shutil
import sys
import types

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sinks")


def golden_records():
    """The records the fixtures hold (also rebuilt by the tests)."""
    rng = np.random.default_rng(2024)
    p0 = rng.random(40)
    p0 /= p0.sum()
    p1 = rng.random(40) ** 9
    edge = np.array([0.0, -0.0, 1.0, 0.5, 0.1, 1 / 3, 2.0 ** -13, 1e-4, 9.99e-5, 1e-5, 1e16, 1e15,
                     9999999999999998.0, 123456789.0, 5e-324, 2.2250738585072014e-308,
                     1.7976931348623157e308, 1e22, 0.30000000000000004, np.nan, np.inf, -np.inf,
                     -1.5e-7, 12345678901234567890.0])
    coined = [(0, 0, p0), (5, 5, p1), (10, 10, edge)]
    dt = 0.1
    ctqw = [(k, k * dt, p) for k, p in ((0, p1), (3, p0), (7, edge))]
    return coined, ctqw


GRAPH_COINED = {"family": "cycle", "n": 40}
GRAPH_CTQW = {"family": "grid", "nx": 8, "ny": 5, "periodic": True}


def main():
    sys.path.insert(0, REF_SRC)
    from qwalk import cli  # reference package
    from pathlib import Path

    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    coined, ctqw = golden_records()
    for name, model, desc, recs in (("coined", "coined", GRAPH_COINED, coined),
                                    ("ctqw", "ctqw", GRAPH_CTQW, ctqw)):
        records = [cli.DistributionRecord(k, t, p) for k, t, p in recs]
        plan = types.SimpleNamespace(model=model, graph_desc=desc)
        cli._write_json_sink(Path(OUT) / f"{name}.json", plan, records)
        cli._write_csv_sink(Path(OUT) / f"{name}.csv", records)
        cli._write_frames_sink(Path(OUT) / f"{name}_frames", records)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
