"""Shared test configuration.

Markers: `gpu` — needs a B200 (run with `-m gpu` on the GPU box).  Everything
else runs on CPU.  The oracle under `oracle/` is test infrastructure: tests
use it only as the checker.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a B200 GPU")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def golden_group(z, prefix: str) -> dict:
    p = prefix + "/"
    return {k[len(p):]: z[k] for k in z.files if k.startswith(p)}


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import qwalk_oracle
    return qwalk_oracle


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (den if den > 0 else 1.0)
