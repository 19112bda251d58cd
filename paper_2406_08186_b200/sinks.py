"""On-disk sinks of probability distributions (reference cli.py:390-432).

The formats the reference's `qwalk simulate` writes downstream of the reducer,
byte for byte, with the per-value text produced by libqwb200's threaded
formatter (`qwb_format_json_floats` / `qwb_format_csv_rows`, csrc/sinks.cpp)
instead of a Python loop over every vertex:

* JSON (`_write_json_sink`, cli.py:398-408): one document
  `{"schema":1,"model":...,"graph":...,"snapshots":[{"k":..,"t":..,"p":[..]},..]}`
  written with separators (",", ":") and a trailing newline;
* CSV (`_write_csv_rows` / `_write_csv_sink`, cli.py:411-421): header
  `snapshot,t,vertex,probability`, one row per (snapshot, vertex);
* frames (`_write_frames_sink`, cli.py:424-431): `frame_{k:05d}.csv` per
  snapshot with header `vertex,probability`.

Records are `DistributionRecord(k, t, p)` (cli.py:95-99): the snapshot index,
its time (the index for coined walks, k * delta_t for CTQW) and the vertex
probabilities (numpy float64, or a torch tensor, which is copied to the host).
"""

from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N

_CHUNK = 1 << 22   # values formatted per native call (bounds the text buffer)


@dataclass(frozen=True)
class DistributionRecord:
    """One saved snapshot (reference cli.py:95-99)."""

    k: int
    t: float
    p: np.ndarray


def records(sim_range, probs, times=None) -> list[DistributionRecord]:
    """Pair snapshot indices, times and distributions as the reference's
    `_execute` does (cli.py:384-387); times default to the indices (coined)."""
    idx = list(sim_range.indices()) if hasattr(sim_range, "indices") else list(sim_range)
    times = idx if times is None else list(times)
    return [DistributionRecord(k, t, p) for k, t, p in zip(idx, times, probs)]


def _host_f64(p) -> np.ndarray:
    if hasattr(p, "detach"):   # torch tensor (device or host)
        p = p.detach().to("cpu").numpy()
    a = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    if a.ndim != 1:
        raise ValueError("p: a distribution must be one-dimensional")
    return a


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _buffer(n: int, per_item: int) -> np.ndarray:
    return np.empty(min(n, _CHUNK) * per_item + 1, dtype=np.uint8)


def _json_floats(a: np.ndarray, f) -> None:
    """Writes "p0,p1,...": the body of a JSON "p" list."""
    lib = N.load()
    buf = _buffer(a.size, 25)
    for lo in range(0, a.size, _CHUNK):
        blk = a[lo:lo + _CHUNK]
        n = lib.qwb_format_json_floats(blk.ctypes.data, blk.size, buf.ctypes.data, buf.size, _threads())
        if n < 0:
            raise RuntimeError("qwb_format_json_floats: buffer too small")
        if lo:
            f.write(b",")
        f.write(memoryview(buf)[:n])


def _csv_rows(a: np.ndarray, prefix: str, f) -> None:
    """Writes one "<prefix><vertex>,<p>" line per vertex."""
    lib = N.load()
    pre = prefix.encode()
    buf = _buffer(a.size, len(pre) + 47)
    for lo in range(0, a.size, _CHUNK):
        blk = a[lo:lo + _CHUNK]
        n = lib.qwb_format_csv_rows(blk.ctypes.data, blk.size, lo, pre, len(pre), buf.ctypes.data, buf.size,
                                    _threads())
        if n < 0:
            raise RuntimeError("qwb_format_csv_rows: buffer too small")
        f.write(memoryview(buf)[:n])


def _json_scalar(x) -> str:
    if isinstance(x, (bool, np.bool_)):
        return json.dumps(bool(x))
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return json.dumps(float(x))


def write_json_sink(path, model: str, graph_desc: dict, recs) -> None:
    """The reference's JSON sink (cli.py:398-408) for model "coined"/"ctqw"
    and the config's graph description."""
    head = json.dumps({"schema": 1, "model": model, "graph": graph_desc}, separators=(",", ":"))
    with open(path, "wb") as f:
        f.write(head[:-1].encode() + b',"snapshots":[')
        for i, r in enumerate(recs):
            if i:
                f.write(b",")
            f.write(f'{{"k":{_json_scalar(r.k)},"t":{_json_scalar(r.t)},"p":['.encode())
            _json_floats(_host_f64(r.p), f)
            f.write(b"]}")
        f.write(b"]}\n")


def _csv_field(x) -> str:
    if isinstance(x, (int, np.integer)) and not isinstance(x, (bool, np.bool_)):
        return str(int(x))
    return str(float(x)) if isinstance(x, (float, np.floating)) else str(x)


def write_csv_sink(path, recs) -> None:
    """The reference's CSV sink (cli.py:411-421)."""
    with open(path, "wb") as f:
        f.write(b"snapshot,t,vertex,probability\n")
        for r in recs:
            _csv_rows(_host_f64(r.p), f"{_csv_field(r.k)},{_csv_field(r.t)},", f)


def write_frames_sink(dir_path, recs) -> None:
    """The reference's frames sink (cli.py:424-431): one CSV per snapshot."""
    d = Path(dir_path)
    d.mkdir(parents=True, exist_ok=True)
    for r in recs:
        with open(d / f"frame_{r.k:05d}.csv", "wb") as f:
            f.write(b"vertex,probability\n")
            _csv_rows(_host_f64(r.p), "", f)


def format_float(x: float, json_style: bool = False) -> str:
    """Python's float repr (JSON spelling of non-finite values if json_style),
    computed natively; exposed for tests."""
    buf = C.create_string_buffer(40)
    n = N.load().qwb_format_f64_repr(float(x), int(json_style), buf)
    return buf.raw[:n].decode()
