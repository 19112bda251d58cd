"""ctypes binding of libqwb200.so (the C ABI declared in include/qwb200.h).

The product has no CPU fallback: if the library is missing or no B200 is
visible, every compute entry point raises.  Status codes are mapped onto the
reference's exception classes (errors.py of qwalk 0.1.0).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libqwb200.so")

QWB_OK = 0
STATUS_TO_EXC = {
    1: E.DimensionMismatch,
    2: E.NonFiniteEntry,
    3: E.NotOnDevice,
    4: E.EngineStopped,
    5: E.AlreadyStopped,
    6: E.UnsupportedEngineKind,
    7: E.SeriesNotConverged,
    8: E.MarkedVertexOutOfRange,
    9: E.UnsupportedGraphForPersistentShift,
    10: ValueError,
    20: E.DeviceError,
    21: E.DeviceError,
    22: E.DeviceError,
}

FAMILY = {"generic": 0, "cycle": 1, "line": 2, "grid": 3, "hypercube": 4}
SHIFT = {"flipflop": 0, "persistent": 1, "none": 2}


class qwb_z(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_dbl = C.c_double
_p_i64 = C.POINTER(C.c_int64)
_p_int = C.POINTER(C.c_int)
_p_dbl = C.POINTER(C.c_double)

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES = {
    "qwb_init": [_i32, C.POINTER(_vp)],
    "qwb_shutdown": [_vp],
    "qwb_last_error": [_vp],
    "qwb_version": [],
    "qwb_device_count": [_p_int],
    "qwb_family_adjacency": [_vp, _i32, _p_i64, _vp, _vp, _p_i64, _vp],
    "qwb_coined_operator": [_vp, _i64, _vp, _vp, _vp, _i64, _i32, _i32, _p_i64, _vp, _vp, _vp,
                            _p_i64, _vp],
    "qwb_shift_sources": [_vp, _i64, _vp, _vp, _i32, _i32, _p_i64, _vp, _vp],
    "qwb_hamiltonian": [_vp, _i64, _vp, _vp, _dbl, _vp, _i64, _vp, _vp, _vp, _vp],
    "qwb_inf_norm": [_vp, _i64, _vp, _vp, _p_dbl, _vp],
    "qwb_csr_prepare": [_vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp],
    "qwb_spmv": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "qwb_csr_run": [_vp, _i64, _vp, _vp, _vp, _vp, _p_i64, _i64, _vp, _vp, _vp],
    "qwb_marked_bitmap": [_vp, _i64, _vp, _i64, _vp, _vp],
    "qwb_lattice_to_planes": [_vp, _i64, _i64, _vp, _vp, _vp],
    "qwb_lattice_from_planes": [_vp, _i64, _i64, _vp, _vp, _vp],
    "qwb_lattice_run": [_vp, _i64, _i64, _i32, _vp, _p_i64, _i64, _vp, _vp, _i64, _p_i64, _i32, _vp,
                        _p_int, _vp],
    "qwb_lattice_fused_depth": [_i64, _i64, _i64, _p_int, _p_int],
    "qwb_lattice_step": [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp],
    "qwb_lattice_probability": [_vp, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_to_planes": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_from_planes": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_probability": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_step": [_vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _vp],
    "qwb_slab_exchange_local": [_vp, _i64, _i32, _p_i64, C.POINTER(_vp), _i32, _vp],
    "qwb_csr_halo_exchange": [_vp, _i64, _vp, _vp, _p_i64, _p_i64, C.POINTER(C.c_int), _i32, _vp, _vp],
    "qwb_slab_ghost_rows": [_i64, _i64, _i64, _i64, _p_int],
    "qwb_slab_depth": [_p_int],
    "qwb_slab_to_planes_g": [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_from_planes_g": [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_probability_g": [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "qwb_slab_advance_local": [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i32, _i32,
                               _vp],
    "qwb_slab_run_fused": [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32,
                           _p_int, _vp],
    "qwb_slab_ghost_exchange_local": [_vp, _i64, _i64, _i32, _p_i64, C.POINTER(_vp), _i32, _vp],
    "qwb_comm_unique_id": [_vp],
    "qwb_comm_init": [_vp, _vp, _i32, _i32],
    "qwb_comm_destroy": [_vp],
    "qwb_slab_run": [_vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i64, _i32, _i32, _p_int, _vp],
    "qwb_prob_arcs": [_vp, _i64, _vp, _vp, _vp, _vp],
    "qwb_prob_abs2": [_vp, _i64, _vp, _vp, _vp],
    "qwb_axpy": [_vp, _i64, qwb_z, _vp, _vp, _vp, _vp],
    "qwb_scale": [_vp, _i64, qwb_z, _vp, _vp, _vp],
    "qwb_dot": [_vp, _i64, _vp, _vp, C.POINTER(qwb_z), _vp],
    "qwb_norm": [_vp, _i64, _vp, _p_dbl, _vp],
    "qwb_check_finite": [_vp, _i64, _vp, _p_int, _vp],
    "qwb_taylor_evolve_csr": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _i32, _p_int, _vp],
    "qwb_taylor_evolve_hypercube_sharded": [_vp, _i32, _i32, _dbl, _vp, _vp, _vp, _i64, _dbl, _dbl, _i32,
                                            _p_int, _vp],
    "qwb_taylor_evolve_hypercube_shards_local": [_vp, _i32, _i32, _dbl, _vp, C.POINTER(_vp), C.POINTER(_vp),
                                                 _i64, _dbl, _dbl, _i32, _p_int, _vp],
    "qwb_taylor_evolve_hypercube": [_vp, _i32, _dbl, _vp, _vp, _vp, _i64, _dbl, _dbl, _i32, _p_int,
                                    _vp],
    "qwb_hypercube_apply": [_vp, _i32, _dbl, _vp, _vp, _vp, _vp],
    "qwb_format_f64_repr": [_dbl, _i32, _vp],
    "qwb_format_json_floats": [_vp, _i64, _vp, _i64, _i32],
    "qwb_format_csv_rows": [_vp, _i64, _i64, C.c_char_p, _i64, _vp, _i64, _i32],
}
_RESTYPES = {"qwb_last_error": C.c_char_p, "qwb_version": C.c_char_p,
             "qwb_format_json_floats": C.c_int64, "qwb_format_csv_rows": C.c_int64}

_lock = threading.Lock()
_lib = None


def library_path() -> str:
    return LIB_PATH


def load() -> C.CDLL:
    """Load libqwb200.so (once).  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise E.DeviceError(
                f"libqwb200.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2406_08186_b200._build` (there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return sorted(SIGNATURES)


def last_error(ctx=None) -> str:
    msg = load().qwb_last_error(ctx)
    return msg.decode() if msg else ""


def check(status: int, ctx=None) -> None:
    if status == QWB_OK:
        return
    exc = STATUS_TO_EXC.get(int(status), E.DeviceError)
    raise exc(last_error(ctx) or f"libqwb200 status {status}")


def call(name: str, *args, ctx=None) -> None:
    check(getattr(load(), name)(*args), ctx)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else int(t.data_ptr())


def i64_array(values) -> C.Array:
    vals = [int(v) for v in values]
    arr = (C.c_int64 * max(1, len(vals)))(*vals)
    return arr
