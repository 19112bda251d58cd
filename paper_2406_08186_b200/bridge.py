"""The B200 core as engine kind "b200" of the UNMODIFIED reference package.

The reference's extension point for a new compute engine is its engine API
(`qwalk.backend`: `init_engine` / `stop_engine`, `move_to_device`,
`matvec_mul`, `vector_axpy` / `vector_scale` / `vector_dot` /
`vector_norm`; backend.py:243-464) — the "homogeneous linear-algebra API"
that its Neblina bridge implements.  It has no dynamic plugin
loader: a maintainer adds an `EngineKind` member and a branch
per operation.  `install(qwalk)` does exactly that from the outside, so the
reference's own `coined.simulate`, `ctqw.evolve_state`, `ctqw.simulate` and
CLI run on the GPU through libqwb200's C ABI:

    import qwalk
    from paper_2406_08186_b200 import bridge
    bridge.install(qwalk)
    eng = qwalk.init_engine("b200")
    states = qwalk.coined.simulate(eng, spec, (0, 10, 1), psi0)

Each operation keeps the reference's contract (backend.py:259-267, SPEC.md:
115-118): operands are validated (finite entries, dimensions, engine
ownership) with the reference's own exception classes, results come back as
new host `ComplexVector`s, one operation at a time per engine.  Because the
API returns host vectors, every step through it moves the state over PCIe
both ways; the walk-level entry points of `paper_2406_08186_b200` keep the
state in HBM instead.  Other engine kinds are passed to the original
functions untouched.

INTEGRATION.md §B shows the equivalent in-tree change to backend.py.
"""

from __future__ import annotations

from . import backend as QB
from . import errors as QE

KIND = "b200"
_PATCHED = ("init_engine", "stop_engine", "move_to_device", "matvec_mul", "vector_axpy", "vector_scale",
            "vector_dot", "vector_norm")


class B200Engine:
    """The reference's Engine for kind "b200": one libqwb200 context on one GPU."""

    def __init__(self, device: int | None = None):
        self.core = QB.init_engine(KIND, device=device)
        self.kind = KIND
        self.thread_count = 1

    @property
    def state(self) -> str:
        return self.core.state

    def _require_running(self) -> None:
        if self.core.state != "initialized":
            raise _ref_errors().EngineStopped("engine has been stopped")

    def __repr__(self):
        return f"Engine({KIND}, device={self.core.device}, {self.state})"


class _DeviceVec:
    """Payload of the reference's DeviceVector for a b200 engine: HBM storage."""

    __slots__ = ("tensor",)

    def __init__(self, tensor):
        self.tensor = tensor

    @property
    def dim(self) -> int:
        return int(self.tensor.shape[0])


class _DeviceCsr:
    """Payload of the reference's DeviceMatrix for a b200 engine."""

    __slots__ = ("csr",)

    def __init__(self, csr):
        self.csr = csr

    @property
    def n_rows(self) -> int:
        return self.csr.n_rows

    @property
    def n_cols(self) -> int:
        return self.csr.n_cols


_REF = {}


def _ref_errors():
    return _REF["errors"]


def _translate(exc: QE.QuantumWalkError):
    """Our exception -> the reference's class of the same name."""
    cls = getattr(_ref_errors(), type(exc).__name__, None)
    return cls(str(exc)) if cls is not None else exc


def install(qwalk) -> None:
    """Add engine kind "b200" to the imported reference package `qwalk`
    (idempotent).  Patches the engine functions in qwalk.backend and the names
    its modules imported from it (coined, ctqw, the package namespace)."""
    if getattr(qwalk, "_b200_bridge", False):
        return
    import importlib
    B = qwalk.backend
    RE = importlib.import_module(qwalk.__name__ + ".errors")
    _REF["errors"] = RE
    orig = {name: getattr(B, name) for name in _PATCHED}

    def is_b200(engine) -> bool:
        return isinstance(engine, B200Engine)

    def take_vec(engine, h):
        if not isinstance(h, B.DeviceVector) or not isinstance(h.vector, _DeviceVec):
            raise RE.NotOnDevice("operand must be moved to the device first")
        if h.engine is not engine:
            raise RE.NotOnDevice("operand was moved to a different engine")
        return h.vector.tensor

    def take_mat(engine, h):
        if not isinstance(h, B.DeviceMatrix) or not isinstance(h.matrix, _DeviceCsr):
            raise RE.NotOnDevice("operand must be moved to the device first")
        if h.engine is not engine:
            raise RE.NotOnDevice("operand was moved to a different engine")
        return h.matrix.csr

    def host_vector(t):
        return B.ComplexVector(QB.to_host(t))

    def init_engine(kind="serial", thread_count=None, *args, **kw):
        if str(getattr(kind, "value", kind)).lower() == KIND:
            return B200Engine(kw.get("device"))
        return orig["init_engine"](kind, thread_count, *args, **kw)

    def stop_engine(engine):
        if not is_b200(engine):
            return orig["stop_engine"](engine)
        if engine.core.state != "initialized":
            raise RE.AlreadyStopped("engine already stopped")
        QB.stop_engine(engine.core)

    def move_to_device(engine, obj):
        if not is_b200(engine):
            return orig["move_to_device"](engine, obj)
        engine._require_running()
        try:
            if isinstance(obj, B.ComplexVector):
                t = QB.to_device(engine.core, obj.entries)
                QB._require_finite(engine.core, t)
                return B.DeviceVector(engine, _DeviceVec(t))
            if isinstance(obj, B.CsrMatrix):
                m = QB.CsrMatrix(obj.n_rows, obj.n_cols, obj.row_offsets, obj.col_indices, obj.values)
                return B.DeviceMatrix(engine, _DeviceCsr(QB.upload_csr(engine.core, m)))
        except QE.QuantumWalkError as exc:
            raise _translate(exc) from None
        if isinstance(obj, B.DenseMatrix):
            raise RE.NotOnDevice("dense matrices are not supported by the b200 engine (CSR only)")
        raise RE.NotOnDevice(f"cannot move object of type {type(obj).__name__}")

    def matvec_mul(engine, v, m):
        if not is_b200(engine):
            return orig["matvec_mul"](engine, v, m)
        engine._require_running()
        x = take_vec(engine, v)
        csr = take_mat(engine, m)
        if csr.n_cols != x.shape[0]:
            raise RE.DimensionMismatch(f"matrix has {csr.n_cols} columns but vector has dim {x.shape[0]}")
        return host_vector(QB.spmv_device(engine.core, csr, x))

    def vector_axpy(engine, alpha, x, y):
        if not is_b200(engine):
            return orig["vector_axpy"](engine, alpha, x, y)
        engine._require_running()
        xe, ye = take_vec(engine, x), take_vec(engine, y)
        if xe.shape != ye.shape:
            raise RE.DimensionMismatch("axpy operands must have equal dimension")
        return host_vector(_axpy(engine.core, complex(alpha), xe, ye))

    def vector_scale(engine, alpha, x):
        if not is_b200(engine):
            return orig["vector_scale"](engine, alpha, x)
        engine._require_running()
        return host_vector(_scale(engine.core, complex(alpha), take_vec(engine, x)))

    def vector_dot(engine, x, y):
        if not is_b200(engine):
            return orig["vector_dot"](engine, x, y)
        engine._require_running()
        xe, ye = take_vec(engine, x), take_vec(engine, y)
        if xe.shape != ye.shape:
            raise RE.DimensionMismatch("dot operands must have equal dimension")
        return QB.vector_dot(engine.core, QB.DeviceVector(engine.core, xe), QB.DeviceVector(engine.core, ye))

    def vector_norm(engine, x):
        if not is_b200(engine):
            return orig["vector_norm"](engine, x)
        engine._require_running()
        return QB.device_norm(engine.core, take_vec(engine, x))

    new = {"init_engine": init_engine, "stop_engine": stop_engine, "move_to_device": move_to_device,
           "matvec_mul": matvec_mul, "vector_axpy": vector_axpy, "vector_scale": vector_scale,
           "vector_dot": vector_dot, "vector_norm": vector_norm}
    # the engine module itself, and every module that imported the names
    for mod in [B, qwalk] + [importlib.import_module(qwalk.__name__ + "." + m) for m in ("coined", "ctqw")]:
        for name, fn in new.items():
            if getattr(mod, name, None) is orig[name]:
                setattr(mod, name, fn)
    qwalk._b200_bridge = True


def _axpy(core, a: complex, xe, ye):
    from . import _native as N
    out = QB.empty_z(core, xe.shape[0])
    core.call("qwb_axpy", xe.shape[0], N.qwb_z(a.real, a.imag), N.ptr(xe), N.ptr(ye), N.ptr(out), core.stream())
    return out


def _scale(core, a: complex, xe):
    from . import _native as N
    out = QB.empty_z(core, xe.shape[0])
    core.call("qwb_scale", xe.shape[0], N.qwb_z(a.real, a.imag), N.ptr(xe), N.ptr(out), core.stream())
    return out


def installed(qwalk) -> bool:
    return bool(getattr(qwalk, "_b200_bridge", False))


__all__ = ["install", "installed", "B200Engine", "KIND"]
