"""ctypes binding of the plain C oracle (oracle/rd_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
package. It shares no code with ``paper_1901_06535_b200`` (the CUDA path); the
only module both sides use is ``rdinputs`` (seeded inputs, no method
arithmetic).

Every function cites the PAPER.md passage it follows; see rd_oracle.h and
DESIGN.md §3 for the readings (ghost = edge cell, canonical expression tree,
constants rounded once, events before their step, probes every ``stride``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_SRC = [os.path.join(_HERE, n) for n in ("rd_oracle.c", "rd_oracle.h", "oracle_body.h")]

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liborc.so with gcc (plain C, no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(p) for p in _SRC)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        cmd = ["gcc", *CFLAGS, "-o", _LIB_PATH, os.path.join(_HERE, "rd_oracle.c"), "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB_PATH


ORC_REACTION_OFF = 1
_KIND = {"disc": 1, "rect": 2, "half_disc": 3}
SHAPE_MASK_PHI = 1


class _Params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("eps", "f", "q", "Du", "dt", "dx")]


class _Shape(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("dir", C.c_int32),
        ("cy2", C.c_int64), ("cx2", C.c_int64), ("r", C.c_int64),
        ("y0", C.c_int64), ("x0", C.c_int64), ("y1", C.c_int64), ("x1", C.c_int64),
        ("flags", C.c_uint32), ("pad_", C.c_uint32), ("mask_phi", C.c_double),
    ]


class _Rect(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("y0", "x0", "y1", "x1")]


class _Event(C.Structure):
    _fields_ = [("shape", _Shape), ("value", C.c_double), ("at_step", C.c_int64)]


class _Probe(C.Structure):
    _fields_ = [("rect", _Rect), ("threshold", C.c_double), ("stride", C.c_int64)]


class _Fault(C.Structure):
    _fields_ = [("step", C.c_int64), ("i", C.c_int64), ("j", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64 = C.c_int64
        for sfx in ("f64", "f32"):
            getattr(L, f"orc_reaction_{sfx}").restype = C.c_double
            getattr(L, f"orc_reaction_{sfx}").argtypes = [C.c_double] * 3 + [C.POINTER(_Params), C.POINTER(C.c_double)]
            getattr(L, f"orc_laplacian_{sfx}").argtypes = [i64, i64, P, P, C.POINTER(_Params)]
            getattr(L, f"orc_step_{sfx}").argtypes = [i64, i64, P, P, P, P, P, C.POINTER(_Params), C.c_uint32]
            getattr(L, f"orc_stamp_{sfx}").restype = i64
            getattr(L, f"orc_stamp_{sfx}").argtypes = [i64, i64, P, P, C.POINTER(_Shape), C.c_double]
            getattr(L, f"orc_probe_max_{sfx}").restype = C.c_double
            getattr(L, f"orc_probe_max_{sfx}").argtypes = [i64, i64, P, C.POINTER(_Rect)]
            getattr(L, f"orc_run_{sfx}").restype = C.c_int
            getattr(L, f"orc_run_{sfx}").argtypes = [
                i64, i64, P, P, P, C.POINTER(_Params), C.c_uint32, i64, i64,
                C.POINTER(_Event), i64, C.POINTER(_Probe), i64, C.POINTER(C.c_int64), C.POINTER(_Fault), i64, P]
            getattr(L, f"orc_timelapse_record_{sfx}").argtypes = [i64, i64, P, P]
            getattr(L, f"orc_rest_fill_{sfx}").argtypes = [i64, i64, P, P, P, C.POINTER(_Params)]
        L.orc_rest_state.restype = C.c_double
        L.orc_rest_state.argtypes = [C.c_double, C.POINTER(_Params)]
        L.orc_shape_contains.restype = C.c_int
        L.orc_shape_contains.argtypes = [C.POINTER(_Shape), i64, i64]
        L.orc_params_default.argtypes = [C.POINTER(_Params)]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


@dataclass
class Params:
    """Table 1; phi is per cell and passed as a plane."""
    eps: float = 0.0243
    f: float = 1.4
    q: float = 0.002
    Du: float = 0.45
    dt: float = 0.001
    dx: float = 0.25

    def c(self) -> _Params:
        return _Params(self.eps, self.f, self.q, self.Du, self.dt, self.dx)


def _sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise TypeError(f"oracle supports float64/float32, not {dt}")


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


def shape_struct(s: dict) -> _Shape:
    """Convert a neutral shape dict (rdinputs) to the oracle's struct."""
    out = _Shape()
    out.kind = _KIND[s["kind"]]
    out.dir = int(s.get("dir", 0))
    out.cy2 = int(s.get("cy2", 0))
    out.cx2 = int(s.get("cx2", 0))
    out.r = int(s.get("r", 0))
    out.y0, out.x0, out.y1, out.x1 = (int(s.get(k, 0)) for k in ("y0", "x0", "y1", "x1"))
    if s.get("mask_phi") is not None:
        out.flags = SHAPE_MASK_PHI
        out.mask_phi = float(s["mask_phi"])
    return out


def reaction(u: float, v: float, phi: float, params: Params = Params(), dtype=np.float64):
    """(du/dt reaction part, dv/dt) of Eq. 1 in precision dtype."""
    dv = C.c_double()
    du = getattr(lib(), f"orc_reaction_{_sfx(dtype)}")(u, v, phi, C.byref(params.c()), C.byref(dv))
    return du, dv.value


def laplacian(u: np.ndarray, params: Params = Params()) -> np.ndarray:
    """Five-node Laplacian with ghost = edge."""
    u = np.ascontiguousarray(u)
    out = np.empty_like(u)
    getattr(lib(), f"orc_laplacian_{_sfx(u.dtype)}")(u.shape[0], u.shape[1], _ptr(u), _ptr(out), C.byref(params.c()))
    return out


def step(u, v, phi, params: Params = Params(), reaction_off: bool = False):
    """One synchronous forward-Euler step."""
    u = np.ascontiguousarray(u)
    v = np.ascontiguousarray(v, dtype=u.dtype)
    phi = np.ascontiguousarray(phi, dtype=u.dtype)
    uo, vo = np.empty_like(u), np.empty_like(v)
    getattr(lib(), f"orc_step_{_sfx(u.dtype)}")(
        u.shape[0], u.shape[1], _ptr(u), _ptr(v), _ptr(phi), _ptr(uo), _ptr(vo), C.byref(params.c()),
        ORC_REACTION_OFF if reaction_off else 0)
    return uo, vo


def stamp(u: np.ndarray, phi: np.ndarray, shape: dict, value: float = 1.0) -> int:
    """u := value on the shape's cells, clipped. In place."""
    s = shape_struct(shape)
    return getattr(lib(), f"orc_stamp_{_sfx(u.dtype)}")(u.shape[0], u.shape[1], _ptr(u), _ptr(phi), C.byref(s), value)


def shape_contains(shape: dict, i: int, j: int) -> bool:
    return bool(lib().orc_shape_contains(C.byref(shape_struct(shape)), i, j))


def probe_max(u: np.ndarray, rect) -> float:
    """max of u over [y0,y1)x[x0,x1)."""
    y0, x0, y1, x1 = rect
    r = _Rect(y0, x0, y1, x1)
    return getattr(lib(), f"orc_probe_max_{_sfx(u.dtype)}")(u.shape[0], u.shape[1], _ptr(u), C.byref(r))


@dataclass
class RunResult:
    u: np.ndarray
    v: np.ndarray
    first_fire: list = field(default_factory=list)
    status: int = 0
    fault: tuple | None = None
    max_u: np.ndarray | None = None


def rest_state(phi: float, params: Params = Params()) -> float:
    """u* = v* of the homogeneous medium with excitability phi, by fp64
    bisection."""
    return lib().orc_rest_state(float(phi), C.byref(params.c()))


def rest_fill(phi: np.ndarray, params: Params = Params()):
    """Quiescent initial planes u = v = u*(phi) per cell."""
    phi = np.ascontiguousarray(phi)
    u, v = np.empty_like(phi), np.empty_like(phi)
    getattr(lib(), f"orc_rest_fill_{_sfx(phi.dtype)}")(phi.shape[0], phi.shape[1], _ptr(phi), _ptr(u), _ptr(v),
                                                        C.byref(params.c()))
    return u, v


def timelapse_record(u: np.ndarray, max_u: np.ndarray) -> None:
    """max_u := pointwise max(max_u, u), in place."""
    getattr(lib(), f"orc_timelapse_record_{_sfx(u.dtype)}")(u.shape[0], u.shape[1], _ptr(np.ascontiguousarray(u)),
                                                            _ptr(max_u))


def run(u, v, phi, n_steps: int, events=(), probes=(), params: Params = Params(),
        step0: int = 0, reaction_off: bool = False, timelapse_stride: int = 0, max_u=None) -> RunResult:
    """Run one instance for n_steps.

    events: iterable of (shape_dict, value, at_step); probes: iterable of
    (rect(y0,x0,y1,x1), threshold, stride). With timelapse_stride > 0 the
    timelapse max_u (initial value max_u, default -inf) is recorded after every
    step that is a multiple of it. Returns copies of u, v (and max_u).
    """
    u = np.array(u, copy=True, order="C")
    v = np.array(v, copy=True, order="C", dtype=u.dtype)
    phi = np.ascontiguousarray(phi, dtype=u.dtype)
    ev = (_Event * max(1, len(events)))()
    for k, (shape, value, at) in enumerate(events):
        ev[k].shape = shape_struct(shape)
        ev[k].value = float(value)
        ev[k].at_step = int(at)
    pr = (_Probe * max(1, len(probes)))()
    for k, (rect, thr, stride) in enumerate(probes):
        pr[k].rect = _Rect(*rect)
        pr[k].threshold = float(thr)
        pr[k].stride = int(stride)
    ff = (C.c_int64 * max(1, len(probes)))(*([-1] * max(1, len(probes))))
    fault = _Fault(-1, -1, -1)
    mu = None
    if timelapse_stride > 0:
        mu = (np.full(u.shape, -np.inf, dtype=u.dtype) if max_u is None
              else np.array(max_u, dtype=u.dtype, copy=True, order="C"))
    st = getattr(lib(), f"orc_run_{_sfx(u.dtype)}")(
        u.shape[0], u.shape[1], _ptr(u), _ptr(v), _ptr(phi), C.byref(params.c()),
        ORC_REACTION_OFF if reaction_off else 0, step0, n_steps, ev, len(events), pr, len(probes), ff,
        C.byref(fault), int(timelapse_stride), _ptr(mu) if mu is not None else None)
    return RunResult(u, v, [ff[k] for k in range(len(probes))], st,
                     (fault.step, fault.i, fault.j) if st != 0 else None, mu)


def run_batch(u, v, phi, n_steps: int, events_per=None, probes_per=None, params: Params = Params()):
    """The batched mode (a8) as B independent oracle runs, instance by instance."""
    B = u.shape[0]
    out = []
    for b in range(B):
        out.append(run(u[b], v[b], phi[b], n_steps,
                       events=(events_per[b] if events_per else ()),
                       probes=(probes_per[b] if probes_per else ()), params=params))
    return out


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(n)
