"""B200-native Oregonator reaction-diffusion engine (RDCSim hot path, arXiv 1901.06535).

Thin Python binding of the C ABI in include/rd.h. The module-level functions
carry the C names (rd_create, rd_stimulate, rd_step, rd_read_fields, rd_probe,
...) and only marshal arguments; ``Sim`` is a convenience wrapper over them.
Every step of the hot path runs in librd.so's sm_100a kernels; if the
extension is missing, calls raise (there is no CPU fallback).

PyTorch is optional here and only used for streams (``Sim.set_stream``) and
process groups (``paper_1901_06535_b200.dist``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (RD_DISC, RD_ECUDA, RD_EINVAL, RD_ENCCL, RD_ENOMEM, RD_ENONFINITE, RD_EPARAM, RD_ERANGE, RD_F32, RD_F64, RD_HALF_DISC, RD_NO_CHECKPOINT,  # noqa: F401
                   RD_NO_GRAPH, RD_OK, RD_REACTION_OFF, RD_RECT, RD_SHAPE_MASK_PHI, TRANSPORTS, load)

__all__ = ["RDError", "Sim", "rd_params_default", "rd_create", "rd_create_slab", "rd_destroy", "rd_stimulate",
           "rd_step", "rd_read_fields", "rd_write_fields", "rd_probe", "rd_probe_latch", "rd_probe_result",
           "rd_get_step", "rd_get_fault", "rd_checkpoint", "rd_step_unchecked", "rd_step_begin", "rd_step_finish", "RD_BLOCK_PUSH", "rd_plane_origins", "rd_set_peer", "rd_push_ghosts", "rd_flag_ptr", "rd_ipc_export", "rd_ipc_map", "rd_stream_signal", "rd_stream_wait", "rd_read_flags", "rd_restore", "rd_set_stream", "rd_row_ptr", "rd_timelapse", "rd_read_timelapse", "stream_handle", "rd_set_params", "rd_init_rest", "rd_fill_noise", "rd_paint_phi", "rd_get_stats", "rd_set_profiling",
           "rd_reset_stats", "rd_last_error", "load", "rd_get_geometry", "rd_arena_bytes", "rd_create_device",
           "rd_field_ptr", "rd_dist_unique_id", "rd_dist_local_id", "rd_dist_shm_id", "rd_create_dist", "rd_write_fields_async",
           "rd_commit_fields", "rd_read_fields_async", "rd_io_wait"]

_KIND = {"disc": RD_DISC, "rect": RD_RECT, "half_disc": RD_HALF_DISC}
_DT = {np.dtype(np.float32): RD_F32, np.dtype(np.float64): RD_F64}


class RDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_lib.ERRNAMES.get(code, code)}: {msg}")
        self.code = code


def _check(rc: int, handle=None, create: bool = False):
    if rc != RD_OK:
        L = load()
        msg = (L.rd_create_error() if create else L.rd_last_error(handle)) or b""
        raise RDError(rc, msg.decode(errors="replace"))


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
        raise ValueError("host buffers must be C-contiguous numpy arrays")
    return a.ctypes.data_as(C.c_void_p)


_GEOM = {}  # handle address -> rd_get_geometry (dropped by rd_destroy)


def _geom(h) -> dict:
    key = getattr(h, "value", h)
    g = _GEOM.get(key)
    if g is None:
        g = _GEOM[key] = rd_get_geometry(h)
    return g


def _host(a: np.ndarray | None, h, rows: int | None = None, what: str = "buffer", writable: bool = False):
    """Validate a host buffer the C side reads or writes as rows x width
    elements of the handle's dtype (owned rows by default): the C side copies
    exactly that many bytes, so a short or mistyped array must not get
    through."""
    if a is None:
        return None
    g = _geom(h)
    dt = np.dtype(np.float32 if g["dtype"] == RD_F32 else np.float64)
    n = (g["height"] if rows is None else rows) * g["width"]
    if not isinstance(a, np.ndarray):
        raise ValueError(f"{what}: expected a numpy array")
    if a.dtype != dt:
        raise ValueError(f"{what}: dtype {a.dtype} does not match the handle's {dt}")
    if a.size != n:
        raise ValueError(f"{what}: {a.size} elements, expected {n} ({n // g['width']} rows x {g['width']})")
    if not a.flags.c_contiguous:
        raise ValueError(f"{what}: must be C-contiguous")
    if writable and not a.flags.writeable:
        raise ValueError(f"{what}: must be writable")
    return a.ctypes.data_as(C.c_void_p)


def _check_map(phi, dt, n: int, what: str):
    if phi is not None and phi.size != n:
        raise ValueError(f"{what}: {phi.size} elements, expected {n}")


def _shape(s: dict) -> _lib.rd_shape:
    out = _lib.rd_shape()
    out.kind = _KIND[s["kind"]]
    out.dir = int(s.get("dir", 0))
    for k in ("cy2", "cx2", "r", "y0", "x0", "y1", "x1"):
        setattr(out, k, int(s.get(k, 0)))
    if s.get("mask_phi") is not None:
        out.flags = RD_SHAPE_MASK_PHI
        out.mask_phi = float(s["mask_phi"])
    return out


# ----------------------------------------------------------------- C names

def rd_params_default() -> _lib.rd_params:
    p = _lib.rd_params()
    load().rd_params_default(C.byref(p))
    return p


def rd_create(width: int, height: int, phi_map: np.ndarray | None, *, batch: int = 1, dtype=np.float32,
              tb_depth: int = 0, flags: int = 0, params: _lib.rd_params | None = None, pitch: int = 0):
    """rd_create(grid, params, phi_map): phi_map is [batch][height][width] on
    the host, or None for phi = 0 (paint it with rd_paint_phi)."""
    dt = np.dtype(dtype)
    phi = None if phi_map is None else np.ascontiguousarray(phi_map, dtype=dt)
    _check_map(phi, dt, batch * height * width, "phi_map")
    g = _lib.rd_grid(width, height, batch, _DT[dt], tb_depth, flags, pitch)
    p = params or rd_params_default()
    h = C.c_void_p()
    _check(load().rd_create(C.byref(g), C.byref(p), _ptr(phi), C.byref(h)), create=True)
    return h


def rd_create_slab(width: int, height: int, phi_slab: np.ndarray, row0: int, height_global: int, halo: int, *,
                   batch: int = 1, dtype=np.float32, tb_depth: int = 0, flags: int = 0, params=None):
    dt = np.dtype(dtype)
    phi = None if phi_slab is None else np.ascontiguousarray(phi_slab, dtype=dt)
    lo, hi = max(0, row0 - halo), min(height_global, row0 + height + halo)
    _check_map(phi, dt, batch * (hi - lo) * width, "phi_slab (owned + ghost rows)")
    g = _lib.rd_grid(width, height, batch, _DT[dt], tb_depth, flags, 0)
    p = params or rd_params_default()
    h = C.c_void_p()
    _check(load().rd_create_slab(C.byref(g), C.byref(p), _ptr(phi), row0, height_global, halo, C.byref(h)),
           create=True)
    return h


def rd_destroy(h) -> None:
    _GEOM.pop(getattr(h, "value", h), None)
    _check(load().rd_destroy(h), h)


def rd_get_geometry(h) -> dict:
    """Where the handle's rows sit: width, height (owned rows), height_global,
    row0, pitch, batch, dtype, halo, tb_depth, rank, world, transport,
    flag_selftest."""
    g = _lib.rd_geometry()
    _check(load().rd_get_geometry(h, C.byref(g)), h)
    d = {k: getattr(g, k) for k, _ in g._fields_ if k != "pad"}
    d["transport"] = TRANSPORTS.get(d["transport"], d["transport"])
    return d


def rd_arena_bytes(width: int, height: int, *, batch: int = 1, dtype=np.float32, pitch: int = 0) -> int:
    g = _lib.rd_grid(width, height, batch, _DT[np.dtype(dtype)], 0, 0, pitch)
    n = C.c_size_t()
    _check(load().rd_arena_bytes(C.byref(g), C.byref(n)), create=True)
    return n.value


def rd_create_device(width: int, height: int, arena_ptr: int, arena_bytes: int, phi_ptr: int | None, *,
                     batch: int = 1, dtype=np.float32, tb_depth: int = 0, flags: int = 0, params=None, pitch: int = 0):
    """rd_create over a caller-owned DEVICE arena (e.g. a torch uint8 CUDA
    tensor of rd_arena_bytes bytes): phi_ptr is a device map [batch][H][W]
    (or None). The caller keeps the arena alive until rd_destroy."""
    g = _lib.rd_grid(width, height, batch, _DT[np.dtype(dtype)], tb_depth, flags, pitch)
    p = params or rd_params_default()
    h = C.c_void_p()
    _check(load().rd_create_device(C.byref(g), C.byref(p), C.c_void_p(arena_ptr), int(arena_bytes),
                                   C.c_void_p(phi_ptr) if phi_ptr else None, C.byref(h)), create=True)
    return h


def rd_field_ptr(h, b: int, plane: int) -> tuple[int, int]:
    """(device pointer of cell (0, 0), row pitch in elements) of instance b's
    current u (0), v (1) or phi (2); valid until the next rd_step."""
    p, pitch = C.c_void_p(), C.c_int64()
    _check(load().rd_field_ptr(h, int(b), int(plane), C.byref(p), C.byref(pitch)), h)
    return p.value, pitch.value


def rd_dist_unique_id() -> bytes:
    """128-byte rendezvous id for ranks in several processes (NCCL unique id)."""
    buf = C.create_string_buffer(128)
    _check(load().rd_dist_unique_id(buf), create=True)
    return buf.raw


def rd_dist_local_id() -> bytes:
    """128-byte rendezvous id for ranks that are host threads of this process."""
    buf = C.create_string_buffer(128)
    _check(load().rd_dist_local_id(buf), create=True)
    return buf.raw


def rd_dist_shm_id() -> bytes:
    """128-byte rendezvous id for ranks that are processes of this box, without
    NCCL (a POSIX shared-memory segment carries the control plane)."""
    buf = C.create_string_buffer(128)
    _check(load().rd_dist_shm_id(buf), create=True)
    return buf.raw


def rd_create_dist(width: int, height_global: int, phi_rows: np.ndarray | None, rank: int, world: int, uid: bytes, *,
                   batch: int = 1, dtype=np.float32, tb_depth: int = 0, flags: int = 0, params=None):
    """rd_create_dist (collective): rank's row slab of the global grid.
    phi_rows: host [batch][rows][width] of the OWNED rows (see slab_rows), or
    None for phi = 0."""
    dt = np.dtype(dtype)
    phi = None if phi_rows is None else np.ascontiguousarray(phi_rows, dtype=dt)
    base, extra = divmod(height_global, world)
    rows = base + (1 if rank < extra else 0)
    _check_map(phi, dt, batch * rows * width, "phi_rows (owned rows)")
    if len(uid) != 128:
        raise ValueError("uid must be the 128 bytes of rd_dist_unique_id / rd_dist_local_id / rd_dist_shm_id")
    g = _lib.rd_grid(width, height_global, batch, _DT[dt], tb_depth, flags, 0)
    p = params or rd_params_default()
    h = C.c_void_p()
    _check(load().rd_create_dist(C.byref(g), C.byref(p), _ptr(phi), int(rank), int(world),
                                 C.create_string_buffer(uid, 128), C.byref(h)), create=True)
    return h


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream as an explicit handle


def stream_handle(stream) -> int:
    """cudaStream_t of a torch.cuda.Stream (or an int). torch's default stream
    reports handle 0, which rd_set_stream would read as "the handle's own
    stream": map it to cudaStreamLegacy so the engine really shares it."""
    ptr = int(getattr(stream, "cuda_stream", stream) or 0)
    return ptr if ptr else CUDA_STREAM_LEGACY


def rd_set_stream(h, stream_ptr: int | None) -> None:
    """stream_ptr: a cudaStream_t (int), None = the handle's own stream."""
    _check(load().rd_set_stream(h, C.c_void_p(stream_ptr) if stream_ptr else None), h)


def rd_stimulate(h, b: int, shape: dict, value: float = 1.0, at_step: int = 0) -> None:
    s = _shape(shape)
    _check(load().rd_stimulate(h, b, C.byref(s), float(value), int(at_step)), h)


def rd_step(h, n: int) -> None:
    _check(load().rd_step(h, int(n)), h)


def rd_checkpoint(h) -> None:
    _check(load().rd_checkpoint(h), h)


def rd_step_unchecked(h, n: int) -> None:
    _check(load().rd_step_unchecked(h, int(n)), h)


RD_BLOCK_PUSH = 1


def rd_step_begin(h, k: int, flags: int = 0) -> bool:
    """Open a slab block of k steps and launch its interior rows (they need
    no ghost rows) so they overlap the halo exchange; False: the block is not
    one plain launch -- step it with rd_step_unchecked after the exchange.
    flags=RD_BLOCK_PUSH: the edge bands push their send rows into the
    neighbours' ghost rows (peer memory) instead of a separate exchange."""
    started = C.c_int32(0)
    _check(load().rd_step_begin(h, int(k), int(flags), C.byref(started)), h)
    return bool(started.value)


def rd_plane_origins(h):
    """((u0, u1), (v0, v1), instance stride bytes): this handle's (row 0,
    col 0) device pointers of both buffers."""
    p = [C.c_void_p() for _ in range(4)]
    st = C.c_int64()
    _check(load().rd_plane_origins(h, *[C.byref(x) for x in p], C.byref(st)), h)
    return (p[0].value, p[1].value), (p[2].value, p[3].value), st.value


def rd_set_peer(h, side: int, u, v, rows: int, stride_bytes: int) -> None:
    """Register the slab neighbour above (side 0) / below (side 1) by its
    plane origins (u = (u0, u1), v = (v0, v1)) valid in this process; u=None
    clears."""
    if u is None:
        _check(load().rd_set_peer(h, int(side), None, None, None, None, 0, 0), h)
    else:
        _check(load().rd_set_peer(h, int(side), u[0], u[1], v[0], v[1], int(rows), int(stride_bytes)), h)


def rd_push_ghosts(h) -> None:
    _check(load().rd_push_ghosts(h), h)


def rd_flag_ptr(h, side: int) -> int:
    p = C.c_void_p()
    _check(load().rd_flag_ptr(h, int(side), C.byref(p)), h)
    return p.value


def rd_ipc_export(h):
    """(64-byte cudaIpcMemHandle, this process's base address of the plane allocation)."""
    buf = C.create_string_buffer(64)
    base = C.c_void_p()
    _check(load().rd_ipc_export(h, buf, C.byref(base)), h)
    return buf.raw, base.value


def rd_ipc_map(h, handle64: bytes) -> int:
    """Open a neighbour's exported handle here; returns the mapped base."""
    base = C.c_void_p()
    _check(load().rd_ipc_map(h, C.create_string_buffer(handle64, 64), C.byref(base)), h)
    return base.value


def rd_stream_signal(h, flag_ptr: int, value: int) -> None:
    _check(load().rd_stream_signal(h, flag_ptr, int(value)), h)


def rd_stream_wait(h, flag_ptr: int, value: int) -> None:
    _check(load().rd_stream_wait(h, flag_ptr, int(value)), h)


def rd_step_finish(h) -> None:
    """Close the block opened by rd_step_begin once the exchange has landed:
    edge bands, buffer flip, mirrors, step, probes."""
    _check(load().rd_step_finish(h), h)


def rd_read_flags(h) -> tuple[bool, bool]:
    nf, ie = C.c_int32(), C.c_int32()
    _check(load().rd_read_flags(h, C.byref(nf), C.byref(ie)), h)
    return bool(nf.value), bool(ie.value)


def rd_restore(h) -> None:
    _check(load().rd_restore(h), h)


def rd_get_step(h) -> int:
    return int(load().rd_get_step(h))


def rd_get_fault(h) -> tuple:
    f = _lib.rd_fault()
    _check(load().rd_get_fault(h, C.byref(f)), h)
    return (f.step, f.b, f.i, f.j)


def rd_read_fields(h, b: int, u_out: np.ndarray | None, v_out: np.ndarray | None) -> None:
    _check(load().rd_read_fields(h, b, _host(u_out, h, what="u_out", writable=True),
                                 _host(v_out, h, what="v_out", writable=True)), h)


def rd_write_fields(h, b: int, u: np.ndarray | None, v: np.ndarray | None) -> None:
    _check(load().rd_write_fields(h, b, _host(u, h, what="u"), _host(v, h, what="v")), h)


def rd_write_fields_async(h, b: int, u: np.ndarray | None, v: np.ndarray | None) -> None:
    """Start uploading u, v (pinned host arrays the caller keeps alive until
    rd_commit_fields / rd_io_wait) into the handle's staging block."""
    _check(load().rd_write_fields_async(h, b, _host(u, h, what="u"), _host(v, h, what="v")), h)


def rd_commit_fields(h) -> None:
    _check(load().rd_commit_fields(h), h)


def rd_read_fields_async(h, b: int, u_out: np.ndarray | None, v_out: np.ndarray | None) -> None:
    """Snapshot the fields and start copying them to u_out, v_out (valid after
    rd_io_wait; the caller keeps the arrays alive until then)."""
    _check(load().rd_read_fields_async(h, b, _host(u_out, h, what="u_out", writable=True),
                                       _host(v_out, h, what="v_out", writable=True)), h)


def rd_io_wait(h) -> None:
    _check(load().rd_io_wait(h), h)


def rd_read_fields_device(h, b: int, u_ptr: int | None, v_ptr: int | None) -> None:
    _check(load().rd_read_fields_device(h, b, C.c_void_p(u_ptr) if u_ptr else None,
                                        C.c_void_p(v_ptr) if v_ptr else None), h)


def rd_write_fields_device(h, b: int, u_ptr: int | None, v_ptr: int | None) -> None:
    _check(load().rd_write_fields_device(h, b, C.c_void_p(u_ptr) if u_ptr else None,
                                         C.c_void_p(v_ptr) if v_ptr else None), h)


def rd_probe(h, b: int, rect, threshold: float = 0.1) -> tuple[bool, float]:
    r = _lib.rd_rect(*rect)
    fired, m = C.c_int32(), C.c_double()
    _check(load().rd_probe(h, b, C.byref(r), float(threshold), C.byref(fired), C.byref(m)), h)
    return bool(fired.value), m.value


def rd_probe_latch(h, b: int, rect, threshold: float = 0.1, stride: int = 50) -> int:
    r = _lib.rd_rect(*rect)
    pid = C.c_int32()
    _check(load().rd_probe_latch(h, b, C.byref(r), float(threshold), int(stride), C.byref(pid)), h)
    return pid.value


def rd_probe_result(h, pid: int) -> int:
    out = C.c_int64()
    _check(load().rd_probe_result(h, pid, C.byref(out)), h)
    return out.value


def rd_set_params(h, b: int, params: _lib.rd_params) -> None:
    _check(load().rd_set_params(h, int(b), C.byref(params)), h)


def rd_paint_phi(h, b: int, rect, value: float) -> None:
    r = None if rect is None else C.byref(_lib.rd_rect(*rect))
    _check(load().rd_paint_phi(h, int(b), r, float(value)), h)


def rd_fill_noise(h, b: int = -1, planes: int = 3, seed: int = 1, amplitude: float = 0.1) -> None:
    _check(load().rd_fill_noise(h, int(b), int(planes), int(seed), float(amplitude)), h)


def rd_init_rest(h, b: int = -1) -> None:
    _check(load().rd_init_rest(h, int(b)), h)


def rd_timelapse(h, stride: int) -> None:
    _check(load().rd_timelapse(h, int(stride)), h)


def rd_read_timelapse(h, b: int, out: np.ndarray) -> None:
    _check(load().rd_read_timelapse(h, b, _host(out, h, what="max_u_out", writable=True)), h)


def rd_row_ptr(h, b: int, plane: int, row: int) -> tuple[int, int]:
    p, pitch = C.c_void_p(), C.c_int64()
    _check(load().rd_row_ptr(h, b, plane, row, C.byref(p), C.byref(pitch)), h)
    return p.value, pitch.value


def rd_set_profiling(h, on: bool) -> None:
    _check(load().rd_set_profiling(h, 1 if on else 0), h)


def rd_get_stats(h) -> dict:
    s = _lib.rd_stats()
    _check(load().rd_get_stats(h, C.byref(s)), h)
    return {k: getattr(s, k) for k, _ in s._fields_ if not k.startswith("pad")}


def rd_reset_stats(h) -> None:
    _check(load().rd_reset_stats(h), h)


def rd_last_error(h) -> str:
    return (load().rd_last_error(h) or b"").decode(errors="replace")


# ------------------------------------------------------------- convenience

class Sim:
    """Owning wrapper over an rd_sim handle (one instance batch on one GPU)."""

    def __init__(self, phi: np.ndarray | None = None, *, dtype=np.float32, tb_depth: int = 0, flags: int = 0,
                 params=None, pitch: int = 0, shape: tuple | None = None):
        """phi: host map [B][H][W] (or [H][W]); or phi=None with shape=(B, H, W)
        for phi = 0 on the device (then paint_phi)."""
        if phi is not None:
            phi = np.asarray(phi)
            if phi.ndim == 2:
                phi = phi[None]
            self.B, self.H, self.W = phi.shape
        else:
            self.B, self.H, self.W = shape
        self.dtype = np.dtype(dtype)
        self.h = rd_create(self.W, self.H, phi, batch=self.B, dtype=dtype, tb_depth=tb_depth, flags=flags,
                           params=params, pitch=pitch)

    def close(self):
        if getattr(self, "h", None):
            rd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def stimulate(self, shape: dict, value: float = 1.0, at_step: int = 0, b: int = -1):
        rd_stimulate(self.h, b, shape, value, at_step)

    def step(self, n: int):
        rd_step(self.h, n)

    @property
    def step_count(self) -> int:
        return rd_get_step(self.h)

    def read(self, b: int = 0):
        u = np.empty((self.H, self.W), dtype=self.dtype)
        v = np.empty((self.H, self.W), dtype=self.dtype)
        rd_read_fields(self.h, b, u, v)
        return u, v

    def write(self, b: int, u: np.ndarray | None, v: np.ndarray | None):
        rd_write_fields(self.h, b, None if u is None else np.ascontiguousarray(u, dtype=self.dtype),
                        None if v is None else np.ascontiguousarray(v, dtype=self.dtype))

    def probe(self, b: int, rect, threshold: float = 0.1):
        return rd_probe(self.h, b, rect, threshold)

    def probe_latch(self, b: int, rect, threshold: float = 0.1, stride: int = 50) -> int:
        return rd_probe_latch(self.h, b, rect, threshold, stride)

    def probe_result(self, pid: int) -> int:
        return rd_probe_result(self.h, pid)

    def set_params(self, b: int, params) -> None:
        """Per-instance Eq. 1 parameters (b = -1: all instances)."""
        rd_set_params(self.h, b, params)

    def paint_phi(self, value: float, rect=None, b: int = -1) -> None:
        """phi := value on rect (y0, x0, y1, x1) or the whole grid (None)."""
        rd_paint_phi(self.h, b, rect, value)

    def fill_noise(self, b: int = -1, planes: int = 3, seed: int = 1, amplitude: float = 0.1) -> None:
        """Seeded U[0, amplitude) noise in u/v on the device."""
        rd_fill_noise(self.h, b, planes, seed, amplitude)

    def init_rest(self, b: int = -1) -> None:
        """Quiescent start: u = v = u*(phi) per cell."""
        rd_init_rest(self.h, b)

    def timelapse(self, stride: int) -> None:
        rd_timelapse(self.h, stride)

    def read_timelapse(self, b: int = 0) -> np.ndarray:
        out = np.empty((self.H, self.W), dtype=self.dtype)
        rd_read_timelapse(self.h, b, out)
        return out

    def fault(self):
        return rd_get_fault(self.h)

    def set_stream(self, stream) -> None:
        """Issue work on a torch.cuda.Stream (or raw cudaStream_t int)."""
        rd_set_stream(self.h, stream_handle(stream))

    def stats(self) -> dict:
        return rd_get_stats(self.h)
