"""ctypes declarations of include/rd.h (argument marshalling only).

Every compute step runs in librd.so's CUDA kernels. There is no CPU fallback:
if the extension is missing this module raises on first use.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librd.so")

RD_OK, RD_EINVAL, RD_EPARAM, RD_ERANGE, RD_ENONFINITE, RD_ECUDA, RD_ENCCL, RD_ENOMEM = 0, -1, -2, -3, -4, -5, -6, -7
RD_F32, RD_F64 = 1, 2
RD_REACTION_OFF, RD_NO_CHECKPOINT, RD_NO_GRAPH = 1, 2, 4
RD_DISC, RD_RECT, RD_HALF_DISC = 1, 2, 3
RD_SHAPE_MASK_PHI = 1
RD_MAX_TB = 8
RD_TRANSPORT_NONE, RD_TRANSPORT_P2P, RD_TRANSPORT_NCCL, RD_TRANSPORT_LOCAL = 0, 1, 2, 3
TRANSPORTS = {0: "none", 1: "p2p", 2: "nccl", 3: "local"}

ERRNAMES = {0: "RD_OK", -1: "RD_EINVAL", -2: "RD_EPARAM", -3: "RD_ERANGE", -4: "RD_ENONFINITE",
            -5: "RD_ECUDA", -6: "RD_ENCCL", -7: "RD_ENOMEM"}


class rd_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("eps", "f", "q", "Du", "dt", "dx")]


class rd_grid(C.Structure):
    _fields_ = [("width", C.c_int64), ("height", C.c_int64), ("batch", C.c_int32), ("dtype", C.c_int32),
                ("tb_depth", C.c_int32), ("flags", C.c_uint32), ("pitch", C.c_int64)]


class rd_shape(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dir", C.c_int32), ("cy2", C.c_int64), ("cx2", C.c_int64),
                ("r", C.c_int64), ("y0", C.c_int64), ("x0", C.c_int64), ("y1", C.c_int64), ("x1", C.c_int64),
                ("flags", C.c_uint32), ("reserved", C.c_uint32), ("mask_phi", C.c_double)]


class rd_rect(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("y0", "x0", "y1", "x1")]


class rd_fault(C.Structure):
    _fields_ = [("step", C.c_int64), ("b", C.c_int32), ("pad", C.c_int32), ("i", C.c_int64), ("j", C.c_int64)]


class rd_stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("step_launches", C.c_int64), ("cell_updates", C.c_int64),
                ("step_kernel_ms", C.c_double), ("timed_launches", C.c_int64), ("tb_depth", C.c_int32),
                ("phi_uniform", C.c_int32), ("replays", C.c_int64), ("arith_mode", C.c_int32), ("kernel", C.c_int32)]


class rd_geometry(C.Structure):
    _fields_ = [("width", C.c_int64), ("height", C.c_int64), ("height_global", C.c_int64), ("row0", C.c_int64),
                ("pitch", C.c_int64), ("phi_rows_lo", C.c_int64), ("phi_rows_hi", C.c_int64),
                ("exchanges", C.c_int64), ("batch", C.c_int32), ("dtype", C.c_int32), ("halo", C.c_int32),
                ("tb_depth", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("transport", C.c_int32),
                ("flag_selftest", C.c_int32)]


# (name, restype, argtypes) of every symbol include/rd.h declares
P, i32, i64, u32, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
SYMBOLS = [
    ("rd_abi_version", C.c_int32, []),
    ("rd_params_default", None, [C.POINTER(rd_params)]),
    ("rd_create", C.c_int, [C.POINTER(rd_grid), C.POINTER(rd_params), P, C.POINTER(P)]),
    ("rd_create_slab", C.c_int, [C.POINTER(rd_grid), C.POINTER(rd_params), P, i64, i64, i32, C.POINTER(P)]),
    ("rd_destroy", C.c_int, [P]),
    ("rd_arena_bytes", C.c_int, [C.POINTER(rd_grid), C.POINTER(C.c_size_t)]),
    ("rd_create_device", C.c_int, [C.POINTER(rd_grid), C.POINTER(rd_params), P, C.c_size_t, P, C.POINTER(P)]),
    ("rd_field_ptr", C.c_int, [P, i32, i32, C.POINTER(P), C.POINTER(i64)]),
    ("rd_get_geometry", C.c_int, [P, C.POINTER(rd_geometry)]),
    ("rd_dist_unique_id", C.c_int, [P]),
    ("rd_dist_local_id", C.c_int, [P]),
    ("rd_dist_shm_id", C.c_int, [P]),
    ("rd_create_dist", C.c_int, [C.POINTER(rd_grid), C.POINTER(rd_params), P, i32, i32, P, C.POINTER(P)]),
    ("rd_set_stream", C.c_int, [P, P]),
    ("rd_write_fields", C.c_int, [P, i32, P, P]),
    ("rd_read_fields", C.c_int, [P, i32, P, P]),
    ("rd_read_fields_device", C.c_int, [P, i32, P, P]),
    ("rd_write_fields_device", C.c_int, [P, i32, P, P]),
    ("rd_write_fields_async", C.c_int, [P, i32, P, P]),
    ("rd_commit_fields", C.c_int, [P]),
    ("rd_read_fields_async", C.c_int, [P, i32, P, P]),
    ("rd_io_wait", C.c_int, [P]),
    ("rd_stimulate", C.c_int, [P, i32, C.POINTER(rd_shape), dbl, i64]),
    ("rd_step", C.c_int, [P, i64]),
    ("rd_checkpoint", C.c_int, [P]),
    ("rd_step_unchecked", C.c_int, [P, i64]),
    ("rd_step_begin", C.c_int, [P, i64, i32, C.POINTER(i32)]),
    ("rd_step_finish", C.c_int, [P]),
    ("rd_plane_origins", C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(i64)]),
    ("rd_set_peer", C.c_int, [P, i32, P, P, P, P, i64, i64]),
    ("rd_push_ghosts", C.c_int, [P]),
    ("rd_flag_ptr", C.c_int, [P, i32, C.POINTER(P)]),
    ("rd_ipc_export", C.c_int, [P, P, C.POINTER(P)]),
    ("rd_ipc_map", C.c_int, [P, P, C.POINTER(P)]),
    ("rd_stream_signal", C.c_int, [P, P, u32]),
    ("rd_stream_wait", C.c_int, [P, P, u32]),
    ("rd_read_flags", C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("rd_restore", C.c_int, [P]),
    ("rd_get_step", C.c_int64, [P]),
    ("rd_get_fault", C.c_int, [P, C.POINTER(rd_fault)]),
    ("rd_probe", C.c_int, [P, i32, C.POINTER(rd_rect), dbl, C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("rd_probe_latch", C.c_int, [P, i32, C.POINTER(rd_rect), dbl, i32, C.POINTER(C.c_int32)]),
    ("rd_probe_result", C.c_int, [P, i32, C.POINTER(C.c_int64)]),
    ("rd_set_params", C.c_int, [P, i32, C.POINTER(rd_params)]),
    ("rd_init_rest", C.c_int, [P, i32]),
    ("rd_fill_noise", C.c_int, [P, i32, C.c_uint32, C.c_uint64, dbl]),
    ("rd_paint_phi", C.c_int, [P, i32, C.POINTER(rd_rect), dbl]),
    ("rd_timelapse", C.c_int, [P, i32]),
    ("rd_read_timelapse", C.c_int, [P, i32, P]),
    ("rd_row_ptr", C.c_int, [P, i32, i32, i64, C.POINTER(P), C.POINTER(C.c_int64)]),
    ("rd_set_profiling", C.c_int, [P, i32]),
    ("rd_get_stats", C.c_int, [P, C.POINTER(rd_stats)]),
    ("rd_reset_stats", C.c_int, [P]),
    ("rd_last_error", C.c_char_p, [P]),
    ("rd_create_error", C.c_char_p, []),
]

_lib = None


def _nccl_hint() -> None:
    """Point librd's run-time NCCL lookup (RD_NCCL_LIB) at the copy torch
    links against, if the environment ships one: librd opens NCCL only for
    rd_create_dist, and a process can hold one libnccl.so.2, so it must be
    the one a later `import torch` expects."""
    if os.environ.get("RD_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for d in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(d, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["RD_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def load(path: str | None = None):
    """dlopen librd.so and declare every rd.h symbol. Raises if it is missing."""
    global _lib
    _nccl_hint()
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"CUDA extension {p} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, res, args in SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
