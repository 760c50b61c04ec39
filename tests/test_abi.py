"""The C-ABI library (no GPU needed): it loads, exports every symbol
include/rd.h declares, matches the Python declarations, and validates
arguments before touching the device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1901_06535_b200 as rd
from paper_1901_06535_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rd.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rd_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rd_\w+)", out))
    for n in names:
        assert n in exported, n
        assert getattr(lib, n) is not None
    assert sorted(n for n, _, _ in _lib.SYMBOLS) == names


def test_struct_layouts_match_header():
    """Sizes of the ABI structs as a C compiler lays them out."""
    code = r'''
#include <stdio.h>
#include "rd.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(rd_params), sizeof(rd_grid), sizeof(rd_shape),
 sizeof(rd_rect), sizeof(rd_fault), sizeof(rd_stats), sizeof(rd_geometry));return 0;}
'''
    exe = "/tmp/rd_sizes"
    subprocess.run(["gcc", "-x", "c", "-I", os.path.join(ROOT, "include"), "-o", exe, "-"], input=code, text=True,
                   check=True)
    sizes = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    ours = [C.sizeof(t) for t in (_lib.rd_params, _lib.rd_grid, _lib.rd_shape, _lib.rd_rect, _lib.rd_fault,
                                  _lib.rd_stats, _lib.rd_geometry)]
    assert sizes == ours


def test_abi_version_and_defaults(table1):
    assert _lib.load().rd_abi_version() == 2
    p = rd.rd_params_default()
    for k in ("eps", "f", "q", "Du", "dt", "dx"):
        assert getattr(p, k) == table1[k]


@pytest.mark.parametrize("field,value", [("eps", 0.0), ("q", 1.5), ("dt", -1.0), ("dt", 0.04), ("f", float("nan"))])
def test_param_validation_before_device(field, value):
    """SPEC.md:28 invariants are rejected with RD_EPARAM (no device needed);
    dt=0.04 violates dt*Du/dx^2 < 0.25."""
    p = rd.rd_params_default()
    setattr(p, field, value)
    with pytest.raises(rd.RDError) as e:
        rd.rd_create(8, 8, np.zeros((8, 8), np.float32), params=p)
    assert e.value.code == _lib.RD_EPARAM


def test_dims_validation_before_device():
    with pytest.raises(rd.RDError) as e:
        rd.rd_create(2, 8, np.zeros((8, 2), np.float32))
    assert e.value.code == _lib.RD_EINVAL
    with pytest.raises(rd.RDError) as e:
        rd.rd_create(8, 8, np.zeros((8, 8), np.float32), tb_depth=99)
    assert e.value.code == _lib.RD_EINVAL


def test_no_cpu_fallback(monkeypatch, tmp_path):
    """The product path fails loudly when the CUDA extension is missing."""
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="not built"):
        _lib.load(str(tmp_path / "missing.so"))


def test_dist_and_device_calls_validate_before_device():
    """The multi-GPU and caller-memory calls reject bad arguments without a
    device: an unknown in-process id, a rank outside the world, a NULL arena;
    rd_arena_bytes needs no device at all; the in-process id is tagged."""
    uid = rd.rd_dist_local_id()
    assert uid[:8] == b"RDLOCAL1" and len(uid) == 128
    bogus = b"RDLOCAL1" + b"\xff" * 8 + bytes(112)
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_dist(64, 64, None, 0, 2, bogus)
    assert e.value.code == _lib.RD_EINVAL
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_dist(64, 64, None, 3, 2, uid)
    assert e.value.code == _lib.RD_EINVAL
    with pytest.raises(ValueError):
        rd.rd_create_dist(64, 64, np.zeros((10, 64), np.float32), 0, 2, uid)  # not the 32 owned rows
    n = rd.rd_arena_bytes(100, 50, dtype=np.float32)
    pitch = (8 + 100 + 8 + 16 + 31) // 32 * 32
    assert n == 7 * (50 + 2 * (8 + 24)) * pitch * 4 + 256
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_device(100, 50, 0, n, None)
    assert e.value.code == _lib.RD_EINVAL


def test_shm_id_names_a_segment_of_this_box():
    """rd_dist_shm_id creates the POSIX shared-memory segment its 128 bytes
    name (the control plane of one-box process groups, no NCCL); a world
    larger than a segment holds is refused before any device work."""
    import os
    import struct
    uid = rd.rd_dist_shm_id()
    assert uid[:8] == b"RDSHM001" and len(uid) == 128
    name = lambda u: "/dev/shm/rd_dist_%016x" % struct.unpack("<Q", u[8:16])[0]  # noqa: E731
    path = name(uid)
    try:
        assert os.path.exists(path) and os.path.getsize(path) > 64 * 256
        other = rd.rd_dist_shm_id()
        os.unlink(name(other))
        assert other[8:16] != uid[8:16]
        with pytest.raises(rd.RDError) as e:
            rd.rd_create_dist(64, 1024, None, 0, 65, uid)
        assert e.value.code == _lib.RD_EINVAL
    finally:
        os.unlink(path)
