"""Kernel-level checks that need a GPU but no oracle: the fast fp32 division
(rdk::div_fast_f32) is bit-identical to IEEE div.rn on the whole input domain
the reaction can produce, for Table-1 q and other q values."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def divcheck(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cuda") / "divcheck")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe,
                    os.path.join(HERE, "cuda", "divcheck.cu")], check=True)
    return exe


@pytest.mark.parametrize("q", ["0.002", "0.5", "1e-12", "0.999"])
def test_fast_division_exhaustive(divcheck, q):
    out = subprocess.run([divcheck, q], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout)
    assert r["tested"] > 4_000_000_000
    assert r["mismatch_guarded"] == 0, r
