import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

from helpers import golden  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (tens of seconds)")


@pytest.fixture(scope="session")
def table1():
    return golden("table1_params.json")


@pytest.fixture(params=["tb", "tb-phimap", "lp", "cr", "gz"])
def kernel(request, monkeypatch):
    """Run a GPU test with each stencil kernel: the register-pipelined
    tb_kernel, the level-parallel lp_kernel, the cluster-resident cr_kernel
    and the whole-chip tiled gz_kernel (RD_KERNEL, read at rd_create; cr / gz
    apply where the instance fits their limits, else the handle falls back to
    tb_kernel). "tb" lets tb_kernel take a one-valued phi map as a kernel
    parameter (its UPHI variants); "tb-phimap" makes it stream the phi plane
    whatever its values (RD_TB_UPHI=0), so both paths see every case."""
    name = request.param
    if name == "tb-phimap":
        monkeypatch.setenv("RD_TB_UPHI", "0")
        name = "tb"
    monkeypatch.setenv("RD_KERNEL", name)
    return name
