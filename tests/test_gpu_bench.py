"""bench.py keeps the driver's contract: one JSON line from a short run, with
every key the round-end driver and the judge read (metric, value, config,
roofline, cpu_baseline, e2e, gpu_launches, clocks, ...), and the reference
arm's line (impl = reference, the oracle on the host cores)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    d = _line(["--timesteps", "20", "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--cpu-seconds", "1",
               "--e2e-pipeline-steps", "3"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["vs_baseline"] is None and d["dtype"] == "f32"
    assert "workload" in d["config"] and "configs[3]" in d["config"]["workload"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("alu", "hbm", "tensor") and 0 < r["frac"] and r["achieved"] > 0 and r["peak"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] >= 1 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["pipeline"] == 2 and e["steps"] == 3 and e["serial"]["value"] > 0 and e["serial"]["steps"] == 1
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=900)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "configs[3]" in d["config"]["workload"]


def test_bench_two_ranks_under_torchrun():
    """The driver's N > 1 launch (torchrun, one process per rank) of the
    weak-scaling line: 16384 rows per rank, row slabs with halo exchange.
    Both ranks share this box's one GPU, so the exchange runs over gloo
    (host-staged halos; RD_BENCH_BACKEND) -- a functional check of the
    N > 1 code path and its JSON line, not a measurement."""
    env = dict(os.environ, RD_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--timesteps", "8", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["steps"] == 3
    assert "configs[4]" in d["config"]["workload"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
