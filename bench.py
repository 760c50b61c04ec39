#!/usr/bin/env python
"""Benchmark of the Oregonator forward-Euler hot path (BASELINE.json metric:
"Gcell-updates/s and % of B200 HBM roofline at 1/2/4/8 GPUs").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One bench "step" = rd_step(T) with T = --timesteps (default 1000) time steps of
the whole hot path (a1-a8: due stimuli, K-step blocked stencil launches, the
non-finite health check, probe latches) over the workload:
  N = 1: configs[3] "c4_roofline" 16384 x 16384 fp32, noise + 64 half-discs;
         K = 10 x 1000 = the config's 10000 timed steps. The line also carries
         per_config (configs[0..2] in fp32 and fp64: rate, kernel, probe
         outcomes vs the paper's, the oracle's rate) and fp32_error (R-17).
  N > 1: configs[4] weak scaling, a 16384-row slab per GPU of a
         (16384 N) x 16384 grid with 16 N obstacles, each rank an
         rd_create_dist handle (halo exchange inside librd); beside it
         "strong": configs[4] at 65536 x 65536 split over the N GPUs.
Inputs (5 planes x 1 GiB per GPU) are far larger than L2 (126 MB), so no
flush is needed between steps. Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gcell-updates/s and % of B200 HBM roofline at 1/2/4/8 GPUs"
UNIT = "Gcell-updates/s"
BYTES_PER_CELL = {np.dtype(np.float32): 20, np.dtype(np.float64): 40}  # read u,v,phi + write u,v


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ALU roofline of the temporally blocked kernel: the canonical
# tree is 13 add/sub + 9 mul + 1 div = 23 fp32 operations per cell-update
# (R-8); the FP32 pipe peak is 148 SMs x 128 lanes x clocks.max.sm, one
# operation per lane per cycle (B200_PROFILING.md: 148 SMs, 1965 MHz).
OPS_PER_CELL = 23
FP32_LANES = 148 * 128


def alu_peak_tops():
    mhz, src = 1965.0, "B200_PROFILING.md clocks.max.sm"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mhz, src = float(json.load(fh)["sm_max_mhz"]), "MEASURED_PEAKS.json sm_max_mhz"
    except Exception:
        pass
    return FP32_LANES * mhz * 1e6 / 1e12, f"derived: 148 SMs x 128 FP32 lanes x {mhz:.0f} MHz ({src})"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(world: int, T: int, tb_depth: int, scaling: str = "weak", strong_grid: int = 65536) -> dict:
    """The `config` of the JSON line -- the same for our arm and the
    reference arm (BASELINE.json configs[3] at N = 1,
    configs[4] weak scaling at N > 1; --scaling strong: configs[4] at its full
    65536 x 65536 over N GPUs)."""
    if scaling == "strong":
        G = strong_grid
        d = {"workload": f"configs[4] strong scaling: {G}x{G} fp32 row slabs over N GPUs (rd_create_dist), "
                         "256 obstacles phi=0.2 per 65536^2, masked half-discs", "grid": [G, G]}
        return dict(d, time_steps_per_step=T, tb_depth=tb_depth,
                    l2=f"inputs larger than L2 (5 planes of {G * G * 4 / 1e9:.1f}/N GB per GPU); no flush needed",
                    parallelism=f"row slabs x{world}")
    if world == 1:
        d = {"workload": "configs[3] c4_roofline: 16384x16384 fp32, phi=0.054, u,v~U[0,0.1) seed 1, "
                         "64 half-discs r=8 seed 2, no-flux", "grid": [16384, 16384]}
    else:
        d = {"workload": f"configs[4] weak scaling: ({16384 * world})x16384 fp32 row slabs (rd_create_dist), "
                         "16 obstacles/GPU phi=0.2, masked half-discs", "grid": [16384 * world, 16384]}
    return dict(d, time_steps_per_step=T, tb_depth=tb_depth,
                l2="inputs larger than L2 (5 x 1 GiB planes per GPU); no flush needed",
                parallelism=f"row slabs x{world}" if world > 1 else "single GPU")


def host_cores() -> int:
    """Host cores this process may run on (the oracle's OpenMP threads)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def max_over_ranks(x: float, world: int) -> float:
    """Device-timed milliseconds -> max over ranks (all_reduce MAX)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------- rank context

class ProcCtx:
    """One process per GPU (the driver's torchrun launch): torch.distributed
    for the rendezvous id, barriers and the max over ranks -- never for the
    halo data, which librd moves itself (rd_create_dist)."""

    def __init__(self, world, rank, local):
        self.world, self.rank, self.local, self.functional = world, rank, local, False

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    def max(self, x: float) -> float:
        return max_over_ranks(x, self.world)

    def uid(self) -> bytes:
        from paper_1901_06535_b200.dist import shm_id, unique_id
        if os.environ.get("RD_BENCH_SHM") == "1" and self.world > 1:
            # one-box process group without NCCL (rd_dist_shm_id): ranks may share a GPU
            import torch.distributed as dist
            obj = [shm_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            return obj[0]
        return unique_id()


class ThreadCtx:
    """RD_BENCH_THREADS=1: the N ranks as host threads of ONE process on one
    GPU (rd_dist_local_id) -- a functional check of the N > 1 code path and
    its JSON line on a one-GPU box, not a measurement (the ranks share SMs)."""

    def __init__(self, world, rank, shared):
        self.world, self.rank, self.local, self.functional = world, rank, 0, True
        self.shared = shared

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        self.shared["barrier"].wait()
        torch.cuda.synchronize()

    def max(self, x: float) -> float:
        sh = self.shared
        sh["vals"][self.rank] = x
        sh["barrier"].wait()
        m = max(sh["vals"])
        sh["barrier"].wait()
        return m

    def uid(self) -> bytes:
        import paper_1901_06535_b200 as rd
        if self.rank == 0:
            self.shared["uid"] = rd.rd_dist_local_id()
        self.shared["barrier"].wait()
        u = self.shared["uid"]
        self.shared["barrier"].wait()
        return u


# ------------------------------------------------------------- our arm

def e2e_pipelined(rd, sim, pu, pv, T, steps, cells):
    """e2e on ONE handle from ONE host thread with the library's asynchronous
    host I/O (include/rd.h: rd_write_fields_async / rd_commit_fields /
    rd_read_fields_async / rd_io_wait). Every step is a job: its inputs are
    copied in from pinned host memory and its result out to pinned host
    memory, inside the timed region; job i+1's upload and job i-1's download
    run on the copy engines while job i's stencil launches own the SMs (the
    first upload and the last download are exposed). Timed on the host clock
    between two device synchronisations."""
    import torch
    h = sim.h
    rd.rd_set_stream(h, 0)  # back to the handle's own stream
    outs = [(torch.empty(pu.shape, dtype=torch.float32, pin_memory=True).numpy(),
             torch.empty(pu.shape, dtype=torch.float32, pin_memory=True).numpy()) for _ in range(2)]
    # untimed: allocate the staging blocks, touch every buffer once
    rd.rd_write_fields_async(h, 0, pu, pv)
    rd.rd_commit_fields(h)
    rd.rd_read_fields_async(h, 0, *outs[0])
    rd.rd_read_fields_async(h, 0, *outs[1])
    rd.rd_io_wait(h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rd.rd_write_fields_async(h, 0, pu, pv)
    rd.rd_commit_fields(h)
    for i in range(steps):
        if i + 1 < steps:
            rd.rd_write_fields_async(h, 0, pu, pv)  # the next job's inputs, under this job's steps
        sim.step(T)
        rd.rd_read_fields_async(h, 0, *outs[i % 2])  # snapshot, drained under the next job's steps
        if i + 1 < steps:
            rd.rd_commit_fields(h)
    rd.rd_io_wait(h)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    return {"value": cells * T * steps / secs / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 2 * cells * 4, "d2h_bytes_per_step": 2 * cells * 4, "steps": steps,
            "pipeline": 2, "timer": "host clock between device synchronisations",
            "api": "one handle, one host thread: rd_write_fields_async(host pinned) of the next job + rd_step + "
                   "rd_read_fields_async(host pinned) + rd_commit_fields, every step; rd_io_wait at the end"}


def load_traffic(workload: str, kernel: str, cells_per_launch: float):
    """DRAM bytes per launch of `kernel` on `workload` from a committed ncu
    --set full capture (profiles/traffic_rNN.json) -- only if the capture is
    of this very workload, kernel and launch size (its cell-update count
    stored beside it); else None."""
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")), reverse=True):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        for e in d.get("entries", []):
            # the same launch size within 1%: a 1000-step segment at depth 6 is cut into 165 launches
            # of 6 steps and 2 of 5 (5.99 on average); the capture is of a 6-step launch
            if (e.get("workload") == workload and e.get("kernel") == kernel
                    and abs(e.get("cell_updates_per_launch", -1) - cells_per_launch) <= 0.01 * cells_per_launch):
                return e["dram_bytes_per_launch"], (f"{os.path.relpath(f, ROOT)} (a launch of "
                                                    f"{e['cell_updates_per_launch']:.0f} cell-updates)")
    return None, None


def roofline_of(st, ms, workload_tag, dtype):
    """ALU roofline of the dominant kernel with the one-step
    HBM view beside it, from the stencil launches' summed CUDA-event times
    inside the timed region (rd_set_profiling)."""
    hbm, hbm_src = peaks()
    kms = st["step_kernel_ms"]
    k_launches = max(1, st["timed_launches"])
    bpc = BYTES_PER_CELL[dtype]
    achieved = bpc * st["cell_updates"] / (kms / 1e3) / 1e9 if kms > 0 else None
    alu, alu_src = alu_peak_tops()
    ops = OPS_PER_CELL * st["cell_updates"] / (kms / 1e3) / 1e12 if kms > 0 else None
    # the handle found phi to be one value: tb_kernel takes it as a parameter (its UPHI variants)
    kernel = f"tb_kernel<float,K={st['tb_depth']}{',uphi' if st.get('phi_uniform') else ''}>"
    cpl = st["cell_updates"] / k_launches
    traffic, tsrc = load_traffic(workload_tag, kernel, cpl)
    return {"bound": "alu", "achieved": ops, "peak": alu, "unit": "TFLOP/s",
            "frac": (ops / alu) if ops else None, "traffic": traffic,
            "traffic_source": tsrc or "no ncu capture of this workload/kernel/launch size: null",
            "kernel": kernel, "peak_source": alu_src,
            "algorithmic_ops_per_cell_update": OPS_PER_CELL,
            "ops": "fp32 add/sub/mul/div of the canonical Eq.-1 tree (13 + 9 + 1), R-8",
            "cell_updates_per_launch": cpl, "avg_launch_ms": kms / k_launches,
            "kernel_share_of_step": kms / ms if ms else None,
            "hbm_view": {"achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if achieved else None, "peak_source": hbm_src,
                         "algorithmic_bytes_per_cell_update": bpc, "one_step_roofline_gcells": hbm / bpc,
                         "note": ("SURVEY 8(d)'s 20 B per cell-update (read u, v, phi; write u, v); this workload's "
                                  "phi is one value, which the kernel takes as a parameter (16 B)"
                                  if st.get("phi_uniform") else None)}}


def timed(ctx, stepper, h, T, steps, warmup, clocks_index):
    """W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
    events on the engine's stream (torch's current), clocks sampled during
    the timed region. Returns (device ms of this rank, stats, clocks)."""
    import torch
    import paper_1901_06535_b200 as rd
    stream = torch.cuda.current_stream()
    rd.rd_set_stream(h, rd.stream_handle(stream))
    for _ in range(warmup):
        stepper(T)
    ctx.barrier()
    rd.rd_reset_stats(h)
    rd.rd_set_profiling(h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(clocks_index) if ctx.rank == 0 else None
    if clk:
        clk.__enter__()
    try:
        ctx.barrier()
        e0.record(stream)
        for _ in range(steps):
            stepper(T)
        e1.record(stream)
        ctx.barrier()
    finally:
        if clk:
            clk.__exit__()
    ms = e0.elapsed_time(e1)
    st = rd.rd_get_stats(h)
    rd.rd_set_profiling(h, False)
    return ms, st, (clk.summary() if clk else None)


def per_config(cpu_seconds: float):
    """configs[0..2] -- the 128^2 disc, the AND-gate batch and the diode batch
    (§4) -- in fp32 and fp64 through rd_step, each run in
    full (second of two runs: the first warms module loads and clocks): device
    time, Gcell/s, the stencil kernel, the probe outcomes against the paper's
    (rdinputs expect), and the oracle's own rate on the host cores on a
    bounded sample of the same instance (cpu_baseline)."""
    import torch
    import paper_1901_06535_b200 as rd
    from rdinputs import config
    out = []
    for n in (1, 2, 3):
        for dt in (np.float32, np.float64):
            w = config(n, dtype=dt)
            phi = np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)])
            for rep in range(2):
                sim = rd.Sim(phi, dtype=dt)
                for b in range(w.B):
                    for shape, val, at in w.events[b]:
                        sim.stimulate(shape, val, at, b=b)
                pids = ([[sim.probe_latch(b, r, t, s) for (r, t, s) in w.probes[b]] for b in range(w.B)]
                        if w.probes else [])
                stream = torch.cuda.current_stream()
                sim.set_stream(stream)
                rd.rd_reset_stats(sim.h)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                sim.step(w.steps)
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                st = sim.stats()
                fires = [[sim.probe_result(p) for p in ps] for ps in pids]
                sim.close()
            cells = w.B * w.H * w.W * w.steps
            got = [any(f >= 0 for f in fs) for fs in fires] if fires else None
            exp = w.expect.get("fires")
            e = {"config": f"configs[{n - 1}] {w.name}", "dtype": np.dtype(dt).name, "batch": w.B,
                 "grid": [w.H, w.W], "time_steps": w.steps, "device_ms": ms,
                 "gcell_updates_per_s": cells / (ms / 1e3) / 1e9,
                 "stencil_kernel": ["tb_kernel", "lp_kernel", "cr_kernel", "gz_kernel"][st["kernel"]],
                 "kernel_launches": st["launches"], "first_fire": fires, "fires": got, "expected_fires": exp,
                 "outcome_ok": (got == exp) if exp is not None else None}
            if cpu_seconds > 0:
                e["cpu_baseline"] = oracle_rate(w, dt, cpu_seconds)
            out.append(e)
    return out


def oracle_rate(w, dt, seconds: float):
    """The oracle (as it stands, on all host cores) on instance 0 of w for a
    bounded number of its steps."""
    import oracle
    oracle.set_num_threads(host_cores())
    u0, v0 = w.init_planes(0)
    phi = w.phi_plane(0).astype(dt)
    t = time.perf_counter()
    oracle.run(u0.astype(dt), v0.astype(dt), phi, 20, events=w.events[0])
    t1 = (time.perf_counter() - t) / 20
    n = int(max(20, min(w.steps, seconds / max(t1, 1e-6))))
    t = time.perf_counter()
    oracle.run(u0.astype(dt), v0.astype(dt), phi, n, events=w.events[0])
    el = time.perf_counter() - t
    return {"value": w.H * w.W * n / el / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"instance 0, first {n} of {w.steps} time steps"}


def config4_fp64(T: int = 200):
    """configs[3]'s grid and inputs in fp64 (north_star: the stencil kernel "in
    fp32 and fp64"): T time steps of rd_step, device-timed after one warm-up
    call, with the one-step HBM roofline (40 B per cell-update) beside it."""
    import torch
    import paper_1901_06535_b200 as rd
    from rdinputs import config
    w = config(4)
    dt = np.dtype(np.float64)
    with rd.Sim(None, shape=(1, w.H, w.W), dtype=dt) as sim:
        sim.paint_phi(0.054)
        sim.fill_noise(seed=1)
        for shape, val, at in w.events[0]:
            sim.stimulate(shape, val, at)
        stream = torch.cuda.current_stream()
        sim.set_stream(stream)
        sim.step(T)
        rd.rd_reset_stats(sim.h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        sim.step(T)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = sim.stats()
    hbm, _ = peaks()
    g = w.H * w.W * T / (ms / 1e3) / 1e9
    return {"config": "configs[3] c4_roofline grid and inputs, fp64", "dtype": "float64", "grid": [w.H, w.W],
            "time_steps": T, "device_ms": ms, "gcell_updates_per_s": g, "tb_depth": st["tb_depth"],
            "stencil_kernel": ["tb_kernel", "lp_kernel", "cr_kernel", "gz_kernel"][st["kernel"]],
            "frac_of_one_step_hbm_roofline": g / (hbm / BYTES_PER_CELL[dt])}


def fp32_error():
    """BASELINE.json north_star's literal fp32 check, reported (reading R-17):
    max |u_fp32 - u_fp64| on config 1 after 300 and 1000 steps, both computed
    by this engine (its fp64 path equals the fp64 oracle bitwise; its fp32
    path the oracle's fp32 mode)."""
    import paper_1901_06535_b200 as rd
    from rdinputs import config
    res = {}
    for steps in (300, 1000):
        f = {}
        for dt in (np.float32, np.float64):
            w = config(1, dtype=dt)
            with rd.Sim(w.phi_plane(0).astype(dt)[None], dtype=dt) as sim:
                for shape, val, at in w.events[0]:
                    sim.stimulate(shape, val, at)
                sim.step(steps)
                f[dt] = sim.read(0)
        du = np.abs(f[np.float32][0].astype(np.float64) - f[np.float64][0])
        dv = np.abs(f[np.float32][1].astype(np.float64) - f[np.float64][1])
        res[f"step{steps}"] = {"max_abs_du": float(du.max()), "max_abs_dv": float(dv.max()),
                               "cells_over_2e-3": int(np.count_nonzero(np.maximum(du, dv) > 2e-3))}
    res.update(tolerance=2e-3, config="configs[0] 128x128 disc",
               reading="DESIGN.md R-17: gated bitwise against the oracle's fp32 mode and <= 2e-3 vs fp64 up to "
                       "step 300; the step-1000 gap is the refractory wake amplifying rounding, reported not gated")
    return res


def run_single(args):
    """N = 1: configs[3] (16384^2 fp32) -- the metric's own configuration."""
    import torch
    import paper_1901_06535_b200 as rd
    from rdinputs import config
    ctx = ProcCtx(1, 0, 0)
    dtype = np.dtype(np.float32)
    T = args.timesteps
    w = config(4)
    H, W = w.H, w.W
    # inputs built on the device: phi = 0.054, seeded U[0,0.1) noise
    # (rd_fill_noise == rdinputs.noise_plane bitwise), 64 half-discs
    sim = rd.Sim(None, shape=(1, H, W), dtype=dtype, tb_depth=args.tb)
    h = sim.h
    sim.paint_phi(0.054)
    sim.fill_noise(seed=1)
    u0, v0 = sim.read(0)  # host copies for the e2e leg and the CPU baseline
    phi = np.full((H, W), 0.054, dtype=dtype)
    for shape, val, at in w.events[0]:
        sim.stimulate(shape, val, at)
    cells = H * W
    ms, st, clk = timed(ctx, sim.step, h, T, args.steps, args.warmup, 0)
    value = cells * T * args.steps / (ms / 1e3) / 1e9
    roofline = roofline_of(st, ms, "c4_roofline", dtype)
    stream = torch.cuda.current_stream()

    # e2e through the public API with pinned host buffers: every step writes
    # u, v from the host, steps, and reads u, v back
    e2e = None
    if args.e2e_steps > 0:
        pu = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy()
        pv = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy()
        pu[...] = u0
        pv[...] = v0
        ou = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy()
        ov = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy()
        ctx.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            rd.rd_write_fields(h, 0, pu, pv)
            sim.step(T)
            rd.rd_read_fields(h, 0, ou, ov)
        b.record(stream)
        ctx.barrier()
        ems = a.elapsed_time(b)
        e2e = {"value": cells * T * args.e2e_steps / (ems / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * cells * 4, "d2h_bytes_per_step": 2 * cells * 4,
               "steps": args.e2e_steps, "api": "rd_write_fields(host pinned) + rd_step + rd_read_fields(host)"}
        if args.e2e_pipeline > 1:
            serial = e2e
            e2e = e2e_pipelined(rd, sim, pu, pv, T, args.e2e_pipeline_steps, cells)
            e2e["serial"] = {"value": serial["value"], "steps": serial["steps"], "api": serial["api"]}
    launches = st["launches"]
    # config 4's phi is one value, which tb_kernel takes as a kernel parameter
    # (rd_stats.phi_uniform); beside the line's value goes the rate of the
    # general kernel that streams the phi plane (maps with more than one
    # value: config 5, the circuits), on the same handle: RD_TB_UPHI=0 and a
    # repaint make the handle re-derive its choice
    streamed = None
    if st.get("phi_uniform"):
        rd.rd_set_stream(h, rd.stream_handle(stream))
        os.environ["RD_TB_UPHI"] = "0"
        try:
            sim.paint_phi(0.054)
            sms, sst, sclk = timed(ctx, sim.step, h, T, max(2, args.steps // 3), 1, 0)
            streamed = {"value": cells * T * max(2, args.steps // 3) / (sms / 1e3) / 1e9, "unit": UNIT,
                        "phi_uniform": sst.get("phi_uniform"), "sm_mhz": (sclk or {}).get("sm_mhz"),
                        "avg_launch_ms": sst["step_kernel_ms"] / max(1, sst["timed_launches"]),
                        "what": "the same workload with tb_kernel streaming the phi plane (RD_TB_UPHI=0)"}
        finally:
            os.environ.pop("RD_TB_UPHI", None)
    sim.close()
    cpu = None if args.no_cpu_baseline else cpu_baseline(u0, v0, phi, args.cpu_seconds)
    hbm, _ = peaks()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(1, T, st["tb_depth"]),
            "frac_of_one_step_hbm_roofline": value / (hbm / BYTES_PER_CELL[dtype]),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "phi_uniform": bool(st.get("phi_uniform")), "phi_streamed": streamed}
    if not args.no_configs:
        line["per_config"] = per_config(0 if args.no_cpu_baseline else args.config_cpu_seconds)
        line["fp32_error"] = fp32_error()
        line["fp64_large"] = config4_fp64()
    return line


def dist_run(args, ctx, strong: bool):
    """One N > 1 line: configs[4] weak (16384 rows per GPU) or strong (the
    --strong-grid^2 grid, 65536^2 by default, split over the ranks), each rank
    an rd_create_dist slab; rd_step runs the whole distributed super-step in
    librd. Returns this rank's timing and stats."""
    import torch
    import paper_1901_06535_b200 as rd
    from paper_1901_06535_b200.dist import DistSim
    from rdinputs import config
    world, rank = ctx.world, ctx.rank
    dtype = np.dtype(np.float32)
    T = args.strong_timesteps if strong else args.timesteps
    if strong:
        G = args.strong_grid
        w = config(5, H=G, W=G, n_obstacles=max(1, 256 * G * G // (65536 * 65536)))
    else:
        w = config(5, H=16384 * world, W=16384, n_obstacles=16 * world)
    H, W = w.H, w.W
    sim = DistSim(W, H, rank, world, None, uid=ctx.uid(), dtype=dtype, tb_depth=args.tb)
    try:
        sim.paint_phi(0.054)
        for rect in w.meta["obstacles"]:
            sim.paint_phi(0.2, rect)
        sim.fill_noise(seed=1)
        for shape, val, at in w.events[0]:
            sim.stimulate(shape, val, at)
        cells = sim.rows * W
        u0 = v0 = None
        if not strong and args.e2e_steps > 0:
            u0, v0 = sim.read_owned(0)
        ms, st, clk = timed(ctx, sim.step, sim.h, T, args.steps, args.warmup, ctx.local)
        ms_max = ctx.max(ms)
        geo = sim.geometry()
        e2e = None
        if not strong and args.e2e_steps > 0:
            # per rank: owned rows in from pinned host memory, step (halos
            # inside librd), owned rows out; max over ranks
            pu = torch.empty((sim.rows, W), dtype=torch.float32, pin_memory=True).numpy()
            pv = torch.empty((sim.rows, W), dtype=torch.float32, pin_memory=True).numpy()
            pu[...] = u0
            pv[...] = v0
            ou = np.empty_like(pu)
            ov = np.empty_like(pv)
            stream = torch.cuda.current_stream()
            ctx.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.e2e_steps):
                rd.rd_write_fields(sim.h, 0, pu, pv)
                sim.step(T)
                rd.rd_read_fields(sim.h, 0, ou, ov)
            b.record(stream)
            ctx.barrier()
            ems = ctx.max(a.elapsed_time(b))
            e2e = {"value": H * W * T * args.e2e_steps / (ems / 1e3) / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": 2 * cells * 4, "d2h_bytes_per_step": 2 * cells * 4,
                   "steps": args.e2e_steps,
                   "api": "per rank: rd_write_fields(host pinned, owned rows) + rd_step (rd_create_dist: halos "
                          "inside librd) + rd_read_fields(host); bytes per rank, time max over ranks"}
    finally:
        sim.close()
    value = H * W * T * args.steps / (ms_max / 1e3) / 1e9
    return {"value": value, "ms_per_step": ms_max / args.steps, "rank_ms_per_step": ms / args.steps,
            "T": T, "grid": [H, W], "st": st, "clk": clk, "geo": geo, "e2e": e2e,
            "roofline": roofline_of(st, ms, "c5_strong" if strong else "c5_weak", dtype)}


def run_dist(args, ctx):
    """N > 1 (and --scaling strong at N = 1): the weak line with the strong
    result beside it (BASELINE.json north_star: "8-GPU scaling efficiency
    >=85% on the largest grid" is the strong number)."""
    world = ctx.world
    hbm, _ = peaks()
    weak = None if args.scaling == "strong" else dist_run(args, ctx, strong=False)
    strong = None
    if args.scaling == "strong" or (world > 1 and not args.no_strong):
        strong = dist_run(args, ctx, strong=True)
    if ctx.rank != 0:
        return None
    main = weak or strong
    scaling = "weak" if weak else "strong"
    st = main["st"]
    line = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(world, main["T"], st["tb_depth"], scaling, args.strong_grid),
            "frac_of_one_step_hbm_roofline": main["value"] / world / (hbm / BYTES_PER_CELL[np.dtype(np.float32)]),
            "roofline": main["roofline"], "cpu_baseline": None, "e2e": main["e2e"],
            "gpu_launches": st["launches"], "clocks": main["clk"],
            "transport": main["geo"]["transport"], "halo_exchanges_rank0": main["geo"]["exchanges"]}
    if main["e2e"] is None:
        line["e2e"] = {"skipped": "--scaling strong: host copies of the 65536^2 grid (17/N GB per plane) are "
                                  "not staged; the weak line carries e2e"}
    if weak and strong:
        line["strong"] = {"value": strong["value"], "unit": UNIT, "ms_per_step": strong["ms_per_step"],
                          "rank0_ms_per_step": strong["rank_ms_per_step"], "time_steps_per_step": strong["T"],
                          "config": config_dict(world, strong["T"], strong["st"]["tb_depth"], "strong",
                                                args.strong_grid),
                          "roofline": strong["roofline"], "transport": strong["geo"]["transport"]}
    if ctx.functional:
        line["functional_check"] = ("RD_BENCH_THREADS / RD_BENCH_SHM: the ranks shared a GPU; the numbers are not "
                                    "a measurement")
    return line


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    threads = os.environ.get("RD_BENCH_THREADS") == "1" and args.gpus > 1
    if threads:
        world = args.gpus
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world == 1 and args.scaling != "strong":
        line = run_single(args)
    elif threads:
        shared = {"barrier": threading.Barrier(world), "vals": [0.0] * world}
        out = [None] * world
        errs = []

        def body(r):
            try:
                torch.cuda.set_device(local)
                out[r] = run_dist(args, ThreadCtx(world, r, shared))
            except BaseException as e:  # noqa: BLE001 -- surfaced below
                errs.append(e)
                shared["barrier"].abort()

        ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        line = out[0]
    else:
        if world > 1:
            import torch.distributed as dist
            if os.environ.get("RD_BENCH_SHM") == "1":
                # RD_BENCH_SHM=1: the torchrun launch on a box with fewer GPUs than ranks. torch's process
                # group is gloo, librd's is the shared-memory one; the ranks' processes share devices.
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        ctx = ProcCtx(world, rank, local)
        ctx.functional = world > torch.cuda.device_count()
        line = run_dist(args, ctx)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def cpu_baseline(u0, v0, phi, seconds: float):
    """The oracle, as it stands, on the host cores: a bounded sample of the same
    workload (the full grid for a few time steps, fp32 mode)."""
    import oracle
    oracle.set_num_threads(host_cores())
    H, W = u0.shape
    t = time.perf_counter()
    oracle.run(u0, v0, phi, 1)
    t1 = time.perf_counter() - t
    n = int(max(1, min(20, seconds / max(t1, 1e-3))))
    t = time.perf_counter()
    oracle.run(u0, v0, phi, n)
    el = time.perf_counter() - t
    return {"value": H * W * n / el / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"full {H}x{W} grid, {n} time steps, fp32 mode (config-4 inputs, no stimuli)",
            "seconds": el}


# ------------------------------------------------------- reference arm

def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) timed as it
    stands on the host cores, on our arm's config/metric/unit. Each bench step
    is a bounded sample of that workload: four time steps of a 16384 x 16384
    grid (N = 1: the config-4 grid; N > 1: rank 0's slab of the config-5
    weak-scaling grid, obstacles included) in one oracle call, after an
    untimed step 0 that applies the stimuli, so the run ends within minutes.
    Under torchrun rank 0 alone works; the other ranks exit without work."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from rdinputs import config
    oracle.set_num_threads(host_cores())  # torchrun sets OMP_NUM_THREADS=1; rank 0 alone works here
    if world == 1 and args.scaling == "weak":
        w = config(4)
        sample = "4 time steps of the full 16384x16384 config-4 grid per bench step (after step 0's stimuli)"
    else:
        w = config(5, H=16384, W=16384, n_obstacles=16)
        sample = ("4 time steps of one 16384x16384 slab of the config-5 geometry (16 obstacles) per bench step "
                  "(after step 0); the metric is a per-cell rate")
    u, v = w.init_planes(0)
    phi = w.phi_plane(0).astype(np.float32)
    # untimed: step 0 with the stimuli (our arm stamps them before its timed
    # region too), then the warm-up steps
    r = oracle.run(u, v, phi, 1, events=w.events[0])
    cu, cv, s0 = r.u, r.v, 1
    n = 4  # time steps per bench step: one oracle call, amortising its marshalling
    for _ in range(args.warmup):
        r = oracle.run(cu, cv, phi, n, step0=s0)
        cu, cv, s0 = r.u, r.v, s0 + n
    t = time.perf_counter()
    for _ in range(args.steps):
        r = oracle.run(cu, cv, phi, n, step0=s0)
        cu, cv, s0 = r.u, r.v, s0 + n
    el = time.perf_counter() - t
    value = w.H * w.W * n * args.steps / el / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(world, args.timesteps, args.tb or 4, args.scaling),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--timesteps", type=int, default=1000, help="time steps per bench step")
    ap.add_argument("--tb", type=int, default=0, help="temporal-blocking depth (0 = auto)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-pipeline", type=int, default=2,
                    help="N = 1: 2 = e2e with the library's asynchronous host I/O (copies of the neighbouring jobs "
                         "under a job's steps), 1 = the serial write/step/read only")
    ap.add_argument("--e2e-pipeline-steps", type=int, default=24)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="the line's workload: weak (N = 1: configs[3]; N > 1: configs[4] with 16384 rows per GPU, "
                         "the strong result beside it) or strong (configs[4] 65536^2 split over N, any N)")
    ap.add_argument("--strong-grid", type=int, default=65536, help="side of the strong-scaling grid")
    ap.add_argument("--strong-timesteps", type=int, default=200, help="time steps per bench step, strong line")
    ap.add_argument("--no-strong", action="store_true", help="N > 1: skip the strong-scaling result")
    ap.add_argument("--no-configs", action="store_true", help="N = 1: skip per_config and fp32_error")
    ap.add_argument("--config-cpu-seconds", type=float, default=2.0,
                    help="oracle seconds per per_config entry (its cpu_baseline)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
