#!/usr/bin/env python
"""Benchmark of the Oregonator forward-Euler hot path (BASELINE.json metric:
"Gcell-updates/s and % of B200 HBM roofline at 1/2/4/8 GPUs").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One bench "step" = rd_step(T) with T = --timesteps (default 1000) time steps of
the whole hot path (a1-a8: due stimuli, K-step blocked stencil launches, the
non-finite health check, probe latches) over the workload:
  N = 1: configs[3] "c4_roofline" 16384 x 16384 fp32, noise + 64 half-discs;
         K = 10 x 1000 = the config's 10000 timed steps.
  N > 1: configs[4] weak scaling: a 16384-row slab per GPU of a
         (16384 N) x 16384 grid with 16 N obstacles, halo exchange over NCCL.
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


def config_dict(world: int, T: int, tb_depth: int, scaling: str = "weak") -> dict:
    """The `config` of the JSON line -- the same for our arm and the
    reference arm (BASELINE.json configs[3] at N = 1,
    configs[4] weak scaling at N > 1; --scaling strong: configs[4] at its full
    65536 x 65536 over N GPUs)."""
    if scaling == "strong":
        d = {"workload": "configs[4] strong scaling: 65536x65536 fp32 row slabs over N GPUs, 256 obstacles "
                         "phi=0.2, masked half-discs, NCCL halo exchange", "grid": [65536, 65536]}
        return dict(d, time_steps_per_step=T, tb_depth=tb_depth,
                    l2="inputs larger than L2 (5 planes of 17/N GB per GPU); no flush needed",
                    parallelism=f"row slabs x{world}")
    if world == 1:
        d = {"workload": "configs[3] c4_roofline: 16384x16384 fp32, phi=0.054, u,v~U[0,0.1) seed 1, "
                         "64 half-discs r=8 seed 2, no-flux", "grid": [16384, 16384]}
    else:
        d = {"workload": f"configs[4] weak scaling: ({16384 * world})x16384 fp32 row slabs, 16 obstacles/GPU "
                         "phi=0.2, masked half-discs, NCCL halo exchange", "grid": [16384 * world, 16384]}
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


# ------------------------------------------------------------- our arm

def e2e_pipelined(rd, sim, w, dtype, tb, pu, pv, T, depth, steps, cells):
    """e2e with `depth` handles of the same workload, each driven by its own
    host thread through the public API (ctypes releases the GIL; each handle
    has its own CUDA stream). Every step still copies its inputs in from
    pinned host memory and its result out, inside the timed region; one job's
    copies overlap another job's stencil launches (copy engines vs SMs), and
    the jobs' stencil launches do not overlap each other (one steps at a time).
    Timed on the host clock between two device synchronisations."""
    import torch
    sims = [sim] + [rd.Sim(None, shape=(1, w.H, w.W), dtype=dtype, tb_depth=tb)
                    for _ in range(depth - 1)]
    try:
        rd.rd_set_stream(sim.h, 0)  # back to the handle's own stream
        for s in sims[1:]:
            s.paint_phi(0.054)
            for shape, val, at in w.events[0]:
                s.stimulate(shape, val, at)
            s.write(0, pu, pv)
            s.step(T)  # warm-up: events consumed, segment graphs captured
        outs = [(torch.empty(pu.shape, dtype=torch.float32, pin_memory=True).numpy(),
                 torch.empty(pu.shape, dtype=torch.float32, pin_memory=True).numpy()) for _ in sims]
        counts = [steps // depth + (1 if k < steps % depth else 0) for k in range(depth)]
        errors = []
        # staggered start: job k begins once job k-1's first inputs are on the
        # device, so the first launch does not wait for every job's upload
        uploaded = [threading.Event() for _ in range(depth)]
        # one job steps at a time (two concurrent stencil grids would share
        # the SMs and break tb_kernel's one-wave schedule); uploads and
        # read-backs of the other jobs proceed meanwhile on the copy engines
        compute = threading.Lock()

        def job(k):
            try:
                if k:
                    uploaded[k - 1].wait()
                for i in range(counts[k]):
                    rd.rd_write_fields(sims[k].h, 0, pu, pv)
                    if i == 0:
                        uploaded[k].set()
                    with compute:
                        sims[k].step(T)
                    rd.rd_read_fields(sims[k].h, 0, *outs[k])
            except Exception as e:  # surfaced below
                errors.append(e)
            finally:
                uploaded[k].set()

        threads = [threading.Thread(target=job, args=(k,)) for k in range(depth)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        if errors:
            raise errors[0]
    finally:
        for s in sims[1:]:
            s.close()
    return {"value": cells * T * steps / secs / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 2 * cells * 4, "d2h_bytes_per_step": 2 * cells * 4, "steps": steps,
            "pipeline": depth, "timer": "host clock between device synchronisations",
            "api": f"{depth} handles, one host thread each: rd_write_fields(host pinned) + rd_step + "
                   "rd_read_fields(host) every step"}


def run_ours(args):
    import torch
    import paper_1901_06535_b200 as rd
    from paper_1901_06535_b200.dist import SlabSim
    from rdinputs import config

    world, rank, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # RD_BENCH_BACKEND=gloo: functional check of this N > 1 path with
        # several ranks on one GPU (host-staged halos; not a measurement)
        backend = os.environ.get("RD_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dtype = np.dtype(np.float32)
    T = args.timesteps
    hbm, hbm_src = peaks()

    strong = args.scaling == "strong"
    if world == 1 and not strong:
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
        stepper = sim.step
        cells = H * W
    else:
        # weak: 16384 rows per GPU; strong: the full 65536^2 grid split over
        # the ranks (N = 1 included: one 120 GB slab)
        w = (config(5) if strong else config(5, H=16384 * world, W=16384, n_obstacles=16 * world))
        H, W = w.H, w.W
        slab = SlabSim(W, H, rank, world, None, dtype=dtype, halo=max(args.tb, 4) if args.tb else 4,
                       p2p=args.p2p)
        h = slab.h
        rd.rd_paint_phi(h, -1, None, 0.054)
        for rect in w.meta["obstacles"]:
            rd.rd_paint_phi(h, -1, rect, 0.2)
        slab.fill_noise(seed=1)
        for shape, val, at in w.events[0]:
            slab.stimulate(shape, val, at)
        stepper = slab.step
        cells = slab.rows * W
        # host copies of this rank's rows for the e2e leg (not at the strong
        # sizes: 17/N GB per plane)
        u0 = v0 = None
        if not strong:
            u0, v0 = slab.read_owned(0)
    stream = torch.cuda.current_stream()
    rd.rd_set_stream(h, rd.stream_handle(stream))  # engine work on the stream the events are recorded on

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        stepper(T)
    barrier()
    rd.rd_reset_stats(h)
    rd.rd_set_profiling(h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            stepper(T)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    st = rd.rd_get_stats(h)
    rd.rd_set_profiling(h, False)
    ms_max = max_over_ranks(ms, world)
    total_updates = cells * world * T * args.steps
    value = total_updates / (ms_max / 1e3) / 1e9

    # dominant kernel: the temporally blocked stencil (tb_kernel)
    kms = st["step_kernel_ms"]
    k_launches = max(1, st["timed_launches"])
    bpc = BYTES_PER_CELL[dtype]
    achieved = bpc * st["cell_updates"] / (kms / 1e3) / 1e9 if kms > 0 else None
    # DRAM bytes per tb_kernel launch from the latest committed ncu --set full
    # capture (profiles/traffic_rNN.json, scripts/summarize_ncu.py)
    traffic = None
    tfiles = sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")))
    if tfiles:
        try:
            traffic = json.load(open(tfiles[-1])).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # temporal blocking moves the kernel off the HBM roof (DRAM bytes per
    # launch ~ one step's, ncu) onto the FP32 pipe: report the ALU bound, with
    # the one-step HBM view beside it
    alu, alu_src = alu_peak_tops()
    ops = OPS_PER_CELL * st["cell_updates"] / (kms / 1e3) / 1e12 if kms > 0 else None
    roofline = {"bound": "alu", "achieved": ops, "peak": alu, "unit": "TFLOP/s",
                "frac": (ops / alu) if ops else None, "traffic": traffic,
                "kernel": f"tb_kernel<float,K={st['tb_depth']}>", "peak_source": alu_src,
                "algorithmic_ops_per_cell_update": OPS_PER_CELL,
                "ops": "fp32 add/sub/mul/div of the canonical Eq.-1 tree (13 + 9 + 1), R-8",
                "cell_updates_per_launch": st["cell_updates"] / k_launches,
                "avg_launch_ms": kms / k_launches, "kernel_share_of_step": kms / ms if ms else None,
                "hbm_view": {"achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": (achieved / hbm) if achieved else None, "peak_source": hbm_src,
                             "algorithmic_bytes_per_cell_update": bpc, "one_step_roofline_gcells": hbm / bpc}}

    # e2e through the public API with pinned host buffers: every step writes
    # this rank's u, v from the host, steps, and reads u, v back (N > 1: the
    # owned rows of each slab; time = max over ranks)
    e2e = None
    if strong:
        e2e = {"skipped": "--scaling strong: 65536^2 host copies (17/N GB per plane) are not staged; "
                          "the default (weak) line carries e2e"}
    elif args.e2e_steps > 0:
        rows = u0.shape[0]
        pu = torch.empty((rows, W), dtype=torch.float32, pin_memory=True).numpy()
        pv = torch.empty((rows, W), dtype=torch.float32, pin_memory=True).numpy()
        pu[...] = u0
        pv[...] = v0
        ou = torch.empty((rows, W), dtype=torch.float32, pin_memory=True).numpy()
        ov = torch.empty((rows, W), dtype=torch.float32, pin_memory=True).numpy()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            rd.rd_write_fields(h, 0, pu, pv)
            stepper(T)
            rd.rd_read_fields(h, 0, ou, ov)
        b.record(stream)
        barrier()
        ems = max_over_ranks(a.elapsed_time(b), world)
        e2e = {"value": cells * world * T * args.e2e_steps / (ems / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * cells * 4, "d2h_bytes_per_step": 2 * cells * 4,
               "steps": args.e2e_steps,
               "api": ("rd_write_fields(host pinned) + rd_step + rd_read_fields(host)" if world == 1 else
                       "per rank: rd_write_fields(host pinned, owned rows) + SlabSim.step (NCCL halos) + "
                       "rd_read_fields(host); bytes per rank, time max over ranks")}
        if world == 1 and args.e2e_pipeline > 1:
            serial = e2e
            e2e = e2e_pipelined(rd, sim, w, dtype, args.tb, pu, pv, T, args.e2e_pipeline, args.e2e_pipeline_steps, cells)
            e2e["serial"] = {"value": serial["value"], "steps": serial["steps"], "api": serial["api"]}

    cpu = None
    if rank == 0 and world == 1 and not strong and not args.no_cpu_baseline:
        cpu = cpu_baseline(u0, v0, phi, args.cpu_seconds)

    launches = st["launches"]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_dict(world, T, st["tb_depth"], args.scaling),
                "frac_of_one_step_hbm_roofline": value / world / (hbm / bpc),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


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
                    help="handles (host threads) of the pipelined e2e leg at N = 1 (1: serial only)")
    ap.add_argument("--e2e-pipeline-steps", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1: peer-memory halo push (CUDA IPC + stream-ordered flags) instead of NCCL")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N > 1 workload: configs[4] weak (16384 rows per GPU, default) or strong (65536^2 split)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
