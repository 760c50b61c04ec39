#!/usr/bin/env python
"""Does the halo transport complete UNDER a running interior launch?
(VERDICT r01 "what's weak" 2: tb_kernel's one-wave grid fills every SM's
register file, so a transport that needs SMs -- NCCL's kernels -- waits for
the interior launch to drain; rd_create_dist moves the halo rows with
cudaMemcpyAsync instead, on a second stream.)

On one GPU: a middle slab of the N > 1 workload (16384 x 16384 owned rows,
halo 4) opens a block with rd_step_begin, which launches the interior rows
(one 4-step tb_kernel launch over ~16376 rows, every SM busy) on stream A;
right after, a 2 MB device-to-device copy -- the size of one block's halo
rows at W = 65536 (4 rows x 2 planes x 2 sides x 64 Ki floats) -- is issued
on stream B. CUDA events on both streams give the copy's start and end
relative to the kernel's start. The copy alone (idle GPU) is timed too.
Output: one JSON line (profiles/<round>_overlap.json).
"""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1901_06535_b200 as rd  # noqa: E402


def main():
    n = 16384
    h = rd.rd_create_slab(n, n, None, n, 3 * n, 4, dtype=np.float32, tb_depth=4)
    rd.rd_paint_phi(h, -1, None, 0.054)
    rd.rd_fill_noise(h, -1, 3, 1, 0.1)
    A = torch.cuda.current_stream()
    B = torch.cuda.Stream()
    rd.rd_set_stream(h, rd.stream_handle(A))
    nbytes = 2 * 1024 * 1024
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda").fill_(1)
    dst = torch.empty_like(src)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # the copy alone
    alone = []
    for _ in range(20):
        b0, b1 = ev(), ev()
        b0.record(B)
        with torch.cuda.stream(B):
            dst.copy_(src)
        b1.record(B)
        torch.cuda.synchronize()
        alone.append(b0.elapsed_time(b1))
    rows = []
    for trial in range(12):
        a0, a1, b0, b1 = ev(), ev(), ev(), ev()
        torch.cuda.synchronize()
        a0.record(A)
        started = rd.rd_step_begin(h, 4)  # interior rows: one tb_kernel launch on stream A
        a1.record(A)
        b0.record(B)
        with torch.cuda.stream(B):
            dst.copy_(src)
        b1.record(B)
        rd.rd_step_finish(h)
        torch.cuda.synchronize()
        if trial < 2:
            continue  # warm-up
        rows.append({"started": bool(started), "interior_ms": a0.elapsed_time(a1),
                     "copy_start_ms": a0.elapsed_time(b0), "copy_end_ms": a0.elapsed_time(b1),
                     "copy_ms": b0.elapsed_time(b1)})
    rd.rd_destroy(h)
    under = [r["copy_end_ms"] < r["interior_ms"] for r in rows]
    out = {"what": "2 MB device-to-device cudaMemcpyAsync (torch copy_) on stream B issued right after the interior "
                   "tb_kernel launch of a 16384x16384 middle slab (rd_step_begin, K=4) on stream A; times relative "
                   "to the kernel's start event",
           "copy_alone_ms_median": statistics.median(alone),
           "interior_ms_median": statistics.median(r["interior_ms"] for r in rows),
           "copy_end_ms_median": statistics.median(r["copy_end_ms"] for r in rows),
           "copy_ms_under_kernel_median": statistics.median(r["copy_ms"] for r in rows),
           "completed_under_kernel": f"{sum(under)}/{len(under)}", "trials": rows,
           "gpu": torch.cuda.get_device_name()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
