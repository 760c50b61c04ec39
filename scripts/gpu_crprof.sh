#!/bin/bash
# cr_kernel profile on config 2 (fp32): timing run, then one ncu --set full
# capture of a cr_kernel launch (development helper).
set -e
mkdir -p gpurun_out
python scripts/bench_configs.py --configs 1,2,3 --dtype f32 > gpurun_out/cr_bench.jsonl 2>&1
cat gpurun_out/cr_bench.jsonl
ncu --set full --import-source on --clock-control none -k regex:cr_kernel -s 0 -c 1 -f -o gpurun_out/cr_c2 \
  python scripts/bench_configs.py --configs 2 --dtype f32 --repeat 1 > gpurun_out/cr_ncu.log 2>&1 || tail -5 gpurun_out/cr_ncu.log
