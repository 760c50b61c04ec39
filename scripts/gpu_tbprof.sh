#!/bin/bash
# One ncu --set full capture of a tb_kernel launch on config 4 (after a plain
# run of the same command) -> gpurun_out/prof_full.ncu-rep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD2="python bench.py --timesteps 100 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 20 -c 1 -f -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
