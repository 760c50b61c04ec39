#!/bin/bash
# DRAM bytes and instructions per cell-update of tb_kernel at each temporal-
# blocking depth K = 1..6 on config 4 ("Record dram__bytes ...
# for each k"): a plain bench run per K (device-timed Gcell/s), then an ncu
# pass over three tb_kernel launches of the same command.
# Output: gpurun_out/kt_<K>.json (bench line), gpurun_out/kt_<K>.csv (ncu).
# RD_TB_UPHI=0 in the environment measures the kernel that streams the phi
# plane (config 4's one-valued map otherwise goes in as a parameter, K <= 4);
# KT_TAG=<suffix> names the output files kt<suffix>_<K>.*.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active
for K in ${KS:-1 2 3 4 5 6}; do
  CMD="python bench.py --tb $K --timesteps 60 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  $CMD > gpurun_out/kt${KT_TAG}_$K.json 2> gpurun_out/kt${KT_TAG}_$K.err
  echo "K=$K plain rc=$?"
  ncu --metrics $M --clock-control none -k regex:tb_kernel -s 6 -c 3 --csv --log-file gpurun_out/kt${KT_TAG}_$K.csv \
      python bench.py --tb $K --timesteps 60 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  echo "K=$K ncu rc=$?"
done
