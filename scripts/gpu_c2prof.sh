cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for kern in tb lp; do
RD_KERNEL=$kern python scripts/bench_configs.py --configs 2 --dtype f32 > gpurun_out/c2_$kern.log 2>&1 && \
RD_KERNEL=$kern ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -s 3000 -c 40 --csv --log-file gpurun_out/c2_$kern.csv python scripts/bench_configs.py --configs 2 --dtype f32 > gpurun_out/c2_ncu_$kern.log 2>&1
done
echo done
