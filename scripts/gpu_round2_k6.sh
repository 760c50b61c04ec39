# Round-2 final profile after the depth-6 default for large fp32 grids: the
# default bench line, the reference arm, the strong N = 1 line, the ncu launch
# list of the bench command, one --set full capture of the default tb_kernel on
# config 4 (phi as a parameter, K = 6) and one of the streaming kernel
# (RD_TB_UPHI=0), the fp32 size sweep.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --scaling strong --steps 3 --warmup 3 > gpurun_out/bench_strong.log 2>/dev/null; echo "strong rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --e2e-pipeline 1 --no-cpu-baseline --no-configs"
timeout 300 $CMD > gpurun_out/plain_list.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "launch list rc=$?"
CMD2="python bench.py --timesteps 96 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 20 -c 1 -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv 2>/dev/null
RD_TB_UPHI=0 timeout 300 $CMD2 > gpurun_out/plain_streamed.log 2>&1 && \
RD_TB_UPHI=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 20 -c 1 -o gpurun_out/prof_streamed $CMD2 > gpurun_out/ncu_streamed.log 2>&1
echo "streamed rc=$?"
ncu -i gpurun_out/prof_streamed.ncu-rep --page raw --csv > gpurun_out/prof_streamed_raw.csv 2>/dev/null && rm -f gpurun_out/prof_streamed.ncu-rep
timeout 600 python scripts/bench_sizes.py > gpurun_out/bench_sizes.log 2>&1; echo "sizes rc=$?"
