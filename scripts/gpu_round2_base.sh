# Round-2 baseline on the current HEAD: the GPU suite, the default bench line,
# the reference arm, the ncu launch list of the bench command and one --set full
# capture of tb_kernel (config 4) and gz_kernel (config 3 fp32).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
if [ -z "$RD_SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t_all.log
fi
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_reference.log | cut -c1-300
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --e2e-pipeline 1 --no-cpu-baseline --no-configs"
timeout 300 $CMD > gpurun_out/plain_list.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "launch list rc=$?"
CMD2="python bench.py --timesteps 100 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 20 -c 1 -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
CMD3="python scripts/bench_configs.py --configs 3 --dtype f32 --repeat 1"
timeout 300 $CMD3 > gpurun_out/plain_cr.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gz_kernel -s 0 -c 1 -o gpurun_out/prof_gz $CMD3 > gpurun_out/ncu_gz.log 2>&1
echo "gz rc=$?"
# gpurun merges at most 64 MiB back: keep the tb_kernel report, export the raw page of the others
ncu -i gpurun_out/prof_gz.ncu-rep --page raw --csv > gpurun_out/prof_gz_raw.csv 2>/dev/null && rm -f gpurun_out/prof_gz.ncu-rep
timeout 600 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 > gpurun_out/bench_configs.log 2>&1; echo "configs rc=$?"
# fp64 on the config-4 grid: one --set full capture of tb_kernel<double, K=4> (LEAN)
CMD4='python -c "import bench; print(bench.config4_fp64(40))"'
timeout 300 bash -c "$CMD4" > gpurun_out/plain_f64.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 12 -c 1 -o gpurun_out/prof_tb_f64 bash -c "$CMD4" > gpurun_out/ncu_f64.log 2>&1
echo "f64 rc=$?"
ncu -i gpurun_out/prof_tb_f64.ncu-rep --page raw --csv > gpurun_out/prof_tb_f64_raw.csv 2>/dev/null && rm -f gpurun_out/prof_tb_f64.ncu-rep
# throughput against grid size with the default kernel choice (gz_kernel -> tb_kernel hand-over)
timeout 600 python scripts/bench_sizes.py > gpurun_out/bench_sizes.log 2>&1; echo "sizes rc=$?"
timeout 600 python scripts/bench_sizes.py --dtype f64 --sizes 128,256,512,1024,1536,2048,4096,8192 > gpurun_out/bench_sizes_f64.log 2>&1; echo "sizes f64 rc=$?"
