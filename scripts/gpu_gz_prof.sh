# ncu --set full of one gz_kernel launch (config 3 fp32, 20000 steps).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python scripts/bench_configs.py --configs 3 --dtype f32 --repeat 1"
RD_KERNEL=gz RD_GZ_K=${K:-12} timeout 300 $CMD > gpurun_out/plain_gz.log 2>&1 && \
RD_KERNEL=gz RD_GZ_K=${K:-12} timeout 900 ncu --set full --clock-control none --import-source on -k regex:gz_kernel -s 0 -c 1 -o gpurun_out/prof_gz $CMD > gpurun_out/ncu_gz.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_gz.log
