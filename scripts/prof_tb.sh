# ncu --set full of one tb_kernel launch (K from $1) on config 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K=${1:-4}
CMD="python bench.py --timesteps 100 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --tb $K"
$CMD > gpurun_out/plain_k$K.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 10 -c 1 -o gpurun_out/prof_k$K $CMD > gpurun_out/ncu_k$K.log 2>&1
echo "rc=$?"
