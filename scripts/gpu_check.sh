set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or ragged or batched or splitting or reaction or masked or probes or nonfinite or write_fields" 2>&1 | tail -25
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/bench1.log 2>&1; tail -3 gpurun_out/bench1.log
