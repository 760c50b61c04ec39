cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -8
for k in 2 3 4 5 6; do
  python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --tb $k 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('tb', d['config']['tb_depth'], 'value', round(d['value'],1), 'kernel_ms', round(r['avg_launch_ms'],3), 'frac', round(r['frac'],3), d['clocks'])"
done
