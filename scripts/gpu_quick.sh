cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('tb', d['config']['tb_depth'], 'value', round(d['value'],1), 'kernel_ms', round(r['avg_launch_ms'],3), 'frac', round(r['frac'],3), d['clocks'])"
timeout 300 python scripts/bench_configs.py --configs 1,2,3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],1), 'ms', d['launches'], 'launches', d['first_fire'])"
