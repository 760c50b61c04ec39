# A/B of the packed-fp32 row_update (RD_PACK) against the scalar default:
# the f32x2 mix microbenchmark, then bench lines of each build, then parity
# tests of the packed build.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/f32x2_mix scripts/f32x2_mix.cu && /tmp/f32x2_mix > gpurun_out/f32x2_mix.txt 2>&1; cat gpurun_out/f32x2_mix.txt
bq() { timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$1', 'value', round(d['value'],1), 'kernel_ms', round(r['avg_launch_ms'],4), d['clocks']['sm_mhz'], 'per GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))"; }
bq scalar; 
RD_NVCC_DEFS=-DRD_PACK python -c "from paper_1901_06535_b200 import _build; _build.build(force=True)" > gpurun_out/build_pack.log 2>&1 || echo build failed
bq packed; bq packed
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/t_pack.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_pack.log
python -c "from paper_1901_06535_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
bq scalar
