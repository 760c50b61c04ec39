# gz_kernel bring-up: its own tests, then the parity/fuzz suites (every
# kernel-parametrised case runs on gz too), then per-config throughput with
# RD_KERNEL=gz at several block depths next to the default choice.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gz.py -x -q -p no:cacheprovider > gpurun_out/t_gz.log 2>&1; echo gz tests rc=$?; tail -15 gpurun_out/t_gz.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/t_par.log 2>&1; echo parity rc=$?; tail -15 gpurun_out/t_par.log
pc() { python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$1', d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],2), 'ms', d['stencil_kernel'], d['launches'], d['first_fire'])"; }
timeout 300 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 2>/dev/null | pc default
for K in 4 8 12 16; do
RD_KERNEL=gz RD_GZ_K=$K timeout 300 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 2>/dev/null | pc gz_k$K
done
