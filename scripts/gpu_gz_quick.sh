# gz_kernel quick A/B: gz tests, configs 2-3 at the model's k and at KS, then
# the phase-timing build at k = 8 (configs 2-3).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gz.py -x -q -p no:cacheprovider > gpurun_out/t_gz.log 2>&1; echo gz tests rc=$?; tail -2 gpurun_out/t_gz.log
pc() { python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$1', d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],2), 'ms', d['stencil_kernel'])"; }
timeout 300 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 2>/dev/null | pc default
for K in ${KS:-8}; do
  RD_KERNEL=gz RD_GZ_K=$K timeout 300 python scripts/bench_configs.py --configs 2,3 --repeat 2 2>/dev/null | pc "k$K"
done
KS=8 bash scripts/gpu_gz_phase.sh 2>&1 | grep -v 'poll passes'
