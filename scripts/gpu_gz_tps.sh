# gz_kernel: one vs two tiles per SM (RD_GZ_TPS) and the block depth, configs 1-3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gz.py -x -q -p no:cacheprovider > gpurun_out/t_gz.log 2>&1; echo gz tests rc=$?; tail -2 gpurun_out/t_gz.log
RD_GZ_TPS=2 timeout 900 python -m pytest tests/test_gpu_gz.py -x -q -p no:cacheprovider > gpurun_out/t_gz2.log 2>&1; echo gz tps2 tests rc=$?; tail -2 gpurun_out/t_gz2.log
pc() { python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$1', d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],2), 'ms', d['stencil_kernel'])"; }
for TPS in 1 2 0; do for K in 6 8 10; do
  RD_GZ_TPS=$TPS RD_KERNEL=gz RD_GZ_K=$K timeout 300 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 2>/dev/null | pc "tps$TPS k$K"
done; done
