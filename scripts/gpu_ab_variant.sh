cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
RD_TB_VARIANT=full python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs > gpurun_out/ab_full_$i.json 2>>gpurun_out/ab.err
python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs > gpurun_out/ab_lean_$i.json 2>>gpurun_out/ab.err
done
for f in gpurun_out/ab_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), d['clocks']['sm_mhz'], round(d['roofline']['avg_launch_ms'],4))"; done
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/t_all.log
