# tb_kernel change check: GPU suite, the bench line (no per-config/e2e legs),
# and one --set full capture of the K=4 LEAN launch for the instruction count.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t_all.log
for i in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs > gpurun_out/tbq_$i.json 2>gpurun_out/tbq.err
python -c "
import json; d=json.loads(open('gpurun_out/tbq_$i.json').read().strip().splitlines()[-1]); r=d['roofline']
print('value', round(d['value'],1), 'kernel_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), d['clocks'], 'per GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))"
done
CMD2="python bench.py --timesteps 100 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 20 -c 1 -o gpurun_out/prof_tb $CMD2 > gpurun_out/ncu_tb.log 2>&1
echo "ncu rc=$?"
