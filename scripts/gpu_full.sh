# The full GPU suite, smoke, and the per-config default choice.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python scripts/bench_configs.py --configs 1,2,3 --repeat 2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],2), 'ms', d['stencil_kernel'], d['first_fire'])"
