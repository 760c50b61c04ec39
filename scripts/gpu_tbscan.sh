cd $GRAFT_REPO_ROOT
for tb in 1 2 3 4; do
timeout 300 python scripts/bench_configs.py --configs 1,2,3 --tb $tb 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('tb', d['tb_depth'], d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],1), 'ms', d['launches'], 'launches')"
done
