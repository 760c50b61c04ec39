cd $GRAFT_REPO_ROOT
for hb in 1 2 3 4 6 8 12 20; do
RD_HB=$hb timeout 300 python scripts/bench_configs.py --configs 2,3 --dtype f32 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('hb $hb', d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],1), 'ms')"
done
