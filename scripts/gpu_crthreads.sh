#!/bin/bash
# cr_kernel block-size sweep on configs 1-3 (development helper)
for nt in 512 768 1024; do
  echo "== RD_CR_THREADS=$nt"
  RD_CR_THREADS=$nt python scripts/bench_configs.py --configs 1,2,3 --dtype f32 | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print(r['config'], r['dtype'], round(r['device_ms'], 3), 'ms', round(r['gcell_updates_per_s'], 1), 'Gcell/s')"
done
echo "== f64 default"
python scripts/bench_configs.py --configs 1,2,3 --dtype f64 | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print(r['config'], r['dtype'], round(r['device_ms'], 3), 'ms', round(r['gcell_updates_per_s'], 1), 'Gcell/s')"
