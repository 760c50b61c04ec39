#!/bin/bash
# Row-block height scan on config 4 (bench line; development helper)
for hb in 0 512 683 964 1366 2048; do
  RD_HB=$hb timeout 300 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('hb', $hb, round(d['value'],1), 'launch_ms', round(r['avg_launch_ms'],4), 'mhz', d['clocks']['sm_mhz'])"
done
