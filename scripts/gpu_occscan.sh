#!/bin/bash
# Occupancy sweep of tb_kernel on config 4 (development helper): RD_TB_DSMEM adds
# dynamic shared memory to every launch so fewer one-warp CTAs fit per SM.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for ds in 0 1536 3072 5600 9000 15000; do
  RD_TB_DSMEM=$ds timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('dsmem', $ds, round(d['value'],1), 'launch_ms', round(r['avg_launch_ms'],4), 'mhz', d['clocks']['sm_mhz'], 'per GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))"
done
