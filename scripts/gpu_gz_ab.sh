# A/B of gz_kernel build variants (RD_NVCC_DEFS) on configs 2/3 at k = 8.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
pc() { python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$1', d['config'], d['dtype'], round(d['gcell_updates_per_s'],1), 'Gcell/s', round(d['device_ms'],2), 'ms', d['stencil_kernel'])"; }
for DEFS in "$@"; do
  RD_NVCC_DEFS="$DEFS" python -c "from paper_1901_06535_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo "build failed: $DEFS"
  for K in 6 8 10; do
    RD_KERNEL=gz RD_GZ_K=$K timeout 300 python scripts/bench_configs.py --configs 2,3 --repeat 2 2>/dev/null | pc "[$DEFS] k$K"
  done
done
