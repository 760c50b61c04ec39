# gz_kernel phase timing (measurement build -DRD_GZ_PROF), configs 2 and 3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RD_NVCC_DEFS="-DRD_GZ_PROF $EXTRA" python -c "from paper_1901_06535_b200 import _build; _build.build(force=True)" > gpurun_out/build_prof.log 2>&1 || { echo build failed; tail gpurun_out/build_prof.log; }
for K in ${KS:-8}; do for c in "3 f32" "3 f64" "2 f32" "2 f64"; do set -- $c
  echo "== k=$K config $1 $2"; RD_KERNEL=gz RD_GZ_K=$K timeout 120 python scripts/gz_phase_prof.py --config $1 --dtype $2 2>&1 | tail -5
done; done
