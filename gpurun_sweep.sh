for K in 3 4 5 6; do for HB in 0 4 6 8 10 12 16; do
  if [ $HB = 0 ]; then unset RD_HB; else export RD_HB=$HB; fi
  RD_TB_DEPTH=$K RD_KERNEL=tb timeout 200 python scripts/bench_configs.py --configs 2,3 --dtype f64 --repeat 2 | sed "s/^/K$K HB$HB /" >> gpurun_out/sweep2.txt
done; done
