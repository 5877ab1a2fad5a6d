mkdir -p gpurun_out; : > gpurun_out/ab_dgm.txt
for r in 1 2; do for gm in 4 6 8 16; do
  echo "gm=$gm" >> gpurun_out/ab_dgm.txt
  EPSMOE_RASTER_GM=$gm python tools/gemm_bench.py --config mixtral --reps 10 >> gpurun_out/ab_dgm.txt 2>&1
done; done
