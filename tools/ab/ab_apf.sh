# GEMM: L2 bulk prefetch of the next raster block's A rows (EPSMOE_A_PF=1) vs none
O=gpurun_out/ab_apf; mkdir -p $O; : > $O/gemm.txt
for r in 1 2 3; do for cfg in dsv2 dsv2_lite mixtral; do for v in 0 1; do
  echo "[EPSMOE_A_PF=$v]" >> $O/gemm.txt
  EPSMOE_A_PF=$v python tools/gemm_bench.py --config $cfg --reps 20 >> $O/gemm.txt 2>&1
done; done; done
