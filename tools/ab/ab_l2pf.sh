# GEMM producer L2 prefetch distance (EPSMOE_L2_PF k-blocks ahead, crossing into the next ticket)
O=gpurun_out/ab_l2pf; mkdir -p $O; : > $O/gemm.txt
for r in 1 2; do for cfg in dsv2 dsv2_lite mixtral; do for d in 0 4 8 16; do
  echo "[EPSMOE_L2_PF=$d]" >> $O/gemm.txt
  EPSMOE_L2_PF=$d python tools/gemm_bench.py --config $cfg --reps 20 >> $O/gemm.txt 2>&1
done; done; done
