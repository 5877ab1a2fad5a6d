# Where the expert GEMMs' output-store cost comes from: stores to the real rows (0), none (1), or into
# a 256-row window that stays in L2 (3: same TMA store traffic, no DRAM writes)
O=gpurun_out/ab_store2; mkdir -p $O; : > $O/gemm.txt
for r in 1 2; do for cfg in dsv2 dsv2_lite mixtral; do for d in 0 1 3; do
  echo "[EPSMOE_GEMM_DIAG=$d]" >> $O/gemm.txt
  EPSMOE_GEMM_DIAG=$d python tools/gemm_bench.py --config $cfg --reps 20 >> $O/gemm.txt 2>&1
done; done; done
