# Is an epilogue stall free under the power cap?  Normal (double-buffered TMEM accumulator) vs DIAG=10 (the MMA
# waits for the previous tile's drain), and DIAG=8 for reference; isolated GEMMs, CUDA events, interleaved x3 + ncu.
set -x
O=gpurun_out/${1:-r02q}
mkdir -p $O
for rep in 1 2 3; do for d in 0 10 8; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_GEMM_DIAG=$d timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/diag=$d /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for d in 0 10; do
EPSMOE_GEMM_DIAG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 2 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_diag$d.csv 2>/dev/null
done
