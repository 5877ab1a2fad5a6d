# How the expert GEMMs' time under the power cap scales with operand bytes: normal vs B loads skipped (DIAG=6)
# vs A loads skipped (7) vs no loads (5), isolated DSv2 / Lite GEMMs, CUDA events (sustained), interleaved x3 + ncu.
set -x
O=gpurun_out/${1:-r02o}
mkdir -p $O
for rep in 1 2 3; do for d in 0 6 7 5; do for c in dsv2 dsv2_lite; do
  EPSMOE_GEMM_DIAG=$d timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/diag=$d /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for d in 0 6 7; do
EPSMOE_GEMM_DIAG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 2 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_diag$d.csv 2>/dev/null
done
