# Ceilings of the expert GEMMs: normal vs load pipeline alone (DIAG=4) vs MMA issue alone (DIAG=5),
# isolated DSv2 / Mixtral shapes, interleaved x3, + ncu of each mode.
set -x
O=gpurun_out/${1:-r02k}
mkdir -p $O
for rep in 1 2 3; do for d in 0 4 5 1; do for c in dsv2 mixtral; do
  EPSMOE_GEMM_DIAG=$d timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/diag=$d /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
for d in 0 4 5 1; do
EPSMOE_GEMM_DIAG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 4 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_diag$d.csv 2>/dev/null
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv >> $O/smi.txt
