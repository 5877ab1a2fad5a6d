# Does the load energy sit in L2 reads or in SM ingest?  Half tiles off (full tiles only), isolated DSv2 /
# Lite GEMMs, CUDA events (sustained), interleaved x3:
#   0 normal | 8 peer CTA loads no B (L2 reads -25%, ingest -25%) | 9 leader multicasts its B half to both
#   (L2 reads -25%, ingest unchanged) | 6 no B at all (-50% / -50%)
set -x
O=gpurun_out/${1:-r02p}
mkdir -p $O
export EPSMOE_HALF_TILES=0
for d in 9 8; do EPSMOE_GEMM_DIAG=$d timeout 120 python tools/gemm_bench.py --config dsv2_lite --reps 2 > $O/smoke_diag$d.txt 2>&1; echo "rc=$?" >> $O/smoke_diag$d.txt; done
for rep in 1 2 3; do for d in 0 8 9 6; do for c in dsv2 dsv2_lite; do
  EPSMOE_GEMM_DIAG=$d timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/diag=$d /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum
for d in 0 8 9; do
EPSMOE_GEMM_DIAG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 2 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_diag$d.csv 2>/dev/null
done
