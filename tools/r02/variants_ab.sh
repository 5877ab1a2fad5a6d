# Same-box A/B of compiled variants (tools/ab/lib_*.so) on the isolated DSv2 / Lite GEMMs, interleaved x3, + ncu tensor-pipe.
set -x
O=gpurun_out/${1:-r02g}
V=${VARIANTS:-head m0h0 m0h1 m1h0 m1h1}
mkdir -p $O
for rep in 1 2 3; do for v in $V; do
  for c in dsv2 dsv2_lite; do
  EPSMOE_LIB=$PWD/tools/ab/lib_$v.so timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/$v /" >> $O/ab.txt
  done
done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in $V; do
EPSMOE_LIB=$PWD/tools/ab/lib_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 4 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_$v.csv 2>/dev/null
done
