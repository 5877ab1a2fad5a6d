# A/B (VARIANTS, interleaved, isolated GEMMs on dsv2 / lite / mixtral) then the GPU suite with the in-tree build.
set -x
O=gpurun_out/${1:-r02h}
V=${VARIANTS:-head dec}
mkdir -p $O
for rep in 1 2 3; do for v in $V; do
  for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_LIB=$PWD/tools/ab/lib_$v.so timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/$v /" >> $O/ab.txt
  done
done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in $V; do
EPSMOE_LIB=$PWD/tools/ab/lib_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 4 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_$v.csv 2>/dev/null
done
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -25 > $O/pytest_gpu.txt
