# Same-box A/B: HEAD build (tools/ab/lib_head.so) vs working tree, isolated DSv2 GEMMs, interleaved.
set -x
O=gpurun_out/${1:-r02f}
mkdir -p $O
for rep in 1 2 3; do
  EPSMOE_LIB=$PWD/tools/ab/lib_head.so timeout 300 python tools/gemm_bench.py --config dsv2 --reps 10 2>&1 | sed "s/^/head /" >> $O/ab.txt
  EPSMOE_MMA_WARP=0 EPSMOE_HALF_TAG=0 timeout 300 python tools/gemm_bench.py --config dsv2 --reps 10 2>&1 | sed "s/^/new00 /" >> $O/ab.txt
  EPSMOE_MMA_WARP=1 EPSMOE_HALF_TAG=0 timeout 300 python tools/gemm_bench.py --config dsv2 --reps 10 2>&1 | sed "s/^/new10 /" >> $O/ab.txt
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
EPSMOE_LIB=$PWD/tools/ab/lib_head.so timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_head.csv 2>/dev/null
EPSMOE_MMA_WARP=0 EPSMOE_HALF_TAG=0 timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_new00.csv 2>/dev/null
EPSMOE_MMA_WARP=1 EPSMOE_HALF_TAG=0 timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_new10.csv 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $O/smi.txt
