# GEMM change check (tag = $1): GPU tests, isolated GEMM timings, bench line, ncu tensor-pipe of GateUp / Down.
set -x
O=gpurun_out/${1:-r02d}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -25 > $O/pytest_gpu.txt
for c in dsv2 mixtral dsv2_lite; do timeout 300 python tools/gemm_bench.py --config $c --reps 10 > $O/gemm_$c.txt 2>&1; done
timeout 600 python bench.py > $O/bench_dsv2.json 2> $O/bench_dsv2.err
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k regex:"gemm_kernel" --csv \
    python tools/gemm_bench.py --config dsv2 --reps 2 > $O/ncu_gemms_dsv2.csv 2> $O/ncu_gemms.err
