# A/B: Down epilogue bulk stores as 32 x 32 boxes (64 B per row) vs 32 x 64 boxes (full 128-B lines).
set -x
O=gpurun_out/${1:-r02m}
mkdir -p $O
EPSMOE_STORE64=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py -q -x 2>&1 | tail -3 > $O/pytest_store64.txt
for rep in 1 2 3; do for v in 0 1; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_STORE64=$v timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/s64=$v /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum
for v in 0 1; do
EPSMOE_STORE64=$v timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 4 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_s64_$v.csv 2>/dev/null
done
for rep in 1 2; do for v in 0 1; do
  EPSMOE_STORE64=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/s64=$v /" >> $O/bench_ab.txt
done; done
