# Multicast clusters (EPSMOE_MC): hang check, GPU parity, isolated GEMM A/B, layer A/B.
set -x
O=gpurun_out/${1:-r02r}
mkdir -p $O
EPSMOE_MC=1 timeout 60 python tools/gemm_bench.py --config dsv2_lite --reps 2 > $O/first.txt 2>&1; echo "rc=$?" >> $O/first.txt
grep -q "rc=0" $O/first.txt || exit 3
EPSMOE_MC=1 EPSMOE_HALF_TILES=0 timeout 60 python tools/gemm_bench.py --config dsv2_lite --reps 2 >> $O/first.txt 2>&1; echo "rc=$?" >> $O/first.txt
EPSMOE_MC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py -q -x 2>&1 | tail -5 > $O/pytest_mc.txt
for rep in 1 2 3; do for v in 0 1; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_MC=$v timeout 120 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/mc=$v /" >> $O/ab.txt
done; done; done
for rep in 1 2; do for v in 0 1; do
  EPSMOE_MC=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/mc=$v /" >> $O/bench_ab.txt
done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum
for v in 0 1; do
EPSMOE_MC=$v timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel" -c 4 --csv python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_mc$v.csv 2>/dev/null
done
