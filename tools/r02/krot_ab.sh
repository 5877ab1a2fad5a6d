# k-block rotation per n-tile (EPSMOE_KROT): parity (incl. EP invariance) with rotation, layer A/B, decode GEMM ncu.
set -x
O=gpurun_out/${1:-r02z}
mkdir -p $O
EPSMOE_KROT=7 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py tests/test_gpu_fullsize.py tests/test_gpu_ep.py -m gpu -q -x 2>&1 | tail -3 > $O/pytest_krot7.txt
for rep in 1 2 3; do for v in 0 1 7; do for c in mixtral_decode dsv2_decode mixtral dsv2; do
  EPSMOE_KROT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/krot=$v /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.min.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in 0 1 7; do
  EPSMOE_KROT=$v timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel<[01]" -c 4 --csv python tools/gemm_bench.py --config mixtral_decode --reps 1 > $O/ncu_mixdec_krot$v.csv 2>/dev/null
done
