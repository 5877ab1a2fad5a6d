# Round evidence refresh: GPU tests, bench lines, ncu launch list, ncu full of the expert GEMMs.
set -x
TAG=${1:-r01b}
O=gpurun_out/$TAG
mkdir -p $O
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.txt
python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.txt 2>&1
python bench.py > $O/bench_dsv2.json 2> $O/bench_dsv2.err
python bench.py --config mixtral > $O/bench_mixtral.json 2> $O/bench_mixtral.err
python bench.py --config dsv2_lite > $O/bench_dsv2_lite.json 2> $O/bench_dsv2_lite.err
python bench.py --config dsv2_decode --no-cpu-baseline > $O/bench_dsv2_decode.json 2> $O/bench_dsv2_decode.err
python bench.py --config mixtral_decode --no-cpu-baseline > $O/bench_mixtral_decode.json 2> $O/bench_mixtral_decode.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_dsv2.json 2> $O/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_dsv2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
# HBM-bound kernels (router GEMM, gate top-k, permute, combine): DRAM bytes and duration per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"permute_kernel|combine_kernel|gate_topk|gemm_kernel<2" -c 8 --csv \
    --log-file $O/hbm_kernels_dsv2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for cfg in dsv2 mixtral dsv2_lite; do
  ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 2 -o $O/gemms_$cfg -f \
      python tools/gemm_bench.py --config $cfg --reps 1 > $O/ncu_$cfg.log 2>&1
  ncu -i $O/gemms_$cfg.ncu-rep --page raw --csv > $O/gemms_${cfg}_raw.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
