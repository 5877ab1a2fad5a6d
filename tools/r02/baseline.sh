# Round-2 baseline: GPU tests, bench line, ncu full (with source) of the Down GEMM on DSv2 shapes.
set -x
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_dsv2.json 2> $O/bench_dsv2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel<1" -s 2 -c 1 -o $O/down_dsv2 -f \
    python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_down.log 2>&1
ncu -i $O/down_dsv2.ncu-rep --page raw --csv > $O/down_dsv2_raw.csv 2>/dev/null
ncu -i $O/down_dsv2.ncu-rep --page source --csv > $O/down_dsv2_source.csv 2>/dev/null
ncu -i $O/down_dsv2.ncu-rep --page details --csv > $O/down_dsv2_details.csv 2>/dev/null
