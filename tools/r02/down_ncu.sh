# ncu --set full (with source) of the Down GEMM on DSv2 shapes + epilogue diag A/B
set -x
O=gpurun_out/r02b
mkdir -p $O

timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<\\(int\\)1, \\(int\\)2" -s 2 -c 1 -o $O/down_dsv2 -f \
    python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_down.log 2>&1
ncu -i $O/down_dsv2.ncu-rep --page raw --csv > $O/down_dsv2_raw.csv 2>/dev/null
ncu -i $O/down_dsv2.ncu-rep --page source --csv > $O/down_dsv2_source.csv 2>/dev/null
ncu -i $O/down_dsv2.ncu-rep --page details --csv > $O/down_dsv2_details.csv 2>/dev/null
