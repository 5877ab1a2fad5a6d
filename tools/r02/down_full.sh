# ncu --set full with source of the DSv2 Down GEMM (in-tree build), raw + source csv.
set -x
O=gpurun_out/${1:-r02i}
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<\\(int\\)1, \\(int\\)2" -s 2 -c 1 -o $O/down -f \
    python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_down.log 2>&1
ncu -i $O/down.ncu-rep --page raw --csv > $O/down_raw.csv 2>/dev/null
ncu -i $O/down.ncu-rep --page source --csv > $O/down_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<\\(int\\)0, \\(int\\)2" -s 2 -c 1 -o $O/gateup -f \
    python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_gateup.log 2>&1
ncu -i $O/gateup.ncu-rep --page raw --csv > $O/gateup_raw.csv 2>/dev/null
ncu -i $O/gateup.ncu-rep --page source --csv > $O/gateup_source.csv 2>/dev/null
rm -f $O/*.ncu-rep
