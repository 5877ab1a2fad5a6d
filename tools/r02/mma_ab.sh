# A/B of the MMA issuer variants on the isolated DSv2 / Lite / Mixtral GEMMs + ncu source of the warp variant's Down.
set -x
O=gpurun_out/${1:-r02e}
mkdir -p $O
for rep in 1 2; do
for mw in 0 1; do for ht in 0 1; do
  for c in dsv2 dsv2_lite mixtral; do
    EPSMOE_MMA_WARP=$mw EPSMOE_HALF_TAG=$ht timeout 300 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/mw=$mw ht=$ht /" >> $O/ab.txt
  done
done; done; done
for mw in 0 1; do
EPSMOE_MMA_WARP=$mw timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<\\(int\\)1, \\(int\\)2" -s 2 -c 1 -o $O/down_mw$mw -f \
    python tools/gemm_bench.py --config dsv2 --reps 1 > $O/ncu_down_mw$mw.log 2>&1
ncu -i $O/down_mw$mw.ncu-rep --page raw --csv > $O/down_mw${mw}_raw.csv 2>/dev/null
ncu -i $O/down_mw$mw.ncu-rep --page source --csv > $O/down_mw${mw}_source.csv 2>/dev/null
rm -f $O/down_mw$mw.ncu-rep
done
for i in 1 2 3; do for mw in 0 1; do
EPSMOE_MMA_WARP=$mw timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x 2>&1 | tail -3 | sed "s/^/mw=$mw run=$i /" >> $O/multiproc.txt
done; done
