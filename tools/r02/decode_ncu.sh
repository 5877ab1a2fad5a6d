# Decode GEMMs under ncu --set full: Mixtral / DSv2 decode GateUp + Down (gemm_bench), and the
# DSv2 decode router inside the layer.  Raw CSVs for the HBM-fraction analysis.
set -x
O=gpurun_out/${1:-r02m}
mkdir -p $O
for cfg in mixtral_decode dsv2_decode; do
  timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 4 -c 2 -o $O/dec_$cfg -f \
      python tools/gemm_bench.py --config $cfg --reps 1 > $O/ncu_$cfg.log 2>&1
  ncu -i $O/dec_$cfg.ncu-rep --page raw --csv > $O/dec_${cfg}_raw.csv 2>/dev/null
done
timeout 600 ncu --set full --clock-control none -k regex:"gemm_kernel<2" -s 2 -c 1 -o $O/router_dsv2_decode -f \
    python bench.py --config dsv2_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_router.log 2>&1
ncu -i $O/router_dsv2_decode.ncu-rep --page raw --csv > $O/router_dsv2_decode_raw.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config mixtral_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/launches_mixtral_decode.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config dsv2_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/launches_dsv2_decode.csv 2>/dev/null
rm -f $O/*.ncu-rep
