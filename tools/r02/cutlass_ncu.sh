# ncu --set full of our grouped GEMMs and torch._grouped_mm (CUTLASS) on the same problems.
set -x
O=gpurun_out/${1:-r02r}
mkdir -p $O
for cfg in dsv2 dsv2_lite; do
  for g in "" "--gateup"; do
    n=down; [ -n "$g" ] && n=gateup
    timeout 900 ncu --set full --clock-control none -c 16 -o $O/${cfg}_$n -f \
        python tools/down_vs_cutlass.py --config $cfg $g > $O/ncu_${cfg}_$n.log 2>&1
    ncu -i $O/${cfg}_$n.ncu-rep --page raw --csv > $O/${cfg}_${n}_raw.csv 2>/dev/null
  done
done
rm -f $O/*.ncu-rep
