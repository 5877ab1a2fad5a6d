# Down GEMM knobs (scheduler, raster, TMA stores) vs torch._grouped_mm (CUTLASS) in the same process.
O=gpurun_out/${1:-r02t}
mkdir -p $O
for c in dsv2 dsv2_lite; do
  for kv in "X=0" "EPSMOE_DYN_SCHED=0" "EPSMOE_RASTER_GM=1" "EPSMOE_RASTER_GM=2" "EPSMOE_RASTER_GM=8" "EPSMOE_RASTER_GM=16" "EPSMOE_TMA_STORE=0" "X=1"; do
    env $kv timeout 300 python tools/down_ab_cutlass.py --config $c --rounds 12 2>>$O/err.txt | sed "s/^/$kv /" >> $O/knobs.txt
  done
done
