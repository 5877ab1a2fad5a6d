# Ticket-queue depth 4 vs 8 (EPSMOE_TQ), Down vs CUTLASS in isolation; static Down for reference.
O=gpurun_out/${1:-r02w}
mkdir -p $O
for rep in 1 2; do for v in tq4 tq8 static; do for c in dsv2 dsv2_lite; do
  if [ $v = static ]; then E="EPSMOE_DYN_SCHED=0 EPSMOE_LIB=$PWD/tools/ab/lib_tq4.so"; else E="EPSMOE_LIB=$PWD/tools/ab/lib_$v.so"; fi
  env $E timeout 300 python tools/down_ab_cutlass.py --config $c --rounds 12 2>>$O/err.txt | sed "s/^/$v /" >> $O/down.txt
done; done; done
