# SM partition for the shared-experts || routing phase (ep == 1): the shared GEMMs on fewer SMs
# (EPSMOE_SHARED_CTAS) and the permute kept off the GEMM SMs by a shared-memory reservation
# (EPSMOE_ROUTE_SMEM), interleaved bench A/B.
O=gpurun_out/${1:-r02pa}
mkdir -p $O
for rep in 1 2 3; do
  for v in "X=0" "EPSMOE_SHARED_CTAS=132 EPSMOE_ROUTE_SMEM=16384" "EPSMOE_SHARED_CTAS=140 EPSMOE_ROUTE_SMEM=16384" "EPSMOE_SHARED_CTAS=124 EPSMOE_ROUTE_SMEM=16384" "EPSMOE_SHARED_CTAS=132"; do
    for c in dsv2 dsv2_lite; do
      env $v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/[$v] /" >> $O/ab.txt
    done
  done
done
