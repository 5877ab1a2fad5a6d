# Multicast clusters A/B: 0 off | 1 clusters + companions | 2 unit tickets on pairs only | 3 clusters only; + traces.
set -x
O=gpurun_out/${1:-r02v}
mkdir -p $O
for v in 0 1 3; do EPSMOE_TRACE=1 EPSMOE_MC=$v timeout 60 python tools/gemm_bench.py --config dsv2 --reps 1 > $O/trace_mc$v.txt 2>&1; done
for rep in 1 2 3; do for v in 0 1 2 3; do for c in dsv2 dsv2_lite; do
  EPSMOE_MC=$v timeout 120 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/mc=$v /" >> $O/ab.txt
done; done; done
