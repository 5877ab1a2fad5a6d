# Clusters of 4 in lockstep with vs without the A multicast (DIAG=11), clusters only (MC=3) and hybrid (MC=1).
set -x
O=gpurun_out/${1:-r02w}
mkdir -p $O
for rep in 1 2 3; do for v in "0 0" "3 0" "3 11" "1 0" "1 11"; do set -- $v; for c in dsv2 dsv2_lite; do
  EPSMOE_MC=$1 EPSMOE_GEMM_DIAG=$2 timeout 120 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/mc=$1,d=$2 /" >> $O/ab.txt
done; done; done
