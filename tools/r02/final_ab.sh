# Same-box A/B of the GEMM diag hooks (a9131db vs working tree), then the round's evidence refresh.
set -x
O=gpurun_out/${1:-r02x}
mkdir -p $O
for rep in 1 2 3; do for v in head cur; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_LIB=$PWD/tools/ab/lib_$v.so timeout 120 python tools/gemm_bench.py --config $c --reps 10 2>&1 | sed "s/^/$v /" >> $O/ab.txt
done; done; done
