# Split-K router for E <= 64 (R19): GPU suite, then A/B vs HEAD (no split anywhere).
set -x
O=gpurun_out/${1:-r02o}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest_gpu.txt
for rep in 1 2 3; do for v in head cur; do for c in mixtral_decode mixtral dsv2_lite dsv2; do
  L=""; [ $v = head ] && L="EPSMOE_LIB=$PWD/tools/ab/lib_head.so"
  env $L timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
done; done; done
