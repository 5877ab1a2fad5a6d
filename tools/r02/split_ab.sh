# Column-split permute / combine for small batches: GPU suite (parity, stage-wise, EP), decode bench A/B vs HEAD.
set -x
O=gpurun_out/${1:-r02y}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest_gpu.txt
for rep in 1 2 3; do for v in head cur; do for c in dsv2_decode mixtral_decode; do
  L=""; [ $v = head ] && L="EPSMOE_LIB=$PWD/tools/ab/lib_head.so"
  env $L timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
done; done; done
M=gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none -c 40 --csv python bench.py --config dsv2_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_decode_cur.csv 2>/dev/null
EPSMOE_LIB=$PWD/tools/ab/lib_head.so timeout 300 ncu --metrics $M --clock-control none -c 40 --csv python bench.py --config dsv2_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_decode_head.csv 2>/dev/null
