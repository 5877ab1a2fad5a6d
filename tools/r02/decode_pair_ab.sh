# Weight-streaming launches take CTA pairs when their last wave is the emptier one: GPU suite, A/B vs HEAD.
set -x
O=gpurun_out/${1:-r02n}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest_gpu.txt
for rep in 1 2 3; do for v in head cur; do for c in mixtral_decode dsv2_decode; do
  L=""; [ $v = head ] && L="EPSMOE_LIB=$PWD/tools/ab/lib_head.so"
  env $L timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
done; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config mixtral_decode --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/launches_mixtral_decode.csv 2>/dev/null
