# Split-K router (R19): GPU suite, then A/B against EPSMOE_ROUTER_KSPLIT=1 (the unsplit router,
# same library) on the decode and prefill lines, interleaved, plus ncu router / gate times.
set -x
O=gpurun_out/${1:-r02l}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest_gpu.txt
for rep in 1 2 3; do for v in ks1 cur; do for c in dsv2_decode mixtral_decode dsv2 mixtral; do
  E=""; [ $v = ks1 ] && E="EPSMOE_ROUTER_KSPLIT=1"
  env $E timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
done; done; done
for v in ks1 cur; do
  E=""; [ $v = ks1 ] && E="EPSMOE_ROUTER_KSPLIT=1"
  for c in dsv2_decode dsv2; do
    env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel<2|gate_topk" --csv \
      python bench.py --config $c --graph off --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_${c}_$v.csv 2>/dev/null
  done
done
