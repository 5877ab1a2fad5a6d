# The first async host call after a sync takes the standalone call's token slicing: host-path tests, e2e A/B vs HEAD.
set -x
O=gpurun_out/${1:-r02fc}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py -m gpu -q -x -k "forward_host" 2>&1 | tail -3 > $O/pytest.txt
for rep in 1 2 3; do for v in head cur; do for c in dsv2 mixtral dsv2_lite mixtral_decode; do
  L=""; [ $v = head ] && L="EPSMOE_LIB=$PWD/tools/ab/lib_head.so"
  env $L timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
done; done; done
