# Tickets published one tile ahead: parity, Down vs CUTLASS in isolation, layer A/B (EPSMOE_TICKET_AHEAD 0 / 1).
set -x
O=gpurun_out/${1:-r02v}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3 > $O/pytest.txt
for rep in 1 2; do for v in 0 1; do for c in dsv2 dsv2_lite; do
  EPSMOE_TICKET_AHEAD=$v timeout 300 python tools/down_ab_cutlass.py --config $c --rounds 12 2>>$O/err.txt | sed "s/^/ahead=$v /" >> $O/down.txt
done; done; done
for rep in 1 2 3; do for v in 0 1; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_TICKET_AHEAD=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/ahead=$v /" >> $O/ab.txt
done; done; done
