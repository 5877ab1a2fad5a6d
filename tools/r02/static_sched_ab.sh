# Static round-robin tile scheduling (cursor decode) for the DownGemm / all GEMMs vs dynamic tickets:
# parity suite with every GEMM static, then bench A/B (EPSMOE_DYN_SCHED = 1 dynamic, 2 Down static, 0 all static).
set -x
O=gpurun_out/${1:-r02u}
mkdir -p $O
EPSMOE_DYN_SCHED=0 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3 > $O/pytest_static.txt
for rep in 1 2 3; do for v in 1 2 0; do for c in dsv2 dsv2_lite mixtral; do
  EPSMOE_DYN_SCHED=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | sed "s/^/dyn=$v /" >> $O/ab.txt
done; done; done
