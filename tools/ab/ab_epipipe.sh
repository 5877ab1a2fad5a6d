# DownGemm epilogue: pipelined TMEM loads + two staging buffers (EPSMOE_EPI_PIPE=1) vs one buffer (0)
O=gpurun_out/ab_epipipe; mkdir -p $O; : > $O/gemm.txt
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > $O/pytest_parity.txt
for r in 1 2 3; do
for cfg in dsv2 mixtral dsv2_lite; do
for env in "EPSMOE_EPI_PIPE=0" "EPSMOE_EPI_PIPE=1" "EPSMOE_GEMM_DIAG=1"; do
  echo "[$env]" >> $O/gemm.txt
  env $env python tools/gemm_bench.py --config $cfg --reps 10 >> $O/gemm.txt 2>&1
done; done; done
for r in 1 2; do
for env in "EPSMOE_EPI_PIPE=0" "EPSMOE_EPI_PIPE=1"; do
  echo "[$env]" >> $O/bench.txt
  env $env python bench.py --steps 30 --no-cpu-baseline --e2e-steps 1 >> $O/bench.txt 2>&1
done; done
