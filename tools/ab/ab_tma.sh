set -x
python -m pytest tests -m gpu -x -q -k "gemm or parity or ep or fullsize" 2>&1 | tail -8 > gpurun_out/ab_pytest.log
for v in 0 1 0 1; do
  echo "TMA_STORE=$v" >> gpurun_out/ab_gemm.log
  EPSMOE_TMA_STORE=$v python tools/gemm_bench.py --config dsv2 >> gpurun_out/ab_gemm.log 2>&1
  EPSMOE_TMA_STORE=$v python tools/gemm_bench.py --config mixtral >> gpurun_out/ab_gemm.log 2>&1
done
for v in 0 1; do
  EPSMOE_TMA_STORE=$v python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_bench_$v.json 2>gpurun_out/ab_bench_$v.err
done
