# compute-sanitizer memcheck / racecheck / synccheck over small GPU cases
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
      -k "layer_parity_grid and tiny or grouped_gemm_swiglu_and_down and 300 or router_gemm_exact and 128 or fig_eps or empty_and_single" \
      > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_ep.py -q -x -p no:cacheprovider -k "p2p_put_all2all and 2-2-1-False-False and 1 or local_reduce_ep1" \
  > gpurun_out/san/memcheck_ep.txt 2>&1
echo "memcheck_ep rc=$?" >> gpurun_out/san/summary.txt
