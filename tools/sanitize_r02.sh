# Round-2 compute-sanitizer pass over the kernels changed this round: decoded tile tickets (GEMMs),
# NaN-safe gate (R18), column-split permute / combine for few rows, tile-count grids for dense GEMMs,
# shared experts beside the router; plus the EP put plane.  Small cases only (sanitizers are slow).
O=gpurun_out/san_r02
mkdir -p $O
: > $O/summary.txt
SEL="layer_parity_grid or empty_and_single or grouped_gemm_swiglu_and_down and counts0 or router_exact_on_grid_large_h_with_bias and 1088 or fused_shared_down and 700"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_stagewise.py -q -x -p no:cacheprovider \
      -k "$SEL or nan_token or dense_chunks_with_fused" > $O/$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_ep.py -q -x -p no:cacheprovider -k "p2p_put_all2all and 2-2-1-False-False and 1 or local_reduce_ep1" \
  > $O/memcheck_ep.txt 2>&1
echo "memcheck_ep rc=$?" >> $O/summary.txt
