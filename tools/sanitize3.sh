# compute-sanitizer over this round's later paths: GEMM half tiles (M = 128 2-CTA MMA, 64-row boxes),
# the copy-engine all2all plane, the comm-only measurement mode
mkdir -p gpurun_out/san3; : > gpurun_out/san3/summary.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "tile_shape or grouped_gemm_swiglu_and_down and 256 or layer_parity_grid and e160" \
  > gpurun_out/san3/memcheck_half_tiles.txt 2>&1
echo "memcheck_half_tiles rc=$?" >> gpurun_out/san3/summary.txt
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tile_shape" \
  > gpurun_out/san3/synccheck_half_tiles.txt 2>&1
echo "synccheck_half_tiles rc=$?" >> gpurun_out/san3/summary.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_ep.py -q -x -p no:cacheprovider \
    -k "p2p_put_all2all and 2-2-1-False-False and 1-2 or comm_only or ranks_with_no_tokens and 2" \
  > gpurun_out/san3/memcheck_ce_comm_only.txt 2>&1
echo "memcheck_ce_comm_only rc=$?" >> gpurun_out/san3/summary.txt
