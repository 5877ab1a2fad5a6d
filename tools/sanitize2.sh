# memcheck over the feature paths: FP8 dispatch, LocalReduce (EP 2), token slices, device-limited routing,
# fused DownGemm+combine scatter, EPI_COMBINE / gather options
mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_ep.py -q -x -p no:cacheprovider \
    -k "fp8_dispatch_ep_equals_ep1_and_oracle and 2-2 or local_reduce_ep_vs_oracle and 2-1 or token_sliced and 4-2-4 or p2p_put_all2all and 2-2-1-False-True or device_limited" \
  > gpurun_out/san/memcheck_features.txt 2>&1
echo "memcheck_features rc=$?" >> gpurun_out/san/summary2.txt
EPSMOE_FUSE_COMBINE=1 EPSMOE_GATHER=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "layer_parity_grid and mid_shared" \
  > gpurun_out/san/memcheck_options.txt 2>&1
echo "memcheck_options rc=$?" >> gpurun_out/san/summary2.txt
