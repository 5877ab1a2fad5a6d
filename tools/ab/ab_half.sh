# Half tiles: a group's last m-tile with <= 128 rows as an M = 128 2-CTA MMA (EPSMOE_HALF_TILES=1) vs M = 256
O=gpurun_out/ab_half; mkdir -p $O; : > $O/gemm.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -25 > $O/pytest.txt
for r in 1 2 3; do for cfg in dsv2 dsv2_lite mixtral; do for v in 0 1; do
  echo "[EPSMOE_HALF_TILES=$v]" >> $O/gemm.txt
  EPSMOE_HALF_TILES=$v timeout 120 python tools/gemm_bench.py --config $cfg --reps 20 >> $O/gemm.txt 2>&1
done; done; done
