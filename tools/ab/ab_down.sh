# Down-GEMM knobs on dsv2 shapes (tools/gemm_bench.py)
mkdir -p gpurun_out; : > gpurun_out/ab_down.txt
for r in 1 2; do
for env in "" "EPSMOE_RASTER_GM=1" "EPSMOE_RASTER_GM=2" "EPSMOE_RASTER_GM=8" "EPSMOE_DYN_SCHED=0" "EPSMOE_TMA_STORE=0" "EPSMOE_GEMM_DIAG=1" "EPSMOE_GEMM_DIAG=2"; do
  echo "[$env]" >> gpurun_out/ab_down.txt
  env $env python tools/gemm_bench.py --config dsv2 --reps 10 >> gpurun_out/ab_down.txt 2>&1
done
echo "[tile128]" >> gpurun_out/ab_down.txt
python tools/gemm_bench.py --config dsv2 --reps 10 --tile-m 128 >> gpurun_out/ab_down.txt 2>&1
done
