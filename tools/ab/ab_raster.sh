mkdir -p gpurun_out; : > gpurun_out/ab_raster.txt
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab_raster.txt
for r in 1 2; do for cfg in mixtral dsv2 dsv2_lite; do
  python bench.py --config $cfg --no-cpu-baseline --steps 20 --e2e-steps 2 > gpurun_out/ab_r.json 2>>gpurun_out/ab_r.err
  python - $cfg >> gpurun_out/ab_raster.txt <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_r.json"))
print(sys.argv[1], "layer", round(d["ms_per_step"], 3), {k: d["stages_ms"][k] for k in ("gateup", "down", "shared")}, d["clocks"]["sm_mhz"])
PY
done; done
